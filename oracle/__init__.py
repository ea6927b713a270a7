"""oracle -- TEST INFRASTRUCTURE ONLY (the checker, never the product).

Two CPU checkers for the collective-emulation hot path:

* ``oracle.port``  -- ctypes over ``liboracle.so``, the plain-C restatement in
  ``cemu_oracle.c`` (every function cites the reference file:line it follows).
* ``oracle.ref``   -- ctypes over ``_ref/libcemu_ref.so``, the reference's own
  ``cemu_core`` compiled from /root/reference by ``oracle/Makefile`` plus the
  ``ref_shim.cpp`` C-ABI driver.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product package ``paper_2405_02969_b200`` never does.
"""
