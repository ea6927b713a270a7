"""Wire-format interop: a B200 communicator in wire mode
against the reference's own emulator.

The reference EmulatorServer (proj/src/emulator.cpp, compiled from the
reference sources into oracle/_ref) serves in a thread of this process; the
B200 communicator dials it, handshakes (HELLO/TOPO with the config digest and
plan) and runs its collectives over the CEMU frame protocol with the buffer
on the GPU.  Checked:

* results bit-equal to the reference's own WorkerSession against the same
  emulator (oracle/_ref), to the oracle's zero-payload restatement and to
  this library's device zero-payload mode;
* the reference engine releases every to-real step no earlier than the
  device model's floor for it, in order (the call record holds both);
* plan and digest mismatches fail loudly with the reference's wording.
"""
from __future__ import annotations

import socket
import time

import numpy as np
import pytest
import torch

import paper_2405_02969_b200 as pb
from gpu_util import assert_bit_equal, host_input, to_np
from oracle import port as P
from oracle import ref as R

pytestmark = pytest.mark.gpu

if not R.available():
    pytest.skip("oracle/_ref not built", allow_module_level=True)


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def wire_config(W: int, alpha=500.0, beta=0.0001, gamma=0.0, kind="alpha_beta") -> str:
    p0, pe = _port(), _port()
    lines = [f"world_size = {W}", "real_ranks = 0", "bucket_bytes = 65536", f"delay.kind = {kind}",
             f"link.alpha_us = {alpha}", f"link.beta_us_per_byte = {beta}", f"link.gamma_us_per_byte = {gamma}",
             "delay.fixed_us = 0", "delay.inject_us = 0", f"endpoint.0 = 127.0.0.1:{p0}"]
    lines += [f"endpoint.{r} = 127.0.0.1:{pe}" for r in range(1, W)]
    return "\n".join(lines) + "\n"


def start_emulator(W: int, **kw):
    """A reference emulator on fresh ports: the ports come from bind(0) and
    are released before the emulator binds them, so another socket can take
    one in between (a long test session); retry with new ones."""
    last = None
    for _ in range(5):
        text = wire_config(W, **kw)
        try:
            return text, R.Emulator(text)
        except R.RefError as e:
            last = e
    raise last


def test_digests_agree_with_the_reference_parser(cuda):
    text = wire_config(8)
    assert pb.JobConfig.parse(text).digest == R.config_digest(text)


@pytest.mark.parametrize("W", [2, 4, 8])
def test_wire_allreduce_and_allgather_equal_the_reference_worker(cuda, W):
    count, sc = 4096 + 4 * W, 1000
    plan = [pb.CollectivePlanEntry("allreduce", count * 4, 4), pb.CollectivePlanEntry("allgather", sc, 1)]
    text, emu = start_emulator(W, alpha=50.0)
    with emu:
        comm = pb.Communicator(text, 0, 0)
        comm.attach_emulator(plan)
        for it in range(2):  # op ids 0..3 over the two plan entries
            h = host_input(2, count, seed=W + it)
            x = h.cuda()
            comm.all_reduce(x, x)
            got = to_np(x)
            ref = to_np(h).copy()
            R.emulated_collective(W, 0, ref.view(np.uint8), count * 4, 4)  # the reference worker, fresh emulator
            assert_bit_equal(got, ref, f"wire allreduce W={W} it={it}")
            want = P.allreduce(2, P.PAYLOAD_ZERO, W, [0], 0, 1, [to_np(h)], count)
            assert_bit_equal(got, want, "vs oracle zero payload")

            own = host_input(1, sc, seed=it)
            full = torch.zeros(sc * W, dtype=torch.uint8, device="cuda")
            comm.all_gather(own.cuda(), full)
            ref = np.zeros(sc * W, dtype=np.uint8)
            ref[:sc] = to_np(own)
            R.emulated_collective(W, 1, ref, sc, 1)
            assert_bit_equal(to_np(full), ref, f"wire allgather W={W} it={it}")
        comm.close()  # BYE
        # the emulator counts a session when its handler returns, just after the BYE
        deadline = time.time() + 5
        while emu.sessions < 1 and time.time() < deadline:
            time.sleep(0.01)
        assert emu.sessions >= 1


def test_wire_float_buffer_folds_as_int32_lanes_like_the_reference(cuda):
    """collective.cpp:343-350: elem_size 4 sums int32 bit patterns; with the
    emulator's zero payload the result equals the device zero mode (-0.0
    kept, not turned into +0.0 by a float add)."""
    W = 4
    h = host_input(7, 8192, seed=3)
    h[::7] = -0.0
    text, emu = start_emulator(W, alpha=20.0)
    with emu:
        comm = pb.Communicator(text, 0, 0)
        comm.attach_emulator([pb.CollectivePlanEntry("allreduce", h.numel() * 4, 4)])
        y = torch.empty(h.numel(), device="cuda")
        comm.all_reduce(h.cuda(), y)  # out of place
        comm.close()
    zero = pb.Communicator(f"world_size = {W}\nreal_ranks = 0\nbucket_bytes = 1\npayload.mode = zero\n", 0, 0)
    z = torch.empty_like(y)
    zero.all_reduce(h.cuda(), z)
    torch.cuda.synchronize()
    zero.close()
    assert_bit_equal(to_np(y), to_np(z), "wire fp32 vs device zero mode")


def test_reference_engine_releases_no_earlier_than_the_device_floors(cuda):
    W = 4
    text, emu = start_emulator(W, alpha=3000.0, beta=0.001, gamma=0.0001)  # floors of several ms per step
    nbytes = 1 << 16
    with emu:
        comm = pb.Communicator(text, 0, 0)
        comm.attach_emulator([pb.CollectivePlanEntry("allreduce", nbytes, 4)])
        x = torch.zeros(nbytes // 4, dtype=torch.int32, device="cuda")
        comm.all_reduce(x, x)
        rec = comm.call_record()
        log = comm.event_log(rec["call_id"])
        comm.close()
    K = rec["steps"]
    assert K == 2 * (W - 1)
    floors = np.array(rec["floors_us"])
    want_floors = P.release_floors(P.delay_model(1, 0, 3000.0, 0.001, 0.0001, 0.0, 0.0, 1, 0.0, 0.0),
                                   0, W, nbytes, K, 0)
    assert floors.tolist() == list(want_floors)
    rel_us = (np.array(rec["release_ns"]) - rec["t_start_ns"]) / 1e3
    assert np.all(np.diff(rel_us) >= 0), rel_us  # in order
    assert np.all(rel_us >= floors - 1.0), (rel_us, floors)  # never early (1 us clock tolerance)
    late = rel_us - floors
    assert np.all(late < 50_000), late  # the reference's CPU poller overshoot is ~1 ms
    assert rec["model_latency_us"] == int(floors.max())
    sends = [l.split() for l in log if " to_real " in l]
    assert [int(f[4]) for f in sends] == list(range(K))  # step order, reference EventLog format


def test_wire_mode_errors_are_loud(cuda):
    W = 4
    text, emu = start_emulator(W)
    with emu:
        comm = pb.Communicator(text, 0, 0)
        comm.attach_emulator([pb.CollectivePlanEntry("allreduce", 64, 4)])
        x = torch.zeros(16, dtype=torch.int32, device="cuda")
        with pytest.raises(pb.CemuError, match="does not match the declared plan"):
            comm.all_gather(x[:4], x)
        with pytest.raises(pb.CemuError, match=r"buffer size 32 does not match plan entry \(64\)"):
            comm.all_reduce(x[:8], x[:8])
        with pytest.raises(pb.CemuError, match="allreduce and allgather only"):
            comm.reduce_scatter(x, x[:4])
        comm.close()
        # a config that differs from the emulator's: digest rejected by the peer
        other = text.replace("link.alpha_us = 500.0", "link.alpha_us = 501.0")
        assert other != text
        c2 = pb.Communicator(other, 0, 0)
        with pytest.raises(pb.CemuError, match="config digest mismatch"):
            c2.attach_emulator([pb.CollectivePlanEntry("allreduce", 64, 4)])
        c2.close()


# ---- failure paths, against a scripted fake emulator ------------------------
import json as _json
import struct
import threading
import time


def _frame(t, op=0, seq=0, src=0, dst=0, chunk=0, payload=b""):
    return struct.pack("<4sBBIIHHHI", b"CEMU", 1, t, op, seq, src, dst, chunk, len(payload)) + payload


def _read_frame(conn):
    def exact(n):
        b = b""
        while len(b) < n:
            c = conn.recv(n - len(b))
            if not c:
                raise EOFError
            b += c
        return b
    h = exact(24)
    magic, ver, t, op, seq, src, dst, chunk, n = struct.unpack("<4sBBIIHHHI", h)
    return t, op, seq, src, dst, chunk, exact(n) if n else b""


class FakeEmulator:
    """Accepts one session, answers the handshake, then follows `script`:
    "silent" (never answers), "error" (ERROR on OPEN_OP), "bad_chunk"
    (DATA for the wrong chunk)."""

    def __init__(self, text: str, script: str):
        pe = int(text.split("endpoint.1 = 127.0.0.1:")[1].split()[0])
        self.digest = pb.JobConfig.parse(text).digest
        self.world = pb.JobConfig.parse(text).world_size
        self.script = script
        self.sock = socket.socket()
        self.sock.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
        self.sock.bind(("127.0.0.1", pe))
        self.sock.listen(1)
        self.th = threading.Thread(target=self._serve, daemon=True)
        self.th.start()

    def _serve(self):
        conn, _ = self.sock.accept()
        self.conn = conn
        t, *_ , payload = _read_frame(conn)
        assert t == 1  # HELLO
        hello = _json.loads(payload)
        topo = _json.dumps({"rank": -1, "world_size": self.world, "config_digest": self.digest,
                            "plan": hello["plan"]}).encode()
        conn.sendall(_frame(2, payload=topo))
        try:
            t, op, seq, *_ = _read_frame(conn)  # OPEN_OP
            if self.script == "error":
                conn.sendall(_frame(5, payload=b"injected failure"))
            elif self.script == "bad_chunk":
                _read_frame(conn)  # the worker's DATA for position 0
                conn.sendall(_frame(4, op=op, seq=0, src=self.world - 1, dst=0, chunk=99, payload=b"\0" * 16))
            while True:  # "silent": swallow everything, answer nothing
                _read_frame(conn)
        except (EOFError, OSError):
            pass

    def close(self):
        try:
            self.conn.close()
        except Exception:
            pass
        self.sock.close()


@pytest.mark.parametrize("script,match", [("error", "peer reported error: injected failure"),
                                          ("bad_chunk", "protocol mismatch")])
def test_wire_peer_errors_surface(cuda, script, match):
    W = 4
    text = wire_config(W)
    fake = FakeEmulator(text, script)
    comm = pb.Communicator(text, 0, 0)
    comm.attach_emulator([pb.CollectivePlanEntry("allreduce", 64, 4)])
    x = torch.zeros(16, dtype=torch.int32, device="cuda")
    with pytest.raises(pb.CemuError, match=match):
        comm.all_reduce(x, x)
    with pytest.raises(pb.CemuError):  # the session stays failed, as the reference's does
        comm.all_reduce(x, x)
    comm.close()
    fake.close()


def test_wire_detach_from_a_silent_emulator_is_bounded(cuda):
    W = 4
    text = wire_config(W)
    fake = FakeEmulator(text, "silent")
    comm = pb.Communicator(text, 0, 0)
    comm.attach_emulator([pb.CollectivePlanEntry("allreduce", 64, 4)])
    t0 = time.perf_counter()
    comm.detach_emulator()  # BYE goes out, no BYE comes back
    assert time.perf_counter() - t0 < 10
    comm.close()
    fake.close()
