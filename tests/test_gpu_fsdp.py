"""GPU: the FSDP trace at 1024 emulated ranks (config 5) reproduces its ideal
timeline within 1% for every cost model, on a Llama-3-8B-shaped slice
(embed, 2 blocks, head), and the full what-if table's ordering holds."""
from __future__ import annotations

import pytest

from paper_2405_02969_b200 import fsdp

pytestmark = pytest.mark.gpu


def test_fsdp_slice_all_cost_models(cuda):
    units = fsdp.llama3_8b_units()
    sl = [units[0], units[1], units[2], units[-1]]
    res = fsdp.whatif_table(1024, iterations=2, units=sl)
    assert res["max_rel_err"] < 0.01, res["rows"]
    t = {(r["algo"], r["inter_bw_x"]): r["iteration_ms"] for r in res["rows"]}
    assert t[("tree", 1.0)] < t[("ring", 1.0)]
    for algo in ("ring", "tree", "hierarchical"):
        assert t[(algo, 2.0)] < t[(algo, 1.0)]
