"""FSDP trace (config 5) host side: Llama-3-8B shapes, the cost-model configs,
and the ideal-timeline calculator on hand-checkable schedules (CPU)."""
from __future__ import annotations

import paper_2405_02969_b200 as pb
from paper_2405_02969_b200 import fsdp
from paper_2405_02969_b200 import schedule as S


def test_llama3_8b_shapes():
    units = fsdp.llama3_8b_units()
    assert len(units) == 34
    total = sum(p for _, p in units)
    assert 8.02e9 < total < 8.04e9  # Llama-3-8B: 8.03 B parameters
    block = dict(units)["block0"]
    assert 218.0e6 < block < 218.2e6
    plan = fsdp.unit_plan(units, 1024)
    assert plan[1]["shard"] * 1024 >= block and plan[1]["bwd_us"] == 2 * plan[1]["fwd_us"]


def test_cost_configs_parse_and_models_order():
    for algo in ("ring", "tree", "hierarchical"):
        for s in (1.0, 2.0):
            cfg = pb.JobConfig.parse(fsdp.cost_config(1024, algo, s))
            assert cfg.world_size == 1024
    # one block's all-gather at 1024 ranks: hierarchical (NVLink carries 7/8) < tree < ring
    shard = fsdp.unit_plan(fsdp.llama3_8b_units(), 1024)[1]["shard"] * 2
    def ag(algo, bw):
        n = fsdp.NET
        m = S.delay_model(S.ALPHA_BETA, {"ring": 0, "tree": 1, "hierarchical": 2}[algo], n["alpha_inter_us"],
                          n["beta_inter_us_per_byte"] / bw, n["gamma_us_per_byte"], 0, 0, n["gpus_per_node"],
                          n["alpha_intra_us"], n["beta_intra_us_per_byte"])
        return S.model_total_us(m, S.ALLGATHER, 1024, shard)
    assert ag("hierarchical", 1) < ag("tree", 1) < ag("ring", 1)
    assert ag("ring", 2) < ag("ring", 1)


def test_ideal_timeline_hand_computed():
    plan = [{"fwd_us": 10, "bwd_us": 20}, {"fwd_us": 10, "bwd_us": 20}]
    # zero-latency network: pure compute
    assert fsdp.ideal_iteration_us(plan, [0, 0], [0, 0]) == 60
    # AG 5 each, RS 7 each:
    # fwd: AG0 0->5, compute0 5-15 (AG1 issued at 5: 5->10), compute1 15-25
    # bwd: AGb1 issued 25 -> 30; compute1b 30-50 (AGb0 issued 30 -> 35); RS1 at 50 -> 57
    #      compute0b 50-70; RS0 at 70 -> 77
    assert fsdp.ideal_iteration_us(plan, [5, 5], [7, 7]) == 77
