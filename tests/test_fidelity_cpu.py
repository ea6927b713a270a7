"""CPU: the calibration side of the emulated-vs-baseline fidelity check
(paper_2405_02969_b200/fidelity.py) -- the alpha-beta fit and the latency
table the delay-model plugin interpolates."""
from __future__ import annotations

import math

import pytest

from paper_2405_02969_b200 import fidelity as F


@pytest.mark.parametrize("k", [2, 4, 8])
def test_alpha_beta_fit_recovers_an_affine_ring(k):
    alpha, beta = 3.5, 2.0e-6
    sizes = [4096 << i for i in range(14)]
    us = [2 * (k - 1) * alpha + 2 * (k - 1) / k * m * beta for m in sizes]
    fit = F.fit_alpha_beta(sizes, us, k)
    assert fit["alpha_us"] == pytest.approx(alpha, rel=1e-9)
    assert fit["beta_us_per_byte"] == pytest.approx(beta, rel=1e-9)
    cfg = F.ab_config(k, fit)  # a config the library parses: plain floats, no numpy reprs
    assert "np." not in cfg and f"world_size = {k}" in cfg


def test_table_plugin_hits_the_measured_points_and_interpolates_log_log():
    sizes, us = [4096, 65536, 1 << 20, 16 << 20], [10.0, 12.0, 20.0, 80.0]
    p = F.table_plugin(sizes, us)
    for s, u in zip(sizes, us):
        assert p.at(s) == pytest.approx(u)
    mid = p.at(math.sqrt(65536 * (1 << 20)))   # geometric midpoint -> geometric mean
    assert mid == pytest.approx(math.sqrt(12.0 * 20.0))
    assert p.at(64 << 20) == pytest.approx(80.0 * 4 ** (math.log(80 / 20) / math.log(16)))  # end slope
    offs = p(0, 4, 1 << 20, 6)  # K release offsets, evenly spread, the last = the call's latency
    assert offs[-1] == pytest.approx(20.0) and offs == sorted(offs) and len(offs) == 6


def test_size_plugin_from_service_samples():
    p, table = F.size_plugin([(1 << 20, 10.0), (1 << 20, 14.0), (4 << 20, 30.0)])
    assert table == {1 << 20: 12.0, 4 << 20: 30.0}
    assert p.at(1 << 20) == pytest.approx(12.0)
    p1, t1 = F.size_plugin([(32 << 20, 100.0), (32 << 20, 110.0)])  # one bucket size: constant
    assert p1.at(32 << 20) == pytest.approx(105.0) and p1.at(16 << 20) == pytest.approx(105.0)
