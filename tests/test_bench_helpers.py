"""Host-side helpers of bench.py (CPU): the H_t count behind the training
roofline's byte figure, the conversion-peak models, the multi-rank hooks."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import oracle  # noqa: E402


def test_updated_units_matches_oracle_lattice():
    """H_t = #{u : g2(u, c_t) <= r2_t} (R5) recomputed with the oracle's
    lattice distance and schedule."""
    rows, cols, topo, T, sigma0 = 7, 9, 1, 1000, 4.5
    rng = np.random.default_rng(1)
    log = rng.integers(0, rows * cols, size=40).astype(np.int32)
    t0 = 300
    H = bench.updated_units(rows, cols, topo, log, t0, T, sigma0)
    for s, c in enumerate(log):
        _, sigma, rr = oracle.schedule(t0 + s, T, 0.1, sigma0)
        cnt = sum(1 for u in range(rows * cols) if oracle.lattice_g2(rows, cols, topo, u, int(c)) <= rr)
        assert H[s] == cnt


def test_conversion_peak_models():
    cpk, src = bench.conv_peak_per_s()
    assert 3e12 < cpk < 6e12 and "F2F" in src
    tf, src2 = bench.tf32_peak_tflops()
    assert 500 < tf < 1200


def test_one_device_hook(monkeypatch):
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setenv("LOCAL_RANK", "1")
    assert bench.dist_env() == (1, 2, 1)
    monkeypatch.setenv("BENCH_ONE_DEVICE", "1")
    assert bench.dist_env() == (1, 2, 0)
