"""Short-prototype training kernel (SOM_TRAIN_SHORT_ROWS, train_small.cu)
against the oracle: the map-size study of the paper (Table 3, P:298-309:
weight length 64, square maps) and other d <= 128.

Bar (BASELINE.json north_star): BMU sequence identical, weights within 1e-4
max-abs.  The kernel's neighbourhood is RN32(alpha * (Er * Ec)) from
separable tables (R26), a few fp64 ulp from the oracle's
RN32(alpha * exp(-g2/2sigma^2)), so a weight may differ from the oracle's by
an ulp where h rounds differently; the count is reported and bounded."""
import math

import numpy as np
import pytest

import oracle
from synth import init_rows, uniform_matrix

pytestmark = pytest.mark.gpu

W_TOL = 1e-4
SHORT = 4          # SOM_TRAIN_SHORT_ROWS
KERNEL_SHORT = 5   # som_last_train_config kernel id


@pytest.fixture(scope="module")
def som():
    from paper_1905_09598_b200 import som as s
    s.lib()
    return s


def _run(som, rows, cols, topo, X, W0, epochs, sigma0, seed, t_end=-1, grid=0, mode=SHORT, cutoff=1e-4):
    n, d = X.shape
    T = epochs * n
    te = T if t_end < 0 else t_end
    with som.SOM(rows, cols, d, topo) as m:
        som.som_set_train_mode(m.h, mode)
        if grid:
            som.som_set_train_grid(m.h, grid)
        m.set_weights(W0)
        log = np.full(te, -7, np.int32)
        m.train_online(X, epochs=epochs, alpha0=0.1, sigma0=sigma0, seed=seed, t_end=t_end, bmu_log=log,
                       cutoff=cutoff)
        W = m.get_weights()
        g, k = som.som_last_train_config(m.h)
    Wo, logo = oracle.train_online(W0, rows, cols, topo, X, epochs, 0.1, sigma0, seed, eps=cutoff, t_end=t_end)
    assert k == KERNEL_SHORT
    return W, log, Wo, logo, g


def _check(W, log, Wo, logo, label):
    assert np.array_equal(log, logo), f"{label}: first BMU mismatch at step {np.flatnonzero(log != logo)[:1]}"
    err = np.abs(W.astype(np.float64) - Wo).max()
    assert err <= W_TOL, err
    ndiff = int(np.count_nonzero(W != Wo))
    assert ndiff <= max(8, W.size // 10000), ndiff
    print(f" [{label}: {ndiff} of {W.size} weights differ, max {err:.1e}]", end="")


@pytest.mark.parametrize("side,topo,epochs,t_end", [
    (16, 1, 10, -1),      # Table 3 smallest map, full schedule (T = 20000)
    (16, 0, 10, -1),
    (32, 1, 4, -1),
    (64, 1, 2, 3000),     # several register rounds per thread
    (128, 0, 1, 400),     # 16 rounds at G = 128
    (256, 1, 1, 60),      # 256x256: 4 register rounds per thread at G = 128
])
def test_table3_maps_d64(som, side, topo, epochs, t_end):
    X = uniform_matrix(2000, 64, side)
    W0 = init_rows(X, side * side, side + 1) if side * side <= 2000 else \
        uniform_matrix(side * side, 64, side + 2)
    W, log, Wo, logo, g = _run(som, side, side, topo, X, W0, epochs, side / 2.0, seed=side, t_end=t_end)
    _check(W, log, Wo, logo, f"{side}x{side} d=64 G={g}")


def test_streamed_variant_small_grid(som):
    """Force the global-memory (streamed) variant on a mid-size map by
    limiting the grid: 64x64 units over 4 CTAs = 8 rounds per thread."""
    X = uniform_matrix(1000, 64, 7)
    W0 = uniform_matrix(64 * 64, 64, 8)
    W, log, Wo, logo, g = _run(som, 64, 64, 1, X, W0, 1, 32.0, seed=7, t_end=300, grid=4)
    assert g == 4
    _check(W, log, Wo, logo, "64x64 streamed G=4")


@pytest.mark.parametrize("d", [4, 12, 32, 100, 128])
def test_other_short_dims(som, d):
    """Lane groups of 1, 4, 8, 32 lanes, partly idle lanes (d = 12, 100)."""
    X = uniform_matrix(500, d, d)
    W0 = init_rows(X, 12 * 15, d + 1)
    W, log, Wo, logo, g = _run(som, 12, 15, 1, X, W0, 3, 7.5, seed=d)
    _check(W, log, Wo, logo, f"12x15 d={d}")


def test_no_cutoff_and_rect(som):
    X = uniform_matrix(400, 64, 3)
    W0 = init_rows(X, 20 * 20, 4)
    W, log, Wo, logo, g = _run(som, 20, 20, 0, X, W0, 3, 10.0, seed=3, cutoff=0.0)
    _check(W, log, Wo, logo, "20x20 rect eps=0")


def test_auto_picks_short_rows_and_resume(som):
    """AUTO uses the short-row kernel for d <= 128; a split t-range resumes
    exactly (the pending update is flushed at the end of each call)."""
    X = uniform_matrix(300, 64, 11)
    W0 = init_rows(X, 100, 12)
    with som.SOM(10, 10, 64, 1) as m:
        m.set_weights(W0)
        la = np.empty(900, np.int32)
        m.train_online(X, epochs=3, alpha0=0.1, sigma0=5.0, seed=4, bmu_log=la)
        _, k = som.som_last_train_config(m.h)
        Wa = m.get_weights()
        m.set_weights(W0)
        lb1 = np.empty(333, np.int32)
        lb2 = np.empty(900 - 333, np.int32)
        m.train_online(X, epochs=3, alpha0=0.1, sigma0=5.0, seed=4, t_end=333, bmu_log=lb1)
        m.train_online(X, epochs=3, alpha0=0.1, sigma0=5.0, seed=4, t_begin=333, bmu_log=lb2)
        Wb = m.get_weights()
    assert k == KERNEL_SHORT
    assert np.array_equal(Wa, Wb) and np.array_equal(la, np.concatenate([lb1, lb2]))
