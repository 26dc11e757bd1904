"""CSR-input training (som_train_online_csr) against the
dense oracle.

The sparse distance path computes the same real number as the definition
(R25), so the bar is the training bar of BASELINE.json north_star: the BMU
log identical to the dense oracle's, weights within 1e-4 (in practice bit
for bit: the update is the same Eq. 1 arithmetic)."""
import math

import numpy as np
import pytest

import oracle
from synth import bank_corpus, init_rows

pytestmark = pytest.mark.gpu

W_TOL = 1e-4
W_GLOBAL = 2


@pytest.fixture(scope="module")
def som():
    from paper_1905_09598_b200 import som as s
    s.lib()
    return s


def _train_csr(som, rows, cols, topo, C, W0, epochs, alpha0, sigma0, seed, mode=W_GLOBAL, grid=0, cutoff=1e-4,
               t_ranges=None):
    T = epochs * C.n
    with som.SOM(rows, cols, C.d, topo) as m:
        som.som_set_train_mode(m.h, mode)
        som.som_set_train_grid(m.h, grid)
        m.set_weights(W0)
        logs = []
        for tb, te in (t_ranges or [(0, T)]):
            log = np.full(te - tb, -7, np.int32)
            m.train_online_csr(C.indptr, C.indices, C.data, C.n, epochs, alpha0=alpha0, sigma0=sigma0, seed=seed,
                               cutoff=cutoff, t_begin=tb, t_end=te, bmu_log=log)
            logs.append(log)
        _, kernel = som.som_last_train_config(m.h)
        W = m.get_weights()
    return W, np.concatenate(logs), kernel


def _check(W, log, Wo, logo):
    bad = np.flatnonzero(log != logo)
    assert bad.size == 0, f"first BMU mismatch at step {bad[0]} of {log.size}"
    err = np.abs(W.astype(np.float64) - Wo).max()
    assert err <= W_TOL, err
    assert np.count_nonzero(W != Wo) <= W.size // 1000   # normally bit for bit


@pytest.mark.parametrize("rows,cols,topo,n,d,epochs,sigma0,grid", [
    (12, 15, 1, 1500, 3000, 4, 3.0, 0),      # hex, sigma shrinks from partial to 1: both paths each step
    (9, 11, 0, 800, 2000, 6, 6.0, 13),       # rect, ragged: 99 units over 13 CTAs
    (20, 20, 1, 1000, 4096, 3, 10.0, 0),     # c2-like map, full -> partial neighbourhood
    (5, 7, 1, 300, 12000, 4, 2.0, 5),        # wide rows: 6 float4 chunks per thread (no x cache)
])
def test_csr_training_matches_dense_oracle(som, rows, cols, topo, n, d, epochs, sigma0, grid):
    C = bank_corpus(n, d, seed=n + d)
    X = C.dense()
    W0 = init_rows(X, rows * cols, 17)
    W, log, kernel = _train_csr(som, rows, cols, topo, C, W0, epochs, 0.1, sigma0, 5, grid=grid)
    assert kernel == 4, kernel
    Wo, logo = oracle.train_online(W0, rows, cols, topo, X, epochs, 0.1, sigma0, 5)
    _check(W, log, Wo, logo)


def test_csr_training_resume_and_empty_rows(som):
    """Documents with no terms (D_u = |w_u|^2) and a t-range split into three
    calls reproduce the single dense oracle run."""
    C = bank_corpus(600, 2500, seed=8)
    # empty every 7th row
    keep = np.ones(C.nnz, bool)
    rows_ = np.repeat(np.arange(C.n), np.diff(C.indptr))
    keep[np.isin(rows_, np.arange(0, C.n, 7))] = False
    indptr = np.zeros(C.n + 1, np.int64)
    np.cumsum(np.bincount(rows_[keep], minlength=C.n), out=indptr[1:])
    C.indptr, C.indices, C.data = indptr, C.indices[keep].copy(), C.data[keep].copy()
    X = C.dense()
    assert (np.abs(X).sum(1) == 0).sum() >= C.n // 7
    W0 = init_rows(X, 80, 3) + np.float32(0.01)
    T = 5 * C.n
    W, log, kernel = _train_csr(som, 8, 10, 1, C, W0, 5, 0.2, 4.0, 11,
                                t_ranges=[(0, 1000), (1000, 1001), (1001, T)])
    assert kernel == 4
    Wo, logo = oracle.train_online(W0, 8, 10, 1, X, 5, 0.2, 4.0, 11)
    _check(W, log, Wo, logo)


def test_csr_training_no_cutoff_and_auto(som):
    """cutoff 0 (every unit adapts: the dense path every step) and AUTO mode
    on a small map (register kernel on the densified rows)."""
    C = bank_corpus(400, 1000, seed=9)
    X = C.dense()
    W0 = init_rows(X, 48, 4)
    W, log, kernel = _train_csr(som, 6, 8, 1, C, W0, 3, 0.1, 3.0, 2, cutoff=0.0)
    assert kernel == 4
    Wo, logo = oracle.train_online(W0, 6, 8, 1, X, 3, 0.1, 3.0, 2, eps=0.0)
    _check(W, log, Wo, logo)
    W, log, kernel = _train_csr(som, 6, 8, 1, C, W0, 3, 0.1, 3.0, 2, mode=0)
    assert kernel in (1, 2), kernel
    Wo, logo = oracle.train_online(W0, 6, 8, 1, X, 3, 0.1, 3.0, 2)
    _check(W, log, Wo, logo)


def test_csr_training_equals_dense_training_c3_prefix(som):
    """c3 shape (50x50 hex, 10k terms), first 3,000 steps: the sparse kernel
    and the dense global-W kernel give the same BMU log and weights, and
    both match the oracle."""
    C = bank_corpus(5000, 10000, seed=31)
    X = C.dense()
    W0 = init_rows(X, 2500, 1031)
    steps = 3000
    W, log, kernel = _train_csr(som, 50, 50, 1, C, W0, 100, 0.1, 25.0, 1, t_ranges=[(0, steps)])
    assert kernel == 4
    Wo, logo = oracle.train_online(W0, 50, 50, 1, X, 100, 0.1, 25.0, 1, t_begin=0, t_end=steps)
    _check(W, log, Wo, logo)


def test_csr_training_late_schedule(som):
    """Late in the schedule (sigma near its floor) almost every unit takes the
    sparse path: steps [T - 4000, T) from a mid-training codebook."""
    C = bank_corpus(2000, 6000, seed=12)
    X = C.dense()
    W0 = init_rows(X, 900, 7)
    T = 20 * C.n
    Wm, _ = oracle.train_online(W0, 30, 30, 1, X, 20, 0.1, 15.0, 4, t_begin=0, t_end=200)
    W, log, kernel = _train_csr(som, 30, 30, 1, C, Wm, 20, 0.1, 15.0, 4, t_ranges=[(T - 4000, T)])
    assert kernel == 4
    Wo, logo = oracle.train_online(Wm, 30, 30, 1, X, 20, 0.1, 15.0, 4, t_begin=T - 4000, t_end=T)
    _check(W, log, Wo, logo)


@pytest.mark.parametrize("defect", ["unsorted", "range", "rowptr"])
def test_csr_validation(som, defect):
    C = bank_corpus(50, 200, seed=3)
    indptr, col, val = C.indptr.copy(), C.indices.copy(), C.data.copy()
    if defect == "unsorted":
        p0 = indptr[4]
        col[p0], col[p0 + 1] = col[p0 + 1], col[p0]
    elif defect == "range":
        col[-1] = 200
    else:
        indptr[10] = indptr[11] + 1
    W0 = init_rows(C.dense(), 12, 1)
    with som.SOM(3, 4, 200, 1) as m:
        m.set_weights(W0)
        with pytest.raises(som.SomError):
            m.train_online_csr(indptr, col, val, C.n, 2)
        b1 = np.empty(C.n, np.int32)
        with pytest.raises(som.SomError):
            som.som_map_csr(m.h, indptr, col, val, C.n, b1)
        assert np.array_equal(m.get_weights(), W0)


@pytest.mark.parametrize("cover,expect", [("0.6", 12), ("0", 4), ("1.01", 4)])
def test_dense_then_sparse_kernel12(som, monkeypatch, cover, expect):
    """AUTO with rows too long for kernel 4's TMA ring (d = 13,000: 7 float4
    per thread): the dense pipelined kernel 3 while the cutoff disk holds >=
    SOM_DENSE_COVER of the units on average, then kernel 4 (kernel id 12,
    two launches; the CSR rows densified on the device), against the oracle
    over the whole schedule; SOM_DENSE_COVER=0 / > 1 keep kernel 4
    throughout."""
    monkeypatch.setenv("SOM_DENSE_COVER", cover)
    C = bank_corpus(200, 13000, seed=213)
    X = C.dense()
    W0 = init_rows(X, 12 * 12, 213)
    W, log, kernel = _train_csr(som, 12, 12, 1, C, W0, 2, 0.1, 6.0, 9, mode=0, grid=16)
    assert kernel == expect, kernel
    Wo, logo = oracle.train_online(W0, 12, 12, 1, X, 2, 0.1, 6.0, 9)
    _check(W, log, Wo, logo)
