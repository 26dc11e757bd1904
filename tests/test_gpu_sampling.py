"""Per-epoch permutation sampling (R8b: the option beside P:162's
uniform random selection, R8) through every training kernel family, against
the oracle running the same counter-based permutation: BMU log identical,
weights within 1e-4 (observed bit-identical).  Resume across a t-range
split, zero rows (the permutation runs over the non-zero rows), and the
argument check."""
import numpy as np
import pytest

import oracle
from synth import bank_corpus, init_rows

pytestmark = pytest.mark.gpu
PERMUTE = 1


@pytest.fixture(scope="module")
def som():
    from paper_1905_09598_b200 import som as s
    s.lib()
    return s


@pytest.mark.parametrize("rows,cols,n,d,mode,csr,grid,expect", [
    (10, 10, 200, 500, 3, False, 0, 2),      # W in registers
    (12, 12, 300, 1000, 1, False, 0, 1),     # W in shared memory
    (16, 16, 300, 2048, 2, True, 0, 4),      # CSR, W streamed (kernel 4)
    (20, 20, 400, 6000, 0, True, 16, 10),    # CSR, tiered storage (kernel 10)
    (16, 16, 300, 64, 0, False, 0, 5),       # short rows
])
def test_permutation_sampling_matches_oracle(som, rows, cols, n, d, mode, csr, grid, expect, monkeypatch):
    monkeypatch.setenv("SOM_TIER_HANDOVER", "0")
    C = bank_corpus(n, d, seed=n + d)
    X = C.dense()
    W0 = init_rows(X, rows * cols, 5)
    epochs, sigma0, seed = 3, max(rows, cols) / 2.0, 17
    T = epochs * n
    with som.SOM(rows, cols, d, 1) as m:
        som.som_set_train_mode(m.h, mode)
        if grid:
            som.som_set_train_grid(m.h, grid)
        m.set_weights(W0)
        log = np.full(T, -1, np.int32)
        for a, b in ((0, T // 3 + 7), (T // 3 + 7, T)):
            if csr:
                m.train_online_csr(C.indptr, C.indices, C.data, n, epochs, 0.1, sigma0, seed, t_begin=a, t_end=b,
                                   bmu_log=log[a:b], sampling=PERMUTE)
            else:
                m.train_online(X, epochs, 0.1, sigma0, seed, t_begin=a, t_end=b, bmu_log=log[a:b], sampling=PERMUTE)
        k = som.som_last_train_config(m.h)[1]
        W = m.get_weights()
    assert k == expect, k
    Wo, logo = oracle.train_online(W0, rows, cols, 1, X, epochs, 0.1, sigma0, seed, sampling=PERMUTE)
    assert np.array_equal(log, logo), f"first BMU mismatch at {int(np.argmax(log != logo))}"
    assert np.abs(W.astype(np.float64) - Wo).max() <= 1e-4
    # the draws differ from R8's: the trajectory is not the with-replacement one
    _, log_r8 = oracle.train_online(W0, rows, cols, 1, X, epochs, 0.1, sigma0, seed)
    assert not np.array_equal(log, log_r8)


def test_permutation_sampling_zero_rows_and_bad_mode(som):
    C = bank_corpus(250, 512, seed=71)
    X = C.dense()
    X[::7] = 0.0                               # drawable rows: the non-zero ones
    W0 = init_rows(np.delete(X, np.arange(0, 250, 7), 0), 100, 72)
    with som.SOM(10, 10, 512, 0) as m:
        m.set_weights(W0)
        log = np.empty(2 * 250, np.int32)
        m.train_online(X, 2, 0.1, 5.0, 23, bmu_log=log, sampling=PERMUTE)
        W = m.get_weights()
        with pytest.raises(som.SomError, match="SOM_EINVAL"):
            m.train_online(X, 2, 0.1, 5.0, 23, sampling=2)
    Wo, logo = oracle.train_online(W0, 10, 10, 0, X, 2, 0.1, 5.0, 23, sampling=PERMUTE)
    assert np.array_equal(log, logo)
    assert np.abs(W.astype(np.float64) - Wo).max() <= 1e-4
