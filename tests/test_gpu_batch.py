"""Batch SOM (som_train_batch / _csr, batch.cu, R27) against the
oracle's batch map (or_train_batch: sums over documents in index order,
straight from the definition).

Bar (BASELINE.json north_star): weights within 1e-4 max-abs, BMUs of the
final map identical.  The kernel regroups sum_i h(c_i,u) x_i as
sum_c h(c,u) S_c and takes h from separable tables (R26): both are exact in
real arithmetic and a few fp64 ulp apart, far below the fp32 rounding of W,
so the weights normally agree bit for bit; the count of differing weights
is reported and bounded."""
import numpy as np
import pytest

import oracle
from synth import bank_corpus, init_rows, uniform_matrix

pytestmark = pytest.mark.gpu

W_TOL = 1e-4


@pytest.fixture(scope="module")
def som():
    from paper_1905_09598_b200 import som as s
    s.lib()
    return s


def _check(W, b, Wo, bo, label):
    err = np.abs(W.astype(np.float64) - Wo).max()
    assert err <= W_TOL, err
    ndiff = int(np.count_nonzero(W != Wo))
    assert ndiff <= max(4, W.size // 10000), ndiff
    assert np.array_equal(b, bo), f"{label}: final BMUs differ on {np.count_nonzero(b != bo)} rows"
    print(f" [{label}: {ndiff} of {W.size} weights differ, max {err:.1e}]", end="")


@pytest.mark.parametrize("rows,cols,topo,n,d,epochs,csr", [
    (10, 10, 0, 200, 500, 10, False),   # c1 shape, dense rows
    (10, 10, 0, 200, 500, 10, True),    # the same from CSR (sparse-identity BMUs, CSR sums)
    (8, 12, 1, 600, 300, 6, True),
    (20, 20, 1, 3000, 1000, 3, True),   # N = 400 > one GEMM tile, ragged
    (3, 70, 1, 400, 64, 4, False),      # 3 x 70: unit tiles cross lattice rows
])
def test_batch_matches_oracle(som, rows, cols, topo, n, d, epochs, csr):
    C = bank_corpus(n, d, seed=rows * cols + d)
    X = C.dense()
    W0 = init_rows(X, rows * cols, 5)
    sigma0 = max(rows, cols) / 2.0
    with som.SOM(rows, cols, d, topo) as m:
        m.set_weights(W0)
        if csr:
            b = m.train_batch_csr(C.indptr, C.indices, C.data, C.n, epochs, sigma0)
        else:
            b = m.train_batch(X, epochs, sigma0)
        W = m.get_weights()
    Wo, bo = oracle.train_batch(W0, rows, cols, topo, X, epochs, sigma0)
    _check(W, b, Wo, bo, f"{rows}x{cols} n={n} d={d} E={epochs} {'csr' if csr else 'dense'}")


@pytest.mark.parametrize("kind,cutoff", [(1, 1e-4), (2, 0.0), (0, 1e-2)])
def test_batch_schedules(som, kind, cutoff):
    X = uniform_matrix(500, 40, kind + 3)
    W0 = init_rows(X, 6 * 7, 9)
    with som.SOM(6, 7, 40, 1) as m:
        m.set_weights(W0)
        b = m.train_batch(X, 5, 3.5, kind=kind, cutoff=cutoff)
        W = m.get_weights()
    Wo, bo = oracle.train_batch(W0, 6, 7, 1, X, 5, 3.5, kind=kind, eps=cutoff)
    _check(W, b, Wo, bo, f"kind={kind} eps={cutoff}")


def test_batch_kmeans_limit_and_empty_units(som):
    """sigma0 = sigma_min = 0.1: only the BMU itself weighs in, an epoch is a
    Lloyd step; a unit far from all rows keeps its weights."""
    X = uniform_matrix(400, 16, 21)
    W0 = uniform_matrix(20, 16, 22)
    W0[19] += 4.0
    with som.SOM(4, 5, 16, 0) as m:
        m.set_weights(W0)
        b = m.train_batch(X, 3, 0.1, sigma_min=0.1)
        W = m.get_weights()
    Wo, bo = oracle.train_batch(W0, 4, 5, 0, X, 3, 0.1, sigma_min=0.1)
    _check(W, b, Wo, bo, "k-means limit")
    assert np.array_equal(W[19], W0[19])


def test_batch_one_unit_zero_epochs_and_errors(som):
    X = uniform_matrix(100, 8, 31)
    with som.SOM(1, 1, 8, 0) as m:
        m.set_weights(np.zeros((1, 8), np.float32))
        b = m.train_batch(X, 2, 1.0)
        W = m.get_weights()
        assert np.all(b == 0)
        np.testing.assert_allclose(W[0], X.astype(np.float64).mean(0), rtol=0, atol=2e-7)
        m.set_weights(np.ones((1, 8), np.float32))
        m.train_batch(X, 0, 1.0)
        assert np.array_equal(m.get_weights(), np.ones((1, 8), np.float32))
        with pytest.raises(som.SomError) as e:
            som.som_train_batch(m.h, X, 0, 1, 1.0)
        assert e.value.status == som.SOM_EEMPTY
        with pytest.raises(som.SomError) as e:
            som.som_train_batch(m.h, X, 100, 1, -1.0)
        assert e.value.status == som.SOM_EINVAL


def test_batch_c3_shape_timing(som):
    """A c3-shaped batch epoch (50x50 map, 50k CSR docs x 10k terms): every
    step on the GPU; checked against the oracle on the final BMUs of a
    document sample via the exact mapping of the returned weights."""
    C = bank_corpus(50000, 10000, seed=77)
    W0 = init_rows(C.dense()[:5000], 2500, 78)
    with som.SOM(50, 50, 10000, 1) as m:
        m.set_weights(W0)
        b = m.train_batch_csr(C.indptr, C.indices, C.data, C.n, 2, 25.0)
        ms, units, launches = som.som_last_stats(m.h)
        W = m.get_weights()
    sample = np.arange(0, C.n, 97)
    Xs = C.dense()[sample]
    ob, _, _, m12, _ = oracle.map_docs(W, Xs, want_margins=True)
    ok = m12 > 1e-6
    assert np.array_equal(b[sample][ok], ob[ok])
    print(f" [c3-shaped batch SOM: 2 epochs of 50k docs in {ms:.1f} ms, {launches} launches]", end="")
