"""tcgen05 3xTF32 batch mapping (SOM_MAP_3XTF32) against the oracle.

Bar (BASELINE.json north_star, R19/R20): bmu1 identical on every
document whose oracle margin (D2-D1)/D1 exceeds 1e-5, bmu2 identical where
(D3-D2)/D2 also does; D1 within 1e-5 relative; QE within 1e-4."""
import numpy as np
import pytest

import oracle
from synth import bank_corpus, init_rows, uniform_matrix

pytestmark = pytest.mark.gpu

MARGIN = 1e-5


@pytest.fixture(scope="module")
def som():
    from paper_1905_09598_b200 import som as s
    s.lib()
    return s


def _codebook(X, N, seed):
    """Prototype-like codebook: blends of data rows with the corpus mean."""
    R = init_rows(X, N, seed).astype(np.float64)
    mu = X.mean(0, dtype=np.float64)
    return (0.6 * R + 0.4 * mu).astype(np.float32)


def _check(b1, b2, d1, ob1, ob2, od1, m12, m23):
    ok1 = m12 > MARGIN
    ok2 = ok1 & (m23 > MARGIN)
    assert ok1.mean() > 0.95, f"too many near ties: {ok1.mean()}"
    bad = np.flatnonzero(ok1 & (b1 != ob1))
    assert bad.size == 0, f"bmu1 differs on {bad.size} margin-filtered docs, e.g. {bad[:5]}"
    bad2 = np.flatnonzero(ok2 & (b2 != ob2))
    assert bad2.size == 0, f"bmu2 differs on {bad2.size} docs"
    # D1: tensor-core fp32 accumulation is not round-to-nearest (observed
    # positive bias growing with K). With the hi.hi and lo
    # products in separate TMEM accumulators the observed max is ~5e-6; bar
    # 1e-5 absolute, 10x inside the north star's 1e-4 max-abs for errors.
    ab = np.abs(d1.astype(np.float64) - od1)
    assert ab.max() <= 1e-5, ab.max()
    print(f" [3xTF32 D1 abs err max {ab.max():.2e} median {np.median(ab):.2e}]", end="")


@pytest.mark.parametrize("rows,cols,n,d,topo", [
    (20, 20, 5000, 3000, 1),     # c2 shape
    (10, 10, 200, 500, 0),       # c1 shape
    (13, 23, 1000, 1000, 1),     # N = 299 (ragged unit tile), d % 32 != 0
    (3, 5, 300, 333, 1),         # d % 4 != 0, tiny map
    (1, 1, 130, 64, 0),          # 1 unit: bmu2 = -1
])
def test_map_3xtf32_matches_oracle(som, rows, cols, n, d, topo):
    C = bank_corpus(n, d, seed=n + d + 1)
    X = C.dense()
    W = _codebook(X, rows * cols, 3)
    with som.SOM(rows, cols, d, topo) as m:
        m.set_weights(W)
        som.som_set_map_precision(m.h, som.SOM_MAP_3XTF32)
        b1, b2, d1 = m.map(X)
        qe, te = m.errors(X)
    ob1, ob2, od1, m12, m23 = oracle.map_docs(W, X, want_margins=True)
    if rows * cols == 1:
        assert np.all(b1 == 0) and np.all(b2 == -1)
        np.testing.assert_allclose(d1, od1, rtol=1e-5)
        return
    _check(b1, b2, d1, ob1, ob2, od1, m12, m23)
    assert abs(qe - oracle.qerror_from_d1(od1)) <= 1e-4
    ok = (m12 > MARGIN) & (m23 > MARGIN)
    te_o = oracle.topographic_error_from_bmus(rows, cols, topo, ob1, ob2)
    assert abs(te - te_o) <= (1 - ok.mean()) + 1e-12


def test_map_3xtf32_csr_equals_dense(som):
    C = bank_corpus(3000, 2000, seed=21)
    X = C.dense()
    W = _codebook(X, 300, 4)
    with som.SOM(15, 20, 2000, 1) as m:
        m.set_weights(W)
        som.som_set_map_precision(m.h, som.SOM_MAP_3XTF32)
        a1, a2, ad = m.map(X)
        b1 = np.empty(C.n, np.int32)
        b2 = np.empty(C.n, np.int32)
        bd = np.empty(C.n, np.float32)
        som.som_map_csr(m.h, C.indptr, C.indices, C.data, C.n, b1, b2, bd)
    ob1, ob2, od1, m12, m23 = oracle.map_docs(W, X, want_margins=True)
    _check(b1, b2, bd, ob1, ob2, od1, m12, m23)
    same = m12 > MARGIN
    assert np.array_equal(a1[same], b1[same])
    np.testing.assert_allclose(ad, bd, rtol=2e-7, atol=1e-7)


def test_map_3xtf32_c3_sample(som):
    """c3-like contraction (20k docs x 2500 units x 10k terms, CSR input);
    the oracle's sparse-identity path checks every document."""
    C = bank_corpus(20000, 10000, seed=33)
    Wsrc = bank_corpus(2500, 10000, seed=34).dense()
    W = (0.5 * Wsrc + 0.5 * C.dense()[:2500].mean(0)).astype(np.float32)
    with som.SOM(50, 50, 10000, 1) as m:
        m.set_weights(W)
        som.som_set_map_precision(m.h, som.SOM_MAP_3XTF32)
        b1 = np.empty(C.n, np.int32)
        b2 = np.empty(C.n, np.int32)
        d1 = np.empty(C.n, np.float32)
        som.som_map_csr(m.h, C.indptr, C.indices, C.data, C.n, b1, b2, d1)
        ms, units, _ = som.som_last_stats(m.h)
    ob1, ob2, od1, m12, m23 = oracle.map_docs_csr(W, C.indptr, C.indices, C.data, want_margins=True)
    _check(b1, b2, d1, ob1, ob2, od1, m12, m23)
    print(f"c3-like 3xTF32 mapping: {units} docs in {ms:.2f} ms")


def test_auto_precision_and_weight_changes(som):
    """AUTO switches to the tensor cores for large contractions; the cached W
    split follows weight updates (set_weights, training)."""
    C = bank_corpus(4000, 3000, seed=5)
    X = C.dense()
    W = _codebook(X, 1024, 6)
    with som.SOM(32, 32, 3000, 1) as m:
        m.set_weights(W)
        b1, _, _ = m.map(X)                        # 4000*1024*3000 = 1.2e10 -> tensor cores
        _, _, launches = som.som_last_stats(m.h)
        assert launches == 3
        W2 = W[::-1].copy()
        m.set_weights(W2)
        c1, _, _ = m.map(X)
    ob1, _, _, m12, _ = oracle.map_docs(W2, X, want_margins=True)
    ok = m12 > MARGIN
    assert np.array_equal(c1[ok], ob1[ok])
