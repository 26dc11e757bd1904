"""tcgen05 3xTF32 batch mapping (SOM_MAP_3XTF32) against the oracle.

The tensor cores are a filter (R20b): 4 candidates per document
from the 3xTF32 contraction, rescored by the exact fp64 definition (R10) and
certified against a bound on the approximation error, else mapped exactly
over every unit.  Bar: bmu1, bmu2 and D1 equal the oracle's on EVERY
document — no margin filter — including exact ties (duplicate prototypes:
lowest index first, R9) and documents placed at near-ties, which must take
the exact fallback."""
import numpy as np
import pytest

import oracle
from synth import bank_corpus, init_rows

pytestmark = pytest.mark.gpu


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


def _check_all(b1, b2, d1, ob1, ob2, od1):
    bad = np.flatnonzero(b1 != ob1)
    assert bad.size == 0, f"bmu1 differs on {bad.size} docs, e.g. {bad[:5]}"
    bad2 = np.flatnonzero(b2 != ob2)
    assert bad2.size == 0, f"bmu2 differs on {bad2.size} docs, e.g. {bad2[:5]}"
    diff = np.flatnonzero(d1 != od1.astype(np.float32))
    assert diff.size == 0, f"D1 differs on {diff.size} docs (max {np.abs(d1[diff] - od1[diff]).max():.3g})"


def _map_tc(som, m, X=None, csr=None):
    som.som_set_map_precision(m.h, som.SOM_MAP_3XTF32)
    if csr is None:
        b1, b2, d1 = m.map(X)
    else:
        n = csr.n
        b1, b2, d1 = np.empty(n, np.int32), np.empty(n, np.int32), np.empty(n, np.float32)
        som.som_map_csr(m.h, csr.indptr, csr.indices, csr.data, n, b1, b2, d1)
    return b1, b2, d1, som.som_last_map_fallbacks(m.h)


@pytest.mark.parametrize("rows,cols,n,d,topo", [
    (20, 20, 5000, 3000, 1),     # c2 shape
    (10, 10, 200, 500, 0),       # c1 shape
    (13, 23, 1000, 1000, 1),     # N = 299 (ragged unit tile), d % 32 != 0
    (3, 5, 300, 333, 1),         # d % 4 != 0, tiny map
    (2, 2, 150, 40, 0),          # N = 4: every unit a candidate
    (1, 1, 130, 64, 0),          # 1 unit: bmu2 = -1
])
def test_map_3xtf32_exact_on_every_document(som, rows, cols, n, d, topo):
    C = bank_corpus(n, d, seed=n + d + 1)
    X = C.dense()
    W = _codebook(X, rows * cols, 3)
    with som.SOM(rows, cols, d, topo) as m:
        m.set_weights(W)
        b1, b2, d1, nf = _map_tc(som, m, X=X)
        som.som_set_map_precision(m.h, som.SOM_MAP_3XTF32)
        qe, te = m.errors(X)
    ob1, ob2, od1 = oracle.map_docs(W, X)
    _check_all(b1, b2, d1, ob1, ob2, od1)
    assert abs(qe - oracle.qerror_from_d1(od1)) <= 1e-12
    assert te == oracle.topographic_error_from_bmus(rows, cols, topo, ob1, ob2)
    print(f" [{rows}x{cols} d={d}: {nf} of {n} docs by the exact fallback]", end="")


def test_map_3xtf32_ties_and_near_ties(som):
    """Where the tensor-core filter cannot decide: eight prototypes within a
    few fp32 ulps of each other (the 3xTF32 error exceeds their spread: the
    certificate fails and the sparse-identity scan decides) and six exact
    duplicates (ties at every precision: the dense scan over every unit
    decides, lowest index first, R9).  Identical to the oracle on every
    document, dense and CSR input."""
    C = bank_corpus(1500, 1500, seed=41)
    X = C.dense()
    W = _codebook(X, 256, 42)
    base = W[40].copy()
    for j in range(8):                           # units 40..47: base + j ulps on one element each
        W[40 + j] = base
        k = int(np.flatnonzero(base)[j % np.count_nonzero(base)])
        W[40 + j, k] = np.nextafter(base[k], np.float32(2.0)) if j else base[k]
        for _ in range(j // 2):
            W[40 + j, k] = np.nextafter(W[40 + j, k], np.float32(2.0))
    W[100:106] = W[60]                           # units 60, 100..105: exact duplicates
    rng = np.random.default_rng(43)
    near = (base + rng.random((40, 1500)).astype(np.float32) * 1e-4 * (base > 0)).astype(np.float32)
    Xt = np.concatenate([X, near, np.repeat(W[60:61], 10, 0)])
    from scipy import sparse
    Ct = sparse.csr_matrix(Xt)
    with som.SOM(16, 16, 1500, 1) as m:
        m.set_weights(W)
        b1, b2, d1, nf = _map_tc(som, m, X=Xt)
        c1 = np.empty(Xt.shape[0], np.int32)
        c2 = np.empty(Xt.shape[0], np.int32)
        cd = np.empty(Xt.shape[0], np.float32)
        som.som_set_map_precision(m.h, som.SOM_MAP_3XTF32)
        som.som_map_csr(m.h, Ct.indptr.astype(np.int64), Ct.indices.astype(np.int32), Ct.data.astype(np.float32),
                        Xt.shape[0], c1, c2, cd)
        nf_csr = som.som_last_map_fallbacks(m.h)
    ob1, ob2, od1 = oracle.map_docs(W, Xt)
    _check_all(b1, b2, d1, ob1, ob2, od1)
    _check_all(c1, c2, cd, ob1, ob2, od1)
    assert nf >= 10 and nf_csr >= 10, (nf, nf_csr)
    assert np.all(b1[-10:] == 60) and np.all(b2[-10:] == 100)
    print(f" [{nf} (dense) / {nf_csr} (CSR) of {Xt.shape[0]} docs took a fallback]", end="")


def test_map_3xtf32_csr_equals_dense(som):
    C = bank_corpus(3000, 2000, seed=21)
    X = C.dense()
    W = _codebook(X, 300, 4)
    with som.SOM(15, 20, 2000, 1) as m:
        m.set_weights(W)
        a1, a2, ad, _ = _map_tc(som, m, X=X)
        b1, b2, bd, nf = _map_tc(som, m, csr=C)
    ob1, ob2, od1 = oracle.map_docs(W, X)
    _check_all(b1, b2, bd, ob1, ob2, od1)
    assert np.array_equal(a1, b1) and np.array_equal(a2, b2) and np.array_equal(ad, bd)


def test_map_3xtf32_c3_sample(som):
    """c3-like contraction (20k docs x 2500 units x 10k terms, CSR input):
    every document against the oracle's sparse-identity mapping (R25 — its
    D1 may differ from the dense definition's in the last fp32 ulp)."""
    C = bank_corpus(20000, 10000, seed=33)
    Wsrc = bank_corpus(2500, 10000, seed=34).dense()
    W = (0.5 * Wsrc + 0.5 * C.dense()[:2500].mean(0)).astype(np.float32)
    with som.SOM(50, 50, 10000, 1) as m:
        m.set_weights(W)
        b1, b2, d1, nf = _map_tc(som, m, csr=C)
        ms, units, _ = som.som_last_stats(m.h)
    ob1, ob2, od1 = oracle.map_docs_csr(W, C.indptr, C.indices, C.data)
    assert np.array_equal(b1, ob1) and np.array_equal(b2, ob2)
    ulp = np.spacing(od1.astype(np.float32))
    assert np.all(np.abs(d1.astype(np.float64) - od1) <= ulp)
    print(f" [c3-like 3xTF32 mapping: {units} docs in {ms:.2f} ms, {nf} exact fallbacks]", end="")


def test_auto_precision_and_weight_changes(som):
    """AUTO switches to the tensor cores for large dense contractions; the
    cached W split follows weight updates (set_weights)."""
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
        c1, c2, cd = m.map(X)
    ob1, ob2, od1 = oracle.map_docs(W2, X)
    _check_all(c1, c2, cd, ob1, ob2, od1)


def test_tc_many_work_items_per_cta(som):
    """More (128-document block, 128-unit tile) work items than CTAs: 10,240
    documents x 2 unit tiles = 160 items on <= 148 persistent CTAs, so CTAs
    run several tiles and alternate the two TMEM accumulator buffers (the
    epilogue of one tile overlapping the MMAs of the next).  Every document
    exact."""
    C = bank_corpus(10240, 512, seed=15)
    X = C.dense()
    W = _codebook(X, 16 * 16, 16)
    with som.SOM(16, 16, 512, 1) as m:
        m.set_weights(W)
        b1, b2, d1, fb = _map_tc(som, m, X)
    ob1, ob2, od1 = oracle.map_docs(W, X)
    _check_all(b1, b2, d1, ob1, ob2, od1)
    print(f" [fallbacks {fb}]", end="")
