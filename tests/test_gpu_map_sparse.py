"""Exact sparse batch mapping (SOM_MAP_SPARSE_F64, map_sparse.cu) against
the oracle.

The kernel evaluates the sparse identity (R25)
    D_u = RN32(max(0, (|x|^2 - 2 sum_{k in nz(x)} x_k w_uk) + |w_u|^2))
in fp64.  It equals the definition (R10) in real arithmetic; the two fp64
evaluations differ by a few fp64 ulp, so the fp32 D agrees with the oracle
except when the exact sum lies within ~1e-16 relative of an fp32 rounding
boundary; where D itself is ~0 the fp64 error of the expansion (a few ulp
of |x|^2 + |w|^2, absolute) dominates.  Bar: D1 within one fp32 ulp of the
oracle's or 1e-14 absolute (observed: equal except D = 0 documents),
bmu1 identical on every document whose oracle margin (D2-D1)/D1 exceeds
1e-6 (16 fp32 ulp; the 3xTF32 path needs 1e-5), bmu2 likewise with
(D3-D2)/D2; QE within 1e-6 and TE exact on the same filter.  Both oracle
paths are used: the dense definition (or_map) and the sparse identity
(or_map_csr)."""
import numpy as np
import pytest

import oracle
from synth import bank_corpus, init_rows

pytestmark = pytest.mark.gpu

MARGIN = 1e-6
ULP = 2.0 ** -23


@pytest.fixture(scope="module")
def som():
    from paper_1905_09598_b200 import som as s
    s.lib()
    return s


def _codebook(X, N, seed):
    R = init_rows(X, N, seed).astype(np.float64)
    mu = X.mean(0, dtype=np.float64)
    return (0.6 * R + 0.4 * mu).astype(np.float32)


def _map_sparse(som, m, rowptr, col, val, n):
    som.som_set_map_precision(m.h, som.SOM_MAP_SPARSE_F64)
    return m.map_csr(rowptr, col, val, n)


def _check(b1, b2, d1, ob1, ob2, od1, m12, m23):
    ok1 = m12 > MARGIN
    ok2 = ok1 & (m23 > MARGIN)
    assert ok1.mean() > 0.98, f"too many near ties: {ok1.mean()}"
    bad = np.flatnonzero(ok1 & (b1 != ob1))
    assert bad.size == 0, f"bmu1 differs on {bad.size} margin-filtered docs, e.g. {bad[:5]}"
    bad2 = np.flatnonzero(ok2 & (b2 != ob2))
    assert bad2.size == 0, f"bmu2 differs on {bad2.size} docs"
    same = b1 == ob1
    # R25: the expansion's fp64 error is absolute, a few ulp of |x|^2 + |w|^2
    # (~1e-16 here): within one fp32 ulp relative, or 1e-14 absolute where D
    # is ~0 (a document equal to its prototype: D = 0 exactly in the oracle)
    err = np.abs(d1[same].astype(np.float64) - od1[same])
    assert np.all(err <= ULP * od1[same] + 1e-14), err.max(initial=0.0)
    return int(np.count_nonzero(d1 != od1))


@pytest.mark.parametrize("rows,cols,n,d,topo,cfg", [
    (20, 20, 5000, 3000, 1, None),    # c2 shape (N = 400: 2 x 256-unit tiles, ragged)
    (20, 20, 5000, 3000, 1, "d4"),    # same, fp64 W^T
    (10, 10, 200, 500, 0, None),      # c1 shape
    (13, 23, 1000, 1000, 1, "d1"),    # N = 299, 64-unit tiles (5, ragged), fp64 W^T
    (13, 23, 1000, 1000, 1, "d2"),
    (13, 23, 1000, 1000, 1, "f2"),    # fp32 W^T, 128-unit tiles
    (13, 23, 1000, 1000, 1, "f8"),    # fp32 W^T, 512-unit tiles (1 ragged tile)
    (3, 5, 300, 333, 1, "f4"),        # tiny map, odd d
    (1, 1, 130, 64, 0, None),         # 1 unit: bmu2 = -1
    (50, 50, 4000, 10000, 1, None),   # c3 map, 10 tiles of 256 (ragged)
])
def test_map_sparse_matches_oracle(som, monkeypatch, rows, cols, n, d, topo, cfg):
    if cfg is not None:     # W^T storage (d = fp64, f = fp32) and tile width 64 J
        monkeypatch.setenv("SOM_SPARSE_F32", "1" if cfg[0] == "f" else "0")
        monkeypatch.setenv("SOM_SPARSE_J", cfg[1:])
    C = bank_corpus(n, d, seed=n + d + 7)
    X = C.dense()
    N = rows * cols
    W = _codebook(X, N, 5)
    with som.SOM(rows, cols, d, topo) as m:
        m.set_weights(W)
        b1, b2, d1 = _map_sparse(som, m, C.indptr, C.indices, C.data, C.n)
        qe, te = m.errors_csr(C.indptr, C.indices, C.data, C.n)
    ob1, ob2, od1, m12, m23 = oracle.map_docs(W, X, want_margins=True)
    if N == 1:
        assert np.all(b1 == 0) and np.all(b2 == -1)
        rel = np.abs(d1.astype(np.float64) - od1) / od1
        assert rel.max() <= ULP
        return
    ndiff = _check(b1, b2, d1, ob1, ob2, od1, m12, m23)
    print(f" [D1 differs from the dense definition on {ndiff}/{n} docs (<= 1 ulp)]", end="")
    assert abs(qe - oracle.qerror_from_d1(od1)) <= 1e-6
    ok = (m12 > MARGIN) & (m23 > MARGIN)
    te_o = oracle.topographic_error_from_bmus(rows, cols, topo, ob1, ob2)
    assert abs(te - te_o) <= (1 - ok.mean()) + 1e-12


def test_map_sparse_vs_sparse_oracle_c5_shape(som):
    """c5-shaped contraction (100x100 map, 20k terms) on a 20k-document
    sample; the oracle's sparse-identity path (or_map_csr) checks every
    document."""
    C = bank_corpus(20000, 20000, seed=55)
    Wsrc = bank_corpus(10000, 20000, seed=56).dense()
    W = (0.5 * Wsrc + 0.5 / np.sqrt(20000)).astype(np.float32)
    del Wsrc
    with som.SOM(100, 100, 20000, 1) as m:
        m.set_weights(W)
        b1, b2, d1 = _map_sparse(som, m, C.indptr, C.indices, C.data, C.n)
        ms, units, launches = som.som_last_stats(m.h)
    ob1, ob2, od1, m12, m23 = oracle.map_docs_csr(W, C.indptr, C.indices, C.data, want_margins=True)
    ndiff = _check(b1, b2, d1, ob1, ob2, od1, m12, m23)
    print(f" [c5-shaped sparse mapping: {units} docs in {ms:.2f} ms, {ndiff} D1 differ by <= 1 ulp]", end="")


def test_map_sparse_edge_rows(som):
    """Empty rows (D = |w|^2: the unit of smallest norm), rows with more than
    32 non-zeros (several fetch rounds), a row with every term set, and
    negative / large values (the identity does not assume TF-IDF ranges)."""
    rng = np.random.default_rng(3)
    d, N = 700, 37
    rows_nz = [0, 1, 31, 32, 33, 64, 65, 200, d, 0, 5]
    indptr = np.zeros(len(rows_nz) + 1, np.int64)
    cols, vals = [], []
    for i, k in enumerate(rows_nz):
        c = np.sort(rng.choice(d, size=k, replace=False)).astype(np.int32)
        cols.append(c)
        vals.append(rng.normal(0, 1, size=k).astype(np.float32) * (10.0 if i == 4 else 1.0))
        indptr[i + 1] = indptr[i] + k
    col = np.concatenate(cols)
    val = np.concatenate(vals)
    n = len(rows_nz)
    W = rng.normal(0, 0.5, size=(N, d)).astype(np.float32)
    W[7] *= 0.01                      # smallest norm: the BMU of an empty row
    X = np.zeros((n, d), np.float32)
    for i in range(n):
        X[i, col[indptr[i]:indptr[i + 1]]] = val[indptr[i]:indptr[i + 1]]
    with som.SOM(1, N, d, 0) as m:
        m.set_weights(W)
        b1, b2, d1 = _map_sparse(som, m, indptr, col, val, n)
    ob1, ob2, od1, m12, m23 = oracle.map_docs(W, X, want_margins=True)
    assert b1[0] == 7 and b1[9] == 7
    assert np.array_equal(b1, ob1) and np.array_equal(b2, ob2)
    rel = np.abs(d1.astype(np.float64) - od1) / np.maximum(od1, 1e-30)
    assert rel.max() <= ULP


def test_map_sparse_auto_and_cache(som):
    """AUTO picks the sparse path for TF-IDF rows; the cached W^T follows
    weight changes (set_weights and training)."""
    C = bank_corpus(3000, 2000, seed=12)
    X = C.dense()
    W = _codebook(X, 150, 2)
    with som.SOM(10, 15, 2000, 1) as m:
        m.set_weights(W)
        a1, _, ad = m.map_csr(C.indptr, C.indices, C.data, C.n)
        W2 = W[::-1].copy()
        m.set_weights(W2)
        c1, _, cd = m.map_csr(C.indptr, C.indices, C.data, C.n)
        m.train_online_csr(C.indptr, C.indices, C.data, C.n, 1, t_end=500)
        W3 = m.get_weights()
        e1, _, ed = m.map_csr(C.indptr, C.indices, C.data, C.n)
        som.som_set_map_precision(m.h, som.SOM_MAP_EXACT_F64)
        x1, _, xd = m.map_csr(C.indptr, C.indices, C.data, C.n)
    for Wk, b, dd in ((W, a1, ad), (W2, c1, cd), (W3, e1, ed)):
        ob1, _, od1, m12, _ = oracle.map_docs(Wk, X, want_margins=True)
        ok = m12 > MARGIN
        assert np.array_equal(b[ok], ob1[ok])
        assert np.abs(dd.astype(np.float64) - od1).max() <= ULP * od1.max()
    ob1, _, od1 = oracle.map_docs(W3, X)
    assert np.array_equal(x1, ob1) and np.array_equal(xd, od1)   # the exact dense path stays bit-exact


@pytest.mark.parametrize("cfg", ["f8", "f4"])
def test_integer_widening_is_exact(som, monkeypatch, cfg):
    """fp32 W^T with half the values widened on the integer pipe (W holds
    only +0 and positive normals: codebook rows are TF-IDF documents, so
    most entries are exact zeros; one -0 is normalised): results equal the
    F2F-only kernel bit for bit and the oracle."""
    C = bank_corpus(3000, 4000, seed=71)
    X = C.dense()
    W = init_rows(X, 1024, 72).copy()
    W[5, 7] = -0.0
    assert (W == 0).mean() > 0.9
    monkeypatch.setenv("SOM_SPARSE_F32", "1")
    monkeypatch.setenv("SOM_SPARSE_J", cfg[1:])
    outs = []
    for icv in ("1", "0"):
        monkeypatch.setenv("SOM_SPARSE_ICV", icv)
        with som.SOM(32, 32, 4000, 1) as m:
            m.set_weights(W)
            outs.append(_map_sparse(som, m, C.indptr, C.indices, C.data, C.n))
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)
    ob1, ob2, od1, m12, m23 = oracle.map_docs(W, X, want_margins=True)
    _check(*outs[0], ob1, ob2, od1, m12, m23)


def test_dense_rows_through_sparse_path(som):
    """SOM_MAP_SPARSE_F64 on dense rows: the rows are put in CSR form on the
    device (column order), so every output equals the CSR-input call bit for
    bit; QE/TE through som_errors likewise."""
    C = bank_corpus(4000, 3000, seed=81)
    X = C.dense()
    W = _codebook(X, 400, 82)
    with som.SOM(20, 20, 3000, 1) as m:
        m.set_weights(W)
        som.som_set_map_precision(m.h, som.SOM_MAP_SPARSE_F64)
        a = m.map(X)
        qa, ta = m.errors(X)
        b = m.map_csr(C.indptr, C.indices, C.data, C.n)
        qb, tb = m.errors_csr(C.indptr, C.indices, C.data, C.n)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
    assert qa == qb and ta == tb
    ob1, ob2, od1, m12, m23 = oracle.map_docs(W, X, want_margins=True)
    _check(*a, ob1, ob2, od1, m12, m23)
