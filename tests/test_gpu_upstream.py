"""Upstream steps on the GPU (R28-R31) against the
oracle: TF-IDF + L2 rows (som_tfidf_csr), top-2 PCA (som_pca_top2[_csr]),
PCA-plane linear init (som_init_linear), Fig. 2 sizing (som_map_geometry),
and the whole chain from raw counts to a trained map.

Bars: TF-IDF values within 1 fp32 ulp (the device log and the oracle's glibc
log may differ in the last fp64 bit; observed equal); eigenvalues within
1e-9 relative and eigenvectors within 1e-6 max-abs of LAPACK's (subspace
iteration stops at residual 1e-12 * pc1); init weights within 1e-6; sizing
exact."""
import numpy as np
import pytest

import oracle
from synth import bank_corpus, uniform_matrix

pytestmark = pytest.mark.gpu

ULP = 2.0 ** -23


@pytest.fixture(scope="module")
def som():
    from paper_1905_09598_b200 import som as s
    s.lib()
    return s


def _counts_corpus(n, d, seed):
    """Raw term counts with the corpus' sparsity pattern (integers 1..5), plus
    a column present in every row (idf 0) and an all-ubiquitous row."""
    C = bank_corpus(n, d, seed=seed)
    rng = np.random.default_rng(seed)
    cnt = rng.integers(1, 6, size=C.nnz).astype(np.float32)
    return C.indptr.copy(), C.indices.copy(), cnt


@pytest.mark.parametrize("n,d", [(500, 300), (5000, 3000), (7, 5)])
def test_tfidf_matches_oracle(som, n, d):
    rp, ci, cnt = _counts_corpus(n, d, n + d)
    ov, oz = oracle.tfidf_csr(rp, ci, cnt, d)
    with som.SOM(2, 2, d, 1) as m:
        out = np.empty_like(cnt)
        z = som.som_tfidf_csr(m.h, rp, ci, cnt, n, out)
    rel = np.abs(out.astype(np.float64) - ov) / np.maximum(np.abs(ov), 1e-30)
    assert rel.max() <= ULP and z == oz
    print(f" [tfidf {n}x{d}: {np.count_nonzero(out != ov)} values differ (<= 1 ulp)]", end="")


def test_tfidf_ubiquitous_term_and_zero_row(som):
    rp = np.array([0, 2, 4, 5], np.int64)
    ci = np.array([0, 2, 1, 2, 2], np.int32)
    cnt = np.array([1, 5, 2, 1, 7], np.float32)
    with som.SOM(1, 2, 3, 0) as m:
        out = np.empty(5, np.float32)
        z = som.som_tfidf_csr(m.h, rp, ci, cnt, 3, out)
    assert out.tolist() == [1.0, 0.0, 1.0, 0.0, 0.0] and z == 1


def _check_pca(got, ref):
    pc1, pc2, v1, v2, mu = got
    opc1, opc2, ov1, ov2, omu = ref
    assert abs(pc1 - opc1) <= 1e-9 * opc1 and abs(pc2 - opc2) <= 1e-9 * opc1
    assert np.abs(mu - omu).max() <= 1e-12
    assert np.abs(v1 - ov1).max() <= 1e-6 and np.abs(v2 - ov2).max() <= 1e-6


@pytest.mark.parametrize("n,d,csr", [(400, 50, False), (2000, 300, True), (3000, 1000, True), (300, 9, False)])
def test_pca_matches_lapack(som, n, d, csr):
    C = bank_corpus(n, d, seed=n + 3 * d)
    X = C.dense()
    ref = oracle.pca_top2(X)
    with som.SOM(2, 3, d, 1) as m:
        got = m.pca_top2(csr=(C.indptr, C.indices, C.data, C.n)) if csr else m.pca_top2(X)
        ms, _, launches = som.som_last_stats(m.h)
    _check_pca(got, ref)
    print(f" [pca {n}x{d}: {ms:.1f} ms, {launches} launches]", end="")


def test_pca_degenerate_collinear_and_constant(som):
    X = np.array([[1, 0], [-1, 0], [2, 0], [-2, 0]], np.float32)
    with som.SOM(1, 2, 2, 0) as m:
        pc1, pc2, v1, v2, mu = m.pca_top2(X)
    assert abs(pc1 - 10.0 / 3.0) < 1e-12 and abs(pc2) < 1e-12 and np.allclose(v1, [1, 0])
    Xc = np.ones((5, 4), np.float32)
    with som.SOM(1, 2, 4, 0) as m:
        pc1, pc2, v1, v2, mu = m.pca_top2(Xc)
    assert pc1 == 0.0 and pc2 == 0.0 and np.allclose(mu, 1.0)


def test_linear_init_matches_oracle(som):
    X = uniform_matrix(300, 40, 3)
    pc1, pc2, v1, v2, mu = oracle.pca_top2(X)
    with som.SOM(6, 9, 40, 1) as m:
        m.init_linear(mu, v1, v2, pc1, pc2)
        W = m.get_weights()
    Wo = oracle.linear_init(6, 9, mu, v1, v2, pc1, pc2)
    assert np.abs(W.astype(np.float64) - Wo).max() <= 1e-6
    assert np.count_nonzero(W != Wo) <= W.size // 1000


@pytest.mark.parametrize("m_,pc1,pc2", [(400, 1.0, 1.0), (4, 1.0, 1.0), (100, 10.0, 0.05), (513, 3.0, 1.0),
                                        (676, 0.0, 0.0), (10 ** 6, 5.0, 2.0)])
def test_map_geometry_matches_fig2(som, m_, pc1, pc2):
    assert som.som_map_geometry(m_, pc1, pc2) == oracle.map_geometry(m_, pc1, pc2)


def test_upstream_chain_counts_to_trained_map(som):
    """Raw counts -> TF-IDF -> PCA -> Fig. 2 sizing -> linear init -> online
    training on the GPU; the oracle runs the same chain from the same counts."""
    n, d = 600, 400
    rp, ci, cnt = _counts_corpus(n, d, 9)
    val, _ = oracle.tfidf_csr(rp, ci, cnt, d)
    X = np.zeros((n, d), np.float32)
    for i in range(n):
        X[i, ci[rp[i]:rp[i + 1]]] = val[rp[i]:rp[i + 1]]
    opc1, opc2, ov1, ov2, omu = oracle.pca_top2(X)
    orows, ocols, oitr = oracle.map_geometry(n, opc1, opc2)
    W0o = oracle.linear_init(orows, ocols, omu, ov1, ov2, opc1, opc2)
    epochs = max(1, min(3, oitr // n))
    Wo, logo = oracle.train_online(W0o, orows, ocols, 1, X, epochs, 0.1, max(orows, ocols) / 2.0, 5)
    with som.SOM(2, 2, d, 1) as pre:
        gv = np.empty_like(cnt)
        som.som_tfidf_csr(pre.h, rp, ci, cnt, n, gv)
        pc1, pc2, v1, v2, mu = pre.pca_top2(csr=(rp, ci, gv, n))
    rows, cols, itr = som.som_map_geometry(n, pc1, pc2)
    assert (rows, cols, itr) == (orows, ocols, oitr)
    with som.SOM(rows, cols, d, 1) as m:
        m.init_linear(mu, v1, v2, pc1, pc2)
        log = np.empty(epochs * n, np.int32)
        m.train_online_csr(rp, ci, gv, n, epochs, alpha0=0.1, sigma0=max(rows, cols) / 2.0, seed=5, bmu_log=log)
        W = m.get_weights()
    assert np.abs(W.astype(np.float64) - Wo).max() <= 1e-4
    agree = np.mean(log == logo)
    assert agree >= 0.99, agree
    print(f" [chain: {rows}x{cols} map, {epochs} epochs, BMU agreement {agree:.4f}]", end="")


def test_upstream_validation(som):
    """Arguments are checked before any side effect (som.h conventions)."""
    with som.SOM(2, 2, 5, 1) as m:
        W0 = np.arange(20, dtype=np.float32).reshape(4, 5)
        m.set_weights(W0)
        rp = np.array([0, 2, 3], np.int64)
        ci = np.array([0, 7, 1], np.int32)           # column 7 >= dim 5
        cnt = np.ones(3, np.float32)
        out = np.empty(3, np.float32)
        with pytest.raises(som.SomError) as e:
            som.som_tfidf_csr(m.h, rp, ci, cnt, 2, out)
        assert e.value.status == som.SOM_EINVAL
        with pytest.raises(som.SomError) as e:
            m.pca_top2(np.ones((1, 5), np.float32))   # n = 1
        assert e.value.status == som.SOM_EINVAL
        with pytest.raises(som.SomError):
            som.som_init_linear(m.h, np.zeros(5), np.zeros(5), np.zeros(5), float("nan"), 1.0)
        assert np.array_equal(m.get_weights(), W0)
        with pytest.raises(som.SomError):
            som.som_map_geometry(0, 1.0, 1.0)
        with pytest.raises(som.SomError):
            som.som_map_geometry(10, -1.0, 1.0)
        with pytest.raises(som.SomError) as e:
            m.train_batch_csr(rp, ci, cnt, 2, 1, 1.0)  # malformed CSR: weights untouched
        assert np.array_equal(m.get_weights(), W0)
