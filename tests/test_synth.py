"""Input generator properties (synth/ holds no SOM arithmetic)."""
import numpy as np

from synth import bank_corpus


def test_corpus_deterministic_and_normalised():
    a = bank_corpus(300, 2000, seed=7)
    b = bank_corpus(300, 2000, seed=7)
    assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
    assert np.array_equal(a.data, b.data)
    X = a.dense()
    norms = np.sqrt((X.astype(np.float64) ** 2).sum(1))
    assert np.all(np.abs(norms - 1.0) < 1e-6)          # P:174 normalised rows
    assert np.all(a.data > 0)                          # non-negative, no explicit zeros
    assert np.all(np.diff(a.indptr) > 0)               # no zero rows (R17)
    for i in range(a.n):
        cols = a.indices[a.indptr[i]:a.indptr[i + 1]]
        assert np.all(np.diff(cols) > 0)


def test_idf_eq2_weights_are_count_times_idf():
    # Eq. 2: w = count * ln(n/df), then L2-normalised; so within a
    # row, w_k / ln(n/df_k) is proportional to an integer count.
    C = bank_corpus(400, 600, seed=3)
    df = np.bincount(C.indices, minlength=C.d)
    assert np.all(df < C.n)                            # idf 0 terms are never stored
    for i in range(0, C.n, 37):
        cols = C.indices[C.indptr[i]:C.indptr[i + 1]]
        vals = C.data[C.indptr[i]:C.indptr[i + 1]].astype(np.float64)
        ratio = vals / np.log(C.n / df[cols])
        ok = False
        for cmin in range(1, 8):
            cnt = ratio / ratio.min() * cmin
            if np.all(np.abs(cnt - np.rint(cnt)) < 1e-4 * cnt):
                ok = True
                break
        assert ok


def test_bank_shape_nnz():
    C = bank_corpus(513, 3917, seed=1)                # Axis shape, Table 1
    assert 25 < C.nnz / C.n < 70
