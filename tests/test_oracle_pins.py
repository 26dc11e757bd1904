"""Pins for the oracle: each check ties oracle/ to something other than itself
(hand-computed values, published KATs, closed forms, brute force through a
different library routine, invariants).  CPU only."""
import json
import math
import os
import struct
from fractions import Fraction

import numpy as np
import pytest

import oracle
from synth import bank_corpus, init_rows, uniform_matrix

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _bits(a):
    return [f"{struct.unpack('<I', struct.pack('<f', float(v)))[0]:08x}" for v in np.ravel(a)]


def _rn_f32(q: Fraction) -> np.float32:
    """Exact round-to-nearest-even of a rational to binary32 (normal range)."""
    if q == 0:
        return np.float32(0.0)
    sign = -1 if q < 0 else 1
    q = abs(q)
    e = math.floor(math.log2(q.numerator) - math.log2(q.denominator))
    while Fraction(2) ** e > q:
        e -= 1
    while Fraction(2) ** (e + 1) <= q:
        e += 1
    scaled = q / Fraction(2) ** (e - 23)          # in [2^23, 2^24)
    m = math.floor(scaled)
    rem = scaled - m
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and m % 2 == 1):
        m += 1
    return np.float32(sign * m * 2.0 ** (e - 23))


# ------------------------------------------------------------------ sampler
def test_splitmix64_published_kat():
    g = _gold("splitmix64_kat.json")
    got = [f"{oracle.splitmix64(0, t):016x}" for t in range(3)]
    assert got == g["seed0_first3"]


def test_sample_index_survey_regression_and_range():
    g = _gold("splitmix64_kat.json")
    assert [oracle.sample_index(1, t, 200) for t in range(10)] == g["survey_A9_seed1_n200_i0_9"]
    assert [oracle.sample_index(42, t, 5000) for t in range(10)] == g["survey_A9_seed42_n5000_i0_9"]
    idx = np.array([oracle.sample_index(7, t, 13) for t in range(20000)])
    assert idx.min() == 0 and idx.max() == 12
    # uniform with replacement (R8): chi-square-ish sanity, 13 bins
    cnt = np.bincount(idx, minlength=13)
    assert np.all(np.abs(cnt - 20000 / 13) < 5 * math.sqrt(20000 / 13))


# ----------------------------------------------------------------- schedule
def test_schedule_endpoints_closed_form():
    a0, s0 = 0.1, 5.0
    a, s, r2 = oracle.schedule(0, 2000, a0, s0)
    assert a == a0 and s == s0                          # alpha_0 = alpha0 exactly (R6)
    assert math.isclose(r2, 2 * 25 * math.log(1e4), rel_tol=1e-15)
    # alpha(T-1) / (alpha0/100) = exp(ln100 (1 - ((T-1)/T)^2)): 1.0046 at T=2000 (SURVEY [A2])
    a, _, _ = oracle.schedule(1999, 2000, a0, s0)
    assert abs(a / (a0 / 100) - 1.0046) < 1e-4
    a, _, _ = oracle.schedule(499999, 500000, a0, s0)
    assert abs(a / (a0 / 100) - 1.0000184) < 1e-6
    # sigma floor (R3): sigma0 = 0.5 is floored to sigma_min = 1
    _, s, _ = oracle.schedule(0, 10, 0.1, 0.5)
    assert s == 1.0
    # eps = 0 -> no cutoff
    _, _, r2 = oracle.schedule(3, 10, 0.1, 2.0, eps=0.0)
    assert r2 == math.inf
    # monotone non-increasing in t for all three decay kinds, all end at 1 %
    for kind in (0, 1, 2):
        al = [oracle.schedule(t, 100, 1.0, 10.0, kind=kind)[0] for t in range(101)]
        assert all(x >= y for x, y in zip(al, al[1:]))
        assert math.isclose(al[-1], 0.01, rel_tol=1e-12)


# ------------------------------------------------------------------ lattice
def test_lattice_spec_examples():
    g = _gold("lattice.json")
    cols = 7
    for (iu, ju), (iv, jv), want in g["hex_pairs_g2"]:
        assert oracle.lattice_g2(6, cols, 1, iu * cols + ju, iv * cols + jv) == want
    for (iu, ju), (iv, jv), want in g["rect_pairs_g2"]:
        assert oracle.lattice_g2(6, cols, 0, iu * cols + ju, iv * cols + jv) == want


def test_lattice_symmetry_and_spec_positions():
    rows, cols = 6, 7
    N = rows * cols
    for topo in (0, 1):
        for u in range(N):
            for v in range(N):
                g = oracle.lattice_g2(rows, cols, topo, u, v)
                assert g == oracle.lattice_g2(rows, cols, topo, v, u)
                assert g * 4 == int(g * 4)                  # multiples of 1/4: exact
                # SPEC S:164 planar positions, evaluated independently in float
                iu, ju, iv, jv = u // cols, u % cols, v // cols, v % cols
                if topo == 1:
                    pu = (ju + 0.5 * (iu % 2), iu * math.sqrt(3) / 2)
                    pv = (jv + 0.5 * (iv % 2), iv * math.sqrt(3) / 2)
                else:
                    pu, pv = (ju, iu), (jv, iv)
                ref = (pu[0] - pv[0]) ** 2 + (pu[1] - pv[1]) ** 2
                assert abs(g - ref) < 1e-12


def test_hex_neighbour_histogram():
    g = _gold("lattice.json")
    rows, cols = 6, 7
    hist = {}
    for u in range(rows * cols):
        c = sum(oracle.lattice_g2(rows, cols, 1, u, v) == 1.0 for v in range(rows * cols))
        hist[str(c)] = hist.get(str(c), 0) + 1
    assert hist == g["hex_6x7_neighbour_histogram"]
    # rectangular: interior units have exactly 4
    c = sum(oracle.lattice_g2(6, 7, 0, 2 * 7 + 3, v) == 1.0 for v in range(42))
    assert c == 4


# ----------------------------------------------------- worked example (Eq. 1)
@pytest.mark.parametrize("topo,key", [(0, "rect"), (1, "hex")])
def test_worked_example_2x2(topo, key):
    g = _gold("worked_example_2x2.json")
    W = np.array(g["W"], np.float32)
    x = np.array(g["x"], np.float32)
    c, D, _ = oracle.bmu(W, x)
    assert c == g["bmu"] and D == np.float32(g["D2"][c])
    W1 = oracle.update(W.copy(), 2, 2, topo, x, c, g["alpha"], g["sigma"], math.inf)
    assert _bits(W1) == [b for row in g[key]["W_new_bits"] for b in row]
    # independent derivation: exact rational evaluation of fmaf(h, RN(x-w), w)
    for u in range(4):
        g2 = g[key]["g2"][u]
        assert oracle.lattice_g2(2, 2, topo, u, c) == g2
        h = np.float32(g["alpha"] * math.exp(-g2 / 2.0))
        if key == "rect":
            assert abs(float(h) - g["rect"]["h"][u]) < 1e-9
        for k in range(2):
            diff = _rn_f32(Fraction(float(x[k])) - Fraction(float(W[u, k])))
            want = _rn_f32(Fraction(float(h)) * Fraction(float(diff)) + Fraction(float(W[u, k])))
            assert W1[u, k] == want
    U = oracle.umatrix(W, 2, 2, topo)
    np.testing.assert_allclose(U, g[key]["U"], rtol=0, atol=1e-7)


def test_tie_rule():
    g = _gold("worked_example_2x2.json")
    W = np.array(g["W"], np.float32)
    c, D, m = oracle.bmu(W, np.array(g["tie"]["x_all_equal"], np.float32))
    assert c == g["tie"]["bmu_all_equal"] and m == 0.0
    b1, b2, d1 = oracle.map_docs(W, np.array([g["tie"]["map_x"]], np.float32))
    assert (b1[0], b2[0]) == (g["tie"]["map_bmu1"], g["tie"]["map_bmu2"])
    # rect: 1 and 0 adjacent -> TE contribution 0
    assert oracle.topographic_error_from_bmus(2, 2, 0, b1, b2) == 0.0


def test_spec_update_examples():
    # 1-unit map, alpha = 0.1 at t = 0: w = (0), x = (1) -> w' = (0.1)
    W = np.zeros((1, 1), np.float32)
    W1, log = oracle.train_online(W, 1, 1, 0, np.ones((1, 1), np.float32), epochs=1,
                                  alpha0=0.1, sigma0=1.0, seed=3)
    assert W1[0, 0] == np.float32(0.1) and log[0] == 0
    # S:213 h = 0 -> unchanged; alpha = 0 here
    W = uniform_matrix(4, 5, 1)
    W1 = oracle.update(W.copy(), 2, 2, 0, uniform_matrix(1, 5, 2)[0], 0, 0.0, 1.0, math.inf)
    assert np.array_equal(W1, W)


# -------------------------------------------------------------- BMU / map
def test_bmu_and_map_brute_force():
    for seed in range(5):
        W = uniform_matrix(23, 17, seed)
        X = uniform_matrix(40, 17, 100 + seed)
        b1, b2, d1, m12, _ = oracle.map_docs(W, X, want_margins=True)
        for i in range(40):
            # different summation (numpy pairwise) in fp64, then fp32 key (R9, R10)
            acc = np.sum((X[i].astype(np.float64) - W.astype(np.float64)) ** 2, axis=1)
            D = acc.astype(np.float32)
            order = np.lexsort((np.arange(23), D))
            assert b1[i] == order[0] and b2[i] == order[1]
            assert d1[i] == D[order[0]]
            c, Dc, _ = oracle.bmu(W, X[i])
            assert c == order[0] and Dc == D[order[0]]


def test_map_csr_identity_matches_dense():
    C = bank_corpus(150, 400, seed=5)
    X = C.dense()
    W = init_rows(X, 30, 9) * np.float32(0.5) + np.float32(0.01)
    a = oracle.map_docs(W, X)
    b = oracle.map_docs_csr(W, C.indptr, C.indices, C.data)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    np.testing.assert_allclose(a[2], b[2], rtol=2e-7, atol=0)


def test_qerror_spec_examples():
    # S:230 single prototype equal to every row -> 0
    X = np.tile(uniform_matrix(1, 6, 3), (5, 1))
    assert oracle.qerror(X[:1], X) == 0.0
    # S:231 unit-norm rows, single zero prototype -> 1.0
    C = bank_corpus(50, 100, seed=1)
    assert abs(oracle.qerror(np.zeros((1, 100), np.float32), C.dense()) - 1.0) < 1e-6
    # S:232 rows {(0),(2)}, one prototype (1) -> 1.0
    assert oracle.qerror(np.array([[1.0]], np.float32), np.array([[0.0], [2.0]], np.float32)) == 1.0


def test_one_unit_map_degenerate():
    X = uniform_matrix(10, 4, 0)
    W1, log = oracle.train_online(X[:1], 1, 1, 1, X, epochs=2, alpha0=0.1, sigma0=0.5, seed=1)
    assert np.all(log == 0)
    assert oracle.topographic_error(W1, 1, 1, 1, X) == 0.0
    assert oracle.umatrix(W1, 1, 1, 1)[0] == 0.0


# ---------------------------------------------------------------- invariants
def test_zero_rate_leaves_weights_bit_identical():
    C = bank_corpus(60, 80, seed=2)
    X = C.dense()
    W0 = init_rows(X, 12, 2)
    W1, _ = oracle.train_online(W0, 3, 4, 1, X, epochs=3, alpha0=0.0, sigma0=2.0, seed=4)
    assert np.array_equal(W1, W0)


def test_t_range_resume_is_exact():
    C = bank_corpus(50, 60, seed=3)
    X = C.dense()
    W0 = init_rows(X, 9, 3)
    Wa, la = oracle.train_online(W0, 3, 3, 1, X, epochs=4, alpha0=0.1, sigma0=1.5, seed=11)
    Wb, lb1 = oracle.train_online(W0, 3, 3, 1, X, epochs=4, alpha0=0.1, sigma0=1.5, seed=11,
                                  t_begin=0, t_end=77)
    Wb, lb2 = oracle.train_online(Wb, 3, 3, 1, X, epochs=4, alpha0=0.1, sigma0=1.5, seed=11,
                                  t_begin=77, t_end=-1)
    assert np.array_equal(Wa, Wb) and np.array_equal(la, np.concatenate([lb1, lb2]))


def test_thread_count_invariance():
    C = bank_corpus(100, 3000, seed=4)
    X = C.dense()
    W0 = init_rows(X, 100, 4)
    nt = oracle.num_threads()
    try:
        oracle.set_num_threads(1)
        W1, l1 = oracle.train_online(W0, 10, 10, 1, X, epochs=1, alpha0=0.1, sigma0=5, seed=2)
        oracle.set_num_threads(max(nt, 4))
        W2, l2 = oracle.train_online(W0, 10, 10, 1, X, epochs=1, alpha0=0.1, sigma0=5, seed=2)
    finally:
        oracle.set_num_threads(nt)
    assert np.array_equal(W1, W2) and np.array_equal(l1, l2)


def test_eq1_contraction_and_convex_hull():
    # S:244 |x - w'| = (1 - h)|x - w| (up to fp32 rounding); S:247 convex hull
    rng = np.random.default_rng(0)
    W = rng.uniform(0, 1, (6, 9)).astype(np.float32)
    x = rng.uniform(0, 1, 9).astype(np.float32)
    W1 = oracle.update(W.copy(), 2, 3, 1, x, 4, 0.3, 1.2, math.inf)
    for u in range(6):
        g2 = oracle.lattice_g2(2, 3, 1, u, 4)
        h = float(np.float32(0.3 * math.exp(-g2 / (2 * 1.2 * 1.2))))
        np.testing.assert_allclose(np.abs(x - W1[u]), (1 - h) * np.abs(x - W[u]), atol=3e-7)
    C = bank_corpus(80, 50, seed=6)
    X = C.dense()
    W0 = init_rows(X, 16, 6)
    Wf, _ = oracle.train_online(W0, 4, 4, 1, X, epochs=5, alpha0=0.5, sigma0=2.0, seed=1)
    lo = np.minimum(X.min(0), W0.min(0))
    hi = np.maximum(X.max(0), W0.max(0))
    assert np.all(Wf >= lo - 1e-6) and np.all(Wf <= hi + 1e-6)


def test_fixed_point_identical_rows():
    # k identical rows, long schedule -> QE -> 0 within 1e-3
    row = uniform_matrix(1, 40, 8)
    X = np.tile(row, (7, 1))
    W0 = uniform_matrix(9, 40, 5) * np.float32(0.2)
    Wf, _ = oracle.train_online(W0, 3, 3, 1, X, epochs=300, alpha0=0.5, sigma0=1.5, seed=5, eps=0.0)
    assert oracle.qerror(Wf, X) <= 1e-3


def test_topology_preservation_three_clusters():
    # SPEC acceptance 5: intra-cluster BMU grid distance < inter
    wins = 0
    for seed in range(10):
        rng = np.random.default_rng(seed)
        centers = rng.uniform(0, 1, (3, 30)) * 4
        X = np.concatenate([c + 0.05 * rng.standard_normal((100, 30)) for c in centers]).astype(np.float32)
        lab = np.repeat(np.arange(3), 100)
        W0 = init_rows(X, 36, seed)
        Wf, _ = oracle.train_online(W0, 6, 6, 1, X, epochs=5, alpha0=0.1, sigma0=3.0, seed=seed)
        b1, _, _ = oracle.map_docs(Wf, X)
        sub = rng.choice(300, 90, replace=False)
        intra, inter = [], []
        for a in sub:
            for b in sub:
                if a < b:
                    g = math.sqrt(oracle.lattice_g2(6, 6, 1, b1[a], b1[b]))
                    (intra if lab[a] == lab[b] else inter).append(g)
        wins += np.mean(intra) < np.mean(inter)
    assert wins >= 9


def test_qe_improves_on_bank_corpus():
    # SPEC acceptance 6: final QE <= 0.8 x initial QE
    C = bank_corpus(200, 500, seed=1)
    X = C.dense()
    W0 = uniform_matrix(100, 500, 1) * np.float32(0.1)   # random initial codebook
    q0 = oracle.qerror(W0, X)
    Wf, _ = oracle.train_online(W0, 10, 10, 0, X, epochs=10, alpha0=0.1, sigma0=5.0, seed=1)
    assert oracle.qerror(Wf, X) <= 0.8 * q0


# ------------------------------------------------------------ batch SOM (R27)
def _f32(v):
    return struct.unpack("f", struct.pack("f", float(v)))[0]


def test_batch_closed_form_two_units():
    """1x2 map, two documents, one epoch, no cutoff: each document's BMU is
    the unit it sits next to, h = 1 at distance 0 and q = exp(-1/(2 sigma0^2))
    between the units (tau = 0, f = 1, floor sigma_min below sigma0), so
        W0' = (x1 + q x2) / (1 + q),  W1' = (q x1 + x2) / (q + 1),
    evaluated here in exact rational arithmetic from the fp64 q and rounded
    once to fp32."""
    sigma0 = 0.8
    x1 = np.array([0.125, 0.75, 0.3], np.float32)
    x2 = np.array([0.9, 0.0625, 0.55], np.float32)
    W0 = np.stack([x1 + np.float32(0.01), x2 - np.float32(0.01)]).astype(np.float32)
    W, b = oracle.train_batch(W0, 1, 2, 0, np.stack([x1, x2]), 1, sigma0, sigma_min=0.1, eps=0.0)
    q = Fraction(math.exp(-1.0 / (2.0 * sigma0 * sigma0)))
    for k in range(3):
        a1, a2 = Fraction(float(x1[k])), Fraction(float(x2[k]))
        assert W[0, k] == _f32((a1 + q * a2) / (1 + q))
        assert W[1, k] == _f32((q * a1 + a2) / (q + 1))
    assert list(b) == [0, 1]


def test_batch_reduces_to_kmeans_step():
    """With a neighbourhood radius below the smallest lattice distance
    (sigma0 = sigma_min = 0.1, eps = 1e-4: r2 = 0.18 < 1) only the BMU
    itself gets weight, and one epoch is one Lloyd (k-means) step: every
    unit becomes the mean of its documents, units without documents keep
    their weights.  Checked against numpy's own argmin and mean."""
    X = uniform_matrix(300, 7, 5).astype(np.float64)
    W0 = uniform_matrix(12, 7, 6)
    W0[11] += 5.0                     # far from every document: keeps its row
    d2 = ((X[:, None, :] - W0[None, :, :].astype(np.float64)) ** 2).sum(-1)
    srt = np.sort(d2, axis=1)
    assert ((srt[:, 1] - srt[:, 0]) / srt[:, 0]).min() > 1e-9      # no near ties
    c = d2.argmin(1)
    W, _ = oracle.train_batch(W0, 3, 4, 1, X.astype(np.float32), 1, 0.1, sigma_min=0.1, eps=1e-4)
    for u in range(12):
        if np.any(c == u):
            np.testing.assert_allclose(W[u], X[c == u].mean(0), rtol=0, atol=2e-7)
        else:
            assert np.array_equal(W[u], W0[u])
    assert np.array_equal(W[11], W0[11])


def test_batch_one_unit_is_the_mean_and_hull():
    X = uniform_matrix(200, 9, 8)
    W, b = oracle.train_batch(uniform_matrix(1, 9, 9), 1, 1, 0, X, 3, 2.0)
    np.testing.assert_allclose(W[0], X.astype(np.float64).mean(0), rtol=0, atol=2e-7)
    assert np.all(b == 0)
    W2, _ = oracle.train_batch(uniform_matrix(20, 9, 10), 4, 5, 1, X, 4, 2.5, eps=0.0)
    assert np.all(W2 >= X.min(0) - 1e-7) and np.all(W2 <= X.max(0) + 1e-7)   # weighted means


def test_batch_fixed_point_and_zero_epochs():
    x = uniform_matrix(1, 6, 11)
    X = np.repeat(x, 40, axis=0)
    W0 = uniform_matrix(9, 6, 12)
    W, _ = oracle.train_batch(W0, 3, 3, 0, X, 1, 1.5, eps=0.0)
    np.testing.assert_allclose(W, np.repeat(x, 9, axis=0), rtol=0, atol=1e-7)
    W3, _ = oracle.train_batch(W0, 3, 3, 0, X, 0, 1.5)
    assert np.array_equal(W3, W0)


# ------------------------------------------------- upstream (NEXT-3: R28-R31)
def _csr(rows, d):
    indptr = [0]
    col, val = [], []
    for r in rows:
        for t, c in sorted(r.items()):
            col.append(t)
            val.append(c)
        indptr.append(len(col))
    return (np.array(indptr, np.int64), np.array(col, np.int32), np.array(val, np.float32))


def test_tfidf_spec_examples():
    """IDF = ln(N/df) (ln 10 = 2.302585 for df = 1 of 10); a term in
    every document weighs 0; L2 normalisation [3,4] -> [0.6, 0.8], [5] -> [1]."""
    # doc0: a x3, b x4; doc1: c x1 -> idf(a) = idf(b) = idf(c) = ln 2
    rp, ci, va = _csr([{0: 3, 1: 4}, {2: 1}], 3)
    out, zr = oracle.tfidf_csr(rp, ci, va, 3)
    assert out.tolist() == [_f32(0.6), _f32(0.8), 1.0] and zr == 0
    # z (term 2) in every document: explicit zero; doc2 has only z: a zero row
    rp, ci, va = _csr([{0: 1, 2: 5}, {1: 2, 2: 1}, {2: 7}], 3)
    out, zr = oracle.tfidf_csr(rp, ci, va, 3)
    assert out.tolist() == [1.0, 0.0, 1.0, 0.0, 0.0] and zr == 1
    # ln 10: term 0 in one document of ten, together with term 1 (in all ten):
    rows = [{0: 2, 1: 1}] + [{1: 1, 2 + i: 1} for i in range(9)]
    rp, ci, va = _csr(rows, 11)
    out, _ = oracle.tfidf_csr(rp, ci, va, 11)
    assert out[0] == 1.0 and out[1] == 0.0          # 2 ln 10 / |2 ln 10|, and idf 0
    # two terms with different idf: doc0 = (a:1, b:1), a in 2 of 4 docs (ln 2), b in 1 (ln 4 = 2 ln 2)
    rp, ci, va = _csr([{0: 1, 1: 1}, {0: 1}, {2: 1}, {3: 1}], 4)
    out, _ = oracle.tfidf_csr(rp, ci, va, 4)
    assert out[0] == _f32(1 / math.sqrt(5)) and out[1] == _f32(2 / math.sqrt(5))


def test_pca_spec_examples_and_invariants():
    pc1, pc2, v1, v2, mu = oracle.pca_top2(np.array([[1, 0], [-1, 0], [2, 0], [-2, 0]], np.float64))
    assert np.allclose(v1, [1, 0]) and abs(pc2) < 1e-12 and abs(pc1 - 10.0 / 3.0) < 1e-12   # var = 10/3
    pc1, pc2, v1, v2, mu = oracle.pca_top2(np.array([[1, 0], [0, 1], [-1, 0], [0, -1]], np.float64))
    assert abs(pc1 - pc2) < 1e-12 and abs(pc1 - 2.0 / 3.0) < 1e-12
    X = uniform_matrix(50, 8, 3).astype(np.float64)
    pc1, pc2, v1, v2, mu = oracle.pca_top2(X)
    Xc = X - X.mean(0)
    # the eigenvalue is the variance of the projection (closed form), maximal over directions
    assert abs(np.var(Xc @ v1, ddof=1) - pc1) < 1e-12 and abs(np.var(Xc @ v2, ddof=1) - pc2) < 1e-12
    assert abs(v1 @ v2) < 1e-12 and abs(np.linalg.norm(v1) - 1) < 1e-12
    rng = np.random.default_rng(4)
    for _ in range(200):
        u = rng.normal(size=8)
        u /= np.linalg.norm(u)
        assert np.var(Xc @ u, ddof=1) <= pc1 + 1e-12
        u -= (u @ v1) * v1
        u /= np.linalg.norm(u)
        assert np.var(Xc @ u, ddof=1) <= pc2 + 1e-12       # second largest on the complement of v1
    assert v1[np.argmax(np.abs(v1))] > 0 and v2[np.argmax(np.abs(v2))] > 0          # R29 sign rule


def test_linear_init_plane_and_corners():
    X = uniform_matrix(80, 6, 5).astype(np.float64)
    pc1, pc2, v1, v2, mu = oracle.pca_top2(X)
    W = oracle.linear_init(4, 5, mu, v1, v2, pc1, pc2).astype(np.float64)
    B = np.stack([v1, v2])
    resid = (W - mu) - ((W - mu) @ B.T) @ B
    assert np.abs(resid).max() < 1e-6                       # on the principal plane (fp32 rounding)
    np.testing.assert_allclose(W[0], mu - math.sqrt(pc1) * v1 - math.sqrt(pc2) * v2, atol=1e-6)
    np.testing.assert_allclose(W[19], mu + math.sqrt(pc1) * v1 + math.sqrt(pc2) * v2, atol=1e-6)
    W1 = oracle.linear_init(1, 1, mu, v1, v2, pc1, pc2)
    assert np.array_equal(W1[0], mu.astype(np.float32))   # 1x1 map: the mean


def test_map_geometry_fig2_traces():
    """S:152-160 hand traces of Fig. 2."""
    assert oracle.map_geometry(400, 1.0, 1.0) == (9, 11, 20800)
    assert oracle.map_geometry(4, 1.0, 1.0) == (3, 3, 1808)
    r, c, _ = oracle.map_geometry(100, 10.0, 0.05)       # pc2 * munits < pc1 -> r = 1
    assert (r, c) == oracle.map_geometry(100, 1.0, 1.0)[:2] == (6, 8)


# ------------------------------------------- round 2: discriminating pins
@pytest.mark.parametrize("topo,key", [(0, "rect"), (1, "hex")])
def test_topographic_error_nonzero_closed_form(topo, key):
    """A non-zero TE fixed by hand (tests/golden/te_2x2_docs.json): the BMU
    pairs, which pairs are lattice-adjacent, TE = k/n exactly, and the zero
    row left out of both QE and TE."""
    g = _gold("te_2x2_docs.json")
    W = np.array(g["W"], np.float32)
    X = np.array(g["docs"], np.float32)
    b1, b2, d1 = oracle.map_docs(W, X)
    assert [[int(a), int(b)] for a, b in zip(b1, b2)] == g["bmu_pairs"]
    np.testing.assert_allclose(d1, [min(r) for r in g["D_hand"]], rtol=1e-6, atol=1e-7)
    nonadj = {tuple(sorted(p)) for p in g[key]["nonadjacent_pairs"]}
    for u in range(4):
        for v in range(u + 1, 4):
            assert (oracle.lattice_g2(2, 2, topo, u, v) != 1.0) == ((u, v) in nonadj)
    keep = oracle.keep_mask(len(X), oracle.nonzero_rows(X))
    assert keep.tolist() == g["keep"]
    k, n = g[key]["te"]
    assert oracle.topographic_error_from_bmus(2, 2, topo, b1, b2, keep) == k / n
    assert oracle.topographic_error(W, 2, 2, topo, X) == k / n
    k2, n2 = g[key]["te_if_zero_row_counted"]
    assert oracle.topographic_error_from_bmus(2, 2, topo, b1, b2) == k2 / n2
    qe = (0.4 + 1.0 + 0.3 + 2 * math.sqrt(6.85) + math.sqrt(12.5)) / 6
    assert abs(oracle.qerror(W, X) - qe) < 1e-6


def test_decay_kinds_mid_schedule_closed_forms():
    """The three decay forms of R1 at tau = 1/2 and 1/4 with k = ln 100:
    Gaussian f = 100^(-tau^2), linear f = 1 - 0.99 tau, exponential
    f = 100^(-tau) — alpha_t = alpha0 f and sigma_t = sigma0 f (above the
    floor).  A squared tau in the linear or exponential kind, or a missing
    square in the Gaussian one, fails here."""
    T = 1000
    want = {0: {500: 10 ** -0.5, 250: 100 ** (-1 / 16)},
            1: {500: 0.505, 250: 1 - 0.99 / 4},
            2: {500: 0.1, 250: 100 ** -0.25}}
    for kind, pts in want.items():
        for t, f in pts.items():
            a, s, r2 = oracle.schedule(t, T, 1.0, 40.0, kind=kind)
            assert math.isclose(a, f, rel_tol=1e-14), (kind, t, a, f)
            assert math.isclose(s, 40.0 * f, rel_tol=1e-14)
            assert math.isclose(r2, 2 * (40.0 * f) ** 2 * math.log(1e4), rel_tol=1e-13)


def test_zero_rows_never_drawn_and_not_scored():
    """all-zero rows stay in X but are excluded from the draws:
    draw t takes the i_t-th non-zero row, i_t = sample_index(seed, t, n_nz).
    So X with zero rows inserted trains exactly like the zero-free X when T
    is the same (epochs * n = epochs' * n_nz) — and a corpus of zero rows
    only is EmptyData."""
    C = bank_corpus(40, 60, seed=9)
    Xnz = C.dense()
    X = np.zeros((60, 60), np.float32)
    pos = np.sort(np.random.default_rng(1).choice(60, 40, replace=False))
    X[pos] = Xnz
    assert np.array_equal(oracle.nonzero_rows(X), pos)
    W0 = init_rows(Xnz, 9, 2)
    # T = 2 * 60 = 3 * 40 = 120 steps on both
    Wa, la = oracle.train_online(W0, 3, 3, 1, X, epochs=2, alpha0=0.1, sigma0=1.5, seed=7)
    Wb, lb = oracle.train_online(W0, 3, 3, 1, Xnz, epochs=3, alpha0=0.1, sigma0=1.5, seed=7)
    assert np.array_equal(Wa, Wb) and np.array_equal(la, lb)
    assert oracle.qerror(Wa, X) == oracle.qerror(Wa, Xnz)
    assert oracle.topographic_error(Wa, 3, 3, 1, X) == oracle.topographic_error(Wa, 3, 3, 1, Xnz)
    with pytest.raises(ValueError, match="EmptyData"):
        oracle.train_online(W0, 3, 3, 1, np.zeros((5, 60), np.float32), epochs=1, alpha0=0.1, sigma0=1.5, seed=7)
    # CSR: explicit zeros do not make a row non-zero
    rp = np.array([0, 2, 3, 3], np.int64)
    va = np.array([0.5, 0.0, 0.0], np.float32)
    assert oracle.nonzero_rows_csr(rp, va).tolist() == [0]


def test_csr_training_equals_dense_training():
    """or_train_online_csr densifies x_t per step: the same trajectory as the
    dense oracle on the dense copy, including a corpus with zero rows (an
    explicit-zero CSR entry does not make a row non-zero)."""
    C = bank_corpus(80, 120, seed=12)
    W0 = init_rows(C.dense(), 16, 3)
    Wa, la = oracle.train_online(W0, 4, 4, 1, C.dense(), epochs=3, alpha0=0.2, sigma0=2.0, seed=5)
    Wb, lb = oracle.train_online_csr(W0, 4, 4, 1, C.indptr, C.indices, C.data, epochs=3, alpha0=0.2, sigma0=2.0,
                                     seed=5)
    assert np.array_equal(Wa, Wb) and np.array_equal(la, lb)
    # zero rows: rows 3 and 7 emptied (row 7 keeps an explicit 0.0 entry)
    rp, ci, va = C.indptr.copy(), C.indices.copy(), C.data.copy()
    va[rp[3]:rp[4]] = 0.0
    va[rp[7]:rp[8]] = 0.0
    X = C.dense()
    X[3] = 0.0
    X[7] = 0.0
    Wa, la = oracle.train_online(W0, 4, 4, 1, X, epochs=2, alpha0=0.2, sigma0=2.0, seed=6)
    Wb, lb = oracle.train_online_csr(W0, 4, 4, 1, rp, ci, va, epochs=2, alpha0=0.2, sigma0=2.0, seed=6)
    assert np.array_equal(Wa, Wb) and np.array_equal(la, lb)


def test_permutation_sampler_is_a_permutation_per_epoch():
    """R8b (per-epoch permutation option of P:162's random
    selection): within each epoch of m steps every index of [0, m) is drawn
    exactly once (brute force over several m, including powers of two and
    their neighbours, where the cycle-walking domain is tight or loose), and
    consecutive epochs use different orders."""
    for m in (1, 2, 3, 4, 5, 7, 8, 9, 31, 32, 33, 100, 1000, 5000):
        orders = []
        for e in range(3):
            draws = [oracle.perm_index(42, e * m + p, m) for p in range(m)]
            assert sorted(draws) == list(range(m)), (m, e)
            orders.append(draws)
        if m >= 5:
            assert orders[0] != orders[1] and orders[1] != orders[2]
    # seed-dependence and counter-based resume: the same t gives the same draw
    assert [oracle.perm_index(1, t, 100) for t in range(100)] != [oracle.perm_index(2, t, 100) for t in range(100)]
    assert oracle.perm_index(7, 12345, 5000) == oracle.perm_index(7, 12345, 5000)


def test_permutation_sampling_training_draws_every_row_once():
    """Online training with R8b on a 1x1 map: the single prototype's
    trajectory w <- fmaf(h, RN32(x - w), w) (Eq. 1, R11; h = RN32(alpha_t)
    since g2 = 0) is replayed by hand along the draws perm_index gives over
    the non-zero rows (zero rows are never drawn); the first epoch
    draws every non-zero row once."""
    rng = np.random.default_rng(3)
    X = rng.random((9, 4)).astype(np.float32)
    X[[2, 5]] = 0.0                       # zero rows: drawable rows m = 7
    nz = [i for i in range(9) if X[i].any()]
    draws = [nz[oracle.perm_index(11, t, len(nz))] for t in range(len(nz))]
    assert sorted(draws) == nz
    # the oracle's training with sampling=1 follows exactly these draws: with
    # a 1x1 map and eps = 0 the prototype after step t is
    # fmaf(alpha_t, x - w, w), so replay it here with the same arithmetic
    W0 = np.zeros((1, 4), np.float32)
    W, log = oracle.train_online(W0, 1, 1, 0, X, 1, 0.5, 1.0, 11, eps=0.0, sampling=1)
    T = X.shape[0]                    # T = epochs * n steps (R7); epochs of R8b are m = 7 steps
    w = W0[0].astype(np.float64)
    for t in range(T):
        a, _, _ = oracle.schedule(t, T, 0.5, 1.0, eps=0.0)
        h = float(np.float32(a))      # g2 = 0: h = RN32(alpha) (R4)
        x = X[nz[oracle.perm_index(11, t, len(nz))]].astype(np.float64)
        diff = (x.astype(np.float32) - w.astype(np.float32)).astype(np.float64)   # RN32(x - w) (R11)
        w = np.float32(h * diff + w).astype(np.float64)   # fmaf: one rounding of the exact h*diff + w
    assert np.array_equal(W[0], w.astype(np.float32))
