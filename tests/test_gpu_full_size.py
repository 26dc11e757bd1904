"""Full-size run of BASELINE.json configs[4] (c5): batch BMU mapping of
10,000,000 CSR documents x 20,000 terms onto a 100x100 map on one B200, in
the launch configuration bench.py times (som_map_csr, AUTO = the exact sparse
path, chunked by the library).  The oracle checks sampled documents one by
one (its sparse-identity mapping, or_map_csr) and the error sums are checked
against the per-document outputs.

The corpus is generated as 50 seeded blocks of 200,000 documents (same
generator, same shapes) in parallel host processes."""
import multiprocessing as mp

import numpy as np
import pytest

import oracle
from synth import bank_corpus

pytestmark = pytest.mark.gpu

N_DOCS, D, BLOCK = 10_000_000, 20_000, 200_000


def _block(k):
    C = bank_corpus(BLOCK, D, seed=9000 + k)
    return C.indptr, C.indices, C.data


@pytest.fixture(scope="module")
def corpus():
    with mp.get_context("fork").Pool(min(16, mp.cpu_count())) as pool:
        parts = pool.map(_block, range(N_DOCS // BLOCK))
    nnz = sum(p[1].size for p in parts)
    rowptr = np.empty(N_DOCS + 1, np.int64)
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float32)
    rowptr[0] = 0
    r, o = 0, 0
    for ip, ci, va in parts:
        m = ip.size - 1
        rowptr[r + 1:r + m + 1] = ip[1:] + o
        col[o:o + ci.size] = ci
        val[o:o + va.size] = va
        r += m
        o += ci.size
    return rowptr, col, val


def test_c5_full_size_mapping(corpus):
    import torch

    from paper_1905_09598_b200 import som
    rowptr, col, val = corpus
    W = (0.5 * bank_corpus(10000, D, seed=8999).dense() + 0.5 / np.sqrt(D)).astype(np.float32)
    rp, ci, va = (torch.from_numpy(a).cuda() for a in (rowptr, col, val))
    b1 = torch.empty(N_DOCS, dtype=torch.int32, device="cuda")
    b2 = torch.empty(N_DOCS, dtype=torch.int32, device="cuda")
    d1 = torch.empty(N_DOCS, dtype=torch.float32, device="cuda")
    with som.SOM(100, 100, D, 1) as m:
        m.set_weights(W)
        som.som_map_csr(m.h, rp, ci, va, N_DOCS, b1, b2, d1)
        ms, units, launches = som.som_last_stats(m.h)
        qe, te = som.som_errors_csr(m.h, rp, ci, va, N_DOCS)
    b1, b2, d1 = (t.cpu().numpy() for t in (b1, b2, d1))
    # sampled documents, one by one through the oracle
    rng = np.random.default_rng(5)
    idx = np.sort(rng.choice(N_DOCS, size=2000, replace=False))
    sp = np.zeros(idx.size + 1, np.int64)
    sp[1:] = np.cumsum(rowptr[idx + 1] - rowptr[idx])
    sc = np.concatenate([col[rowptr[i]:rowptr[i + 1]] for i in idx])
    sv = np.concatenate([val[rowptr[i]:rowptr[i + 1]] for i in idx])
    ob1, ob2, od1, m12, m23 = oracle.map_docs_csr(W, sp, sc, sv, want_margins=True)
    ok = m12 > 1e-6
    assert ok.mean() > 0.98
    assert np.array_equal(b1[idx][ok], ob1[ok])
    ok2 = ok & (m23 > 1e-6)
    assert np.array_equal(b2[idx][ok2], ob2[ok2])
    err = np.abs(d1[idx].astype(np.float64) - od1)
    assert np.all(err <= 2.0 ** -23 * od1 + 1e-14)
    # error sums over all 10M documents agree with the per-document outputs
    assert abs(qe - np.sqrt(d1.astype(np.float64)).mean()) <= 1e-9
    assert np.all(b1 >= 0) and np.all(b1 < 10000) and np.all(b2 != b1)
    print(f" [c5 full size: {N_DOCS} docs in {ms:.0f} ms = {N_DOCS / ms * 1e3 / 1e6:.2f} M docs/s, "
          f"{launches} launches, QE {qe:.6f}, TE {te:.4f}]", end="")


def test_c3_full_schedule_tail():
    """BASELINE.json configs[2] (c3: 50x50 hex, 50,000 x 10,000 TF-IDF,
    10 epochs = 500,000 steps) trained on the GPU in the bench's launch
    configuration; the last 100 steps (smallest radius, alpha near alpha0/100)
    are re-run by the oracle from the GPU's weights at step 499,900 (the
    t-range resume is exact, tests/test_gpu_parity.py) and must give the same
    BMU log and weights; the final QE must beat the initial codebook's."""
    from paper_1905_09598_b200 import som
    from synth import init_rows
    C = bank_corpus(50000, 10000, seed=3)
    X = C.dense()
    W0 = init_rows(X, 2500, 1003)
    T, t0 = 500000, 499900
    with som.SOM(50, 50, 10000, 1) as m:
        m.set_weights(W0)
        qe0, _ = m.errors(X)
        m.train_online(X, epochs=10, alpha0=0.1, sigma0=25.0, seed=3, t_end=t0)
        ms, units, _ = som.som_last_stats(m.h)
        Wt0 = m.get_weights()
        log = np.empty(T - t0, np.int32)
        m.train_online(X, epochs=10, alpha0=0.1, sigma0=25.0, seed=3, t_begin=t0, bmu_log=log)
        W = m.get_weights()
        qe1, te1 = m.errors(X)
    Wo, logo = oracle.train_online(Wt0, 50, 50, 1, X, 10, 0.1, 25.0, 3, t_begin=t0)
    assert np.array_equal(log, logo)
    assert np.abs(W.astype(np.float64) - Wo).max() <= 1e-4
    assert qe1 < qe0
    print(f" [c3 full schedule: {units} steps in {ms / 1e3:.2f} s = {1e3 * ms / units:.1f} us/step, "
          f"QE {qe0:.4f} -> {qe1:.4f}, TE {te1:.4f}]", end="")
