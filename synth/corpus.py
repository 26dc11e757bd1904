"""Seeded synthetic "four-bank-complaint-shaped" TF-IDF corpora.

Input generation only: this module holds none of the SOM arithmetic and is
the one module both the oracle side (tests) and the product side (bench,
tests) draw inputs from.  Recipe:

* Shape: the paper's Table 1 gives only documents x features
  (440-676 docs x 3,917-4,545 terms).  Configs c1-c5 (BASELINE.json) set n, V.
* Topics: K = 5 product topics (loans, credit cards, ATM, account charges,
  mobile/internet banking), each with 3 sub-topics (e.g. car
  loans P:246, CPP P:278).  A topic owns a block of V/(2K) terms.
* Tokens: with probability ``lam`` from the document's topic block (a
  Zipf(1.05) over ranks; the top 20 % of ranks are shared by the sub-topics,
  the rest are permuted per sub-topic), otherwise from a Zipf(1.05)
  background over all V terms.
* Length: lognormal with mean 60 tokens, sigma_log 0.6 (not in the paper).
* Weights: raw term counts, IDF = ln(n/df) (Eq. 2, natural
  log as S:66), rows L2-normalised in fp64, stored as fp32.
  A row that ends up all-zero (every term has idf 0) is redrawn, so the
  corpus never holds a zero row (reading R17).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Corpus:
    n: int
    d: int
    indptr: np.ndarray   # int64 [n+1]
    indices: np.ndarray  # int32 [nnz], ascending within a row
    data: np.ndarray     # float32 [nnz], > 0
    topic: np.ndarray    # int32 [n]

    def dense(self) -> np.ndarray:
        X = np.zeros((self.n, self.d), dtype=np.float32)
        rows = np.repeat(np.arange(self.n), np.diff(self.indptr))
        X[rows, self.indices] = self.data
        return X

    @property
    def nnz(self) -> int:
        return int(self.indices.shape[0])


def _zipf_cdf(m: int, s: float) -> np.ndarray:
    w = 1.0 / np.arange(1, m + 1, dtype=np.float64) ** s
    c = np.cumsum(w)
    return c / c[-1]


def _draw_tokens(rng, n, V, topic, sub, K, n_sub, lam, mean_len, sigma_log, s, perms, bg_perm):
    B = max(1, V // (2 * K))
    mu = np.log(mean_len) - 0.5 * sigma_log ** 2
    L = np.maximum(3, np.rint(rng.lognormal(mu, sigma_log, size=n))).astype(np.int64)
    doc = np.repeat(np.arange(n, dtype=np.int64), L)
    M = doc.shape[0]
    from_topic = rng.random(M) < lam
    term = np.empty(M, dtype=np.int64)
    # topic tokens
    cdf_b = _zipf_cdf(B, s)
    nt = int(from_topic.sum())
    r = np.minimum(np.searchsorted(cdf_b, rng.random(nt), side="right"), B - 1)
    td = doc[from_topic]
    k = topic[td]
    term[from_topic] = (k * B) % V + perms[k, sub[td], r]
    # background tokens
    cdf_v = _zipf_cdf(V, s)
    nb = M - nt
    rb = np.minimum(np.searchsorted(cdf_v, rng.random(nb), side="right"), V - 1)
    term[~from_topic] = bg_perm[rb]
    return doc, np.minimum(term, V - 1)


def bank_corpus(n_docs: int, n_terms: int, seed: int, n_topics: int = 5, n_sub: int = 3,
                lam: float = 0.3, mean_len: float = 60.0, sigma_log: float = 0.6,
                zipf_s: float = 1.05) -> Corpus:
    """Generate a TF-IDF, L2-normalised document-term matrix (CSR)."""
    n, V, K = int(n_docs), int(n_terms), int(n_topics)
    if n < 1 or V < 1:
        raise ValueError("n_docs and n_terms must be >= 1")
    rng = np.random.default_rng(np.random.SeedSequence([0x50A1, seed]))
    B = max(1, V // (2 * K))
    core = max(1, B // 5)
    perms = np.empty((K, n_sub, B), dtype=np.int64)
    for k in range(K):
        for j in range(n_sub):
            tail = core + rng.permutation(B - core) if B > core else np.empty(0, np.int64)
            perms[k, j] = np.concatenate([np.arange(core), tail])[:B]
    bg_perm = rng.permutation(V)
    topic = rng.integers(0, K, size=n).astype(np.int64)
    sub = rng.integers(0, n_sub, size=n).astype(np.int64)

    doc, term = _draw_tokens(rng, n, V, topic, sub, K, n_sub, lam, mean_len, sigma_log,
                             zipf_s, perms, bg_perm)
    for _attempt in range(64):
        key = doc * V + term
        ukey, cnt = np.unique(key, return_counts=True)
        pd, pt = ukey // V, ukey % V
        df = np.bincount(pt, minlength=V)
        idf = np.zeros(V, dtype=np.float64)
        nz = df > 0
        idf[nz] = np.log(n / df[nz])                 # Eq. 2, natural log
        w = cnt.astype(np.float64) * idf[pt]
        keep = w > 0.0
        pd, pt, w = pd[keep], pt[keep], w[keep]
        sq = np.bincount(pd, weights=w * w, minlength=n)
        zero = np.flatnonzero(sq == 0.0)
        if zero.size == 0:
            break
        # redraw the zero rows' tokens and try again
        d2, t2 = _draw_tokens(rng, zero.size, V, topic[zero], sub[zero], K, n_sub, lam,
                              mean_len, sigma_log, zipf_s, perms, bg_perm)
        keep_tok = ~np.isin(doc, zero)
        doc = np.concatenate([doc[keep_tok], zero[d2]])
        term = np.concatenate([term[keep_tok], t2])
    else:
        raise RuntimeError("could not draw a corpus without zero rows")
    norm = np.sqrt(sq)
    data = (w / norm[pd]).astype(np.float32)
    counts = np.bincount(pd, minlength=n)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    return Corpus(n=n, d=V, indptr=indptr, indices=pt.astype(np.int32), data=data,
                  topic=topic.astype(np.int32))


def init_rows(X: np.ndarray, N: int, seed: int) -> np.ndarray:
    """Seeded codebook for tests: N rows of X, without replacement when N <= n."""
    rng = np.random.default_rng(np.random.SeedSequence([0x1A17, seed]))
    n = X.shape[0]
    idx = rng.choice(n, size=N, replace=N > n)
    return np.ascontiguousarray(X[idx], dtype=np.float32)


def uniform_matrix(n: int, d: int, seed: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    rng = np.random.default_rng(np.random.SeedSequence([0x0F32, seed]))
    return rng.uniform(lo, hi, size=(n, d)).astype(np.float32)


# Workload presets (BASELINE.json configs; epochs for c3/c4 and topology for
# c3-c5 are DESIGN.md proposals).  topo: 0 = rectangular, 1 = hexagonal.
CONFIGS = {
    "c1": dict(rows=10, cols=10, topo=0, n=200, d=500, epochs=10, sigma0=5.0),
    "c2": dict(rows=20, cols=20, topo=1, n=5000, d=3000, epochs=100, sigma0=10.0),
    "c3": dict(rows=50, cols=50, topo=1, n=50000, d=10000, epochs=10, sigma0=25.0),
    "c4": dict(rows=100, cols=100, topo=1, n=200000, d=20000, epochs=2, sigma0=50.0),
    "c5": dict(rows=100, cols=100, topo=1, n=10_000_000, d=20000, epochs=0, sigma0=50.0),
}
