"""Kernel 10 (train_tier.cu): online training with the map held in the SM's
storage tiers — rows in tensor memory (tcgen05.ld/st), rows in shared
memory, the rest streamed through a chunked TMA ring — against the dense
oracle.  Bar (BASELINE.json north_star): BMU log identical, weights within
1e-4 (observed bit-identical: the update is Eq. 1's arithmetic, the
distances R10 via the sparse identity R25).  Covers every chunk count KJ
the kernel instantiates (4..8), maps with few and many streamed rows per CTA
(grid forced small), ring depth 2 and no shared-memory rows, the late
schedule (few updated units: the speculative sparse terms carry most keys)
with a resume split, the no-cutoff schedule, zero rows and dense rows
converted on the device."""
import numpy as np
import pytest

import oracle
from synth import bank_corpus, init_rows

pytestmark = pytest.mark.gpu
KERNEL_TIER = 10


@pytest.fixture(autouse=True)
def _tier_on(monkeypatch):
    monkeypatch.setenv("SOM_TRAIN_TIER", "1")
    monkeypatch.setenv("SOM_TIER_HANDOVER", "0")   # kernel 10 for the whole range


@pytest.fixture(scope="module")
def som():
    from paper_1905_09598_b200 import som as s
    s.lib()
    return s


def _run(som, rows, cols, C, W0, epochs, sigma0, seed, t_end=-1, cutoff=1e-4, csr=True, t_split=None, topo=1,
         grid=0):
    T = epochs * C.n
    te = T if t_end < 0 else t_end
    with som.SOM(rows, cols, C.d, topo) as m:
        if grid:
            som.som_set_train_grid(m.h, grid)
        m.set_weights(W0)
        log = np.full(te, -7, np.int32)
        cuts = [0, te] if t_split is None else [0, t_split, te]
        for a, b in zip(cuts, cuts[1:]):
            if csr:
                m.train_online_csr(C.indptr, C.indices, C.data, C.n, epochs, alpha0=0.1, sigma0=sigma0, seed=seed,
                                   cutoff=cutoff, t_begin=a, t_end=b, bmu_log=log[a:b])
            else:
                m.train_online(C.dense(), epochs, alpha0=0.1, sigma0=sigma0, seed=seed, cutoff=cutoff, t_begin=a,
                               t_end=b, bmu_log=log[a:b])
        g, k = som.som_last_train_config(m.h)
        W = m.get_weights()
    return W, log, k


def _check(W, log, Wo, logo):
    bad = np.flatnonzero(log != logo)
    assert bad.size == 0, f"first BMU mismatch at step {bad[0]} of {log.size}"
    assert np.abs(W.astype(np.float64) - Wo).max() <= 1e-4
    return bool(np.array_equal(W, Wo))


@pytest.mark.parametrize("rows,cols,d,n,steps,grid", [
    (20, 20, 6000, 1200, 400, 16),      # KJ 4, 25 units per CTA: 8 TMEM + smem rows + a long stream
    (20, 20, 7600, 1200, 400, 20),      # KJ 5
    (24, 24, 9000, 1200, 300, 24),      # KJ 6
    (50, 50, 10000, 3000, 300, 0),      # KJ 7: the c3 map (148 CTAs, 16-17 units each)
    (30, 30, 12000, 1000, 300, 40),     # KJ 8 (ragged last chunk: 3000 float4 = 7 x 384 + 312)
    (40, 40, 7000, 800, 300, 148),      # 1,600 units on 148 CTAs: 10-11 rows each, no streamed row
])
@pytest.mark.parametrize("ndw", ["16", "12"])
def test_tier_matches_oracle(som, monkeypatch, rows, cols, d, n, steps, grid, ndw):
    """KJ counts are those of 12 data warps; SOM_TIER_NDW=16 (the default
    where a row needs 4-5 float4 chunks per thread of 16 warps) covers
    d = 7600 ... 10000 with 16 data warps and 128-column TMEM groups."""
    monkeypatch.setenv("SOM_TIER_NDW", ndw)
    C = bank_corpus(n, d, seed=d + n)
    X = C.dense()
    W0 = init_rows(X, rows * cols, 31)
    sigma0 = max(rows, cols) / 2.0
    W, log, k = _run(som, rows, cols, C, W0, 1, sigma0, 3, t_end=steps, grid=grid)
    assert k == KERNEL_TIER, k
    Wo, logo = oracle.train_online(W0, rows, cols, 1, X, 1, 0.1, sigma0, 3, t_end=steps)
    bit = _check(W, log, Wo, logo)
    print(f" [{rows}x{cols} d={d} grid={grid}: bit-identical W {bit}]", end="")


@pytest.mark.parametrize("ring,nsm", [("2", "0"), ("5", "1"), ("16", "4")])
def test_tier_ring_depths_and_late_schedule(som, monkeypatch, ring, nsm):
    """Ring depths 2..16 chunks and 0..4 shared-memory rows; the whole
    schedule on a small corpus (the neighbourhood shrinks to sigma_min: few
    rows per step, the speculative sparse terms carry most units), resumed
    across a split."""
    monkeypatch.setenv("SOM_TIER_RING", ring)
    monkeypatch.setenv("SOM_TIER_NSM", nsm)
    C = bank_corpus(300, 8000, seed=77)
    X = C.dense()
    W0 = init_rows(X, 40 * 40, 77)
    W, log, k = _run(som, 40, 40, C, W0, 3, 20.0, 5, t_split=517, grid=64)
    assert k == KERNEL_TIER
    Wo, logo = oracle.train_online(W0, 40, 40, 1, X, 3, 0.1, 20.0, 5)
    _check(W, log, Wo, logo)


def test_tier_no_cutoff_and_dense_input(som):
    """cutoff 0 (plain Eq. 1 on every unit every step: only the dense pass)
    and dense rows converted to CSR on the device (AUTO)."""
    C = bank_corpus(500, 6000, seed=78)
    X = C.dense()
    W0 = init_rows(X, 1600, 78)
    W, log, k = _run(som, 40, 40, C, W0, 1, 20.0, 6, t_end=250, cutoff=0.0, csr=False, grid=100)
    assert k == KERNEL_TIER
    Wo, logo = oracle.train_online(W0, 40, 40, 1, X, 1, 0.1, 20.0, 6, eps=0.0, t_end=250)
    _check(W, log, Wo, logo)


def test_tier_zero_rows_rect(som):
    C = bank_corpus(400, 6400, seed=79)
    rp, ci, va = C.indptr, C.indices, C.data.copy()
    for i in range(0, C.n, 9):
        va[rp[i]:rp[i + 1]] = 0.0
    X = C.dense()
    X[::9] = 0.0
    Cz = type(C)(C.n, C.d, rp, ci, va, C.topic)
    W0 = init_rows(np.delete(X, np.arange(0, C.n, 9), 0), 1600, 79)
    W, log, k = _run(som, 40, 40, Cz, W0, 2, 20.0, 8, t_end=600, topo=0, grid=100)
    assert k == KERNEL_TIER
    Wo, logo = oracle.train_online(W0, 40, 40, 0, X, 2, 0.1, 20.0, 8, t_end=600)
    _check(W, log, Wo, logo)


def test_tier_c3_late_window_equals_kernel4(som, monkeypatch):
    """c3 (50x50 hex, 50,000 x 10,000): 2,000 steps late in the schedule
    (sigma at its floor) from the same weights, kernel 10 vs kernel 4: BMU
    logs and weights identical bit for bit."""
    import torch
    from synth import CONFIGS
    cfg = CONFIGS["c3"]
    C = bank_corpus(cfg["n"], cfg["d"], seed=301)
    rp, ci, va = (torch.from_numpy(a).cuda() for a in (C.indptr, C.indices, C.data))
    m = som.SOM(50, 50, cfg["d"], 1)
    som.som_init_random_csr(m.h, rp, ci, va, C.n, 1301)
    W0 = m.get_weights()
    t0, t1 = 470000, 472000
    out = {}
    for tier in ("0", "1"):
        monkeypatch.setenv("SOM_TRAIN_TIER", tier)
        m.set_weights(W0)
        som.som_train_online_csr(m.h, rp, ci, va, C.n, cfg["epochs"], 0.1, cfg["sigma0"], None, 1, t0, t1, None)
        k = som.som_last_train_config(m.h)[1]
        log = torch.empty(t1 - t0, dtype=torch.int32, device="cuda")
        som.som_train_online_csr(m.h, rp, ci, va, C.n, cfg["epochs"], 0.1, cfg["sigma0"], None, 1, t1, t1 + 2000, log)
        out[tier] = (k, m.get_weights(), log.cpu().numpy())
    m.close()
    assert out["0"][0] == 4 and out["1"][0] == KERNEL_TIER
    assert np.array_equal(out["0"][2], out["1"][2])
    assert np.array_equal(out["0"][1], out["1"][1])


@pytest.mark.parametrize("cover", ["0.4", "0.9", "0.15"])
def test_tier_handover_to_kernel4(som, monkeypatch, cover):
    """AUTO with SOM_TRAIN_TIER=1: kernel 10 while the cutoff disk holds at
    least SOM_TIER_COVER of the units on average over winner positions,
    kernel 4 from the first step where it does not (kernel id 11, two
    launches): the whole schedule against the oracle, at the default
    threshold and at two other split points."""
    monkeypatch.setenv("SOM_TIER_HANDOVER", "1")
    monkeypatch.setenv("SOM_TIER_COVER", cover)
    C = bank_corpus(300, 8000, seed=91)
    X = C.dense()
    W0 = init_rows(X, 40 * 40, 91)
    W, log, k = _run(som, 40, 40, C, W0, 3, 20.0, 9, grid=64)
    assert k == 11, k
    Wo, logo = oracle.train_online(W0, 40, 40, 1, X, 3, 0.1, 20.0, 9)
    _check(W, log, Wo, logo)


@pytest.mark.parametrize("tier,t0", [("1", 0), ("0", 460000)])
def test_c3_exchange_variants_identical(som, monkeypatch, tier, t0):
    """The three in-GPU exchange variants (som_internal.h: 0 tagged
    all-gather, 1 atomic max + arrival counter, 2 the counter-hinted
    all-gather, the default at G = 148) on c3 windows of kernel 10 (early,
    every unit updated) and kernel 4 (late): the same BMU log and weights
    bit for bit."""
    import torch
    from synth import CONFIGS
    cfg = CONFIGS["c3"]
    C = bank_corpus(cfg["n"], cfg["d"], seed=301)
    rp, ci, va = (torch.from_numpy(a).cuda() for a in (C.indptr, C.indices, C.data))
    monkeypatch.setenv("SOM_TRAIN_TIER", tier)
    m = som.SOM(50, 50, cfg["d"], 1)
    som.som_init_random_csr(m.h, rp, ci, va, C.n, 1301)
    W0 = m.get_weights()
    out = {}
    for mode in ("0", "1", "2"):
        monkeypatch.setenv("SOM_XCHG_ATOMIC", mode)
        m.set_weights(W0)
        log = torch.empty(1500, dtype=torch.int32, device="cuda")
        som.som_train_online_csr(m.h, rp, ci, va, C.n, cfg["epochs"], 0.1, cfg["sigma0"], None, 1, t0, t0 + 1500, log)
        out[mode] = (som.som_last_train_config(m.h), m.get_weights(), log.cpu().numpy())
    m.close()
    assert out["2"][0][0] == 148 and out["2"][0][1] == (KERNEL_TIER if tier == "1" else 4), out["2"][0]
    for mode in ("0", "1"):
        assert np.array_equal(out[mode][2], out["2"][2]), f"mode {mode}: BMU log differs"
        assert np.array_equal(out[mode][1], out["2"][1]), f"mode {mode}: weights differ"
