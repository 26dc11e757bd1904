"""Parity of the CUDA path (libsom via the C ABI) against the oracle.

Bar (BASELINE.json north_star): BMU sequences and mapping indices identical;
weights and errors within 1e-4 max-abs; integer outputs bit-exact."""
import math

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


def _train_both(som, rows, cols, topo, X, W0, epochs, alpha0, sigma0, seed, mode=0, kind=0, cutoff=1e-4,
                t_begin=0, t_end=-1, k=math.log(100.0)):
    n, d = X.shape
    with som.SOM(rows, cols, d, topo) as m:
        som.som_set_train_mode(m.h, mode)
        m.set_weights(W0)
        T = epochs * n
        te = T if t_end < 0 else t_end
        log = np.full(max(te - t_begin, 0), -7, np.int32)
        m.train_online(X, epochs=epochs, alpha0=alpha0, sigma0=sigma0, seed=seed, kind=kind, cutoff=cutoff,
                       t_begin=t_begin, t_end=t_end, bmu_log=log, k=k)
        W = m.get_weights()
    Wo, logo = oracle.train_online(W0, rows, cols, topo, X, epochs, alpha0, sigma0, seed, kind=kind, k=k,
                                   eps=cutoff, t_begin=t_begin, t_end=t_end)
    return W, log, Wo, logo


def _assert_train(W, log, Wo, logo):
    assert np.array_equal(log, logo), f"first BMU mismatch at step {np.flatnonzero(log != logo)[:1]}"
    err = np.abs(W.astype(np.float64) - Wo).max() if W.size else 0.0
    assert err <= W_TOL, err


# --------------------------------------------------------------- training
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_c1_full_training(som, seed):
    """c1: 10x10 rect, 200 x 500 TF-IDF, 10 epochs (T = 2000), full schedule."""
    C = bank_corpus(200, 500, seed=seed)
    X = C.dense()
    W0 = init_rows(X, 100, seed + 1000)
    W, log, Wo, logo = _train_both(som, 10, 10, 0, X, W0, 10, 0.1, 5.0, seed)
    _assert_train(W, log, Wo, logo)
    # the strict contract normally reproduces the weights bit for bit
    assert np.count_nonzero(W != Wo) <= W.size // 1000


@pytest.mark.parametrize("mode", [1, 2])
def test_c1_hex_smem_and_global(som, mode):
    C = bank_corpus(200, 500, seed=4)
    X = C.dense()
    W0 = init_rows(X, 100, 4)
    W, log, Wo, logo = _train_both(som, 10, 10, 1, X, W0, 5, 0.1, 5.0, 9, mode=mode)
    _assert_train(W, log, Wo, logo)


@pytest.mark.parametrize("kind,cutoff", [(1, 1e-4), (2, 1e-3), (0, 0.0)])
def test_decay_kinds_and_no_cutoff(som, kind, cutoff):
    C = bank_corpus(150, 300, seed=5)
    X = C.dense()
    W0 = init_rows(X, 48, 5)
    W, log, Wo, logo = _train_both(som, 6, 8, 1, X, W0, 4, 0.2, 4.0, 5, kind=kind, cutoff=cutoff)
    _assert_train(W, log, Wo, logo)


@pytest.mark.parametrize("rows,cols,d,n,mode", [
    (1, 1, 7, 5, 0),          # 1-unit map: BMU always 0
    (1, 13, 33, 40, 0),       # 1 x N strip, ragged d
    (17, 19, 501, 90, 0),     # N = 323 > 148 CTAs, d % 4 != 0 (smem)
    (17, 19, 501, 90, 2),     # same, global W with scalar rows
    (12, 25, 1030, 60, 2),    # global W, float4 rows, N = 300
    (3, 2, 4, 1, 0),          # n = 1
])
def test_ragged_shapes(som, rows, cols, d, n, mode):
    X = uniform_matrix(n, d, rows * 100 + cols)
    X /= np.linalg.norm(X, axis=1, keepdims=True).astype(np.float32)
    W0 = uniform_matrix(rows * cols, d, 7) * np.float32(0.05)
    W, log, Wo, logo = _train_both(som, rows, cols, 1, X, W0, 3, 0.3, max(rows, cols) / 2.0, 77, mode=mode)
    _assert_train(W, log, Wo, logo)


def test_t_range_resume_matches_one_call(som):
    C = bank_corpus(120, 256, seed=6)
    X = C.dense()
    W0 = init_rows(X, 64, 6)
    with som.SOM(8, 8, 256, 1) as m:
        m.set_weights(W0)
        la = np.empty(600, np.int32)
        m.train_online(X, epochs=5, alpha0=0.1, sigma0=4.0, seed=3, bmu_log=la)
        Wa = m.get_weights()
        m.set_weights(W0)
        lb1 = np.empty(123, np.int32)
        lb2 = np.empty(477, np.int32)
        m.train_online(X, epochs=5, alpha0=0.1, sigma0=4.0, seed=3, t_begin=0, t_end=123, bmu_log=lb1)
        m.train_online(X, epochs=5, alpha0=0.1, sigma0=4.0, seed=3, t_begin=123, t_end=-1, bmu_log=lb2)
        Wb = m.get_weights()
    assert np.array_equal(Wa, Wb) and np.array_equal(la, np.concatenate([lb1, lb2]))


def test_zero_rate_and_zero_epochs_leave_weights(som):
    C = bank_corpus(80, 128, seed=7)
    X = C.dense()
    W0 = init_rows(X, 20, 7)
    with som.SOM(4, 5, 128, 1) as m:
        m.set_weights(W0)
        m.train_online(X, epochs=3, alpha0=0.0, sigma0=2.0, seed=1)
        assert np.array_equal(m.get_weights(), W0)
        m.train_online(X, epochs=0, alpha0=0.5, sigma0=2.0, seed=1)
        assert np.array_equal(m.get_weights(), W0)


def test_c2_prefix(som):
    """c2 shape: 20x20 hex, 5000 x 3000, 100 epochs; first 1500 steps via the t-range."""
    C = bank_corpus(5000, 3000, seed=1)
    X = C.dense()
    W0 = init_rows(X, 400, 1001)
    W, log, Wo, logo = _train_both(som, 20, 20, 1, X, W0, 100, 0.1, 10.0, 1, t_begin=0, t_end=1500)
    _assert_train(W, log, Wo, logo)


def test_device_tensors_through_abi(som):
    import torch
    C = bank_corpus(200, 500, seed=2)
    X = C.dense()
    W0 = init_rows(X, 100, 2)
    Xt = torch.from_numpy(X).cuda()
    with som.SOM(10, 10, 500, 0) as m:
        m.set_weights(torch.from_numpy(W0).cuda())
        log = torch.empty(400, dtype=torch.int32, device="cuda")
        som.som_train_online(m.h, Xt, 200, 2, 0.1, 5.0, None, 11, 0, -1, log)
        Wd = torch.empty(100, 500, device="cuda")
        som.som_get_weights(m.h, Wd)
    Wo, logo = oracle.train_online(W0, 10, 10, 0, X, 2, 0.1, 5.0, 11)
    _assert_train(Wd.cpu().numpy(), log.cpu().numpy(), Wo, logo)


# ---------------------------------------------------------------- mapping
@pytest.mark.parametrize("rows,cols,d,n,topo", [(10, 10, 500, 200, 0), (7, 19, 333, 1000, 1),
                                                (20, 20, 3000, 5000, 1), (1, 1, 5, 9, 1), (2, 1, 17, 130, 0)])
def test_map_exact_matches_oracle(som, rows, cols, d, n, topo):
    C = bank_corpus(n, d, seed=n + d) if d >= 50 and n >= 50 else None
    X = C.dense() if C is not None else uniform_matrix(n, d, 3)
    W0 = init_rows(X, rows * cols, 5) * np.float32(0.7) + np.float32(0.001)
    with som.SOM(rows, cols, d, topo) as m:
        m.set_weights(W0)
        b1, b2, d1 = m.map(X)
        qe, te = m.errors(X)
        U = m.umatrix()
    ob1, ob2, od1 = oracle.map_docs(W0, X)
    assert np.array_equal(b1, ob1) and np.array_equal(b2, ob2)
    assert np.array_equal(d1, od1)
    assert abs(qe - oracle.qerror_from_d1(od1)) <= 1e-12 * max(1.0, qe)
    assert te == oracle.topographic_error_from_bmus(rows, cols, topo, ob1, ob2)
    np.testing.assert_allclose(U, oracle.umatrix(W0, rows, cols, topo), rtol=1e-6, atol=1e-7)


def test_map_csr_matches_dense(som):
    C = bank_corpus(3000, 2000, seed=9)
    X = C.dense()
    W0 = init_rows(X, 150, 9)
    with som.SOM(10, 15, 2000, 1) as m:
        m.set_weights(W0)
        a = m.map(X)
        som.som_set_map_precision(m.h, som.SOM_MAP_EXACT_F64)   # densified CSR through the exact path
        b1 = np.empty(C.n, np.int32)
        b2 = np.empty(C.n, np.int32)
        d1 = np.empty(C.n, np.float32)
        som.som_map_csr(m.h, C.indptr, C.indices, C.data, C.n, b1, b2, d1)
    assert np.array_equal(a[0], b1) and np.array_equal(a[1], b2) and np.array_equal(a[2], d1)


def test_init_random_rows_distinct(som):
    X = uniform_matrix(50, 12, 4)
    with som.SOM(5, 6, 12, 1) as m:
        m.init_random(X, seed=3)
        W = m.get_weights()
    rows = [int(np.flatnonzero((X == w).all(1))[0]) for w in W]
    assert len(set(rows)) == 30


def test_validation_errors(som):
    X = uniform_matrix(10, 4, 1)
    with som.SOM(2, 2, 4, 1) as m:
        with pytest.raises(som.SomError) as e:
            som.som_train_online(m.h, X, 0, 1, 0.1, 1.0, None, 1)
        assert e.value.status == som.SOM_EEMPTY
        with pytest.raises(som.SomError) as e:
            som.som_train_online(m.h, X, 10, 1, 1.5, 1.0, None, 1)
        assert e.value.status == som.SOM_EINVAL
        with pytest.raises(som.SomError) as e:
            som.som_train_online(m.h, X, 10, 1, 0.1, 1.0, None, 1, 5, 11)
        assert e.value.status == som.SOM_EINVAL
        with pytest.raises(som.SomError) as e:
            som.som_errors(m.h, X, 0)
        assert e.value.status == som.SOM_EEMPTY
        # the handle still works after argument errors
        m.train_online(X, epochs=1, alpha0=0.1, sigma0=1.0, seed=1)


@pytest.mark.parametrize("grid", [1, 7, 32, 64, 148])
def test_register_kernel_grid_invariance(som, grid):
    """Results do not depend on the number of persistent CTAs."""
    C = bank_corpus(400, 1200, seed=12)
    X = C.dense()
    W0 = init_rows(X, 80, 12)
    with som.SOM(8, 10, 1200, 1) as m:
        som.som_set_train_mode(m.h, som.SOM_TRAIN_W_REGISTERS if grid >= 10 else som.SOM_TRAIN_AUTO)
        som.som_set_train_grid(m.h, grid)
        m.set_weights(W0)
        log = np.empty(1600, np.int32)
        m.train_online(X, epochs=4, alpha0=0.1, sigma0=5.0, seed=12, bmu_log=log)
        W = m.get_weights()
        g, kern = som.som_last_train_config(m.h)
    assert g == min(grid, 80)
    Wo, logo = oracle.train_online(W0, 8, 10, 1, X, 4, 0.1, 5.0, 12)
    _assert_train(W, log, Wo, logo)


def test_c2_kernel_variants_agree(som):
    """c2 shape, 3000 steps: register, shared and global placements give the same result."""
    C = bank_corpus(5000, 3000, seed=2)
    X = C.dense()
    W0 = init_rows(X, 400, 1002)
    out = {}
    for mode in (som.SOM_TRAIN_W_REGISTERS, som.SOM_TRAIN_W_SHARED, som.SOM_TRAIN_W_GLOBAL):
        with som.SOM(20, 20, 3000, 1) as m:
            som.som_set_train_mode(m.h, mode)
            m.set_weights(W0)
            log = np.empty(3000, np.int32)
            m.train_online(X, epochs=100, alpha0=0.1, sigma0=10.0, seed=2, t_end=3000, bmu_log=log)
            out[mode] = (m.get_weights(), log, som.som_last_train_config(m.h))
    W1, l1, c1 = out[som.SOM_TRAIN_W_REGISTERS]
    assert c1[1] == 2
    for mode in (som.SOM_TRAIN_W_SHARED, som.SOM_TRAIN_W_GLOBAL):
        assert np.array_equal(out[mode][1], l1) and np.array_equal(out[mode][0], W1)


@pytest.mark.slow
def test_c2_full_schedule(som):
    """c2 in full: 20x20 hex, 5000 x 3000, 100 epochs = 500,000 steps
    (BASELINE.json configs[1]).  The oracle runs on all host cores (OpenMP
    over units; each unit's sum stays sequential).  BMU sequence identical
    over the whole schedule, weights within 1e-4."""
    C = bank_corpus(5000, 3000, seed=1)
    X = C.dense()
    W0 = init_rows(X, 400, 1001)
    W, log, Wo, logo = _train_both(som, 20, 20, 1, X, W0, 100, 0.1, 10.0, 1)
    _assert_train(W, log, Wo, logo)
    print(f" [c2 full: 500000 steps, BMU log identical, max|dW| = {np.abs(W - Wo).max():.3g}, "
          f"bit-identical weights: {np.array_equal(W, Wo)}]", end="")


def test_c3_prefix_global_kernel(som, monkeypatch):
    """c3 shape (50x50 hex, 10k terms; W = 100 MB streams from L2/HBM): the
    pipelined global-memory kernel (dense rows kept dense:
    SOM_TRAIN_DENSE_CSR=0), first 150 steps, against the oracle."""
    monkeypatch.setenv("SOM_TRAIN_DENSE_CSR", "0")
    C = bank_corpus(3000, 10000, seed=3)
    X = C.dense()
    W0 = init_rows(X, 2500, 1003)
    with som.SOM(50, 50, 10000, 1) as m:
        m.set_weights(W0)
        log = np.empty(150, np.int32)
        m.train_online(X, epochs=10, alpha0=0.1, sigma0=25.0, seed=3, t_end=150, bmu_log=log)
        assert som.som_last_train_config(m.h)[1] == 3
        W = m.get_weights()
    Wo, logo = oracle.train_online(W0, 50, 50, 1, X, 10, 0.1, 25.0, 3, t_end=150)
    _assert_train(W, log, Wo, logo)


@pytest.mark.parametrize("ring", [True, False])
def test_c2_shape_global_kernels_ring_and_registers(som, monkeypatch, ring):
    """Both global-memory kernels (TMA row ring; register-pipelined) on the
    c2 shape agree with the oracle over 1500 steps."""
    if not ring:
        monkeypatch.setenv("SOM_NO_TMA_RING", "1")
    C = bank_corpus(5000, 3000, seed=4)
    X = C.dense()
    W0 = init_rows(X, 400, 1004)
    W, log, Wo, logo = _train_both(som, 20, 20, 1, X, W0, 100, 0.1, 10.0, 4, mode=2, t_end=1500)
    _assert_train(W, log, Wo, logo)


@pytest.mark.parametrize("csr", [False, True])
def test_c4_shape_prefix(som, csr):
    """c4 map and vocabulary (100x100 hex, 20k terms; W = 800 MB streams from
    HBM): the first 40 steps, dense rows (TMA row-ring kernel) and CSR rows
    (sparse-distance kernel), against the oracle.  2,000 documents keep the
    oracle's dense copy small; the kernels only see the map and row shapes."""
    C = bank_corpus(2000, 20000, seed=44)
    X = C.dense()
    W0 = init_rows(X, 10000, 1044) if X.shape[0] >= 10000 else \
        (0.5 * init_rows(bank_corpus(10000, 20000, seed=45).dense(), 10000, 1) + 0.5 * X.mean(0)).astype(np.float32)
    steps = 40
    with som.SOM(100, 100, 20000, 1) as m:
        m.set_weights(W0)
        log = np.empty(steps, np.int32)
        if csr:
            m.train_online_csr(C.indptr, C.indices, C.data, C.n, 2, alpha0=0.1, sigma0=50.0, seed=4, t_end=steps,
                               bmu_log=log)
        else:
            m.train_online(X, epochs=2, alpha0=0.1, sigma0=50.0, seed=4, t_end=steps, bmu_log=log)
        ms, _, _ = som.som_last_stats(m.h)
        g, k = som.som_last_train_config(m.h)
        W = m.get_weights()
    Wo, logo = oracle.train_online(W0, 100, 100, 1, X, 2, 0.1, 50.0, 4, t_end=steps)
    _assert_train(W, log, Wo, logo)
    print(f" [c4 prefix {'csr' if csr else 'dense'}: kernel {k}, G={g}, {1000 * ms / steps:.1f} us/step]", end="")
