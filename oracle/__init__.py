"""Oracle for the CUDASOM hot path (arXiv 1905.09598) — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product (``paper_1905_09598_b200``) never imports it and shares no code with
it.  The arithmetic lives in ``som_oracle.c`` (plain C, fp64 accumulation,
built with ``-O2 -ffp-contract=off``); this module only marshals numpy
arrays through ctypes.  See the C file for the paper passage each function
follows, and DESIGN.md §3 for the readings where the paper is silent.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "som_oracle.c")
_LIB = os.path.join(_HERE, "libsom_oracle.so")

RECT, HEX = 0, 1
DECAY_GAUSSIAN, DECAY_LINEAR, DECAY_EXP = 0, 1, 2
LN100 = float(np.log(100.0))


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i32, i64, u64, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
        P = ctypes.c_void_p
        L.or_splitmix64.restype = u64
        L.or_splitmix64.argtypes = [u64, i64]
        L.or_sample_index.restype = i64
        L.or_sample_index.argtypes = [u64, i64, i64]
        L.or_perm_index.restype = i64
        L.or_perm_index.argtypes = [u64, i64, i64]
        L.or_schedule.restype = None
        L.or_schedule.argtypes = [ctypes.c_int, f64, i64, i64, f64, f64, f64, f64, P, P, P]
        L.or_lattice_g2.restype = f64
        L.or_lattice_g2.argtypes = [i32, i32, i32, i64, i64]
        L.or_bmu.restype = i64
        L.or_bmu.argtypes = [P, i64, i64, P, P, P]
        L.or_update.restype = None
        L.or_update.argtypes = [P, i32, i32, i32, i64, P, i64, f64, f64, f64]
        L.or_train_online.restype = ctypes.c_int
        L.or_train_online.argtypes = [P, i32, i32, i32, i64, P, i64, i32, f64, f64, i32,
                                      f64, f64, f64, i32, u64, i64, i64, P, P]
        L.or_train_online_csr.restype = ctypes.c_int
        L.or_train_online_csr.argtypes = [P, i32, i32, i32, i64, P, P, P, i64, i32, f64, f64, i32,
                                          f64, f64, f64, i32, u64, i64, i64, P]
        L.or_map.restype = None
        L.or_map.argtypes = [P, i64, i64, P, i64, P, P, P, P, P]
        L.or_map_csr.restype = None
        L.or_map_csr.argtypes = [P, P, i64, i64, P, P, P, i64, P, P, P, P, P]
        L.or_train_batch.restype = ctypes.c_int
        L.or_train_batch.argtypes = [P, i32, i32, i32, i64, P, i64, i32, f64, i32, f64, f64, f64, P]
        L.or_tfidf_csr.restype = None
        L.or_tfidf_csr.argtypes = [P, P, P, i64, i64, P, P]
        L.or_row_sqnorm.restype = None
        L.or_row_sqnorm.argtypes = [P, i64, i64, P]
        L.or_qerror_from_d1.restype = f64
        L.or_qerror_from_d1.argtypes = [P, i64]
        L.or_qerror_masked.restype = f64
        L.or_qerror_masked.argtypes = [P, P, i64]
        L.or_topographic_error_masked.restype = f64
        L.or_topographic_error_masked.argtypes = [i32, i32, i32, P, P, P, i64]
        L.or_nonzero_rows.restype = i64
        L.or_nonzero_rows.argtypes = [P, i64, i64, P]
        L.or_nonzero_rows_csr.restype = i64
        L.or_nonzero_rows_csr.argtypes = [P, P, i64, P]
        L.or_topographic_error_from_bmus.restype = f64
        L.or_topographic_error_from_bmus.argtypes = [i32, i32, i32, P, P, i64]
        L.or_umatrix.restype = None
        L.or_umatrix.argtypes = [P, i32, i32, i32, i64, P]
        L.or_num_threads.restype = ctypes.c_int
        L.or_set_num_threads.restype = None
        L.or_set_num_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


# ------------------------------------------------------------------ sampler
def splitmix64(seed: int, t: int) -> int:
    return int(lib().or_splitmix64(seed & (2**64 - 1), t))


def sample_index(seed: int, t: int, n: int) -> int:
    return int(lib().or_sample_index(seed & (2**64 - 1), t, n))


def perm_index(seed: int, t: int, m: int) -> int:
    """R8b: the draw of step t under per-epoch permutation sampling."""
    return int(lib().or_perm_index(seed & (2**64 - 1), t, m))


# ----------------------------------------------------------------- schedule
def schedule(t, T, alpha0, sigma0, kind=DECAY_GAUSSIAN, k=LN100, sigma_min=1.0, eps=1e-4):
    a, s, r = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    lib().or_schedule(kind, k, t, T, alpha0, sigma0, sigma_min, eps,
                      ctypes.byref(a), ctypes.byref(s), ctypes.byref(r))
    return a.value, s.value, r.value


def lattice_g2(rows, cols, topo, u, v) -> float:
    return float(lib().or_lattice_g2(rows, cols, topo, u, v))


# ------------------------------------------------------------ BMU / update
def bmu(W, x):
    W, x = _f32(W), _f32(x)
    N, d = W.shape
    D = ctypes.c_float()
    m = ctypes.c_double()
    c = lib().or_bmu(_p(W), N, d, _p(x), ctypes.byref(D), ctypes.byref(m))
    return int(c), np.float32(D.value), m.value


def update(W, rows, cols, topo, x, c, alpha, sigma, r2):
    """Apply one Eq. 1 step in place to a float32 (N, d) array; returns W."""
    assert W.dtype == np.float32 and W.flags.c_contiguous
    x = _f32(x)
    lib().or_update(_p(W), rows, cols, topo, W.shape[1], _p(x), c, alpha, sigma, r2)
    return W


def train_online(W, rows, cols, topo, X, epochs, alpha0, sigma0, seed,
                 kind=DECAY_GAUSSIAN, k=LN100, sigma_min=1.0, eps=1e-4,
                 t_begin=0, t_end=-1, want_margins=False, sampling=0):
    """Online SOM on a copy of W.  Returns (W', bmu_log[, margins])."""
    W = np.array(W, dtype=np.float32, copy=True, order="C")
    X = _f32(X)
    n, d = X.shape
    assert W.shape == (rows * cols, d)
    T = epochs * n
    te = T if t_end < 0 else t_end
    steps = max(te - t_begin, 0)
    log = np.empty(steps, dtype=np.int32)
    margins = np.empty(steps, dtype=np.float64) if want_margins else None
    rc = lib().or_train_online(_p(W), rows, cols, topo, d, _p(X), n, epochs, alpha0, sigma0,
                               kind, k, sigma_min, eps, sampling, seed & (2**64 - 1), t_begin, te,
                               _p(log), _p(margins))
    if rc == -2:
        raise ValueError("or_train_online: EmptyData (every row is zero, S:219)")
    if rc != 0:
        raise ValueError("or_train_online: bad arguments")
    return (W, log, margins) if want_margins else (W, log)


def train_online_csr(W, rows, cols, topo, rowptr, col, val, epochs, alpha0, sigma0, seed,
                     kind=DECAY_GAUSSIAN, k=LN100, sigma_min=1.0, eps=1e-4, t_begin=0, t_end=-1, sampling=0):
    """Online SOM on CSR rows (x_t densified per step).  Returns (W', bmu_log)."""
    W = np.array(W, dtype=np.float32, copy=True, order="C")
    rowptr = np.ascontiguousarray(rowptr, np.int64)
    col = np.ascontiguousarray(col, np.int32)
    val = _f32(val)
    n = rowptr.shape[0] - 1
    d = W.shape[1]
    T = epochs * n
    te = T if t_end < 0 else t_end
    log = np.empty(max(te - t_begin, 0), dtype=np.int32)
    rc = lib().or_train_online_csr(_p(W), rows, cols, topo, d, _p(rowptr), _p(col), _p(val), n, epochs, alpha0,
                                   sigma0, kind, k, sigma_min, eps, sampling, seed & (2**64 - 1), t_begin, te,
                                   _p(log))
    if rc == -2:
        raise ValueError("or_train_online_csr: EmptyData (every row is zero, S:219)")
    if rc != 0:
        raise ValueError("or_train_online_csr: bad arguments")
    return W, log


# --------------------------------------------------------------- mapping
def train_batch(W, rows, cols, topo, X, epochs, sigma0, kind=DECAY_GAUSSIAN, k=LN100, sigma_min=1.0,
                eps=1e-4):
    """Batch SOM (R27) on a copy of W.  Returns (W', BMUs after the last epoch)."""
    W = np.array(W, dtype=np.float32, copy=True, order="C")
    X = _f32(X)
    n, d = X.shape
    assert W.shape == (rows * cols, d)
    b = np.empty(n, np.int32)
    r = lib().or_train_batch(_p(W), rows, cols, topo, d, _p(X), n, epochs, sigma0, kind, k, sigma_min, eps, _p(b))
    if r != 0:
        raise ValueError("or_train_batch: bad arguments")
    return W, b


def tfidf_csr(rowptr, col, counts, d):
    """Eq. 2 TF-IDF + L2 row normalisation (R28).  Returns (values, zero_rows)."""
    rowptr = np.ascontiguousarray(rowptr, np.int64)
    col = np.ascontiguousarray(col, np.int32)
    counts = _f32(counts)
    out = np.empty_like(counts)
    zr = ctypes.c_int64()
    lib().or_tfidf_csr(_p(rowptr), _p(col), _p(counts), rowptr.shape[0] - 1, d, _p(out), ctypes.byref(zr))
    return out, zr.value


def map_docs(W, X, want_margins=False):
    W, X = _f32(W), _f32(X)
    N, d = W.shape
    n = X.shape[0]
    b1 = np.empty(n, np.int32)
    b2 = np.empty(n, np.int32)
    d1 = np.empty(n, np.float32)
    m12 = np.empty(n, np.float64)
    m23 = np.empty(n, np.float64)
    lib().or_map(_p(W), N, d, _p(X), n, _p(b1), _p(b2), _p(d1), _p(m12), _p(m23))
    if want_margins:
        return b1, b2, d1, m12, m23
    return b1, b2, d1


def map_docs_csr(W, rowptr, col, val, want_margins=False):
    W = _f32(W)
    N, d = W.shape
    rowptr = np.ascontiguousarray(rowptr, np.int64)
    col = np.ascontiguousarray(col, np.int32)
    val = _f32(val)
    n = rowptr.shape[0] - 1
    wsq = np.empty(N, np.float64)
    lib().or_row_sqnorm(_p(W), N, d, _p(wsq))
    b1 = np.empty(n, np.int32)
    b2 = np.empty(n, np.int32)
    d1 = np.empty(n, np.float32)
    m12 = np.empty(n, np.float64)
    m23 = np.empty(n, np.float64)
    lib().or_map_csr(_p(W), _p(wsq), N, d, _p(rowptr), _p(col), _p(val), n,
                     _p(b1), _p(b2), _p(d1), _p(m12), _p(m23))
    if want_margins:
        return b1, b2, d1, m12, m23
    return b1, b2, d1


from .upstream import linear_init, map_geometry, pca_top2  # noqa: E402,F401


def nonzero_rows(X):
    """Indices of the rows of X holding a non-zero value."""
    X = _f32(X)
    idx = np.empty(X.shape[0], np.int64)
    m = lib().or_nonzero_rows(_p(X), X.shape[0], X.shape[1], _p(idx))
    return idx[:m]


def nonzero_rows_csr(rowptr, val):
    rowptr = np.ascontiguousarray(rowptr, np.int64)
    val = _f32(val)
    idx = np.empty(rowptr.shape[0] - 1, np.int64)
    m = lib().or_nonzero_rows_csr(_p(rowptr), _p(val), rowptr.shape[0] - 1, _p(idx))
    return idx[:m]


def keep_mask(n, nz_idx):
    keep = np.zeros(n, np.uint8)
    keep[nz_idx] = 1
    return keep


def qerror_from_d1(d1, keep=None) -> float:
    """QE (R14) over the rows with keep[i] != 0 (all rows if keep is None):
    zero rows are not scored."""
    d1 = _f32(d1)
    if keep is None:
        return float(lib().or_qerror_from_d1(_p(d1), d1.shape[0]))
    keep = np.ascontiguousarray(keep, np.uint8)
    return float(lib().or_qerror_masked(_p(d1), _p(keep), d1.shape[0]))


def qerror(W, X) -> float:
    _, _, d1 = map_docs(W, X)
    return qerror_from_d1(d1, keep_mask(X.shape[0], nonzero_rows(X)))


def topographic_error_from_bmus(rows, cols, topo, b1, b2, keep=None) -> float:
    b1 = np.ascontiguousarray(b1, np.int32)
    b2 = np.ascontiguousarray(b2, np.int32)
    if keep is None:
        return float(lib().or_topographic_error_from_bmus(rows, cols, topo, _p(b1), _p(b2), b1.shape[0]))
    keep = np.ascontiguousarray(keep, np.uint8)
    return float(lib().or_topographic_error_masked(rows, cols, topo, _p(b1), _p(b2), _p(keep), b1.shape[0]))


def topographic_error(W, rows, cols, topo, X) -> float:
    b1, b2, _ = map_docs(W, X)
    return topographic_error_from_bmus(rows, cols, topo, b1, b2, keep_mask(X.shape[0], nonzero_rows(X)))


def umatrix(W, rows, cols, topo):
    W = _f32(W)
    U = np.empty(rows * cols, np.float32)
    lib().or_umatrix(_p(W), rows, cols, topo, W.shape[1], _p(U))
    return U


def num_threads() -> int:
    return int(lib().or_num_threads())


def set_num_threads(nt: int) -> None:
    lib().or_set_num_threads(nt)
