"""Thin Python binding of libsom (include/som.h): argument marshalling only.

Every function has the name of the C entry point it calls and the same
argument order.  Arrays may be numpy arrays (host memory) or torch tensors
(host or CUDA); the library detects where each pointer lives.  All compute
runs in libsom's sm_100a kernels — there is no Python or CPU fallback: if
libsom.so is missing or no B200 is present, the calls raise.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SOM_LIB", os.path.join(_HERE, "libsom.so"))   # SOM_LIB: A/B a second build

SOM_OK, SOM_EINVAL, SOM_EDIM, SOM_EEMPTY, SOM_ENOMEM, SOM_ECUDA, SOM_ENCCL, SOM_ESTATE, SOM_EUNSUPPORTED = range(9)
SOM_RECT, SOM_HEX = 0, 1
SOM_DECAY_GAUSSIAN, SOM_DECAY_LINEAR, SOM_DECAY_EXP = 0, 1, 2
SOM_MAP_AUTO, SOM_MAP_EXACT_F64, SOM_MAP_3XTF32, SOM_MAP_SPARSE_F64 = 0, 1, 2, 3
SOM_TRAIN_AUTO, SOM_TRAIN_W_SHARED, SOM_TRAIN_W_GLOBAL, SOM_TRAIN_W_REGISTERS = 0, 1, 2, 3
SOM_SHARD_DOCS, SOM_SHARD_NEURONS = 1, 2
SOM_XCHG_MAILBOX, SOM_XCHG_NCCL = 0, 1
SOM_SAMPLE_REPLACE, SOM_SAMPLE_PERMUTE = 0, 1

_STATUS = {0: "SOM_OK", 1: "SOM_EINVAL", 2: "SOM_EDIM", 3: "SOM_EEMPTY", 4: "SOM_ENOMEM", 5: "SOM_ECUDA",
           6: "SOM_ENCCL", 7: "SOM_ESTATE", 8: "SOM_EUNSUPPORTED"}


class SomError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class som_schedule(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("k", ctypes.c_double), ("sigma_min", ctypes.c_double),
                ("cutoff", ctypes.c_double), ("sampling", ctypes.c_int32)]


_lib = None

# every symbol include/som.h declares (tests check the library exports them)
EXPORTS = ["som_schedule_default", "som_create", "som_destroy", "som_set_weights", "som_get_weights",
           "som_init_random", "som_train_online", "som_train_online_csr", "som_set_train_mode", "som_set_train_grid", "som_set_trace", "som_last_train_config", "som_last_spec_fallbacks", "som_last_map_fallbacks", "som_map", "som_map_csr", "som_set_map_precision",
           "som_train_batch", "som_train_batch_csr", "som_tfidf_csr", "som_pca_top2", "som_pca_top2_csr",
           "som_init_linear", "som_map_geometry",
           "som_qerror", "som_topographic_error", "som_errors", "som_errors_csr", "som_umatrix", "som_set_stream",
           "som_last_stats", "som_last_error", "som_version", "som_comm_init", "som_comm_local_units",
           "som_comm_mailbox_ipc", "som_comm_set_peers_ipc", "som_comm_set_peers_dev", "som_comm_mailbox_ptr",
           "som_comm_unique_id", "som_comm_init_nccl", "som_set_exchange", "som_init_random_csr", "som_fit",
           "som_fit_csr", "som_last_phases"]


def lib():
    """Load libsom.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    P, i32, i64, u64, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
    sig = {
        "som_schedule_default": [P],
        "som_create": [i32, i32, i32, i32, i32, P],
        "som_set_weights": [P, P],
        "som_get_weights": [P, P],
        "som_init_random": [P, P, i64, u64],
        "som_train_online": [P, P, i64, i32, f64, f64, P, u64, i64, i64, P],
        "som_train_online_csr": [P, P, P, P, i64, i32, f64, f64, P, u64, i64, i64, P],
        "som_train_batch": [P, P, i64, i32, f64, P, P],
        "som_tfidf_csr": [P, P, P, P, i64, P, P],
        "som_pca_top2": [P, P, i64, P, P, P, P],
        "som_pca_top2_csr": [P, P, P, P, i64, P, P, P, P],
        "som_init_linear": [P, P, P, P, f64, f64],
        "som_map_geometry": [i64, f64, f64, P, P, P],
        "som_train_batch_csr": [P, P, P, P, i64, i32, f64, P, P],
        "som_map": [P, P, i64, P, P, P],
        "som_map_csr": [P, P, P, P, i64, P, P, P],
        "som_set_map_precision": [P, i32],
        "som_set_train_mode": [P, i32],
        "som_set_train_grid": [P, i32],
        "som_set_trace": [P, P, i32],
        "som_last_train_config": [P, P, P],
        "som_last_spec_fallbacks": [P, P],
        "som_last_map_fallbacks": [P, P],
        "som_qerror": [P, P, i64, P],
        "som_topographic_error": [P, P, i64, P],
        "som_errors": [P, P, i64, P, P],
        "som_errors_csr": [P, P, P, P, i64, P, P],
        "som_umatrix": [P, P],
        "som_set_stream": [P, P],
        "som_last_stats": [P, P, P, P],
        "som_comm_init": [P, i32, i32],
        "som_comm_local_units": [P, P],
        "som_comm_mailbox_ipc": [P, P],
        "som_comm_set_peers_ipc": [P, P],
        "som_comm_set_peers_dev": [P, P],
        "som_comm_mailbox_ptr": [P, P],
        "som_comm_unique_id": [P],
        "som_comm_init_nccl": [P, i32, i32, P, i32],
        "som_set_exchange": [P, i32],
        "som_init_random_csr": [P, P, P, P, i64, u64],
        "som_fit": [P, P, i64, i32, f64, f64, P, u64, u64, P, P, P, P, P, P],
        "som_fit_csr": [P, P, P, P, i64, i32, f64, f64, P, u64, u64, P, P, P, P, P, P],
        "som_last_phases": [P, P, P],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    L.som_destroy.argtypes = [P]
    L.som_destroy.restype = None
    L.som_last_error.argtypes = []
    L.som_last_error.restype = ctypes.c_char_p
    L.som_version.argtypes = []
    L.som_version.restype = ctypes.c_char_p
    _lib = L
    return L


def _check(st: int):
    if st != SOM_OK:
        raise SomError(st, lib().som_last_error().decode())


# (rows*cols, dim) of every live handle, for the size checks below (the C
# ABI takes plain pointers and cannot see buffer sizes)
_dims: dict[int, tuple[int, int]] = {}


def _numel(a) -> int:
    return int(a.size) if isinstance(a, np.ndarray) else int(a.numel())


def _need(a, count: int, what: str):
    """SOM_EDIM unless a holds at least `count` elements (None passes)."""
    if a is not None and _numel(a) < count:
        raise SomError(SOM_EDIM, f"{what}: {_numel(a)} elements, need {count}")


def _check_rows(h, X, n: int, what: str = "X"):
    """X must be (>= n, dim) or hold >= n * dim elements."""
    if X is None or n <= 0:
        return
    d = _dims.get(_hv(h))
    if d is None:
        return
    if getattr(X, "ndim", 1) == 2 and X.shape[1] != d[1]:
        raise SomError(SOM_EDIM, f"{what} has {X.shape[1]} columns, the map has dim {d[1]}")
    _need(X, n * d[1], what)


def _hv(h) -> int:
    return h.value if isinstance(h, ctypes.c_void_p) else int(h or 0)


def _ptr(a, dtype=None, writable=False):
    """Raw pointer of a contiguous numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        if dtype is not None and a.dtype != np.dtype(dtype):
            raise TypeError(f"expected {np.dtype(dtype)}, got {a.dtype}")
        if writable and not a.flags.writeable:
            raise ValueError("output array is read-only")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):   # torch.Tensor
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        if dtype is not None:
            want = {np.float32: "torch.float32", np.int32: "torch.int32", np.int64: "torch.int64",
                    np.float64: "torch.float64"}[dtype]
            if str(a.dtype) != want:
                raise TypeError(f"expected {want}, got {a.dtype}")
        return a.data_ptr()
    raise TypeError(f"unsupported array type {type(a)}")


# ------------------------------------------------------------------ ABI calls
def som_schedule_default() -> som_schedule:
    s = som_schedule()
    _check(lib().som_schedule_default(ctypes.byref(s)))
    return s


def som_create(rows: int, cols: int, dim: int, topology: int, device: int = 0) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    _check(lib().som_create(rows, cols, dim, topology, device, ctypes.byref(h)))
    _dims[_hv(h)] = (rows * cols, dim)
    return h


def som_destroy(h) -> None:
    _dims.pop(_hv(h), None)
    lib().som_destroy(h)


def _check_map(h, w, what):
    d = _dims.get(_hv(h))
    if d is not None:
        _need(w, d[0] * d[1], what)


def som_set_weights(h, w) -> None:
    _check_map(h, w, "w")
    _check(lib().som_set_weights(h, _ptr(w, np.float32)))


def som_get_weights(h, w) -> None:
    _check_map(h, w, "w")
    _check(lib().som_get_weights(h, _ptr(w, np.float32, writable=True)))


def som_init_random(h, X, n: int, seed: int) -> None:
    _check_rows(h, X, n)
    _check(lib().som_init_random(h, _ptr(X, np.float32), n, seed & (2**64 - 1)))


def _check_log(bmu_log, t_begin, t_end, n, epochs):
    if bmu_log is not None:
        te = epochs * n if t_end == -1 else t_end
        _need(bmu_log, max(te - t_begin, 0), "bmu_log")


def _check_csr(rowptr, col, val, n):
    _need(rowptr, n + 1, "rowptr")
    if col is not None and val is not None and _numel(col) != _numel(val):
        raise SomError(SOM_EDIM, "col and val differ in length")


def som_train_online(h, X, n: int, epochs: int, alpha0: float, sigma0: float, sched: som_schedule | None,
                     seed: int, t_begin: int = 0, t_end: int = -1, bmu_log=None) -> None:
    _check_rows(h, X, n)
    _check_log(bmu_log, t_begin, t_end, n, epochs)
    sp = ctypes.byref(sched) if sched is not None else None
    _check(lib().som_train_online(h, _ptr(X, np.float32), n, epochs, alpha0, sigma0, sp, seed & (2**64 - 1),
                                  t_begin, t_end, _ptr(bmu_log, np.int32, writable=True)))


def som_train_online_csr(h, rowptr, col, val, n: int, epochs: int, alpha0: float, sigma0: float,
                         sched: som_schedule | None, seed: int, t_begin: int = 0, t_end: int = -1,
                         bmu_log=None) -> None:
    _check_csr(rowptr, col, val, n)
    _check_log(bmu_log, t_begin, t_end, n, epochs)
    sp = ctypes.byref(sched) if sched is not None else None
    _check(lib().som_train_online_csr(h, _ptr(rowptr, np.int64), _ptr(col, np.int32), _ptr(val, np.float32), n,
                                      epochs, alpha0, sigma0, sp, seed & (2**64 - 1), t_begin, t_end,
                                      _ptr(bmu_log, np.int32, writable=True)))


def som_train_batch(h, X, n: int, epochs: int, sigma0: float, sched: som_schedule | None = None, bmu=None) -> None:
    _check_rows(h, X, n)
    _need(bmu, n, "bmu")
    _check(lib().som_train_batch(h, _ptr(X, np.float32), n, epochs, sigma0,
                                 ctypes.byref(sched) if sched is not None else None, _ptr(bmu, np.int32, True)))


def som_train_batch_csr(h, rowptr, col, val, n: int, epochs: int, sigma0: float, sched: som_schedule | None = None,
                        bmu=None) -> None:
    _check_csr(rowptr, col, val, n)
    _need(bmu, n, "bmu")
    _check(lib().som_train_batch_csr(h, _ptr(rowptr, np.int64), _ptr(col, np.int32), _ptr(val, np.float32), n,
                                     epochs, sigma0, ctypes.byref(sched) if sched is not None else None,
                                     _ptr(bmu, np.int32, True)))


def som_tfidf_csr(h, rowptr, col, counts, n: int, out) -> int:
    z = ctypes.c_int64()
    _check(lib().som_tfidf_csr(h, _ptr(rowptr, np.int64), _ptr(col, np.int32), _ptr(counts, np.float32), n,
                               _ptr(out, np.float32, True), ctypes.byref(z)))
    return z.value


def som_pca_top2(h, X, n: int, mean, v1, v2, pc) -> None:
    _check(lib().som_pca_top2(h, _ptr(X, np.float32), n, _ptr(mean, np.float64, True), _ptr(v1, np.float64, True),
                              _ptr(v2, np.float64, True), _ptr(pc, np.float64, True)))


def som_pca_top2_csr(h, rowptr, col, val, n: int, mean, v1, v2, pc) -> None:
    _check(lib().som_pca_top2_csr(h, _ptr(rowptr, np.int64), _ptr(col, np.int32), _ptr(val, np.float32), n,
                                  _ptr(mean, np.float64, True), _ptr(v1, np.float64, True),
                                  _ptr(v2, np.float64, True), _ptr(pc, np.float64, True)))


def som_init_linear(h, mean, v1, v2, pc1: float, pc2: float) -> None:
    _check(lib().som_init_linear(h, _ptr(mean, np.float64), _ptr(v1, np.float64), _ptr(v2, np.float64), pc1, pc2))


def som_map_geometry(m: int, pc1: float, pc2: float) -> tuple[int, int, int]:
    r, c, t = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64()
    _check(lib().som_map_geometry(m, pc1, pc2, ctypes.byref(r), ctypes.byref(c), ctypes.byref(t)))
    return r.value, c.value, t.value


def som_map(h, X, n: int, bmu1, bmu2=None, d2=None) -> None:
    _check_rows(h, X, n)
    for a, nm in ((bmu1, "bmu1"), (bmu2, "bmu2"), (d2, "d2")):
        _need(a, n, nm)
    _check(lib().som_map(h, _ptr(X, np.float32), n, _ptr(bmu1, np.int32, True), _ptr(bmu2, np.int32, True),
                         _ptr(d2, np.float32, True)))


def som_map_csr(h, rowptr, col, val, n: int, bmu1, bmu2=None, d2=None) -> None:
    _check_csr(rowptr, col, val, n)
    for a, nm in ((bmu1, "bmu1"), (bmu2, "bmu2"), (d2, "d2")):
        _need(a, n, nm)
    _check(lib().som_map_csr(h, _ptr(rowptr, np.int64), _ptr(col, np.int32), _ptr(val, np.float32), n,
                             _ptr(bmu1, np.int32, True), _ptr(bmu2, np.int32, True), _ptr(d2, np.float32, True)))


def som_set_train_mode(h, mode: int) -> None:
    _check(lib().som_set_train_mode(h, mode))


def som_set_trace(h, device_buf, steps: int) -> None:
    _check(lib().som_set_trace(h, _ptr(device_buf), steps))


def som_set_train_grid(h, grid: int) -> None:
    _check(lib().som_set_train_grid(h, grid))


def som_last_train_config(h) -> tuple[int, int]:
    g, k = ctypes.c_int32(), ctypes.c_int32()
    _check(lib().som_last_train_config(h, ctypes.byref(g), ctypes.byref(k)))
    return g.value, k.value



def som_last_map_fallbacks(h) -> int:
    n = ctypes.c_int64()
    _check(lib().som_last_map_fallbacks(h, ctypes.byref(n)))
    return n.value


def som_last_spec_fallbacks(h) -> int:
    n = ctypes.c_int64()
    _check(lib().som_last_spec_fallbacks(h, ctypes.byref(n)))
    return int(n.value)

def som_set_map_precision(h, precision: int) -> None:
    _check(lib().som_set_map_precision(h, precision))


def som_qerror(h, X, n: int) -> float:
    _check_rows(h, X, n)
    q = ctypes.c_double()
    _check(lib().som_qerror(h, _ptr(X, np.float32), n, ctypes.byref(q)))
    return q.value


def som_topographic_error(h, X, n: int) -> float:
    _check_rows(h, X, n)
    t = ctypes.c_double()
    _check(lib().som_topographic_error(h, _ptr(X, np.float32), n, ctypes.byref(t)))
    return t.value


def som_errors(h, X, n: int) -> tuple[float, float]:
    _check_rows(h, X, n)
    q, t = ctypes.c_double(), ctypes.c_double()
    _check(lib().som_errors(h, _ptr(X, np.float32), n, ctypes.byref(q), ctypes.byref(t)))
    return q.value, t.value


def som_errors_csr(h, rowptr, col, val, n: int) -> tuple[float, float]:
    _check_csr(rowptr, col, val, n)
    q, t = ctypes.c_double(), ctypes.c_double()
    _check(lib().som_errors_csr(h, _ptr(rowptr, np.int64), _ptr(col, np.int32), _ptr(val, np.float32), n,
                                ctypes.byref(q), ctypes.byref(t)))
    return q.value, t.value


def som_umatrix(h, U) -> None:
    d = _dims.get(_hv(h))
    if d is not None:
        _need(U, d[0], "U")
    _check(lib().som_umatrix(h, _ptr(U, np.float32, True)))


def som_set_stream(h, stream) -> None:
    """stream: a torch.cuda.Stream, a raw cudaStream_t int, or None."""
    raw = None if stream is None else (stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
    _check(lib().som_set_stream(h, raw))


def som_last_stats(h) -> tuple[float, int, int]:
    ms, units, launches = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int32()
    _check(lib().som_last_stats(h, ctypes.byref(ms), ctypes.byref(units), ctypes.byref(launches)))
    return ms.value, units.value, launches.value


def som_comm_init(h, rank: int, world: int) -> None:
    _check(lib().som_comm_init(h, rank, world))


def som_comm_local_units(h) -> int:
    v = ctypes.c_int32()
    _check(lib().som_comm_local_units(h, ctypes.byref(v)))
    return v.value


def som_comm_mailbox_ipc(h) -> bytes:
    buf = (ctypes.c_uint8 * 64)()
    _check(lib().som_comm_mailbox_ipc(h, buf))
    return bytes(buf)


def som_comm_set_peers_ipc(h, handles: list[bytes]) -> None:
    blob = b"".join(handles)
    buf = (ctypes.c_uint8 * len(blob)).from_buffer_copy(blob)
    _check(lib().som_comm_set_peers_ipc(h, buf))


def som_comm_set_peers_dev(h, mailboxes: list[int]) -> None:
    arr = (ctypes.c_void_p * len(mailboxes))(*mailboxes)
    _check(lib().som_comm_set_peers_dev(h, arr))


def som_comm_mailbox_ptr(h) -> int:
    v = ctypes.c_void_p()
    _check(lib().som_comm_mailbox_ptr(h, ctypes.byref(v)))
    return v.value or 0


def som_comm_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().som_comm_unique_id(buf))
    return bytes(buf)


def som_comm_init_nccl(h, rank: int, world: int, uid: bytes, shard_mode: int) -> None:
    if len(uid) != 128:
        raise SomError(SOM_EINVAL, "NCCL unique id must be 128 bytes")
    buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    _check(lib().som_comm_init_nccl(h, rank, world, buf, shard_mode))


def som_set_exchange(h, mode: int) -> None:
    _check(lib().som_set_exchange(h, mode))


def som_init_random_csr(h, rowptr, col, val, n: int, seed: int) -> None:
    _check_csr(rowptr, col, val, n)
    _check(lib().som_init_random_csr(h, _ptr(rowptr, np.int64), _ptr(col, np.int32), _ptr(val, np.float32), n,
                                     seed & (2**64 - 1)))


def _fit_outputs(h, n, bmu1, bmu2, d2, U):
    for a, nm in ((bmu1, "bmu1"), (bmu2, "bmu2"), (d2, "d2")):
        _need(a, n, nm)
    d = _dims.get(_hv(h))
    if d is not None:
        _need(U, d[0], "U")


def som_fit(h, X, n: int, epochs: int, alpha0: float, sigma0: float, sched: som_schedule | None, seed: int,
            init_seed: int, bmu1=None, bmu2=None, d2=None, U=None) -> tuple[float, float]:
    _check_rows(h, X, n)
    _fit_outputs(h, n, bmu1, bmu2, d2, U)
    q, t = ctypes.c_double(), ctypes.c_double()
    sp = ctypes.byref(sched) if sched is not None else None
    _check(lib().som_fit(h, _ptr(X, np.float32), n, epochs, alpha0, sigma0, sp, seed & (2**64 - 1),
                         init_seed & (2**64 - 1), _ptr(bmu1, np.int32, True), _ptr(bmu2, np.int32, True),
                         _ptr(d2, np.float32, True), ctypes.byref(q), ctypes.byref(t), _ptr(U, np.float32, True)))
    return q.value, t.value


def som_fit_csr(h, rowptr, col, val, n: int, epochs: int, alpha0: float, sigma0: float, sched: som_schedule | None,
                seed: int, init_seed: int, bmu1=None, bmu2=None, d2=None, U=None) -> tuple[float, float]:
    _check_csr(rowptr, col, val, n)
    _fit_outputs(h, n, bmu1, bmu2, d2, U)
    q, t = ctypes.c_double(), ctypes.c_double()
    sp = ctypes.byref(sched) if sched is not None else None
    _check(lib().som_fit_csr(h, _ptr(rowptr, np.int64), _ptr(col, np.int32), _ptr(val, np.float32), n, epochs,
                             alpha0, sigma0, sp, seed & (2**64 - 1), init_seed & (2**64 - 1),
                             _ptr(bmu1, np.int32, True), _ptr(bmu2, np.int32, True), _ptr(d2, np.float32, True),
                             ctypes.byref(q), ctypes.byref(t), _ptr(U, np.float32, True)))
    return q.value, t.value


def som_last_phases(h) -> tuple[list[float], float]:
    ms = (ctypes.c_double * 5)()
    tr = ctypes.c_double()
    _check(lib().som_last_phases(h, ms, ctypes.byref(tr)))
    return list(ms), tr.value


def som_last_error() -> str:
    return lib().som_last_error().decode()


def som_version() -> str:
    return lib().som_version().decode()


# ----------------------------------------------------- convenience wrapper
class SOM:
    """Owning handle: ``SOM(rows, cols, dim, topology)``; methods call the ABI."""

    def __init__(self, rows: int, cols: int, dim: int, topology: int = SOM_HEX, device: int = 0):
        self.rows, self.cols, self.dim, self.topology = rows, cols, dim, topology
        self.N = rows * cols
        self.h = som_create(rows, cols, dim, topology, device)

    def close(self):
        if self.h:
            som_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_weights(self, w):
        som_set_weights(self.h, w)

    def get_weights(self, out=None):
        if out is None:
            out = np.empty((self.N, self.dim), np.float32)
        som_get_weights(self.h, out)
        return out

    def init_random(self, X, seed: int):
        som_init_random(self.h, X, X.shape[0], seed)

    def train_online(self, X, epochs: int, alpha0: float = 0.1, sigma0: float | None = None, seed: int = 1,
                     kind: int = SOM_DECAY_GAUSSIAN, k: float = math.log(100.0), sigma_min: float = 1.0,
                     cutoff: float = 1e-4, t_begin: int = 0, t_end: int = -1, bmu_log=None,
                     sampling: int = SOM_SAMPLE_REPLACE):
        if sigma0 is None:
            sigma0 = max(self.rows, self.cols) / 2.0
        s = som_schedule(kind, k, sigma_min, cutoff, sampling)
        som_train_online(self.h, X, X.shape[0], epochs, alpha0, sigma0, s, seed, t_begin, t_end, bmu_log)
        return bmu_log

    def train_online_csr(self, rowptr, col, val, n: int, epochs: int, alpha0: float = 0.1,
                         sigma0: float | None = None, seed: int = 1, kind: int = SOM_DECAY_GAUSSIAN,
                         k: float = math.log(100.0), sigma_min: float = 1.0, cutoff: float = 1e-4,
                         t_begin: int = 0, t_end: int = -1, bmu_log=None, sampling: int = SOM_SAMPLE_REPLACE):
        if sigma0 is None:
            sigma0 = max(self.rows, self.cols) / 2.0
        s = som_schedule(kind, k, sigma_min, cutoff, sampling)
        som_train_online_csr(self.h, rowptr, col, val, n, epochs, alpha0, sigma0, s, seed, t_begin, t_end, bmu_log)
        return bmu_log

    def map(self, X, want_bmu2: bool = True, want_d2: bool = True):
        n = X.shape[0]
        b1 = np.empty(n, np.int32)
        b2 = np.empty(n, np.int32) if want_bmu2 else None
        d2 = np.empty(n, np.float32) if want_d2 else None
        som_map(self.h, X, n, b1, b2, d2)
        return b1, b2, d2

    def train_batch(self, X, epochs: int, sigma0: float | None = None, kind: int = SOM_DECAY_GAUSSIAN,
                    k: float = math.log(100.0), sigma_min: float = 1.0, cutoff: float = 1e-4, want_bmu: bool = True):
        if sigma0 is None:
            sigma0 = max(self.rows, self.cols) / 2.0
        b = np.empty(X.shape[0], np.int32) if want_bmu else None
        som_train_batch(self.h, X, X.shape[0], epochs, sigma0, som_schedule(kind, k, sigma_min, cutoff), b)
        return b

    def train_batch_csr(self, rowptr, col, val, n: int, epochs: int, sigma0: float | None = None,
                        kind: int = SOM_DECAY_GAUSSIAN, k: float = math.log(100.0), sigma_min: float = 1.0,
                        cutoff: float = 1e-4, want_bmu: bool = True):
        if sigma0 is None:
            sigma0 = max(self.rows, self.cols) / 2.0
        b = np.empty(n, np.int32) if want_bmu else None
        som_train_batch_csr(self.h, rowptr, col, val, n, epochs, sigma0, som_schedule(kind, k, sigma_min, cutoff), b)
        return b

    def pca_top2(self, X=None, csr=None):
        """(pc1, pc2, v1, v2, mean) of dense rows X or csr = (rowptr, col, val, n)."""
        mean, v1, v2, pc = np.empty(self.dim), np.empty(self.dim), np.empty(self.dim), np.empty(2)
        if csr is not None:
            som_pca_top2_csr(self.h, *csr[:3], csr[3], mean, v1, v2, pc)
        else:
            som_pca_top2(self.h, X, X.shape[0], mean, v1, v2, pc)
        return float(pc[0]), float(pc[1]), v1, v2, mean

    def init_linear(self, mean, v1, v2, pc1: float, pc2: float):
        som_init_linear(self.h, mean, v1, v2, pc1, pc2)

    def map_csr(self, rowptr, col, val, n: int, want_bmu2: bool = True, want_d2: bool = True):
        b1 = np.empty(n, np.int32)
        b2 = np.empty(n, np.int32) if want_bmu2 else None
        d2 = np.empty(n, np.float32) if want_d2 else None
        som_map_csr(self.h, rowptr, col, val, n, b1, b2, d2)
        return b1, b2, d2

    def errors(self, X):
        return som_errors(self.h, X, X.shape[0])

    def errors_csr(self, rowptr, col, val, n: int):
        return som_errors_csr(self.h, rowptr, col, val, n)

    def set_map_precision(self, precision: int):
        som_set_map_precision(self.h, precision)

    def umatrix(self):
        U = np.empty(self.N, np.float32)
        som_umatrix(self.h, U)
        return U

    def last_stats(self):
        return som_last_stats(self.h)
