"""ctypes binding of libfctn_b200.so (the C ABI in include/fctn_b200.h).

There is no fallback: if the library is missing or cannot be loaded the
import of the device path raises.  Loading the library does not need a GPU;
creating a context does.
"""
from __future__ import annotations

import ctypes as C
import os
import sys
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfctn_b200.so")

F64, F32 = 0, 1
ALG_PLAIN, ALG_ACCEL = 0, 1
SIGN_PD, SIGN_PRINTED = 0, 1
ST_OBJECTIVE, ST_DIFF_SQ, ST_BASE_SQ, ST_DATA_SQ, ST_XNEW_SQ = 0, 1, 2, 3, 4
ST_PENALTY, ST_STEP_FAC, ST_FNORM_MAX, ST_DEVICE_MS, ST_COUNT = 5, 6, 7, 8, 16
CT_FLOPS, CT_MK, CT_COMPOSE, CT_HITS, CT_LAUNCHES, CT_COUNT = 0, 1, 2, 3, 4, 8

EXPORTS = [
    "fctn_create", "fctn_upload", "fctn_upload_f64", "fctn_get_x_f64", "fctn_set_factors", "fctn_set_rank", "fctn_get_factors", "fctn_get_x",
    "fctn_objective", "fctn_sweep", "fctn_plan_sweeps", "fctn_nccl_unique_id", "fctn_set_comm", "fctn_set_comm_host", "fctn_set_comm_loopback",
    "fctn_sync", "fctn_selftest_stream", "fctn_selftest_chol", "fctn_selftest_eigh", "fctn_timer", "fctn_set_profiling", "fctn_get_profile", "fctn_last_error", "fctn_version",
    "fctn_quality", "fctn_quality_ctx", "fctn_destroy", "fctn_trim_cache",
]
Q_PSNR, Q_SSIM, Q_ERR_SQ, Q_REF_SQ, Q_OFF_ERR_SQ, Q_OFF_REF_SQ, Q_OFF_COUNT, Q_COUNT = 0, 1, 2, 3, 4, 5, 6, 8
K_CLASSES = ["merge", "stream_y", "gram", "reduce", "chol", "compose", "dft", "fgram", "zpass", "ysmall", "mbuild",
             "eigh"]

_lib = None

HOST_ALLREDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int64)
HOST_ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64)


class _HostBlock:
    """An anonymous mapping (advised for transparent huge pages) that exports
    its bytes (PEP 688) and goes back to the pool when the last array or view
    over it is gone, so a later download of the same size finds its pages
    already faulted in."""

    def __init__(self, mm, nbytes):
        self.mm, self.nbytes = mm, nbytes

    def __buffer__(self, flags):
        return memoryview(self.mm)

    def __release_buffer__(self, view):
        view.release()

    def __del__(self):
        try:
            _host_pool_put(self.mm, self.nbytes)
        except Exception:  # interpreter shutdown
            pass


_HOST_POOL = {}  # nbytes -> [mmap, ...]
_HOST_POOL_IDLE = [0]
_HOST_POOL_LOCK = threading.Lock()


def _host_pool_cap() -> int:
    return int(float(os.environ.get("FCTN_HOSTPOOL_GB", "8")) * (1 << 30))


def _host_pool_put(mm, nbytes):
    with _HOST_POOL_LOCK:
        if _HOST_POOL_IDLE[0] + nbytes <= _host_pool_cap():
            _HOST_POOL.setdefault(nbytes, []).append(mm)
            _HOST_POOL_IDLE[0] += nbytes
            return
    mm.close()


def trim_host_pool():
    """Unmap every idle download buffer."""
    with _HOST_POOL_LOCK:
        for blocks in _HOST_POOL.values():
            for mm in blocks:
                mm.close()
        _HOST_POOL.clear()
        _HOST_POOL_IDLE[0] = 0


def trim_cache():
    """Return the idle device blocks of closed contexts to the driver
    (fctn_trim_cache) and unmap the idle host download buffers."""
    lib().fctn_trim_cache()
    trim_host_pool()


def _host_empty(dims) -> np.ndarray:
    """F-order float64 array for a large download.  The first-touch page
    faults of a fresh 2 GB array cost as much as the transfer (and several
    times more when the kernel has no huge pages to give), so large results
    live in pooled anonymous mappings: the block returns to the pool when the
    caller drops the array (and every view of it), and the next download of
    that size reuses the faulted pages.  FCTN_HOSTPOOL_GB bounds the idle
    bytes (default 8, 0 disables pooling)."""
    n = int(np.prod(dims))
    nbytes = n * 8
    if nbytes < (64 << 20):
        return np.empty(dims, dtype=np.float64, order="F")
    import mmap
    mm = None
    with _HOST_POOL_LOCK:
        blocks = _HOST_POOL.get(nbytes)
        if blocks:
            mm = blocks.pop()
            _HOST_POOL_IDLE[0] -= nbytes
    if mm is None:
        mm = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        try:
            mm.madvise(mmap.MADV_HUGEPAGE)
        except (AttributeError, OSError):
            pass
    if sys.version_info < (3, 12):  # no __buffer__ protocol for Python classes: unpooled mapping
        return np.frombuffer(mm, dtype=np.float64, count=n).reshape(dims, order="F")
    return np.frombuffer(_HostBlock(mm, nbytes), dtype=np.float64, count=n).reshape(dims, order="F")


def slab_of(I0: int, rank: int, nranks: int):
    """Standard partition of mode 0 (fctn_set_comm)."""
    return rank * I0 // nranks, (rank + 1) * I0 // nranks


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(lib().fctn_nccl_unique_id(buf))
    return bytes(buf)


class NativeError(RuntimeError):
    pass


def lib():
    """Load (once) and type the shared library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2510_22506_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    P = C.c_void_p
    i64p = C.POINTER(C.c_int64)
    f64p = C.POINTER(C.c_double)
    L.fctn_create.argtypes = [C.c_int, C.c_int, C.c_int, i64p, i64p, f64p, f64p, C.c_int, C.c_double, C.c_int,
                              C.c_int64, C.POINTER(P)]
    L.fctn_upload.argtypes = [P, P, P]
    L.fctn_upload_f64.argtypes = [P, P, P]
    L.fctn_get_x_f64.argtypes = [P, P]
    L.fctn_set_factors.argtypes = [P, C.POINTER(P), i64p, C.c_int]
    L.fctn_set_rank.argtypes = [P, i64p]
    L.fctn_get_factors.argtypes = [P, C.POINTER(P)]
    L.fctn_get_x.argtypes = [P, P]
    L.fctn_objective.argtypes = [P, f64p, i64p]
    L.fctn_sweep.argtypes = [P, C.POINTER(C.c_int32), C.c_int, C.c_double, C.c_double, f64p, i64p]
    L.fctn_plan_sweeps.argtypes = [C.c_int, i64p, i64p, C.c_int, C.c_int64, C.c_int, C.POINTER(C.c_int32), i64p]
    L.fctn_nccl_unique_id.argtypes = [P]
    L.fctn_set_comm.argtypes = [P, P, C.c_int, C.c_int, C.c_int64, C.c_int64]
    L.fctn_set_comm_host.argtypes = [P, HOST_ALLREDUCE, HOST_ALLGATHER, P, C.c_int, C.c_int, C.c_int64, C.c_int64]
    L.fctn_set_comm_loopback.argtypes = [P, C.c_int, C.c_int, C.c_int64, C.c_int64]
    L.fctn_sync.argtypes = [P]
    L.fctn_selftest_chol.argtypes = [C.c_int, C.c_int64, C.c_int64, P, P, P, P, C.c_int, f64p]
    L.fctn_selftest_eigh.argtypes = [C.c_int, C.c_int64, P, P, P, C.c_int, f64p, C.POINTER(C.c_int)]
    L.fctn_selftest_stream.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64, P, P,
                                       f64p]
    L.fctn_timer.argtypes = [P, C.c_int, f64p]
    L.fctn_set_profiling.argtypes = [P, C.c_int]
    L.fctn_get_profile.argtypes = [P, f64p, i64p, f64p]
    L.fctn_quality.argtypes = [C.c_int, C.c_int, C.c_int, i64p, P, P, P, C.c_double, f64p]
    L.fctn_quality_ctx.argtypes = [P, P, C.c_int, C.c_int, C.c_double, f64p]
    L.fctn_last_error.argtypes = [P]
    L.fctn_last_error.restype = C.c_char_p
    L.fctn_version.argtypes = []
    L.fctn_version.restype = C.c_char_p
    L.fctn_destroy.argtypes = [P]
    L.fctn_destroy.restype = None
    for name in EXPORTS:
        if not hasattr(L, name):
            raise ImportError(f"{LIB_PATH} does not export {name}")
    _lib = L
    return L


def _i64(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int64))
    return a, a.ctypes.data_as(C.POINTER(C.c_int64))


def _f64(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a, a.ctypes.data_as(C.POINTER(C.c_double))


def check(rc: int, handle=None, numeric_exc=None):
    if rc == 0:
        return
    msg = lib().fctn_last_error(handle).decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise (numeric_exc or NativeError)(msg)
    raise NativeError(msg)


def plan_sweeps(dims, rank_tri, algorithm: int, cache_budget: int, orders) -> np.ndarray:
    """Shape-only replay of the reference FLOP meter and cache hits."""
    orders = np.ascontiguousarray(np.asarray(orders, dtype=np.int32))
    n = len(dims)
    ns = orders.shape[0]
    d, dp = _i64(dims)
    r, rp = _i64(rank_tri)
    out = np.zeros((ns, CT_COUNT), dtype=np.int64)
    rc = lib().fctn_plan_sweeps(n, dp, rp, algorithm, int(cache_budget), ns,
                                orders.ctypes.data_as(C.POINTER(C.c_int32)),
                                out.ctypes.data_as(C.POINTER(C.c_int64)))
    check(rc)
    return out


def selftest_stream(x, m, k, use_tc=True, device=0):
    """Y = X_(k) M^T through the library's K2 path (kernel unit tests).
    x: F-order tensor (float32 or float64); m: (p, S) F-order with p in X's
    column order (modes before k fastest)."""
    dt = F32 if x.dtype == np.float32 else F64
    x = np.asfortranarray(x)
    m = np.asfortranarray(m, dtype=x.dtype)
    dims = x.shape
    I = dims[k]
    P = int(np.prod(dims[:k])) if k > 0 else 1
    Q = int(np.prod(dims[k + 1:])) if k + 1 < len(dims) else 1
    S = m.shape[1]
    y = np.zeros((I, S), dtype=np.float64, order="F")
    rc = lib().fctn_selftest_stream(int(device), dt, int(bool(use_tc)), I, P, Q, S, x.ctypes.data_as(C.c_void_p),
                                    m.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.POINTER(C.c_double)))
    check(rc)
    return y


def quality(est: np.ndarray, truth: np.ndarray, mask=None, peak: float = 1.0, device: int = 0) -> np.ndarray:
    """Raw quality sums (FCTN_Q_*) of two host tensors on the device."""
    dt = F32 if (est.dtype == np.float32 and truth.dtype == np.float32) else F64
    npd = np.float32 if dt == F32 else np.float64
    e = np.asfortranarray(est, dtype=npd)
    t = np.asfortranarray(truth, dtype=npd)
    m = None
    if mask is not None:
        m = np.asfortranarray(mask)
        m = m.view(np.uint8) if m.dtype == np.bool_ else np.asfortranarray(m != 0, dtype=np.uint8)
    d, dp = _i64(e.shape)
    out = np.zeros(Q_COUNT, dtype=np.float64)
    check(lib().fctn_quality(int(device), dt, e.ndim, dp, e.ctypes.data_as(C.c_void_p), t.ctypes.data_as(C.c_void_p),
                             None if m is None else m.ctypes.data_as(C.c_void_p), float(peak),
                             out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def selftest_chol(G, mu, Fr, Fi, reps=1, device=0):
    """Per-frequency SPD solves (G + mu_w I) a = F_w on the device; returns
    (Fr_out, Fi_out, best ms per launch).  F arrays are (H1, S)."""
    G = np.asfortranarray(G, dtype=np.float64)
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    H1, S = Fr.shape
    fr = np.asfortranarray(Fr, dtype=np.float64).copy(order="F")
    fi = np.asfortranarray(Fi, dtype=np.float64).copy(order="F")
    ms = C.c_double()
    rc = lib().fctn_selftest_chol(int(device), S, H1, G.ctypes.data_as(C.c_void_p), mu.ctypes.data_as(C.c_void_p),
                                  fr.ctypes.data_as(C.c_void_p), fi.ctypes.data_as(C.c_void_p), int(reps),
                                  C.byref(ms))
    check(rc)
    return fr, fi, float(ms.value)


def selftest_eigh(G, V0=None, reps=1, device=0):
    """G = V diag(phi) V^T on the device (eigh.cu); returns (V, phi, best ms,
    Jacobi sweeps).  V0: warm-start basis (identity by default)."""
    G = np.asfortranarray(G, dtype=np.float64)
    S = G.shape[0]
    V = np.asfortranarray(np.eye(S) if V0 is None else V0, dtype=np.float64).copy(order="F")
    phi = np.zeros(S)
    ms = C.c_double()
    sw = C.c_int()
    rc = lib().fctn_selftest_eigh(int(device), S, G.ctypes.data_as(C.c_void_p), V.ctypes.data_as(C.c_void_p),
                                  phi.ctypes.data_as(C.c_void_p), int(reps), C.byref(ms), C.byref(sw))
    check(rc)
    return V, phi, float(ms.value), int(sw.value)


class Context:
    """Owns one device context (one GPU, one CUDA stream)."""

    def __init__(self, device, dtype: int, dims, rank_tri, lams, deltas, sign: int, rho: float,
                 algorithm: int, cache_budget: int, numeric_exc=None):
        self._numeric = numeric_exc
        L = lib()
        self.dims = tuple(int(d) for d in dims)
        self.n = len(self.dims)
        self.dtype = dtype
        self.np_dtype = np.float64 if dtype == F64 else np.float32
        d, dp = _i64(self.dims)
        r, rp = _i64(rank_tri)
        lm, lp = _f64(lams)
        dl, dlp = _f64(deltas)
        h = C.c_void_p()
        rc = L.fctn_create(int(device), dtype, self.n, dp, rp, lp, dlp, sign, float(rho), algorithm,
                           int(cache_budget), C.byref(h))
        if rc:
            msg = L.fctn_last_error(None).decode()
            if rc == 1:
                raise ValueError(msg)
            raise NativeError(msg)
        self.h = h
        self.rank_tri = tuple(int(v) for v in rank_tri)
        self._stats = np.zeros(ST_COUNT, dtype=np.float64)
        self._counters = np.zeros(CT_COUNT, dtype=np.int64)

    def _check(self, rc):
        check(rc, self.h, self._numeric)

    def close(self):
        if getattr(self, "h", None):
            lib().fctn_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def upload(self, values: np.ndarray, mask: np.ndarray):
        if tuple(values.shape) != self.dims or tuple(mask.shape) != self.dims:
            raise ValueError(f"expected a tensor of extents {self.dims} (this rank's slab), got {values.shape}")
        x = np.asfortranarray(values, dtype=self.np_dtype)
        m = np.asfortranarray(mask, dtype=np.uint8)
        self._check(lib().fctn_upload(self.h, x.ctypes.data_as(C.c_void_p), m.ctypes.data_as(C.c_void_p)))

    def upload_f64(self, values: np.ndarray, mask: np.ndarray):
        """fp64 values (F order) and a bool/uint8 mask; the fp32 variant converts
        on the device (no host-side cast pass)."""
        if tuple(values.shape) != self.dims or tuple(mask.shape) != self.dims:
            raise ValueError(f"expected a tensor of extents {self.dims} (this rank's slab), got {values.shape}")
        x = np.asfortranarray(values, dtype=np.float64)
        m = np.asfortranarray(mask)
        m = m.view(np.uint8) if m.dtype == np.bool_ else np.asfortranarray(m, dtype=np.uint8)
        self._check(lib().fctn_upload_f64(self.h, x.ctypes.data_as(C.c_void_p), m.ctypes.data_as(C.c_void_p)))

    def get_x_f64(self) -> np.ndarray:
        out = _host_empty(self.dims)
        self._check(lib().fctn_get_x_f64(self.h, out.ctypes.data_as(C.c_void_p)))
        return out

    def set_rank(self, rank_tri):
        r, rp = _i64(rank_tri)
        self._check(lib().fctn_set_rank(self.h, rp))
        self.rank_tri = tuple(int(v) for v in rank_tri)

    def set_factors(self, unfoldings, versions, reset_cache: bool):
        arrs = [np.asfortranarray(a, dtype=np.float64) for a in unfoldings]
        ptrs = (C.c_void_p * self.n)(*[a.ctypes.data for a in arrs])
        v, vp = _i64(versions)
        self._check(lib().fctn_set_factors(self.h, ptrs, vp, int(bool(reset_cache))))

    def get_factors(self, shapes):
        arrs = [np.empty(s, dtype=np.float64, order="F") for s in shapes]
        ptrs = (C.c_void_p * self.n)(*[a.ctypes.data for a in arrs])
        self._check(lib().fctn_get_factors(self.h, ptrs))
        return arrs

    def get_x(self) -> np.ndarray:
        out = np.empty(self.dims, dtype=self.np_dtype, order="F")
        self._check(lib().fctn_get_x(self.h, out.ctypes.data_as(C.c_void_p)))
        return out

    def objective(self):
        v = C.c_double()
        ct = np.zeros(CT_COUNT, dtype=np.int64)
        self._check(lib().fctn_objective(self.h, C.byref(v), ct.ctypes.data_as(C.POINTER(C.c_int64))))
        return float(v.value), ct

    def sweep(self, order, extrapolation=None):
        o = np.ascontiguousarray(np.asarray(order, dtype=np.int32))
        ex, a, b = (0, 0.0, 0.0) if extrapolation is None else (1, float(extrapolation[0]), float(extrapolation[1]))
        self._check(lib().fctn_sweep(self.h, o.ctypes.data_as(C.POINTER(C.c_int32)), ex, a, b,
                                     self._stats.ctypes.data_as(C.POINTER(C.c_double)),
                                     self._counters.ctypes.data_as(C.POINTER(C.c_int64))))
        return self._stats.copy(), self._counters.copy()

    def sync(self):
        self._check(lib().fctn_sync(self.h))

    def quality(self, truth: np.ndarray, use_mask: bool, peak: float = 1.0) -> np.ndarray:
        """Raw quality sums (FCTN_Q_*) of the resident X against a host truth
        tensor (this rank's slab when sharded)."""
        if tuple(truth.shape) != self.dims:
            raise ValueError("tensors must have identical shapes")
        t = truth if truth.dtype in (np.float32, np.float64) else truth.astype(np.float64)
        t = np.asfortranarray(t)
        out = np.zeros(Q_COUNT, dtype=np.float64)
        self._check(lib().fctn_quality_ctx(self.h, t.ctypes.data_as(C.c_void_p), F32 if t.dtype == np.float32 else F64,
                                           int(bool(use_mask)), float(peak),
                                           out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def set_comm_nccl(self, uid: bytes, rank: int, nranks: int):
        lo, hi = slab_of(self.dims[0], rank, nranks)
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        self._check(lib().fctn_set_comm(self.h, buf, rank, nranks, lo, hi))
        self._set_slab(lo, hi)

    def set_comm_loopback(self, rank: int, nranks: int):
        """Device-side loop-back collectives (timing model / tests): this rank's
        slab with every kernel at its nranks-GPU shape, sweeps graph-replayed."""
        lo, hi = slab_of(self.dims[0], rank, nranks)
        self._check(lib().fctn_set_comm_loopback(self.h, rank, nranks, lo, hi))
        self._set_slab(lo, hi)

    def set_comm_host(self, allreduce, allgather, rank: int, nranks: int):
        """allreduce(np.ndarray) sums in place across ranks; allgather(send) ->
        np.ndarray of nranks*len(send) in rank order.  Both on float64."""
        lo, hi = slab_of(self.dims[0], rank, nranks)

        def _ar(_u, ptr, n):
            try:
                a = np.ctypeslib.as_array(ptr, shape=(n,))
                allreduce(a)
                return 0
            except Exception:  # pragma: no cover
                return 1

        def _ag(_u, sptr, rptr, n):
            try:
                snd = np.ctypeslib.as_array(sptr, shape=(n,))
                rcv = np.ctypeslib.as_array(rptr, shape=(n * nranks,))
                rcv[:] = allgather(snd.copy())
                return 0
            except Exception:  # pragma: no cover
                return 1

        self._host_cbs = (HOST_ALLREDUCE(_ar), HOST_ALLGATHER(_ag))  # keep alive
        self._check(lib().fctn_set_comm_host(self.h, self._host_cbs[0], self._host_cbs[1], None, rank, nranks, lo,
                                             hi))
        self._set_slab(lo, hi)

    def _set_slab(self, lo, hi):
        self.slab = (lo, hi)
        self.dims = (hi - lo,) + self.dims[1:]

    def timer_start(self):
        self._check(lib().fctn_timer(self.h, 0, None))

    def timer_stop(self) -> float:
        v = C.c_double()
        self._check(lib().fctn_timer(self.h, 1, C.byref(v)))
        return float(v.value)

    def set_profiling(self, on: bool):
        self._check(lib().fctn_set_profiling(self.h, int(bool(on))))

    def get_profile(self) -> dict:
        ms = np.zeros(12)
        n = np.zeros(12, dtype=np.int64)
        b = np.zeros(12)
        self._check(lib().fctn_get_profile(self.h, ms.ctypes.data_as(C.POINTER(C.c_double)),
                                           n.ctypes.data_as(C.POINTER(C.c_int64)),
                                           b.ctypes.data_as(C.POINTER(C.c_double))))
        return {K_CLASSES[i]: {"ms": float(ms[i]), "launches": int(n[i]), "bytes": float(b[i])}
                for i in range(12) if n[i] > 0}
