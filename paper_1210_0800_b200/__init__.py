"""paper_1210_0800_b200 -- B200-native complex dd/qd modified Gram-Schmidt
least squares (Verschelde & Yoffe, arXiv:1210.0800), behind the reference
``xqr`` API.

Host-side mirror of the reference interface for Python callers (tests, the
bench, notebooks).  Every call goes through the C ABI of
``libxqr_b200.so`` (``include/xqr_b200.h``) into hand-written sm_100a
kernels.  There is no CPU fallback: without the built library or a CUDA
device the calls raise.

Names, argument meaning and errors follow the reference:

===========================  ======================================================
this module                  reference (``/root/reference/proj/include/xqr``)
===========================  ======================================================
``mgs_qr(a)``                ``mgs_qr<R>(col_matrix<R>)``            mgs.hpp:84-106
``lsq_solve(a, b)``          ``lsq_solve<R>(a, b)``                  mgs.hpp:131-158
``back_substitute(r, y)``    ``back_substitute<R>(r, y)``            mgs.hpp:110-126
``par_mgs_qr(a, w, mode)``   ``par_mgs_qr(a, workers, mode)``        parallel.hpp:35-99
``par_lsq_solve(a, b, w)``   ``par_lsq_solve(a, b, workers)``        parallel.hpp:105-153
``par_back_substitute``      ``par_back_substitute(r, y, workers)``  parallel.hpp:157-183
``breakdown_error`` ...      ``errors.hpp:13-51``
===========================  ======================================================

Array convention: a matrix is a float64 array of shape ``(n_cols, m_rows, 2,
L)`` (column-major complex entries; real limbs then imaginary limbs) -- the
memory image of ``col_matrix<R>``; a vector is ``(len, 2, L)``; a real is
``(L,)``.  L = 1 (double), 2 (double_double), 4 (quad_double).
"""
from __future__ import annotations

import ctypes
import math
import os
import threading

import numpy as np

__all__ = [
    "error", "overflow_error", "domain_error", "dimension_error", "breakdown_error",
    "usage_error", "cuda_error", "normalize_mode", "Context", "context", "library_path",
    "mgs_qr", "lsq_solve", "back_substitute", "par_mgs_qr", "par_lsq_solve",
    "par_back_substitute", "mgs_qr_batched", "lsq_solve_batched", "arith", "real_traits",
    "residual_max_entry", "orthogonality_defect", "residual_max_entry_batched",
    "orthogonality_defect_batched", "accuracy_sweep", "gen_systems",
]

HERE = os.path.dirname(os.path.abspath(__file__))
library_path = os.environ.get("XQR_B200_LIB") or os.path.join(HERE, "libxqr_b200.so")


# ---- errors (errors.hpp:13-51) ------------------------------------------------
class error(RuntimeError):
    """Base class of everything the library raises (errors.hpp:13-16)."""


class overflow_error(error):
    """A finite-precision operation left the representable range (errors.hpp:19-22)."""


class domain_error(error):
    """Invalid operand: division by zero, ... (errors.hpp:24-27)."""


class dimension_error(error):
    """Operand shapes disagree (errors.hpp:29-32)."""


class breakdown_error(error):
    """Rank deficiency while orthogonalizing; ``column`` is 1-based (errors.hpp:34-41)."""

    def __init__(self, column: int):
        super().__init__(f"orthogonalization breakdown at column {column}")
        self.column = column


class usage_error(error):
    """Bad arguments or configuration (errors.hpp:49-52)."""


class cuda_error(error):
    """CUDA runtime failure (no reference counterpart: the reference is CPU-only)."""


XQR_OK, XQR_BREAKDOWN, XQR_OVERFLOW, XQR_DOMAIN, XQR_DIMENSION, XQR_USAGE, XQR_CUDA = (
    0, 1, 2, 3, 4, 5, 16)


def _raise(code: int, column: int = 0, what: str = "") -> None:
    if code == XQR_OK:
        return
    if code == XQR_BREAKDOWN:
        raise breakdown_error(column)
    if code == XQR_OVERFLOW:
        raise overflow_error(what or "overflow")
    if code == XQR_DOMAIN:
        raise domain_error(what or "domain error")
    if code == XQR_DIMENSION:
        raise dimension_error(what or "dimension mismatch")
    if code == XQR_USAGE:
        raise usage_error(what or "usage error")
    raise cuda_error(what or f"CUDA failure ({code})")


class normalize_mode:
    """parallel.hpp:23.  Both modes give bitwise-identical factors; the
    device always normalises the pivot once."""

    designated = "designated"
    redundant = "redundant"


class real_traits:
    """real_type.hpp:22-47, indexed by limb count."""

    name = {1: "d", 2: "dd", 4: "qd"}
    decimal_digits = {1: 15, 2: 31, 4: 62}
    epsilon = {1: 2.0 ** -52, 2: 2.0 ** -104, 4: 2.0 ** -209}


# ---- C ABI ----------------------------------------------------------------------
class xqr_status(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("column", ctypes.c_int32), ("system", ctypes.c_int64)]


_dp = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_ci = ctypes.c_int
_sp = ctypes.POINTER(xqr_status)

_lib = None
_lib_lock = threading.Lock()

_SIGNATURES = {
    "xqr_version": ([], _ci),
    "xqr_ctx_create": ([_ci, ctypes.POINTER(_vp)], _ci),
    "xqr_ctx_destroy": ([_vp], None),
    "xqr_ctx_set_stream": ([_vp, _vp], _ci),
    "xqr_ctx_stream": ([_vp], _vp),
    "xqr_ctx_synchronize": ([_vp], _ci),
    "xqr_ctx_last_error": ([_vp], ctypes.c_char_p),
    "xqr_mgs_qr": ([_vp, _ci, _i64, _i64, _dp, _dp, _dp, _sp], _ci),
    "xqr_lsq_solve": ([_vp, _ci, _i64, _i64, _dp, _dp, _dp, _dp, _sp], _ci),
    "xqr_back_substitute": ([_vp, _ci, _i64, _i64, _dp, _i64, _dp, _dp, _sp], _ci),
    "xqr_mgs_qr_batched": ([_vp, _ci, _i64, _i64, _i64, _dp, _dp, _dp, _sp], _ci),
    "xqr_lsq_solve_batched": ([_vp, _ci, _i64, _i64, _i64, _dp, _dp, _dp, _dp, _sp], _ci),
    "xqr_mgs_qr_batched_device": ([_vp, _ci, _i64, _i64, _i64, _vp, _vp, _vp, _vp], _ci),
    "xqr_lsq_solve_batched_device": ([_vp, _ci, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp], _ci),
    "xqr_back_substitute_batched_device": ([_vp, _ci, _i64, _i64, _vp, _vp, _vp, _vp], _ci),
    "xqr_arith": ([_vp, _ci, _ci, _i64, _dp, _dp, _dp, ctypes.POINTER(ctypes.c_int32)], _ci),
    "xqr_residual_max_entry": ([_vp, _ci, _i64, _i64, _dp, _dp, _dp, _dp, _sp], _ci),
    "xqr_orthogonality_defect": ([_vp, _ci, _i64, _i64, _dp, _dp, _sp], _ci),
    "xqr_residual_max_entry_batched": ([_vp, _ci, _i64, _i64, _i64, _dp, _dp, _dp, _dp, _sp], _ci),
    "xqr_orthogonality_defect_batched": ([_vp, _ci, _i64, _i64, _i64, _dp, _dp, _sp], _ci),
    "xqr_residual_max_entry_batched_device": ([_vp, _ci, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp], _ci),
    "xqr_orthogonality_defect_batched_device": ([_vp, _ci, _i64, _i64, _i64, _vp, _vp, _vp], _ci),
    "xqr_gen_systems": ([_ci, _i64, _i64, _i64, ctypes.c_double, ctypes.c_uint64, _i64, _ci, _dp,
                         _dp], _ci),
    "xqr_gen_systems_dist": ([_ci, _i64, _i64, _i64, ctypes.c_double, _ci, ctypes.c_uint64, _i64, _ci,
                              _dp, _dp], _ci),
    "xqr_ctx_launch_count": ([_vp], _i64),
    "xqr_ctx_grid_fallbacks": ([_vp], _i64),
    "xqr_fp64_peak": ([_vp, _ci, _dp], _ci),
    "xqr_ctx_last_kernel_ms": ([_vp], ctypes.c_float),
}


def load_library() -> ctypes.CDLL:
    """Load ``libxqr_b200.so`` (built in-tree by ``__graft_entry__.build()``).
    Raises if it is missing -- there is no fallback."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(library_path):
                raise cuda_error(f"{library_path} is not built; run __graft_entry__.build()")
            lib = ctypes.CDLL(library_path)
            for name, (args, res) in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


class Context:
    """One CUDA device + stream + workspace (``xqr_ctx``).  Single-threaded,
    like the C ABI; :func:`context` hands out one per (thread, device)."""

    def __init__(self, device: int = 0):
        lib = load_library()
        h = _vp()
        rc = lib.xqr_ctx_create(device, ctypes.byref(h))
        if rc:
            raise cuda_error(f"xqr_ctx_create(device={device}) failed ({rc})")
        self._lib = lib
        self.handle = h
        self.device = device

    def close(self):
        if self.handle:
            self._lib.xqr_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def last_error(self) -> str:
        return (self._lib.xqr_ctx_last_error(self.handle) or b"").decode()

    def set_stream(self, stream_ptr: int):
        self._lib.xqr_ctx_set_stream(self.handle, _vp(stream_ptr))

    def synchronize(self):
        rc = self._lib.xqr_ctx_synchronize(self.handle)
        if rc:
            _raise(rc, what=self.last_error())

    @property
    def launch_count(self) -> int:
        return int(self._lib.xqr_ctx_launch_count(self.handle))

    def fp64_peak(self, op: int = 0) -> float:
        """Measured FP64 lane-instructions/s of this device (op 0: DADD, 1: DFMA)."""
        v = ctypes.c_double()
        rc = self._lib.xqr_fp64_peak(self.handle, op, ctypes.byref(v))
        self.check(rc)
        return float(v.value)

    @property
    def grid_fallbacks(self) -> int:
        """Single systems re-routed to the one-CTA kernel (grid not placeable)."""
        return int(self._lib.xqr_ctx_grid_fallbacks(self.handle))

    @property
    def last_kernel_ms(self) -> float:
        return float(self._lib.xqr_ctx_last_kernel_ms(self.handle))

    def check(self, rc: int, st: xqr_status | None = None):
        if rc:
            col = st.column if st is not None else 0
            _raise(rc, col, self.last_error())

    # device-pointer entry points (asynchronous on the ctx stream)
    def lsq_solve_batched_device(self, limbs, batch, m, n, d_a, d_b, d_x, d_z, d_st):
        rc = self._lib.xqr_lsq_solve_batched_device(self.handle, limbs, batch, m, n, _vp(d_a),
                                                    _vp(d_b), _vp(d_x), _vp(d_z), _vp(d_st))
        self.check(rc)

    def mgs_qr_batched_device(self, limbs, batch, m, n, d_a, d_q, d_r, d_st):
        rc = self._lib.xqr_mgs_qr_batched_device(self.handle, limbs, batch, m, n, _vp(d_a),
                                                 _vp(d_q), _vp(d_r), _vp(d_st))
        self.check(rc)


_tls = threading.local()


def context(device: int = 0) -> Context:
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


def _f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(_dp)


def _limbs_of(a) -> int:
    L = a.shape[-1]
    if L not in (1, 2, 4):
        raise usage_error("limb count must be 1, 2 or 4")
    return L


# ---- the reference API ----------------------------------------------------------
def mgs_qr(a, device: int = 0):
    """mgs.hpp:84-106.  Returns (q, r): q (n, m, 2, L), r (n, n, 2, L)."""
    if a.ndim != 4 or a.shape[2] != 2:
        raise dimension_error("matrix must have shape (n, m, 2, L)")
    n, m, _, L = a.shape
    _limbs_of(a)
    ctx = context(device)
    a, pa = _f64(a)
    q = np.zeros_like(a)
    r = np.zeros((n, n, 2, L))
    st = xqr_status()
    rc = ctx._lib.xqr_mgs_qr(ctx.handle, L, m, n, pa, q.ctypes.data_as(_dp), r.ctypes.data_as(_dp),
                             ctypes.byref(st))
    ctx.check(rc, st)
    return q, r


def lsq_solve(a, b, device: int = 0):
    """mgs.hpp:131-158.  Returns (x, z): x (n, 2, L), z = residual norm (L,)."""
    if a.ndim != 4 or a.shape[2] != 2:
        raise dimension_error("matrix must have shape (n, m, 2, L)")
    n, m, _, L = a.shape
    _limbs_of(a)
    if b.shape != (m, 2, L):
        raise dimension_error("right-hand side length mismatch")
    ctx = context(device)
    a, pa = _f64(a)
    b, pb = _f64(b)
    x = np.zeros((n, 2, L))
    z = np.zeros(L)
    st = xqr_status()
    rc = ctx._lib.xqr_lsq_solve(ctx.handle, L, m, n, pa, pb, x.ctypes.data_as(_dp),
                                z.ctypes.data_as(_dp), ctypes.byref(st))
    ctx.check(rc, st)
    return x, z


def back_substitute(r, y, device: int = 0):
    """mgs.hpp:110-126.  r (cols, rows, 2, L) upper triangular, y (n, 2, L)."""
    cols, rows, _, L = r.shape
    _limbs_of(r)
    ctx = context(device)
    r, pr = _f64(r)
    y, py = _f64(y)
    x = np.zeros((y.shape[0], 2, L))
    st = xqr_status()
    rc = ctx._lib.xqr_back_substitute(ctx.handle, L, rows, cols, pr, y.shape[0], py,
                                      x.ctypes.data_as(_dp), ctypes.byref(st))
    ctx.check(rc, st)
    return x


def residual_max_entry(a, q, r, device: int = 0):
    """mgs.hpp:161-178: max entry modulus of A - QR (working precision).
    a, q (n, m, 2, L); r (n, n, 2, L).  Returns an (L,) array."""
    n, m, _, L = a.shape
    if q.shape != a.shape or r.shape != (n, n, 2, L):
        raise dimension_error("factor shapes do not match the input matrix")
    ctx = context(device)
    a, pa = _f64(a)
    q, pq = _f64(q)
    r, pr = _f64(r)
    out = np.zeros(L)
    st = xqr_status()
    rc = ctx._lib.xqr_residual_max_entry(ctx.handle, L, m, n, pa, pq, pr, out.ctypes.data_as(_dp),
                                         ctypes.byref(st))
    ctx.check(rc, st)
    return out


def orthogonality_defect(q, device: int = 0):
    """mgs.hpp:208-222: max entry modulus of Q^H Q - I (tree inner products)."""
    n, m, _, L = q.shape
    ctx = context(device)
    q, pq = _f64(q)
    out = np.zeros(L)
    st = xqr_status()
    rc = ctx._lib.xqr_orthogonality_defect(ctx.handle, L, m, n, pq, out.ctypes.data_as(_dp),
                                           ctypes.byref(st))
    ctx.check(rc, st)
    return out


def residual_max_entry_batched(a, q, r, device: int = 0):
    """Batched residual_max_entry: a, q (batch, n, m, 2, L), r (batch, n, n, 2, L);
    returns (out (batch, L), codes)."""
    batch, n, m, _, L = a.shape
    ctx = context(device)
    a, pa = _f64(a)
    q, pq = _f64(q)
    r, pr = _f64(r)
    out = np.zeros((batch, L))
    st = (xqr_status * max(batch, 1))()
    rc = ctx._lib.xqr_residual_max_entry_batched(ctx.handle, L, batch, m, n, pa, pq, pr,
                                                 out.ctypes.data_as(_dp), st)
    if rc >= XQR_DIMENSION:  # shape, usage, device: the whole call
        _raise(rc, 0, ctx.last_error())
    return out, np.array([st[i].code for i in range(batch)], dtype=np.int32)


def orthogonality_defect_batched(q, device: int = 0):
    batch, n, m, _, L = q.shape
    ctx = context(device)
    q, pq = _f64(q)
    out = np.zeros((batch, L))
    st = (xqr_status * max(batch, 1))()
    rc = ctx._lib.xqr_orthogonality_defect_batched(ctx.handle, L, batch, m, n, pq,
                                                   out.ctypes.data_as(_dp), st)
    if rc >= XQR_DIMENSION:  # shape, usage, device: the whole call
        _raise(rc, 0, ctx.last_error())
    return out, np.array([st[i].code for i in range(batch)], dtype=np.int32)


def _check_workers(workers):
    # worker_pool(0) throws usage_error (worker_pool.hpp:26)
    if int(workers) < 1:
        raise usage_error("worker count must be at least 1")


def par_mgs_qr(a, workers, mode=normalize_mode.designated, device: int = 0):
    """parallel.hpp:35-99: bitwise equal to mgs_qr; the device decomposition
    replaces the worker pool, so `workers` and `mode` only get validated."""
    _check_workers(workers)
    if mode not in (normalize_mode.designated, normalize_mode.redundant):
        raise usage_error("unknown normalize_mode")
    return mgs_qr(a, device)


def par_lsq_solve(a, b, workers, device: int = 0):
    """parallel.hpp:105-153."""
    _check_workers(workers)
    return lsq_solve(a, b, device)


def par_back_substitute(r, y, workers, device: int = 0):
    """parallel.hpp:157-183."""
    _check_workers(workers)
    return back_substitute(r, y, device)


def lsq_solve_batched(a, b, device: int = 0, raise_first: bool = False):
    """Many independent systems of one shape: a (batch, n, m, 2, L), b (batch,
    m, 2, L).  Returns (x, z, codes, columns).  Failed systems keep their
    status instead of raising unless raise_first."""
    batch, n, m, _, L = a.shape
    ctx = context(device)
    a, pa = _f64(a)
    b, pb = _f64(b)
    x = np.zeros((batch, n, 2, L))
    z = np.zeros((batch, L))
    st = (xqr_status * max(batch, 1))()
    rc = ctx._lib.xqr_lsq_solve_batched(ctx.handle, L, batch, m, n, pa, pb, x.ctypes.data_as(_dp),
                                        z.ctypes.data_as(_dp), st)
    codes = np.array([st[i].code for i in range(batch)], dtype=np.int32)
    cols = np.array([st[i].column for i in range(batch)], dtype=np.int32)
    if rc and (raise_first or rc >= XQR_DIMENSION):  # shape, usage, device: the whole call
        i = int(np.nonzero(codes)[0][0]) if codes.any() else 0
        _raise(rc, int(cols[i]) if batch else 0, ctx.last_error())
    return x, z, codes, cols


def mgs_qr_batched(a, device: int = 0, raise_first: bool = False):
    """a (batch, n, m, 2, L) -> (q, r, codes, columns)."""
    batch, n, m, _, L = a.shape
    ctx = context(device)
    a, pa = _f64(a)
    q = np.zeros_like(a)
    r = np.zeros((batch, n, n, 2, L))
    st = (xqr_status * max(batch, 1))()
    rc = ctx._lib.xqr_mgs_qr_batched(ctx.handle, L, batch, m, n, pa, q.ctypes.data_as(_dp),
                                     r.ctypes.data_as(_dp), st)
    codes = np.array([st[i].code for i in range(batch)], dtype=np.int32)
    cols = np.array([st[i].column for i in range(batch)], dtype=np.int32)
    if rc and (raise_first or rc >= XQR_DIMENSION):  # shape, usage, device: the whole call
        i = int(np.nonzero(codes)[0][0]) if codes.any() else 0
        _raise(rc, int(cols[i]) if batch else 0, ctx.last_error())
    return q, r, codes, cols


MODULUS_DIST = {"log": 0, "linear": 1}  # random.hpp:44 modulus_dist


def gen_systems(limbs: int, batch: int, m: int, n: int, g: float = 1.0, seed: int = 1,
                first_stream: int = 0, threads: int | None = None, rhs: bool = True,
                dist: str = "log"):
    """The reference generator (experiment.hpp:64-79) on the host: returns
    a (batch, n, m, 2, L) and b (batch, m, 2, L).  first_stream=-1 draws one
    system from split_mix64(seed) itself (the reference's single-system
    experiments); otherwise system s uses split_mix64(seed).split(first_stream+s).
    dist: "log" (log-uniform modulus, the default) or "linear" (random.hpp:57-71)."""
    lib = load_library()
    if dist not in MODULUS_DIST:
        raise usage_error(f"unknown modulus distribution '{dist}'")
    a = np.zeros((batch, n, m, 2, limbs))
    b = np.zeros((batch, m, 2, limbs)) if rhs else None
    threads = threads or min(32, os.cpu_count() or 1)
    rc = lib.xqr_gen_systems_dist(limbs, batch, m, n, g, MODULUS_DIST[dist], seed, first_stream, threads,
                                  a.ctypes.data_as(_dp), b.ctypes.data_as(_dp) if rhs else None)
    if rc:
        _raise(rc, what="gen_systems")
    return (a, b) if rhs else a


def accuracy_sweep(limbs: int, m: int = 32, n: int = 32, g_values=(1.0,), trials: int = 100,
                   seed: int = 1, device: int = 0, dist: str = "log"):
    """The reference's accuracy sweep (run_accuracy_sweep, experiment.hpp:117-176,
    paper Table 2) on the device: for each g (index gi), `trials` matrices
    drawn from split_mix64(seed).split(gi*trials + t), mgs_qr of each (one
    batched launch), e = residual_max_entry (device metric), log10(e's
    leading limb).  As in the reference's trial loop, only breakdown_error
    excludes a trial (counted in `exclusions`); any other error -- of the
    factorisation or of the residual metric -- propagates, the first one in
    trial order.  Returns one dict per g: g, trials (completed),
    exclusions, m_e = min log10 e, M_e = max log10 e, D_e = m_e - M_e,
    log10_e (per completed trial), wall_seconds (GPU generation excluded:
    host generation + solve + metric)."""
    import time

    if trials < 1:
        raise usage_error("trials must be at least 1")
    if m < n or n < 1:
        raise usage_error("need rows >= cols >= 1")
    out = []
    for gi, g in enumerate(g_values):
        t0 = time.perf_counter()
        a = gen_systems(limbs, trials, m, n, float(g), seed, gi * trials, rhs=False, dist=dist)
        q, r, codes, cols = mgs_qr_batched(a, device=device)
        keep = codes == 0
        e = np.zeros((trials, limbs))
        ecodes = np.zeros(trials, dtype=np.int32)
        if keep.any():
            e[keep], ecodes[keep] = residual_max_entry_batched(a[keep], q[keep], r[keep], device=device)
        # the reference's loop raises at the first trial whose factorisation
        # fails with anything but a breakdown, or whose metric fails
        bad = ((codes != XQR_OK) & (codes != XQR_BREAKDOWN)) | (ecodes != XQR_OK)
        if bad.any():
            t = int(np.nonzero(bad)[0][0])
            code = int(codes[t]) if codes[t] != XQR_OK else int(ecodes[t])
            _raise(code, int(cols[t]), f"accuracy trial {t} (g={g})")
        # std::log10 of the leading limb (experiment.hpp:130): C libm's log10, as
        # math.log10 calls it (numpy's vectorised log10 can differ by an ulp)
        log10_e = np.array([math.log10(v) for v in e[keep, 0]], dtype=np.float64)
        rec = {"g": float(g), "m": m, "n": n, "limbs": limbs, "trials": int(keep.sum()),
               "exclusions": int((codes == XQR_BREAKDOWN).sum()), "log10_e": log10_e.tolist()}
        if len(log10_e):
            rec["m_e"] = float(log10_e.min())
            rec["M_e"] = float(log10_e.max())
            rec["D_e"] = rec["m_e"] - rec["M_e"]
        else:
            rec["m_e"] = rec["M_e"] = rec["D_e"] = float("nan")
        rec["wall_seconds"] = time.perf_counter() - t0
        out.append(rec)
    return out


def arith(limbs: int, op: int, a, b=None, device: int = 0):
    """Elementwise device arithmetic (test instrumentation): op codes as
    ``xqr_arith``.  Returns (out, codes)."""
    ctx = context(device)
    a, pa = _f64(a)
    pb = None
    if b is not None:
        b, pb = _f64(b)
    stride = 2 * limbs if 5 <= op <= 7 else limbs
    count = a.size // stride
    out = np.zeros_like(a)
    codes = np.zeros(count, dtype=np.int32)
    rc = ctx._lib.xqr_arith(ctx.handle, limbs, op, count, pa, pb, out.ctypes.data_as(_dp),
                            codes.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    ctx.check(rc)
    return out, codes
