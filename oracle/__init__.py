"""CPU ORACLE -- test infrastructure only.

Python (ctypes + numpy) access to

* ``_build/libxqr_oracle.so`` -- the plain-C restatement of the reference hot
  path (``xqr_oracle.c``; every function cites the reference file:line), and
* ``_ref/libxqr_ref.so`` -- the unmodified reference headers compiled in place
  (``ref_shim.cpp``), present wherever ``/root/reference`` was available at
  build time (the built .so travels to the GPU box).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module.  The product (``paper_1210_0800_b200``) never
does.

Array convention (same as the product's C ABI): a matrix is a float64 numpy
array of shape ``(n_cols, m_rows, 2, L)`` -- column-major complex entries, the
real part's L limbs then the imaginary part's -- i.e. the memory image of the
reference ``col_matrix<R>`` columns laid end to end.  A vector is
``(len, 2, L)``; a real is ``(L,)``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "_build", "libxqr_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libxqr_ref.so")
REF_LIB_V4 = os.path.join(HERE, "_ref", "libxqr_ref_v4.so")
REF_BUILD_INFO = os.path.join(HERE, "_ref", "BUILD_INFO.json")


def host_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    fl = set(line.split(":", 1)[1].split())
                    return {"avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl", "fma"} <= fl
    except OSError:
        pass
    return False


def reference_build() -> dict:
    """Which reference build reference() loads here, with its compiler and flags."""
    import json

    info = {}
    try:
        info = json.load(open(REF_BUILD_INFO))
    except (OSError, ValueError):
        pass
    v4 = os.path.exists(REF_LIB_V4) and host_has_avx512()
    return {"lib": os.path.basename(REF_LIB_V4 if v4 else REF_LIB), "compiler": info.get("compiler"),
            "flags": info.get("v4" if v4 else "portable")}
REF_INC = "/root/reference/proj/include"

_dp = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.c_int64


class Status(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("column", ctypes.c_int32), ("system", ctypes.c_int64)]


def build(ref: bool | None = None) -> None:
    """Compile the C restatement (and the reference shim when the reference
    tree is present)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref is None:
        ref = os.path.isdir(REF_INC)
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _ptr(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


class Oracle:
    """One CPU implementation of the hot path (`port` or `reference`)."""

    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_LIB if kind == "port" else (
            REF_LIB_V4 if os.path.exists(REF_LIB_V4) and host_has_avx512() else REF_LIB)
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = ctypes.CDLL(path)
        p = "xo_" if kind == "port" else "ref_"
        self._p = p
        L = self.lib
        sp = ctypes.POINTER(Status)
        ci = ctypes.c_int
        self._mgs = getattr(L, p + "mgs_qr")
        self._mgs.argtypes = [ci, _i64, _i64, _dp, _dp, _dp, sp]
        self._lsq = getattr(L, p + "lsq_solve")
        self._lsq.argtypes = [ci, _i64, _i64, _dp, _dp, _dp, _dp, sp]
        self._bs = getattr(L, p + "back_substitute")
        self._bs.argtypes = [ci, _i64, _i64, _dp, _i64, _dp, _dp, sp]
        self._res = getattr(L, p + "residual_max_entry")
        self._res.argtypes = [ci, _i64, _i64, _dp, _dp, _dp, _dp, sp]
        self._orth = getattr(L, p + "orthogonality_defect")
        self._orth.argtypes = [ci, _i64, _i64, _dp, _dp, sp]
        self._gen = getattr(L, p + "gen_system")
        self._gen.argtypes = [ci, _i64, _i64, ctypes.c_double, ctypes.c_uint64, _i64, _dp, _dp]
        self._sm = getattr(L, p + "splitmix_next")
        self._sm.argtypes = [ctypes.c_uint64, _i64, _i64, ctypes.POINTER(ctypes.c_uint64)]
        self._sm.restype = None
        self._arith = getattr(L, p + "arith")
        self._arith.argtypes = [ci, ci, _i64, _dp, _dp, _dp, ctypes.POINTER(ctypes.c_int32)]
        if kind == "reference":
            self._plsq = L.ref_par_lsq_solve
            self._plsq.argtypes = [ci, _i64, _i64, _dp, _dp, _dp, _dp, ci, sp]
            self._pmgs = L.ref_par_mgs_qr
            self._pmgs.argtypes = [ci, _i64, _i64, _dp, _dp, _dp, ci, ci, sp]
            self._acc = L.ref_accuracy_csv
            self._acc.argtypes = [ci, _i64, _i64, _dp, ci, _i64, ctypes.c_uint64, ci, ctypes.c_char_p, _i64]
            self._batch = L.ref_lsq_solve_batch
            self._batch.argtypes = [ci, _i64, _i64, _i64, _dp, _dp, _dp, _dp, ci,
                                    ctypes.POINTER(ctypes.c_int32)]

    # -- generator -----------------------------------------------------------
    def gen_system(self, limbs, m, n, g=1.0, seed=1, stream=-1, rhs=True):
        a = np.zeros((n, m, 2, limbs))
        b = np.zeros((m, 2, limbs)) if rhs else None
        rc = self._gen(limbs, m, n, g, seed, stream, _ptr(a), _ptr(b))
        if rc:
            raise ValueError(f"gen_system failed ({rc})")
        return (a, b) if rhs else a

    def splitmix(self, seed, count, stream=-1):
        out = np.zeros(count, dtype=np.uint64)
        self._sm(seed, stream, count, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
        return out

    # -- hot path ------------------------------------------------------------
    def mgs_qr(self, a):
        n, m, _, L = a.shape
        q = np.zeros_like(a)
        r = np.zeros((n, n, 2, L))
        st = Status()
        self._mgs(L, m, n, _ptr(np.ascontiguousarray(a)), _ptr(q), _ptr(r), ctypes.byref(st))
        return q, r, (st.code, st.column)

    def lsq_solve(self, a, b):
        n, m, _, L = a.shape
        x = np.zeros((n, 2, L))
        z = np.zeros(L)
        st = Status()
        self._lsq(L, m, n, _ptr(np.ascontiguousarray(a)), _ptr(np.ascontiguousarray(b)), _ptr(x),
                  _ptr(z), ctypes.byref(st))
        return x, z, (st.code, st.column)

    def par_lsq_solve(self, a, b, workers):
        n, m, _, L = a.shape
        x = np.zeros((n, 2, L))
        z = np.zeros(L)
        st = Status()
        self._plsq(L, m, n, _ptr(np.ascontiguousarray(a)), _ptr(np.ascontiguousarray(b)), _ptr(x),
                   _ptr(z), workers, ctypes.byref(st))
        return x, z, (st.code, st.column)

    def par_mgs_qr(self, a, workers, redundant=False):
        n, m, _, L = a.shape
        q = np.zeros_like(a)
        r = np.zeros((n, n, 2, L))
        st = Status()
        self._pmgs(L, m, n, _ptr(np.ascontiguousarray(a)), _ptr(q), _ptr(r), workers,
                   int(redundant), ctypes.byref(st))
        return q, r, (st.code, st.column)

    def lsq_solve_batch(self, a, b, threads):
        batch, n, m, _, L = a.shape
        x = np.zeros((batch, n, 2, L))
        z = np.zeros((batch, L))
        codes = np.zeros(batch, dtype=np.int32)
        self._batch(L, batch, m, n, _ptr(np.ascontiguousarray(a)), _ptr(np.ascontiguousarray(b)),
                    _ptr(x), _ptr(z), threads, codes.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
        return x, z, codes

    def accuracy_csv(self, limbs, m, n, g_values, trials, seed=1, linear=False):
        """The reference's run_accuracy_sweep + accuracy_csv text (reference build only)."""
        g = np.ascontiguousarray(g_values, dtype=np.float64)
        buf = ctypes.create_string_buffer(1 << 16)
        rc = self._acc(limbs, m, n, _ptr(g), len(g), trials, seed, int(linear), buf, len(buf))
        return buf.value.decode(), rc

    def back_substitute(self, r, y):
        rc_, rn, _, L = r.shape
        x = np.zeros((y.shape[0], 2, L))
        st = Status()
        self._bs(L, rn, rc_, _ptr(np.ascontiguousarray(r)), y.shape[0],
                 _ptr(np.ascontiguousarray(y)), _ptr(x), ctypes.byref(st))
        return x, (st.code, st.column)

    def residual_max_entry(self, a, q, r):
        n, m, _, L = a.shape
        out = np.zeros(L)
        st = Status()
        self._res(L, m, n, _ptr(np.ascontiguousarray(a)), _ptr(np.ascontiguousarray(q)),
                  _ptr(np.ascontiguousarray(r)), _ptr(out), ctypes.byref(st))
        return out, (st.code, st.column)

    def orthogonality_defect(self, q):
        n, m, _, L = q.shape
        out = np.zeros(L)
        st = Status()
        self._orth(L, m, n, _ptr(np.ascontiguousarray(q)), _ptr(out), ctypes.byref(st))
        return out, (st.code, st.column)

    def arith(self, limbs, op, a, b=None):
        a = np.ascontiguousarray(a, dtype=np.float64)
        out = np.zeros_like(a)
        stride = 2 * limbs if 5 <= op <= 7 else limbs
        count = a.size // stride
        codes = np.zeros(count, dtype=np.int32)
        bb = None if b is None else np.ascontiguousarray(b, dtype=np.float64)
        self._arith(limbs, op, count, _ptr(a), _ptr(bb), _ptr(out),
                    codes.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
        return out, codes


REF_IO_TOOL = os.path.join(HERE, "_ref", "ref_io_tool")


class RefIO:
    """The reference's own matrix_io / shortest (oracle/ref_io_tool.cpp, run as
    a subprocess), for the file-format tests.  Reference build only."""

    def _run(self, args, data: bytes) -> bytes:
        return subprocess.run([REF_IO_TOOL] + args, input=data, capture_output=True, check=True).stdout

    def write_matrix(self, a) -> str:
        a = np.ascontiguousarray(a, dtype=np.float64)
        n, m, _, L = a.shape
        return self._run(["write", str(L), str(m), str(n)], a.tobytes()).decode()

    def read_matrix(self, text: str):
        """(array, limbs) or raises ValueError(line)."""
        out = self._run(["read"], text.encode())
        head, _, body = out.partition(b"\n")
        tok = head.split()
        if tok[0] == b"error":
            raise ValueError(int(tok[1]))
        m, n, L = int(tok[1]), int(tok[2]), int(tok[3])
        return np.frombuffer(body, dtype=np.float64).reshape(n, m, 2, L).copy(), L

    def shortest_many(self, vals):
        out = self._run(["shortest"], np.asarray(vals, dtype=np.float64).tobytes())
        return out.decode().split("\n")[: len(vals)]


def ref_io() -> RefIO | None:
    return RefIO() if os.path.exists(REF_IO_TOOL) else None


def port() -> Oracle:
    return Oracle("port")


def reference() -> Oracle | None:
    return Oracle("reference") if os.path.exists(REF_LIB) else None
