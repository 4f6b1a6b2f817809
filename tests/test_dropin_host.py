"""CPU: the drop-in headers' host side (include/xqr/*.hpp) against the
reference compiled in place (oracle/_ref) -- no GPU needed.

* the value types' operators (double_double / quad_double + - * / sqrt
  renormalize, cplx * / +; double_double.hpp:41-122, quad_double.hpp:216-370,
  complex.hpp:26-65), bit for bit and exception for exception, over every
  operand class of tests/arith_cases.py;
* mgs_qr driven through the detail:: building blocks (mgs.hpp:36-80) the way
  the reference's own tests drive them (test_mgs.cpp:120-146), against the
  reference's mgs_qr;
* to_double_double / real_cast / abs2 / cabs (quad_double.hpp:30-34,
  real_type.hpp:50-73, complex.hpp:77-85);
* the reference's unmodified experiment.hpp compiles against include/ with no
  other reference header (the GPU suite runs it: test_dropin_gpu.py).
"""
import ctypes
import os
import subprocess

import numpy as np
import pytest

from arith_cases import operand_pairs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "host_ops.cpp")
LIB = os.path.join(ROOT, "tests", "cpp", "_build", "libxqr_hostops.so")
INC = os.path.join(ROOT, "include")
REF_INC = "/root/reference/proj/include"
dp = ctypes.POINTER(ctypes.c_double)


@pytest.fixture(scope="module")
def hostops():
    deps = [SRC] + [os.path.join(dp_, f) for dp_, _, fs in os.walk(INC) for f in fs]
    deps.append(os.path.join(ROOT, "paper_1210_0800_b200", "csrc", "xarith.cuh"))
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(d) for d in deps):
        os.makedirs(os.path.dirname(LIB), exist_ok=True)
        subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-I", INC, SRC,
                        "-o", LIB], check=True)
    lib = ctypes.CDLL(LIB)
    lib.xq_arith.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, dp, dp, dp,
                             ctypes.POINTER(ctypes.c_int32)]
    lib.xq_mgs_by_parts.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, dp, dp, dp]
    lib.xq_misc.argtypes = [dp, dp, dp]
    return lib


def _arith(lib, limbs, op, a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    out = np.zeros_like(a)
    stride = 2 * limbs if 5 <= op <= 7 else limbs
    count = a.size // stride
    codes = np.zeros(count, dtype=np.int32)
    lib.xq_arith(limbs, op, count, a.ctypes.data_as(dp), b.ctypes.data_as(dp), out.ctypes.data_as(dp),
                 codes.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    return out, codes


@pytest.mark.parametrize("L", [1, 2, 4])
@pytest.mark.parametrize("op", [0, 1, 2, 3, 4, 5, 6, 7, 8])
def test_value_type_operators_equal_reference(hostops, ref, L, op):
    rng = np.random.default_rng(6200 + 10 * L + op)
    count = {0: 20000, 1: 20000, 2: 10000, 7: 10000, 8: 10000, 5: 3000}.get(op, 1500)
    cplx = 5 <= op <= 7
    a, b = operand_pairs(rng, count, L, (lambda v: ref.arith(L, 8, v)[0]) if L > 1 else (lambda v: v),
                         parts=2 if cplx else 1)
    if op == 4:
        a = np.abs(a)
    if op in (3, 6):  # division: zero divisors raise domain_error in both
        b[:16] = 0.0
    if L > 1:  # overflow raises overflow_error in both
        a[16:24, ..., 0] = 1e300
        b[16:24, ..., 0] = 1e300 if op != 3 else 1e-300
    want, wcodes = ref.arith(L, op, a, b)
    got, gcodes = _arith(hostops, L, op, a, b)
    assert np.array_equal(gcodes, wcodes), f"exceptions differ at {np.nonzero(gcodes != wcodes)[0][:5]}"
    ok = wcodes == 0
    g = got.reshape(count, -1)[ok].view(np.uint64)
    w = want.reshape(count, -1)[ok].view(np.uint64)
    bad = np.argwhere(g != w)
    assert len(bad) == 0, f"op {op} L {L}: {len(bad)} limbs differ, first row {bad[0][0]}"


@pytest.mark.parametrize("L", [1, 2, 4])
@pytest.mark.parametrize("m,n", [(8, 8), (17, 9), (33, 33)])
def test_detail_building_blocks_equal_reference_mgs(hostops, ref, L, m, n):
    a, _ = ref.gen_system(L, m, n, 1.0, 900 + m + n)
    for plant in (False, True):
        if plant:
            a = a.copy()
            a[n - 1] = a[0]  # breakdown at the last column (1-based n)
        q = np.zeros_like(a)
        r = np.zeros((n, n, 2, L))
        rc = hostops.xq_mgs_by_parts(L, m, n, a.ctypes.data_as(dp), q.ctypes.data_as(dp), r.ctypes.data_as(dp))
        wq, wr, st = ref.mgs_qr(a)
        assert rc == st[0]
        if rc == 0:
            assert np.array_equal(q.view(np.uint64), wq.view(np.uint64))
            assert np.array_equal(r.view(np.uint64), wr.view(np.uint64))


def test_casts_and_moduli(hostops, port):
    rng = np.random.default_rng(77)
    for _ in range(200):
        x = port.arith(4, 8, rng.standard_normal((1, 4)) * np.array([1, 2.0 ** -54, 2.0 ** -108, 2.0 ** -162]))[0][0]
        z = port.arith(4, 8, (rng.standard_normal((2, 4)) * np.array([1, 2.0 ** -54, 2.0 ** -108,
                                                                        2.0 ** -162])))[0].reshape(-1)
        out = np.zeros(14)
        hostops.xq_misc(np.ascontiguousarray(x).ctypes.data_as(dp), np.ascontiguousarray(z).ctypes.data_as(dp),
                        out.ctypes.data_as(dp))
        # to_double_double: two_sum of the heads, the tails folded in rounded
        s = x[0] + x[1]
        bb = s - x[0]
        e = (x[0] - (s - bb)) + (x[1] - bb)
        t = e + (x[2] + x[3])
        hi = s + t
        lo = t - (hi - s)
        assert out[0] == hi and out[1] == lo
        assert out[2] == hi and out[3] == lo and out[4] == 0.0 and out[5] == 0.0  # widening is exact
        # abs2 = re*re + im*im in quad-double; cabs = its sqrt (the port's ops)
        re, im = z[:4], z[4:]
        want = port.arith(4, 0, port.arith(4, 2, re[None], re[None])[0], port.arith(4, 2, im[None], im[None])[0])[0][0]
        assert np.array_equal(out[6:10].view(np.uint64), want.view(np.uint64))
        assert np.array_equal(out[10:14].view(np.uint64), port.arith(4, 4, want[None])[0][0].view(np.uint64))


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="needs the reference tree")
def test_reference_experiment_compiles_against_dropin(tmp_path):
    """The unmodified experiment.hpp (the hot path's harness caller,
    SURVEY.md §8b) compiles against include/, and every other xqr header it
    pulls in resolves to include/, not to the reference."""
    src = tmp_path / "t.cpp"
    src.write_text('#include "xqr/experiment.hpp"\nint main() { return 0; }\n')
    p = subprocess.run(["g++", "-std=c++20", "-ffp-contract=off", "-fsyntax-only", "-H", "-I", INC, "-I", REF_INC,
                        str(src)], capture_output=True, text=True)
    assert p.returncode == 0, p.stderr[-2000:]
    xqr_headers = [ln.split()[-1] for ln in p.stderr.splitlines() if "xqr/" in ln and ln.startswith(".")]
    from_ref = [h for h in xqr_headers if h.startswith(REF_INC)]
    assert from_ref == [f"{REF_INC}/xqr/experiment.hpp"], from_ref
