"""CPU: the product's device arithmetic source (csrc/xarith*.cuh), compiled for
the host, against the oracle -- bit for bit, every op, every operand class
(tests/arith_cases.py).  Lets arithmetic changes be proven on the CPU before
they reach the GPU; the GPU suite repeats the check on the device build."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

from arith_cases import operand_pairs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "arith_host.cpp")
LIB = os.path.join(ROOT, "tests", "cpp", "_build", "libxarith_host.so")
CSRC = os.path.join(ROOT, "paper_1210_0800_b200", "csrc")


@pytest.fixture(scope="module", params=[0, 1, 2], ids=["batched-build", "grid-build", "register-build"])
def host(request):
    """The arithmetic as the batched kernels compile it (-DXB_XSMEM=1: the
    merge's output slots in memory), as the single-system kernels do
    (-DXB_SHIFT_TAIL=1: in-place leftover folds after shifted merges), and
    the plain register form."""
    lib_path = {0: LIB.replace(".so", "_xs.so"), 1: LIB.replace(".so", "_tail.so"), 2: LIB}[request.param]
    flags = {0: ["-DXB_XSMEM=1"], 1: ["-DXB_SHIFT_TAIL=1"], 2: []}[request.param]
    deps = [SRC] + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.startswith("xarith")]
    if not os.path.exists(lib_path) or os.path.getmtime(lib_path) < max(os.path.getmtime(d) for d in deps):
        os.makedirs(os.path.dirname(lib_path), exist_ok=True)
        subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-shared", "-fPIC",
                        *flags, SRC, "-o", lib_path], check=True)
    lib = ctypes.CDLL(lib_path)
    dp = ctypes.POINTER(ctypes.c_double)
    lib.xh_arith.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, dp, dp, dp,
                             ctypes.POINTER(ctypes.c_int32)]

    def run(limbs, op, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        out = np.zeros_like(a)
        stride = 2 * limbs if 5 <= op <= 7 else limbs
        count = a.size // stride
        codes = np.zeros(count, dtype=np.int32)
        lib.xh_arith(limbs, op, count, a.ctypes.data_as(dp), b.ctypes.data_as(dp),
                     out.ctypes.data_as(dp), codes.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
        return out, codes

    return run


@pytest.mark.parametrize("L", [2, 4])
@pytest.mark.parametrize("op", [0, 1, 2, 3, 4, 5, 6, 7, 8])
def test_host_arith_bitwise(port, host, L, op):
    rng = np.random.default_rng(7000 + 10 * L + op)
    count = {0: 400000, 1: 200000, 2: 60000, 7: 60000, 5: 12000}.get(op, 6000)
    cplx = 5 <= op <= 7
    renorm = lambda x: port.arith(L, 8, x)[0]
    a, b = operand_pairs(rng, count, L, renorm, parts=2 if cplx else 1)
    if op == 4:
        a = np.abs(a)
    want, wcodes = port.arith(L, op, a, b)
    got, gcodes = host(L, op, a, b)
    assert np.array_equal(gcodes, wcodes)
    ok = wcodes == 0
    g = got.reshape(count, -1)[ok].view(np.uint64)
    w = want.reshape(count, -1)[ok].view(np.uint64)
    bad = np.argwhere(g != w)
    assert len(bad) == 0, f"op {op} L {L}: {len(bad)} limbs differ, first row {bad[0][0]}"
