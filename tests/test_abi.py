"""CPU tests of the drop-in boundary: the C-ABI library loads without a GPU,
exports every symbol include/xqr_b200.h declares, refuses to run without a
device (no CPU fallback), and the host-side argument validation raises the
reference's exception types before touching the device."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1210_0800_b200 as xqr

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "xqr_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(xqr_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_python_bindings():
    declared = header_functions()
    assert declared, "no functions parsed from the header"
    assert sorted(xqr.exported_symbols()) == declared


def test_library_exports_every_declared_symbol():
    lib = xqr.load_library()
    for name in header_functions():
        assert hasattr(lib, name), name
    assert lib.xqr_version() >= 100


def test_library_is_sm100a():
    # the fatbin carries sm_100a SASS (cuobjdump lists the arch)
    import shutil
    import subprocess

    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", xqr.library_path], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_cpp_dropin_headers_compile():
    # include/xqr/*.hpp: the reference API re-exported over the C ABI
    import shutil
    import subprocess
    import tempfile

    if not shutil.which("g++"):
        pytest.skip("no g++")
    src = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
    with tempfile.TemporaryDirectory() as d:
        r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"),
                            "-I", os.path.join(ROOT, "oracle"),
                            src], capture_output=True, text=True, cwd=d)
        assert r.returncode == 0, r.stderr


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib = xqr.load_library()
    h = ctypes.c_void_p()
    assert lib.xqr_ctx_create(0, ctypes.byref(h)) == xqr.XQR_CUDA
    with pytest.raises(xqr.cuda_error):
        xqr.Context(0)


def test_host_validation_raises_reference_types():
    a = np.zeros((3, 4, 2, 2))
    with pytest.raises(xqr.dimension_error):
        xqr.lsq_solve(a, np.zeros((5, 2, 2)))
    with pytest.raises(xqr.usage_error):
        xqr.par_lsq_solve(a, np.zeros((4, 2, 2)), 0)
    with pytest.raises(xqr.usage_error):
        xqr.par_mgs_qr(a, 2, mode="bogus")
    with pytest.raises(xqr.usage_error):
        xqr.mgs_qr(np.zeros((2, 2, 2, 3)))
    e = xqr.breakdown_error(7)
    assert e.column == 7 and isinstance(e, xqr.error)
