"""Run the C++ drop-in test binary (tests/cpp/test_dropin.cpp, built by
__graft_entry__.build()): the reference API compiled against include/xqr/*.hpp,
executed on the B200, compared bitwise with the CPU oracle."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_build", "test_dropin")


def test_cpp_dropin_binary():
    assert os.path.exists(BIN), "run __graft_entry__.build() first"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("PASS")


def test_generator_matches_oracle(port):
    import numpy as np

    import paper_1210_0800_b200 as xqr

    for L in (1, 2, 4):
        a, b = xqr.gen_systems(L, 3, 9, 7, 1.0, 5, 2)
        for s in range(3):
            wa, wb = port.gen_system(L, 9, 7, 1.0, 5, 2 + s)
            assert np.array_equal(a[s].view(np.uint64), wa.view(np.uint64))
            assert np.array_equal(b[s].view(np.uint64), wb.view(np.uint64))
        a1, b1 = xqr.gen_systems(L, 1, 6, 6, 2.0, 11, -1)
        wa, wb = port.gen_system(L, 6, 6, 2.0, 11, -1)
        assert np.array_equal(a1[0].view(np.uint64), wa.view(np.uint64))
