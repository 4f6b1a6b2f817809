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


EXP = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_build", "test_experiment")


def _fields(csv_text):
    return [ln.split(",")[:-1] for ln in csv_text.splitlines()]


@pytest.mark.parametrize("prec,limbs,m,n,trials,gs", [
    ("cdd", 2, 16, 16, 12, [1.0, 8.0]),
    ("cqd", 4, 12, 9, 6, [0.0, 17.0, 32.0]),
    ("cd", 1, 8, 8, 30, [16.0]),
])
def test_reference_experiment_harness_on_dropin(ref, prec, limbs, m, n, trials, gs):
    """The reference's unmodified experiment.hpp built against include/
    (tests/cpp/test_experiment.cpp): its accuracy sweep -- mgs_qr on the B200,
    residual_max_entry on the B200, breakdown exclusions -- prints the same
    CSV as the reference's own sweep (oracle/_ref), field for field except the
    wall time."""
    if not os.path.exists(EXP):
        pytest.skip("test_experiment not built (needs the reference tree at build time)")
    p = subprocess.run([EXP, "accuracy", prec, str(m), str(n), str(trials), "7"] + [repr(g) for g in gs],
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr
    want, rc = ref.accuracy_csv(limbs, m, n, gs, trials, 7)
    assert rc == 0
    assert _fields(p.stdout) == _fields(want)


def test_reference_overhead_bench_on_dropin():
    """experiment.hpp's overhead bench (experiment.hpp:242-285: real-double
    baseline, then cd / cdd / cqd mgs_qr on the B200 with
    timing_sink + to_double(f.r(0,0).re)) runs through the drop-in."""
    if not os.path.exists(EXP):
        pytest.skip("test_experiment not built")
    p = subprocess.run([EXP, "overhead", "16", "16", "3"], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr
    rows = [ln.split(",") for ln in p.stdout.splitlines()]
    assert rows[0] == ["kind", "precision", "m", "n", "reps", "wall_seconds", "factor_vs_baseline"]
    assert [r[1] for r in rows[1:]] == ["d", "cd", "cdd", "cqd"]
