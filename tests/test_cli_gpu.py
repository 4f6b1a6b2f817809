"""GPU: the command line on the B200 path against the reference -- output
files byte-identical to the reference's write_matrix of the oracle's factors,
the same stdout lines, the reference's exit codes (test_cli.cpp:91-172)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1210_0800_b200 import matrix_io
from paper_1210_0800_b200.cli import shortest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def cli(*args):
    p = subprocess.run([sys.executable, "-m", "paper_1210_0800_b200.cli", *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=300)
    return p.returncode, p.stdout, p.stderr


@pytest.mark.parametrize("L,name", [(1, "cd"), (2, "cdd"), (4, "cqd")])
def test_qr_and_solve_files(port, tmp_path, L, name):
    import oracle

    rio = oracle.ref_io()
    a, b = port.gen_system(L, 12, 7, 1.0, 11)
    fa, fb = tmp_path / "a.mat", tmp_path / "b.mat"
    fa.write_text(matrix_io.matrix_text(a))
    fb.write_text(matrix_io.matrix_text(b[None]))
    rc, out, err = cli("qr", str(fa), "--precision", name)
    assert rc == 0, err
    q, r, _ = port.mgs_qr(a)
    want_q = rio.write_matrix(q) if rio else matrix_io.matrix_text(q)
    want_r = rio.write_matrix(r) if rio else matrix_io.matrix_text(r)
    assert (tmp_path / "a.mat.q").read_text() == want_q
    assert (tmp_path / "a.mat.r").read_text() == want_r
    res, _ = port.residual_max_entry(a, q, r)
    dfc, _ = port.orthogonality_defect(q)
    assert out.splitlines() == [f"residual_max_entry {shortest(res[0])}",
                                f"orthogonality_defect {shortest(dfc[0])}"]
    rc, out, err = cli("solve", str(fa), str(fb), "--x-out", str(tmp_path / "x.mat"), "--workers", "4")
    assert rc == 0, err
    x, z, _ = port.lsq_solve(a, b)
    assert (tmp_path / "x.mat").read_text() == (rio.write_matrix(x[None]) if rio else matrix_io.matrix_text(x[None]))
    assert out.splitlines() == [f"residual_norm {shortest(z[0])}"]


def test_exit_codes(port, tmp_path):
    a = port.gen_system(2, 6, 4, 1.0, 3, rhs=False)
    a[2] = a[0]  # rank deficient: breakdown at column 3
    f = tmp_path / "a.mat"
    f.write_text(matrix_io.matrix_text(a))
    rc, out, err = cli("qr", str(f))
    assert rc == 4 and err.startswith("numerical:")
    rc, _, err = cli("qr", str(f), "--precision", "cqd")
    assert rc == 3 and err.startswith("data:")
    rc, _, err = cli("qr", str(f), "--precision", "cxx")
    assert rc == 2 and err.startswith("usage:")
    bad = tmp_path / "bad.mat"
    bad.write_text("2 1 d\n0x1p+0 0x0p+0\n0xZp+0 0x0p+0\n")
    rc, _, err = cli("qr", str(bad))
    assert rc == 3 and "line 3" in err
    rc, _, _ = cli("qr")
    assert rc == 2


def _fields(csv_text):
    """rows without the wall_seconds column (timing differs by construction)"""
    return [ln.split(",")[:-1] for ln in csv_text.splitlines()]


@pytest.mark.parametrize("args,limbs,gs,trials,linear", [
    (["--precision", "cdd", "--m", "8", "--n", "8", "--g", "1", "8", "--trials", "10"], 2, [1.0, 8.0], 10, False),
    (["--precision", "cqd", "--m", "12", "--n", "9", "--g", "0", "--g", "17", "--g", "32",
      "--trials", "7", "--seed", "5"], 4, [0.0, 17.0, 32.0], 7, False),
    (["--precision", "cd", "--m", "10", "--n", "10", "--g", "1,16", "--trials", "5",
      "--modulus-dist", "linear"], 1, [1.0, 16.0], 5, True),
])
def test_accuracy_csv_matches_reference(ref, args, limbs, gs, trials, linear):
    """xqr_main.cpp:216-226: one sweep over every g (rows after the first draw
    split(gi*trials + t)), the reference's accuracy_csv header and `accuracy,`
    rows -- field for field against the reference's own sweep, except the
    wall time."""
    rc, out, err = cli("accuracy", *args)
    assert rc == 0, err
    m, n = int(args[args.index("--m") + 1]), int(args[args.index("--n") + 1])
    seed = int(args[args.index("--seed") + 1]) if "--seed" in args else 1
    want, wrc = ref.accuracy_csv(limbs, m, n, gs, trials, seed, linear)
    assert wrc == 0
    assert out.splitlines()[0] == "kind,precision,m,n,g,trials,exclusions,m_e,M_e,D_e,wall_seconds"
    assert _fields(out) == _fields(want)


@pytest.mark.parametrize("prec,limbs,m,g,trials", [("cd", 1, 8, 16.0, 50), ("cdd", 2, 16, 64.0, 50),
                                                     ("cd", 1, 32, 100.0, 20)])
def test_accuracy_breakdowns_excluded_like_reference(ref, prec, limbs, m, g, trials):
    """Wide magnitude ranges make near-singular matrices: breakdowns are
    counted as exclusions exactly as the reference's trial loop counts them
    (cd 8x8 g=16: 6 of 50; cdd 16x16 g=64: 26 of 50; cd 32x32 g=100: all, so
    m_e / M_e / D_e are nan)."""
    rc, out, err = cli("accuracy", "--precision", prec, "--m", str(m), "--n", str(m), "--g", str(g),
                       "--trials", str(trials))
    assert rc == 0, err
    want, _ = ref.accuracy_csv(limbs, m, m, [g], trials)
    assert _fields(out) == _fields(want)
    assert int(_fields(out)[1][6]) > 0


def test_accuracy_requires_precision():
    rc, _, _ = cli("accuracy", "--m", "8", "--n", "8")
    assert rc == 2
