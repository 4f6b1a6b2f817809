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


def test_accuracy_csv():
    rc, out, err = cli("accuracy", "--precision", "cdd", "--m", "8", "--n", "8", "--g", "1,8",
                       "--trials", "10")
    assert rc == 0, err
    lines = out.splitlines()
    assert lines[0] == "precision,m,n,g,trials,exclusions,m_e,M_e,D_e,wall_seconds"
    assert len(lines) == 3 and lines[1].startswith("cdd,8,8,1,10,0,")
