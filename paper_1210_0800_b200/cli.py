"""xqr command line on the B200 path (the reference CLI's qr / solve /
accuracy subcommands, tools/xqr_main.cpp:121-196, :249-328):

    python -m paper_1210_0800_b200.cli qr A.mat [--q-out P] [--r-out P] [--precision cdd]
                                                 [--workers N] [--normalize-mode M]
    python -m paper_1210_0800_b200.cli solve A.mat b.mat [--x-out P] [--precision cqd]
    python -m paper_1210_0800_b200.cli accuracy [--precision cdd] [--m 32] [--n 32]
                                               [--g 1 4 8] [--trials 100] [--seed 1]
                                               [--modulus-dist log|linear] [--paper-scale] [--out F]

Files are the reference's matrix format (matrix_io.py); outputs are written
atomically (temp + rename, xqr_main.cpp:42-58); stdout prints the same
`residual_max_entry` / `orthogonality_defect` / `residual_norm` lines in
shortest round-trip decimal.  Exit codes: 0 ok, 2 usage, 3 data, 4 numerical
(xqr_main.cpp:330-360).  The factorisation, solve and metrics run on the GPU.
"""
from __future__ import annotations

import argparse
import os
import re
import sys

import numpy as np

from . import matrix_io

PRECISION_LIMBS = {"cd": 1, "cdd": 2, "cqd": 4}


class data_error(RuntimeError):
    pass


def shortest(v: float) -> str:
    """std::to_chars(double) -- shortest round-trip, fixed or scientific,
    whichever is shorter (fixed on a tie) -- as experiment.hpp:376-380."""
    v = float(v)
    if v != v:
        return "nan" if np.signbit(v) == 0 else "-nan"
    if v in (float("inf"), float("-inf")):
        return "inf" if v > 0 else "-inf"
    if v == 0.0:
        return "-0" if np.signbit(v) else "0"
    sign = "-" if v < 0 else ""
    r = repr(abs(v))
    m = re.fullmatch(r"(\d+)(?:\.(\d*))?(?:e([+-]\d+))?", r)
    ip, fp, ex = m.group(1), m.group(2) or "", int(m.group(3) or 0)
    digits = (ip + fp).lstrip("0")
    # decimal exponent of the leading digit
    lead = len(ip.lstrip("0")) - 1 if ip.lstrip("0") else -(len(fp) - len(fp.lstrip("0")) + 1)
    e = lead + ex
    digits = digits.rstrip("0") or "0"
    k = len(digits)
    if e >= k - 1:
        fixed = "%.0f" % abs(v)  # the exact integer, as printf %f prints it
    elif e >= 0:
        fixed = digits[:e + 1] + "." + digits[e + 1:]
    else:
        fixed = "0." + "0" * (-e - 1) + digits
    sci = digits[0] + ("." + digits[1:] if k > 1 else "") + "e" + ("-" if e < 0 else "+") + f"{abs(e):02d}"
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def write_file_atomic(path: str, text: str) -> None:
    tmp = path + ".tmp"
    try:
        with open(tmp, "w") as f:
            f.write(text)
        os.replace(tmp, path)
    except OSError as exc:
        try:
            os.remove(tmp)
        except OSError:
            pass
        raise data_error(f"cannot write '{path}': {exc}") from None


def read_matrix_file(path: str):
    try:
        return matrix_io.read_matrix(path)
    except OSError:
        raise data_error(f"cannot open '{path}'") from None
    except matrix_io.parse_error as e:
        raise data_error(f"{path}: {e}") from None


def require_precision(flag, limbs, path):
    if not flag:
        return
    want = PRECISION_LIMBS.get(flag)
    if want is None:
        from . import usage_error

        raise usage_error(f"unknown precision token '{flag}'")
    if want != limbs:
        have = {v: k for k, v in PRECISION_LIMBS.items()}[limbs]
        raise data_error(f"{path}: expected precision '{flag}', file holds '{have}'")


def run_qr(o) -> None:
    import paper_1210_0800_b200 as xqr

    a, L = read_matrix_file(o.input)
    require_precision(o.precision, L, o.input)
    if o.normalize_mode not in ("designated", "redundant"):
        raise xqr.usage_error(f"unknown normalize mode '{o.normalize_mode}'")
    if o.workers == 1:
        q, r = xqr.mgs_qr(a)
    else:
        q, r = xqr.par_mgs_qr(a, o.workers, o.normalize_mode)
    write_file_atomic(o.q_out or o.input + ".q", matrix_io.matrix_text(q))
    write_file_atomic(o.r_out or o.input + ".r", matrix_io.matrix_text(r))
    resid = xqr.residual_max_entry(a, q, r)[0]
    defect = xqr.orthogonality_defect(q)[0]
    print(f"residual_max_entry {shortest(resid)}")
    print(f"orthogonality_defect {shortest(defect)}")


def run_solve(o) -> None:
    import paper_1210_0800_b200 as xqr

    a, L = read_matrix_file(o.input)
    require_precision(o.precision, L, o.input)
    b, Lb = read_matrix_file(o.rhs)
    if Lb != L:
        raise data_error(f"{o.rhs}: right-hand side precision differs from the matrix")
    if b.shape[0] != 1 or b.shape[1] != a.shape[1]:
        raise data_error(f"{o.rhs}: right-hand side must be a {a.shape[1]}x1 column")
    x, z = (xqr.lsq_solve(a, b[0]) if o.workers == 1 else xqr.par_lsq_solve(a, b[0], o.workers))
    write_file_atomic(o.x_out or o.input + ".x", matrix_io.matrix_text(x[None]))
    print(f"residual_norm {shortest(z[0])}")


ACCURACY_CSV_HEADER = "kind,precision,m,n,g,trials,exclusions,m_e,M_e,D_e,wall_seconds"


def accuracy_csv(precision: str, records) -> str:
    """experiment.hpp:412-433 accuracy_csv: header, then one `accuracy,` row
    per g in shortest round-trip decimal."""
    lines = [ACCURACY_CSV_HEADER + "\n"]
    for rec in records:
        lines.append(f"accuracy,{precision},{rec['m']},{rec['n']},{shortest(rec['g'])},{rec['trials']},"
                     f"{rec['exclusions']},{shortest(rec['m_e'])},{shortest(rec['M_e'])},"
                     f"{shortest(rec['D_e'])},{shortest(rec['wall_seconds'])}\n")
    return "".join(lines)


def run_accuracy(o) -> None:
    """accuracy sweep on the GPU (xqr_main.cpp:216-226 -> run_accuracy_sweep,
    experiment.hpp:157-176): ONE sweep over every g, so g index gi draws the
    streams split(gi*trials + t) exactly as the reference; CSV as the
    reference's accuracy_csv."""
    import paper_1210_0800_b200 as xqr

    L = PRECISION_LIMBS.get(o.precision)
    if L is None:
        raise xqr.usage_error(f"unknown precision token '{o.precision}'")
    if o.modulus_dist not in xqr.MODULUS_DIST:
        raise xqr.usage_error(f"unknown modulus distribution '{o.modulus_dist}'")
    trials = o.trials * 10 if o.paper_scale else o.trials
    # --g is repeatable and takes several values (CLI11 vector option); a
    # comma-separated list is accepted too
    gs = [float(t) for tok in (o.g or ["1"]) for t in str(tok).split(",") if t]
    records = xqr.accuracy_sweep(L, o.m, o.n, gs, trials, o.seed, dist=o.modulus_dist)
    text = accuracy_csv(o.precision, records)
    if o.out:
        write_file_atomic(o.out, text)
    else:
        sys.stdout.write(text)


def main(argv=None) -> int:
    import paper_1210_0800_b200 as xqr

    ap = argparse.ArgumentParser(prog="xqr", description="QR / least squares in cd, cdd, cqd on a B200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    q = sub.add_parser("qr")
    q.add_argument("input")
    q.add_argument("--precision", default="")
    q.add_argument("--q-out", default="")
    q.add_argument("--r-out", default="")
    q.add_argument("--workers", type=int, default=int(os.environ.get("XQR_WORKERS", "1")))
    q.add_argument("--normalize-mode", default="designated")
    s = sub.add_parser("solve")
    s.add_argument("input")
    s.add_argument("rhs")
    s.add_argument("--precision", default="")
    s.add_argument("--x-out", default="")
    s.add_argument("--workers", type=int, default=int(os.environ.get("XQR_WORKERS", "1")))
    a = sub.add_parser("accuracy")
    a.add_argument("--precision", required=True)
    a.add_argument("--m", type=int, default=32)
    a.add_argument("--n", type=int, default=32)
    a.add_argument("--g", action="extend", nargs="+", default=None)
    a.add_argument("--trials", type=int, default=100)
    a.add_argument("--seed", type=int, default=1)
    a.add_argument("--modulus-dist", default="log")
    a.add_argument("--paper-scale", action="store_true")
    a.add_argument("--out", default="")
    try:
        o = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    try:
        if o.workers < 1 if hasattr(o, "workers") else False:
            raise xqr.usage_error("worker count must be at least 1")
        {"qr": run_qr, "solve": run_solve, "accuracy": run_accuracy}[o.cmd](o)
    except xqr.usage_error as e:
        print(f"usage: {e}", file=sys.stderr)
        return 2
    except (data_error, xqr.dimension_error) as e:
        print(f"data: {e}", file=sys.stderr)
        return 3
    except (xqr.breakdown_error, xqr.overflow_error, xqr.domain_error) as e:
        print(f"numerical: {e}", file=sys.stderr)
        return 4
    except Exception as e:  # noqa: BLE001
        print(f"error: {e}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
