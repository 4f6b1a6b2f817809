"""Matrix files of the reference (matrix_io.hpp:25-117, hexfloat.hpp:18-58):
a header `rows cols precision` (d, dd or qd), then one complex entry per line,
column-major, each spelled as C99 hex-float components -- the real part's
limbs, then the imaginary part's.  Write-then-read reproduces every bit; the
text is byte-identical to the reference's write_matrix
(tests/test_matrix_io.py checks it against the reference itself).

Arrays use the package convention: (n_cols, m_rows, 2, L) float64.
"""
from __future__ import annotations

import math
import re

import numpy as np

NAMES = {1: "d", 2: "dd", 4: "qd"}
LIMBS = {v: k for k, v in NAMES.items()}


class parse_error(ValueError):
    """Malformed input file; `line` is 1-based (errors.hpp:41-46)."""

    def __init__(self, line: int, what: str):
        super().__init__(f"line {line}: {what}")
        self.line = line


# ---- hex-float tokens (hexfloat.hpp:18-34) -------------------------------------------
def hex_token(v: float) -> str:
    """C99 `%a` as glibc prints it: shortest hex fraction, no trailing zeros."""
    if not math.isfinite(v):
        from . import overflow_error

        raise overflow_error("cannot serialize non-finite value")
    if v == 0.0:
        return "-0x0p+0" if math.copysign(1.0, v) < 0 else "0x0p+0"
    h = float.hex(v)  # [-]0x1.hhhhhhhhhhhhhp[+-]d  (or 0x0.h...p-1022 for subnormals)
    m = re.fullmatch(r"(-?)0x([01])\.([0-9a-f]+)p([+-]\d+)", h)
    sign, lead, frac, exp = m.groups()
    frac = frac.rstrip("0")
    body = f"0x{lead}.{frac}" if frac else f"0x{lead}"
    e = int(exp)
    return f"{sign}{body}p{'+' if e >= 0 else '-'}{abs(e)}"


def parse_numeric_token(tok: str, line: int) -> float:
    """strtod on one whole token (hexfloat.hpp:26-34): hex or decimal, finite."""
    if not tok:
        raise parse_error(line, "empty numeric token")
    try:
        if re.fullmatch(r"[+-]?0[xX][0-9a-fA-F]*\.?[0-9a-fA-F]*([pP][+-]?\d+)?", tok):
            t = tok
            neg = t.startswith("-")
            t = t.lstrip("+-")
            if "p" not in t.lower():
                t += "p0"
            v = float.fromhex(t)
            v = -v if neg else v
        else:
            if not re.fullmatch(r"[+-]?(\d+\.?\d*|\.\d+)([eE][+-]?\d+)?|[+-]?(inf|infinity|nan)", tok,
                                re.IGNORECASE):
                raise ValueError
            v = float(tok)
    except (ValueError, OverflowError):
        raise parse_error(line, f"bad numeric token '{tok}'") from None
    if not math.isfinite(v):
        raise parse_error(line, f"non-finite value '{tok}'")
    return v


# ---- limb renormalisation on read (hexfloat.hpp:49-58) --------------------------------
def _qts(a: float, b: float):
    s = a + b
    return s, b - (s - a)


def _renorm4(c0, c1, c2, c3):
    """quad_double.hpp:157-200 on host doubles (IEEE binary64, no contraction)."""
    if math.isinf(c0):
        return c0, c1, c2, c3
    t, c3 = _qts(c2, c3)
    t, c2 = _qts(c1, t)
    c0, c1 = _qts(c0, t)
    s0, s1, s2, s3 = c0, c1, 0.0, 0.0
    if s1 != 0.0:
        s1, s2 = _qts(s1, c2)
        if s2 != 0.0:
            s2, s3 = _qts(s2, c3)
        else:
            s1, s2 = _qts(s1, c3)
    else:
        s0, s1 = _qts(s0, c2)
        if s1 != 0.0:
            s1, s2 = _qts(s1, c3)
        else:
            s0, s1 = _qts(s0, c3)
    return s0, s1, s2, s3


def _from_components(comps, L):
    if L == 1:
        return comps
    if L == 2:
        return list(_qts(comps[0], comps[1]))
    return list(_renorm4(*comps))


# ---- files ------------------------------------------------------------------------------
def matrix_text(a) -> str:
    """write_matrix (matrix_io.hpp:25-34)."""
    a = np.asarray(a, dtype=np.float64)
    n, m, _, L = a.shape
    out = [f"{m} {n} {NAMES[L]}\n"]
    for j in range(n):
        for i in range(m):
            out.append(" ".join(hex_token(float(v)) for v in a[j, i].reshape(-1)) + "\n")
    return "".join(out)


def write_matrix(path: str, a) -> None:
    with open(path, "w") as f:
        f.write(matrix_text(a))


def parse_matrix(text: str):
    """read_matrix (matrix_io.hpp:91-109): returns (array, limbs)."""
    lines = text.split("\n")
    if text.endswith("\n"):
        lines = lines[:-1]
    if not lines:
        raise parse_error(1, "missing header")
    toks = lines[0].split()
    if len(toks) != 3:
        raise parse_error(1, "header must be 'rows cols precision'")
    for t in toks[:2]:
        if not t.isdigit():
            raise parse_error(1, f"bad dimension '{t}'")
    m, n = int(toks[0]), int(toks[1])
    if toks[2] not in LIMBS:
        raise parse_error(1, f"unknown precision '{toks[2]}'")
    L = LIMBS[toks[2]]
    if n == 0 or m < n:
        raise parse_error(1, "dimensions must satisfy rows >= cols >= 1")
    a = np.zeros((n, m, 2, L))
    ln = 1
    for j in range(n):
        for i in range(m):
            if ln >= len(lines):
                raise parse_error(ln + 1, "unexpected end of file")
            tk = lines[ln].split()
            ln += 1
            if len(tk) != 2 * L:
                raise parse_error(ln, f"expected {2 * L} components per entry")
            comps = [parse_numeric_token(t, ln) for t in tk]
            a[j, i, 0] = _from_components(comps[:L], L)
            a[j, i, 1] = _from_components(comps[L:], L)
    for rest in lines[ln:]:
        ln += 1
        if rest.split():
            raise parse_error(ln, "trailing content after last entry")
    return a, L


def read_matrix(path: str):
    with open(path) as f:
        return parse_matrix(f.read())
