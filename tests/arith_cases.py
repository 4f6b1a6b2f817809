"""Operand generators for the arithmetic parity tests (host and device).

Classes are chosen to drive every data-dependent branch of the reference
quad-double code (quad_double.hpp:60-257: the magnitude merge, the zero tests
of quick_three_accum and of both renorm trees):

* generic: testsupport::random_dd/random_qd style full-limb operands
  (tests/support/random_values.hpp:15-38), renormalised;
* widened: lower limbs exactly 0 (random.hpp:70 -- the generator's inputs);
* offset: b scaled by 2^e for e in 0..260, so the merge interleaves a's and
  b's limbs in every pattern and one operand can be exhausted early;
* cancel: b = -a with perturbed tails, so leading limbs cancel exactly and
  zero error terms appear mid-merge;
* sparse: random limbs zeroed (zeros inside the limb sequence);
* ties: equal magnitudes, opposite signs, signed zeros;
* dyadic: short-mantissa limbs spaced ~54 bits apart, so partial sums are
  exact and zero error terms appear inside otherwise regular merges;
* newton: x and a correction 1-3 limbs below it (x + x*(1 - b*x) and the
  sqrt/division corrections), either operand first -- the shifted merges,
  including the ones whose loop exits early and folds leftovers.
"""
import numpy as np


def random_operands(rng, count, L, emin=-40, emax=40, parts=1):
    e = rng.integers(emin, emax + 1, size=(count, parts))
    mant = 1.0 + rng.random((count, parts))
    sgn = np.where(rng.random((count, parts)) < 0.5, -1.0, 1.0)
    out = np.zeros((count, parts, L))
    out[..., 0] = np.ldexp(sgn * mant, e)
    for l in range(1, L):
        out[..., l] = out[..., l - 1] * 2.0 ** -54 * (2 * rng.random((count, parts)) - 1)
    return out


def operand_pairs(rng, count, L, renorm, parts=1):
    """(a, b) arrays of shape (count, parts, L) mixing all classes; `renorm`
    renormalises an (N, L) array (the oracle's op 8)."""
    per = count // 8
    a = random_operands(rng, count, L, parts=parts)
    b = random_operands(rng, count, L, parts=parts)
    if L > 1:
        a = renorm(a.reshape(-1, L)).reshape(a.shape)
        b = renorm(b.reshape(-1, L)).reshape(b.shape)
    s = 0
    # widened
    a[s:s + per // 2, ..., 1:] = 0.0
    b[s + per // 4:s + per, ..., 1:] = 0.0
    s += per
    # offset: b scaled by 2^-e, e in 0..260 (exact scaling keeps b renormalised)
    e = rng.integers(0, 261, size=(per, parts, 1))
    sg = np.where(rng.random((per, parts, 1)) < 0.5, -1.0, 1.0)
    b[s:s + per] = np.ldexp(b[s:s + per], -e) * sg
    sw = rng.random(per) < 0.5
    tmp = a[s:s + per][sw].copy()
    a[s:s + per][sw] = b[s:s + per][sw]
    b[s:s + per][sw] = tmp
    s += per
    # cancel: b = -a, tail limbs perturbed from some position on
    b[s:s + per] = -a[s:s + per]
    if L > 1:
        pos = rng.integers(1, L + 1, size=per)
        for i in range(per):
            if pos[i] < L:
                b[s + i, ..., pos[i]:] = random_operands(rng, 1, L - pos[i], -200, -120, parts)[0]
        b[s:s + per] = renorm(b[s:s + per].reshape(-1, L)).reshape(b[s:s + per].shape)
    s += per
    # sparse: zero random limbs
    mask = rng.random((per, parts, L)) < 0.35
    a[s:s + per][mask] = 0.0
    mask = rng.random((per, parts, L)) < 0.35
    b[s:s + per][mask] = 0.0
    s += per
    # ties / signed zeros
    b[s:s + per // 2] = a[s:s + per // 2]
    a[s + per // 2:s + per, ..., 0] = -0.0
    b[s + per // 2:s + per, ..., 0] = np.where(rng.random((per - per // 2, parts)) < 0.5, 0.0, -0.0)
    flip = rng.random((per, parts, L)) < 0.5
    b[s:s + per][flip] = -b[s:s + per][flip]
    s += per
    # dyadic: mantissas k/8, exponent gaps 53..56
    for arr in (a, b):
        e0 = rng.integers(-4, 5, size=(per, parts))
        mant = rng.integers(8, 16, size=(per, parts, L)) / 8.0
        sg = np.where(rng.random((per, parts, L)) < 0.5, -1.0, 1.0)
        gaps = np.cumsum(rng.integers(53, 57, size=(per, parts, L)), axis=-1) - 53
        arr[s:s + per] = sg * np.ldexp(mant, e0[..., None] - gaps)
    s += per
    # newton: b = a correction S limbs (54 S bits, +-4) below a, either order
    if L > 1:
        c = random_operands(rng, per, L, -2, 2, parts)
        c = renorm(c.reshape(-1, L)).reshape(c.shape)
        shift = 54 * rng.integers(1, 4, size=(per, parts, 1)) + rng.integers(-4, 5, size=(per, parts, 1))
        sg = np.where(rng.random((per, parts, 1)) < 0.5, -1.0, 1.0)
        b[s:s + per] = sg * np.ldexp(c, -shift)
        sw = rng.random(per) < 0.5
        tmp = a[s:s + per][sw].copy()
        a[s:s + per][sw] = b[s:s + per][sw]
        b[s:s + per][sw] = tmp
    return np.ascontiguousarray(a), np.ascontiguousarray(b)
