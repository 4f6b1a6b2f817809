"""GPU: randomized shapes, magnitudes and precisions against the oracle, bit
for bit (errors included) -- a sweep across every kernel the routing can pick
(one CTA, the double-double grid, the quad-double clusters at each cluster
size, batched systems).  XQR_FUZZ_CASES scales it (default 48)."""
import os

import numpy as np
import pytest

import paper_1210_0800_b200 as xqr

pytestmark = pytest.mark.gpu


def same(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)
    b = np.ascontiguousarray(b, dtype=np.float64).view(np.uint64)
    return np.array_equal(a, b)


def check(port, a, b, what):
    x, z, st = port.lsq_solve(a, b)
    q, r, sq = port.mgs_qr(a)
    for call, want, ref_st in ((lambda: xqr.lsq_solve(a, b), (x, z), st),
                               (lambda: xqr.mgs_qr(a), (q, r), sq)):
        if ref_st[0] == 0:
            got = call()
            assert all(same(g, w) for g, w in zip(got, want)), what
        else:
            exc = {1: xqr.breakdown_error, 2: xqr.overflow_error, 3: xqr.domain_error}[ref_st[0]]
            with pytest.raises(exc) as e:
                call()
            if ref_st[0] == 1:
                assert e.value.column == ref_st[1], what


def test_fuzz_single_systems(port):
    rng = np.random.default_rng(20261017)
    cases = int(os.environ.get("XQR_FUZZ_CASES", "48"))
    for c in range(cases):
        L = int(rng.choice([1, 2, 4]))
        sizes = [2, 7, 16, 31, 33, 64, 65, 100, 129, 200, 256, 257, 300]
        if os.environ.get("XQR_FUZZ_BIG") == "1":  # tall systems too (slower oracle)
            sizes += [400, 511, 512, 700, 1024, 1100, 2048]
        m = int(rng.choice(sizes))
        if L == 4 and os.environ.get("XQR_FUZZ_BIG") != "1":
            m = min(m, 257)
        n = int(rng.integers(1, min(m, 64 if L == 4 else 96, 24 if m > 512 else 96) + 1))
        g = float(rng.choice([1.0, 1.0, 4.0, 8.0, 16.0]))
        a, b = port.gen_system(L, m, n, g, int(rng.integers(1, 1 << 30)))
        if rng.random() < 0.15 and n > 2:  # a dependent column somewhere
            a[int(rng.integers(1, n))] = a[0]
        check(port, a, b, f"case {c}: L={L} m={m} n={n} g={g}")


def test_fuzz_batches(port):
    rng = np.random.default_rng(77)
    for c in range(int(os.environ.get("XQR_FUZZ_CASES", "48")) // 8):
        L = int(rng.choice([1, 2, 4]))
        m = int(rng.choice([8, 32, 33, 64, 100]))
        n = int(rng.integers(1, min(m, 40) + 1))
        batch = int(rng.integers(2, 6))
        A = np.stack([port.gen_system(L, m, n, 1.0, 1000 * c + s)[0] for s in range(batch)])
        B = np.stack([port.gen_system(L, m, n, 1.0, 1000 * c + s)[1] for s in range(batch)])
        if n > 1:
            A[batch // 2, n - 1] = A[batch // 2, 0]  # one system breaks down
        x, z, codes, cols = xqr.lsq_solve_batched(A, B)
        for s in range(batch):
            wx, wz, st = port.lsq_solve(A[s], B[s])
            assert codes[s] == st[0] and (st[0] != 1 or cols[s] == st[1]), f"batch case {c} system {s}"
            if st[0] == 0:
                assert same(x[s], wx) and same(z[s], wz), f"batch case {c} system {s}"
