"""GPU parity: the sm_100a path through the C ABI against the CPU oracle,
bit for bit (the north star's 1e-28*kappa / 1e-60*kappa tolerance is implied:
a bitwise-equal result has zero difference).

Inputs are the reference generator's (experiment.hpp:64-79) so the oracle,
the reference and the device all see identical systems."""
import math
import os

import numpy as np
import pytest

import paper_1210_0800_b200 as xqr

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_same(got, want, what=""):
    g, w = bits(got), bits(want)
    if not np.array_equal(g, w):
        bad = np.argwhere(g != w)
        raise AssertionError(f"{what}: {len(bad)} limbs differ, first at {bad[0].tolist()}: "
                             f"{got.reshape(-1)[np.ravel_multi_index(bad[0], g.shape)]!r} vs "
                             f"{want.reshape(-1)[np.ravel_multi_index(bad[0], w.shape)]!r}")


# ---- elementwise arithmetic (eft.hpp, double_double.hpp, quad_double.hpp, complex.hpp)
def random_operands(rng, count, L, emin=-40, emax=40, cplx=False):
    """testsupport::random_dd/random_qd style operands (random_values.hpp:15-38),
    renormalised by the oracle."""
    parts = 2 if cplx else 1
    e = rng.integers(emin, emax + 1, size=(count, parts))
    mant = 1.0 + rng.random((count, parts))
    sgn = np.where(rng.random((count, parts)) < 0.5, -1.0, 1.0)
    out = np.zeros((count, parts, L))
    out[..., 0] = np.ldexp(sgn * mant, e)
    for l in range(1, L):
        out[..., l] = out[..., l - 1] * 2.0 ** -54 * (2 * rng.random((count, parts)) - 1)
    return out


@pytest.mark.parametrize("L", [1, 2, 4])
@pytest.mark.parametrize("op", [0, 1, 2, 3, 4, 5, 6, 7, 8])
def test_arith_bitwise(port, L, op):
    rng = np.random.default_rng(1000 * L + op)
    count = 20000 if L == 4 else 100000
    cplx = 5 <= op <= 7
    a = random_operands(rng, count, L, cplx=cplx)
    b = random_operands(rng, count, L, cplx=cplx)
    if op == 4:
        a = np.abs(a)
    if L > 1:  # renormalise the operands with the oracle (quad_double.hpp:209-213)
        a = port.arith(L, 8, a.reshape(-1, L))[0].reshape(a.shape)
        b = port.arith(L, 8, b.reshape(-1, L))[0].reshape(b.shape)
    # special operands: zeros, zero lower limbs, equal magnitudes
    a[:8] = 0.0
    a[8:16, ..., 1:] = 0.0
    b[16:24] = a[16:24]
    b[24:32] = -a[24:32]
    want, wcodes = port.arith(L, op, a, b)
    got, gcodes = xqr.arith(L, op, a, b)
    assert np.array_equal(gcodes, wcodes)
    ok = wcodes == 0
    assert_same(got.reshape(count, -1)[ok], want.reshape(count, -1)[ok], f"op {op} L {L}")


# ---- the hot path ------------------------------------------------------------------------
GRID = [(d, s) for d in (8, 32, 33, 64) for s in range(20)]  # acceptance.cpp:266-268


@pytest.mark.parametrize("L", [1, 2, 4])
def test_criterion7_grid_bitwise(port, L):
    """acceptance.cpp:264-317's grid: dims {8,32,33,64} x 20 seeds; GPU == CPU."""
    for dim, seed in GRID:
        if L == 4 and dim == 64 and seed % 4:
            continue
        a, b = port.gen_system(L, dim, dim, 1.0, seed * 1009 + dim)
        q, r, st = port.mgs_qr(a)
        gq, gr = xqr.mgs_qr(a)
        assert_same(gq, q, f"Q dim={dim} seed={seed}")
        assert_same(gr, r, f"R dim={dim} seed={seed}")
        x, z, st = port.lsq_solve(a, b)
        gx, gz = xqr.lsq_solve(a, b)
        assert_same(gx, x, f"x dim={dim} seed={seed}")
        assert_same(gz, z, f"z dim={dim} seed={seed}")


@pytest.mark.parametrize("L", [1, 2, 4])
@pytest.mark.parametrize("m,n", [(1, 1), (2, 1), (12, 7), (40, 1), (31, 31), (65, 3), (100, 50),
                                 (129, 20), (200, 200), (300, 17)])
def test_shapes_bitwise(port, L, m, n):
    if L == 4 and m * n > 20000:
        pytest.skip("oracle too slow for this shape in qd")
    a, b = port.gen_system(L, m, n, 1.0, 1000 + m * 7 + n)
    q, r, _ = port.mgs_qr(a)
    gq, gr = xqr.mgs_qr(a)
    assert_same(gq, q, "Q")
    assert_same(gr, r, "R")
    x, z, _ = port.lsq_solve(a, b)
    gx, gz = xqr.lsq_solve(a, b)
    assert_same(gx, x, "x")
    assert_same(gz, z, "z")


@pytest.mark.parametrize("L", [2, 4])
def test_wide_magnitude_range_bitwise(port, L):
    # g = 8, 16: entries spread over 1e-16..1e16 (Table 2 sweep, experiment.hpp:157-176)
    for g in (8.0, 16.0):
        a, b = port.gen_system(L, 24, 24, g, 77)
        q, r, st = port.mgs_qr(a)
        if st[0]:
            with pytest.raises(xqr.breakdown_error) as e:
                xqr.mgs_qr(a)
            assert e.value.column == st[1]
            continue
        gq, gr = xqr.mgs_qr(a)
        assert_same(gq, q, f"Q g={g}")
        assert_same(gr, r, f"R g={g}")


@pytest.mark.parametrize("L", [1, 2, 4])
def test_breakdown_column(L):
    # test_mgs.cpp:70-90
    col = np.zeros((3, 2, L))
    for i in range(3):
        col[i, 0, 0] = i + 1.0
        col[i, 1, 0] = 0.5
    a = np.stack([col, col])
    with pytest.raises(xqr.breakdown_error) as e:
        xqr.mgs_qr(a)
    assert e.value.column == 2
    with pytest.raises(xqr.breakdown_error) as e:
        xqr.mgs_qr(np.zeros((2, 2, 2, L)))
    assert e.value.column == 1


@pytest.mark.parametrize("L", [1, 2, 4])
def test_lsq_breakdown_and_zero_residual(port, L):
    # b in the range of A: z == 0 exactly is legitimate (mgs.hpp:128-130)
    a = np.zeros((3, 3, 2, L))
    for k in range(3):
        a[k, k, 0, 0] = 1.0
    b = np.zeros((3, 2, L))
    b[:, 0, 0] = [1.5, 0.25, -1.0]
    b[:, 1, 0] = [-2.0, 3.0, 0.5]
    x, z = xqr.lsq_solve(a, b)
    assert_same(x, b)
    assert not bits(z).any()
    # dependent columns: breakdown at 2 in lsq_solve too
    a2, b2 = port.gen_system(L, 6, 3, 1.0, 5)
    a2[2] = a2[0]
    x, z, st = port.lsq_solve(a2, b2)
    with pytest.raises(xqr.breakdown_error) as e:
        xqr.lsq_solve(a2, b2)
    assert e.value.column == st[1] == 3


@pytest.mark.parametrize("L", [2, 4])
def test_overflow_reported(port, L):
    a = np.zeros((2, 2, 2, L))
    a[0, 0, 0, 0] = 1e300
    a[0, 1, 0, 0] = 1e300
    a[1, 0, 0, 0] = 1.0
    a[1, 1, 1, 0] = 1.0
    assert port.mgs_qr(a)[2][0] == 2
    with pytest.raises(xqr.overflow_error):
        xqr.mgs_qr(a)


def assert_same_nan(got, want, what=""):
    """Bitwise where the oracle is a number; NaN where it is NaN (the GPU's
    canonical NaN and x86's default NaN differ in sign and payload bits)."""
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(got), nan), f"{what}: NaN positions differ"
    assert_same(np.where(nan, 0.0, got), np.where(nan, 0.0, want), what)


def test_cd_overflow_propagates(port):
    """complex<double> arithmetic is unchecked in the reference
    (real_type.hpp:19): Inf/NaN propagate and no overflow_error is raised,
    unlike dd/qd (test_overflow_reported).  A column norm that overflows
    to Inf still trips the breakdown test (mgs.hpp:84-92), as in the
    reference; a back substitution that overflows just returns Inf/NaN."""
    a = np.zeros((2, 2, 2, 1))
    a[0, 0, 0, 0] = 1e300
    a[0, 1, 0, 0] = 1e300
    a[1, 0, 0, 0] = 1.0
    a[1, 1, 1, 0] = 1.0
    q, r, st = port.mgs_qr(a)
    assert st[0] == 1
    with pytest.raises(xqr.breakdown_error) as e:
        xqr.mgs_qr(a)
    assert e.value.column == st[1]
    a = np.zeros((2, 2, 2, 1))
    a[0, :, 0, 0] = (1e150, 1e150)  # |a_0|^2 finite, r_01 * q_0 overflows
    a[1, :, 0, 0] = (1e300, -1e300)
    a[1, 1, 1, 0] = 1.0
    q, r, st = port.mgs_qr(a)
    if st[0] == 1:
        with pytest.raises(xqr.breakdown_error):
            xqr.mgs_qr(a)
    else:
        assert st[0] == 0
        gq, gr = xqr.mgs_qr(a)
        assert_same_nan(gq, q, "Q")
        assert_same_nan(gr, r, "R")
    rng = np.random.default_rng(5)
    rr, y = _upper(rng, 40, 1)
    rr[30, :30, :, 0] = 1e300
    y[30, :, 0] = 1e300
    x, st = port.back_substitute(rr, y)
    assert st == (0, 0)
    assert_same_nan(xqr.back_substitute(rr, y), x, "back substitution")


@pytest.mark.parametrize("L", [2, 4])
@pytest.mark.parametrize("m,n", [(70, 20), (24, 12), (300, 50)])
def test_single_system_grid_error_paths(port, L, m, n):
    """The whole-GPU single-system kernels (xgrid1 for dd, m >= 64; xgrid2 for
    qd, m >= 16) report the reference's first error: a breakdown in the middle
    of the factorisation, an overflow, and wide-range data (g = 16)."""
    def check(call_port, call_dev, *args):
        want = call_port(*args)
        st = want[-1]
        if st[0] == 0:
            got = call_dev(*args)
            for g, w in zip(got, want[:-1]):
                assert_same(g, w)
        elif st[0] == 1:
            with pytest.raises(xqr.breakdown_error) as e:
                call_dev(*args)
            assert e.value.column == st[1]
        else:
            with pytest.raises({2: xqr.overflow_error, 3: xqr.domain_error}[st[0]]):
                call_dev(*args)
        return st

    a, b = port.gen_system(L, m, n, 1.0, 404 + m)
    a[n // 2] = a[1]  # dependent column
    assert check(port.mgs_qr, xqr.mgs_qr, a)[0] == 1
    assert check(port.lsq_solve, xqr.lsq_solve, a, b)[0] == 1
    a, b = port.gen_system(L, m, n, 1.0, 405 + m)
    a[n - 2, :, 0, 0] *= 1e300  # overflow inside the sweep
    a[n - 2, :, 1, 0] *= 1e300
    assert check(port.mgs_qr, xqr.mgs_qr, a)[0] == 2
    assert check(port.lsq_solve, xqr.lsq_solve, a, b)[0] == 2
    for seed in range(3):
        a, b = port.gen_system(L, m, n, 16.0, 900 + seed)
        check(port.mgs_qr, xqr.mgs_qr, a)
        check(port.lsq_solve, xqr.lsq_solve, a, b)


@pytest.mark.parametrize("L", [1, 2, 4])
def test_back_substitute_api(port, L):
    rng = np.random.default_rng(L)
    for n in (1, 2, 7, 33, 70):
        r = np.zeros((n, n, 2, L))
        for j in range(n):
            for i in range(j + 1):
                r[j, i, :, 0] = rng.uniform(-1, 1, 2)
            r[j, j, :, 0] += (1.5, 0.25)
        y = np.zeros((n, 2, L))
        y[..., 0] = rng.uniform(-1, 1, (n, 2))
        x, st = port.back_substitute(r, y)
        assert st == (0, 0)
        assert_same(xqr.back_substitute(r, y), x, f"n={n}")
    # zero diagonal -> domain_error (mgs.hpp:119-121); shapes -> dimension_error
    r = np.zeros((2, 2, 2, L))
    r[0, 0, 0, 0] = 1.0
    y = np.ones((2, 2, L))
    with pytest.raises(xqr.domain_error):
        xqr.back_substitute(r, y)
    with pytest.raises(xqr.dimension_error):
        xqr.back_substitute(np.zeros((2, 3, 2, L)), y)
    with pytest.raises(xqr.dimension_error):
        xqr.back_substitute(np.eye(3)[:, :, None, None] * np.ones((1, 1, 2, L)), y)


def _upper(rng, n, L):
    r = np.zeros((n, n, 2, L))
    for j in range(n):
        r[j, : j + 1, :, 0] = rng.uniform(-1, 1, (j + 1, 2))
        r[j, j, :, 0] += (1.5, 0.25)
    y = np.zeros((n, 2, L))
    y[..., 0] = rng.uniform(-1, 1, (n, 2))
    return r, y


@pytest.mark.parametrize("L", [1, 2, 4])
def test_back_substitute_flow(port, L):
    """Single-system back substitution runs the warp-pipelined sweep
    (flow_back_substitute): sizes with one and several unknowns per lane
    pair, and the reference's first error when several are planted --
    an overflowing update above a zero diagonal (the overflow comes first in
    program order, mgs.hpp:117-124) and the other way round."""
    rng = np.random.default_rng(100 + L)
    for n in (16, 17, 193, 241, 255, 256, 257, 300, 513):
        r, y = _upper(rng, n, L)
        x, st = port.back_substitute(r, y)
        assert st == (0, 0)
        assert_same(xqr.back_substitute(r, y), x, f"n={n}")
    # n = 300: several unknowns per thread; n = 200: the one-per-thread sweep
    for n, k_over, k_zero in ((300, 250, 100), (300, 40, 200), (300, 299, 17), (300, 5, 6),
                              (200, 150, 60), (200, 30, 120), (200, 199, 1)):
        r, y = _upper(rng, n, L)
        r[k_over, : k_over, :, 0] = 1e300  # x_j -= r_jk x_k overflows at step k_over
        y[k_over, :, 0] = 1e300
        r[k_zero, k_zero] = 0.0  # zero diagonal -> domain_error at step k_zero
        _, st = port.back_substitute(r, y)
        assert st[0] in (2, 3)
        with pytest.raises({2: xqr.overflow_error, 3: xqr.domain_error}[st[0]]):
            xqr.back_substitute(r, y)


@pytest.mark.parametrize("L", [2, 4])
def test_batched_matches_single(port, L):
    """Batched systems (split streams, random.hpp:38-40) == the oracle per system;
    a rank-deficient system in the middle keeps its own status."""
    batch, m, n = 37, 20, 16
    a = np.zeros((batch, n, m, 2, L))
    b = np.zeros((batch, m, 2, L))
    for s in range(batch):
        a[s], b[s] = port.gen_system(L, m, n, 1.0, 5, s)
    a[11, 5] = a[11, 2]  # breakdown at column 6
    x, z, codes, cols = xqr.lsq_solve_batched(a, b)
    for s in range(batch):
        wx, wz, st = port.lsq_solve(a[s], b[s])
        assert (codes[s], cols[s]) == st, s
        if st[0] == 0:
            assert_same(x[s], wx, f"x[{s}]")
            assert_same(z[s], wz, f"z[{s}]")
    assert codes[11] == 1 and cols[11] == 6
    q, r, codes, cols = xqr.mgs_qr_batched(a)
    for s in (0, 11, 36):
        wq, wr, st = port.mgs_qr(a[s])
        assert (codes[s], cols[s]) == st
        if st[0] == 0:
            assert_same(q[s], wq)
            assert_same(r[s], wr)


@pytest.mark.parametrize("pinned", [False, True])
def test_batched_pipeline_chunks(port, monkeypatch, pinned):
    """The host-buffer batch is split into chunks pipelined over two streams
    (capi.cu solve_host_batched); force small, uneven chunks and check every
    system, its status index, and the pinned (direct DMA) input path."""
    import torch

    L, batch, m, n = 4, 23, 12, 9
    a = np.zeros((batch, n, m, 2, L))
    b = np.zeros((batch, m, 2, L))
    for s in range(batch):
        a[s], b[s] = port.gen_system(L, m, n, 1.0, 9, s)
    a[17, 4] = a[17, 1]  # breakdown at column 5
    if pinned:
        a = torch.from_numpy(a).pin_memory().numpy()
        b = torch.from_numpy(b).pin_memory().numpy()
    monkeypatch.setenv("XQR_CHUNK", "5")
    x, z, codes, cols = xqr.lsq_solve_batched(a, b)
    q, r, qcodes, qcols = xqr.mgs_qr_batched(a)
    for s in range(batch):
        wx, wz, st = port.lsq_solve(a[s], b[s])
        assert (codes[s], cols[s]) == st, s
        if st[0] == 0:
            assert_same(x[s], wx, f"x[{s}]")
            assert_same(z[s], wz, f"z[{s}]")
        wq, wr, st = port.mgs_qr(a[s])
        assert (qcodes[s], qcols[s]) == st, s
        if st[0] == 0:
            assert_same(q[s], wq, f"q[{s}]")
            assert_same(r[s], wr, f"r[{s}]")
    assert codes[17] == 1 and cols[17] == 5


@pytest.mark.parametrize("L", [1, 2, 4])
@pytest.mark.parametrize("m,n", [(8, 8), (33, 33), (40, 7), (64, 64), (129, 20)])
def test_metrics_bitwise(port, L, m, n):
    """Device residual_max_entry / orthogonality_defect (mgs.hpp:161-222) ==
    the oracle's, on a factorisation and on a perturbed one."""
    if L == 4 and m * n > 3000:
        pytest.skip("oracle too slow for this shape in qd")
    a, _ = port.gen_system(L, m, n, 1.0, 31 * m + n)
    q, r, st = port.mgs_qr(a)
    assert st[0] == 0
    q2 = q.copy()
    q2[n // 2, m // 3, 0, 0] *= 1.0 + 2.0 ** -20
    for qq in (q, q2):
        want, wst = port.residual_max_entry(a, qq, r)
        got = xqr.residual_max_entry(a, qq, r)
        assert_same(got, want, "residual")
        want, wst = port.orthogonality_defect(qq)
        got = xqr.orthogonality_defect(qq)
        assert_same(got, want, "defect")
    # batched forms agree with the single-system forms
    ab, qb, rb = np.stack([a, a]), np.stack([q, q2]), np.stack([r, r])
    res, codes = xqr.residual_max_entry_batched(ab, qb, rb)
    assert not codes.any()
    assert_same(res[1], port.residual_max_entry(a, q2, r)[0], "batched residual")
    dfc, codes = xqr.orthogonality_defect_batched(qb)
    assert_same(dfc[1], port.orthogonality_defect(q2)[0], "batched defect")


@pytest.mark.parametrize("L", [1, 2, 4])
def test_accuracy_sweep_matches_reference_loop(port, L):
    """accuracy_sweep (paper Table 2 harness, experiment.hpp:117-176) on the
    GPU == the reference's serial loop run on the oracle, trial by trial
    (including breakdown exclusions at large g)."""
    g_values, trials, m = (1.0, 8.0, 150.0), 12, 10
    recs = xqr.accuracy_sweep(L, m, m, g_values, trials, seed=20260901)
    for gi, (g, rec) in enumerate(zip(g_values, recs)):
        want, excl = [], 0
        for t in range(trials):
            a = port.gen_system(L, m, m, g, 20260901, gi * trials + t, rhs=False)
            q, r, st = port.mgs_qr(a)
            if st[0] == 1:
                excl += 1
                continue
            e, _ = port.residual_max_entry(a, q, r)
            want.append(math.log10(e[0]))  # std::log10 (experiment.hpp:130)
        assert rec["exclusions"] == excl
        assert np.array_equal(np.array(rec["log10_e"]), np.array(want)), g


def test_par_api_routes_to_device(port):
    a, b = port.gen_system(2, 33, 33, 1.0, 7)
    x, z, _ = port.lsq_solve(a, b)
    for w in (1, 2, 8):
        gx, gz = xqr.par_lsq_solve(a, b, w)
        assert_same(gx, x)
        assert_same(gz, z)
    q, r, _ = port.mgs_qr(a)
    for mode in (xqr.normalize_mode.designated, xqr.normalize_mode.redundant):
        gq, gr = xqr.par_mgs_qr(a, 4, mode)
        assert_same(gq, q)
        assert_same(gr, r)


# ---- golden fixtures: the BASELINE configs at full size ------------------------------
@pytest.mark.parametrize("name", ["cdd_32x32", "cdd_256x256", "cqd_256x256", "cqd_512x256",
                                  "cqd_128x128_s0", "cqd_128x128_s3"])
def test_golden_bench_configs(port, name):
    g = np.load(os.path.join(GOLDEN, f"bench_{name}.npz"))
    L, m, n = int(g["limbs"]), int(g["m"]), int(g["n"])
    a, b = port.gen_system(L, m, n, 1.0, int(g["seed"]), int(g["stream"]))
    x, z = xqr.lsq_solve(a, b)
    assert_same(x, g["x"], f"{name} x")
    assert_same(z, g["z"], f"{name} z")


# ---- single-system grid kernels at their shape boundaries -----------------------------
# xgrid2 (qd, m >= 16): cluster size 1/2/4 and 1/2/4 rows per lane pair switch
# at m = 64, 128, 256, 512; xgrid1 (dd, m >= 64): rows per thread switch at
# 256 and 512.  Few columns keep the oracle fast; every result bitwise.
@pytest.mark.parametrize("L,m", [(4, m) for m in (16, 17, 63, 64, 65, 127, 129, 255, 257, 511, 513, 1000,
                                                   1024)] + [(2, m) for m in (64, 65, 255, 257, 511, 513, 1024)])
def test_grid_shape_boundaries(port, L, m):
    for n in (4, 9):
        a, b = port.gen_system(L, m, n, 1.0, 7000 + m + n)
        q, r, _ = port.mgs_qr(a)
        gq, gr = xqr.mgs_qr(a)
        assert_same(gq, q, f"Q m={m} n={n}")
        assert_same(gr, r, f"R m={m} n={n}")
        x, z, _ = port.lsq_solve(a, b)
        gx, gz = xqr.lsq_solve(a, b)
        assert_same(gx, x, f"x m={m} n={n}")
        assert_same(gz, z, f"z m={m} n={n}")


@pytest.mark.parametrize("m,n,force", [(300, 60, None), (512, 45, None), (200, 90, "1")])
def test_grid_paired_bulk_updates(port, monkeypatch, m, n, force):
    """xgrid2 updates trailing columns two at a time (lockstep pairs) when a
    cluster owns more than one: on by default for 256 < m <= 512 (8-CTA
    clusters, 37 of them: pairs form once n + 1 > 37), forced on for m = 200
    (4-CTA clusters, 74 of them).  Bitwise against the oracle."""
    if force:
        monkeypatch.setenv("XQR_GRID_PAIR", force)
    a, b = port.gen_system(4, m, n, 1.0, 8100 + m + n)
    q, r, _ = port.mgs_qr(a)
    gq, gr = xqr.mgs_qr(a)
    assert_same(gq, q, "Q")
    assert_same(gr, r, "R")
    x, z, _ = port.lsq_solve(a, b)
    gx, gz = xqr.lsq_solve(a, b)
    assert_same(gx, x, "x")
    assert_same(gz, z, "z")


# ---- the reference's known answers (test_mgs.cpp) through the device ------------------
@pytest.mark.parametrize("L", [1, 2, 4])
@pytest.mark.parametrize("n", [4, 64, 200, 1100, 1400])
def test_known_answer_identity_device(L, n):
    """test_mgs.cpp:45-55 (identity factors to identity) at the CTA size and
    at grid-kernel sizes; lsq_solve on I returns b with z = 0 (:220-228)."""
    a = np.zeros((n, n, 2, L))
    for k in range(n):
        a[k, k, 0, 0] = 1.0
    q, r = xqr.mgs_qr(a)
    assert_same(q, a, "Q")
    assert_same(r, a, "R")
    rng = np.random.default_rng(n + L)
    b = np.zeros((n, 2, L))
    b[..., 0] = rng.uniform(-1, 1, (n, 2))
    x, z = xqr.lsq_solve(a, b)
    assert_same(x, b, "x")
    assert not np.any(z.view(np.uint64)), "z must be +0"


@pytest.mark.parametrize("L", [1, 2, 4])
@pytest.mark.parametrize("n", [2, 64])
def test_known_answer_breakdowns_device(L, n):
    """test_mgs.cpp:70-90: a zero matrix breaks down at column 1; a repeated
    column at its (1-based) index -- on the CTA and the grid kernels."""
    with pytest.raises(xqr.breakdown_error) as e:
        xqr.mgs_qr(np.zeros((n, n, 2, L)))
    assert e.value.column == 1
    a = np.zeros((n, n, 2, L))
    rng = np.random.default_rng(3)
    a[..., 0] = rng.uniform(-1, 1, (n, n, 2))
    a[1] = a[0]
    with pytest.raises(xqr.breakdown_error) as e:
        xqr.mgs_qr(a)
    assert e.value.column == 2


def test_known_answer_three_four_five_device():
    """test_mgs.cpp:57-68: (3, 4) normalises exactly to r = 5, q = (0.6, 0.8)."""
    a = np.zeros((1, 2, 2, 1))
    a[0, 0, 0, 0], a[0, 1, 0, 0] = 3.0, 4.0
    q, r = xqr.mgs_qr(a)
    assert r[0, 0, 0, 0] == 5.0 and r[0, 0, 1, 0] == 0.0
    assert q[0, 0, 0, 0] == 0.6 and q[0, 1, 0, 0] == 0.8


@pytest.mark.parametrize("L", [1, 2, 4])
@pytest.mark.parametrize("m,n", [(3, 5), (3, 0), (0, 0), (16, 17), (64, 65)])
def test_dimension_errors_device(port, L, m, n):
    """Shapes the reference rejects with dimension_error (mgs.hpp, matrix.hpp:
    m < n, empty) are rejected the same way by the device API, single and
    batched, including sizes that would otherwise route to the grid kernels."""
    a = np.zeros((n, m, 2, L))
    b = np.zeros((m, 2, L))
    assert port.mgs_qr(a)[2][0] == 4 and port.lsq_solve(a, b)[2][0] == 4
    with pytest.raises(xqr.dimension_error):
        xqr.mgs_qr(a)
    with pytest.raises(xqr.dimension_error):
        xqr.lsq_solve(a, b)
    with pytest.raises(xqr.dimension_error):
        xqr.lsq_solve_batched(a[None], b[None])


# ---- single systems beyond 1024 rows (grid kernels only) ------------------------------
@pytest.mark.parametrize("L,m", [(4, 1025), (4, 1500), (4, 2048), (2, 1025), (2, 2048), (1, 1300)])
def test_tall_single_systems(port, L, m):
    """m in (1024, 2048]: qd on 8-CTA clusters with 4 rows per lane pair, dd / d
    on the CTA-per-column kernel with 8 rows per thread; bitwise, plus the
    device metrics.  Batches of such systems run system by system on the grid
    kernels (one CTA per system holds at most 1024 rows) with the same bits."""
    for n in (3, 9):
        a, b = port.gen_system(L, m, n, 1.0, 9100 + m + n)
        q, r, _ = port.mgs_qr(a)
        gq, gr = xqr.mgs_qr(a)
        assert_same(gq, q, f"Q m={m} n={n}")
        assert_same(gr, r, f"R m={m} n={n}")
        x, z, _ = port.lsq_solve(a, b)
        gx, gz = xqr.lsq_solve(a, b)
        assert_same(gx, x, f"x m={m} n={n}")
        assert_same(gz, z, f"z m={m} n={n}")
        assert_same(xqr.residual_max_entry(a, q, r), port.residual_max_entry(a, q, r)[0], "residual")
        assert_same(xqr.orthogonality_defect(q), port.orthogonality_defect(q)[0], "orthogonality")
    a2, b2 = port.gen_system(L, m, n, 1.0, 9200 + m)
    A = np.stack([a, a2])
    B = np.stack([b, b2])
    bx, bz, codes, _ = xqr.lsq_solve_batched(A, B)
    assert not codes.any()
    assert_same(bx[0], x, "batched x[0]")
    assert_same(bx[1], port.lsq_solve(a2, b2)[0], "batched x[1]")
    bq, br, codes, _ = xqr.mgs_qr_batched(A)
    assert not codes.any()
    assert_same(bq[0], q, "batched q[0]")
    assert_same(br[1], port.mgs_qr(a2)[1], "batched r[1]")


def test_tall_batch_device_api(port):
    """The device-pointer batched call with m > 1024: system by system on the
    grid kernels, statuses carry their system index."""
    torch = pytest.importorskip("torch")
    L, m, n = 4, 1100, 5
    sys_ab = [port.gen_system(L, m, n, 1.0, 9300 + s) for s in range(3)]
    A = np.stack([ab[0] for ab in sys_ab])
    A[1, 2] = A[1, 0]  # system 1 breaks down at column 3
    B = np.stack([ab[1] for ab in sys_ab])
    ctx = xqr.context(0)
    da, db = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dx = torch.zeros((3, n, 2, L), dtype=torch.float64, device="cuda")
    dz = torch.zeros((3, L), dtype=torch.float64, device="cuda")
    dst = torch.zeros((3, 2), dtype=torch.int64, device="cuda")
    try:
        ctx.lsq_solve_batched_device(L, 3, m, n, da.data_ptr(), db.data_ptr(), dx.data_ptr(),
                                     dz.data_ptr(), dst.data_ptr())
    except xqr.breakdown_error:
        pass  # the call reports the first failing system; statuses are per system
    torch.cuda.synchronize()
    st = dst.cpu().numpy()
    code = st[:, 0] & 0xFFFFFFFF
    col = st[:, 0] >> 32
    assert list(code) == [0, 1, 0] and col[1] == 3 and list(st[:, 1]) == [0, 1, 2]
    for s in (0, 2):
        x, z, _ = port.lsq_solve(A[s], B[s])
        assert_same(dx[s].cpu().numpy(), x, f"x[{s}]")
        assert_same(dz[s].cpu().numpy(), z, f"z[{s}]")


# ---- routing when the persistent grid cannot be placed -----------------------------------
@pytest.mark.parametrize("L,m,n", [(4, 64, 64), (4, 40, 33), (2, 96, 96), (2, 64, 20)])
def test_grid_unplaceable_reroutes_to_cta(port, monkeypatch, L, m, n):
    """XQR_GRID_MAX_SMS=0 emulates a device partition on which the cooperative
    grid cannot be made co-resident: the single system is re-routed to the
    one-CTA kernel (no error, same bits, counted in grid_fallbacks); with a
    few SMs the grid runs narrower and still gives the same bits."""
    a, b = port.gen_system(L, m, n, 1.0, 4400 + m + n)
    x, z, st = port.lsq_solve(a, b)
    q, r, st2 = port.mgs_qr(a)
    assert st[0] == 0 and st2[0] == 0
    ctx = xqr.context(0)
    for sms, rerouted in (("0", True), ("3", False)):
        monkeypatch.setenv("XQR_GRID_MAX_SMS", sms)
        before = ctx.grid_fallbacks
        gx, gz = xqr.lsq_solve(a, b)
        gq, gr = xqr.mgs_qr(a)
        assert_same(gx, x, f"x sms={sms}")
        assert_same(gz, z, f"z sms={sms}")
        assert_same(gq, q, f"q sms={sms}")
        assert_same(gr, r, f"r sms={sms}")
        assert (ctx.grid_fallbacks - before == 2) == rerouted


def test_grid_unplaceable_tall_system_fails_loudly(port, monkeypatch):
    """m > 1024 has no one-CTA kernel: an unplaceable grid is a cuda_error,
    never a silent fallback."""
    a, b = port.gen_system(4, 1100, 3, 1.0, 77)
    monkeypatch.setenv("XQR_GRID_MAX_SMS", "0")
    with pytest.raises(xqr.cuda_error):
        xqr.lsq_solve(a, b)


# ---- the grid kernels place every shape they are routed (no silent re-route) ------------
@pytest.mark.parametrize("L,m,n", [(1, 256, 8), (2, 256, 8), (2, 300, 8), (2, 512, 8), (2, 1024, 6),
                                   (2, 2048, 4), (4, 256, 8), (4, 512, 8), (4, 1024, 6), (4, 2048, 4)])
def test_grid_shapes_place_without_reroute(port, L, m, n):
    """Every row count the grid kernels serve launches on the full B200 (a
    launch that fails for lack of shared memory would be re-routed to the
    one-CTA kernel: the same bits, but tens of times slower -- only the
    fallback counter shows it)."""
    a, b = port.gen_system(L, m, n, 1.0, 9100 + m + n)
    ctx = xqr.context(0)
    before = ctx.grid_fallbacks
    xqr.lsq_solve(a, b)
    xqr.mgs_qr(a)
    assert ctx.grid_fallbacks == before


# ---- both schedules of the double / double-double grid kernel --------------------------
@pytest.mark.parametrize("chain", ["0", "1"])
@pytest.mark.parametrize("L,m,n", [(2, 256, 40), (2, 300, 24), (1, 128, 64), (2, 64, 64)])
def test_grid1_schedules_bitwise(port, monkeypatch, chain, L, m, n):
    """The dd/d grid kernel's cyclic schedule and its chain mode (CTA 0 runs
    every pivot, the other CTAs the earlier projections) give the reference's
    bits for QR and least squares."""
    monkeypatch.setenv("XQR_GRID_CHAIN", chain)
    a, b = port.gen_system(L, m, n, 4.0, 5200 + m + n)
    x, z, st = port.lsq_solve(a, b)
    q, r, st2 = port.mgs_qr(a)
    assert st[0] == 0 and st2[0] == 0
    gx, gz = xqr.lsq_solve(a, b)
    gq, gr = xqr.mgs_qr(a)
    assert_same(gx, x, "x")
    assert_same(gz, z, "z")
    assert_same(gq, q, "q")
    assert_same(gr, r, "r")


# ---- the batched pre-pass's maximum column norm at the extremes ------------------------
@pytest.mark.parametrize("L", [1, 2, 4])
@pytest.mark.parametrize("scale", [505, 511, -500, -530, 0])
def test_batched_prepass_extreme_and_tied_norms(port, L, scale):
    """The batched kernels take square roots only for the columns that can
    hold the largest norm (within 2^-40 of the largest s_j) and for extreme
    magnitudes.  A batch mixing one column scaled by 2^scale (huge: near or
    past overflow; tiny: below 2^-1000), exact duplicates of the largest
    column (tied norms) and columns a last-limb step below it must give the
    reference's results or error, system by system."""
    rng = np.random.default_rng(6100 + L + scale)
    m, n, batch = 48, 12, 4
    A = np.stack([port.gen_system(L, m, n, 1.0, 300 + s)[0] for s in range(batch)])
    B = np.stack([port.gen_system(L, m, n, 1.0, 300 + s)[1] for s in range(batch)])
    A[0, 3] = A[0, 3] * 2.0 ** scale          # one extreme column
    A[1, 5] = A[1, 2]                         # a tied (duplicate) column: breakdown
    A[2, 7, :, :, -1] = np.nextafter(A[2, 7, :, :, -1], np.inf)  # last limbs nudged
    A[2, 8] = A[2, 7]
    A[2, 8, :, :, -1] = np.nextafter(A[2, 8, :, :, -1], -np.inf)
    x, z, codes, cols = xqr.lsq_solve_batched(A, B)
    for s in range(batch):
        wx, wz, st = port.lsq_solve(A[s], B[s])
        assert codes[s] == st[0], f"system {s}: code {codes[s]} vs {st[0]}"
        if st[0] == 1:
            assert cols[s] == st[1], f"system {s}"
        if st[0] == 0:
            if L == 1:
                assert_same_nan(x[s], wx, f"x[{s}]")
            else:
                assert_same(x[s], wx, f"x[{s}]")
                assert_same(z[s], wz, f"z[{s}]")


@pytest.mark.gpu
@pytest.mark.parametrize("m,n", [(200, 200), (240, 230)])
def test_batched_qd_back_substitution_many_blocks(port, m, n):
    """The batched quad-double kernels' warp-specialised back substitution
    with more unknowns than one sweep of the updaters off the finisher's
    SMSP (16 per warp), so the warps on the finisher's SMSP take the next
    blocks and some updaters carry two: each system bitwise equal to the
    single-system solve of the same data (itself pinned to the oracle)."""
    batch = 2
    a = np.zeros((batch, n, m, 2, 4))
    b = np.zeros((batch, m, 2, 4))
    for s in range(batch):
        a[s], b[s] = port.gen_system(4, m, n, 1.0, 77, s)
    x, z, codes, cols = xqr.lsq_solve_batched(a, b)
    for s in range(batch):
        gx, gz = xqr.lsq_solve(a[s], b[s])
        assert codes[s] == 0 and cols[s] == 0
        assert_same(x[s], gx, f"x[{s}]")
        assert_same(z[s], gz, f"z[{s}]")
