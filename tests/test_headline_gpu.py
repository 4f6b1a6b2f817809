"""GPU: the headline batched kernel pinned at its benchmark shape.

BASELINE.json configs[4] is a batch of cqd 128x128 least-squares systems;
bench.py times it through ``xqr_lsq_solve_batched[_device]``, which runs the
CTA-per-system kernel ``mgs_cta_kernel<L=4, LV=3, NW=8, LSQ, MINB=2>`` (and
``<4,3,8,QR,2>`` for ``mgs_qr_batched``).  Single-system ``lsq_solve`` of the
same shape routes to the cluster grid kernel instead, so the golden-config
test in test_parity_gpu.py does not cover this instance.  Here one full wave
of the batched kernel (2 CTAs x SMs systems, streams 0..wave-1 of
split_mix64(1), experiment.hpp:64-79) is solved and checked bit for bit:

* streams 0-3 against the reference's own results (tests/golden, generated
  from oracle/_ref by tests/golden/make_golden.py);
* a spread of further streams against the reference compiled in place
  (oracle/_ref, run here on the host), or the C restatement where it is absent;
* the device-pointer entry point against the host-buffer one, system by
  system, over the whole wave (acceptance.cpp:264-317 determinism pattern).
"""
import hashlib
import os

import numpy as np
import pytest

import paper_1210_0800_b200 as xqr

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
L, M, N = 4, 128, 128


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def digest(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def wave():
    torch = pytest.importorskip("torch")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    return 2 * sms  # resident CTAs of the cqd m <= 128 kernel: 2 per SM


@pytest.fixture(scope="module")
def systems(wave):
    return xqr.gen_systems(L, wave, M, N, 1.0, 1, 0)


@pytest.fixture(scope="module")
def checker():
    """The reference compiled in place when present (fast, threaded), else the port."""
    import oracle

    ref = oracle.reference()
    return ref if ref is not None else oracle.port()


def _check_streams(wave):
    extra = [4, 5, 6, 7, 31, 32, 63, 100, 147, wave // 2, wave - 2, wave - 1]
    return sorted(set(s for s in extra if s < wave))


@pytest.fixture(scope="module")
def host_result(systems):
    a, b = systems
    x, z, codes, cols = xqr.lsq_solve_batched(a, b)
    return x, z, codes, cols


def test_headline_batch_golden_streams(systems, host_result):
    x, z, codes, _ = host_result
    assert not codes.any()
    for s in range(4):
        g = np.load(os.path.join(GOLDEN, f"bench_cqd_128x128_s{s}.npz"))
        assert int(g["stream"]) == s and int(g["m"]) == M
        assert digest(systems[0][s], systems[1][s]) == str(g["a_digest"]), "generator drifted"
        assert np.array_equal(bits(x[s]), bits(g["x"])), f"x of stream {s}"
        assert np.array_equal(bits(z[s]), bits(g["z"])), f"z of stream {s}"


def test_headline_batch_vs_reference(systems, host_result, checker, wave):
    a, b = systems
    x, z, _, _ = host_result
    idx = _check_streams(wave)
    if checker.kind == "reference":
        wx, wz, wcodes = checker.lsq_solve_batch(a[idx], b[idx], threads=min(32, os.cpu_count() or 1))
        assert not wcodes.any()
    else:
        outs = [checker.lsq_solve(a[s], b[s]) for s in idx]
        wx = np.stack([o[0] for o in outs])
        wz = np.stack([o[1] for o in outs])
    for k, s in enumerate(idx):
        assert np.array_equal(bits(x[s]), bits(wx[k])), f"x of stream {s} ({checker.kind})"
        assert np.array_equal(bits(z[s]), bits(wz[k])), f"z of stream {s} ({checker.kind})"


def test_headline_batch_device_entry_equals_host(systems, host_result, wave):
    torch = pytest.importorskip("torch")
    a, b = systems
    x, z, _, _ = host_result
    ctx = xqr.context(0)
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    dx = torch.zeros((wave, N, 2, L), dtype=torch.float64, device="cuda")
    dz = torch.zeros((wave, L), dtype=torch.float64, device="cuda")
    dst = torch.full((wave, 2), -1, dtype=torch.int64, device="cuda")
    ctx.lsq_solve_batched_device(L, wave, M, N, da.data_ptr(), db.data_ptr(), dx.data_ptr(),
                                 dz.data_ptr(), dst.data_ptr())
    torch.cuda.synchronize()
    st = dst.cpu().numpy()
    assert not (st[:, 0] & 0xFFFFFFFF).any()
    assert np.array_equal(st[:, 1], np.arange(wave))
    assert np.array_equal(bits(dx.cpu().numpy()), bits(x))
    assert np.array_equal(bits(dz.cpu().numpy()), bits(z))


def test_headline_qr_batch(systems, checker, wave):
    """mgs_qr_batched at 128x128 (the <4,3,8,QR,2> instance): Q and R digests
    of streams 0-3 equal the reference's (tests/golden qr_digest), more
    streams against the reference, and the device-pointer call equals the
    host-buffer one."""
    torch = pytest.importorskip("torch")
    a = systems[0]
    q, r, codes, _ = xqr.mgs_qr_batched(a)
    assert not codes.any()
    for s in range(4):
        g = np.load(os.path.join(GOLDEN, f"bench_cqd_128x128_s{s}.npz"))
        assert digest(q[s], r[s]) == str(g["qr_digest"]), f"Q/R of stream {s}"
    for s in (5, wave - 1):
        wq, wr, st = checker.mgs_qr(a[s])
        assert st[0] == 0
        assert np.array_equal(bits(q[s]), bits(wq)), f"q of stream {s}"
        assert np.array_equal(bits(r[s]), bits(wr)), f"r of stream {s}"
    ctx = xqr.context(0)
    da = torch.from_numpy(a).cuda()
    dq = torch.zeros_like(da)
    dr = torch.full((wave, N, N, 2, L), 7.0, dtype=torch.float64, device="cuda")
    dst = torch.zeros((wave, 2), dtype=torch.int64, device="cuda")
    ctx.mgs_qr_batched_device(L, wave, M, N, da.data_ptr(), dq.data_ptr(), dr.data_ptr(), dst.data_ptr())
    torch.cuda.synchronize()
    assert not (dst.cpu().numpy()[:, 0] & 0xFFFFFFFF).any()
    assert np.array_equal(bits(dq.cpu().numpy()), bits(q))
    assert np.array_equal(bits(dr.cpu().numpy()), bits(r))


def test_headline_batch_planted_errors(systems, checker):
    """Failures inside a full-shape batch stay per system: a planted rank
    deficiency (breakdown at its 1-based column, mgs.hpp:50) and an overflow
    (double_double.hpp:34-37 / quad_double.hpp:202-205) do not disturb the
    neighbours, which stay bitwise equal to the reference."""
    a, b = systems
    a = a[:8].copy()
    b = b[:8].copy()
    a[2, 77] = a[2, 5]           # column 78 repeats column 6
    a[5, 3, 9, 0, 0] = 1e300     # squares overflow
    x, z, codes, cols = xqr.lsq_solve_batched(a, b)
    for s in range(8):
        wx, wz, st = checker.lsq_solve(a[s], b[s])
        assert (codes[s], cols[s]) == st, s
        if st[0] == 0:
            assert np.array_equal(bits(x[s]), bits(wx)), s
            assert np.array_equal(bits(z[s]), bits(wz)), s
    assert codes[2] == xqr.XQR_BREAKDOWN and cols[2] == 78
    assert codes[5] == xqr.XQR_OVERFLOW


@pytest.mark.parametrize("L2", [2, 4])
@pytest.mark.parametrize("op", [0, 1, 2, 3, 4, 5, 6, 7, 8])
def test_arith_edge_classes_vs_reference(L2, op):
    """Device arithmetic against the reference's own operators (oracle/_ref;
    the port where the reference build is absent) over every operand class
    of tests/arith_cases.py -- merge orders, exhausted limbs, cancellation,
    signed zeros, shifted Newton operands (test_quad_double.cpp:25-70)."""
    import sys

    import oracle

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from arith_cases import operand_pairs

    chk = oracle.reference() or oracle.port()
    rng = np.random.default_rng(5100 + 10 * L2 + op)
    count = {0: 40000, 1: 40000, 2: 20000, 7: 20000, 8: 20000, 5: 4000}.get(op, 2000)
    cplx = 5 <= op <= 7
    a, b = operand_pairs(rng, count, L2, lambda v: chk.arith(L2, 8, v)[0], parts=2 if cplx else 1)
    if op == 4:
        a = np.abs(a)
    want, wcodes = chk.arith(L2, op, a, b)
    got, gcodes = xqr.arith(L2, op, a, b)
    assert np.array_equal(gcodes, wcodes)
    ok = wcodes == 0
    g = bits(got).reshape(count, -1)[ok]
    w = bits(want).reshape(count, -1)[ok]
    bad = np.argwhere(g != w)
    assert len(bad) == 0, f"op {op} L {L2}: {len(bad)} limbs differ ({chk.kind}), first row {bad[0][0]}"


def _in_fresh_thread(fn):
    """Run fn as the first library call of a new thread (a fresh ctx with an
    empty arena); return its result or re-raise its exception."""
    import threading

    box = {}

    def work():
        try:
            box["out"] = fn()
        except BaseException as e:  # noqa: BLE001
            box["err"] = e

    t = threading.Thread(target=work)
    t.start()
    t.join()
    if "err" in box:
        raise box["err"]
    return box["out"]


@pytest.mark.parametrize("L2", [2, 4])
@pytest.mark.parametrize("k", [1, 2, 3])
def test_metric_on_fresh_context(L2, k):
    """A metric call as the FIRST call of a thread (fresh ctx, empty arena;
    e.g. orthogonality_defect(identity(2)) needs more scratch than its
    copied input): the metric scratch is sized together with the inputs, so
    nothing is reallocated under live device pointers."""
    import oracle

    port = oracle.port()
    q = np.zeros((k, k, 2, L2))
    for i in range(k):
        q[i, i, 0, 0] = 1.0
    assert np.array_equal(_in_fresh_thread(lambda: xqr.orthogonality_defect(q)), np.zeros(L2))
    a, _ = port.gen_system(L2, k + 1, k, 1.0, 3)
    qq, rr, _ = port.mgs_qr(a)
    got = _in_fresh_thread(lambda: xqr.residual_max_entry(a, qq, rr))
    assert np.array_equal(bits(got), bits(port.residual_max_entry(a, qq, rr)[0]))
