"""Reproduce the paper's accuracy table (Table 2) and its quality-up comparison
on the B200:

  * Table 2: 1,000 QR decompositions of random 32x32
    complex matrices, modulus log-uniform in [10^-g, 10^g]; m_e / M_e = min /
    max log10 of the max-entry residual e (mgs.hpp:161-178).  Complex double
    and double-double for g = 1, 4, 8, 12, 16; double-double and quad-double
    for g = 17, 20, 24, 28, 32.  GPU: batched mgs_qr + batched device metric,
    the reference's own trial streams (experiment.hpp:117-176).
  * Quality-up: on the same A and b, the time of
    complex quad-double on the GPU against complex double-double on one CPU
    core (the reference itself, oracle/_ref), with the accuracy each buys
    (residual e, orthogonality defect, least-squares residual z).

    python tools/paper_tables.py [--trials 1000] [--out profiles/r01_paper_tables.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1210_0800_b200 as xqr  # noqa: E402

NAMES = {1: "cd", 2: "cdd", 4: "cqd"}


def table2(trials):
    rows = []
    for limbs, gs in ((1, (1, 4, 8, 12, 16)), (2, (1, 4, 8, 12, 16, 17, 20, 24, 28, 32)),
                      (4, (17, 20, 24, 28, 32))):
        t0 = time.perf_counter()
        recs = xqr.accuracy_sweep(limbs, 32, 32, gs, trials, seed=20260901)
        dt = time.perf_counter() - t0
        for r in recs:
            r.pop("log10_e")
            r["precision"] = NAMES[limbs]
            rows.append(r)
        print(f"table2 {NAMES[limbs]}: {len(gs)} g values x {trials} trials in {dt:.1f} s", flush=True)
    return rows


def device_solve_ms(limbs, a, b, reps=3):
    import torch

    m, n = a.shape[1], a.shape[0]
    ctx = xqr.context(0)
    da = torch.from_numpy(a[None]).cuda()
    db = torch.from_numpy(b[None]).cuda()
    dx = torch.zeros((1, n, 2, limbs), dtype=torch.float64, device="cuda")
    dz = torch.zeros((1, limbs), dtype=torch.float64, device="cuda")
    dst = torch.zeros(2, dtype=torch.int64, device="cuda")
    stream = torch.cuda.Stream()  # a real stream handle shared by torch events and the ctx
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    call = lambda: ctx.lsq_solve_batched_device(limbs, 1, m, n, da.data_ptr(), db.data_ptr(),
                                                dx.data_ptr(), dz.data_ptr(), dst.data_ptr())
    call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def quality_up(sizes, cpu_qd_max):
    import oracle  # CPU baseline leg: the reference compiled in place

    ref = oracle.reference() or oracle.port()
    out = []
    for n in sizes:
        row = {"n": n}
        for limbs in (2, 4):
            a, b = xqr.gen_systems(limbs, 1, n, n, 1.0, 1, -1)
            a, b = a[0], b[0]
            rec = {"gpu_ms": device_solve_ms(limbs, a, b)}
            x, z = xqr.lsq_solve(a, b)
            q, r = xqr.mgs_qr(a)
            rec["residual_e"] = float(xqr.residual_max_entry(a, q, r)[0])
            rec["orthogonality_defect"] = float(xqr.orthogonality_defect(q)[0])
            rec["z"] = float(z[0])
            if limbs == 2 or n <= cpu_qd_max:
                t0 = time.perf_counter()
                cx, cz, st = ref.lsq_solve(a, b)
                rec["cpu_ms_1core"] = 1e3 * (time.perf_counter() - t0)
                rec["cpu_bitwise_equal"] = bool(np.array_equal(cx.view(np.uint64), x.view(np.uint64)))
            row[NAMES[limbs]] = rec
        if "cpu_ms_1core" in row["cdd"]:
            row["quality_up_gpu_cqd_vs_cpu_cdd"] = row["cdd"]["cpu_ms_1core"] / row["cqd"]["gpu_ms"]
        out.append(row)
        print(f"quality-up n={n}: {json.dumps(row)}", flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=1000)
    ap.add_argument("--sizes", default="32,80,256")
    ap.add_argument("--cpu-qd-max", type=int, default=80)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_paper_tables.json"))
    args = ap.parse_args()
    res = {"table2": table2(args.trials),
           "quality_up": quality_up([int(v) for v in args.sizes.split(",")], args.cpu_qd_max),
           "host_cores": os.cpu_count()}
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
    print("wrote", args.out)


if __name__ == "__main__":
    main()
