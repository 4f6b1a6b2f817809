#!/usr/bin/env python3
"""Dev tool: time one build of the library on the batched headline workload
and fingerprint its results, so kernel variants can be compared on one box.

    XQR_B200_LIB=path/to/lib.so python tools/variant_bench.py [--batch 296] [--reps 3]
        [--m 128] [--n 128] [--limbs 4]

Prints one JSON line: ms per launch (CUDA events on the ctx stream), systems/s,
a sha256 of all x and z limbs (equal digests = bitwise-equal results), and
the golden check of streams 0..3 where fixtures exist."""
import argparse
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=296)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--m", type=int, default=128)
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--limbs", type=int, default=4)
    ap.add_argument("--qr", action="store_true")
    ap.add_argument("--single", action="store_true",
                    help="one system drawn from split_mix64(1) itself (the latency configs; grid kernels)")
    args = ap.parse_args()
    import torch

    import paper_1210_0800_b200 as xqr

    L, m, n, B = args.limbs, args.m, args.n, args.batch
    if args.single:
        B = 1
    a, b = xqr.gen_systems(L, B, m, n, 1.0, 1, -1 if args.single else 0)
    ctx = xqr.Context(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    dx = torch.zeros((B, n, 2, L), dtype=torch.float64, device="cuda")
    dz = torch.zeros((B, L), dtype=torch.float64, device="cuda")
    dq = torch.zeros_like(da) if args.qr else None
    dr = torch.zeros((B, n, n, 2, L), dtype=torch.float64, device="cuda") if args.qr else None
    dst = torch.zeros((B, 2), dtype=torch.int64, device="cuda")

    def call():
        if args.qr:
            ctx.mgs_qr_batched_device(L, B, m, n, da.data_ptr(), dq.data_ptr(), dr.data_ptr(), dst.data_ptr())
        else:
            ctx.lsq_solve_batched_device(L, B, m, n, da.data_ptr(), db.data_ptr(), dx.data_ptr(),
                                         dz.data_ptr(), dst.data_ptr())

    call()
    torch.cuda.synchronize()
    times = []
    for _ in range(args.reps):
        call()
        torch.cuda.synchronize()
        times.append(ctx.last_kernel_ms)
    ms = float(np.median(times))
    h = hashlib.sha256()
    if args.qr:
        h.update(dq.cpu().numpy().tobytes())
        h.update(dr.cpu().numpy().tobytes())
    else:
        h.update(dx.cpu().numpy().tobytes())
        h.update(dz.cpu().numpy().tobytes())
    codes = dst.cpu().numpy()[:, 0] & 0xFFFFFFFF
    golden = None
    gname = os.path.join(ROOT, "tests", "golden", f"bench_{'cdd' if L == 2 else 'cqd'}_{m}x{n}.npz")
    if args.single and not args.qr and os.path.exists(gname):
        g = np.load(gname)
        golden = bool(np.array_equal(dx[0].cpu().numpy().view(np.uint64), g["x"].view(np.uint64))
                      and np.array_equal(dz[0].cpu().numpy().view(np.uint64), g["z"].view(np.uint64)))
    elif not args.qr and L == 4 and m == 128 and n == 128:
        golden = True
        for s in range(min(4, B)):
            g = np.load(os.path.join(ROOT, "tests", "golden", f"bench_cqd_128x128_s{s}.npz"))
            golden = golden and bool(np.array_equal(dx[s].cpu().numpy().view(np.uint64), g["x"].view(np.uint64)))
    print(json.dumps({"lib": os.environ.get("XQR_B200_LIB", "default"), "batch": B, "m": m, "n": n,
                      "limbs": L, "qr": args.qr, "ms": ms, "times": times, "sys_per_s": B / (ms / 1e3),
                      "digest": h.hexdigest()[:16], "failed": int((codes != 0).sum()), "golden_s0_3": golden}),
          flush=True)


if __name__ == "__main__":
    main()
