"""Latency of single small systems through the device call (dev tool):
    python tools/small_latency.py          # grid kernels (default routing)
    XQR_FORCE_CTA=1 python tools/small_latency.py   # one-CTA kernel
"""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1210_0800_b200 as xqr
ctx = xqr.context(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
for L, m, n in [tuple(int(v) for v in c.split(",")) for c in (sys.argv[1:] or ["4,16,16", "4,32,32", "4,48,48", "4,64,64", "4,80,80", "2,64,64", "2,128,128"])]:
    a, b = xqr.gen_systems(L, 1, m, n, 1.0, 1, -1)
    da = torch.from_numpy(a).cuda(); db = torch.from_numpy(b).cuda()
    dx = torch.zeros((1, n, 2, L), dtype=torch.float64, device="cuda"); dz = torch.zeros((1, L), dtype=torch.float64, device="cuda")
    dst = torch.zeros((1, 2), dtype=torch.int64, device="cuda")
    call = lambda: ctx.lsq_solve_batched_device(L, 1, m, n, da.data_ptr(), db.data_ptr(), dx.data_ptr(), dz.data_ptr(), dst.data_ptr())
    call(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): call()
    e1.record(); torch.cuda.synchronize()
    print(f"L={L} {m}x{n}: {e0.elapsed_time(e1)/5*1e3:.0f} us", flush=True)
