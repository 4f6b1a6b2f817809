"""Dev: end-to-end latency of single-system lsq_solve through the host-buffer
C ABI (median of 20 after 3 warm-ups), for the latency configs.
    python tools/e2e_single.py"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1210_0800_b200 as xqr  # noqa: E402

for L, m, n in ((2, 256, 256), (4, 256, 256), (4, 512, 256)):
    a, b = xqr.gen_systems(L, 1, m, n, 1.0, 1, -1)
    for _ in range(3):
        xqr.lsq_solve(a[0], b[0])
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        xqr.lsq_solve(a[0], b[0])
        ts.append(time.perf_counter() - t0)
    print(f"L={L} {m}x{n}: e2e {statistics.median(ts) * 1e3:.3f} ms", flush=True)
