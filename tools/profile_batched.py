"""One batched lsq_solve launch (for ncu): python tools/profile_batched.py L m n batch [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1210_0800_b200 as xqr  # noqa: E402

L, m, n, batch = (int(v) for v in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 1
ctx = xqr.Context(0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx.set_stream(s.cuda_stream)
a, b = xqr.gen_systems(L, batch, m, n, 1.0, 1, 0 if batch > 1 else -1)
da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
dx = torch.zeros((batch, n, 2, L), dtype=torch.float64, device="cuda")
dz = torch.zeros((batch, L), dtype=torch.float64, device="cuda")
dst = torch.zeros((batch, 2), dtype=torch.int64, device="cuda")
for _ in range(reps):
    ctx.lsq_solve_batched_device(L, batch, m, n, da.data_ptr(), db.data_ptr(), dx.data_ptr(),
                                 dz.data_ptr(), dst.data_ptr())
torch.cuda.synchronize()
print("kernel ms (last launch):", ctx.last_kernel_ms, "failed:", int((dst[:, 0] & 0xFFFFFFFF).ne(0).sum()))
