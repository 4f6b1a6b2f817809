"""Compare one shape against the oracle and print where the device differs (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_1210_0800_b200 as xqr  # noqa: E402

L, m, n, seed = (int(v) for v in sys.argv[1:5])
port = oracle.port()
a, b = port.gen_system(L, m, n, 1.0, seed)
q, r, st = port.mgs_qr(a)
gq, gr = xqr.mgs_qr(a)
for name, g, w in (("Q", gq, q), ("R", gr, r)):
    gb, wb = g.view(np.uint64), w.view(np.uint64)
    bad = np.argwhere(gb != wb)
    print(name, "differs at", len(bad), "limbs; first:", bad[:6].tolist())
    if len(bad):
        idx = tuple(bad[0])
        print("   got", g[idx[:-1]], "\n  want", w[idx[:-1]])
x, z, st = port.lsq_solve(a, b)
gx, gz = xqr.lsq_solve(a, b)
print("x equal", np.array_equal(gx.view(np.uint64), x.view(np.uint64)), "z equal",
      np.array_equal(gz.view(np.uint64), z.view(np.uint64)))
