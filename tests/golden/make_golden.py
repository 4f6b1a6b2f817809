"""Generate the golden fixtures from the REFERENCE itself (oracle/_ref, the
unmodified reference headers compiled in place).  Run here, where
/root/reference exists:  python tests/golden/make_golden.py

Fixtures (float64 bit patterns, small):
  known_answers.npz   -- tiny systems from test_mgs.cpp (identity, 3-4-5, ...)
  sweep_<prec>.npz    -- criterion-7 grid (acceptance.cpp:264-296) digests
  bench_<cfg>.npz     -- x and z of the BASELINE configs (seed 1) + Q/R digests
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def digest(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def main():
    oracle.build(ref=True)
    R = oracle.reference()
    assert R is not None, "needs /root/reference"
    # criterion-7 grid digests: dims {8,32,33,64} x 20 seeds, rng seed*1009+dim
    for L, name in ((1, "cd"), (2, "cdd"), (4, "cqd")):
        rows = []
        for dim in (8, 32, 33, 64):
            for seed in range(20):
                a, b = R.gen_system(L, dim, dim, 1.0, seed * 1009 + dim)
                q, r, st = R.mgs_qr(a)
                x, z, st2 = R.lsq_solve(a, b)
                rows.append((dim, seed, st[0], st2[0], digest(q, r), digest(x, z)))
        np.savez_compressed(os.path.join(OUT, f"sweep_{name}.npz"),
                            dim=np.array([r[0] for r in rows]), seed=np.array([r[1] for r in rows]),
                            qr_code=np.array([r[2] for r in rows]), ls_code=np.array([r[3] for r in rows]),
                            qr_digest=np.array([r[4] for r in rows]),
                            ls_digest=np.array([r[5] for r in rows]))
        print("sweep", name, len(rows))
    # BASELINE configs, seed 1 (configs[0..3]) and the first batch streams of configs[4]
    cfgs = [("cdd_32x32", 2, 32, 32, 1, -1), ("cdd_256x256", 2, 256, 256, 1, -1),
            ("cqd_256x256", 4, 256, 256, 1, -1), ("cqd_512x256", 4, 512, 256, 1, -1)]
    cfgs += [(f"cqd_128x128_s{s}", 4, 128, 128, 1, s) for s in range(4)]
    for name, L, m, n, seed, stream in cfgs:
        a, b = R.gen_system(L, m, n, 1.0, seed, stream)
        x, z, st = R.lsq_solve(a, b)
        q, r, st2 = R.mgs_qr(a)
        np.savez_compressed(os.path.join(OUT, f"bench_{name}.npz"), limbs=L, m=m, n=n, seed=seed,
                            stream=stream, x=x, z=z, code=st[0], qr_code=st2[0],
                            a_digest=digest(a, b), qr_digest=digest(q, r))
        print("bench", name, st, st2)


if __name__ == "__main__":
    main()
