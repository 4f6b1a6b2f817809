"""Phase timing of one single-system grid solve (dev tool): runs lsq_solve on
the reference generator's system with XQR_GRID_TRACE set and prints the
factorisation and back-substitution spans from the device timestamps.

    python tools/trace_single.py [--limbs 4] [--m 256] [--n 256] [--reps 3]
"""
import argparse
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--limbs", type=int, default=4)
    ap.add_argument("--m", type=int, default=256)
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--phases", action="store_true", help="finisher phase cycles (back substitution)")
    ap.add_argument("--pivots", action="store_true", help="per-pivot phases of the factorisation")
    ap.add_argument("--split", action="store_true", help="with --pivots: split the critical update")
    args = ap.parse_args()
    path = os.path.join(tempfile.mkdtemp(), "trace.txt")
    os.environ["XQR_GRID_TRACE"] = path
    import paper_1210_0800_b200 as xqr

    a, b = xqr.gen_systems(args.limbs, 1, args.m, args.n, 1.0, 1, -1)
    for rep in range(args.reps):
        xqr.lsq_solve(a[0], b[0])
        t = np.loadtxt(path, dtype=np.uint64)
        last = t[-1]
        start, grid_end, bs_start, bs_end = int(last[8]), int(last[5]), int(last[6]), int(last[7])
        fact = (grid_end - start) / 1e3 if start else float("nan")
        pre_end = int(last[3]) if args.limbs == 4 else 0  # xgrid2: norm pre-pass done (row n, slot 2)
        if pre_end and start:
            print(f"  pre-pass (column norms + threshold) {(pre_end - start) / 1e3:.1f} us")
        if args.pivots and args.limbs <= 2:
            # xgrid1 stamps: 0 q_{j-1} in hand, 1 column j updated, 4 norm tree,
            # 5 sqrt, 6 reciprocal, 7 divided, 2 published
            T = t[:, 1:9].astype(np.int64)
            rows = [[T[j][0] - T[j - 1][2], T[j][1] - T[j][0], T[j][4] - T[j][1], T[j][5] - T[j][4],
                     T[j][6] - T[j][5], T[j][7] - T[j][6], T[j][2] - T[j][7]]
                    for j in range(2, args.n - 1) if min(T[j][0], T[j][1], T[j][2], T[j][7], T[j - 1][2]) > 0]
            if rows:
                avg = np.array(rows, dtype=np.float64).mean(axis=0) / 1e3
                print("  dd pivots: handoff %.2f, update %.2f, normtree %.2f, sqrt %.2f, recip %.2f, "
                      "divide %.2f, publish %.2f us" % tuple(avg))
            if args.split:
                D = t[:, 9].astype(np.int64)  # dot product of the critical update done
                sp = [[D[j] - T[j][0], T[j][1] - D[j]] for j in range(2, args.n - 1) if min(D[j], T[j][0], T[j][1]) > 0]
                if sp:
                    print("  update split (us): dot %.2f, axpy+sync %.2f" % tuple(np.array(sp, dtype=np.float64).mean(axis=0) / 1e3))
        elif args.pivots:
            # per pivot j (row j of the trace, globaltimer ns): 0 q_{j-1} in hand,
            # 1 column j updated, 4 norm tree, 5 sqrt, 6 reciprocal, 7 divided,
            # 2 published; 3 last cluster done with round j-1
            T = t[:, 1:9].astype(np.int64)
            n = args.n
            rows = []
            for j in range(2, n - 1):
                cur, prv = T[j], T[j - 1]
                if min(cur[0], cur[1], cur[2], cur[4], cur[5], cur[6], cur[7], prv[2]) == 0:
                    continue
                rows.append([cur[0] - prv[2], cur[1] - cur[0], cur[4] - cur[1], cur[5] - cur[4],
                             cur[6] - cur[5], cur[7] - cur[6], cur[2] - cur[7], cur[2] - prv[2]])
            rows = np.array(rows, dtype=np.float64) / 1e3
            names = ["handoff", "update", "normtree", "sqrt", "recip", "divide", "publish", "pivot"]
            if args.split:
                sp = []
                for j in range(2, n - 1):
                    cur = T[j]
                    tt = int(t[j, 16])
                    if min(cur[0], cur[1], cur[3], tt) == 0 or not cur[0] <= tt <= cur[1]:
                        continue  # (no tree stamp in this build: the slot holds back-substitution data)
                    sp.append([cur[3] - cur[0], tt - cur[3], cur[1] - tt])
                if sp:
                    sp = np.array(sp, dtype=np.float64) / 1e3
                    print("  update split (us): leaf %.1f, tree %.1f, axpy+sync %.1f" % tuple(sp.mean(axis=0)))
            for lo, hi in ((0, len(rows) // 3), (len(rows) // 3, 2 * len(rows) // 3), (2 * len(rows) // 3, len(rows))):
                avg = rows[lo:hi].mean(axis=0)
                print(f"  pivots {lo + 2}-{hi + 1}: " + ", ".join(f"{k} {v:.1f}" for k, v in zip(names, avg)) + " us")
        if args.phases:
            n_rows = t.shape[0] - 1
            c = t[1:-1, 9:14].astype(np.int64)  # back-substitution steps k = 1 .. n-1 (SM cycles)
            c = c[c[:, 0] != 0]
            ph = np.diff(c, axis=1).mean(axis=0)
            loop = (c[:-1, 0] - c[1:, 4]).mean() if len(c) > 1 else 0
            print(f"  finisher cycles/step: wait {ph[0]:.0f}, update {ph[1]:.0f}, smith {ph[2]:.0f}, "
                  f"publish {ph[3]:.0f}, loop {loop:.0f}")
            # updater of the finisher's next input: row k-1 slots 5/6 = x_k taken / x_{k-2} updated;
            # x_k published at the end of step k+1 (row k+1 slot 3)
            B = t[:, 9:16].astype(np.int64)
            u = [(B[k - 1, 5] - B[k + 1, 3], B[k - 1, 6] - B[k - 1, 5], B[k - 1, 0] - B[k - 1, 6])
                 for k in range(3, n_rows - 1) if B[k - 1, 5] and B[k - 1, 6] and B[k + 1, 3] and B[k - 1, 0]]
            sp = t[2:-1, 16].astype(np.int64)
            W = (t[2:-1, 10].astype(np.int64) - t[2:-1, 9].astype(np.int64))
            ks = np.arange(2, n_rows)
            for lo in range(0, n_rows, 32):
                sel = (ks >= lo) & (ks < lo + 32) & (t[2:-1, 9] != 0)
                if sel.any():
                    print(f"    steps {lo}-{lo + 31}: wait {W[sel].mean():.0f} cycles, "
                          f"waiting {(sp[sel] > 0).mean() * 100:.0f} %, spins {sp[sel].mean():.1f}")
            if u:
                u = np.array(u, dtype=np.float64).mean(axis=0)
                print(f"  next-input updater cycles: poll {u[0]:.0f}, update {u[1]:.0f}, "
                      f"slack to the finisher {u[2]:.0f}")
        print(f"rep {rep}: factorisation {fact:.1f} us, gap {(bs_start - grid_end) / 1e3:.1f} us, "
              f"back substitution {(bs_end - bs_start) / 1e3:.1f} us", flush=True)


if __name__ == "__main__":
    main()
