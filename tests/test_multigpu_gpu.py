"""GPU: the N > 1 batch-sharded path on one device.

Two processes (gloo over 127.0.0.1, both on cuda:0 -- a one-GPU box runs the
same code path the 8-GPU node runs with one GPU per rank) each solve their
contiguous shard of a global batch of cqd 128x128 systems (BASELINE configs[4]
shape) through the C ABI, with no data collective.  Every rank's results must
equal, bit for bit, the single-process solve of the same global systems
(system s always draws split_mix64(1).split(s)), and rank 0's first streams
the reference's golden x / z.  Then bench.py itself runs under
torch.distributed.run with 2 ranks (BENCH_DIST_BACKEND=gloo) and must print
one JSON line from rank 0 (experiment.hpp:127-137 is the serial loop these
shards replace)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
L, M, N, TOTAL = 4, 128, 128, 10


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    import paper_1210_0800_b200 as xqr
    from paper_1210_0800_b200.sharding import max_over_ranks, shard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    first, cnt = shard(TOTAL, rank, world, "strong")
    a, b = xqr.gen_systems(L, cnt, M, N, 1.0, 1, first)
    x, z, codes, _ = xqr.lsq_solve_batched(a, b)
    # the device-pointer entry point on the same shard
    ctx = xqr.context(0)
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    dx = torch.zeros((cnt, N, 2, L), dtype=torch.float64, device="cuda")
    dz = torch.zeros((cnt, L), dtype=torch.float64, device="cuda")
    dst = torch.zeros((cnt, 2), dtype=torch.int64, device="cuda")
    ctx.lsq_solve_batched_device(L, cnt, M, N, da.data_ptr(), db.data_ptr(), dx.data_ptr(), dz.data_ptr(),
                                 dst.data_ptr())
    torch.cuda.synchronize()
    same = bool(np.array_equal(dx.cpu().numpy().view(np.uint64), x.view(np.uint64)))
    t = max_over_ranks(float(rank + 1), dist, "cpu")
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), first=first, cnt=cnt, x=x, z=z, codes=codes,
             device_equal=same, tmax=t)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_equal_single_run(tmp_path):
    import torch.multiprocessing as mp

    import paper_1210_0800_b200 as xqr

    a, b = xqr.gen_systems(L, TOTAL, M, N, 1.0, 1, 0)
    x1, z1, c1, _ = xqr.lsq_solve_batched(a, b)
    assert not c1.any()
    mp.spawn(_rank, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    seen = 0
    for r in range(2):
        d = np.load(tmp_path / f"rank{r}.npz")
        first, cnt = int(d["first"]), int(d["cnt"])
        assert first == seen and cnt == TOTAL // 2
        seen += cnt
        assert not d["codes"].any()
        assert bool(d["device_equal"]), f"rank {r}: device entry != host entry"
        assert float(d["tmax"]) == 2.0
        assert np.array_equal(d["x"].view(np.uint64), x1[first:first + cnt].view(np.uint64)), f"rank {r} x"
        assert np.array_equal(d["z"].view(np.uint64), z1[first:first + cnt].view(np.uint64)), f"rank {r} z"
        if first == 0:
            for s in range(4):
                g = np.load(os.path.join(GOLDEN, f"bench_cqd_128x128_s{s}.npz"))
                assert np.array_equal(d["x"][s].view(np.uint64), g["x"].view(np.uint64)), f"golden s{s}"
    assert seen == TOTAL


def test_bench_two_ranks_one_line():
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--steps", "1", "--warmup", "1", "--batch", "40", "--e2e-steps", "1", "--no-single", "--no-cpu"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["systems_total"] == 40 and d["config"]["systems_per_gpu"] == 20
    assert d["status"]["failed_systems"] == 0 and d["status"]["bitwise_vs_reference_streams_0_3"]
    assert d["e2e"]["e2e_matches_device"] and d["e2e"]["e2e_bad_systems"] == 0
    assert d["value"] > 0 and d["gpu_launches"] >= 1
