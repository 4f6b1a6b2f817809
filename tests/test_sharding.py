"""CPU: batch sharding across ranks -- disjoint, covering
ranges; each rank's inputs are exactly the single-run draws
(split_mix64(seed).split(s), random.hpp:38-40); the max-over-ranks timing
reduction -- exercised with world_size 2 over gloo on 127.0.0.1."""
import os
import socket

import numpy as np
import pytest

from paper_1210_0800_b200.sharding import max_over_ranks, shard


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("batch", [0, 1, 7, 4096])
def test_shard_ranges(world, batch):
    # strong: contiguous, disjoint, covering [0, batch)
    nxt = 0
    for r in range(world):
        first, cnt = shard(batch, r, world, "strong")
        assert first == nxt and cnt >= 0
        nxt = first + cnt
    assert nxt == batch
    # weak: `batch` per rank, rank r at r*batch
    for r in range(world):
        assert shard(batch, r, world, "weak") == (r * batch, batch)
    with pytest.raises(ValueError):
        shard(batch, world, world)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    import oracle
    import paper_1210_0800_b200 as xqr

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, cnt = shard(5, rank, world, "strong")
    a, b = xqr.gen_systems(2, cnt, 6, 4, 1.0, 1, first)
    port_oracle = oracle.port()
    ok = True
    for s in range(cnt):
        wa, wb = port_oracle.gen_system(2, 6, 4, 1.0, 1, first + s)
        ok = ok and np.array_equal(a[s], wa) and np.array_equal(b[s], wb)
    mx = max_over_ranks(10.0 * (rank + 1), dist, "cpu")
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.array([first, cnt, int(ok), mx]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo(tmp_path, port):
    import torch.multiprocessing as mp

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = [np.load(tmp_path / f"r{r}.npy") for r in range(world)]
    assert [int(r[0]) for r in res] == [0, 3] and [int(r[1]) for r in res] == [3, 2]
    assert all(int(r[2]) == 1 for r in res), "sharded inputs differ from the single-run draws"
    assert all(r[3] == 20.0 for r in res), "max over ranks"
