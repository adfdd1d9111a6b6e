"""The N>1 host path on CPU: world_size 2 over gloo (127.0.0.1).  Plan inputs
are broadcast from rank 0, each rank takes a contiguous shard of the sweep,
the per-rank rows are gathered back in input order and step times are
reduced with MAX — the same calls bench.py makes over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2510_04825_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    env = parallel.dist_env()
    rng = np.random.default_rng(0)
    arrays = {"X": rng.standard_normal((50, 7)), "S": np.arange(10, dtype=np.int64) * 3,
              "w": rng.uniform(0.5, 2, 10), "none": None} if env.rank == 0 else {}
    got = parallel.broadcast_inputs(arrays, src=0)
    assert got["none"] is None
    ref = {"X": np.random.default_rng(0).standard_normal((50, 7))}
    ok_bcast = np.array_equal(got["X"], ref["X"]) and np.array_equal(got["S"], np.arange(10) * 3)
    P = 23
    params = list(np.linspace(0.5, 2.0, P))
    mine = parallel.shard(params, env.world, env.rank)
    local = np.array([[p, p * p, -p] for p in mine])     # stand-in per-p result rows
    full = parallel.gather_rows(local, P)
    ok_gather = np.array_equal(full, np.array([[p, p * p, -p] for p in params]))
    status = parallel.gather_rows(np.full(len(mine), rank, dtype=np.int32), P)
    import torch
    loc = torch.full((4, 3), float(rank))
    allg = torch.empty((4 * world, 3))
    parallel.all_gather_device(allg, loc)
    ok_gather = ok_gather and bool((allg[:4] == 0).all() and (allg[4:] == 1).all())
    t = parallel.max_over_ranks(1.5 + rank)
    parallel.barrier()
    out[rank] = (bool(ok_bcast), bool(ok_gather), float(t), status.tolist())
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_broadcast_shard_gather():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for rank in range(world):
        ok_b, ok_g, t, status = res[rank]
        assert ok_b and ok_g
        assert t == 2.5
        lo, hi = parallel.shard_bounds(23, 2, 0)
        assert status == [0] * (hi - lo) + [1] * (23 - hi)


def test_shard_bounds_cover_and_balance():
    for P in (0, 1, 7, 4096, 1_000_001):
        for world in (1, 2, 3, 8):
            spans = [parallel.shard_bounds(P, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == P
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
