"""The p-sharded multi-rank solve (parallel.py) against the 1-rank solve,
bitwise.  Two ranks run as two processes on cuda:0 with gloo host
collectives (this box has one GPU; the ranks never wait on each other inside
a kernel): rank 0 runs the offline phase, X/S/w are broadcast, each rank
builds its own plan and solves its contiguous shard, the coefficient,
residual and status rows are all-gathered in input order.  Every per-p
reduction has a fixed order and the kernels' launch shapes do not depend on
the batch (K3's split-K is a plan property), so the gathered rows must equal a
single-process solve of the whole sweep bit for bit."""
import os
import socket
import sys
import tempfile
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu

CASES = {"gauss": (2, dict(n=3000), 203), "stencil": (3, dict(grid=120), 301), "affine_c128": (4, dict(grid=60), 157)}


def _rank(rank, world, port, case, out):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK="0")
    import torch
    import torch.distributed as dist

    from paper_2510_04825_b200 import online, parallel, problems
    from paper_2510_04825_b200.offline import RowSelector, SnapshotBasis, offline
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, kw, P = CASES[case]
    prob = problems.build(cfg, **kw)
    arrays = {}
    if rank == 0:
        basis, sel = offline(prob, device=torch.device("cuda:0"))
        arrays = {"X": basis.basis, "S": sel.indices, "w": sel.weights, "sv": basis.singular_values}
    arrays = parallel.broadcast_inputs(arrays, src=0, device_keys=("X",))
    basis = SnapshotBasis(points=tuple(prob.snapshot_points), raw=arrays["X"], basis=arrays["X"],
                          singular_values=arrays["sv"])
    sel = RowSelector(indices=arrays["S"], n=prob.system.n, weights=arrays["w"])
    plan = online.precompute_online(prob.system, basis, sel, device=0)
    params = prob.test_params(P)
    mine = parallel.shard(params, world, rank)
    res = online.solve_params(plan, mine)
    coef = parallel.gather_rows(res.coefficients, P)
    sres = parallel.gather_rows(res.sampled_residual, P)
    st = parallel.gather_rows(res.status, P)
    if rank == 0:
        np.savez(out, coef=coef, sres=sres, status=st, X=arrays["X"], S=arrays["S"],
                 w=np.zeros(0) if arrays["w"] is None else arrays["w"], sv=arrays["sv"])
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("case", sorted(CASES))
def test_two_rank_shards_equal_one_rank_bitwise(case):
    import torch
    import torch.multiprocessing as mp

    from paper_2510_04825_b200 import online, problems
    from paper_2510_04825_b200.offline import RowSelector, SnapshotBasis
    with tempfile.TemporaryDirectory() as tmp:
        out = str(Path(tmp) / "gathered.npz")
        mp.start_processes(_rank, args=(2, _free_port(), case, out), nprocs=2, join=True, start_method="spawn")
        g = dict(np.load(out))
    cfg, kw, P = CASES[case]
    prob = problems.build(cfg, **kw)
    basis = SnapshotBasis(points=tuple(prob.snapshot_points), raw=g["X"], basis=g["X"], singular_values=g["sv"])
    sel = RowSelector(indices=g["S"], n=prob.system.n, weights=g["w"] if g["w"].size else None)
    torch.cuda.set_device(0)
    plan = online.precompute_online(prob.system, basis, sel, device=0)
    one = online.solve_params(plan, prob.test_params(P))
    assert np.all(one.status == 0) and np.array_equal(g["status"], one.status)
    assert np.array_equal(g["coef"], one.coefficients.astype(g["coef"].dtype)), case
    assert np.array_equal(g["sres"], one.sampled_residual), case
