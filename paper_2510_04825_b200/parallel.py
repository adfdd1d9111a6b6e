"""p-value sharding across GPUs (one process per GPU, torch.distributed).

Every parameter value is an independent unit (solve_online "is
pure and safe to invoke concurrently over many p (the intended
parallelization axis)"), so the sweep is split into contiguous shards with no
collective on the data path.  The only collectives are the ones the
north_star names outside the per-p loop:

  * broadcast_inputs: X, S, weights and the operator arrays go from rank 0 to
    every rank once per plan (NCCL broadcast over NVLink on GPUs, gloo in the
    CPU tests) so the offline artefacts are computed once;
  * gather_rows: per-rank result rows are gathered to every rank in input
    order (all_gather of equal-size padded shards);
  * max_over_ranks: device-timed step times are reduced with MAX.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class DistEnv:
    rank: int
    world: int
    local_rank: int

    @property
    def is_root(self) -> bool:
        return self.rank == 0


def dist_env() -> DistEnv:
    return DistEnv(rank=int(os.environ.get("RANK", 0)), world=int(os.environ.get("WORLD_SIZE", 1)),
                   local_rank=int(os.environ.get("LOCAL_RANK", 0)))


def shard_bounds(P: int, world: int, rank: int):
    """Contiguous block [lo, hi) of P items for `rank` (sizes differ by <= 1)."""
    base, extra = divmod(P, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def shard(items, world: int, rank: int):
    lo, hi = shard_bounds(len(items), world, rank)
    return items[lo:hi]


def _device_for(backend: str, local_rank: int):
    import torch
    return torch.device(f"cuda:{local_rank}") if backend == "nccl" else torch.device("cpu")


def broadcast_inputs(arrays: dict, src: int = 0, local_rank: int = 0, device_keys=()) -> dict:
    """Broadcast a dict of numpy arrays from `src` to all ranks (shapes/dtypes
    first as an object, then one tensor broadcast per array).  Under NCCL the
    arrays named in `device_keys` (e.g. the basis X) are returned as CUDA
    tensors on this rank's device -- the plan consumes them in place
    (SAS_FLAG_INPUT_DEVICE), with no device->host->device round trip; every
    other array comes back as numpy."""
    import torch
    import torch.distributed as dist
    backend = dist.get_backend()
    dev = _device_for(backend, local_rank)
    meta = [{k: (None if v is None else (np.asarray(v).shape, str(np.asarray(v).dtype)))
             for k, v in arrays.items()} if dist.get_rank() == src else None]
    dist.broadcast_object_list(meta, src=src)
    out = {}
    for key, spec in sorted(meta[0].items()):
        if spec is None:  # e.g. an unweighted selector
            out[key] = None
            continue
        shape, dtype = spec
        npdt = np.dtype(dtype)
        if dist.get_rank() == src:
            a = np.ascontiguousarray(arrays[key])
            t = torch.from_numpy(a.view(np.uint8).reshape(-1).copy()).to(dev)
        else:
            t = torch.empty(int(np.prod(shape)) * npdt.itemsize, dtype=torch.uint8, device=dev)
        dist.broadcast(t, src=src)
        if key in device_keys and t.is_cuda:
            tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.complex128): torch.complex128}[npdt]
            out[key] = t.view(tdt).reshape(shape)
        else:
            out[key] = t.cpu().numpy().view(npdt).reshape(shape)
    return out


def gather_rows(local: np.ndarray, P: int, local_rank: int = 0) -> np.ndarray:
    """All-gather contiguous shards (rows of `local`) into the full P-row array
    in input order on every rank."""
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = _device_for(dist.get_backend(), local_rank)
    maxrows = max(hi - lo for lo, hi in (shard_bounds(P, world, q) for q in range(world)))
    row_shape = local.shape[1:]
    a = np.ascontiguousarray(local)
    rowbytes = int(np.prod(row_shape, dtype=np.int64)) * a.dtype.itemsize if row_shape else a.dtype.itemsize
    buf = np.zeros(maxrows * rowbytes, dtype=np.uint8)
    buf[:a.size * a.dtype.itemsize] = a.view(np.uint8).reshape(-1)
    t = torch.from_numpy(buf).to(dev)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    rows = []
    for q in range(world):
        lo, hi = shard_bounds(P, world, q)
        chunk = parts[q].cpu().numpy()[:(hi - lo) * rowbytes].view(a.dtype).reshape((hi - lo,) + row_shape)
        rows.append(chunk)
    return np.concatenate(rows, axis=0)


def all_gather_device(out, local):
    """All-gather equal-size shards of a device tensor into `out` in rank order
    (NCCL all_gather_into_tensor on GPUs; a host round trip under gloo)."""
    import torch
    import torch.distributed as dist
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out, local.contiguous())
        return out
    parts = [torch.empty_like(local, device="cpu") for _ in range(dist.get_world_size())]
    dist.all_gather(parts, local.cpu())
    out.copy_(torch.cat(parts, dim=0))
    return out


def max_over_ranks(value: float, local_rank: int = 0) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    dev = _device_for(dist.get_backend(), local_rank)
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(local_rank: int = 0):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        if dist.get_backend() == "nccl":
            dist.barrier(device_ids=[local_rank])
        else:
            dist.barrier()
