"""Multi-GPU plumbing for the K-TanH hot path (host logic only).

BASELINE.json north_star item (c): the flat tensor is split into contiguous
per-GPU shards, one process per GPU, with NO collective on the data path --
K-TanH is elementwise, so there is no reduction or exchange step.  The only
collectives are timing plumbing (a barrier and a max/sum of scalars over
ranks), done with torch.distributed (NCCL on GPUs, gloo on CPU tests).

The shard rule is the library's kt_shard_range (native, include/ktanh.h).
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_ranks():
    """(rank, local_rank, world_size) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def init(backend: str | None = None, device: torch.device | None = None):
    """Initialise the default process group from env:// if WORLD_SIZE > 1."""
    rank, local_rank, world = env_ranks()
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        kw = {"device_id": device} if (backend == "nccl" and device is not None) else {}
        dist.init_process_group(backend, **kw)
    return rank, local_rank, world


def shard_range(n: int, world: int, rank: int, align: int = 16):
    """Contiguous [begin, begin + count) of rank's shard (kt_shard_range)."""
    from . import shard_range as _native
    return _native(n, world, rank, align)


def shard_view(t: torch.Tensor, world: int, rank: int, align: int = 16) -> torch.Tensor:
    """This rank's contiguous slice of a flat tensor (a view, no copy)."""
    flat = t.reshape(-1)
    b, c = shard_range(flat.numel(), world, rank, align)
    return flat[b:b + c]


def _reduce_scalar(v: float, op, device=None) -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(v)
    if dist.get_backend() != "nccl":
        device = torch.device("cpu")            # gloo reduces host tensors
    elif device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    t = torch.tensor([float(v)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=op)
    return float(t.item())


def max_over_ranks(v: float, device=None) -> float:
    return _reduce_scalar(v, dist.ReduceOp.MAX, device)


def sum_over_ranks(v: float, device=None) -> float:
    return _reduce_scalar(v, dist.ReduceOp.SUM, device)


def gather_over_ranks(values, device=None) -> list:
    """Every rank's list of floats (same length on all ranks), in rank order;
    [values] when not distributed.  Timing / bookkeeping plumbing only."""
    vals = [float(v) for v in values]
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [vals]
    if dist.get_backend() != "nccl":
        device = torch.device("cpu")
    elif device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    return [[float(v) for v in p.cpu()] for p in parts]


def barrier():
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def aggregate_throughput(elements_this_rank: int, ms_this_rank: float, device=None):
    """Whole-job throughput: all ranks' elements / the slowest rank's time.
    Returns (elements_total, ms_max, elements_per_second)."""
    total = sum_over_ranks(elements_this_rank, device)
    ms_max = max_over_ranks(ms_this_rank, device)
    return total, ms_max, total / (ms_max / 1e3)
