"""Element sharding across GPUs.

SEM elements are independent: element e reads only u[:,:,:,e], g[...,e] and
the shared d, and writes only w[:,:,:,e].  With the
column-major layouts (fortran.py:638-658) e is the slowest dimension, so an
element range is one contiguous byte range of u, g and w.  Rank r of P owns a
contiguous range of whole logical work-groups (blocks of l.0 elements, so
every shard still satisfies the kernel's ``nelt mod B = 0`` assumption); d is
replicated.  There is no data-path collective: the only communication is one
all-reduce of the fused sum(w*w) verification norm, outside the timed region.
One process per GPU (torch.distributed, NCCL over NVLink on the box, gloo in
the CPU tests).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(nelt, rank, world, block=1):
    """[lo, hi) of the elements rank *rank* of *world* owns.

    Splits whole blocks of *block* elements as evenly as possible; a ragged
    final block (nelt not a multiple of block) goes to the last rank.
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    nblocks = nelt // block
    lo_b = nblocks * rank // world
    hi_b = nblocks * (rank + 1) // world
    lo = lo_b * block
    hi = hi_b * block if rank < world - 1 else nelt
    return lo, hi


def allreduce_sum(value, device=None, group=None):
    """Sum a python float over ranks (NCCL on CUDA, gloo on CPU)."""
    if not dist.is_available() or not dist.is_initialized():
        return float(value)
    backend = dist.get_backend(group)
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) \
            if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.item())


def allreduce_max(value, device=None, group=None):
    if not dist.is_available() or not dist.is_initialized():
        return float(value)
    backend = dist.get_backend(group)
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) \
            if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def shard_params(params, nelt_name, lo, hi):
    """Parameter binding of one shard (the shard is itself a SEM problem)."""
    out = dict(params)
    out[nelt_name] = hi - lo
    return out
