"""Data-parallel plumbing (torch.distributed): the batch dimension m is sharded over ranks,
one process per GPU; the only exchange of the method is the sum of dtheta over ranks
(dtheta is a sum over columns, "d <- A 1"), done with one all_reduce(SUM)
over NCCL (NVLink/NVSwitch) or gloo (CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_columns(m: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous column block [c0, c1) of rank `rank` (sizes differ by at most one)."""
    base, rem = divmod(m, world)
    c0 = rank * base + min(rank, rem)
    return c0, c0 + base + (1 if rank < rem else 0)


def allreduce_dtheta(dtheta: torch.Tensor, group=None, deterministic: bool = False) -> torch.Tensor:
    """dtheta_total = sum over ranks, in place. deterministic=True gathers the per-rank partials
    and sums them in rank order (bitwise reproducible for a fixed world size)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return dtheta
    if dtheta.is_cuda and dist.get_backend(group) == "gloo":
        # gloo (CPU tests, or several ranks sharing one GPU) reduces host tensors: stage through the host
        host = dtheta.cpu()
        allreduce_dtheta(host, group=group, deterministic=deterministic)
        dtheta.copy_(host)
        return dtheta
    if not deterministic:
        dist.all_reduce(dtheta, op=dist.ReduceOp.SUM, group=group)
        return dtheta
    world = dist.get_world_size(group)
    parts = [torch.empty_like(dtheta) for _ in range(world)]
    dist.all_gather(parts, dtheta, group=group)
    acc = parts[0].clone()
    for p in parts[1:]:
        acc += p
    dtheta.copy_(acc)
    return dtheta
