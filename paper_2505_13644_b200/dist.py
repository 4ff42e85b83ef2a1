"""Batch sharding for data-parallel operator evaluation.

Points are independent: rank r of G evaluates the contiguous slice
[offset_r, offset_r + count_r) of the global batch, passing offset_r as
`point_offset` so randomized directions are identical to a 1-GPU run. No
collective is needed inside the method; `gather` concatenates the per-rank
results on every rank (NCCL all_gather over NVLink/NVSwitch, or gloo on CPU).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """(offset, count) of rank's contiguous slice; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world or n_total < 0:
        raise ValueError("bad shard arguments")
    base, rem = divmod(n_total, world)
    count = base + (1 if rank < rem else 0)
    offset = rank * base + min(rank, rem)
    return offset, count


def gather(local: torch.Tensor, n_total: int, group=None) -> torch.Tensor:
    """Concatenate the per-rank slices (in rank order) into the [n_total, ...] result."""
    world = dist.get_world_size(group)
    counts = [shard(n_total, r, world)[1] for r in range(world)]
    cmax = max(counts)
    pad = torch.zeros((cmax,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = torch.empty((world * cmax,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    return torch.cat([out[r * cmax: r * cmax + counts[r]] for r in range(world)])


def allreduce_grads(grads, group=None):
    """Data-parallel training: rank r's ctm_backward gives the gradient of
    its shard's sum_n gop[n] op[n] + gf[n] f[n]; the global gradient is the SUM over ranks
    (a mean loss puts 1/n_total into the cotangents). One flat all_reduce bucket per step
    (C1: 1.27 M parameters, 5 MB), NCCL over NVLink/NVSwitch on GPUs, gloo on CPU.
    grads: [(dW_l, db_l)], summed in place."""
    flat = torch.cat([t.reshape(-1) for pair in grads for t in pair])
    dist.all_reduce(flat, group=group)
    off = 0
    for pair in grads:
        for t in pair:
            n = t.numel()
            t.copy_(flat[off:off + n].view_as(t))
            off += n
    return grads
