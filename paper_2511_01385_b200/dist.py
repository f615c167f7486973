"""Data-parallel plumbing for the rdFFT hot path (one process per GPU).

The transforms and the BCA forward are independent per vector / token, so
the batch is sharded with no collective (weak scaling: every rank owns a full
per-GPU batch).  The BCA backward has one real exchange: dw (fp32,
q_out*q_in*p) is summed over ranks — dw is linear in the tokens, so the sum of
per-shard dw equals the full-batch dw (Eq. 5).  torch.distributed provides the
process group (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) share of `total` units for `rank` (sizes differ by at most 1)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def allreduce_dw(dw: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the BCA weight gradient over data-parallel ranks, in place (fp32)."""
    if dw.dtype != torch.float32:
        raise ValueError("dw must be float32 (P:L486)")
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(dw, op=dist.ReduceOp.SUM, group=group)
    return dw


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
