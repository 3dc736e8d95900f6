"""Pole-sharded multi-GPU stepping ("all the inverse
operators in the approximation of the operator exponential can be applied
independently").  One process per GPU; rank r owns a contiguous range of half
poles; per step every rank computes its partial pole sums E (rexp_step_partial),
the sums are all-reduced over NVLink (NCCL), and every rank runs the velocity
recovery (rexp_step_finish) on the summed E.  The all-reduce is the only
exchange; it carries nE * 2 nrhs * N doubles per step.
"""
from __future__ import annotations


def half_range(nh: int, rank: int, world: int):
    """Contiguous, balanced split of nh half poles: [lo, hi) for this rank."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    if nh < world:
        raise ValueError(f"{nh} half poles cannot be split over {world} ranks")
    return nh * rank // world, nh * (rank + 1) // world


class ShardedStepper:
    """u <- step(u) with poles split over the ranks of `group` (torch.distributed)."""

    def __init__(self, handle, group=None):
        import torch
        self.h = handle
        self.group = group
        self.e = torch.zeros(handle.partial_len, dtype=torch.float64, device=f"cuda:{handle.device}")

    def step(self, u):
        import torch.distributed as dist

        from . import api
        api.step_partial(self.h, u, self.e)
        dist.all_reduce(self.e, group=self.group)
        api.step_finish(self.h, self.e, u)
        return u
