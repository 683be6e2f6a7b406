"""Multi-GPU mat-vec: one process per GPU, torch.distributed (NCCL) for the plumbing.

Design ("replicated global tree, Morton-partitioned targets"):
every rank holds the global point set (all-gathered once at setup), builds the
identical global tree and lists in ``fmm_setup`` (so the interaction lists —
and hence the approximation — are the single-GPU ones, reading R12), and
evaluates only the targets of its contiguous Morton range of leaves
(``world_size``/``rank`` in ``fmm_exec``). Per mat-vec: all-gather of the
charges (8 B/point), local compute, one sum-reduce-scatter of the outputs
back to each caller's slice (non-owned entries are exact zeros, so the sum is
exact and order-independent).

The collective helpers only move bytes; they are unit-tested with the gloo
backend on CPU (tests/test_dist_gloo.py).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def _is_nccl(group=None) -> bool:
    return dist.get_backend(group) == "nccl"


def gather_counts(n_local: int, device, group=None) -> list[int]:
    world = dist.get_world_size(group)
    t = torch.tensor([n_local], dtype=torch.int64, device=device)
    out = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return [int(x.item()) for x in out]


def gather_rows(local: torch.Tensor, counts: list[int], group=None) -> torch.Tensor:
    """Concatenate every rank's rows (rank order) on every rank. local: [n_r, ...]."""
    world = len(counts)
    chunk = max(counts)
    tail = tuple(local.shape[1:])
    pad = torch.zeros((chunk, *tail), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    if _is_nccl(group):
        buf = torch.empty((world * chunk, *tail), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(buf, pad, group=group)
        parts = [buf[r * chunk: r * chunk + counts[r]] for r in range(world)]
    else:
        bufs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(bufs, pad, group=group)
        parts = [bufs[r][: counts[r]] for r in range(world)]
    return torch.cat(parts, 0)


def scatter_sum(global_rows: torch.Tensor, counts: list[int], rank: int, group=None) -> torch.Tensor:
    """Sum ``global_rows`` [N, ...] over ranks and return this rank's slice (rank-order rows)."""
    world = len(counts)
    chunk = max(counts)
    tail = tuple(global_rows.shape[1:])
    pad = torch.zeros((world * chunk, *tail), dtype=global_rows.dtype, device=global_rows.device)
    off = 0
    for r in range(world):
        pad[r * chunk: r * chunk + counts[r]] = global_rows[off: off + counts[r]]
        off += counts[r]
    if _is_nccl(group):
        out = torch.empty((chunk, *tail), dtype=global_rows.dtype, device=global_rows.device)
        dist.reduce_scatter_tensor(out, pad, op=dist.ReduceOp.SUM, group=group)
        return out[: counts[rank]]
    dist.all_reduce(pad, op=dist.ReduceOp.SUM, group=group)
    return pad[rank * chunk: rank * chunk + counts[rank]].clone()


class DistributedPlan:
    """Collective counterpart of :class:`Plan`: each rank passes its caller-side slice."""

    def __init__(self, points_local: torch.Tensor, p: int, ncrit: int, theta: float, group=None,
                 plan_factory=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.counts = gather_counts(points_local.shape[0], points_local.device, group)
        self.n = sum(self.counts)
        xyz = gather_rows(points_local, self.counts, group)
        if plan_factory is None:
            from .fmm import Plan

            plan_factory = Plan
        self.plan = plan_factory(xyz, p, ncrit, theta, rank=self.rank, world=self.world)

    def matvec(self, q_local: torch.Tensor, grad: bool = False):
        q = gather_rows(q_local, self.counts, self.group)
        res = self.plan.matvec(q, grad=grad)
        phi, g = res if grad else (res, None)
        phi_l = scatter_sum(phi, self.counts, self.rank, self.group)
        if not grad:
            return phi_l
        return phi_l, scatter_sum(g, self.counts, self.rank, self.group)

    def stats(self) -> dict:
        return self.plan.stats()
