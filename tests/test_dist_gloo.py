"""Multi-process (world_size 2, gloo, CPU) tests of the multi-GPU host logic in
paper_1602_02244_b200/dist.py: the collectives only move bytes,
so they run unchanged on CPU tensors. The per-rank compute is a test double
(`_OwnRangeDirect`) that mimics libfmm's contract for world > 1: each rank
returns exact values for the targets it owns and exact zeros elsewhere, so
the reduce-scatter reassembles the global result in every caller's slice.
The CUDA mat-vec itself is covered by the -m gpu tests.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import fmm_inputs as F


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _OwnRangeDirect:
    """Test double for Plan(world > 1): direct sum over all points for the owned
    contiguous range of global rows, zeros elsewhere (like fmm_stats own_begin/own_end)."""

    def __init__(self, xyz, p, ncrit, theta, rank=0, world=1):
        self.x = xyz.numpy()
        n = self.x.shape[0]
        self.lo, self.hi = rank * n // world, (rank + 1) * n // world

    def matvec(self, q, grad=False):
        x, qq = self.x, q.numpy()
        n = x.shape[0]
        phi = np.zeros(n)
        g = np.zeros((n, 3))
        for i in range(self.lo, self.hi):
            d = x[i] - x
            r2 = (d * d).sum(1)
            m = r2 > 0
            r = np.sqrt(r2[m])
            phi[i] = (qq[m] / r).sum()
            g[i] = -(qq[m, None] * d[m] / (r**3)[:, None]).sum(0)
        phi_t, g_t = torch.from_numpy(phi), torch.from_numpy(g)
        return (phi_t, g_t) if grad else phi_t

    def stats(self):
        return {"own_begin": self.lo, "own_end": self.hi}


def _worker(rank, world, port, n, counts, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1602_02244_b200.dist import DistributedPlan, gather_counts, gather_rows, scatter_sum

        x, q = F.cube(n, seed=3)
        offs = np.concatenate([[0], np.cumsum(counts)])
        lo, hi = offs[rank], offs[rank + 1]
        xl = torch.from_numpy(x[lo:hi].copy())
        ql = torch.from_numpy(q[lo:hi].copy())
        assert gather_counts(hi - lo, torch.device("cpu")) == list(counts)
        xa = gather_rows(xl, list(counts))
        assert torch.equal(xa, torch.from_numpy(x))
        # scatter_sum of rank-disjoint contributions is exact
        contrib = torch.zeros(n, dtype=torch.float64)
        contrib[rank::world] = torch.arange(n, dtype=torch.float64)[rank::world]
        s = scatter_sum(contrib, list(counts), rank)
        assert torch.equal(s, torch.arange(n, dtype=torch.float64)[lo:hi])
        plan = DistributedPlan(xl, 4, 8, 0.4, plan_factory=_OwnRangeDirect)
        phi, g = plan.matvec(ql, grad=True)
        out[rank] = (phi.numpy().copy(), g.numpy().copy())
    finally:
        dist.destroy_process_group()


def _run(n, counts):
    world = len(counts)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n, counts, out), nprocs=world, join=True)
    return dict(out)


@pytest.mark.parametrize("counts", [(60, 60), (17, 103), (0, 120)])
def test_distributed_plan_reassembles_caller_slices(counts):
    n = sum(counts)
    res = _run(n, counts)
    x, q = F.cube(n, seed=3)
    full = _OwnRangeDirect(torch.from_numpy(x), 4, 8, 0.4)
    phi_ref, g_ref = full.matvec(torch.from_numpy(q), grad=True)
    offs = np.concatenate([[0], np.cumsum(counts)])
    for r in range(len(counts)):
        phi, g = res[r]
        assert phi.shape == (counts[r],) and g.shape == (counts[r], 3)
        np.testing.assert_array_equal(phi, phi_ref.numpy()[offs[r]:offs[r + 1]])
        np.testing.assert_array_equal(g, g_ref.numpy()[offs[r]:offs[r + 1]])
