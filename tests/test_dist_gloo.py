"""Multi-process (world_size 2, gloo, CPU) tests of the collective helpers in
paper_1602_02244_b200/dist.py: they only move bytes, so they run
unchanged on CPU tensors. The whole LET protocol over gloo is in tests/test_let.py;
the CUDA mat-vec itself is covered by the -m gpu tests. `_OwnRangeDirect` is a
test double for the replicated mode of fmm_matvec (world > 1, global q): exact
values for the owned targets, zeros elsewhere, reassembled by scatter_sum.
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
        from paper_1602_02244_b200.dist import all_to_all_v, gather_counts, gather_rows, scatter_sum

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
        # replicated mode: every rank evaluates its owned targets of the global q, scatter_sum reassembles
        plan = _OwnRangeDirect(xa, 4, 8, 0.4, rank=rank, world=world)
        phi, g = plan.matvec(gather_rows(ql, list(counts)), grad=True)
        phi_l = scatter_sum(phi, list(counts), rank)
        g_l = scatter_sum(g, list(counts), rank)
        out[rank] = (phi_l.numpy().copy(), g_l.numpy().copy())
        # uneven all-to-all of rows (width 3): rank r sends (r + 1) * (d + 1) rows to d
        sc = [(rank + 1) * (d + 1) for d in range(world)]
        rc = [(r + 1) * (rank + 1) for r in range(world)]
        send = torch.cat([torch.full((c * 3,), 100.0 * rank + d, dtype=torch.float64) for d, c in enumerate(sc)])
        recv = all_to_all_v(send, sc, rc, 3)
        exp = torch.cat([torch.full((c * 3,), 100.0 * r + rank, dtype=torch.float64) for r, c in enumerate(rc)])
        assert torch.equal(recv, exp)
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
