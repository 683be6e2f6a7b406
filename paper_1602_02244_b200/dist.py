"""Multi-GPU mat-vec: one process per GPU, torch.distributed (NCCL) for the plumbing.

Design (north_star "Morton-ordered domain decomposition, with a
local-essential-tree exchange (boundary multipoles plus halo particles) over
NCCL/NVLink"): every rank builds the same global tree and lists
from the all-gathered points (so the approximation is the single-GPU one,
reading R12) and owns a contiguous Morton range of leaves (cut by estimated
work). Over NCCL the library itself runs everything (collective mode,
include/fmm.h fmm_exec.nccl_id): this module only broadcasts the ncclUniqueId.
Over other backends (gloo: the CPU tests) the library (fmm_let_*) packs and
unpacks device buffers and this module moves them:

    Q      all-to-all-v   charges to their owner and to the ranks whose near
                          field needs them (halo leaves)
    SHARED all-gather     partial multipoles of cells straddling ranks
    M      all-to-all-v   boundary multipoles (own cells used by other ranks' M2L)
    PHI    all-to-all-v   results back to the callers' slices

Only bytes move here; every arithmetic step runs in libfmm kernels. The
collectives are unit-tested with gloo on CPU (tests/test_dist_gloo.py,
tests/test_let.py); ``let_matvec_local`` runs the same protocol for several
plans in ONE process (buffer copies instead of collectives) so the GPU tests
check the multi-rank path against the single-GPU mat-vec on one device.
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


def all_to_all_v(send: torch.Tensor, send_counts: list[int], recv_counts: list[int], width: int = 1,
                 group=None) -> torch.Tensor:
    """Uneven all-to-all of rows of ``width`` doubles (torch.distributed.all_to_all_single)."""
    recv = torch.empty(sum(recv_counts) * width, dtype=send.dtype, device=send.device)
    dist.all_to_all_single(recv, send.reshape(-1), [c * width for c in recv_counts], [c * width for c in send_counts],
                           group=group)
    return recv


class LetBuffers:
    """Per-rank device buffers of the LET protocol, sized from the plan's counts."""

    def __init__(self, plan, grad: bool):
        L = plan.let
        dev = plan.device
        f = dict(dtype=torch.float64, device=dev)
        ncd, world = L["ncd"], plan.world
        self.q_send = torch.empty(sum(L["q_send"]), **f)
        self.shared_send = torch.empty(L["shared"] * ncd, **f)
        self.m_send = torch.empty(sum(L["m_send"]) * ncd, **f)
        self.phi_send = torch.empty(sum(L["phi_send"]), **f)
        self.grad_send = torch.empty(3 * sum(L["phi_send"]), **f) if grad else None
        self.shared_recv = torch.empty(world * L["shared"] * ncd, **f)


class DistributedPlan:
    """Collective counterpart of :class:`Plan`: each rank passes its caller-side slice of the
    points; ``matvec`` takes and returns that rank's slice of q / phi (/ grad)."""

    def __init__(self, points_local: torch.Tensor, p: int, ncrit: int, theta: float, group=None,
                 plan_factory=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.counts = gather_counts(points_local.shape[0], points_local.device, group)
        self.n = sum(self.counts)
        self.collective = False
        if plan_factory is None and self.world > 1 and _is_nccl(group):
            # collective mode (include/fmm.h fmm_exec.nccl_id): libfmm gathers the points, builds
            # the global tree and moves the whole exchange with NCCL on the plan's stream; this
            # layer only hands it the ncclUniqueId (rank 0 makes it, the group broadcasts it)
            from .fmm import Plan, nccl_unique_id

            idt = torch.zeros(128, dtype=torch.uint8, device=points_local.device)
            if self.rank == 0:
                idt.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(idt, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
            self.plan = Plan(points_local, p, ncrit, theta, rank=self.rank, world=self.world,
                             nccl_id=bytes(idt.cpu().numpy().tobytes()))
            self.collective = True
            self.let = None
            self._buf = {}
            return
        xyz = gather_rows(points_local, self.counts, group)
        if plan_factory is None:
            from .fmm import Plan

            plan_factory = Plan
        self.plan = plan_factory(xyz, p, ncrit, theta, rank=self.rank, world=self.world)
        self.let = self.plan.let_setup(self.counts) if self.world > 1 else None
        self._buf = {}

    def _buffers(self, grad):
        if grad not in self._buf:
            self._buf[grad] = LetBuffers(self.plan, grad)
        return self._buf[grad]

    def matvec(self, q_local: torch.Tensor, grad: bool = False):
        if self.world == 1 or self.collective:
            return self.plan.matvec(q_local, grad=grad)
        L, pl, g = self.let, self.plan, self.group
        B = self._buffers(grad)
        ncd = L["ncd"]
        pl.let_pack_q(q_local, B.q_send)
        q_recv = all_to_all_v(B.q_send, L["q_send"], L["q_recv"], 1, g)
        pl.let_upward(q_recv, B.shared_send, B.m_send)
        if L["shared"]:
            if _is_nccl(g):
                dist.all_gather_into_tensor(B.shared_recv, B.shared_send, group=g)
            else:
                parts = list(B.shared_recv.view(self.world, -1).unbind(0))
                dist.all_gather(parts, B.shared_send, group=g)
                B.shared_recv.copy_(torch.stack(parts).reshape(-1))
        m_recv = all_to_all_v(B.m_send, L["m_send"], L["m_recv"], ncd, g)
        pl.let_finish(B.shared_recv, m_recv, B.phi_send, B.grad_send)
        phi_recv = all_to_all_v(B.phi_send, L["phi_send"], L["phi_recv"], 1, g)
        grad_recv = all_to_all_v(B.grad_send, L["phi_send"], L["phi_recv"], 3, g) if grad else None
        n_local = self.counts[self.rank]
        phi = torch.empty(n_local, dtype=torch.float64, device=q_local.device)
        gl = torch.empty(n_local, 3, dtype=torch.float64, device=q_local.device) if grad else None
        pl.let_unpack(phi_recv, grad_recv, phi, gl)
        return (phi, gl) if grad else phi

    def stats(self) -> dict:
        return self.plan.stats()


def _a2a_local(sends: list[torch.Tensor], send_counts: list[list[int]], width: int) -> list[torch.Tensor]:
    """all-to-all-v among in-process 'ranks': recv[d] = concat_r slice of send[r] destined to d."""
    world = len(sends)
    offs = [[0] * (world + 1) for _ in range(world)]
    for r in range(world):
        for d in range(world):
            offs[r][d + 1] = offs[r][d] + send_counts[r][d] * width
    return [torch.cat([sends[r][offs[r][d]:offs[r][d + 1]] for r in range(world)]) for d in range(world)]


def let_matvec_local(plans: list, q_slices: list[torch.Tensor], grad: bool = False):
    """The LET protocol for several plans (ranks 0..world-1 of one world) in ONE process: the
    collectives become buffer copies. Returns each rank's slice of phi (and grad)."""
    world = len(plans)
    Ls = [pl.let for pl in plans]
    ncd = Ls[0]["ncd"]
    Bs = [LetBuffers(pl, grad) for pl in plans]
    for pl, B, q in zip(plans, Bs, q_slices):
        pl.let_pack_q(q, B.q_send)
    q_recv = _a2a_local([B.q_send for B in Bs], [L["q_send"] for L in Ls], 1)
    for pl, B, qr in zip(plans, Bs, q_recv):
        pl.let_upward(qr, B.shared_send, B.m_send)
    shared_all = torch.cat([B.shared_send for B in Bs])
    m_recv = _a2a_local([B.m_send for B in Bs], [L["m_send"] for L in Ls], ncd)
    for pl, B, mr in zip(plans, Bs, m_recv):
        pl.let_finish(shared_all, mr, B.phi_send, B.grad_send)
    phi_recv = _a2a_local([B.phi_send for B in Bs], [L["phi_send"] for L in Ls], 1)
    grad_recv = _a2a_local([B.grad_send for B in Bs], [L["phi_send"] for L in Ls], 3) if grad else [None] * world
    out = []
    for pl, L, pr, gr, q in zip(plans, Ls, phi_recv, grad_recv, q_slices):
        phi = torch.empty(q.shape[0], dtype=torch.float64, device=q.device)
        gl = torch.empty(q.shape[0], 3, dtype=torch.float64, device=q.device) if grad else None
        pl.let_unpack(pr, gr, phi, gl)
        out.append((phi, gl) if grad else phi)
    return out
