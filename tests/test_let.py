"""Multi-GPU LET exchange (paper_1602_02244_b200/csrc/let.cu, dist.py).

CPU (no GPU): the host list builder (fmm_let_lists_host, the code fmm_let_setup
runs) against a brute-force model of what every rank owns, needs and sends, on
trees from the oracle (bit-identical to the GPU's, tests/test_gpu_parity.py);
and the whole protocol over real gloo collectives (world 2 and 3) with a test
double of the plan whose arithmetic is a checksum FMM (monopole "multipoles",
exact near field) computed in numpy from exactly the data the exchange
delivered, compared with the same checksum computed globally.
GPU: the real kernels, several ranks emulated in one process
(dist.let_matvec_local), against the single-GPU mat-vec and the oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import fmm_inputs as F
from oracle import oracle as O
from paper_1602_02244_b200 import _native as N
from paper_1602_02244_b200.fmm import let_lists_host


class Tree:
    """Oracle tree + lists in the form the LET host code takes."""

    def __init__(self, x, p, ncrit, theta):
        self.p = p
        orc = O.Plan(x, p, ncrit, theta)
        c = orc.cells()
        self.n = x.shape[0]
        self.cbeg, self.cend = c["begin"].astype(np.int32), c["end"].astype(np.int32)
        self.nchild = c["nchild"]
        lv = np.nonzero(self.nchild == 0)[0]
        self.leaves = lv[np.argsort(self.cbeg[lv], kind="stable")].astype(np.int32)
        self.p2p, self.m2l = orc.lists()
        _, perm = orc.keys()
        self.perm = perm.astype(np.uint32)

    def lists(self, world, me, caller_off, what):
        return let_lists_host(self.n, world, me, caller_off, self.perm, self.cbeg, self.cend, self.leaves,
                              self.p2p, self.m2l, what, p=self.p)


def caller_offsets(n, counts):
    return np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)


CASES = [("plummer", 3000, 4, 16, 0.5, (1000, 1000, 1000)), ("cube", 4000, 3, 32, 0.4, (4000 - 1234, 1234)),
         ("sphere", 2500, 3, 20, 0.4, (0, 2500, 0, 0)), ("plummer", 1500, 2, 7, 0.3, (300, 700, 500))]


@pytest.mark.parametrize("dist_name,n,p,ncrit,theta,counts", CASES)
def test_let_lists_match_brute_force(dist_name, n, p, ncrit, theta, counts):
    x, _ = F.make(dist_name, n)
    T = Tree(x, p, ncrit, theta)
    W = len(counts)
    co = caller_offsets(n, counts)
    B = T.lists(W, 0, co, N.FMM_LET_RANK_BEGIN)
    # owner ranges: cover [0, n), cut at leaf boundaries, nondecreasing
    assert B[0] == 0 and B[-1] == n and (np.diff(B) >= 0).all()
    leaf_starts = set(T.cbeg[T.leaves].tolist()) | {n}
    assert all(b in leaf_starts for b in B)
    owner = np.searchsorted(B, np.arange(n), side="right") - 1
    caller = np.searchsorted(co, T.perm.astype(np.int64), side="right") - 1
    # brute force: what each rank needs
    need_pos = []
    for d in range(W):
        s = set(range(B[d], B[d + 1]))
        for t, src in T.p2p:
            if owner[T.cbeg[t]] == d and owner[T.cbeg[src]] != d:
                s |= set(range(T.cbeg[src], T.cend[src]))
        need_pos.append(np.array(sorted(s), dtype=np.int64))
    shared = np.array([c for c in range(len(T.cbeg)) if T.cend[c] > T.cbeg[c]
                       and owner[T.cbeg[c]] != owner[T.cend[c] - 1]], dtype=np.int64)
    need_m = [set() for _ in range(W)]
    sh = set(shared.tolist())
    for t, s in T.m2l:
        if s in sh:
            continue
        for d in range(owner[T.cbeg[t]], owner[T.cend[t] - 1] + 1):
            if owner[T.cbeg[s]] != d:
                need_m[d].add(int(s))
    L = {me: {w: T.lists(W, me, co, w) for w in range(N.FMM_LET_PHI_RECV_ROWS + 1) if w != N.FMM_LET_SHARED}
         for me in range(W)}
    for me in range(W):
        assert np.array_equal(L[me][N.FMM_LET_SHARED_CELLS], shared)
        # charges: what me receives from r = needed positions whose caller is r, ascending
        rc = L[me][N.FMM_LET_Q_RECV]
        pos = L[me][N.FMM_LET_Q_RECV_POS]
        off = np.concatenate([[0], np.cumsum(rc)])
        for r in range(W):
            exp = need_pos[me][caller[need_pos[me]] == r]
            assert np.array_equal(pos[off[r]:off[r + 1]], exp)
            # ... and r sends exactly those rows, in that order
            sc = L[r][N.FMM_LET_Q_SEND]
            soff = np.concatenate([[0], np.cumsum(sc)])
            rows = L[r][N.FMM_LET_Q_SEND_ROWS][soff[me]:soff[me + 1]]
            assert np.array_equal(rows + co[r], T.perm[exp].astype(np.int64))
        # boundary multipoles: from owner r, ascending cell order; r's send list matches
        mc = L[me][N.FMM_LET_M_RECV]
        moff = np.concatenate([[0], np.cumsum(mc)])
        cells = L[me][N.FMM_LET_M_RECV_CELLS]
        for r in range(W):
            exp = sorted(c for c in need_m[me] if owner[T.cbeg[c]] == r)
            assert cells[moff[r]:moff[r + 1]].tolist() == exp
            sc = L[r][N.FMM_LET_M_SEND]
            soff = np.concatenate([[0], np.cumsum(sc)])
            assert L[r][N.FMM_LET_M_SEND_CELLS][soff[me]:soff[me + 1]].tolist() == exp
        # results: owner d sends its owned positions whose caller is me; me writes rows perm - co[me]
        pr = L[me][N.FMM_LET_PHI_RECV]
        poff = np.concatenate([[0], np.cumsum(pr)])
        rows = L[me][N.FMM_LET_PHI_RECV_ROWS]
        for d in range(W):
            own = np.arange(B[d], B[d + 1])
            exp = own[caller[own] == me]
            assert np.array_equal(rows[poff[d]:poff[d + 1]], T.perm[exp].astype(np.int64) - co[me])
            sc = L[d][N.FMM_LET_PHI_SEND]
            soff = np.concatenate([[0], np.cumsum(sc)])
            assert np.array_equal(L[d][N.FMM_LET_PHI_SEND_IDX][soff[me]:soff[me + 1]], exp - B[d])


# ------------------------------------------------------------ protocol over gloo
class ChecksumPlan:
    """Test double of Plan for the LET protocol: the same buffers and lists (real host
    code), but a checksum 'FMM' in numpy: M[c] = sum of q over the cell (partial on
    straddling cells), phi_i = sum over the near-field sources of its leaf + sum of M over
    the M2L sources of its leaf and of every ancestor. Only exchanged data is used."""

    def __init__(self, xyz, p, ncrit, theta, rank=0, world=1):
        self.T = Tree(xyz.numpy(), p, ncrit, theta)
        self.rank, self.world, self.p = rank, world, p
        self.device = torch.device("cpu")
        nc = len(self.T.cbeg)
        self.parent = np.full(nc, -1)
        for c in range(nc):  # children are a contiguous block after child_first in the oracle too
            pass
        cbeg, cend = self.T.cbeg, self.T.cend
        order = np.lexsort((-(cend - cbeg), cbeg))
        stack = []
        for c in order:  # parent = smallest enclosing cell (cells nest)
            while stack and not (cbeg[stack[-1]] <= cbeg[c] and cend[c] <= cend[stack[-1]] and stack[-1] != c):
                stack.pop()
            self.parent[c] = stack[-1] if stack else -1
            stack.append(c)

    def let_setup(self, counts):
        T, W, me = self.T, self.world, self.rank
        co = caller_offsets(T.n, counts)
        g = lambda w: T.lists(W, me, co, w)  # noqa: E731
        self.L = {w: g(w) for w in range(N.FMM_LET_PHI_RECV_ROWS + 1) if w != N.FMM_LET_SHARED}
        self.B = self.L[N.FMM_LET_RANK_BEGIN]
        self.let = dict(q_send=list(self.L[N.FMM_LET_Q_SEND]), q_recv=list(self.L[N.FMM_LET_Q_RECV]),
                        m_send=list(self.L[N.FMM_LET_M_SEND]), m_recv=list(self.L[N.FMM_LET_M_RECV]),
                        phi_send=list(self.L[N.FMM_LET_PHI_SEND]), phi_recv=list(self.L[N.FMM_LET_PHI_RECV]),
                        shared=len(self.L[N.FMM_LET_SHARED_CELLS]), rank_begin=list(self.B), ncd=2)
        return self.let

    def let_pack_q(self, q_local, q_send):
        q_send.copy_(q_local[torch.from_numpy(self.L[N.FMM_LET_Q_SEND_ROWS])])

    def let_upward(self, q_recv, shared_send, m_send):
        T = self.T
        self.q = np.full(T.n, np.nan)
        self.q[self.L[N.FMM_LET_Q_RECV_POS]] = q_recv.numpy()
        lo, hi = self.B[self.rank], self.B[self.rank + 1]
        qq = np.nan_to_num(self.q)
        cs = np.concatenate([[0], np.cumsum(np.where((np.arange(T.n) >= lo) & (np.arange(T.n) < hi), qq, 0.0))])
        self.M = cs[np.clip(T.cend, lo, hi)] - cs[np.clip(T.cbeg, lo, hi)]  # own part of every cell
        self.M[np.clip(T.cend, lo, hi) <= np.clip(T.cbeg, lo, hi)] = 0.0
        sh = self.L[N.FMM_LET_SHARED_CELLS]
        shared_send.view(-1, 2)[:, 0] = torch.from_numpy(self.M[sh])
        shared_send.view(-1, 2)[:, 1] = 0.0
        ms = self.L[N.FMM_LET_M_SEND_CELLS]
        m_send.view(-1, 2)[:, 0] = torch.from_numpy(self.M[ms])
        m_send.view(-1, 2)[:, 1] = 0.0

    def let_finish(self, shared_recv, m_recv, phi_send, grad_send=None):
        T = self.T
        sh = self.L[N.FMM_LET_SHARED_CELLS]
        M = np.full(len(T.cbeg), np.nan)
        lo, hi = self.B[self.rank], self.B[self.rank + 1]
        inside = (T.cbeg >= lo) & (T.cend <= hi)
        M[inside] = self.M[inside]
        if len(sh):
            M[sh] = shared_recv.view(self.world, len(sh), 2)[:, :, 0].sum(0).numpy()
        M[self.L[N.FMM_LET_M_RECV_CELLS]] = m_recv.view(-1, 2)[:, 0].numpy()
        m2l_of = {}
        for t, s in T.m2l:
            m2l_of.setdefault(int(t), []).append(int(s))
        p2p_of = {}
        for t, s in T.p2p:
            p2p_of.setdefault(int(t), []).append(int(s))
        phi = np.zeros(hi - lo)
        for leaf in T.leaves:
            if not (lo <= T.cbeg[leaf] < hi):
                continue
            far, c = 0.0, leaf
            while c >= 0:
                far += sum(M[s] for s in m2l_of.get(int(c), []))
                c = self.parent[c]
            near = sum(self.q[T.cbeg[s]:T.cend[s]].sum() for s in p2p_of.get(int(leaf), []))
            phi[T.cbeg[leaf] - lo:T.cend[leaf] - lo] = far + near
        assert np.isfinite(phi).all(), "the exchange did not deliver every needed value"
        phi_send.copy_(torch.from_numpy(phi[self.L[N.FMM_LET_PHI_SEND_IDX]]))

    def let_unpack(self, phi_recv, grad_recv, phi_local, grad_local=None):
        phi_local[torch.from_numpy(self.L[N.FMM_LET_PHI_RECV_ROWS])] = phi_recv

    def checksum_global(self, q_input):
        """Same checksum with all data on one rank (input order)."""
        T = self.T
        q = np.asarray(q_input)[T.perm]
        cs = np.concatenate([[0], np.cumsum(q)])
        M = cs[T.cend] - cs[T.cbeg]
        m2l_of, p2p_of = {}, {}
        for t, s in T.m2l:
            m2l_of.setdefault(int(t), []).append(int(s))
        for t, s in T.p2p:
            p2p_of.setdefault(int(t), []).append(int(s))
        phi = np.zeros(T.n)
        for leaf in T.leaves:
            far, c = 0.0, leaf
            while c >= 0:
                far += sum(M[s] for s in m2l_of.get(int(c), []))
                c = self.parent[c]
            near = sum(q[T.cbeg[s]:T.cend[s]].sum() for s in p2p_of.get(int(leaf), []))
            phi[T.cbeg[leaf]:T.cend[leaf]] = far + near
        out = np.empty(T.n)
        out[T.perm] = phi
        return out


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1602_02244_b200.dist import DistributedPlan

        name, n, p, ncrit, theta, counts = case
        x, q = F.make(name, n)
        co = caller_offsets(n, counts)
        lo, hi = co[rank], co[rank + 1]
        plan = DistributedPlan(torch.from_numpy(x[lo:hi].copy()), p, ncrit, theta, plan_factory=ChecksumPlan)
        phi = plan.matvec(torch.from_numpy(q[lo:hi].copy()))
        out[rank] = phi.numpy().copy()
        if rank == 0:
            out["ref"] = plan.plan.checksum_global(q)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [CASES[0], CASES[1], CASES[3]])
def test_let_protocol_over_gloo(case):
    world = len(case[-1])
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True)
    got = np.concatenate([out[r] for r in range(world)])
    np.testing.assert_allclose(got, out["ref"], rtol=1e-12, atol=1e-9)


# ------------------------------------------------------------ GPU: real kernels
@pytest.mark.gpu
@pytest.mark.parametrize("dist_name,n,p,ncrit,theta,counts,grad", [
    ("plummer", 30000, 8, 64, 0.5, (10000, 10000, 10000), True),
    ("cube", 20000, 10, 64, 0.4, (7000, 13000), False),
    ("sphere", 20000, 12, 128, 0.4, (5000, 5000, 5000, 5000), False),
    ("plummer", 8000, 4, 16, 0.4, (0, 8000), True),
])
def test_let_matvec_matches_single_gpu_and_oracle(dist_name, n, p, ncrit, theta, counts, grad):
    from paper_1602_02244_b200 import Plan
    from paper_1602_02244_b200.dist import let_matvec_local

    x, q = F.make(dist_name, n)
    dev = torch.device("cuda:0")
    xd = torch.from_numpy(x).to(dev)
    qd = torch.from_numpy(q).to(dev)
    W = len(counts)
    co = caller_offsets(n, counts)
    plans = [Plan(xd, p, ncrit, theta, rank=r, world=W) for r in range(W)]
    for pl in plans:
        pl.let_setup(list(counts))
    # potentials: each rank evaluates the pairs of its own leaves once (mutual) and its halo pairs
    # directed (csrc/near_mutual.cu); gradients take the directed near field
    assert all(pl.stats()["near_mutual"] == 1 for pl in plans)
    res = let_matvec_local(plans, [qd[co[r]:co[r + 1]] for r in range(W)], grad=grad)
    single = Plan(xd, p, ncrit, theta).matvec(qd, grad=grad)
    torch.cuda.synchronize()
    for pl in plans:
        pl.sync()
    phi = torch.cat([r[0] if grad else r for r in res]).cpu().numpy()
    ref = (single[0] if grad else single).cpu().numpy()
    assert O.rel_l2(phi, ref) <= 1e-13  # same lists; only summation order of straddling cells differs
    po = O.fmm(x, q, p, ncrit, theta, grad=grad, nthreads=O.default_threads())
    po = po[0] if grad else po
    assert O.rel_l2(phi, po) <= 1e-11
    if grad:
        g = torch.cat([r[1] for r in res]).cpu().numpy()
        assert O.rel_l2(g, single[1].cpu().numpy()) <= 1e-13


# ------------------------------------------------------------ owner cuts
def test_owner_cuts_balance_the_work():
    """Cost-weighted cuts (let.cu let_cuts): on a Plummer tree, the work each
    rank's targets carry — 11 flop per P2P interaction of its leaves plus the M2L pairs of the
    cells overlapping its range — is within 25 % of the mean for 4 ranks, where equal particle
    counts are not (the dense core has more interactions per particle)."""
    x, _ = F.make("plummer", 40000)
    T = Tree(x, 6, 32, 0.5)
    W = 4
    co = caller_offsets(T.n, (T.n // W,) * (W - 1) + (T.n - (W - 1) * (T.n // W),))
    B = T.lists(W, 0, co, N.FMM_LET_RANK_BEGIN)
    m2l_cost = 6.0 * 7**3

    def work(B):
        w = np.zeros(W)
        own = lambda s: np.searchsorted(B, s, side="right") - 1  # noqa: E731
        sz = (T.cend - T.cbeg).astype(np.float64)
        for t, s in T.p2p:
            w[own(T.cbeg[t])] += 11.0 * sz[t] * sz[s]
        for t, _s in T.m2l:
            for r in range(own(T.cbeg[t]), own(T.cend[t] - 1) + 1):
                w[r] += m2l_cost
        return w

    wb = work(np.asarray(B))
    assert wb.max() / wb.mean() <= 1.25, wb
    counts = np.asarray([0] + [np.searchsorted(T.cbeg[T.leaves], r * T.n // W) for r in range(1, W)] + [len(T.leaves)])
    Bc = np.array([T.cbeg[T.leaves][i] if i < len(T.leaves) else T.n for i in counts])
    wc = work(Bc)
    assert wb.max() / wb.mean() < wc.max() / wc.mean()


# ------------------------------------------------------------ GPU: collective mode (NCCL inside libfmm)
@pytest.mark.gpu
@pytest.mark.parametrize("dist_name,n,p,ncrit,theta,grad", [
    ("plummer", 30000, 8, 64, 0.5, True), ("cube", 20000, 10, 64, 0.4, False), ("sphere", 20000, 12, 128, 0.4, False),
    ("plummer", 8000, 3, 16, 0.4, True)])
def test_collective_mode_one_rank(dist_name, n, p, ncrit, theta, grad):
    """fmm_exec.nccl_id (include/fmm.h): the collective setup (NCCL all-gather of counts and points,
    cost-weighted partition, exchange lists and buffers) and the collective mat-vec (charges, shared
    and boundary multipoles, results moved by NCCL on the plan's stream, rank-local M2M / M2L / L2L)
    on a one-rank communicator — every step of the multi-GPU path but the peer transfers — match the
    single-GPU plan and the oracle."""
    from paper_1602_02244_b200 import Plan
    from paper_1602_02244_b200.fmm import nccl_unique_id

    x, q = F.make(dist_name, n)
    dev = torch.device("cuda:0")
    xd, qd = torch.from_numpy(x).to(dev), torch.from_numpy(q).to(dev)
    uid = nccl_unique_id()
    assert len(uid) == 128
    pl = Plan(xd, p, ncrit, theta, rank=0, world=1, nccl_id=uid)
    out = pl.matvec(qd, grad=grad)
    single = Plan(xd, p, ncrit, theta).matvec(qd, grad=grad)
    torch.cuda.synchronize()
    pl.sync()
    phi = (out[0] if grad else out).cpu().numpy()
    ref = (single[0] if grad else single).cpu().numpy()
    assert O.rel_l2(phi, ref) <= 1e-14
    if grad:
        assert O.rel_l2(out[1].cpu().numpy(), single[1].cpu().numpy()) <= 1e-14
    po = O.fmm(x, q, p, ncrit, theta, nthreads=O.default_threads())
    assert O.rel_l2(phi, po) <= 1e-11
    st = pl.stats()
    assert st["own_begin"] == 0 and st["own_end"] == n and st["bytes_by"]["let"] > 0
    ph = pl.matvec_host(q)  # the end-to-end entry point in collective mode
    assert O.rel_l2(ph.numpy(), phi) <= 1e-15
