"""Projected multi-GPU load balance of the LET mat-vec on ONE GPU.

    python tools/let_scaling.py [config] [world ...]       (default: c4 with 2 4 8 ranks)

Builds `world` plans of the same global problem (legacy multi-GPU mode: every rank's plan holds
the global tree, its own cost-weighted Morton range and the exchange lists), runs the whole LET
protocol in one process (dist.let_matvec_local: the collectives become buffer copies), then times
every rank's own work — upward pass of its range, M2L of its targets, L2L, near field — with CUDA
events, one rank after another. Prints (single-GPU mat-vec / world) / max over ranks: the parallel
efficiency the partition allows before any communication cost (the exchange volumes are MB per
mat-vec). Not a multi-GPU measurement.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import fmm_inputs as F  # noqa: E402
from paper_1602_02244_b200 import Plan  # noqa: E402
from paper_1602_02244_b200.dist import LetBuffers, let_matvec_local  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def main():
    args = [a for a in sys.argv[1:]]
    name = args[0] if args and not args[0].isdigit() else "c4"
    worlds = [int(a) for a in args if a.isdigit()] or [2, 4, 8]
    cfg = F.CONFIGS[name]
    x, q = F.make_config(name)
    dev = torch.device("cuda:0")
    xd, qd = torch.from_numpy(x).to(dev), torch.from_numpy(q).to(dev)
    single = Plan(xd, cfg.p, cfg.ncrit, cfg.theta)
    for _ in range(2):
        single.matvec(qd)
    torch.cuda.synchronize()
    t = []
    for _ in range(5):
        a, b = ev(), ev()
        a.record()
        single.matvec(qd)
        b.record()
        b.synchronize()
        t.append(a.elapsed_time(b))
    t1 = float(np.median(t))
    print(f"{name}: single-GPU mat-vec {t1:.2f} ms", flush=True)
    del single
    for W in worlds:
        counts = [(r + 1) * cfg.n // W - r * cfg.n // W for r in range(W)]
        co = np.concatenate([[0], np.cumsum(counts)])
        plans = [Plan(xd, cfg.p, cfg.ncrit, cfg.theta, rank=r, world=W) for r in range(W)]
        for pl in plans:
            pl.let_setup(counts)
        qs = [qd[co[r]:co[r + 1]] for r in range(W)]
        let_matvec_local(plans, qs)  # warm-up: every rank's buffers filled by a real exchange
        torch.cuda.synchronize()
        Bs = [LetBuffers(pl, False) for pl in plans]
        # every rank's received data once more (buffers), then its own steps timed alone
        per = []
        q_recv, shared_all, m_recv = exchange_inputs(plans, Bs, qs)
        for r, (pl, B) in enumerate(zip(plans, Bs)):
            ts = []
            for _ in range(3):
                a, m, b = ev(), ev(), ev()
                a.record()
                pl.let_upward(q_recv[r], B.shared_send, B.m_send)
                m.record()
                pl.let_finish(shared_all, m_recv[r], B.phi_send, None)
                b.record()
                b.synchronize()
                ts.append((a.elapsed_time(m), m.elapsed_time(b)))
            up, fin = np.median(np.array(ts), axis=0)
            st = pl.stats()
            per.append(up + fin)
            print(f"  W={W} rank {r}: range [{st['own_begin']}, {st['own_end']}) upward {up:.2f} ms, "
                  f"M2L+L2L+near {fin:.2f} ms, total {up + fin:.2f} ms", flush=True)
        eff = (t1 / W) / max(per)
        print(f"W={W}: max rank {max(per):.2f} ms, mean {np.mean(per):.2f} ms, single/W {t1 / W:.2f} ms -> "
              f"projected efficiency {eff:.3f} (imbalance max/mean {max(per) / np.mean(per):.3f})", flush=True)
        del plans, Bs
        torch.cuda.empty_cache()


def exchange_inputs(plans, Bs, qs):
    """The received buffers of every rank (one in-process exchange), kept for the timed steps."""
    from paper_1602_02244_b200.dist import _a2a_local

    Ls = [pl.let for pl in plans]
    ncd = Ls[0]["ncd"]
    for pl, B, q in zip(plans, Bs, qs):
        pl.let_pack_q(q, B.q_send)
    q_recv = _a2a_local([B.q_send for B in Bs], [L["q_send"] for L in Ls], 1)
    for pl, B, qr in zip(plans, Bs, q_recv):
        pl.let_upward(qr, B.shared_send, B.m_send)
    shared_all = torch.cat([B.shared_send for B in Bs])
    m_recv = _a2a_local([B.m_send for B in Bs], [L["m_send"] for L in Ls], ncd)
    torch.cuda.synchronize()
    return q_recv, shared_all, m_recv


if __name__ == "__main__":
    main()
