"""NEXT-1: the M2L formulations along the paper's analytic <-> algebraic axis
(Fig 1), measured on one B200: matrix-free O(p^4) per pair (v1), precomputed
dense translation-invariant class operators on DMMA (v2), and the same
operators rotation-factored (v3). Per variant: M2L stage time (CUDA events,
median of the timed mat-vecs), useful flops per pair, and the plan's device bytes by category
(fmm_stats bytes_by: the FMM side of Fig 4). Prints a markdown table.

    python tools/m2l_sweep.py [--configs c2 c3] [--steps 5]
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import fmm_inputs as F  # noqa: E402


def run(name, variant, steps):
    os.environ["FMM_M2L_VARIANT"] = str(variant)
    from paper_1602_02244_b200 import Plan

    cfg = F.CONFIGS[name]
    x, q = F.make_config(name)
    dev = torch.device("cuda:0")
    pl = Plan(torch.from_numpy(x).to(dev), cfg.p, cfg.ncrit, cfg.theta)
    qd = torch.from_numpy(q).to(dev)
    pl.set_timing(True)
    m2l, tot = [], []
    for i in range(steps + 2):
        pl.matvec(qd, grad=cfg.grad)
        torch.cuda.synchronize()
        st = pl.stats()
        if i >= 2:
            m2l.append(st["t_matvec_ms"][1])
            tot.append(st["t_matvec_ms"][4])
    st = pl.stats()
    out = dict(config=name, variant=st["m2l_variant"], m2l_ms=statistics.median(m2l), matvec_ms=statistics.median(tot),
               pairs=st["n_m2l_pairs"], flops_pair=st["m2l_flops_per_pair"], bytes=st["bytes_device"], by=st["bytes_by"])
    del pl
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["c2", "c3"])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--variants", nargs="+", type=int, default=[1, 2, 3])
    args = ap.parse_args()
    rows = [run(c, v, args.steps) for c in args.configs for v in args.variants]
    print("| config | M2L | M2L ms | mat-vec ms | useful flop/pair | useful TFLOP/s | operators MB | schedule MB | "
          "expansions MB | lists MB | plan MB |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        mb = lambda k: r["by"][k] / 1e6  # noqa: E731
        tf = r["pairs"] * r["flops_pair"] / (r["m2l_ms"] * 1e-3) / 1e12
        print(f"| {r['config']} | v{r['variant']} | {r['m2l_ms']:.3f} | {r['matvec_ms']:.3f} | {r['flops_pair']:.0f} | "
              f"{tf:.2f} | {mb('operators'):.1f} | {mb('schedule'):.1f} | {mb('expansions'):.1f} | {mb('lists'):.1f} | "
              f"{r['bytes'] / 1e6:.1f} |")


if __name__ == "__main__":
    main()
