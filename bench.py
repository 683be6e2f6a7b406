#!/usr/bin/env python
"""bench.py — FMM mat-vec throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

One "step" = one ``fmm_matvec`` (the application phase) over
the configuration's synthetic point set with inputs resident in HBM: charge
gather, P2M, M2M, M2L, L2L, L2P + P2P, un-permute. Default workload:
BASELINE.json configs[2] (N = 10^6 uniform cube, p = 10, ncrit = 64,
theta = 0.4), see DESIGN.md §6. For N > 1 launch under torchrun (one rank per
GPU, NCCL). Prints ONE JSON line on rank 0.

``--impl reference``: the CPU oracle (oracle/, as it stands) on this host's
cores, each step a bounded target sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import fmm_inputs as F  # noqa: E402

METRIC = "FMM mat-vec particles/sec (Laplace 3D, fp64) at 1/2/4/8 B200; % FP64 peak"
UNIT = "particles/s"
SM_COUNT = 148
FP64_FMA_PER_CLK_PER_SM = 64
SM_MAX_MHZ = 1965.0


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def fp64_nominal_tflops():
    pk = peaks()
    mhz = float(pk.get("sm_max_mhz", SM_MAX_MHZ))
    return SM_COUNT * FP64_FMA_PER_CLK_PER_SM * 2 * mhz * 1e6 / 1e12


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * (max(mx) if mx else SM_MAX_MHZ)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ fp64 peak
def fp64_probe(torch, seconds=1.0):
    """Measured DFMA rate (TFLOP/s): burst (one ~0.3 s launch) and sustained (back to back for `seconds`)."""
    from paper_1602_02244_b200 import build

    lib = C.CDLL(build.build_tools())
    lib.fp64_probe_launch.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.fp64_probe_flops.argtypes = [C.c_int, C.c_int, C.c_int64]
    lib.fp64_probe_flops.restype = C.c_double
    seed = torch.tensor([0.9999999, 1e-7, 0.5], dtype=torch.float64, device="cuda")
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    blocks, threads = SM_COUNT * 8, 256

    def run(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        rc = lib.fp64_probe_launch(blocks, threads, iters, C.c_void_p(seed.data_ptr()), C.c_void_p(out.data_ptr()),
                                   C.c_void_p(st.cuda_stream))
        e1.record(st)
        e1.synchronize()
        assert rc == 0, rc
        return lib.fp64_probe_flops(blocks, threads, iters) / (e0.elapsed_time(e1) * 1e-3) / 1e12

    run(1000)
    iters = 20000
    burst = max(run(iters) for _ in range(3))
    t_end = time.time() + seconds
    rates = []
    while time.time() < t_end:
        rates.append(run(iters))
    return {"burst_tflops": burst, "sustained_tflops": statistics.median(rates)}


# ------------------------------------------------------------------ cpu oracle
def morton_segments(pl, n, k, segments=8):
    """k targets as `segments` contiguous Morton-order runs spread over the domain: whole
    leaves, so their M2L / L2L work is shared as in a full mat-vec (a uniform random
    sample would pay one leaf's far field per target)."""
    _, perm = pl.keys()
    seg = max(1, k // segments)
    starts = np.linspace(0, max(0, n - seg), segments).astype(np.int64)
    return np.unique(np.concatenate([perm[s:s + seg] for s in starts]))


def oracle_full(x, q, cfg, nthreads):
    """One complete oracle mat-vec (setup excluded, as for the GPU arm)."""
    from oracle import oracle as O

    pl = O.Plan(x, cfg.p, cfg.ncrit, cfg.theta)
    t0 = time.perf_counter()
    pl.eval(q, nthreads=nthreads, grad=cfg.grad)
    t = time.perf_counter() - t0
    return {"value": cfg.n / t, "t_s": t}


def oracle_rate(x, q, cfg, k, nthreads, reps=1, segments=4):
    """Oracle (as it stands) on a bounded sample: setup once, then sampled-target
    evaluations with 1 and k targets (k in 8 contiguous Morton runs); the full
    mat-vec time is extrapolated as t(1) + (N - 1) * (t(k) - t(1)) / (k - 1)
    (upward pass + per-target work)."""
    from oracle import oracle as O

    t0 = time.perf_counter()
    pl = O.Plan(x, cfg.p, cfg.ncrit, cfg.theta)
    t_setup = time.perf_counter() - t0
    T = morton_segments(pl, cfg.n, k, segments)
    k = len(T)
    t0 = time.perf_counter()
    pl.eval(q, targets=T[:1], nthreads=nthreads, grad=cfg.grad)
    t1 = time.perf_counter() - t0
    tks = []
    for _ in range(reps):
        t0 = time.perf_counter()
        pl.eval(q, targets=T, nthreads=nthreads, grad=cfg.grad)
        tks.append(time.perf_counter() - t0)
    per_target = max(min(tks) - t1, 1e-12) / max(k - 1, 1)
    t_full = t1 + (cfg.n - 1) * per_target
    return {"value": cfg.n / t_full, "t_setup_s": t_setup, "t_sample_s": min(tks), "t_one_s": t1, "k": k,
            "t_full_est_s": t_full, "steps_s": tks}


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ------------------------------------------------------------------- reference arm
def run_reference(args, cfg, rank):
    if rank != 0:
        return  # rank 0 alone runs the CPU oracle
    cores = cpu_cores()
    x, q = F.make_config(cfg.name)
    k = args.ref_targets
    times = []
    res = oracle_rate(x, q, cfg, k, cores, reps=1)  # warm / calibrate
    for _ in range(max(0, args.warmup - 1)):
        oracle_rate(x, q, cfg, k, cores, reps=1)
    res = oracle_rate(x, q, cfg, k, cores, reps=args.steps)
    times = res["steps_s"]
    sample = (f"oracle sampled-target mode: full tree + upward pass, then {res['k']} targets in 4 contiguous "
              f"Morton runs of N={cfg.n}; full mat-vec time extrapolated t1 + (N-1)(tk - t1)/(k-1)")
    line = {
        "impl": "reference", "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * res["t_full_est_s"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(cfg, args.gpus),
        "cpu_baseline": {"value": res["value"], "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "sample_step_s": times,
    }
    print(json.dumps(line), flush=True)


def config_dict(cfg, n_gpus):
    src = f"BASELINE configs[{cfg.index}]" if cfg.index >= 0 else "NEXT-3 paper §4.1 geometry (not a BASELINE config)"
    return {"workload": f"{src}: N={cfg.n} {cfg.dist}, p={cfg.p}, ncrit={cfg.ncrit}, "
                        f"theta={cfg.theta}" + (", with gradients" if cfg.grad else ""),
            "n": cfg.n, "p": cfg.p, "ncrit": cfg.ncrit, "theta": cfg.theta, "grad": cfg.grad,
            "distribution": cfg.dist, "parallelism": f"morton-target-partition x{n_gpus}" if n_gpus > 1 else "1 GPU",
            "l2": "flushed between timed steps (256 MiB write)"}


def run_dry(args, world, rank):
    """The multi-rank launch / timing plumbing with no FMM and no GPU (gloo): every rank
    checks the world, times `--steps` empty steps between barriers, and the max over ranks is
    printed by rank 0 — what the real arm does around fmm_matvec."""
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.init_process_group("gloo")
    t = []
    for _ in range(args.warmup + args.steps):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        t.append(time.perf_counter() - t0)
    tot = torch.tensor([sum(t[args.warmup:])], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks_seen": world, "steps": args.steps,
                          "warmup": args.warmup, "max_over_ranks_s": tot.item()}), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(F.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--grad", action="store_true", help="also return gradients (default: the config's)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-targets", type=int, default=100000)
    ap.add_argument("--cpu-full-max-n", type=int, default=2_000_000)
    ap.add_argument("--ref-targets", type=int, default=100000)
    ap.add_argument("--no-probe", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="launcher / timing plumbing only (no GPU, gloo)")
    args = ap.parse_args()
    cfg = F.CONFIGS[args.config]
    if args.grad:
        cfg = F.Config(**{**cfg.__dict__, "grad": True})
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torchrun (127.0.0.1 rendezvous)
        import socket

        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (launch one rank per GPU)")
    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return
    if args.dry_run:  # launcher check without a GPU (tests/test_bench_launch.py)
        run_dry(args, world, rank)
        return

    import torch
    import torch.distributed as dist

    from paper_1602_02244_b200 import Plan, build
    from paper_1602_02244_b200.dist import DistributedPlan

    build.build()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    assert args.warmup >= 3, "timing rules: at least 3 warm-up steps"

    x, q = F.make_config(cfg.name)
    lo, hi = F.rank_slice(cfg.n, rank, world)
    stream = torch.cuda.current_stream(dev)
    if world > 1:
        plan = DistributedPlan(torch.from_numpy(x[lo:hi]).to(dev), cfg.p, cfg.ncrit, cfg.theta)
        inner = plan.plan
    else:
        plan = Plan(torch.from_numpy(x).to(dev), cfg.p, cfg.ncrit, cfg.theta)
        inner = plan
    q_dev = torch.from_numpy(q[lo:hi]).to(dev)
    st0 = inner.stats()
    # setup (precalculation) timed apart: median of 3 warm plans (1 GPU)
    setup_ms = [st0["t_setup_ms"][3]]
    if world == 1:
        xd = torch.from_numpy(x).to(dev)
        setup_ms = []
        for _ in range(3):
            pl2 = Plan(xd, cfg.p, cfg.ncrit, cfg.theta)
            setup_ms.append(pl2.stats()["t_setup_ms"][3])
            del pl2
        del xd
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step():
        return plan.matvec(q_dev, grad=cfg.grad)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    inner.set_timing(True)
    launches0 = inner.stats()["launches_total"]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    stage = []
    with ClockSampler(local_rank) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            flush.fill_(k & 0xFF)  # evict L2 between timed steps (outside the events)
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
            stage.append(inner.stats()["t_matvec_ms"][:5])  # events of this call (same stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = inner.stats()["launches_total"] - launches0  # this rank's libfmm kernels in the timed region
    inner.set_timing(False)
    ms = [a.elapsed_time(b) for a, b in ev]
    tot = torch.tensor([sum(ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms_per_step = tot.item() / args.steps
    value = cfg.n / (ms_per_step * 1e-3)

    # ---- e2e through the host-buffer ABI entry point (H2D of q, D2H of phi inside the timed region)
    e2e = None
    if world == 1:
        qh = torch.from_numpy(q).pin_memory()
        ph = torch.empty(cfg.n, dtype=torch.float64).pin_memory()
        gh = torch.empty(cfg.n, 3, dtype=torch.float64).pin_memory() if cfg.grad else None
        for _ in range(3):
            plan.matvec_host(qh, grad=cfg.grad, out=(ph, gh))
        t_e2e = []
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            plan.matvec_host(qh, grad=cfg.grad, out=(ph, gh))  # synchronous
            t_e2e.append(time.perf_counter() - t0)
        e2e = {"value": cfg.n / statistics.mean(t_e2e), "unit": UNIT, "h2d_bytes_per_step": 8 * cfg.n,
               "d2h_bytes_per_step": 8 * cfg.n * (4 if cfg.grad else 1), "timing": "host wall clock, synchronous call"}
    else:  # every rank: its pinned host slice of q -> device, DistributedPlan.matvec, its phi slice -> host
        qh = torch.from_numpy(q[lo:hi]).pin_memory()
        ph = torch.empty(hi - lo, dtype=torch.float64).pin_memory()
        gh = torch.empty(hi - lo, 3, dtype=torch.float64).pin_memory() if cfg.grad else None

        def e2e_step():
            qd = qh.to(dev, non_blocking=True)
            out = plan.matvec(qd, grad=cfg.grad)
            phi_d, g_d = out if cfg.grad else (out, None)
            ph.copy_(phi_d, non_blocking=True)
            if g_d is not None:
                gh.copy_(g_d, non_blocking=True)
            torch.cuda.synchronize()

        for _ in range(3):
            e2e_step()
        t_e2e = []
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            e2e_step()
            t_e2e.append(time.perf_counter() - t0)
        tt = torch.tensor([sum(t_e2e)], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": cfg.n / (tt.item() / args.steps), "unit": UNIT, "h2d_bytes_per_step": 8 * cfg.n,
               "d2h_bytes_per_step": 8 * cfg.n * (4 if cfg.grad else 1),
               "timing": "host wall clock per rank (own slices, pinned), max over ranks"}

    # ---- roofline of the dominant kernel: the work the executed formulation does (not a dense
    # equivalent; the paper's point is that the FMM does "only useful Flops")
    st = inner.stats()
    m2l_ms = max(1e-6, statistics.mean(s[1] for s in stage))  # stage events of the inner plan
    near_ms = max(1e-6, statistics.mean(s[2] for s in stage))
    up_ms = statistics.mean(s[0] for s in stage)
    down_ms = statistics.mean(s[3] for s in stage)
    p = cfg.p
    nc = (p + 1) * (p + 2) // 2
    own_frac = (st["own_end"] - st["own_begin"]) / cfg.n
    m2l_flops = st["m2l_flops_per_pair"] * st["n_m2l_pairs"] * (own_frac if world > 1 else 1.0)  # executed form
    m2l_dense_flops = 2.0 * (p + 1) ** 4 * st["n_m2l_pairs"] * (own_frac if world > 1 else 1.0)  # SURVEY 8(d) dense
    p2p_inter = (st["n_p2p_interactions"] - cfg.n) * own_frac
    near_flops = (19.0 if cfg.grad else 11.0) * p2p_inter + (3 if cfg.grad else 1) * 8.0 * nc * cfg.n * own_frac
    nominal = fp64_nominal_tflops()
    probe = None
    if not args.no_probe and rank == 0:
        try:
            probe = fp64_probe(torch)
        except Exception as e:  # measurement helper only
            probe = {"error": str(e)}
    if m2l_ms >= near_ms:
        dom, dflops, dms = "m2l", m2l_flops, m2l_ms
    else:
        dom, dflops, dms = "near (P2P+L2P)", near_flops, near_ms
    achieved = dflops / (dms * 1e-3) / 1e12
    traffic = None  # the ncu capture is of the default workload (configs[2]); other configs report null
    try:
        if args.config == "c3":
            with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")) as f:
                traffic = json.load(f).get(dom, {}).get("bytes")
    except (OSError, ValueError):
        pass
    p2p_m2l_tflops = (m2l_flops + near_flops) / ((m2l_ms + near_ms) * 1e-3) / 1e12
    roofline = {"bound": "alu", "kernel": dom, "achieved": achieved, "peak": nominal, "unit": "TFLOP/s",
                "frac": achieved / nominal, "traffic": traffic,
                "traffic_source": "profiles/traffic.json (ncu --set full, DRAM read+write bytes per launch)",
                "peak_source": "derived (no FP64 entry in MEASURED_PEAKS.json): 148 SM x 64 FP64 FMA/clk x 2 x "
                               "sm_max_mhz; measured_fp64_probe is a DFMA microbenchmark beside it (DESIGN.md §6)",
                "measured_fp64_probe": probe,
                "p2p_m2l_frac": p2p_m2l_tflops / nominal,
                "p2p_m2l_tflops": p2p_m2l_tflops,
                "stages_ms": {"upward": up_ms, "m2l": m2l_ms, "downward": down_ms, "near": near_ms},
                "executed_tflops": {"m2l": m2l_flops / (m2l_ms * 1e-3) / 1e12,
                                    "near": near_flops / (near_ms * 1e-3) / 1e12},
                "convention": "executed formulation: M2L fmm_stats.m2l_flops_per_pair (v4: per-pair rotation "
                              "with the fixed operator, 2 x (FMAs of F, F^T, G, G^T, the z-rotations and the "
                              "Hankel translation)); P2P 11 (phi) / 19 (phi+grad) flop per interaction; L2P "
                              "8 (p+1)(p+2)/2 per particle (x3 with grad)",
                "m2l_formulation": {"variant": st["m2l_variant"], "flops_per_pair": st["m2l_flops_per_pair"]},
                "dense_equivalent": {"m2l_flops_per_pair": 2.0 * (p + 1) ** 4,
                                     "m2l_tflops": m2l_dense_flops / (m2l_ms * 1e-3) / 1e12,
                                     "note": "SURVEY 8(d)'s dense-operator count 2(p+1)^4: the method's speed, "
                                             "not the kernel's fraction of peak"}}

    # ---- CPU oracle baseline (rank 0, N = 1 only, bounded sample)
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        cores = cpu_cores()
        if cfg.n <= args.cpu_full_max_n:
            r = oracle_full(x, q, cfg, cores)
            cpu = {"value": r["value"], "unit": UNIT, "cores": cores, "kind": "oracle",
                   "sample": f"one complete oracle mat-vec of the same workload (N={cfg.n}), {r['t_s']:.1f} s, "
                             f"setup excluded"}
        else:
            r = oracle_rate(x, q, cfg, args.cpu_targets, cores)
            cpu = {"value": r["value"], "unit": UNIT, "cores": cores, "kind": "oracle",
                   "sample": f"oracle sampled-target mode, {r['k']} targets in 4 contiguous Morton runs of "
                             f"N={cfg.n}; t(1 target)={r['t_one_s']:.2f}s, t({r['k']})={r['t_sample_s']:.2f}s, "
                             f"full mat-vec extrapolated {r['t_full_est_s']:.1f}s"}


    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(cfg, world), "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "clocks": clk.summary(), "gpu_launches": launches,
        "setup_ms": statistics.median(setup_ms), "setup_ms_all": setup_ms,
        "counts": {k: st[k] for k in ("n_cells", "n_leaves", "n_p2p_pairs", "n_m2l_pairs", "n_p2p_interactions",
                                      "max_level")},
        "ms_per_step_min": min(ms),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
