"""GPU parity: the CUDA path (through the C ABI) against the independent CPU oracle.

Stage gates: keys / permutation / cell arrays bit-exact, P2P and
M2L lists equal as sets, multipoles <= 1e-13 and locals <= 1e-11 relative per
cell, outputs <= 1e-11 relative L2 (north_star tolerance), both at small sizes
spanning many tiles with ragged leaves and at BASELINE.json's full sizes on a
seeded target sample (oracle sampled-target mode).
"""
import os

import numpy as np
import pytest

import fmm_inputs as F
from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-11  # north_star: rel L2 <= 1e-11 in fp64


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    from paper_1602_02244_b200 import build

    build.build()
    return torch


def to_dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def gpu_fmm(torch, x, q, p, ncrit, theta, grad=False):
    from paper_1602_02244_b200 import Plan

    pl = Plan(to_dev(torch, x), p, ncrit, theta)
    out = pl.matvec(to_dev(torch, q), grad=grad)
    torch.cuda.synchronize()
    pl.sync()
    if grad:
        return pl, out[0].cpu().numpy(), out[1].cpu().numpy()
    return pl, out.cpu().numpy(), None


def test_direct_matches_oracle_direct(torch_cuda):
    from paper_1602_02244_b200 import direct

    torch = torch_cuda
    x, q = F.cube(3001, seed=7)
    t, _ = F.plummer(517, seed=2)
    for tgt in (None, t):
        phi, g = direct(to_dev(torch, x), to_dev(torch, q), None if tgt is None else to_dev(torch, tgt), grad=True)
        po, go = O.direct(x, q, tgt=tgt, grad=True)
        assert O.rel_l2(phi.cpu().numpy(), po) < 1e-13
        assert O.rel_l2(g.cpu().numpy(), go) < 1e-13


def test_direct_worked_example(torch_cuda):
    from paper_1602_02244_b200 import direct

    torch = torch_cuda
    x = np.array([[0.0, 0, 0], [1.0, 0, 0]])
    phi, g = direct(to_dev(torch, x), to_dev(torch, np.array([1.0, -2.0])), grad=True)
    assert phi.cpu().tolist() == [-2.0, 1.0]
    assert g.cpu().tolist() == [[-2.0, 0.0, 0.0], [-1.0, 0.0, 0.0]]


CASES = [
    ("cube", 1000, 4, 32, 0.4),      # configs[0]
    ("cube", 20000, 10, 64, 0.4),    # configs[1..2] recipe at a size the oracle finishes in seconds
    ("plummer", 30000, 8, 64, 0.5),  # configs[3] recipe: adaptive, leaves at many levels
    ("sphere", 30000, 12, 128, 0.4), # configs[4] recipe: 2D manifold
    ("plummer", 5000, 3, 7, 0.3),    # ragged: odd ncrit, deep tree
]


@pytest.mark.parametrize("dist,n,p,ncrit,theta", CASES)
def test_tree_and_lists_match_oracle(torch_cuda, dist, n, p, ncrit, theta):
    torch = torch_cuda
    x, q = F.make(dist, n)
    from paper_1602_02244_b200 import Plan

    pl = Plan(to_dev(torch, x), p, ncrit, theta)
    orc = O.Plan(x, p, ncrit, theta)
    keys, perm = orc.keys()
    assert np.array_equal(pl.export("keys"), keys)
    assert np.array_equal(pl.export("perm").astype(np.int64), perm)
    lo, S, scale = orc.geometry()
    assert np.array_equal(pl.export("geom"), np.array([*lo, S, scale]))
    c = orc.cells()
    assert np.array_equal(pl.export("level"), c["level"])
    assert np.array_equal(pl.export("anchor"), c["anchor"])
    assert np.array_equal(pl.export("begin"), c["begin"])
    assert np.array_equal(pl.export("end"), c["end"])
    assert np.array_equal(pl.export("child"), c["child_first"])
    assert np.array_equal(pl.export("nchild"), c["nchild"])
    assert np.array_equal(pl.export("parent"), c["parent"])
    assert np.array_equal(pl.export("center"), c["center"])
    p2p, m2l = orc.lists()
    for mine, ref in ((pl.export("p2p"), p2p), (pl.export("m2l"), m2l)):
        assert mine.shape == ref.shape
        a = mine.astype(np.int64)
        assert np.array_equal(a[np.lexsort((a[:, 1], a[:, 0]))], ref[np.lexsort((ref[:, 1], ref[:, 0]))])
        assert (np.diff(a[:, 0]) >= 0).all()  # grouped by target
    st = pl.stats()
    assert st["n_cells"] == orc.ncells and st["n_p2p_interactions"] == orc.info("p2p_interactions")


@pytest.mark.parametrize("dist,n,p,ncrit,theta", CASES)
def test_expansions_and_outputs_match_oracle(torch_cuda, dist, n, p, ncrit, theta):
    torch = torch_cuda
    x, q = F.make(dist, n)
    pl, phi, g = gpu_fmm(torch, x, q, p, ncrit, theta, grad=True)
    orc = O.Plan(x, p, ncrit, theta)
    po, go = orc.eval(q, grad=True, nthreads=O.default_threads())
    M, L = orc.expansions()
    Mg, Lg = pl.export("M"), pl.export("L")
    nm = np.linalg.norm(M, axis=1)
    nl = np.linalg.norm(L, axis=1)
    assert (np.linalg.norm(Mg - M, axis=1) <= 1e-13 * nm + 1e-300).all()
    # locals: SURVEY §8(c)'s 1e-12 per cell, or — for a cell whose sum cancels (Plummer-core
    # leaves add 100-175 M2L terms) — a condition-aware bound (R13)
    el = np.linalg.norm(Lg - L, axis=1)
    flagged = np.nonzero(el > 1e-12 * nl + 1e-300)[0]
    assert len(flagged) <= max(2, len(nl) // 500)
    if len(flagged):
        check_local_condition_bound(orc, p, M, L, Lg, flagged)
    assert O.rel_l2(phi, po) <= TOL
    assert O.rel_l2(g, go) <= TOL


def check_local_condition_bound(orc, p, M, L, Lg, cells):
    """Condition-aware gate for local expansions (R13). For target cell A, the GPU's
    own rounding error — its difference from the oracle minus the L2L shift of its parent's
    difference (gated at the parent) — must satisfy
        ||dL_A - L2L(dL_parent)|| <= c u (sum_B ||T_AB M_B|| + ||L2L(L_parent)||),
    u = 2^-53, c = 100 (p+1)^2 (the operation depth of one rotation-form pair, generously): the
    terms' magnitudes, not the cancelled sum's, set the attainable accuracy. The terms are the
    oracle's own operators (m2l, l2l) on the oracle's expansions."""
    cc = orc.cells()
    center, parent = cc["center"], cc["parent"]
    _, m2l = orc.lists()
    u = 2.0**-53
    for a in cells:
        srcs = m2l[m2l[:, 0] == a, 1]
        s = sum(np.linalg.norm(O.m2l(M[b], center[b], center[a], p)) for b in srcs)
        d = Lg[a] - L[a]
        par = parent[a]
        if par >= 0:
            s += np.linalg.norm(O.l2l(L[par], center[par], center[a], p))
            d = d - O.l2l(Lg[par] - L[par], center[par], center[a], p)
        assert np.linalg.norm(d) <= 100 * (p + 1) ** 2 * u * s, (a, np.linalg.norm(d), s)


def test_c1_against_direct_and_survey_truncation(torch_cuda):
    """configs[0]: GPU and oracle have the same truncation error vs O(N^2) direct."""
    torch = torch_cuda
    x, q = F.cube(1000)
    _, phi, g = gpu_fmm(torch, x, q, 4, 32, 0.4, grad=True)
    pd, gd = O.direct(x, q, grad=True)
    po, go = O.fmm(x, q, 4, 32, 0.4, grad=True)
    e_gpu, e_orc = O.rel_l2(phi, pd), O.rel_l2(po, pd)
    assert abs(e_gpu - e_orc) <= 1e-11 + 1e-3 * e_orc
    assert abs(e_orc / 1.584e-4 - 1) < 2e-3  # SURVEY c.4
    assert abs(O.rel_l2(g, gd) - O.rel_l2(go, gd)) <= 1e-11 + 1e-3 * O.rel_l2(go, gd)


@pytest.mark.parametrize("case", ["single", "two", "all_in_one_leaf", "coincident", "tiny_theta", "p0",
                                  "p16", "lattice"])
def test_edge_cases(torch_cuda, case):
    torch = torch_cuda
    rng = np.random.default_rng(1)
    p, ncrit, theta = 4, 16, 0.4
    if case == "single":
        x, q = np.array([[0.3, 0.2, 0.1]]), np.array([2.0])
    elif case == "two":
        x, q = np.array([[0.0, 0, 0], [1.0, 0, 0]]), np.array([1.0, -2.0])
    elif case == "all_in_one_leaf":
        x, q = F.cube(100, seed=3)
        ncrit = 100
    elif case == "coincident":
        x, q = F.cube(500, seed=4)
        x[100:300] = x[5]  # 200 identical points: a deep chain of cells down to level 21
    elif case == "tiny_theta":
        x, q = F.cube(2000, seed=5)
        theta = 1e-6
    elif case == "p0":
        x, q = F.plummer(4000, seed=6)
        p = 0
    elif case == "p16":
        x, q = F.cube(3000, seed=8)
        p, ncrit = 16, 20
    elif case == "lattice":  # points exactly on cell faces (PAPER.md:386 uniform lattices)
        g1 = np.arange(12) / 11.0
        x = np.stack(np.meshgrid(g1, g1, g1, indexing="ij"), -1).reshape(-1, 3)
        q = rng.uniform(-1, 1, len(x))
    _, phi, g = gpu_fmm(torch, x, q, p, ncrit, theta, grad=True)
    po, go = O.fmm(x, q, p, ncrit, theta, grad=True)
    assert np.isfinite(phi).all() and np.isfinite(g).all()
    assert O.rel_l2(phi, po) <= TOL and O.rel_l2(g, go) <= TOL
    if case == "two":
        assert phi.tolist() == [-2.0, 1.0]


def test_determinism_and_input_order(torch_cuda):
    torch = torch_cuda
    from paper_1602_02244_b200 import Plan

    x, q = F.plummer(20000, seed=11)
    pl = Plan(to_dev(torch, x), 8, 64, 0.5)
    qd = to_dev(torch, q)
    a, ga = pl.matvec(qd, grad=True)
    b, gb = pl.matvec(qd, grad=True)
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.equal(ga, gb)  # bitwise (no fp atomics)
    # host-buffer entry point gives the same bits
    ph, gh = pl.matvec_host(q, grad=True)
    assert torch.equal(ph, a.cpu()) and torch.equal(gh, ga.cpu())


def test_usage_and_numeric_errors(torch_cuda):
    torch = torch_cuda
    from paper_1602_02244_b200 import FmmError, Plan

    x, q = F.cube(100)
    bad = x.copy()
    bad[3, 0] = np.nan
    with pytest.raises(FmmError) as e:
        Plan(to_dev(torch, bad), 4, 8, 0.4)
    assert e.value.status == 2
    pl = Plan(to_dev(torch, x), 4, 8, 0.4)
    with pytest.raises(ValueError):
        pl.matvec(to_dev(torch, q[:50]))
    q2 = q.copy()
    q2[7] = np.inf
    with pytest.raises(FmmError) as e:
        pl.matvec_host(q2)
    assert e.value.status == 3
    phi = pl.matvec_host(q)  # the plan stays usable after a numeric error
    assert np.isfinite(phi.numpy()).all()


# 10^4 sampled targets (seed 12345) at every BASELINE config, configs[4] included
FULL = [("c2", 10_000), ("c3", 10_000), ("c4", 10_000), ("c5", 10_000), ("l3", 10_000)]


@pytest.mark.parametrize("name,k", FULL)
def test_full_size_sampled_parity(torch_cuda, name, k):
    """BASELINE.json full sizes, bench launch configuration, on a seeded target sample
    computed one by one by the oracle's sampled-target mode (A15)."""
    if name in ("c4", "c5") and os.environ.get("FMM_SKIP_LARGE"):
        pytest.skip("FMM_SKIP_LARGE set")
    torch = torch_cuda
    cfg = F.CONFIGS[name]
    x, q = F.make_config(name)
    _, phi, g = gpu_fmm(torch, x, q, cfg.p, cfg.ncrit, cfg.theta, grad=cfg.grad)
    T = F.target_sample(cfg.n, k)
    orc = O.Plan(x, cfg.p, cfg.ncrit, cfg.theta)
    res = orc.eval(q, grad=cfg.grad, targets=T, nthreads=O.default_threads())
    po, go = res if cfg.grad else (res, None)
    assert O.rel_l2(phi[T], po) <= TOL
    if cfg.grad:
        assert O.rel_l2(g[T], go) <= TOL
    pd = O.direct(x, q, tgt=x[T][:200], nthreads=O.default_threads())
    assert O.rel_l2(phi[T][:200], pd) < 1e-4  # truncation-level agreement with direct


@pytest.mark.parametrize("variant", ["1", "2", "3", "4"])
@pytest.mark.parametrize("dist,n,p,ncrit,theta", [("plummer", 20000, 6, 32, 0.5), ("plummer", 5000, 1, 7, 0.3),
                                                  ("sphere", 20000, 5, 40, 0.35), ("cube", 20000, 14, 64, 0.4),
                                                  ("plummer", 20000, 9, 40, 0.5), ("sphere", 20000, 12, 128, 0.4),
                                                  ("cube", 20000, 2, 32, 0.5), ("sphere", 20000, 3, 40, 0.4),
                                                  ("plummer", 20000, 4, 16, 0.5), ("cube", 8000, 0, 16, 0.5),
                                                  ("plummer", 20000, 11, 40, 0.5)])
def test_m2l_variants(torch_cuda, monkeypatch, variant, dist, n, p, ncrit, theta):
    """The four M2L formulations — v1 matrix-free O(p^4) per pair (the paper's analytic end),
    v2 precomputed dense translation-invariant operators on DMMA, v3 the
    same operators rotation-factored (p <= 14, else v2) and v4 the per-pair
    rotation with a fixed constant-bank operator on DFMA (2 <= p <= 12, else v3) — match the
    oracle."""
    monkeypatch.setenv("FMM_M2L_VARIANT", variant)
    torch = torch_cuda
    x, q = F.make(dist, n)
    _, phi, g = gpu_fmm(torch, x, q, p, ncrit, theta, grad=True)
    po, go = O.fmm(x, q, p, ncrit, theta, grad=True, nthreads=O.default_threads())
    assert O.rel_l2(phi, po) <= TOL and O.rel_l2(g, go) <= TOL


@pytest.mark.parametrize("variant", ["1", "2"])
@pytest.mark.parametrize("dist,n,p,ncrit,theta,grad", [("plummer", 20000, 4, 64, 0.5, True),
                                                       ("cube", 20000, 4, 200, 0.4, False),
                                                       ("sphere", 20000, 4, 7, 0.4, True),
                                                       ("cube", 3000, 2, 16, 1e-6, True)])
def test_near_variants(torch_cuda, monkeypatch, variant, dist, n, p, ncrit, theta, grad):
    """Near-field kernels (v1 block per leaf; v2 warp per leaf with shared-memory staging,
    lanes-per-target splitting and rsqrt seed + third-order correction) match the oracle;
    ncrit 200 exercises leaves with more than 128 sources (chunked staging) and 64+ targets."""
    monkeypatch.setenv("FMM_NEAR_VARIANT", variant)
    torch = torch_cuda
    x, q = F.make(dist, n)
    _, phi, g = gpu_fmm(torch, x, q, p, ncrit, theta, grad=grad)
    res = O.fmm(x, q, p, ncrit, theta, grad=grad, nthreads=O.default_threads())
    po, go = res if grad else (res, None)
    # all-P2P case: rounding and the one-Newton-step 1/r (<= 1.5 * 2^-40 per interaction, R11)
    tol = 2e-12 if theta < 1e-3 else TOL
    assert O.rel_l2(phi, po) <= tol
    if grad:
        assert O.rel_l2(g, go) <= tol


@pytest.mark.parametrize("variant,par", [("1", "2"), ("2", "2"), ("2", "1")])
@pytest.mark.parametrize("dist,n,p,ncrit,theta", [("plummer", 6000, 0, 16, 0.5), ("cube", 6000, 1, 8, 0.4),
                                                  ("plummer", 6000, 3, 20, 0.5), ("sphere", 8000, 8, 32, 0.4),
                                                  ("plummer", 8000, 11, 40, 0.5), ("cube", 6000, 13, 64, 0.4),
                                                  ("plummer", 4000, 16, 64, 0.5)])
def test_shift_variants(torch_cuda, monkeypatch, variant, par, dist, n, p, ncrit, theta):
    """M2M / L2L (north_star (3)): v1 block per parent with the branchy term sums and v2 the
    level-independent scaled operators A(+,+,+) on DMMA with octant sign maps
    give the oracle's multipoles per cell to 1e-13 and its local expansions to 1e-12 (or the
    condition-aware bound of check_local_condition_bound)."""
    monkeypatch.setenv("FMM_SHIFT_VARIANT", variant)
    monkeypatch.setenv("FMM_SHIFT_PAR", par)
    torch = torch_cuda
    x, q = F.make(dist, n)
    pl, phi, g = gpu_fmm(torch, x, q, p, ncrit, theta, grad=True)
    orc = O.Plan(x, p, ncrit, theta)
    po, go = orc.eval(q, grad=True, nthreads=O.default_threads())
    M, L = orc.expansions()
    Mg, Lg = pl.export("M"), pl.export("L")
    assert (np.linalg.norm(Mg - M, axis=1) <= 1e-13 * np.linalg.norm(M, axis=1) + 1e-300).all()
    nl = np.linalg.norm(L, axis=1)
    flagged = np.nonzero(np.linalg.norm(Lg - L, axis=1) > 1e-12 * nl + 1e-300)[0]
    assert len(flagged) <= max(2, len(nl) // 500)
    if len(flagged):
        check_local_condition_bound(orc, p, M, L, Lg, flagged)
    assert O.rel_l2(phi, po) <= TOL and O.rel_l2(g, go) <= TOL


@pytest.mark.parametrize("split", ["1", "2", "3", "4", "8"])
@pytest.mark.parametrize("dist,n,p,ncrit,theta", [("cube", 30000, 10, 64, 0.4), ("plummer", 20000, 12, 40, 0.5)])
def test_m2l_split_tiles(torch_cuda, monkeypatch, split, dist, n, p, ncrit, theta):
    """M2L v3 with a tile's columns split over several CTAs (partial accumulators summed from
    global scratch in rank order) matches the oracle and the unsplit kernel to rounding."""
    torch = torch_cuda
    x, q = F.make(dist, n)
    monkeypatch.setenv("FMM_M2L_VARIANT", "3")
    monkeypatch.setenv("FMM_M2L_SPLIT", "1")
    _, phi1, g1 = gpu_fmm(torch, x, q, p, ncrit, theta, grad=True)
    monkeypatch.setenv("FMM_M2L_SPLIT", split)
    _, phi, g = gpu_fmm(torch, x, q, p, ncrit, theta, grad=True)
    po, go = O.fmm(x, q, p, ncrit, theta, grad=True, nthreads=O.default_threads())
    assert O.rel_l2(phi, po) <= TOL and O.rel_l2(g, go) <= TOL
    assert O.rel_l2(phi, phi1) <= 1e-14


@pytest.mark.parametrize("variant", ["1", "2", "3", "4"])
def test_stats_bytes_by_category(torch_cuda, monkeypatch, variant):
    """fmm_stats bytes_by (include/fmm.h FMM_B_*) partitions bytes_device; operator tables exist
    only for the precomputed formulations (v2/v3) beside the small M2M/L2L operators."""
    monkeypatch.setenv("FMM_M2L_VARIANT", variant)
    torch = torch_cuda
    x, q = F.cube(20000, seed=2)
    pl, _, _ = gpu_fmm(torch, x, q, 8, 32, 0.4, grad=False)
    st = pl.stats()
    by = st["bytes_by"]
    assert all(v >= 0 for v in by.values()) and sum(by.values()) == st["bytes_device"]
    assert by["other"] < 1024 and by["let"] == 0  # other: the device status word
    nc = 9 * 10 // 2
    assert by["expansions"] >= 2 * 16 * nc * st["n_cells"]
    assert by["particles"] >= 44 * st["n"]
    if variant == "1":
        assert by["operators"] < 1e6 and by["schedule"] == 0
    elif variant == "4":  # the fixed operator lives in constant memory; unit partial sums
        assert by["operators"] < 1e6 and by["schedule"] > 0
    else:
        assert by["operators"] > 1e6 and by["schedule"] > 0


@pytest.mark.parametrize("chunks", ["1", "2", "5"])
@pytest.mark.parametrize("dist,n,p,ncrit,theta", [("plummer", 20000, 8, 32, 0.5), ("cube", 20000, 10, 64, 0.4),
                                                  ("sphere", 20000, 12, 128, 0.4)])
def test_m2l_v4_units(torch_cuda, monkeypatch, chunks, dist, n, p, ncrit, theta):
    """M2L v4 with small work units (1, 2, 5 chunks of 32 pairs): targets cross many unit
    boundaries (partial sums per unit, added in unit order by the fix-up kernel, including units
    that lie wholly inside one target); results match the oracle and the default units."""
    torch = torch_cuda
    x, q = F.make(dist, n)
    monkeypatch.setenv("FMM_M2L_VARIANT", "4")
    _, phi0, g0 = gpu_fmm(torch, x, q, p, ncrit, theta, grad=True)
    monkeypatch.setenv("FMM_V4_UNIT_CHUNKS", chunks)
    for wpc in ("1", "3"):
        monkeypatch.setenv("FMM_V4_WARPS", wpc)
        _, phi, g = gpu_fmm(torch, x, q, p, ncrit, theta, grad=True)
        assert O.rel_l2(phi, phi0) <= 1e-14 and O.rel_l2(g, g0) <= 1e-14
    po, go = O.fmm(x, q, p, ncrit, theta, grad=True, nthreads=O.default_threads())
    assert O.rel_l2(phi, po) <= TOL and O.rel_l2(g, go) <= TOL


@pytest.mark.parametrize("dist,n,p,ncrit,theta,grad", [("cube", 20000, 10, 64, 0.4, True),
                                                       ("plummer", 20000, 6, 32, 0.5, False)])
def test_overlapped_near_field(torch_cuda, monkeypatch, dist, n, p, ncrit, theta, grad):
    """FMM_OVERLAP_NEAR=1: the P2P sums on a low-priority stream beside the far field, L2P after
    L2L (measured not faster, profiles/r2_overlap.md) — results equal the serial path's."""
    torch = torch_cuda
    x, q = F.make(dist, n)
    _, phi0, g0 = gpu_fmm(torch, x, q, p, ncrit, theta, grad=grad)
    monkeypatch.setenv("FMM_OVERLAP_NEAR", "1")
    _, phi, g = gpu_fmm(torch, x, q, p, ncrit, theta, grad=grad)
    assert O.rel_l2(phi, phi0) <= 1e-15
    if grad:
        assert O.rel_l2(g, g0) <= 1e-15


def test_repeated_matvecs_bitwise_equal(torch_cuda, monkeypatch):
    """Stand-in for compute-sanitizer racecheck (closed on this pool, profiles/r2_sanitizer.md):
    a shared-memory race in the warp-cooperative kernels (M2L v4's copy / in-place stages /
    segmented sums, the near field's staging) would show up as run-to-run differences; 12
    repeated mat-vecs, with several M2L v4 unit sizes and warp counts, are bitwise identical."""
    torch = torch_cuda
    from paper_1602_02244_b200 import Plan

    x, q = F.make("plummer", 30000)
    xd, qd = to_dev(torch, x), to_dev(torch, q)
    for uc, wp in (("0", "0"), ("1", "2"), ("3", "5")):
        monkeypatch.setenv("FMM_V4_UNIT_CHUNKS", uc)
        monkeypatch.setenv("FMM_V4_WARPS", wp)
        pl = Plan(xd, 8, 32, 0.5)
        ref = pl.matvec(qd, grad=True)
        for _ in range(12):
            out = pl.matvec(qd, grad=True)
            assert torch.equal(out[0], ref[0]) and torch.equal(out[1], ref[1])


@pytest.mark.parametrize("dist,n,p,ncrit,theta", [("cube", 30000, 10, 64, 0.4), ("plummer", 20000, 6, 32, 0.5),
                                                  ("sphere", 20000, 8, 16, 0.4), ("plummer", 8000, 3, 7, 0.3),
                                                  ("cube", 3000, 2, 16, 1e-6), ("cube", 4000, 4, 1, 0.4),
                                                  ("sphere", 40000, 12, 128, 0.4), ("cube", 20000, 6, 100, 0.4)])
def test_mutual_near_field(torch_cuda, monkeypatch, dist, n, p, ncrit, theta):
    """Potentials-only mat-vecs evaluate each unordered P2P leaf pair once (csrc/near_mutual.cu):
    oracle parity, agreement with the directed P2P (FMM_NEAR_MUTUAL=0) to rounding, and bitwise
    repeatability (its sums have a fixed order: per-task partial slots, no atomics)."""
    torch = torch_cuda
    from paper_1602_02244_b200 import Plan

    x, q = F.make(dist, n)
    xd, qd = to_dev(torch, x), to_dev(torch, q)
    pl = Plan(xd, p, ncrit, theta)
    assert pl.stats()["near_mutual"] == 1
    phi = pl.matvec(qd)
    for _ in range(5):
        assert torch.equal(pl.matvec(qd), phi)
    phi = phi.cpu().numpy()
    ref = O.fmm(x, q, p, ncrit, theta, nthreads=O.default_threads())
    tol = 2e-12 if theta < 1e-3 else TOL  # all-P2P case: as test_near_variants
    assert O.rel_l2(phi, ref) <= tol
    monkeypatch.setenv("FMM_NEAR_MUTUAL", "0")
    pd = Plan(xd, p, ncrit, theta)
    assert pd.stats()["near_mutual"] == 0
    assert O.rel_l2(phi, pd.matvec(qd).cpu().numpy()) <= 1e-14
    # gradients always take the directed path on the same plan
    g = pl.matvec(qd, grad=True)
    gd = pd.matvec(qd, grad=True)
    assert torch.equal(g[0], gd[0]) and torch.equal(g[1], gd[1])


def test_mutual_near_field_limits(torch_cuda):
    """Leaves above 128 particles keep the directed P2P (the mutual kernel's register layout);
    leaves of 65-128 take its 16-group layout, checked against the directed path."""
    torch = torch_cuda
    from paper_1602_02244_b200 import Plan

    x, q = F.make("cube", 16000)  # 16000 / 64 = 250 per level-2 cell: leaves of ~250 particles
    pl = Plan(to_dev(torch, x), 4, 300, 0.4)
    assert pl.stats()["near_mutual"] == 0
    assert pl.matvec(to_dev(torch, q)).shape == (16000,)
    x, q = F.make("cube", 8000)  # 8000 / 64 = 125 per level-2 cell: leaves of ~125 particles
    xd, qd = to_dev(torch, x), to_dev(torch, q)
    pl = Plan(xd, 4, 128, 0.4)  # leaves of <= 128, most of them above 64
    assert pl.stats()["near_mutual"] == 1
    phi = pl.matvec(qd).cpu().numpy()
    po = O.fmm(x, q, 4, 128, 0.4)
    assert O.rel_l2(phi, po) <= 1e-11
