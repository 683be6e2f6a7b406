"""Pins for the whole oracle FMM: worked examples, reductions to
direct summation, the pair-cover invariant of the interaction lists, exact
invariants (linearity, X -> 2X, input order), convergence with p, and the
survey's independent counts.

Paper: FMM approximates the direct N-body sum; the direct
operator is the dense diagonal block and the translations are the
off-diagonal blocks; lists come from a dual tree traversal
with a MAC.
"""
import json
import os

import numpy as np
import pytest

import fmm_inputs as F
from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_worked_example_p2p_sign():
    ex = gold("worked_examples.json")["p2p_sign"]
    for p in (0, 3, 7):
        phi, g = O.fmm(np.array(ex["xyz"]), np.array(ex["q"]), p, 2, 0.4, grad=True)
        assert phi.tolist() == ex["phi"]
        assert g.tolist() == ex["grad"]


def test_worked_example_two_unit_charges_direct():
    ex = gold("worked_examples.json")["two_unit_charges"]
    phi, g = O.direct(np.array(ex["xyz"]), np.array(ex["q"]), grad=True)
    assert phi.tolist() == ex["phi"]
    assert g.tolist() == ex["grad"]


def test_worked_example_quantization_and_keys():
    ex = gold("worked_examples.json")["quantization"]
    pl = O.Plan(np.array(ex["xyz"]), 2, 1, 0.4)
    lo, S, scale = pl.geometry()
    assert lo.tolist() == ex["lo"] and S == ex["S"] and scale == ex["scale"]
    assert pl.info("exp") == ex["exp"]
    keys, perm = pl.keys()
    assert [hex(int(k)) for k in keys] == ex["keys"]
    assert perm.tolist() == [0, 1, 2]
    assert [int(k) >> 60 for k in keys] == ex["level1_digits"]


def test_direct_matches_float64_brute_force():
    rng = np.random.default_rng(3)
    x = rng.random((300, 3))
    q = rng.uniform(-1, 1, 300)
    d = x[:, None, :] - x[None, :, :]
    r = np.sqrt((d**2).sum(-1))
    np.fill_diagonal(r, np.inf)
    phi = (q[None, :] / r).sum(1)
    g = -(q[None, :, None] * d / r[..., None] ** 3).sum(1)
    po, go = O.direct(x, q, grad=True)
    assert np.abs(po - phi).max() < 1e-12
    assert np.abs(go - g).max() < 1e-10


def test_coincident_points_contribute_nothing():
    """Q2: pairs with r^2 == 0 are skipped (self term and duplicates)."""
    x = np.array([[0.0, 0, 0], [0.0, 0, 0], [1.0, 0, 0]])
    q = np.array([1.0, 5.0, 2.0])
    phi = O.direct(x, q)
    assert phi.tolist() == [2.0, 2.0, 6.0]
    assert O.fmm(x, q, 4, 4, 0.4).tolist() == [2.0, 2.0, 6.0]


def test_single_leaf_equals_direct():
    """N <= ncrit -> the root is a leaf -> only the (root, root) P2P pair."""
    x, q = F.cube(200, seed=4)
    phi, g = O.fmm(x, q, 4, 200, 0.4, grad=True)
    pd, gd = O.direct(x, q, grad=True)
    assert O.rel_l2(phi, pd) < 1e-14 and O.rel_l2(g, gd) < 1e-14


def test_tiny_theta_equals_direct():
    """theta -> 0: the MAC never accepts, the M2L list is empty, all work is P2P."""
    x, q = F.cube(1000)
    pl = O.Plan(x, 4, 32, 1e-6)
    assert pl.info("nm2l") == 0
    phi, g = pl.eval(q, grad=True)
    pd, gd = O.direct(x, q, grad=True)
    assert O.rel_l2(phi, pd) < 1e-14 and O.rel_l2(g, gd) < 1e-14


@pytest.mark.parametrize("dist,n,ncrit,theta", [("cube", 1500, 16, 0.4), ("plummer", 2000, 8, 0.5),
                                                ("sphere", 2000, 16, 0.4)])
def test_pair_cover_and_mac(dist, n, ncrit, theta):
    """Every ordered particle pair (i, j) is covered exactly once, by one P2P leaf pair or
    one M2L cell pair; every M2L pair satisfies the MAC and has disjoint ranges
    (the SPEC.md:74,83 pair-cover property, adapted to dual-traversal lists)."""
    x, _ = F.make(dist, n)
    pl = O.Plan(x, 2, ncrit, theta)
    c = pl.cells()
    p2p, m2l = pl.lists()
    cover = np.zeros((n, n), np.int32)
    for lst in (p2p, m2l):
        for A, B in lst:
            cover[c["begin"][A]:c["end"][A], c["begin"][B]:c["end"][B]] += 1
    assert (cover == 1).all()
    H = (1 << (21 - c["level"])).astype(np.int64)
    Cc = (2 * c["anchor"].astype(np.int64) + 1) * H[:, None]
    for A, B in m2l:
        d2 = int(((Cc[A] - Cc[B]) ** 2).sum())
        assert (theta * theta) * d2 > (H[A] + H[B]) ** 2
        assert c["end"][A] <= c["begin"][B] or c["end"][B] <= c["begin"][A]
    leaf = c["child_first"] < 0
    assert leaf[p2p[:, 0]].all() and leaf[p2p[:, 1]].all()


def test_tree_structure_invariants():
    x, _ = F.plummer(3000)
    pl = O.Plan(x, 2, 10, 0.5)
    c = pl.cells()
    keys, perm = pl.keys()
    assert sorted(perm.tolist()) == list(range(3000))  # a permutation
    assert (np.diff(keys.astype(np.uint64)) >= 0).all()
    leaf = c["child_first"] < 0
    cnt = c["end"] - c["begin"]
    assert (cnt[~leaf] > 10).all() and (cnt >= 1).all()
    assert (cnt[leaf] <= 10).all() or (c["level"][leaf][cnt[leaf] > 10] == 21).all()
    lb = np.sort(c["begin"][leaf])
    assert lb[0] == 0 and (np.sort(c["end"][leaf])[:-1] == lb[1:]).all()  # leaves partition [0, N)
    assert (np.diff(c["level"]) >= 0).all()  # breadth-first
    for i in np.nonzero(~leaf)[0]:
        ch = np.arange(c["child_first"][i], c["child_first"][i] + c["nchild"][i])
        assert (c["parent"][ch] == i).all()
        assert c["begin"][ch[0]] == c["begin"][i] and c["end"][ch[-1]] == c["end"][i]


def test_root_monopole_is_total_charge():
    x, q = F.cube(5000, seed=2)
    pl = O.Plan(x, 6, 32, 0.4)
    pl.eval(q)
    M, L = pl.expansions()
    assert abs(M[0, 0] - q.sum()) < 1e-12


def test_linearity_in_q():
    x, q1 = F.cube(2000, seed=1)
    q2 = np.random.default_rng(9).uniform(-1, 1, 2000)
    pl = O.Plan(x, 6, 32, 0.4)
    a = pl.eval(2.5 * q1 - 0.75 * q2)
    b = 2.5 * pl.eval(q1) - 0.75 * pl.eval(q2)
    assert O.rel_l2(a, b) < 1e-14


def test_scaling_X_by_2_is_bitwise():
    """X -> 2X: same normalised geometry (exact 2^-e), so phi/2 and grad/4 exactly."""
    x, q = F.plummer(3000, seed=3)
    a, ga = O.fmm(x, q, 6, 16, 0.5, grad=True)
    b, gb = O.fmm(2 * x, q, 6, 16, 0.5, grad=True)
    assert np.array_equal(a / 2, b) and np.array_equal(ga / 4, gb)


def test_input_order_invariance():
    x, q = F.cube(3000, seed=5)
    a, ga = O.fmm(x, q, 6, 32, 0.4, grad=True)
    sh = np.random.default_rng(0).permutation(3000)
    b, gb = O.fmm(x[sh], q[sh], 6, 32, 0.4, grad=True)
    assert O.rel_l2(a[sh], b) < 1e-14 and O.rel_l2(ga[sh], gb) < 1e-14


def test_convergence_in_p_matches_survey_scratch():
    g = gold("survey_scratch_c1.json")
    x, q = F.cube(1000)
    pd, gd = O.direct(x, q, grad=True)
    prev = (np.inf, np.inf)
    for p in (2, 3, 4, 5, 6, 8, 10, 12):
        phi, gr = O.fmm(x, q, p, 32, 0.4, grad=True)
        e, eg = O.rel_l2(phi, pd), O.rel_l2(gr, gd)
        assert e < prev[0] and eg < prev[1]  # strictly decreasing
        assert abs(e / g["rel_l2_phi_vs_direct"][str(p)] - 1) < 2e-3
        assert abs(eg / g["rel_l2_grad_vs_direct"][str(p)] - 1) < 2e-2
        prev = (e, eg)


def test_counts_c1_match_survey():
    g = gold("survey_scratch_c1.json")["counts"]
    x, _ = F.cube(1000)
    pl = O.Plan(x, 4, 32, 0.4)
    c = pl.cells()
    _, m2l = pl.lists()
    assert pl.ncells == g["cells"] and pl.info("nleaves") == g["leaves"]
    assert pl.info("np2p") == g["p2p_pairs"] and pl.info("nm2l") == g["m2l_pairs"]
    assert int((c["level"][m2l[:, 1]] < c["level"][m2l[:, 0]]).sum()) == g["m2l_source_coarser"]
    assert pl.info("p2p_interactions") == g["p2p_interactions_incl_self"]


def test_counts_c2_match_survey():
    g = gold("survey_scratch_counts.json")["c2"]
    x, _ = F.cube(g["n"])
    pl = O.Plan(x, 10, g["ncrit"], g["theta"])
    c = pl.cells()
    _, m2l = pl.lists()
    assert pl.ncells == g["cells"] and pl.info("nleaves") == g["leaves"]
    assert pl.info("np2p") == g["p2p_pairs"] and pl.info("nm2l") == g["m2l_pairs"]
    assert pl.info("p2p_interactions") == g["p2p_interactions_incl_self"]
    assert int((c["level"][m2l[:, 1]] < c["level"][m2l[:, 0]]).sum()) == g["m2l_source_coarser"]


def test_sampled_target_mode_equals_full():
    """A15: the restricted traversal gives the full run's values at the sampled targets."""
    x, q = F.plummer(20000)
    pl = O.Plan(x, 6, 32, 0.5)
    full, gfull = pl.eval(q, grad=True)
    T = F.target_sample(20000, 200)
    s, gs = pl.eval(q, grad=True, targets=T)
    assert O.rel_l2(s, full[T]) < 1e-15 and O.rel_l2(gs, gfull[T]) < 1e-15


def test_truncation_error_magnitude_c2_sample():
    """Oracle vs direct at C2 (p=10, theta=0.4) sits at the survey's ~1e-6 level."""
    x, q = F.cube(100000)
    pl = O.Plan(x, 10, 64, 0.4)
    T = F.target_sample(100000, 500)
    phi, g = pl.eval(q, grad=True, targets=T)
    pd, gd = O.direct(x, q, tgt=x[T], grad=True)
    assert 1e-7 < O.rel_l2(phi, pd) < 1e-5
    assert 1e-7 < O.rel_l2(g, gd) < 1e-5


@pytest.mark.parametrize("bad", [dict(p=-1), dict(p=17), dict(ncrit=0), dict(theta=0.0), dict(theta=0.6),
                                 dict(theta=float("nan"))])
def test_usage_errors(bad):
    args = dict(p=4, ncrit=8, theta=0.4)
    args.update(bad)
    x, _ = F.cube(10)
    with pytest.raises(O.OracleError) as e:
        O.Plan(x, **args)
    assert e.value.status == 2


def test_nonfinite_inputs():
    x, q = F.cube(10)
    x[3, 1] = np.nan
    with pytest.raises(O.OracleError):
        O.Plan(x, 4, 8, 0.4)
    x, q = F.cube(10)
    q[2] = np.inf
    with pytest.raises(O.OracleError) as e:
        O.Plan(x, 4, 8, 0.4).eval(q)
    assert e.value.status == 3
