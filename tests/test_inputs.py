"""The seeded workload generators (fmm_inputs.py): shapes, ranges and determinism; the NEXT-3
lattice is the paper's §4.1 geometry: exact grid, every point on cell faces."""
import numpy as np

import fmm_inputs as F


def test_lattice_geometry():
    x, q = F.lattice(27)
    assert x.shape == (27, 3) and q.shape == (27,)
    assert np.array_equal(np.unique(x[:, 0]), np.array([-0.5, 0.0, 0.5]))
    x2, q2 = F.lattice(27)
    assert np.array_equal(x, x2) and np.array_equal(q, q2)
    xl, _ = F.make_config("l3")
    assert xl.shape == (1_000_000, 3) and F.CONFIGS["l3"].index == -1
    g = np.unique(xl[:, 2])
    assert g.size == 100 and np.allclose(np.diff(g), 2.0 / 101)


def test_baseline_generators_are_seeded():
    for dist in ("cube", "plummer", "sphere"):
        a, qa = F.make(dist, 1000)
        b, qb = F.make(dist, 1000)
        assert a.shape == (1000, 3) and np.array_equal(a, b) and np.array_equal(qa, qb)
    assert (F.cube(100)[0] >= 0).all() and (F.cube(100)[0] < 1).all()
    assert np.allclose(np.linalg.norm(F.sphere(100)[0], axis=1), 1.0)
    assert (np.linalg.norm(F.plummer(1000)[0], axis=1) <= 100.0 + 1e-9).all()
