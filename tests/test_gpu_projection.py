"""GPU parity of the Prop.1 projection with multi-variable unit atoms (reading R33):
the Dykstra kernel at init and inside the PGD step against oracle/projection.py, and the
projected points satisfying every unit atom under the exact check."""
import numpy as np
import pytest

import fsmt_gen
from fsmt_gen.points import random_points
from oracle import hsmt, projection, semantics, solve

pytestmark = pytest.mark.gpu

TEXT = """p hsmt 3 4
a 0 <= 1 0:1 1:1
a 1 < 0.5 1:2 2:-1
a 2 <= -0.25 0:1 2:1 3:0.5
a 3 <= 0.9 0:1
a 4 >= -0.8 2:1
a 5 <= 0.3 1:1 3:-1
c or 1 +a0
c or 1 -a1
e 2 (not a2)
c or 1 +a3
c or 1 +a4
c or 1 +b0 +a5 -b1
c xor 1 +b1 +b2 +a1
c nae 1 +b0 +b2 +a2
"""
ITERS = 60


def make(text, iters=ITERS):
    import paper_2603_22877_b200 as P
    s = P.Solver(0)
    s.load_formula(text)
    s.build_xbdd()
    s.set_params(eta=0.05, eps=1e-12, proj_iters=iters)
    return s


def test_init_matches_oracle_dykstra():
    f = hsmt.parse(TEXT)
    s = make(TEXT)
    assert s.get_dims()["n_halfspaces"] == 3
    lo, hi = solve.bounds(f)
    H = projection.halfspaces(f)
    R = 70
    s.begin(R, 11)
    a, b = s.get_state()
    for r in (0, 33, 69):
        oa, ob = solve.init_point(f, 11, r, lo, hi, H, ITERS)
        assert np.array_equal(a[:, r], oa.astype(np.float32))
        assert np.max(np.abs(b[:, r] - ob)) <= 2e-5, (r, b[:, r], ob)


def test_step_matches_oracle_and_unit_atoms_hold():
    f = hsmt.parse(TEXT)
    s = make(TEXT)
    lo, hi = solve.bounds(f)
    H = projection.halfspaces(f)
    R = 45
    a, b = random_points(f.n_bool, f.n_real, R, seed=3, b_lo=-2.0, b_hi=2.0)
    s.begin(R, 1)
    s.set_state(a, b)
    kappa, eta = 1.7, 0.05
    s.sweep(kappa, 1)
    s.update(eta, 1e-12)
    a2, b2 = s.get_state()
    w = [c.weight for c in f.constraints]
    for r in range(0, R, 11):
        oa, ob, _, _ = solve.pgd_step(f, a[:, r].astype(np.float64), b[:, r].astype(np.float64), kappa, w, eta, lo, hi,
                                      None, H, ITERS)
        assert np.max(np.abs(a2[:, r] - oa)) <= 1e-5
        assert np.max(np.abs(b2[:, r] - ob)) <= 2e-5, (r, b2[:, r], ob)
    # every unit atom literal (interval and halfspace) holds at every projected point
    x = np.where(a2 < 0, -1, 1).astype(np.int8)
    _, pc = s.verify_batch(x, b2, per_con=True)
    unit = [ci for ci, c in enumerate(f.constraints) if solve.unit_literal(f, c) is not None]
    assert len(unit) == 5
    assert not pc[unit].any()


def test_projection_off_keeps_r15():
    # proj_iters = 0: multi-variable unit atoms stay soft (R15): the step is the plain clamp
    f = hsmt.parse(TEXT)
    s = make(TEXT, iters=0)
    lo, hi = solve.bounds(f)
    R = 33
    a, b = random_points(f.n_bool, f.n_real, R, seed=4, b_lo=-2.0, b_hi=2.0)
    s.begin(R, 1)
    s.set_state(a, b)
    s.sweep(1.0, 1)
    s.update(0.05, 1e-12)
    _, b2 = s.get_state()
    w = [c.weight for c in f.constraints]
    for r in (0, 32):
        _, ob, _, _ = solve.pgd_step(f, a[:, r].astype(np.float64), b[:, r].astype(np.float64), 1.0, w, 0.05, lo, hi)
        assert np.max(np.abs(b2[:, r] - ob)) <= 1e-5


def test_scheduling_dependencies_hard_under_projection():
    # cfg3's dependency constraints (y_j >= y_dep + t_dep) are multi-variable unit atoms:
    # with the R33 projection every returned model satisfies all of them
    inst = fsmt_gen.config("cfg3s")
    f = hsmt.parse(inst.text)
    s = make(inst.text, iters=30)
    nh = s.get_dims()["n_halfspaces"]
    assert nh > 0
    s.set_params(eta=0.03, eta_mode=3, erwa_mode=1, proj_iters=30,
                 kappas=[100.0 ** (i / 9) for i in range(10)])
    res = s.solve(256, 20, 0)
    _, pc = s.verify(res.x, res.y, per_con=True)
    dep = [ci for ci, c in enumerate(f.constraints)
           if solve.unit_literal(f, c) is not None and len(f.atoms[solve.unit_literal(f, c)[0]].coeffs) >= 2]
    assert len(dep) == nh
    assert not np.asarray(pc)[dep].any()
