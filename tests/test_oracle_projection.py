"""Pins of the Prop.1 projection oracle (reading R33, oracle/projection.py) against
what the mathematics fixes: the textbook halfspace / box projections, the KKT conditions
(checked with non-negative least squares), an independent QP solver (scipy SLSQP), Dykstra's
convergence to the exact projection, and the soundness of the R33 margin."""
import numpy as np
import pytest
from scipy.optimize import minimize, nnls

from oracle import hsmt, projection, semantics, solve

UNIT_TEXT = """p hsmt 0 3
a 0 <= 1 0:1 1:1
a 1 < 0.5 1:2 2:-1
a 2 <= -0.25 0:1 2:1
a 3 <= 0.9 0:1
a 4 >= -0.8 2:1
c or 1 +a0
c or 1 -a1
e 2 (not a2)
c or 1 +a3
c or 1 +a4
"""


def random_system(rng, m=3, K=2):
    """K two-variable halfspaces and the box [-1, 1]^m, all holding with slack at a random y0."""
    y0 = rng.uniform(-0.8, 0.8, size=m)
    H = []
    for _ in range(K):
        cols = sorted(rng.choice(m, size=2, replace=False).tolist())
        g = rng.choice([-2.0, -1.0, 1.0, 3.0], size=2)
        H.append((cols, g, float(g @ y0[cols] + rng.uniform(0.05, 0.5))))
    lo = np.full(m, -1.0)
    hi = np.full(m, 1.0)
    return H, lo, hi


def test_single_halfspace_textbook():
    # projection onto {g.b <= h} is bp - max(0, g.bp - h)/||g||^2 g (textbook)
    rng = np.random.default_rng(1)
    for _ in range(20):
        g = rng.normal(size=3)
        h = float(rng.normal())
        bp = rng.normal(size=3) * 2
        want = bp - max(0.0, g @ bp - h) / (g @ g) * g
        inf = np.full(3, np.inf)
        got = projection.project_exact(bp, -inf, inf, [([0, 1, 2], g, h)])
        assert np.allclose(got, want, atol=1e-12)


def test_box_only_is_clamp():
    rng = np.random.default_rng(2)
    bp = rng.normal(size=4) * 2
    lo, hi = np.full(4, -1.0), np.full(4, 0.5)
    assert np.allclose(projection.project_exact(bp, lo, hi, []), np.clip(bp, lo, hi))
    assert np.allclose(projection.dykstra(bp, lo, hi, [], 1), np.clip(bp, lo, hi))


def test_exact_projection_kkt_and_slsqp():
    rng = np.random.default_rng(3)
    for _ in range(25):
        H, lo, hi = random_system(rng)
        bp = rng.normal(size=3) * 1.5
        y = projection.project_exact(bp, lo, hi, H)
        # primal feasibility
        for cols, g, h in H:
            assert g @ y[cols] <= h + 1e-9
        assert np.all(y >= lo - 1e-12) and np.all(y <= hi + 1e-12)
        # KKT: bp - y = sum over active constraints of lam_k * normal_k with lam >= 0 (NNLS residual 0)
        normals = []
        for cols, g, h in H:
            if abs(g @ y[cols] - h) < 1e-9:
                n = np.zeros(3); n[cols] = g; normals.append(n)
        for j in range(3):
            if abs(y[j] - hi[j]) < 1e-12:
                n = np.zeros(3); n[j] = 1; normals.append(n)
            if abs(y[j] - lo[j]) < 1e-12:
                n = np.zeros(3); n[j] = -1; normals.append(n)
        if normals:
            _, res = nnls(np.array(normals).T, bp - y)
            assert res < 1e-9
        else:
            assert np.allclose(y, bp)
        # an independent QP solver
        cons = [{"type": "ineq", "fun": (lambda b, cols=cols, g=g, h=h: h - g @ b[cols])} for cols, g, h in H]
        r = minimize(lambda b: np.sum((b - bp) ** 2), np.clip(bp, lo, hi), method="SLSQP", constraints=cons,
                     bounds=list(zip(lo, hi)), options={"ftol": 1e-14, "maxiter": 500})
        assert np.allclose(r.x, y, atol=1e-6)


def test_dykstra_converges_to_exact():
    rng = np.random.default_rng(4)
    for _ in range(15):
        H, lo, hi = random_system(rng, m=4, K=3)
        bp = rng.normal(size=4) * 1.5
        y = projection.project_exact(bp, lo, hi, H)
        assert np.allclose(projection.dykstra(bp, lo, hi, H, 4000), y, atol=1e-8)


def test_dykstra_is_not_plain_alternating_projection():
    # cyclic projections without Dykstra's corrections reach a feasible point that is in general
    # not the nearest one; with the corrections the limit is the QP minimiser
    rng = np.random.default_rng(6)
    differs = 0
    for _ in range(40):
        H, lo, hi = random_system(rng, m=4, K=3)
        bp = rng.normal(size=4) * 1.5
        y = projection.project_exact(bp, lo, hi, H)
        assert np.allclose(projection.dykstra(bp, lo, hi, H, 4000), y, atol=1e-8)
        x = bp.copy()
        for _ in range(500):
            for cols, g, h in H:
                x[cols] -= max(0.0, g @ x[cols] - h) / (g @ g) * g
            x = np.clip(x, lo, hi)
        differs += np.abs(x - y).max() > 1e-3
    assert differs >= 3


def test_r33_halfspaces_sound():
    f = hsmt.parse(UNIT_TEXT)
    H = projection.halfspaces(f)
    assert len(H) == 3                           # a0, not a1, not a2 (a3, a4 are interval bounds)
    lo, hi = solve.bounds(f)
    rng = np.random.default_rng(5)
    n_in = 0
    for _ in range(4000):
        y = rng.uniform(-1.5, 1.5, size=3).astype(np.float32)
        inside = all(g @ y[cols].astype(np.float64) <= h for cols, g, h in H)
        if inside:
            n_in += 1
            for c in f.constraints[:3]:
                assert semantics.constraint_sat(f, c, np.zeros(0, np.int8), y)
    assert n_in > 100
    # projecting then rounding to fp32 satisfies every unit atom (the margin absorbs the rounding)
    for _ in range(200):
        bp = rng.uniform(-2, 2, size=3)
        y = projection.project_exact(bp, lo.astype(np.float64), hi.astype(np.float64), H).astype(np.float32)
        for c in f.constraints:
            assert semantics.constraint_sat(f, c, np.zeros(0, np.int8), y)
