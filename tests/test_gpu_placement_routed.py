"""The paper's placement family with routing-aware constraints (reading R25; generator
fsmt_gen.placement_routed): place9856s (4 macros x 8 layers, 56 modules) against the oracle in full --
every E_c, objective and gradient with live ERWA counters, exact per-constraint verdicts, and the R33
projection onto the 4 x (pairs) adjacency halfspaces -- and the full 9,856-variable / 415,424-constraint
instance at the bench launch configuration on sampled outputs, plus a solve whose model satisfies every
routing constraint."""
import numpy as np
import pytest

import fsmt_gen
from fsmt_gen.points import random_points, random_counters
from oracle import hsmt, objective, projection, semantics, solve as osolve
from tests.helpers import check_gradient, check_objective

pytestmark = pytest.mark.gpu


def _solver(text, prepare=0):
    import paper_2603_22877_b200 as P
    s = P.Solver(0)
    s.load_formula(text)
    s.build_xbdd()
    if prepare:
        s.prepare(prepare)
    return s


def test_place9856s_sweep_and_check_match_oracle():
    inst = fsmt_gen.config("place9856s")
    f = hsmt.parse(inst.text)
    s = _solver(inst.text)
    assert s.jit_info()["status"] == "active"
    R = 64
    a, b = random_points(f.n_bool, f.n_real, R, seed=51, b_lo=0.0, b_hi=1.0)
    U = random_counters(len(f.constraints), R, seed=52, max_u=5)
    for mode in (0, 1):
        s.set_params(erwa_mode=mode)
        s.begin(R, 3)
        s.set_state(a, b)
        s.set_counters(U)
        for kappa, t in ((0.5, 1), (2.0, 6), (8.0, 11)):
            s.sweep(kappa, t)
            obj, ga, gb = s.get_sweep()
            for r in (0, 33, 63):
                e = 0.0 if mode == 1 else max(t - 2, 0) / 2.0
                w = np.array([c.weight for c in f.constraints]) * 2.0 ** (U[:, r].astype(np.float64) + e)
                C, oga, ogb, terms = objective.objective_and_gradient_grouped(f, a[:, r], b[:, r], kappa, w,
                                                                              want_terms=True)
                E = s.constraint_terms(kappa, r)
                assert np.max(np.abs(E - np.array([terms[i] for i in range(len(f.constraints))]))) <= 1e-6
                what = f"place9856s mode={mode} kappa={kappa} t={t} r={r}"
                check_objective(obj[r], C, float(w.sum()), what=what)
                check_gradient(np.concatenate([ga[:, r], gb[:, r]]), np.concatenate([oga, ogb]),
                               scale_relative=True, what=what)
    x = np.where(a < 0, -1, 1).astype(np.int8)
    u, pc = s.verify_batch(x, b, per_con=True)
    for r in (0, 63):
        want = osolve.violations(f, x[:, r], b[:, r])
        assert np.array_equal(pc[:, r].astype(np.int64), want) and u[r] == want.sum()
    assert s.verify(inst.x_star, inst.y_star) == 0                       # the planted witness


def test_place9856s_routing_projection_matches_oracle():
    """R33: the adjacency atoms of the routing constraints are halfspaces; the Dykstra projection of a
    PGD step matches the oracle's and every routing adjacency atom holds after it."""
    inst = fsmt_gen.config("place9856s")
    f = hsmt.parse(inst.text)
    iters = 40
    s = _solver(inst.text)
    s.set_params(eta=0.05, eps=1e-12, proj_iters=iters)
    nh = s.get_dims()["n_halfspaces"]
    assert nh == 4 * inst.meta["pairs"]
    lo, hi = osolve.bounds(f)
    H = projection.halfspaces(f)
    R = 40
    a, b = random_points(f.n_bool, f.n_real, R, seed=53, b_lo=0.0, b_hi=1.0)
    s.begin(R, 1)
    s.set_state(a, b)
    s.sweep(1.5, 1)
    s.update(0.05, 1e-12)
    a2, b2 = s.get_state()
    w = [c.weight for c in f.constraints]
    for r in (0, 21, 39):
        oa, ob, _, _ = osolve.pgd_step(f, a[:, r].astype(np.float64), b[:, r].astype(np.float64), 1.5, w, 0.05, lo, hi,
                                       None, H, iters)
        assert np.max(np.abs(a2[:, r] - oa)) <= 1e-5
        assert np.max(np.abs(b2[:, r] - ob)) <= 5e-5, (r, np.max(np.abs(b2[:, r] - ob)))


def test_place9856_full_size_sampled():
    inst = fsmt_gen.config("place9856")
    R = 1024
    s = _solver(inst.text, prepare=R)
    assert s.jit_info()["status"].startswith("active; prepared R=1024")
    d = s.get_dims()
    assert (d["n_bool"] + d["n_real"], d["n_cons"]) == (9856, 415424)
    a, b = random_points(d["n_bool"], d["n_real"], R, seed=54, b_lo=0.0, b_hi=1.0)
    U = random_counters(d["n_cons"], R, seed=55, max_u=4)
    s.begin(R, 5)
    s.set_state(a, b)
    s.set_counters(U)
    s.sweep(1.0, 3)
    obj, ga, gb = s.get_sweep()
    assert np.all(np.isfinite(obj)) and np.all(np.isfinite(ga)) and np.all(np.isfinite(gb))
    f = hsmt.parse(inst.text)
    rng = np.random.default_rng(56)
    bsel = np.sort(rng.choice(d["n_bool"], 8, replace=False))
    rsel = np.sort(rng.choice(d["n_real"], 8, replace=False))
    bs, rs = set(bsel.tolist()), set(rsel.tolist())
    touch = [ci for ci, c in enumerate(f.constraints)
             if any((k == "b" and i in bs) or (k == "a" and any(j in rs for j, _ in f.atoms[i].coeffs))
                    for k, i in semantics.slots(c))]
    csel = np.sort(rng.choice(d["n_cons"], 5000, replace=False))
    for r in (0, 700):
        w = np.array([c.weight for c in f.constraints]) * 2.0 ** (U[:, r].astype(np.float64) + 0.5)
        _, oga, ogb = objective.objective_and_gradient_grouped(f, a[:, r], b[:, r], 1.0, w, subset=touch)
        check_gradient(np.concatenate([ga[bsel, r], gb[rsel, r]]), np.concatenate([oga[bsel], ogb[rsel]]),
                       scale_relative=True, what=f"place9856 r={r}")
        E = s.constraint_terms(1.0, r)
        _, _, _, terms = objective.objective_and_gradient_grouped(f, a[:, r], b[:, r], 1.0, subset=csel, want_terms=True)
        assert np.max(np.abs(E[csel] - np.array([terms[ci] for ci in csel]))) <= 1e-6
    x = np.where(a < 0, -1, 1).astype(np.int8)
    u, pc = s.verify_batch(x, b, per_con=True)
    sub = csel[:2000]
    for r in (0, 1023):
        want = np.array([0 if semantics.constraint_sat(f, f.constraints[ci], x[:, r], b[:, r]) else 1 for ci in sub])
        assert np.array_equal(pc[sub, r].astype(int), want)
