"""The paper's random hybrid family (generator fsmt_gen.paper_random, reading R36) at every
n in {100, ..., 1000}: every constraint's E_c and the objective and gradient of sampled restarts
against the fp64 oracle (its O3 Poisson-binomial path for the long symmetric constraints).  CARD
classes beyond the register budget of their xBDD (CARD(50, 25): 650 nodes) run as count classes
(the O((n+k)^2) count-distribution COP of P:254, DESIGN.md §7 item 15); FSMT_JIT_COUNT=1 forces the
count form on the CARD(20, 10) classes of n = 100 as well, and both forms must match the oracle and
each other."""
import os

import numpy as np
import pytest

import fsmt_gen
from fsmt_gen.points import random_points, random_counters
from oracle import hsmt, objective, semantics
from tests.helpers import check_gradient, check_objective

pytestmark = pytest.mark.gpu


def _solver(P, text, env=None):
    env = env or {}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        s = P.Solver(0)
        s.load_formula(text)
        s.build_xbdd()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return s


@pytest.mark.parametrize("n", list(range(100, 1001, 100)))
def test_random_family_parity(n):
    import paper_2603_22877_b200 as P
    inst = fsmt_gen.config(f"rand{n}")
    f = hsmt.parse(inst.text)
    s = _solver(P, inst.text)
    info = s.jit_info()
    # every symmetric constraint runs in a JIT class (xBDD or count form); a constraint that repeats
    # a variable is not symmetric over distinct slots (R5) and may take the generic kernel
    assert info["status"] == "active" and info["jit_cons"] >= len(f.constraints) - 2, info
    R = 64
    Ls = np.array([len(semantics.slots(c)) for c in f.constraints], dtype=np.float64)
    a, b = random_points(f.n_bool, f.n_real, R, seed=n + 1)
    U = random_counters(len(f.constraints), R, seed=n + 2, max_u=3)
    s.begin(R, 3)
    s.set_state(a, b)
    s.set_counters(U)
    for kappa, t in ((0.5, 1), (1.0, 4)):
        s.sweep(kappa, t)
        obj, ga, gb = s.get_sweep()
        for r in (0, 37, 63):
            E = s.constraint_terms(kappa, r)
            w = np.array([c.weight for c in f.constraints]) * 2.0 ** (U[:, r].astype(np.float64) + max(t - 2, 0) / 2.0)
            C, oga, ogb, terms = objective.objective_and_gradient_grouped(f, a[:, r], b[:, r], kappa, w, want_terms=True)
            oE = np.array([terms[i] for i in range(len(f.constraints))])
            # E_c bar: 1e-6, or the fp32 bound of an L-literal pass, 2 L 2^-23 (= 1.2e-5
            # at L = 50: each of the L DP / message steps rounds values <= 1 twice; E = 1 - 2 COP)
            bar = np.maximum(1e-6, 2.0 * Ls * 2.0 ** -23)
            assert np.all(np.isfinite(E)) and np.all(np.abs(E - oE) <= bar), (n, kappa, r, np.max(np.abs(E - oE) / bar))
            check_objective(obj[r], C, float(w.sum()), what=f"rand{n} kappa={kappa} r={r}")
            check_gradient(np.concatenate([ga[:, r], gb[:, r]]), np.concatenate([oga, ogb]), scale_relative=True,
                           what=f"rand{n} kappa={kappa} r={r}")
    # K5: the count classes' exact check counts true literals
    x = np.where(np.random.default_rng(n).random((f.n_bool, R)) < 0.5, -1, 1).astype(np.int8)
    u, pc = s.verify_batch(x, b, per_con=True)
    for r in (0, 63):
        want = np.array([0 if semantics.constraint_sat(f, c, x[:, r], b[:, r]) else 1 for c in f.constraints])
        assert np.array_equal(pc[:, r].astype(int), want) and u[r] == want.sum()


def test_count_form_matches_xbdd_form_cfg2_and_rand100():
    """CARD(20, 10): the 110-node xBDD class (default) and the count class (FSMT_JIT_COUNT=1) agree
    (fp32 rounding) and both match the oracle."""
    import paper_2603_22877_b200 as P
    for name in ("rand100", "cfg2"):
        inst = fsmt_gen.config(name)
        f = hsmt.parse(inst.text)
        xb = _solver(P, inst.text)
        ct = _solver(P, inst.text, {"FSMT_JIT_COUNT": "1"})
        assert "cq0" in ct.jit_source() and "cq0" not in xb.jit_source()
        R = 40
        a, b = random_points(f.n_bool, f.n_real, R, seed=9)
        out = []
        for s in (xb, ct):
            s.begin(R, 1)
            s.set_state(a, b)
            s.sweep(1.3, 1)
            out.append(s.get_sweep())
        for A, B in zip(out[0], out[1]):
            np.testing.assert_allclose(B, A, rtol=1e-5, atol=2e-6)
        for r in (0, R - 1):
            C, oga, ogb = objective.objective_and_gradient_grouped(f, a[:, r], b[:, r], 1.3)
            check_objective(out[1][0][r], C, float(len(f.constraints)), what=f"{name} count")
            check_gradient(out[1][1][:, r], oga, what=f"{name} count grad_a")
            check_gradient(out[1][2][:, r], ogb, what=f"{name} count grad_b")


def test_product_form_matches_xbdd_form_cfg2_and_rand100():
    """OR / NAE / XOR over symmetric literals: the closed-form product classes (default, DESIGN.md
    §7 item 15) and their xBDD classes (FSMT_JIT_PROD=0) agree (fp32 rounding) and both match the
    oracle, with live ERWA counters at t = 4."""
    import paper_2603_22877_b200 as P
    for name in ("rand100", "cfg2"):
        inst = fsmt_gen.config(name)
        f = hsmt.parse(inst.text)
        pr = _solver(P, inst.text)
        xb = _solver(P, inst.text, {"FSMT_JIT_PROD": "0"})
        R = 40
        a, b = random_points(f.n_bool, f.n_real, R, seed=19)
        U = random_counters(len(f.constraints), R, seed=20, max_u=3)
        out = []
        for s in (pr, xb):
            s.begin(R, 1)
            s.set_state(a, b)
            s.set_counters(U)
            s.sweep(0.8, 4)
            out.append(s.get_sweep())
        for A, B in zip(out[0], out[1]):
            np.testing.assert_allclose(A, B, rtol=1e-5, atol=2e-6 * float(np.max(np.abs(B)) or 1.0))
        for r in (0, R - 1):
            w = np.array([c.weight for c in f.constraints]) * 2.0 ** (U[:, r].astype(np.float64) + 1.0)
            C, oga, ogb = objective.objective_and_gradient_grouped(f, a[:, r], b[:, r], 0.8, w)
            for k, (obj, ga, gb) in enumerate(out):
                what = f"{name} {'product' if k == 0 else 'xbdd'} r={r}"
                check_objective(obj[r], C, float(w.sum()), what=what)
                check_gradient(np.concatenate([ga[:, r], gb[:, r]]), np.concatenate([oga, ogb]), scale_relative=True,
                               what=what)


@pytest.mark.parametrize("n", [100, 300])
def test_random_family_solves(n):
    """Alg.2 end to end on the paper's random family: the time-to-SAT recipe of the
    bench (eta 0.4, eta_mode 3, reset-to-0 ERWA, kappa 1 -> 300 geometric then held) reaches SAT
    within its schedule, and the returned model satisfies every constraint under the oracle's
    exact semantics (Thm.1: a rounded model with no violated constraint is a witness)."""
    import paper_2603_22877_b200 as P
    inst = fsmt_gen.config(f"rand{n}")
    f = hsmt.parse(inst.text)
    s = P.Solver(0)
    s.load_formula(inst.text)
    s.build_xbdd()
    kappas = [300.0 ** (i / 19) for i in range(20)] + [300.0] * 200
    s.set_params(kappas=kappas, eta=0.4, eta_mode=3, erwa_mode=1)
    res = s.solve(1024, 2, 0)
    assert res.verdict == P.SAT
    assert all(semantics.eval_formula(f, res.x, res.y)[1])
