"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle on identical seeded inputs.

Rows of SURVEY §8(c)'s parity protocol: P2 (objective/gradient/E_c), P3 (step replay),
P4 (rounding), P5 (verification incl. corrupted models), P6 (ERWA counters), P7 (solve
soundness), P8-style restart-offset independence.  Bars: DESIGN.md §6.
"""
import math

import numpy as np
import pytest

import fsmt_gen
from fsmt_gen.points import random_points, random_counters
from oracle import hsmt, objective, semantics, solve as osolve
from tests.helpers import check_objective, check_gradient, subformula

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu_mod():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2603_22877_b200 as P
    return P


def make(P, text):
    s = P.Solver(0)
    s.load_formula(text)
    s.build_xbdd()
    return s


_PARSED = {}


def parsed(name):
    if name not in _PARSED:
        inst = fsmt_gen.config(name)
        _PARSED[name] = (inst, hsmt.parse(inst.text))
    return _PARSED[name]


def weights_of(f, U, r, t, mode=0):
    e = 0.0 if mode == 1 else max(t - 2, 0) / 2.0
    base = np.array([c.weight for c in f.constraints])
    if U is None:
        return base * 2.0 ** e
    return base * 2.0 ** (U[:, r].astype(np.float64) + e)


# ------------------------------------------------------------------------------------- K0

@pytest.mark.parametrize("name", ["cfg1", "cfg4s", "cfg3s"])
def test_k0_init_bit_exact(gpu_mod, name):
    inst, f = parsed(name)
    s = make(gpu_mod, inst.text)
    seed = 0x0123456789ABCDEF
    s.begin(40, seed, restart_offset=3)
    a, b = s.get_state()
    lo, hi = osolve.bounds(f)
    for r in (0, 1, 17, 39):
        oa, ob = osolve.init_point(f, seed, 3 + r, lo, hi)
        assert np.array_equal(a[:, r], oa.astype(np.float32))
        assert np.array_equal(b[:, r], ob.astype(np.float32))


# ------------------------------------------------------------------------------------- K1 (P2)

@pytest.mark.parametrize("name", ["cfg1", "cfg2s", "cfg3s", "cfg4s"])
@pytest.mark.parametrize("kappa", [0.0, 0.1, 1.0, 2.0])
def test_k1_objective_gradient_small(gpu_mod, name, kappa):
    inst, f = parsed(name)
    s = make(gpu_mod, inst.text)
    R = 70                                              # 3 restart tiles, ragged tail
    lo_b, hi_b = (0.0, 1.0) if name == "cfg4s" else (-1.0, 1.0)
    a, b = random_points(f.n_bool, f.n_real, R, seed=5, b_lo=lo_b, b_hi=hi_b)
    s.begin(R, 1)
    s.set_state(a, b)
    s.sweep(kappa, 1)
    obj, ga, gb = s.get_sweep()
    alpha = sum(c.weight for c in f.constraints)
    for r in (0, 31, 32, 69):
        C, oga, ogb = objective.objective_and_gradient(f, a[:, r], b[:, r], kappa)
        check_objective(obj[r], C, alpha, what=f"{name} r={r}")
        check_gradient(ga[:, r], oga, what=f"{name} grad_a r={r}")
        check_gradient(gb[:, r], ogb, what=f"{name} grad_b r={r}")


@pytest.mark.parametrize("name", ["cfg1", "cfg2s", "cfg4s"])
def test_k1_per_constraint_terms(gpu_mod, name):
    inst, f = parsed(name)
    s = make(gpu_mod, inst.text)
    R = 33
    a, b = random_points(f.n_bool, f.n_real, R, seed=9, b_lo=0.0, b_hi=1.0)
    s.begin(R, 1)
    s.set_state(a, b)
    for r in (0, 32):
        E = s.constraint_terms(1.3, r)
        _, _, _, terms = objective.objective_and_gradient(f, a[:, r], b[:, r], 1.3, want_terms=True)
        want = np.array([terms[i] for i in range(len(f.constraints))])
        assert np.all(np.isfinite(E)) and np.max(np.abs(E - want)) <= 1e-6
        assert np.all(np.abs(E) <= 1.0 + 1e-6)              # range lemma P:1620-1626


@pytest.mark.parametrize("name", ["cfg2s", "cfg4s"])
def test_k1_weighted_later_stage(gpu_mod, name):
    # ERWA weights w = w_c 2^(U + e_t) at stage t = 5 (R18); scale-relative gradient bar (R28)
    inst, f = parsed(name)
    s = make(gpu_mod, inst.text)
    R = 40
    a, b = random_points(f.n_bool, f.n_real, R, seed=11, b_lo=0.0, b_hi=1.0)
    U = random_counters(len(f.constraints), R, seed=12, max_u=4)
    s.begin(R, 1)
    s.set_state(a, b)
    s.set_counters(U)
    s.sweep(1.0, 5)
    obj, ga, gb = s.get_sweep()
    for r in (0, 39):
        w = weights_of(f, U, r, 5)
        C, oga, ogb = objective.objective_and_gradient(f, a[:, r], b[:, r], 1.0, w)
        check_objective(obj[r], C, float(w.sum()), what=name)
        check_gradient(np.concatenate([ga[:, r], gb[:, r]]), np.concatenate([oga, ogb]), scale_relative=True, what=name)


def test_k1_cfg2_full(gpu_mod):
    inst, f = parsed("cfg2")
    s = make(gpu_mod, inst.text)
    R = 1024
    a, b = random_points(f.n_bool, f.n_real, R, seed=3)
    s.begin(R, 2)
    s.set_state(a, b)
    for kappa in (0.1, 1.0, 2.0):
        s.sweep(kappa, 1)
        obj, ga, gb = s.get_sweep()
        for r in (0, 517, 1023):
            C, oga, ogb = objective.objective_and_gradient(f, a[:, r], b[:, r], kappa)
            check_objective(obj[r], C, 2000.0, what=f"cfg2 k={kappa} r={r}")
            check_gradient(ga[:, r], oga, what="cfg2 grad_a")
            check_gradient(gb[:, r], ogb, what="cfg2 grad_b")


@pytest.mark.parametrize("name,R", [("cfg3", 1024), ("cfg4", 1024)])
def test_k1_full_size_sampled(gpu_mod, name, R):
    """Full-size instance at the bench launch configuration; oracle on sampled outputs:
    per-constraint E_c for sampled constraints, gradients of sampled variables (all
    constraints touching them), objective via sum of the kernel's own E_c terms."""
    inst = fsmt_gen.config(name)
    s = make(gpu_mod, inst.text)
    s.prepare(R)                      # the kernels bench.py times (fsmt_prepare(R), DESIGN.md §7 item 11)
    assert f"prepared R={R}" in s.jit_info()["status"]
    d = s.get_dims()
    a, b = random_points(d["n_bool"], d["n_real"], R, seed=4, b_lo=0.0, b_hi=1.0)
    s.begin(R, 4)
    s.set_state(a, b)
    kappa = 1.0
    s.sweep(kappa, 1)
    obj, ga, gb = s.get_sweep()
    assert np.all(np.isfinite(obj)) and np.all(np.isfinite(ga)) and np.all(np.isfinite(gb))
    rng = np.random.default_rng(8)
    bsel = rng.choice(d["n_bool"], 2, replace=False)
    rsel = rng.choice(d["n_real"], 2, replace=False)
    csel = rng.choice(d["n_cons"], 40, replace=False)
    sub, keep = subformula(inst.text, bsel, rsel, extra_constraints=csel)
    fs = hsmt.parse(sub)
    for r in (0, R - 1):
        E = s.constraint_terms(kappa, r)
        # objective = sum of the kernel's terms (fp64), unit weights
        assert abs(obj[r] - math.fsum(E)) <= 1e-6 * d["n_cons"]
        C, oga, ogb, terms = objective.objective_and_gradient_grouped(fs, a[:, r], b[:, r], kappa, want_terms=True)
        idx = {orig: k for k, orig in enumerate(keep)}
        for ci in csel:
            assert abs(E[ci] - terms[idx[ci]]) <= 1e-6, f"E_c mismatch at c={ci}"
        check_gradient(ga[bsel, r], oga[bsel], what=f"{name} grad_a")
        check_gradient(gb[rsel, r], ogb[rsel], what=f"{name} grad_b")


@pytest.mark.parametrize("name,R", [("cfg3", 1024), ("cfg4", 1024)])
def test_k5_full_size_sampled(gpu_mod, name, R):
    """K5 (specialised check) at the bench launch configuration: per-constraint verdicts of
    sampled constraints for sampled restarts are bit-exact against the oracle's exact semantics
    (R22), and the unsat counts equal the per-constraint sums."""
    inst = fsmt_gen.config(name)
    s = make(gpu_mod, inst.text)
    s.prepare(R)                      # the kernels bench.py times
    d = s.get_dims()
    rng = np.random.default_rng(11)
    x = np.where(rng.random((d["n_bool"], R)) < 0.5, -1, 1).astype(np.int8)
    _, y = random_points(0, d["n_real"], R, seed=12, b_lo=0.0, b_hi=1.0)
    unsat, pc = s.verify_batch(x, y, per_con=True)
    assert np.array_equal(unsat.astype(np.int64), pc.sum(axis=0).astype(np.int64))
    csel = np.sort(rng.choice(d["n_cons"], 3000, replace=False))
    sub, keep = subformula(inst.text, extra_constraints=csel)
    fs = hsmt.parse(sub)
    for r in (0, 517, R - 1):
        want = np.array([0 if semantics.constraint_sat(fs, c, x[:, r], y[:, r]) else 1 for c in fs.constraints])
        assert np.array_equal(pc[keep, r].astype(int), want), r


# ------------------------------------------------------------------------------------- K3 (P3)

@pytest.mark.parametrize("name", ["cfg1", "cfg4s", "cfg3s"])
def test_k3_step_replay(gpu_mod, name):
    inst, f = parsed(name)
    s = make(gpu_mod, inst.text)
    R = 36
    s.begin(R, 77)
    lo, hi = osolve.bounds(f)
    eta, eps, kappa = 0.02, 1e-2, 1.5
    for step in range(3):
        a, b = s.get_state()
        s.sweep(kappa, 1)
        gm2 = s.update(eta, eps, want_gm2=True)
        a2, b2 = s.get_state()
        for r in (0, 35):
            oa, ob, ogm2, _ = osolve.pgd_step(f, a[:, r].astype(np.float64), b[:, r].astype(np.float64),
                                              kappa, None, eta, lo, hi)
            frozen = ogm2 <= eps * eps
            assert abs(gm2[r] - ogm2) <= 1e-4 * max(ogm2, 1e-6)
            if not frozen:
                assert np.max(np.abs(a2[:, r] - oa)) <= eta * 1e-5 + 1e-7
                assert np.max(np.abs(b2[:, r] - ob)) <= eta * 1e-5 + 1e-7
            else:
                assert np.array_equal(a2[:, r], a[:, r]) and np.array_equal(b2[:, r], b[:, r])
            assert np.all(a2[:, r] >= -1) and np.all(a2[:, r] <= 1)
            assert np.all(b2[:, r] >= lo) and np.all(b2[:, r] <= hi)


# ------------------------------------------------------------------------------------- K4/K5 (P4-P6)

@pytest.mark.parametrize("rounding", [0, 1])
def test_k4_rounding_bit_exact(gpu_mod, rounding):
    inst, f = parsed("cfg4s")
    s = make(gpu_mod, inst.text)
    s.set_params(rounding=rounding)
    R = 48
    seed = 4242
    s.begin(R, seed, restart_offset=5)
    a = np.random.default_rng(1).uniform(-1, 1, (f.n_bool, R)).astype(np.float32)
    a[0, :4] = [0.0, -0.0, 1.0, -1.0]
    _, b = s.get_state()
    s.set_state(a, b)
    s.stage_end(3)
    x = s.get_rounded()
    for r in range(R):
        want = osolve.round_sign(a[:, r]) if rounding == 0 else osolve.round_philox(a[:, r], seed, 5 + r, 3)
        assert np.array_equal(x[:, r], want)


@pytest.mark.parametrize("name", ["cfg1", "cfg2s", "cfg3s", "cfg4s"])
def test_k5_verify_bit_exact_with_corruptions(gpu_mod, name):
    inst, f = parsed(name)
    s = make(gpu_mod, inst.text)
    rng = np.random.default_rng(2)
    R = 100
    X = np.repeat(inst.x_star[:, None], R, axis=1).copy()
    Y = np.repeat(inst.y_star[:, None], R, axis=1).copy()
    for r in range(1, R):                       # 99 deliberately corrupted models
        if r % 2:
            X[rng.integers(0, f.n_bool), r] *= -1
        else:
            j = rng.integers(0, f.n_real)
            Y[j, r] = np.float32(Y[j, r] + rng.choice([-1, 1]) * rng.uniform(0.01, 0.5))
    u, pc = s.verify_batch(X, Y, per_con=True)
    assert u[0] == 0
    for r in range(R):
        want = osolve.violations(f, X[:, r], Y[:, r])
        assert np.array_equal(pc[:, r].astype(np.int64), want) and u[r] == want.sum()


def test_k5_erwa_counters_and_weights(gpu_mod):
    inst, f = parsed("cfg2s")
    s = make(gpu_mod, inst.text)
    R = 8
    s.begin(R, 3)
    T = 5
    acc = np.zeros((len(f.constraints), R), dtype=np.int64)
    for t in range(1, T + 1):
        a, b = random_points(f.n_bool, f.n_real, R, seed=100 + t)
        s.set_state(a, b)
        unsat = s.stage_end(t)
        for r in range(R):
            u = osolve.violations(f, osolve.round_sign(a[:, r]), b[:, r])
            acc[:, r] += u
            assert unsat[r] == u.sum()
    U = s.get_counters()
    assert np.array_equal(U.astype(np.int64), acc)
    # the weight the kernel uses in stage T+1 equals Alg.2 run literally on the same u sequence
    h = np.zeros(len(f.constraints))
    w = np.ones(len(f.constraints))
    # replay the per-stage u's: acc is the sum; rebuild sequence by re-evaluating
    seqs = []
    for t in range(1, T + 1):
        a, b = random_points(f.n_bool, f.n_real, R, seed=100 + t)
        seqs.append(osolve.violations(f, osolve.round_sign(a[:, 0]), b[:, 0]))
    for t, u in enumerate(seqs, start=1):
        h = osolve.RHO * h + u
        w = w * osolve.GAMMA ** h
        h[:] = 1.0
    assert np.allclose(weights_of(f, U, 0, T + 1), w, rtol=1e-12)


# ------------------------------------------------------------------------------------- solve (P7)

def test_solve_cfg1_sat_and_sound(gpu_mod):
    inst, f = parsed("cfg1")
    s = make(gpu_mod, inst.text)
    s.set_params(eta=0.1)
    for seed in range(4):
        res = s.solve(64, 30, seed)
        assert res.verdict == gpu_mod.SAT
        _, sat = semantics.eval_formula(f, res.x, res.y)
        assert all(sat) and res.stats["host_verified"] == 1


def test_solve_unsat_is_unknown(gpu_mod):
    s = make(gpu_mod, "p hsmt 1 1\na 0 <= 0 0:1\nc or 1 +b0\nc or 1 -b0\nc or 1 +a0\n")
    s.set_params(kappas=[0.5, 1.0, 2.0], eta=0.1)
    res = s.solve(32, 10, 5)
    assert res.verdict == gpu_mod.UNKNOWN and res.stats["best_unsat"] >= 1


@pytest.mark.parametrize("name", ["cfg3s", "cfg4s", "cfg2s"])
def test_solve_structured_small_sound(gpu_mod, name):
    inst, f = parsed(name)
    s = make(gpu_mod, inst.text)
    s.set_params(eta=0.02)
    res = s.solve(256, 40, 11)
    _, sat = semantics.eval_formula(f, res.x, res.y)
    if res.verdict == gpu_mod.SAT:
        assert all(sat)
    else:
        assert sum(not v for v in sat) == res.stats["best_unsat"]


# ------------------------------------------------------------------------------------- P8-style

def test_restart_offset_independence(gpu_mod):
    inst, f = parsed("cfg4s")
    full = make(gpu_mod, inst.text)
    half = make(gpu_mod, inst.text)
    full.begin(64, 99, 0)
    half.begin(32, 99, 32)
    af, bf = full.get_state()
    ah, bh = half.get_state()
    assert np.array_equal(af[:, 32:], ah) and np.array_equal(bf[:, 32:], bh)
    for t in (1, 2, 3):                      # bit-exact (exact on-grid sums, DESIGN.md §7 item 14)
        for k in range(3):
            full.sweep(1.0, t)
            half.sweep(1.0, t)
            of, gaf, gbf = full.get_sweep()
            oh, gah, gbh = half.get_sweep()
            assert np.array_equal(of[32:], oh)
            assert np.array_equal(gaf[:, 32:], gah) and np.array_equal(gbf[:, 32:], gbh)
            full.update(0.02, 1e-2)
            half.update(0.02, 1e-2)
        uf = full.stage_end(t)
        uh = half.stage_end(t)
        assert np.array_equal(uf[32:], uh)
        af, bf = full.get_state()
        ah, bh = half.get_state()
        assert np.array_equal(af[:, 32:], ah) and np.array_equal(bf[:, 32:], bh)
    assert np.array_equal(full.get_counters()[:, 32:], half.get_counters())


# ------------------------------------------------------------------------------------- JIT path

@pytest.mark.parametrize("name", ["cfg3s", "cfg4s"])
def test_jit_active_and_matches_generic(gpu_mod, name, monkeypatch):
    """The JIT-specialised sweep is the one that runs, and it agrees with the generic kernel."""
    inst, f = parsed(name)
    jit = make(gpu_mod, inst.text)
    info = jit.jit_info()
    assert info["status"] == "active" and info["jit_cons"] > 0, info
    monkeypatch.setenv("FSMT_JIT", "0")
    gen = make(gpu_mod, inst.text)
    assert gen.jit_info()["jit_cons"] == 0
    R = 96
    a, b = random_points(f.n_bool, f.n_real, R, seed=31, b_lo=0.0, b_hi=1.0)
    U = random_counters(len(f.constraints), R, seed=32, max_u=3)
    outs = []
    for s in (jit, gen):
        s.begin(R, 5)
        s.set_state(a, b)
        s.set_counters(U)
        assert np.array_equal(s.get_counters(), U)
        s.sweep(1.3, 4)
        outs.append(s.get_sweep())
        E = s.constraint_terms(1.3, 7)
        outs.append((E,))
    (oj, gaj, gbj), (Ej,), (og, gag, gbg), (Eg,) = outs
    assert np.allclose(oj, og, rtol=1e-6, atol=1e-6)
    # weighted (U <= 3, stage 4): scale-relative bar of reading R28
    for gj, gg in ((gaj, gag), (gbj, gbg)):
        assert np.max(np.abs(gj - gg)) <= 1e-5 * max(1.0, float(np.max(np.abs(gg))))
    assert np.max(np.abs(Ej - Eg)) <= 1e-6


@pytest.mark.parametrize("name", ["cfg3s", "cfg4s"])
def test_fsmt_eval_one_call(gpu_mod, name):
    """fsmt_eval (SURVEY §8(b)'s one-call hook) equals set_state + set_counters + sweep + get_sweep
    on the same context and matches the oracle, with and without ERWA counters."""
    inst, f = parsed(name)
    s = make(gpu_mod, inst.text)
    R = 40
    a, b = random_points(f.n_bool, f.n_real, R, seed=31, b_lo=0.0, b_hi=1.0)
    obj, ga, gb = s.eval(a, b, 1.1)
    for r in (0, R - 1):
        C, oga, ogb = objective.objective_and_gradient(f, a[:, r], b[:, r], 1.1)
        check_objective(obj[r], C, float(sum(c.weight for c in f.constraints)), what=f"{name} eval")
        check_gradient(ga[:, r], oga, what=f"{name} eval grad_a")
        check_gradient(gb[:, r], ogb, what=f"{name} eval grad_b")
    rng = np.random.default_rng(2)
    U = rng.integers(0, 4, size=(len(f.constraints), R), dtype=np.uint8)
    obj2, ga2, gb2 = s.eval(a, b, 0.9, U=U, stage_t=5)
    s.set_state(a, b)
    s.set_counters(U)
    s.sweep(0.9, 5)
    o3, g3a, g3b = s.get_sweep()
    np.testing.assert_allclose(obj2, o3, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(ga2, g3a, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(gb2, g3b, rtol=1e-12, atol=1e-12)
    for r in (0, R - 1):
        w = weights_of(f, U, r, 5)
        C, oga, ogb = objective.objective_and_gradient(f, a[:, r], b[:, r], 0.9, w)
        check_objective(obj2[r], C, float(w.sum()), what=f"{name} eval weighted")
        check_gradient(np.concatenate([ga2[:, r], gb2[:, r]]), np.concatenate([oga, ogb]), scale_relative=True,
                       what=f"{name} eval weighted")
