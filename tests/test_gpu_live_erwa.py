"""Parity of the benchmarked module with live ERWA state (VERDICT r1 "next" item 1; SURVEY §8(c) P2
with the weights of Alg.2, R18), and the weight range (R18 at long schedules).

cfg4m is a mid-size placement instance (60 modules, 2,010 constraints) with cfg4's REAL kernel class:
n_m = 32, n_l = 4, so the non-overlap constraint has 7 bit pairs, 25 nodes, 18 slots (the 7-bit
affine groups, aliases, atom pairs and diamonds of the hot kernel).  Every constraint's E_c and every
variable's gradient are compared with the fp64 oracle at 4 restarts spanning 2 warps, for kappa in
{0.1, 1, 2, 10}, stage t in {1, 5, 20} and both ERWA readings, with random counters U in [0, 6]; the
three modules (build-time JIT, U prefetched 3 constraints ahead, fsmt_prepare(R)) must agree bit for
bit (identical per-term arithmetic, exact sums).  Then full cfg4 with fsmt_prepare(1024) (the module
bench.py times) after set_counters at t = 5: 20,000 sampled E_c, 64 variables' gradients, and the hot
kernel's objective for one restart against the oracle's sum over all 705,072 constraints."""
import math
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest

import fsmt_gen
from fsmt_gen.points import random_points, random_counters
from oracle import hsmt, objective
from tests.helpers import check_gradient, check_objective, subformula

pytestmark = pytest.mark.gpu

KAPPAS = (0.1, 1.0, 2.0, 10.0)
STAGES = (1, 5, 20)
MODES = (0, 1)
RESTARTS = (0, 31, 32, 63)
R = 64


def weights(f, U, r, t, mode):
    e = 0.0 if mode == 1 else max(t - 2, 0) / 2.0
    return np.array([c.weight for c in f.constraints]) * 2.0 ** (U[:, r].astype(np.float64) + e)


_F = {}


def _oracle_job(args):
    name, kappa, t, mode, r, a, b, U = args
    if name not in _F:
        _F[name] = hsmt.parse(fsmt_gen.config(name).text)
    f = _F[name]
    C, ga, gb, terms = objective.objective_and_gradient_grouped(f, a, b, kappa, weights(f, U, r, t, mode),
                                                                want_terms=True)
    return (kappa, t, mode, r), (C, ga, gb, np.array([terms[i] for i in range(len(f.constraints))]))


_CASE = {}


def cfg4m_case():
    """Point, counters and oracle values of every (kappa, t, mode, restart) combination (cached)."""
    if not _CASE:
        inst = fsmt_gen.config("cfg4m")
        f = hsmt.parse(inst.text)
        a, b = random_points(f.n_bool, f.n_real, R, seed=61, b_lo=0.0, b_hi=1.0)
        U = random_counters(len(f.constraints), R, seed=62, max_u=6)
        jobs = [("cfg4m", k, t, m, r, a[:, r].astype(np.float64), b[:, r].astype(np.float64), U)
                for k in KAPPAS for t in STAGES for m in MODES for r in RESTARTS]
        with ProcessPoolExecutor(max_workers=max(1, min(32, os.cpu_count() or 1))) as ex:
            orc = dict(ex.map(_oracle_job, jobs))
        _CASE.update(inst=inst, f=f, a=a, b=b, U=U, orc=orc)
    return _CASE


def _solver(P, text, env=None, prepare=0):
    env = env or {}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        s = P.Solver(0)
        s.load_formula(text)
        s.build_xbdd()
        if prepare:
            s.prepare(prepare)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return s


def test_cfg4m_live_erwa_matrix():
    import paper_2603_22877_b200 as P
    c = cfg4m_case()
    inst, f, a, b, U, orc = c["inst"], c["f"], c["a"], c["b"], c["U"], c["orc"]
    modules = {"jit": _solver(P, inst.text), "upf3": _solver(P, inst.text, {"FSMT_JIT_UPF": "3"}),
               "prepared": _solver(P, inst.text, prepare=R)}
    assert modules["prepared"].jit_info()["status"].startswith("active; prepared R=64")
    assert "fsmt_w(" in modules["upf3"].jit_source() and "un2" in modules["upf3"].jit_source()   # prefetch ring
    # the real cfg4 class: 7 bit pairs + 4 atoms (18 slots, 25 nodes)
    assert modules["jit"].get_dims()["max_slots"] == 18 and modules["jit"].get_dims()["max_nodes"] == 25
    for s in modules.values():
        s.set_params(erwa_mode=0)
    out = {}
    for name, s in modules.items():
        for mode in MODES:
            s.set_params(erwa_mode=mode)
            s.begin(R, 5)
            s.set_state(a, b)
            s.set_counters(U)
            for kappa in KAPPAS:
                for t in STAGES:
                    s.sweep(kappa, t)
                    out[(name, kappa, t, mode)] = s.get_sweep()
                E = {r: s.constraint_terms(kappa, r) for r in RESTARTS}
                out[(name, kappa, "E", mode)] = E
    for key, val in out.items():                       # the three modules agree bit for bit
        if key[0] == "jit":
            for other in ("upf3", "prepared"):
                oth = out[(other,) + key[1:]]
                if key[2] == "E":
                    assert all(np.array_equal(val[r], oth[r]) for r in RESTARTS), (other, key)
                else:
                    assert all(np.array_equal(x, y) for x, y in zip(val, oth)), (other, key)
    for kappa in KAPPAS:
        for t in STAGES:
            for mode in MODES:
                obj, ga, gb = out[("prepared", kappa, t, mode)]
                E = out[("prepared", kappa, "E", mode)]
                for r in RESTARTS:
                    C, oga, ogb, oE = orc[(kappa, t, mode, r)]
                    w = weights(f, U, r, t, mode)
                    what = f"cfg4m kappa={kappa} t={t} mode={mode} r={r}"
                    assert np.all(np.isfinite(E[r])) and np.max(np.abs(E[r] - oE)) <= 1e-6, what
                    check_objective(obj[r], C, float(w.sum()), what=what)
                    check_gradient(np.concatenate([ga[:, r], gb[:, r]]), np.concatenate([oga, ogb]),
                                   scale_relative=True, what=what)


_FULL = {}


def _chunk_objective(args):
    lo, hi, a, b, kappa, w = args
    return objective.objective_and_gradient_grouped(_FULL["f"], a, b, kappa, w, subset=range(lo, hi))[0]


def test_cfg4_full_prepared_live_erwa():
    """The exact module bench.py times: cfg4, fsmt_prepare(1024) (U prefetched 3 ahead, R compiled
    in, register cap), counters U ~ [0, 6] at stage t = 5 (verbatim ERWA: w = 2^(U + 1.5))."""
    import multiprocessing as mp
    import paper_2603_22877_b200 as P
    from oracle import semantics
    inst = fsmt_gen.config("cfg4")
    Rf, t, kappa = 1024, 5, 1.0
    s = _solver(P, inst.text, prepare=Rf)
    assert s.jit_info()["status"].startswith("active; prepared R=1024")
    d = s.get_dims()
    a, b = random_points(d["n_bool"], d["n_real"], Rf, seed=71, b_lo=0.0, b_hi=1.0)
    U = random_counters(d["n_cons"], Rf, seed=72, max_u=6)
    s.begin(Rf, 7)
    s.set_state(a, b)
    s.set_counters(U)
    s.sweep(kappa, t)
    obj, ga, gb = s.get_sweep()
    assert np.all(np.isfinite(obj)) and np.all(np.isfinite(ga)) and np.all(np.isfinite(gb))
    f = _FULL.setdefault("f", hsmt.parse(inst.text))
    W = lambda r: np.array([c.weight for c in f.constraints]) * 2.0 ** (U[:, r].astype(np.float64) + 1.5)
    rng = np.random.default_rng(73)
    bsel = np.sort(rng.choice(d["n_bool"], 32, replace=False))
    rsel = np.sort(rng.choice(d["n_real"], 32, replace=False))
    csel = np.sort(rng.choice(d["n_cons"], 20000, replace=False))
    # (1) 20,000 sampled E_c (per-constraint hook) at two restarts
    for r in (3, Rf - 1):
        E = s.constraint_terms(kappa, r)
        _, _, _, terms = objective.objective_and_gradient_grouped(f, a[:, r], b[:, r], kappa, subset=csel,
                                                                  want_terms=True)
        assert np.max(np.abs(E[csel] - np.array([terms[ci] for ci in csel]))) <= 1e-6
    # (2) gradients of 64 variables (every constraint touching them), hot kernel, live weights
    bs, rs = set(bsel.tolist()), set(rsel.tolist())
    touch = [ci for ci, c in enumerate(f.constraints)
             if any((k == "b" and i in bs) or (k == "a" and any(j in rs for j, _ in f.atoms[i].coeffs))
                    for k, i in semantics.slots(c))]
    for r in (3, 517):
        _, oga, ogb = objective.objective_and_gradient_grouped(f, a[:, r], b[:, r], kappa, W(r), subset=touch)
        check_gradient(np.concatenate([ga[bsel, r], gb[rsel, r]]), np.concatenate([oga[bsel], ogb[rsel]]),
                       scale_relative=True, what=f"cfg4 prepared grads r={r}")
    # (3) the hot kernel's objective for one restart vs the oracle over all 705,072 constraints
    r = 517
    w = W(r)
    edges = np.linspace(0, d["n_cons"], 97).astype(int)
    jobs = [(int(lo), int(hi), a[:, r].astype(np.float64), b[:, r].astype(np.float64), kappa, w)
            for lo, hi in zip(edges[:-1], edges[1:])]
    with ProcessPoolExecutor(max_workers=max(1, min(96, os.cpu_count() or 1)), mp_context=mp.get_context("fork")) as ex:
        parts = list(ex.map(_chunk_objective, jobs))
    check_objective(obj[r], math.fsum(parts), float(w.sum()), what="cfg4 prepared objective, all constraints")


# ------------------------------------------------------------------------------ ERWA weight range


@pytest.mark.parametrize("t", [258, 300])
@pytest.mark.parametrize("mode", [0, 1])
def test_erwa_weights_beyond_fp32_range(t, mode):
    """R18 weights w = 2^(U + e_t) with U in {0, 127, 128, 255} and t in {258, 300} (e_t up to 149):
    far beyond fp32 (2^128); the sweep stays finite and matches the fp64 oracle (scale-relative bar,
    R28) in both ERWA readings."""
    import paper_2603_22877_b200 as P
    inst = fsmt_gen.config("cfg4s")
    f = hsmt.parse(inst.text)
    s = _solver(P, inst.text)
    s.set_params(erwa_mode=mode)
    Rr = 40
    a, b = random_points(f.n_bool, f.n_real, Rr, seed=81, b_lo=0.0, b_hi=1.0)
    rng = np.random.default_rng(82)
    U = rng.choice(np.array([0, 127, 128, 255], dtype=np.uint8), size=(len(f.constraints), Rr))
    U[:, 5] = 0                                      # a restart with unit counters
    U[:, 6] = 255                                    # and one with every counter saturated-high
    s.begin(Rr, 3)
    s.set_state(a, b)
    s.set_counters(U)
    s.sweep(1.3, t)
    obj, ga, gb = s.get_sweep()
    assert np.all(np.isfinite(obj)) and np.all(np.isfinite(ga)) and np.all(np.isfinite(gb))
    for r in (0, 5, 6, 39):
        w = weights(f, U, r, t, mode)
        C, oga, ogb = objective.objective_and_gradient(f, a[:, r], b[:, r], 1.3, w)
        check_objective(obj[r], C, float(w.sum()), what=f"t={t} mode={mode} r={r}")
        check_gradient(np.concatenate([ga[:, r], gb[:, r]]), np.concatenate([oga, ogb]), scale_relative=True,
                       what=f"t={t} mode={mode} r={r}")


def test_erwa_300_stages_verbatim_at_the_witness():
    """300 verbatim stages (e_t = 149 at t = 300) at the planted witness: no violations, so U stays 0
    and the weights are 2^149 (old fp32 weights overflowed at t = 258); the sweep at t = 300 is
    finite and matches the oracle; then a 300-stage schedule solve completes."""
    import paper_2603_22877_b200 as P
    inst = fsmt_gen.config("cfg4s")
    f = hsmt.parse(inst.text)
    s = _solver(P, inst.text)
    Rr = 8
    s.begin(Rr, 1)
    a = np.repeat(inst.x_star[:, None].astype(np.float32), Rr, axis=1)
    b = np.repeat(inst.y_star[:, None], Rr, axis=1)
    s.set_state(a, b)
    for t in range(1, 301):
        u = s.stage_end(t)
        assert not u.any()
    assert not s.get_counters().any()
    s.sweep(2.0, 300)
    obj, ga, gb = s.get_sweep()
    assert np.all(np.isfinite(obj)) and np.all(np.isfinite(ga)) and np.all(np.isfinite(gb))
    w = weights(f, np.zeros((len(f.constraints), 1), dtype=np.uint8), 0, 300, 0)
    C, oga, ogb = objective.objective_and_gradient(f, a[:, 0], b[:, 0], 2.0, w)
    check_objective(obj[0], C, float(w.sum()))
    check_gradient(np.concatenate([ga[:, 0], gb[:, 0]]), np.concatenate([oga, ogb]), scale_relative=True)
    s.set_params(kappas=[1.0] * 300, eta=0.05)
    res = s.solve(64, 4, 3)
    assert res.verdict in (P.SAT, P.UNKNOWN)
    assert np.all(np.isfinite(res.y))


def test_erwa_counter_overflow_is_reported():
    """U is a u16 count of violations (R18); the 65536th violation of a constraint in a restart is
    reported as FSMT_ERR_RANGE (the counter is held at 65535), never silently saturated.  A sweep whose
    weights 2^(U + e_t) leave the fp64 range (U = 1000 here) is reported the same way."""
    import paper_2603_22877_b200 as P
    from paper_2603_22877_b200 import native as N
    inst = fsmt_gen.config("cfg4s")
    f = hsmt.parse(inst.text)
    s = _solver(P, inst.text)
    Rr = 8
    s.begin(Rr, 1)
    a, b = random_points(f.n_bool, f.n_real, Rr, seed=5, b_lo=0.0, b_hi=1.0)
    s.set_state(a, b)
    U = np.full((len(f.constraints), Rr), 65534, dtype=np.uint16)
    s.set_counters(U)
    u1 = s.stage_end(1)                               # 65534 -> 65535: fine
    assert u1.sum() > 0
    with pytest.raises(P.FsmtError) as ei:
        s.stage_end(2)                                # 65535 -> 65536: reported
    assert ei.value.status == N.ERR_RANGE
    assert s.get_counters().max() == 65535
    s2 = _solver(P, inst.text)
    s2.begin(Rr, 1)
    s2.set_state(a, b)
    s2.set_counters(np.full((len(f.constraints), Rr), 1000, dtype=np.uint16))
    s2.sweep(1.0, 1)
    with pytest.raises(P.FsmtError) as ei:
        s2.get_sweep()
    assert ei.value.status == N.ERR_RANGE


def test_cfg4_large_r_sampled():
    """SURVEY §8(d) config 5 scale: cfg4 at R = 16,384 restarts (U 23 GB, state 0.7 GB: beyond the
    L2, so the stream values come from HBM) with the kernels fsmt_prepare(16384) builds; the K0 init
    point of sampled restarts in three different warps and restart blocks, sampled variables'
    gradients and E_c against the oracle."""
    import paper_2603_22877_b200 as P
    inst = fsmt_gen.config("cfg4")
    Rl, kappa = 16384, 1.0
    s = _solver(P, inst.text, prepare=Rl)
    assert s.jit_info()["status"].startswith("active; prepared R=16384")
    d = s.get_dims()
    s.begin(Rl, 11)
    s.sweep(kappa, 1)
    obj, ga, gb = s.get_sweep()
    a, b = s.get_state()
    assert np.all(np.isfinite(obj)) and np.all(np.isfinite(ga)) and np.all(np.isfinite(gb))
    f = _FULL.setdefault("f", hsmt.parse(inst.text))
    from oracle import semantics
    rng = np.random.default_rng(91)
    bsel = np.sort(rng.choice(d["n_bool"], 8, replace=False))
    rsel = np.sort(rng.choice(d["n_real"], 8, replace=False))
    bs, rs = set(bsel.tolist()), set(rsel.tolist())
    touch = [ci for ci, c in enumerate(f.constraints)
             if any((k == "b" and i in bs) or (k == "a" and any(j in rs for j, _ in f.atoms[i].coeffs))
                    for k, i in semantics.slots(c))]
    csel = np.sort(rng.choice(d["n_cons"], 4000, replace=False))
    for r in (5, 8191, Rl - 1):
        _, oga, ogb = objective.objective_and_gradient_grouped(f, a[:, r], b[:, r], kappa, subset=touch)
        check_gradient(ga[bsel, r], oga[bsel], what=f"R=16384 grad_a r={r}")
        check_gradient(gb[rsel, r], ogb[rsel], what=f"R=16384 grad_b r={r}")
        E = s.constraint_terms(kappa, r)
        _, _, _, terms = objective.objective_and_gradient_grouped(f, a[:, r], b[:, r], kappa, subset=csel,
                                                                  want_terms=True)
        assert np.max(np.abs(E[csel] - np.array([terms[ci] for ci in csel]))) <= 1e-6
