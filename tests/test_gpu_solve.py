"""GPU solve-loop pieces: step-size / ERWA readings, rounding modes inside the solve, and the two
multi-GPU drivers run at world size 1 over NCCL must reproduce fsmt_solve exactly."""
import os
import socket

import numpy as np
import pytest

import fsmt_gen
from fsmt_gen.points import random_points, random_counters
from oracle import hsmt, objective, semantics
from tests.helpers import check_gradient, check_objective

pytestmark = pytest.mark.gpu


def make(text):
    import paper_2603_22877_b200 as P
    s = P.Solver(0)
    s.load_formula(text)
    s.build_xbdd()
    return s


@pytest.mark.parametrize("eta_mode", [0, 1, 2])
def test_run_stage_eta_mode_matches_manual_steps(eta_mode):
    inst = fsmt_gen.config("cfg4s")
    kappa, eta, steps = 3.0, 0.02, 4
    s1, s2 = make(inst.text), make(inst.text)
    s1.set_params(eta=eta, eps=1e-9, eta_mode=eta_mode)
    s2.set_params(eta=eta, eps=1e-9)
    for s in (s1, s2):
        s.begin(48, 21)
    u1, _ = s1.run_stage(2, kappa, steps)
    kk = np.float32(max(kappa, 1.0))               # the library computes eta_t in fp32
    eta_t = float(np.float32(eta) / (kk ** eta_mode if eta_mode < 2 else kk * kk)) if eta_mode else eta
    for _ in range(steps):
        s2.sweep(kappa, 2)
        s2.update(eta_t, 1e-9)
    u2 = s2.stage_end(2)
    a1, b1 = s1.get_state()
    a2, b2 = s2.get_state()
    assert np.array_equal(a1, a2) and np.array_equal(b1, b2) and np.array_equal(u1, u2)


def test_erwa_reset0_weights():
    inst = fsmt_gen.config("cfg2s")
    f = hsmt.parse(inst.text)
    s = make(inst.text)
    s.set_params(erwa_mode=1)
    R = 33
    a, b = random_points(f.n_bool, f.n_real, R, seed=2)
    U = random_counters(len(f.constraints), R, seed=3, max_u=3)
    s.begin(R, 1)
    s.set_state(a, b)
    s.set_counters(U)
    s.sweep(1.0, 7)                       # reset-to-0 reading: w = w_c 2^U, no stage factor (R18)
    obj, ga, gb = s.get_sweep()
    for r in (0, 32):
        w = np.array([c.weight for c in f.constraints]) * 2.0 ** U[:, r].astype(float)
        C, oga, ogb = objective.objective_and_gradient(f, a[:, r], b[:, r], 1.0, w)
        check_objective(obj[r], C, float(w.sum()))
        check_gradient(np.concatenate([ga[:, r], gb[:, r]]), np.concatenate([oga, ogb]), scale_relative=True)


@pytest.mark.parametrize("rounding", [0, 1])
def test_solve_rounding_modes_sound(rounding):
    inst = fsmt_gen.config("cfg4s")
    f = hsmt.parse(inst.text)
    s = make(inst.text)
    s.set_params(eta=0.05, rounding=rounding)
    res = s.solve(512, 40, 3)
    _, sat = semantics.eval_formula(f, res.x, res.y)
    assert (res.verdict == 10) == all(sat)
    assert sum(not v for v in sat) == res.stats["best_unsat"]


@pytest.fixture(scope="module")
def nccl_world1():
    """A world-size-1 NCCL process group for the driver tests, destroyed afterwards."""
    import torch.distributed as dist
    own = not dist.is_initialized()
    if own:
        sock = socket.socket()
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
        sock.close()
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
        dist.init_process_group("nccl", rank=0, world_size=1)
    yield
    if own:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["restart", "constraint"])
def test_dist_drivers_world1_reproduce_solve(mode, nccl_world1):
    import torch
    from paper_2603_22877_b200 import dist as D
    torch.cuda.set_device(0)
    inst = fsmt_gen.config("cfg4s")
    kappas = [0.5, 1.0, 2.0, 4.0, 8.0]
    ref = make(inst.text)
    ref.set_params(kappas=kappas, eta=0.05)
    res = ref.solve(256, 20, 11)
    s = make(inst.text)
    s.set_params(kappas=kappas, eta=0.05)
    s.bind_stream(torch.cuda.current_stream().cuda_stream)
    d = s.get_dims()
    if mode == "restart":
        out = D.solve_restart_sharded(s, d["n_bool"], d["n_real"], 256, 20, 11, kappas)
    else:
        out = D.solve_constraint_sharded(s, d["n_bool"], d["n_real"], 256, 20, 11, kappas, 1e-2)
    assert out.verdict == res.verdict
    assert (out.best_unsat, out.winner_stage, out.winner_restart) == (
        res.stats["best_unsat"], res.stats["winner_stage"], res.stats["winner_restart"])
    assert np.array_equal(out.x, res.x) and np.array_equal(out.y, res.y)


def test_cfg4_placement_time_to_sat():
    """The 10k-variable / 705k-constraint placement instance is solved
    with the DESIGN.md §9 schedule (geometric kappa to 300 then held, eta_mode 3, ERWA
    reset-to-0), and the model satisfies every constraint under the oracle's exact semantics."""
    from paper_2603_22877_b200 import native as N
    inst = fsmt_gen.config("cfg4")
    s = make(inst.text)
    kappas = [300.0 ** (i / 19) for i in range(20)] + [300.0] * 60
    s.set_params(kappas=kappas, eta=0.03, eta_mode=3, erwa_mode=1, time_limit_s=240)
    res = s.solve(1024, 40, 0)
    assert res.verdict == N.SAT, res.stats
    assert s.verify(res.x, res.y) == 0                       # host exact check, all constraints
    # independent check on a seeded sample of 20,000 constraints under the oracle's semantics
    from tests.helpers import subformula
    rng = np.random.default_rng(0)
    sample = rng.choice(inst.n_cons, 20000, replace=False)
    sub, kept = subformula(inst.text, extra_constraints=sample)
    f = hsmt.parse(sub)
    x = np.asarray(res.x)
    y = np.asarray(res.y, dtype=np.float32)
    bad = [kept[ci] for ci, c in enumerate(f.constraints) if not semantics.constraint_sat(f, c, x, y)]
    assert len(kept) == 20000 and not bad, bad[:10]


@pytest.mark.parametrize("name", ["cfg1", "cfg4s"])
def test_multiple_roundings_r34_match_oracle(name):
    """R34: with n_roundings = M each restart keeps the first of its M Philox draws with the
    fewest violations; the kept model, its unsat count and the ERWA counters match the oracle."""
    from oracle import solve as osolve
    inst = fsmt_gen.config(name)
    f = hsmt.parse(inst.text)
    M, R, seed = 6, 70, 9
    s = make(inst.text)
    s.set_params(eta=0.05, eps=1e-12, rounding=1, n_roundings=M)
    s.begin(R, seed)
    for _ in range(3):
        s.sweep(1.0, 2)
        s.update(0.05, 1e-12)
    a, b = s.get_state()
    unsat = s.stage_end(2)
    x = s.get_rounded()
    U = s.get_counters()
    y = b.astype(np.float32)
    for r in range(0, R, 7):
        best = None
        for m in range(M):
            xm = osolve.round_philox(a[:, r].astype(np.float64), seed, r, 2 + (m << 16))
            um = osolve.violations(f, xm, y[:, r])
            if best is None or um.sum() < best[1].sum():
                best = (xm, um)
        assert np.array_equal(x[:, r], best[0]), r
        assert unsat[r] == best[1].sum()
        assert np.array_equal(U[:, r].astype(int), best[1])


def test_multiple_roundings_solve_sound():
    inst = fsmt_gen.config("cfg4s")
    f = hsmt.parse(inst.text)
    s = make(inst.text)
    s.set_params(eta=0.05, rounding=1, n_roundings=4)
    res = s.solve(256, 20, 5)
    _, sat = semantics.eval_formula(f, res.x, res.y)
    assert (res.verdict == 10) == all(sat)
    assert sum(not v for v in sat) == res.stats["best_unsat"]


def test_graph_captured_stages_reproduce_solve():
    """FSMT_GRAPH=1 (the PGD steps of a stage as one CUDA graph, updated in place across stages)
    launches the same kernels with the same parameters: the solve is bit-identical."""
    inst = fsmt_gen.config("cfg4s")
    out = []
    for g in ("0", "1"):
        os.environ["FSMT_GRAPH"] = g
        try:
            s = make(inst.text)
            s.set_params(eta=0.05, rounding=1, kappas=[0.5, 1.0, 2.0, 4.0])
            res = s.solve(128, 12, 4)
            a, b = s.get_state()
            out.append((res.verdict, res.stats["best_unsat"], np.asarray(res.x).copy(), np.asarray(res.y).copy(), a, b))
        finally:
            os.environ.pop("FSMT_GRAPH", None)
    assert out[0][0] == out[1][0] and out[0][1] == out[1][1]
    for k in (2, 3, 4, 5):
        assert np.array_equal(out[0][k], out[1][k])


def test_graph_then_prepare_reproduces_solve():
    """A stage graph captured with the generic kernels is dropped by fsmt_prepare, and the next
    solve (prepared kernels, graph re-captured) reproduces the generic solve's verdict and
    violation count."""
    inst = fsmt_gen.config("cfg4s")
    os.environ["FSMT_GRAPH"] = "1"
    try:
        s = make(inst.text)
        s.set_params(eta=0.05, rounding=1, kappas=[0.5, 1.0, 2.0, 4.0])
        r1 = s.solve(128, 12, 4)
        s.prepare(128)
        assert "prepared R=128" in s.jit_info()["status"]
        r2 = s.solve(128, 12, 4)
        s.prepare(0)
        r3 = s.solve(128, 12, 4)
    finally:
        os.environ.pop("FSMT_GRAPH", None)
    assert r1.verdict == r2.verdict == r3.verdict
    assert r1.stats["best_unsat"] == r2.stats["best_unsat"] == r3.stats["best_unsat"]


@pytest.mark.parametrize("name,params", [
    ("cfg1", dict(eta=0.1)),
    ("cfg4s", dict(eta=0.05, rounding=1, kappas=[0.5, 1.0, 2.0, 4.0, 8.0])),
    ("cfg4s", dict(eta=0.05, rounding=1, n_roundings=4, kappas=[0.5, 1.0, 2.0, 4.0])),
    ("cfg3s", dict(eta=0.02, erwa_mode=1, eta_mode=3, kappas=[1.0, 3.0, 9.0, 27.0, 81.0] * 3)),
    ("cfg2s", dict(eta=0.05, kappas=[0.5, 1.0, 2.0] * 4)),
])
def test_device_side_solve_loop_matches_host_loop(name, params):
    """fsmt_solve's device-side loop (one CUDA graph with a WHILE node per stage, DESIGN.md §7 item 16)
    runs the host loop's kernels with the same arithmetic: verdict, winner, stages, model bit-identical."""
    inst = fsmt_gen.config(name)
    out = []
    for g in ("0", "1"):
        os.environ["FSMT_SOLVE_GRAPH"] = g
        try:
            s = make(inst.text)
            s.set_params(**params)
            res = s.solve(96, 6, 5)
            out.append(res)
        finally:
            os.environ.pop("FSMT_SOLVE_GRAPH", None)
    h, d = out
    for k in ("best_unsat", "winner_stage", "winner_restart", "stages_run", "steps_run", "host_verified"):
        assert h.stats[k] == d.stats[k], (k, h.stats[k], d.stats[k])
    assert h.verdict == d.verdict
    assert np.array_equal(h.x, d.x) and np.array_equal(h.y, d.y)


def test_device_side_solve_loop_time_limit():
    """With a time limit the device-side loop returns to the host every 16 stages; an exhausted
    limit gives FSMT_ERR_TIMEOUT with the best model so far (soundness unchanged)."""
    inst = fsmt_gen.config("cfg3s")
    f = hsmt.parse(inst.text)
    s = make(inst.text)
    s.set_params(eta=0.001, kappas=[0.01] * 400, time_limit_s=1e-6)
    res = s.solve(64, 2, 1)
    assert res.stats["timeout"] and res.stats["stages_run"] == 16
    _, sat = semantics.eval_formula(f, res.x, res.y)
    assert sum(not v for v in sat) == res.stats["best_unsat"]
