"""The JIT planner's and emitter's optional transformations (DESIGN.md §7, §9 A/B table) each
keep the sweep and the exact check in parity with the oracle: objective, gradients and
per-constraint verdicts on cfg3s / cfg4s / cfg2 under every knob setting."""
import os

import numpy as np
import pytest

import fsmt_gen
from fsmt_gen.points import random_points
from oracle import hsmt, objective, semantics
from tests.helpers import check_gradient, check_objective

pytestmark = pytest.mark.gpu

KNOBS = [
    {},
    {"FSMT_JIT_AFFINE": "0"},
    {"FSMT_JIT_DIAMOND": "0", "FSMT_JIT_ALIAS": "0"},
    {"FSMT_JIT_FOLD": "0", "FSMT_JIT_VFOLD": "0"},
    {"FSMT_JIT_SYM": "0"},
    {"FSMT_JIT_PAIR": "0", "FSMT_JIT_UPF": "0"},
    {"FSMT_JIT_UPF": "3"},
    {"FSMT_JIT_CMP": "0"},
    {"FSMT_JIT_UNROLL": "1"},
    {"FSMT_JIT_VPF": "0"},
    {"FSMT_JIT_VPF": "0", "FSMT_JIT_UNROLL": "2", "FSMT_JIT_UPF": "2"},
    {"FSMT_TILE_VMAX": "16", "FSMT_TILE_RMAX": "16", "FSMT_TILE_CMAX": "3"},
    {"FSMT_JIT_VID32": "1"},
    {"FSMT_TILE_MERGE": "1"},
    {"FSMT_TILE_MERGE": "0"},
]


_ORC = {}


def oracle_case(name):
    """Formula, points and oracle values for restarts 0 and 44 (cached across knob settings)."""
    if name not in _ORC:
        inst = fsmt_gen.config(name)
        f = hsmt.parse(inst.text)
        a, b = random_points(f.n_bool, f.n_real, 45, seed=21, b_lo=0.0, b_hi=1.0)
        w = [c.weight for c in f.constraints]
        x = np.where(a < 0, -1, 1).astype(np.int8)
        vals = {}
        for r in (0, 44):
            C, oga, ogb = objective.objective_and_gradient(f, a[:, r], b[:, r], 1.3, w)
            want = np.array([0 if semantics.constraint_sat(f, c, x[:, r], b[:, r]) else 1 for c in f.constraints])
            vals[r] = (C, oga, ogb, want)
        _ORC[name] = (inst, f, a, b, x, w, vals)
    return _ORC[name]


@pytest.mark.parametrize("knobs", KNOBS, ids=lambda k: ",".join(f"{a}={b}" for a, b in k.items()) or "default")
@pytest.mark.parametrize("name", ["cfg3s", "cfg4s", "cfg2"])
def test_knob_parity(name, knobs):
    import paper_2603_22877_b200 as P
    inst = fsmt_gen.config(name)
    old = {k: os.environ.get(k) for k in knobs}
    os.environ.update(knobs)
    try:
        s = P.Solver(0)
        s.load_formula(inst.text)
        s.build_xbdd()                       # the knobs are read here
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    assert s.jit_info()["jit_classes"] > 0 or (name == "cfg2" and knobs.get("FSMT_JIT_SYM") == "0")
    _, f, a, b, x, w, vals = oracle_case(name)
    R = 45
    s.begin(R, 3)
    s.set_state(a, b)
    s.sweep(1.3, 1)
    obj, ga, gb = s.get_sweep()
    _, pc = s.verify_batch(x, b, per_con=True)
    for r in (0, 44):
        C, oga, ogb, want = vals[r]
        check_objective(obj[r], C, float(sum(w)), what=f"{name} {knobs}")
        check_gradient(ga[:, r], oga, what=f"{name} grad_a {knobs}")
        check_gradient(gb[:, r], ogb, what=f"{name} grad_b {knobs}")
        assert np.array_equal(pc[:, r].astype(int), want)


@pytest.mark.parametrize("name", ["cfg3s", "cfg4s", "cfg2"])
def test_prepared_r_bit_identical(name):
    """fsmt_prepare(R) (restart count compiled in, DESIGN.md §7 item 10) changes no bit: sweep,
    stage end (rounding, exact check, ERWA counters) and a second weighted sweep equal the
    generic kernels'; another R still runs the generic module; and the values match the oracle."""
    import paper_2603_22877_b200 as P
    inst, f, a, b, x, w, vals = oracle_case(name)
    R = 45
    out = []
    for prep in (0, R):
        s = P.Solver(0)
        s.load_formula(inst.text)
        s.build_xbdd()
        if prep:
            s.prepare(prep)
            s.prepare(prep)                  # idempotent
        s.begin(R, 3)
        s.set_state(a, b)
        s.sweep(1.3, 1)
        r1 = s.get_sweep()
        unsat = s.stage_end(1)
        s.sweep(0.7, 3)
        r2 = s.get_sweep()
        _, pc = s.verify_batch(x, b, per_con=True)
        out.append((r1, np.array(unsat), r2, pc, s.get_counters()))
        if prep:
            s.begin(64, 3)                   # not the prepared R: generic module
            s.sweep(1.0, 1)
            assert np.all(np.isfinite(s.get_sweep()[0]))
            s.prepare(0)                     # dropped
    (g1, gu, g2, gpc, gU), (p1, pu, p2, ppc, pU) = out
    # per-term arithmetic is identical and the fp64 sums are exact (on-grid accumulation, DESIGN.md
    # §7 item 14), so every output is bit-identical
    for A, B in zip(g1 + g2, p1 + p2):
        assert np.array_equal(A, B)
    assert np.array_equal(gu, pu) and np.array_equal(gpc, ppc) and np.array_equal(gU, pU)
    for r in (0, 44):
        C, oga, ogb, want = vals[r]
        check_objective(p1[0][r], C, float(sum(w)), what=f"{name} prepared")
        check_gradient(p1[1][:, r], oga, what=f"{name} prepared grad_a")
        check_gradient(p1[2][:, r], ogb, what=f"{name} prepared grad_b")
        assert np.array_equal(ppc[:, r].astype(int), want)


@pytest.mark.parametrize("split", ["2", "5"])
@pytest.mark.parametrize("name", ["cfg3s", "cfg4s", "cfg2"])
def test_tile_split_parity(name, split):
    """The launch-time split of tiles into constraint ranges (FSMT_TILE_SPLIT, read per launch; the
    default splits only tiles of >= 64 constraints when the restarts are few): the exact check (stage
    end, ERWA counters, per-constraint verdicts) is bit-identical to the unsplit launch, and the
    sweep -- whose fp32 partial sums the split regroups -- matches the oracle."""
    import paper_2603_22877_b200 as P
    inst, f, a, b, x, w, vals = oracle_case(name)
    R = 45
    out = []
    for sp in ("1", split):
        old = os.environ.get("FSMT_TILE_SPLIT")
        os.environ["FSMT_TILE_SPLIT"] = sp
        try:
            s = P.Solver(0)
            s.load_formula(inst.text)
            s.build_xbdd()
            s.begin(R, 3)
            s.set_state(a, b)
            s.sweep(1.3, 1)
            r1 = s.get_sweep()
            unsat = s.stage_end(1)
            _, pc = s.verify_batch(x, b, per_con=True)
            out.append((r1, np.array(unsat), pc, s.get_counters()))
        finally:
            if old is None:
                os.environ.pop("FSMT_TILE_SPLIT", None)
            else:
                os.environ["FSMT_TILE_SPLIT"] = old
    (g1, gu, gpc, gU), (p1, pu, ppc, pU) = out
    assert np.array_equal(gu, pu) and np.array_equal(gpc, ppc) and np.array_equal(gU, pU)
    for r in (0, 44):
        C, oga, ogb, want = vals[r]
        check_objective(p1[0][r], C, float(sum(w)), what=f"{name} split {split}")
        check_gradient(p1[1][:, r], oga, what=f"{name} split grad_a")
        check_gradient(p1[2][:, r], ogb, what=f"{name} split grad_b")
        assert np.array_equal(ppc[:, r].astype(int), want)
