"""Edge cases of the boundary: degenerate constraints (constant, duplicated variables -- R5),
formatting (comments, CRLF), the node budget, empty formulas; host side vs the oracle on CPU,
kernels vs the oracle on the GPU."""
import os
import tempfile

import numpy as np
import pytest

from oracle import hsmt, robdd, semantics, objective
from paper_2603_22877_b200 import Solver, FsmtError
from paper_2603_22877_b200 import native as N
from fsmt_gen.points import random_points

DEGENERATE = (
    "p hsmt 3 2\r\n"
    "# comment line\r\n"
    "a 0 <= 0.5 0:1 1:-1   # trailing comment\n"
    "a 1 > -0.25 1:2\n"
    "c xor 1 +b0 -b0\n"                  # constant True (R5: one slot, x xor not x)
    "c or 2 +b1 -b1\n"                   # constant True
    "c nae 1 +b2\n"                      # constant False (single literal NAE)
    "e 0.5 (and b0 (not b0))\n"          # constant False
    "c card 1 1 +b0 +b0 +b1\n"           # duplicated variable: #true <= 1 with b0 counted twice
    "e 1 (xor a0 (not a0) b1)\n"         # duplicated atom
    "c or 1 -a1 +b2\n"
    "e 3 (or (and b0 a0) (and (not b0) a1))\n"
)


def _host(text):
    s = Solver(-1)
    s.load_formula(text)
    s.build_xbdd()
    return s


def test_degenerate_structure_and_verify_match_oracle():
    s = _host(DEGENERATE)
    f = hsmt.parse(DEGENERATE)
    with tempfile.TemporaryDirectory() as d:
        s.dump_structure(d)
        tj = open(os.path.join(d, "templates.jsonl")).read()
        cb = open(os.path.join(d, "constraints.bin"), "rb").read()
    ot, ob = robdd.canonical_dump(f)
    assert tj == ot and cb == ob
    rng = np.random.default_rng(0)
    for _ in range(50):
        x = rng.choice([-1, 1], f.n_bool).astype(np.int8)
        y = rng.uniform(-1, 1, f.n_real).astype(np.float32)
        n, pc = s.verify(x, y, per_con=True)
        want = np.array([0 if semantics.constraint_sat(f, c, x, y) else 1 for c in f.constraints])
        assert np.array_equal(pc.astype(int), want) and n == want.sum()


def test_node_budget_and_empty_formula():
    s = Solver(-1)
    s.load_formula("p hsmt 30 0\nc card 15 1 " + " ".join(f"+b{i}" for i in range(30)) + "\n")
    with pytest.raises(FsmtError) as e:
        s.build_xbdd(node_budget=20)
    assert e.value.status == N.ERR_NODE_BUDGET
    s.build_xbdd()                                   # default budget succeeds
    e = _host("p hsmt 0 0\n")
    assert e.get_dims()["n_cons"] == 0


@pytest.mark.gpu
def test_degenerate_kernels_match_oracle():
    f = hsmt.parse(DEGENERATE)
    s = Solver(0)
    s.load_formula(DEGENERATE)
    s.build_xbdd()
    R = 37
    a, b = random_points(f.n_bool, f.n_real, R, seed=5)
    s.begin(R, 1)
    s.set_state(a, b)
    s.sweep(1.5, 1)
    obj, ga, gb = s.get_sweep()
    w = [c.weight for c in f.constraints]            # the formula's w_c (the oracle defaults to 1)
    for r in (0, 36):
        C, oga, ogb = objective.objective_and_gradient(f, a[:, r], b[:, r], 1.5, w)
        assert abs(obj[r] - C) <= 1e-5 and np.max(np.abs(ga[:, r] - oga)) <= 1e-5 and np.max(np.abs(gb[:, r] - ogb)) <= 1e-5
    X = np.where(a < 0, -1, 1).astype(np.int8)
    u, pc = s.verify_batch(X, b, per_con=True)
    for r in range(R):
        want = np.array([0 if semantics.constraint_sat(f, c, X[:, r], b[:, r]) else 1 for c in f.constraints])
        assert np.array_equal(pc[:, r].astype(int), want)


@pytest.mark.gpu
def test_empty_formula_solve_is_sat():
    s = Solver(0)
    s.load_formula("p hsmt 2 1\n")
    s.build_xbdd()
    res = s.solve(8, 2, 0)
    assert res.verdict == N.SAT
