"""GPU numerics of the smoothed atom probabilities over the whole argument range (Eq.7,
P:224-229; derivative P:1326-1327): single-atom constraints E_c = -d = -erf(u) and
dE/db = -dd/db, u swept over [-7, 7], through the specialised sweep."""
import math

import numpy as np
import pytest

from oracle import hsmt, objective
from tests.helpers import check_gradient

pytestmark = pytest.mark.gpu


def test_atom_probability_accuracy_sweep():
    import paper_2603_22877_b200 as P
    n = 400
    # atom i: q_i y_i <= q0_i with varied coefficients (R18 scale-free), one constraint each
    rng = np.random.default_rng(0)
    lines = [f"p hsmt 0 {n}"]
    qs = rng.choice([-3.0, -1.0, 0.5, 2.0], n)
    for i in range(n):
        lines.append(f"a {i} <= 0.25 {i}:{qs[i]}")
    for i in range(n):
        lines.append(f"e 1 (or a{i} a{i})")          # unit atom; set_state below does not project
    text = "\n".join(lines) + "\n"
    s = P.Solver(0)
    s.load_formula(text)
    s.build_xbdd()
    assert s.jit_info()["jit_cons"] == n
    f = hsmt.parse(text)
    R = 64
    kappa = 2.0
    # u = kappa (q b - q0)/(sqrt2 |q|) spans [-7, 7] across atoms and restarts
    u = np.linspace(-7, 7, n * R).reshape(n, R)
    b = ((u * math.sqrt(2) * np.abs(qs)[:, None] / kappa + 0.25) / qs[:, None]).astype(np.float32)
    s.begin(R, 1)
    s.set_state(None, b)
    s.sweep(kappa, 1)
    obj, ga, gb = s.get_sweep()
    for r in (0, 17, 63):
        E = s.constraint_terms(kappa, r)
        C, _, ogb, terms = objective.objective_and_gradient(f, [], b[:, r], kappa, want_terms=True)
        want = np.array([terms[i] for i in range(n)])
        assert np.max(np.abs(E - want)) <= 2.5e-7, np.max(np.abs(E - want))
        check_gradient(gb[:, r], ogb, atol=1e-5, what="atom sweep")
