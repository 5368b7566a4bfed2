"""Diagnostic: per-constraint terms / gradients of the degenerate edge-case formula, GPU vs oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import hsmt, objective
from paper_2603_22877_b200 import Solver
from fsmt_gen.points import random_points
import tests.test_edge_cases as T

f = hsmt.parse(T.DEGENERATE)
s = Solver(0); s.load_formula(T.DEGENERATE); s.build_xbdd()
R = 37
a, b = random_points(f.n_bool, f.n_real, R, seed=5)
s.begin(R, 1); s.set_state(a, b); s.sweep(1.5, 1)
obj, ga, gb = s.get_sweep()
for r in (0, 36):
    C, oga, ogb, terms = objective.objective_and_gradient(f, a[:, r], b[:, r], 1.5, want_terms=True)
    E = s.constraint_terms(1.5, r)
    print("r", r, "obj", obj[r], C)
    print(" terms gpu", np.round(E, 5))
    print(" terms orc", np.round([terms[i] for i in range(len(f.constraints))], 5))
    print(" ga", ga[:, r], oga); print(" gb", gb[:, r], ogb)
a2, b2 = s.get_state(); print("state a", a2[:, 0], a[:, 0], "b", b2[:, 0], b[:, 0])
