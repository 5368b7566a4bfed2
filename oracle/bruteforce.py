"""Exhaustive SAT for tiny formulas with exact Fourier-Motzkin — oracle, test infrastructure only.

Completeness oracle for Thm.1 pins, following S:163-178: enumerate
every atom truth pattern, keep those that are LRA-consistent (Fourier-Motzkin
over exact rationals, strictness tracked), and for each enumerate the Boolean
vectors; a (Boolean, pattern) pair is a model iff every constraint holds.
"""
from __future__ import annotations

from fractions import Fraction
from itertools import product

from .semantics import constraint_sat_values, slots


def _ineq(atom, truth):
    """Atom (canonical q.y <= q0 | < q0) with a required truth value -> (coeffs, rhs, strict) as '<='/'<'."""
    q = {j: Fraction(c) for j, c in atom.coeffs}
    q0 = Fraction(atom.rhs)
    if truth:
        return q, q0, atom.strict
    # not(q.y <= q0)  <=>  -q.y < -q0 ; not(q.y < q0) <=> -q.y <= -q0
    return {j: -c for j, c in q.items()}, -q0, not atom.strict


def fm_feasible(ineqs, n_vars):
    """Fourier-Motzkin feasibility of sum_j c_j y_j (<|<=) rhs; returns a rational witness or None."""
    stages = [list(ineqs)]
    cur = list(ineqs)
    for e in range(n_vars):
        pos = [x for x in cur if x[0].get(e, 0) > 0]
        neg = [x for x in cur if x[0].get(e, 0) < 0]
        nxt = [x for x in cur if x[0].get(e, 0) == 0]
        for (cp, rp, sp) in pos:
            for (cn, rn, sn) in neg:
                a, b = cp[e], -cn[e]
                co = {}
                for j in set(cp) | set(cn):
                    v = cp.get(j, 0) / a + cn.get(j, 0) / b
                    if j != e and v != 0:
                        co[j] = v
                nxt.append((co, rp / a + rn / b, sp or sn))
        cur = nxt
        stages.append(cur)
    for co, rhs, strict in cur:
        if (0 >= rhs) if strict else (0 > rhs):
            return None
    y = {}
    for e in range(n_vars - 1, -1, -1):
        lo, lo_s, hi, hi_s = None, False, None, False
        for co, rhs, strict in stages[e]:
            c = co.get(e, 0)
            if c == 0:
                continue
            rest = rhs - sum(v * y[j] for j, v in co.items() if j != e)
            bnd = rest / c
            if c > 0:
                if hi is None or bnd < hi or (bnd == hi and strict):
                    hi, hi_s = bnd, strict
            else:
                if lo is None or bnd > lo or (bnd == lo and strict):
                    lo, lo_s = bnd, strict
        if lo is None and hi is None:
            y[e] = Fraction(0)
        elif lo is None:
            y[e] = hi - 1
        elif hi is None:
            y[e] = lo + 1
        elif lo < hi:
            y[e] = (lo + hi) / 2
        else:
            y[e] = lo
    return [y[j] for j in range(n_vars)]


def brute_force_sat(f, limit_bool=16, limit_atoms=16):
    """Returns (x, y) model (x: +-1 list, y: Fractions) or None if unsatisfiable."""
    if f.n_bool > limit_bool or len(f.atoms) > limit_atoms:
        raise ValueError("formula beyond brute-force limits")
    k = len(f.atoms)
    for pattern in product([True, False], repeat=k):
        ineqs = [_ineq(f.atoms[i], pattern[i]) for i in range(k)]
        y = fm_feasible(ineqs, f.n_real)
        if y is None:
            continue
        for xs in product([True, False], repeat=f.n_bool):
            truth = {("b", i): xs[i] for i in range(f.n_bool)}
            truth.update({("a", i): pattern[i] for i in range(k)})
            if all(bool(constraint_sat_values(c, truth)) for c in f.constraints):
                return [(-1 if t else 1) for t in xs], y
    return None


def count_models(f):
    """Number of satisfying (Boolean vector, LRA-consistent atom pattern) pairs."""
    k = len(f.atoms)
    n = 0
    for pattern in product([True, False], repeat=k):
        ineqs = [_ineq(f.atoms[i], pattern[i]) for i in range(k)]
        if fm_feasible(ineqs, f.n_real) is None:
            continue
        for xs in product([True, False], repeat=f.n_bool):
            truth = {("b", i): xs[i] for i in range(f.n_bool)}
            truth.update({("a", i): pattern[i] for i in range(k)})
            if all(bool(constraint_sat_values(c, truth)) for c in f.constraints):
                n += 1
    return n


__all__ = ["fm_feasible", "brute_force_sat", "count_models", "slots"]
