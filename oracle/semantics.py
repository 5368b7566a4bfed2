"""Exact (discrete) semantics of atoms and constraints — oracle, test infrastructure only.

* Atom alpha_i: sum_j q_ij y_j - q_i0 <rel> 0; delta_i = -1 iff True.
  Exact check (reading R22): fp64, s = 0; s += q_j*y_j sequentially in stored
  order (no fused multiply-add: Python floats round every op), then
  ``s <= q0`` (``<`` when strict).
* Constraint f_c : {+-1}^n x R^m -> {+-1}, -1 = True.
  Symmetric kinds: or: #true >= 1; card: #true <= k;
  nae: literals not all equal; xor: odd #true.
* Slots (readings R5, R6): one slot per DISTINCT underlying variable (Boolean
  variable or atom) of a constraint, ordered by first appearance in a
  left-to-right DFS of the expression (literal order for symmetric kinds).
"""
from __future__ import annotations

import numpy as np

from .hsmt import Atom, Constraint, Formula


def eval_atom(atom: Atom, y) -> bool:
    """True iff the canonical atom holds at y, exact fp64 (R22)."""
    s = 0.0
    for j, q in atom.coeffs:
        s = s + q * float(y[j])
    return s < atom.rhs if atom.strict else s <= atom.rhs


def slots(c: Constraint):
    """Distinct variables of c by first appearance (R5, R6): [(kind, idx), ...]."""
    out = []
    seen = set()

    def add(kind, idx):
        if (kind, idx) not in seen:
            seen.add((kind, idx))
            out.append((kind, idx))

    if c.kind == "expr":
        def rec(e):
            if e[0] == "lit":
                add(e[1], e[2])
            elif e[0] == "not":
                rec(e[1])
            else:
                for kid in e[1]:
                    rec(kid)
        rec(c.expr)
    else:
        for kind, idx, _ in c.lits:
            add(kind, idx)
    return out


def _sym_sat(kind, k, count, length):
    if kind == "or":
        return count >= 1
    if kind == "card":
        return count <= k
    if kind == "nae":
        return (count > 0) & (count < length)
    if kind == "xor":
        return (count % 2) == 1
    raise ValueError(kind)


def constraint_sat_values(c: Constraint, truth):
    """Evaluate c given ``truth[(kind, idx)] -> bool or bool ndarray`` (True = literal var True)."""
    if c.kind == "expr":
        def rec(e):
            if e[0] == "lit":
                v = truth[(e[1], e[2])]
                return ~v if (isinstance(v, np.ndarray)) and e[3] else ((not v) if e[3] else v)
            if e[0] == "not":
                v = rec(e[1])
                return ~v if isinstance(v, np.ndarray) else (not v)
            vals = [rec(kid) for kid in e[1]]
            acc = vals[0]
            for v in vals[1:]:
                if e[0] == "and":
                    acc = acc & v
                elif e[0] == "or":
                    acc = acc | v
                else:
                    acc = acc ^ v
            return acc
        return rec(c.expr)
    count = 0
    for kind, idx, neg in c.lits:
        v = truth[(kind, idx)]
        lit = (~v if isinstance(v, np.ndarray) else (not v)) if neg else v
        count = count + (lit.astype(np.int64) if isinstance(lit, np.ndarray) else int(lit))
    return _sym_sat(c.kind, c.k, count, len(c.lits))


def constraint_sat(f: Formula, c: Constraint, x, y) -> bool:
    """f_c(x, y) == -1 ?  x: sequence of +-1 (-1 = True), y: reals."""
    truth = {}
    for kind, idx in slots(c):
        if kind == "b":
            truth[(kind, idx)] = (x[idx] == -1)
        else:
            truth[(kind, idx)] = eval_atom(f.atoms[idx], y)
    return bool(constraint_sat_values(c, truth))


def eval_formula(f: Formula, x, y):
    """(F_w(x,y), per-constraint sat flags) — Eq.3; F_w = -sum w iff all sat (Thm.1)."""
    sat = [constraint_sat(f, c, x, y) for c in f.constraints]
    obj = 0.0
    for c, s in zip(f.constraints, sat):
        obj += c.weight * (-1.0 if s else 1.0)
    return obj, sat


def truth_table(c: Constraint) -> np.ndarray:
    """Satisfaction over all 2^s slot vertices; vertex bit s set <=> slot s True.

    Returns bool array of length 2^s, s = len(slots(c)).
    """
    sl = slots(c)
    s = len(sl)
    idx = np.arange(1 << s, dtype=np.int64)
    truth = {key: ((idx >> pos) & 1).astype(bool) for pos, key in enumerate(sl)}
    out = constraint_sat_values(c, truth)
    return np.broadcast_to(np.asarray(out, dtype=bool), idx.shape).copy()


def shape_key(c: Constraint) -> str:
    """Constraint text with variables renamed by slot position (truth tables are cached by it)."""
    pos = {key: i for i, key in enumerate(slots(c))}
    if c.kind == "expr":
        def rec(e):
            if e[0] == "lit":
                return ("!" if e[3] else "") + f"s{pos[(e[1], e[2])]}"
            if e[0] == "not":
                return f"(not {rec(e[1])})"
            return "(" + e[0] + " " + " ".join(rec(k) for k in e[1]) + ")"
        return rec(c.expr)
    return f"{c.kind}{c.k}:" + ",".join(("-" if n else "+") + f"s{pos[(k, i)]}" for k, i, n in c.lits)
