"""Projection onto the feasible set D (Def.1 / Prop.1) -- oracle, test infrastructure only.

Prop.1: proj_D(a', b') = argmin ||a - a'||^2 + ||b - b'||^2 subject to
-1 <= a_i <= 1 and every unit atomic constraint (a constraint that is one atom literal).
The a-block is a box (clamp).  For the b-block this module holds:

* ``halfspaces(f)`` -- reading R33: each multi-variable unit atom literal becomes the closed
  halfspace g.b <= h with a safety margin (single-variable ones are the R15 interval bounds):
      positive literal  q.b <= q0 (or < q0):       g = q,  h = q0 - delta
      negative literal  not(q.b <= q0) / not(<):   g = -q, h = -q0 - delta
      delta = 2^-17 (|q0| + ||q||_1)               (so the fp32-rounded point passes the exact check)
* ``project_exact(bp, lo, hi, H)`` -- the QP's definition written out: enumerate active sets of
  the inequality system {g_k.b <= h_k} U {b_j <= hi_j} U {-b_j <= -lo_j}, solve each equality-
  constrained least-squares problem in closed form, keep the one that is primal feasible with
  non-negative multipliers (KKT; the minimiser of a strictly convex QP is unique).  Exponential:
  tiny instances only.
* ``dykstra(bp, lo, hi, H, iters)`` -- Dykstra's alternating projection algorithm (Boyle &
  Dykstra 1986), the method the CUDA path runs: sets C_1..C_K = halfspaces in the listed order,
  then C_0 = the box, each with its own correction vector; ``iters`` sweeps.  Converges to
  project_exact as iters -> infinity (pinned in tests/test_oracle_pins.py).
"""
from __future__ import annotations

import itertools

import numpy as np

from .solve import unit_literal

MARGIN = 2.0 ** -17


def halfspaces(f):
    """[(cols, g, h)] for the multi-variable unit atom literals of f, in constraint order (R33)."""
    out = []
    for c in f.constraints:
        u = unit_literal(f, c)
        if u is None:
            continue
        aid, positive = u
        atom = f.atoms[aid]
        if len(atom.coeffs) < 2:
            continue                                   # single-variable: interval bound (R15)
        cols = [j for j, _ in atom.coeffs]
        q = np.array([qj for _, qj in atom.coeffs], dtype=np.float64)
        delta = MARGIN * (abs(atom.rhs) + np.abs(q).sum())
        if positive:
            out.append((cols, q, atom.rhs - delta))
        else:
            out.append((cols, -q, -atom.rhs - delta))
    return out


def _dense(H, m):
    G = np.zeros((len(H), m))
    h = np.zeros(len(H))
    for k, (cols, g, hk) in enumerate(H):
        for j, gj in zip(cols, g):
            G[k, j] += gj
        h[k] = hk
    return G, h


def project_exact(bp, lo, hi, H, tol=1e-10):
    """argmin ||b - bp||^2 s.t. G b <= h, lo <= b <= hi, by active-set enumeration (KKT)."""
    bp = np.asarray(bp, dtype=np.float64)
    m = len(bp)
    G, h = _dense(H, m)
    rows, rhs = [G], [h]
    for j in range(m):
        if np.isfinite(hi[j]):
            e = np.zeros(m); e[j] = 1.0
            rows.append(e[None]); rhs.append(np.array([float(hi[j])]))
        if np.isfinite(lo[j]):
            e = np.zeros(m); e[j] = -1.0
            rows.append(e[None]); rhs.append(np.array([-float(lo[j])]))
    A = np.vstack(rows) if rows else np.zeros((0, m))
    c = np.concatenate(rhs) if rhs else np.zeros(0)
    if np.all(A @ bp <= c + tol):
        return bp.copy()
    n = len(c)
    for size in range(1, min(n, m) + 1):
        for act in itertools.combinations(range(n), size):
            Aa, ca = A[list(act)], c[list(act)]
            M = Aa @ Aa.T
            if np.linalg.matrix_rank(M) < size:
                continue
            lam = np.linalg.solve(M, Aa @ bp - ca)          # stationarity: b = bp - Aa^T lam, Aa b = ca
            if np.any(lam < -tol):
                continue
            b = bp - Aa.T @ lam
            if np.all(A @ b <= c + 1e-9):
                return b
    raise RuntimeError("no KKT point found (infeasible constraint system?)")


def dykstra(bp, lo, hi, H, iters):
    """Dykstra's algorithm in fp64 with the CUDA path's set order and correction bookkeeping.

    Halfspace k: y = x[S] + p_k; x[S] = y - max(0, g.y - h) / ||g||^2 g; p_k = y - x[S].
    Box (last): y = x + p_0; x = clip(y, lo, hi); p_0 = y - x.
    """
    x = np.array(bp, dtype=np.float64)
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    p = [np.zeros(len(cols)) for cols, _, _ in H]
    p0 = np.zeros(len(x))
    for _ in range(iters):
        for k, (cols, g, hk) in enumerate(H):
            y = x[cols] + p[k]
            v = float(g @ y) - hk
            xs = y - (max(v, 0.0) / float(g @ g)) * g
            p[k] = y - xs
            x[cols] = xs
        y = x + p0
        x = np.minimum(np.maximum(y, lo), hi)
        p0 = y - x
    return x
