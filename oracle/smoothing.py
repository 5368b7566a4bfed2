"""Gaussian smoothing of atoms — oracle, test infrastructure only.

Eq.7 (derivation P:830-851):
    d_i(b) = E_{y~N(b, sigma^2 I)} delta_i(y) = erf( (q_i.b - q_i0) / (sqrt(2) ||q_i|| sigma) )
Gradient, P:1326-1327 (the printed exponent at P:855-858 is wrong, reading R2):
    dd_i/db_j = sqrt(2) q_ij / (sqrt(pi) sigma ||q_i||) * exp( -(q_i.b - q_i0)^2 / (2 sigma^2 ||q_i||^2) )
Parametrised by kappa = 1/sigma >= 0 (reading R11): kappa = 0 gives d = 0, dd = 0;
kappa = inf is the sigma = 0 hard switch d = delta (Thm.3).
Randomised rounding (Eq.4): P[x_i = -1] = (1 - a_i)/2.
"""
from __future__ import annotations

import math

from .hsmt import Atom
from .semantics import eval_atom


def round_prob(a_i: float) -> float:
    """P[R(a)_i = -1] = (1 - a_i)/2 (Eq.4)."""
    return (1.0 - a_i) / 2.0


def atom_z(atom: Atom, b) -> float:
    s = 0.0
    for j, q in atom.coeffs:
        s += q * float(b[j])
    return s - atom.rhs


def atom_norm(atom: Atom) -> float:
    return math.sqrt(sum(q * q for _, q in atom.coeffs))


def atom_smooth(atom: Atom, b, kappa: float) -> float:
    """d_i(b) of Eq.7 with sigma = 1/kappa."""
    if math.isinf(kappa):
        return -1.0 if eval_atom(atom, b) else 1.0
    if kappa == 0.0:
        return 0.0
    return math.erf(kappa * atom_z(atom, b) / (math.sqrt(2.0) * atom_norm(atom)))


def atom_smooth_grad(atom: Atom, b, kappa: float):
    """[(j, dd_i/db_j)] from P:1326-1327 (sigma = 1/kappa)."""
    if math.isinf(kappa):
        raise ValueError("gradient undefined at sigma = 0 (S:306)")
    nq = atom_norm(atom)
    z = atom_z(atom, b)
    sigma_inv = kappa
    g = math.exp(-(z * z) * sigma_inv * sigma_inv / (2.0 * nq * nq))
    return [(j, math.sqrt(2.0) * q * sigma_inv / (math.sqrt(math.pi) * nq) * g) for j, q in atom.coeffs]
