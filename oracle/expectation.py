"""E_c and dE_c/dv_s — oracle, test infrastructure only.

Plain definition (Lemma P:812-827 + Thm P:863-868 = Eq.8; exact reformulation
of the xBDD COP by Cor.2 P:998-1013):

    E_c(v) = sum_{z in {+-1}^s} f_c(z) * prod_s (1 + z_s v_s)/2

where v_s = a_i for a Boolean slot and v_s = d_i(b) for an atom slot, and
z_s = -1 means "slot s True".  E_c is multilinear in each v_s, so

    dE_c/dv_s = ( E_c|_{v_s=+1} - E_c|_{v_s=-1} ) / 2              (exact).

Three evaluation paths, all fp64, cross-checked in tests:
  O1 ``enum_*``      the sum above literally, over all 2^s vertices;
  O1'``contract_*``  the same multilinear form evaluated one axis at a time with
                     np.tensordot (library contraction; used for s up to 24);
  O2 ``wfe_*``       Walsh-Fourier coefficients (Thm "WFE" P:739-747, Cor.1
                     P:751-762) by a fast Walsh-Hadamard transform, then
                     Eq.8 sum_U fhat(U) prod_{s in U} v_s;
  O3 ``sym_*``       symmetric kinds by the Poisson-binomial count
                     distribution (the O((n+k)^2) route named at P:254): exact, a
                     different algorithm for the same definition; requires
                     distinct variables per constraint.
"""
from __future__ import annotations

import numpy as np

from .semantics import truth_table, slots, shape_key

# ----------------------------------------------------------------------------- O1


def f_values(table: np.ndarray) -> np.ndarray:
    """f_c(z) in {-1 (True), +1 (False)} per vertex."""
    return np.where(table, -1.0, 1.0)


def enum_expectation(table: np.ndarray, v) -> float:
    """Literal Eq.8: sum over all vertices of f(z) * prod_s P[slot s takes z_s]."""
    s = len(v)
    idx = np.arange(1 << s, dtype=np.int64)
    w = np.ones(1 << s)
    for pos in range(s):
        bit = ((idx >> pos) & 1).astype(bool)              # bit set <=> z_s = -1 (True)
        w = w * np.where(bit, (1.0 - v[pos]) / 2.0, (1.0 + v[pos]) / 2.0)
    return float(f_values(table) @ w)


def enum_gradient(table: np.ndarray, v) -> np.ndarray:
    """dE/dv_s = (E|v_s=+1 - E|v_s=-1)/2, each term by enum_expectation."""
    out = np.zeros(len(v))
    for pos in range(len(v)):
        vp = list(v)
        vp[pos] = 1.0
        vm = list(v)
        vm[pos] = -1.0
        out[pos] = (enum_expectation(table, vp) - enum_expectation(table, vm)) / 2.0
    return out


# ----------------------------------------------------------------------------- O1'


def _tensor(table: np.ndarray, s: int) -> np.ndarray:
    # vertex index = sum_pos bit_pos 2^pos; C-order reshape puts slot s-1 on axis 0,
    # so reverse the axes to have axis t <-> slot t.
    return f_values(table).reshape((2,) * s).transpose(tuple(range(s - 1, -1, -1))) if s else f_values(table).reshape(())


def _vec(vs):
    # index 0 <-> bit 0 <-> z_s = +1 (False): prob (1+v)/2 ; index 1 <-> True: (1-v)/2
    return np.array([(1.0 + vs) / 2.0, (1.0 - vs) / 2.0])


def contract_expectation(table: np.ndarray, v) -> float:
    s = len(v)
    t = _tensor(table, s)
    for pos in range(s - 1, -1, -1):
        t = np.tensordot(t, _vec(v[pos]), axes=([pos], [0]))
    return float(t)


def contract_gradient(table: np.ndarray, v) -> np.ndarray:
    s = len(v)
    base = _tensor(table, s)
    out = np.zeros(s)
    for keep in range(s):
        t = base
        for pos in range(s - 1, -1, -1):
            if pos != keep:
                t = np.tensordot(t, _vec(v[pos]), axes=([pos], [0]))
        # t = [E | slot False, E | slot True]
        out[keep] = (t[0] - t[1]) / 2.0
    return out


# ----------------------------------------------------------------------------- O2


def wfe_coefficients(table: np.ndarray) -> np.ndarray:
    """fhat(U) = E_z[f(z) prod_{s in U} z_s] for every subset mask U (Cor.1 P:758-762)."""
    h = f_values(table).copy()
    n = h.shape[0]
    step = 1
    while step < n:                       # in-place Walsh-Hadamard butterflies
        h = h.reshape(-1, 2, step)
        a = h[:, 0, :].copy()
        b = h[:, 1, :].copy()
        # z = +1 at bit 0, z = -1 at bit 1  =>  chi_U(z) = (-1)^{popcount(idx & U)}
        h[:, 0, :] = a + b
        h[:, 1, :] = a - b
        h = h.reshape(n)
        step *= 2
    return h / n


def wfe_expectation(coef: np.ndarray, v) -> float:
    """Eq.8: sum_U fhat(U) prod_{s in U} v_s."""
    s = len(v)
    idx = np.arange(1 << s, dtype=np.int64)
    mono = np.ones(1 << s)
    for pos in range(s):
        bit = ((idx >> pos) & 1).astype(bool)
        mono = mono * np.where(bit, v[pos], 1.0)
    return float(coef @ mono)


def wfe_sparse(coef: np.ndarray, tol: float = 1e-15):
    nz = np.nonzero(np.abs(coef) > tol)[0]
    return nz.astype(np.int64), coef[nz]


def wfe_sparse_eval(masks: np.ndarray, vals: np.ndarray, s: int, V: np.ndarray):
    """Batched sparse Eq.8 and gradient for many constraints sharing one shape.

    V: (B, s) slot values.  Returns E (B,), dE (B, s).  dE_s = sum_{U ni s} fhat(U) prod_{t in U, t != s} v_t.
    """
    B = V.shape[0]
    bits = ((masks[:, None] >> np.arange(s)[None, :]) & 1).astype(bool)   # (K, s)
    E = np.zeros(B)
    dE = np.zeros((B, s))
    for kk in range(len(masks)):
        cols = np.nonzero(bits[kk])[0]
        if len(cols) == 0:
            E += vals[kk]
            continue
        sub = V[:, cols]
        E += vals[kk] * np.prod(sub, axis=1)
        for ci, col in enumerate(cols):
            others = np.delete(sub, ci, axis=1)
            dE[:, col] += vals[kk] * (np.prod(others, axis=1) if others.shape[1] else 1.0)
    return E, dE


# ----------------------------------------------------------------------------- O3


def _sym_sat_counts(kind, k, L):
    t = np.arange(L + 1)
    if kind == "or":
        return t >= 1
    if kind == "card":
        return t <= k
    if kind == "nae":
        return (t > 0) & (t < L)
    if kind == "xor":
        return (t % 2) == 1
    raise ValueError(kind)


def _count_dist(ps):
    """Poisson-binomial: P[#true = t] for independent literals with P[true] = ps[i]."""
    P = np.zeros(len(ps) + 1)
    P[0] = 1.0
    for i, p in enumerate(ps):
        nxt = P * (1.0 - p)
        nxt[1:] += P[:-1] * p
        P = nxt
    return P


def sym_expectation_and_gradient(c, v):
    """E_c and dE_c/dv_s for symmetric c with distinct variables (slot s = literal s).

    COP = sum_{t sat} P[#true = t]; E = 1 - 2 COP (Alg.F line P:1170).
    Literal l over slot s: P[l true] = (1 - v_s)/2, or (1 + v_s)/2 if negated.
    dCOP/dp_l = P[sat | l true] - P[sat | l false] (leave-one-out count distribution);
    dE/dv_s = -2 * dCOP/dp_l * dp_l/dv_s with dp_l/dv_s = -1/2 (+1/2 if negated).
    """
    L = len(c.lits)
    sat = _sym_sat_counts(c.kind, c.k, L)
    pl = [((1.0 + v[i]) / 2.0 if neg else (1.0 - v[i]) / 2.0) for i, (_, _, neg) in enumerate(c.lits)]
    P = _count_dist(pl)
    cop = float(P[sat].sum())
    grad = np.zeros(L)
    for i, (_, _, neg) in enumerate(c.lits):
        Q = _count_dist(pl[:i] + pl[i + 1:])             # others, length L
        p_true = float(Q[sat[1:]].sum())                 # l true: count shifts by one
        p_false = float(Q[sat[:-1]].sum())
        dcop_dp = p_true - p_false
        grad[i] = -2.0 * dcop_dp * (0.5 if neg else -0.5)
    return 1.0 - 2.0 * cop, grad


# ----------------------------------------------------------------------------- dispatch

_TABLE_CACHE = {}


def cached_table(c):
    key = shape_key(c)
    t = _TABLE_CACHE.get(key)
    if t is None:
        t = truth_table(c)
        _TABLE_CACHE[key] = t
    return t


def is_distinct_symmetric(c) -> bool:
    return c.kind != "expr" and len({(k, i) for k, i, _ in c.lits}) == len(c.lits)


def constraint_expectation_and_gradient(c, v):
    """(E_c, dE_c/dv) for slot values v (ordered as semantics.slots(c))."""
    s = len(v)
    if is_distinct_symmetric(c) and s > 12:
        return sym_expectation_and_gradient(c, v)
    if s > 24:
        raise ValueError(f"constraint with {s} slots is beyond the enumeration oracle")
    table = cached_table(c)
    if s <= 10:
        return enum_expectation(table, v), enum_gradient(table, v)
    return contract_expectation(table, v), contract_gradient(table, v)


__all__ = [
    "enum_expectation", "enum_gradient", "contract_expectation", "contract_gradient",
    "wfe_coefficients", "wfe_expectation", "wfe_sparse", "wfe_sparse_eval",
    "sym_expectation_and_gradient", "constraint_expectation_and_gradient", "cached_table",
    "slots",
]
