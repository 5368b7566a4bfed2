"""C_sigma(a, b) and its gradient — oracle, test infrastructure only.

    C(a,b)   = sum_c w_c E_c(v)                          (Eq.10; Alg.F)
    dC/da_i  = sum_c w_c sum_{s: var(s)=i} dE_c/dv_s     (Alg.B P:1192-1193 with the sign of R1)
    dC/db_j  = sum_c w_c sum_{atom slots s=i} dE_c/dv_s * dd_i/db_j   (Alg.B)

v_s = a_i for Boolean slots, d_i(b) (Eq.7) for atom slots.  Accumulated in fp64
in constraint order.
"""
from __future__ import annotations

import numpy as np

from .expectation import constraint_expectation_and_gradient
from .semantics import slots
from .smoothing import atom_smooth, atom_smooth_grad


def smoothed_atoms(f, b, kappa, needed=None):
    ids = range(len(f.atoms)) if needed is None else needed
    d = {}
    dd = {}
    for i in ids:
        d[i] = atom_smooth(f.atoms[i], b, kappa)
        dd[i] = atom_smooth_grad(f.atoms[i], b, kappa) if np.isfinite(kappa) else []
    return d, dd


def objective_and_gradient(f, a, b, kappa, weights=None, subset=None, want_terms=False):
    """Returns (C, grad_a, grad_b[, E per constraint]) at one restart point.

    weights: per-constraint w_c (default: the formula's weights, Eq.3).  subset: optional
    iterable of constraint indices to restrict the sums to (sampled parity at full size).
    """
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    cons = range(len(f.constraints)) if subset is None else subset
    needed = set()
    cslots = {}
    for ci in cons:
        sl = slots(f.constraints[ci])
        cslots[ci] = sl
        needed.update(i for k, i in sl if k == "a")
    d, dd = smoothed_atoms(f, b, kappa, sorted(needed))
    C = 0.0
    ga = np.zeros(f.n_bool)
    gb = np.zeros(f.n_real)
    terms = {}
    for ci in cons:
        c = f.constraints[ci]
        w = float(c.weight) if weights is None else float(weights[ci])
        sl = cslots[ci]
        v = [a[i] if k == "b" else d[i] for k, i in sl]
        E, dE = constraint_expectation_and_gradient(c, v)
        terms[ci] = E
        C += w * E
        for s, (k, i) in enumerate(sl):
            if k == "b":
                ga[i] += w * dE[s]
            else:
                for j, dij in dd[i]:
                    gb[j] += w * dE[s] * dij
    if want_terms:
        return C, ga, gb, terms
    return C, ga, gb


def objective_and_gradient_grouped(f, a, b, kappa, weights=None, subset=None, want_terms=False):
    """Same sums as objective_and_gradient, with E_c evaluated by the sparse xWFE (O2: Eq.8
    with the Cor.1 coefficients) batched over constraints that share a shape.  Used for the
    large structured configs; pinned against objective_and_gradient in the oracle tests.
    Symmetric constraints with many slots use the O3 path per constraint.
    """
    from .expectation import cached_table, wfe_coefficients, wfe_sparse, wfe_sparse_eval, is_distinct_symmetric
    from .semantics import shape_key
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    cons = list(range(len(f.constraints))) if subset is None else list(subset)
    groups = {}
    cslots = {}
    needed = set()
    for ci in cons:
        c = f.constraints[ci]
        sl = slots(c)
        cslots[ci] = sl
        needed.update(i for k, i in sl if k == "a")
        groups.setdefault(shape_key(c) + "#" + "".join(k for k, _ in sl), []).append(ci)
    d, dd = smoothed_atoms(f, b, kappa, sorted(needed))
    Eall, dEall = {}, {}
    for members in groups.values():
        c0 = f.constraints[members[0]]
        s = len(cslots[members[0]])
        V = np.array([[a[i] if k == "b" else d[i] for k, i in cslots[ci]] for ci in members]).reshape(len(members), s)
        if (is_distinct_symmetric(c0) and s > 12) or s > 24:
            for t, ci in enumerate(members):
                Eall[ci], dEall[ci] = constraint_expectation_and_gradient(f.constraints[ci], V[t])
        else:
            masks, vals = wfe_sparse(wfe_coefficients(cached_table(c0)))
            E, dE = wfe_sparse_eval(masks, vals, s, V)
            for t, ci in enumerate(members):
                Eall[ci], dEall[ci] = float(E[t]), dE[t]
    C = 0.0
    ga = np.zeros(f.n_bool)
    gb = np.zeros(f.n_real)
    for ci in cons:                      # accumulate in constraint order
        w = float(f.constraints[ci].weight) if weights is None else float(weights[ci])
        E, dE = Eall[ci], dEall[ci]
        C += w * E
        for s_, (k, i) in enumerate(cslots[ci]):
            if k == "b":
                ga[i] += w * dE[s_]
            else:
                for j, dij in dd[i]:
                    gb[j] += w * dE[s_] * dij
    if want_terms:
        return C, ga, gb, Eall
    return C, ga, gb
