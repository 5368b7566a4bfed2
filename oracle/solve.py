"""Alg.2 (CLS with annealing) around Alg.1 — oracle, test infrastructure only.

Followed step by step per restart r (restarts are independent):

    init (R20)  a_i <- ((2k+1) - 2^24) 2^-24,  k = Philox(seed; r, i, 0, 0).out0 >> 8
                b_j <- lo_j + (hi_j - lo_j) u (both bounds finite) | 2u - 1 (otherwise),
                       u = (2k+1) 2^-25, k from tag 1; computed in fp64, rounded once to fp32
                (a, b) <- proj(a, b)
    h_c <- 0, w_c <- 1                                          (Alg.2 line 1)
    for t = 1..T  (kappa_t = 1/sigma_t)
        for s = 1..S                                            (Alg.1 while loop, capped: R21)
            g <- grad C(a, b; kappa_t, w)                       (Eq.10, Alg.B with R1)
            (a', b') <- proj((a, b) - eta g)                    (Eq.11-12)
            gm <- ((a, b) - (a', b')) / eta                     (Eq.13)
            if ||gm||^2 <= eps^2: break                         (Eq.14)
            (a, b) <- (a', b')
        (x, y) <- (round(a), b)                                 (Alg.2 line 4; R17)
        for c: u_c <- [f_c(x, y) = +1]; h_c <- rho h_c + u_c; #Unsat += u_c
               if t mod tau = 0: w_c <- w_c gamma^{h_c}; h_c <- 1 (Alg.2 verbatim; R18)
        if #Unsat = 0: return SAT(x, y)
    return UNKNOWN(best)

proj (Def.1/Prop.1; reading R15): a clamped to [-1, 1]; b_j clamped
to [lo_j, hi_j] derived from single-variable unit-atom constraints; other unit
atoms stay soft (objective only, R16).  Bounds are the tightest fp32 values at
which the unit literal holds under the exact check (R15b).
rho = 0.5, gamma = 2, tau = 1.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import philox
from .objective import objective_and_gradient
from .semantics import constraint_sat, eval_atom, slots, truth_table

RHO = 0.5
GAMMA = 2.0
TAU = 1


@dataclass
class Params:
    kappas: list = field(default_factory=lambda: [round(0.1 * i, 10) for i in range(1, 21)])  # R12
    steps: int = 50
    eta: float = 0.05
    eps: float = 1e-2            # P:165, R14
    rounding: str = "sign"       # "sign" | "philox"  (R17)
    erwa_mode: int = 0           # 0: Alg.2 verbatim (h <- 1); 1: reset-to-0 reading (R18)
    eta_mode: int = 0            # 0 eta; 1 eta/kappa; 2 eta/kappa^2; 3 eta for a, eta/kappa^2 for b (R13)
    proj_iters: int = 0          # 0: R15 interval clamps; > 0: Prop.1 QP by that many Dykstra sweeps (R33)
    n_roundings: int = 1         # R34: draws of R(a) per stage with Philox rounding; the best one is kept


# ----------------------------------------------------------------------------- projection bounds


def unit_literal(f, c):
    """(atom_id, positive?) if c is a unit atomic constraint (Prop.1), else None.

    A constraint over exactly one slot, which is an atom, whose truth table is
    'sat iff atom True' (positive) or 'sat iff atom False' (negative).
    """
    sl = slots(c)
    if len(sl) != 1 or sl[0][0] != "a":
        return None
    t = truth_table(c)          # index 0: atom False, index 1: atom True
    if bool(t[1]) and not bool(t[0]):
        return sl[0][1], True
    if bool(t[0]) and not bool(t[1]):
        return sl[0][1], False
    return None


def _f32(x):
    return np.float32(x)


def _holds(atom, positive, j, yv):
    y = {j: float(yv)}
    ok = eval_atom(atom, y)
    return ok if positive else not ok


def bounds(f):
    """Per-real [lo_j, hi_j] as fp32 values (reading R15/R15b)."""
    lo = [np.float32(-np.inf)] * f.n_real
    hi = [np.float32(np.inf)] * f.n_real
    for c in f.constraints:
        u = unit_literal(f, c)
        if u is None:
            continue
        aid, positive = u
        atom = f.atoms[aid]
        if len(atom.coeffs) != 1:
            continue                       # multi-variable unit atom: soft (R15)
        j, q = atom.coeffs[0]
        upper = (q > 0) == positive        # literal bounds y_j from above?
        t = _f32(atom.rhs / q)
        if upper:
            # largest fp32 y with the literal holding
            while _holds(atom, positive, j, np.nextafter(t, np.float32(np.inf))):
                t = np.nextafter(t, np.float32(np.inf))
            while not _holds(atom, positive, j, t):
                t = np.nextafter(t, np.float32(-np.inf))
            hi[j] = min(hi[j], t)
        else:
            while _holds(atom, positive, j, np.nextafter(t, np.float32(-np.inf))):
                t = np.nextafter(t, np.float32(-np.inf))
            while not _holds(atom, positive, j, t):
                t = np.nextafter(t, np.float32(np.inf))
            lo[j] = max(lo[j], t)
    return np.array(lo, dtype=np.float32), np.array(hi, dtype=np.float32)


def project(a, b, lo, hi, H=None, proj_iters=0):
    """Def.1 / Prop.1: a clamped to [-1, 1]; b clamped to the R15 intervals, or (R33, proj_iters > 0
    and multi-variable unit atoms present) projected by Dykstra onto intervals and halfspaces."""
    a2 = np.clip(a, -1.0, 1.0)
    if H and proj_iters > 0:
        from .projection import dykstra
        return a2, dykstra(np.asarray(b, dtype=np.float64), lo, hi, H, proj_iters)
    return a2, np.minimum(np.maximum(b, lo.astype(np.float64)), hi.astype(np.float64))


# ----------------------------------------------------------------------------- init / rounding


def init_point(f, seed, r, lo, hi, H=None, proj_iters=0):
    """Reading R20; returns fp32-representable (a, b) as fp64 arrays."""
    a = np.empty(f.n_bool)
    for i in range(f.n_bool):
        k = philox.draw24(seed, r, i, 0, philox.TAG_INIT_A)
        a[i] = ((2 * k + 1) - 2 ** 24) * 2.0 ** -24
    b = np.empty(f.n_real)
    for j in range(f.n_real):
        k = philox.draw24(seed, r, j, 0, philox.TAG_INIT_B)
        u = (2 * k + 1) * 2.0 ** -25
        l, h = float(lo[j]), float(hi[j])
        if math.isfinite(l) and math.isfinite(h):
            v = l + (h - l) * u
        else:
            v = 2.0 * u - 1.0
        b[j] = float(np.float32(v))
    a, b = project(a, b, lo, hi, H, proj_iters)
    return a, b


def round_sign(a):
    """x = sgn(a) with sgn(0) = +1 (Alg.1 line 10): -1 iff a < 0."""
    return np.where(np.asarray(a) < 0.0, -1, 1).astype(np.int8)


def round_philox(a, seed, r, t):
    """Randomised rounding R(a) (Eq.4; reading R17): -1 iff a < 1 - k 2^-23.

    t is the Philox stage word: stage t's m-th draw (R34) uses t + (m << 16)."""
    x = np.empty(len(a), dtype=np.int8)
    for i, ai in enumerate(a):
        k = philox.draw24(seed, r, i, t, philox.TAG_ROUND)
        x[i] = -1 if float(ai) < 1.0 - k * 2.0 ** -23 else 1
    return x


def violations(f, x, y):
    """u_c = (1/2) f_c(x, y) + 1/2 (Alg.2 line 7): 1 iff c violated (exact, R22)."""
    return np.array([0 if constraint_sat(f, c, x, y) else 1 for c in f.constraints], dtype=np.int64)


# ----------------------------------------------------------------------------- PGD step (for replay)


def pgd_step(f, a, b, kappa, w, eta, lo, hi, eta_b=None, H=None, proj_iters=0):
    """One Alg.1 iteration: returns (a', b', ||gm||^2, C) at (a, b) (Eq.11-14).

    eta_b: optional separate step for the real block (eta_mode 3 reading); default eta.
    H, proj_iters: the R33 projection (oracle/projection.py); default the R15 clamps.
    """
    eta_b = eta if eta_b is None else eta_b
    C, ga, gb = objective_and_gradient(f, a, b, kappa, w)
    a2, b2 = project(np.asarray(a) - eta * ga, np.asarray(b) - eta_b * gb, lo, hi, H, proj_iters)
    gm2 = float(np.sum(((np.asarray(a) - a2) / eta) ** 2) + np.sum(((np.asarray(b) - b2) / eta_b) ** 2))
    return a2, b2, gm2, C


# ----------------------------------------------------------------------------- Alg.2


@dataclass
class RestartResult:
    sat_stage: int          # first stage whose rounded model satisfies all constraints, 0 = never
    x: np.ndarray
    y: np.ndarray
    unsat: int              # unsat count of the returned model
    best_stage: int         # stage at which the returned model was found
    history: list           # per stage: (kappa, steps_taken, unsat)


def solve_restart(f, seed, r, params: Params, lo=None, hi=None):
    if lo is None:
        lo, hi = bounds(f)
    from .projection import halfspaces
    H = halfspaces(f) if params.proj_iters > 0 else None
    a, b = init_point(f, seed, r, lo, hi, H, params.proj_iters)
    C_n = len(f.constraints)
    h = np.zeros(C_n)
    w = np.array([c.weight for c in f.constraints], dtype=np.float64)   # initial w_c (Alg.2 input)
    best = None
    hist = []
    for t, kappa in enumerate(params.kappas, start=1):
        taken = 0
        kk = max(kappa, 1.0)
        eta_t = params.eta / kk ** min(params.eta_mode, 2)
        eta_b = params.eta / kk ** 2 if params.eta_mode >= 2 else eta_t
        if params.eta_mode == 3:
            eta_t = params.eta
        for _ in range(params.steps):
            a2, b2, gm2, _ = pgd_step(f, a, b, kappa, w, eta_t, lo, hi, eta_b, H, params.proj_iters)
            if gm2 <= params.eps ** 2:
                break
            a, b = a2, b2
            taken += 1
        y = np.asarray(b, dtype=np.float32)
        if params.rounding == "sign":
            x = round_sign(a)
            u = violations(f, x, y)
        else:
            # R34: n_roundings draws of R(a), the first with the fewest violations kept
            x, u = None, None
            for m in range(max(1, params.n_roundings)):
                xm = round_philox(a, seed, r, t + (m << 16))
                um = violations(f, xm, y)
                if u is None or um.sum() < u.sum():
                    x, u = xm, um
        n_unsat = int(u.sum())
        for c in range(C_n):
            h[c] = RHO * h[c] + u[c]
            if t % TAU == 0:
                w[c] = w[c] * GAMMA ** h[c]
                h[c] = 1.0 if params.erwa_mode == 0 else 0.0
        hist.append((kappa, taken, n_unsat))
        if best is None or n_unsat < best[0]:
            best = (n_unsat, x.copy(), y.copy(), t)
        if n_unsat == 0:
            return RestartResult(t, x, y, 0, t, hist)
    return RestartResult(0, best[1], best[2], best[0], best[3], hist)


def solve(f, restarts, seed, params: Params, restart_offset=0):
    """Lock-step semantics: SAT at the lexicographically smallest (stage, restart)."""
    lo, hi = bounds(f)
    results = [solve_restart(f, seed, restart_offset + r, params, lo, hi) for r in range(restarts)]
    sat = [(res.sat_stage, r) for r, res in enumerate(results) if res.sat_stage > 0]
    if sat:
        t, r = min(sat)
        return "SAT", r, results
    # best model: lexicographically smallest (unsat, stage, restart)
    r = min(range(restarts), key=lambda i: (results[i].unsat, results[i].best_stage, i))
    return "UNKNOWN", r, results
