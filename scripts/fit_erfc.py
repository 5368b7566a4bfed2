#!/usr/bin/env python
"""Derive the JIT sweep's short erfc coefficients (tiles.cpp kErfcPrelude) and report their
fp32 accuracy.  Two branches split at z = 0.75 (z = |u| >= 0):

  small:  0.5 erfc(z) = 0.5 (1 - z P(z^2)),      P ~ erf(z)/z          (degree 5 in z^2)
  tail:   0.5 erfc(z) = t Q(t) exp(-z^2),        Q ~ 0.5 erfcx(z) / t  (degree 7 in t),
          t = 1 / (1 + z/2), so exp(-z^2) is the dd/db factor already computed

Near-minimax fits by iteratively reweighted least squares (absolute error for P, relative for
Q) against scipy.special in fp64; the fp32 evaluation error is measured on a dense grid.

  python scripts/fit_erfc.py
"""
import numpy as np
from scipy.special import erf, erfc, erfcx

CUT = 0.75
DEG_SMALL, DEG_TAIL = 5, 7


def irls(x, f, deg, rel, iters=80):
    V = np.vander(x, deg + 1, increasing=True)
    w = 1 / np.abs(f) if rel else np.ones_like(f)
    for _ in range(iters):
        c, *_ = np.linalg.lstsq(V * w[:, None], f * w, rcond=None)
        r = (V @ c - f) / (np.abs(f) if rel else 1.0)
        w = w * (1 + 40 * np.abs(r) / np.abs(r).max())
        w /= w.max()
    return c


def horner32(c, x):
    c = c.astype(np.float32)
    q = np.full_like(x, c[-1])
    for k in range(len(c) - 2, -1, -1):
        q = (q * x + c[k]).astype(np.float32)
    return q


def main():
    zs = CUT * 0.5 * (1 - np.cos(np.linspace(0, np.pi, 6000)))
    zs = zs[zs > 1e-7]
    p = irls(zs * zs, erf(zs) / zs, DEG_SMALL, rel=False)
    tmax = 1 / (1 + CUT / 2)
    tt = tmax * 0.5 * (1 - np.cos(np.linspace(0, np.pi, 6000)))
    tt = tt[tt > 1e-6]
    q = irls(tt, 0.5 * erfcx(2 * (1 / tt - 1)) / tt, DEG_TAIL, rel=True)
    z = np.linspace(0, 12, 400001).astype(np.float32)
    small = z < CUT
    z2 = (z * z).astype(np.float32)
    ps = (np.float32(0.5) * (np.float32(1) - (z * horner32(p, z2)).astype(np.float32))).astype(np.float32)
    t = (np.float32(1) / (np.float32(0.5) * z + np.float32(1))).astype(np.float32)
    ez = np.exp(-z.astype(np.float64) ** 2).astype(np.float32)
    pt = (t * horner32(q, t) * ez).astype(np.float32)
    got = np.where(small, ps, pt).astype(np.float64)
    want = 0.5 * erfc(z.astype(np.float64))
    print("P (small, z^2):", ", ".join("%.9e" % v for v in p.astype(np.float32)))
    print("Q (tail, t):   ", ", ".join("%.9e" % v for v in q.astype(np.float32)))
    print("max abs error on 0.5 erfc (fp32 evaluation, exact exp):", np.abs(got - want).max())


if __name__ == "__main__":
    main()
