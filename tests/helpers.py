"""Shared test helpers: tolerances and sub-formula extraction for sampled
full-size parity (the oracle only parses the constraints it needs)."""
from __future__ import annotations

import re

import numpy as np

_ATOM_TOK = re.compile(r"a(\d+)")


def check_objective(gpu, orc, alpha, rel=1e-4, what=""):
    """Reading R27: |dC| <= 1e-4 |C_orc| when |C_orc| >= 0.01 alpha, else <= 1e-6 alpha."""
    gpu = np.asarray(gpu, dtype=np.float64)
    orc = np.asarray(orc, dtype=np.float64)
    assert np.all(np.isfinite(gpu)), f"{what}: non-finite objective"
    bar = np.where(np.abs(orc) >= 0.01 * alpha, rel * np.abs(orc), 1e-6 * alpha)
    err = np.abs(gpu - orc)
    assert np.all(err <= bar), f"{what}: objective error {err.max():.3e} > bar (worst idx {int(np.argmax(err - bar))})"


def check_gradient(gpu, orc, atol=1e-5, scale_relative=False, what=""):
    """Reading R28: |dg| <= 1e-5 (unit weights, kappa <= 2); else 1e-5 * max(1, ||g||_inf)."""
    gpu = np.asarray(gpu, dtype=np.float64)
    orc = np.asarray(orc, dtype=np.float64)
    assert np.all(np.isfinite(gpu)), f"{what}: non-finite gradient"
    bar = atol * (max(1.0, float(np.max(np.abs(orc)))) if scale_relative and orc.size else 1.0)
    err = np.abs(gpu - orc)
    assert err.size == 0 or err.max() <= bar, f"{what}: gradient error {err.max():.3e} > {bar:.3e}"


def subformula(text, bool_vars=(), real_vars=(), extra_constraints=()):
    """HSMT text restricted to the constraints touching the given variables.

    Keeps the header (same variable numbering); atoms referenced by the kept
    constraints are renumbered densely.  Returns (sub_text, original constraint indices).
    """
    lines = [ln for ln in text.splitlines() if ln.strip() and not ln.lstrip().startswith("#")]
    header = lines[0]
    atoms = {}
    cons = []
    for ln in lines[1:]:
        if ln.startswith("a "):
            parts = ln.split()
            atoms[int(parts[1])] = parts
        else:
            cons.append(ln)
    bset = set(int(i) for i in bool_vars)
    rset = set(int(j) for j in real_vars)
    hot_atoms = {aid for aid, p in atoms.items() if any(int(t.split(":")[0]) in rset for t in p[4:])}
    keep = []
    extra = set(int(c) for c in extra_constraints)
    if not bset and not rset:                    # constraints by index only: no scan
        keep = sorted(extra)
        cons_iter = ()
    else:
        cons_iter = enumerate(cons)
    for ci, ln in cons_iter:
        toks = re.findall(r"[+-]?[ab]\d+", ln)
        hit = ci in extra
        for t in toks:
            t = t.lstrip("+-")
            if (t[0] == "b" and int(t[1:]) in bset) or (t[0] == "a" and int(t[1:]) in hot_atoms):
                hit = True
                break
        if hit:
            keep.append(ci)
    used = []
    seen = {}
    out_cons = []
    for ci in keep:
        ln = cons[ci]

        def ren(m):
            aid = int(m.group(1))
            if aid not in seen:
                seen[aid] = len(used)
                used.append(aid)
            return "a" + str(seen[aid])
        body = ln.split(None, 1)
        if ln.startswith("e "):
            w, expr = ln[2:].split(None, 1)
            out_cons.append("e " + w + " " + re.sub(r"(?<![a-z])a(\d+)", ren, expr))
        else:
            out_cons.append(re.sub(r"(?<=[+-])a(\d+)", ren, ln))
    out_atoms = []
    for new, aid in enumerate(used):
        p = atoms[aid]
        out_atoms.append(" ".join(["a", str(new)] + p[2:]))
    return "\n".join([header] + out_atoms + out_cons) + "\n", keep
