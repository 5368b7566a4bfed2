"""Pins of the fp64 oracle against what the paper and mathematics fix (CPU only).

Each test names the passage it pins.  A plausible mistake anywhere in the
oracle (dropped term, wrong sign or index, transposed operand) must fail one of
these.
"""
import json
import math
import os
from itertools import product

import numpy as np
import pytest

from oracle import hsmt, philox, semantics, smoothing, expectation, objective, robdd, bruteforce, solve
import fsmt_gen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


def hx(v):
    return int(v, 16) if isinstance(v, str) else int(v)


# ----------------------------------------------------------------------------- Philox (R17, R20)

def test_philox_known_answers():
    g = load("philox_kat.json")
    for case in g["kat"]:
        out = philox.philox4x32_10([hx(c) for c in case["ctr"]], [hx(k) for k in case["key"]])
        assert [f"{o:08x}" for o in out] == case["out"]


def test_philox_usage_examples():
    g = load("philox_kat.json")["usage"]
    seed = int(g["seed"], 16)
    i = g["init"]
    out0 = philox.philox4x32_10((i["restart"], i["var"], i["stage"], i["tag"]), philox.key_of(seed))[0]
    assert f"{out0:08x}" == i["out0"]
    k = philox.draw24(seed, i["restart"], i["var"], i["stage"], i["tag"])
    assert k == i["k"]
    assert ((2 * k + 1) - 2 ** 24) * 2.0 ** -24 == i["a"]
    r = g["round"]
    k = philox.draw24(seed, r["restart"], r["var"], r["stage"], r["tag"])
    assert k == r["k"] and 1.0 - k * 2.0 ** -23 == r["threshold"]


# ----------------------------------------------------------------------------- parser

def test_parser_examples_and_errors():
    f = hsmt.parse("p hsmt 1 1\na 0 <= 0 0:1\ne 1 (and b0 a0)")
    assert f.n_bool == 1 and f.n_real == 1 and len(f.atoms) == 1 and f.constraints[0].kind == "expr"
    f = hsmt.parse("p hsmt 2 0\nc xor 1 +b0 +b1")
    assert f.constraints[0].kind == "xor" and f.constraints[0].weight == 1.0
    for bad in ["p hsmt 0 1\na 0 = 0 0:1", "p hsmt 1 0\nc or 0 +b0", "p hsmt 1 0\nc or 1", "p hsmt 1 0\nc or 1 +b3",
                "c or 1 +b0", "p hsmt 1 1\na 0 <= 0 0:0", "p hsmt 1 1\na 1 <= 0 0:1", "p hsmt 1 0\ne 1 (foo b0)"]:
        with pytest.raises(hsmt.HsmtError):
            hsmt.parse(bad)


def test_canonicalisation_preserves_truth():
    # canonicalisation preserves eval_atom on random (atom, y) pairs
    rng = np.random.default_rng(0)
    for _ in range(300):
        rel = rng.choice(["<=", "<", ">=", ">"])
        q = rng.integers(-3, 4, size=3)
        q[q == 0] = 1
        q0 = float(rng.integers(-4, 5)) / 2
        y = rng.integers(-4, 5, size=3) / 2.0
        f = hsmt.parse(f"p hsmt 0 3\na 0 {rel} {q0} 0:{q[0]} 1:{q[1]} 2:{q[2]}")
        lhs = float(q @ y)
        want = {"<=": lhs <= q0, "<": lhs < q0, ">=": lhs >= q0, ">": lhs > q0}[rel]
        assert semantics.eval_atom(f.atoms[0], y) == want


def test_eval_examples_spec():
    # S:73-75
    f = hsmt.parse("p hsmt 0 1\na 0 <= 0 0:1\na 1 < 0 0:1")
    assert semantics.eval_atom(f.atoms[0], [-0.5]) and semantics.eval_atom(f.atoms[0], [0.0])
    assert not semantics.eval_atom(f.atoms[1], [0.0])
    f = hsmt.parse("p hsmt 3 0\nc xor 1 +b0 +b1\nc card 1 1 +b0 +b1 +b2")
    assert not semantics.constraint_sat(f, f.constraints[0], [-1, -1, 1], [])
    assert not semantics.constraint_sat(f, f.constraints[1], [-1, -1, 1], [])
    assert semantics.eval_formula(hsmt.parse("p hsmt 0 0\n"), [], []) == (0.0, [])


# ----------------------------------------------------------------------------- smoothing (Eq.7)

def test_smoothing_spec_values():
    f = hsmt.parse("p hsmt 0 1\na 0 <= 0 0:1\na 1 <= 0 0:2")
    assert abs(smoothing.atom_smooth(f.atoms[0], [1.0], 1.0) - 0.682689) < 1e-6
    assert smoothing.atom_smooth(f.atoms[0], [0.0], 1.0) == 0.0
    assert smoothing.atom_smooth(f.atoms[0], [-0.3], math.inf) == -1.0                     # S:302 (sigma=0)
    assert smoothing.atom_smooth(f.atoms[0], [0.7], 0.0) == 0.0                            # R11 kappa = 0
    g = smoothing.atom_smooth_grad(f.atoms[0], [0.0], 1.0)[0][1]
    assert abs(g - 0.797885) < 1e-6
    g2 = smoothing.atom_smooth_grad(f.atoms[1], [0.0], 1.0)[0][1]
    assert abs(g2 - 0.797885) < 1e-6                                                       # S:309 scale invariance


def test_smoothing_gradient_fd_and_erratum():
    # R2: P:1326-1327 is right, P:855-858 is not. q=(1,-2), q0=0.3, b=(0.2,-0.1), sigma=0.8
    f = hsmt.parse("p hsmt 0 2\na 0 <= 0.3 0:1 1:-2")
    at = f.atoms[0]
    b = np.array([0.2, -0.1])
    kappa = 1 / 0.8
    h = 1e-6
    for j in range(2):
        bp, bm = b.copy(), b.copy()
        bp[j] += h
        bm[j] -= h
        fd = (smoothing.atom_smooth(at, bp, kappa) - smoothing.atom_smooth(at, bm, kappa)) / (2 * h)
        an = smoothing.atom_smooth_grad(at, b, kappa)[j][1]
        assert abs(fd - an) <= 1e-7 * max(1, abs(fd))
    fd0 = smoothing.atom_smooth_grad(at, b, kappa)[0][1]
    assert abs(fd0 - 0.445335) < 1e-6
    # the printed P:855-858 exponent gives 0.444271 (must NOT be what the oracle computes)
    z = 0.2 - 2 * -0.1 - 0.3
    nq = math.sqrt(5)
    printed = math.sqrt(2) * 1 / (math.sqrt(math.pi * 5) * 0.8) * math.exp(-z * z / (math.sqrt(2) * nq * 0.8))
    assert abs(printed - 0.444271) < 1e-6 and abs(printed - fd0) > 1e-3


def test_smoothing_monte_carlo():
    # Eq.7 first line: d = E_{y~N(b, sigma^2)} delta(y)
    f = hsmt.parse("p hsmt 0 2\na 0 <= 0.3 0:1 1:-2")
    rng = np.random.default_rng(1)
    b = np.array([0.4, 0.1])
    sigma = 0.6
    ys = b + sigma * rng.standard_normal((400000, 2))
    delta = np.where(ys @ np.array([1.0, -2.0]) <= 0.3, -1.0, 1.0)
    est, se = delta.mean(), delta.std() / math.sqrt(len(delta))
    assert abs(smoothing.atom_smooth(f.atoms[0], b, 1 / sigma) - est) < 4 * se


def test_round_prob():
    assert [smoothing.round_prob(a) for a in (-1, 0, 0.5, 1)] == [1.0, 0.5, 0.25, 0.0]


# ----------------------------------------------------------------------------- expectation (Eq.8, Cor.1)

def _c(text):
    f = hsmt.parse(text)
    return f, f.constraints[0]


def test_wfe_tables_spec():
    # S:145-147
    _, c = _c("p hsmt 2 0\nc or 1 +b0 +b1")
    coef = expectation.wfe_coefficients(semantics.truth_table(c))
    assert np.allclose(coef, [-0.5, 0.5, 0.5, 0.5])          # masks {}, {0}, {1}, {0,1}
    _, c = _c("p hsmt 2 0\nc xor 1 +b0 +b1")
    assert np.allclose(expectation.wfe_coefficients(semantics.truth_table(c)), [0, 0, 0, 1])
    _, c = _c("p hsmt 1 0\nc or 1 +b0")
    assert np.allclose(expectation.wfe_coefficients(semantics.truth_table(c)), [0, 1])


def test_expectation_spec_values():
    _, c = _c("p hsmt 2 0\nc or 1 +b0 +b1")
    t = semantics.truth_table(c)
    assert abs(expectation.enum_expectation(t, [0, 0]) + 0.5) < 1e-15
    # d sat / dp = (0.5, 0.5) at p=(.5,.5): dE/dv = dsat/dp (R1)
    assert np.allclose(expectation.enum_gradient(t, [0, 0]), [0.5, 0.5])
    _, c = _c("p hsmt 2 0\nc xor 1 +b0 +b1")
    t = semantics.truth_table(c)
    assert abs(expectation.enum_expectation(t, [0.5, -0.5]) + 0.25) < 1e-15
    # XOR p=(0.3,0.5) -> dsat/dp = (0, 0.4); v = 1 - 2p
    assert np.allclose(expectation.enum_gradient(t, [1 - 0.6, 1 - 1.0]), [0.0, 0.4])
    assert abs(expectation.enum_expectation(t, [0, 0]) - 0.0) < 1e-15                      # sat 0.5
    _, c = _c("p hsmt 3 0\nc card 1 1 +b0 +b1 +b2")
    E, _ = expectation.sym_expectation_and_gradient(c, [0, 0, 0])
    assert abs((1 - E) / 2 - 0.5) < 1e-15
    _, c = _c("p hsmt 2 0\nc nae 1 +b0 +b1")
    E, _ = expectation.sym_expectation_and_gradient(c, [0, 0])
    assert abs((1 - E) / 2 - 0.5) < 1e-15
    _, c = _c("p hsmt 2 0\nc xor 1 +b0 +b1")
    E, _ = expectation.sym_expectation_and_gradient(c, [-1, -1])
    assert abs((1 - E) / 2 - 0.0) < 1e-15


def _closed_forms(kind, L, k, v, neg):
    lv = [(-x if n else x) for x, n in zip(v, neg)]    # literal relaxed values
    pt = [(1 - x) / 2 for x in lv]                      # P[literal true]
    if kind == "xor":
        return float(np.prod(lv))
    if kind == "or":
        return -1 + 2 * float(np.prod([1 - p for p in pt]))
    if kind == "nae":
        return -1 + 2 * (float(np.prod(pt)) + float(np.prod([1 - p for p in pt])))
    if kind == "card":   # 1 - 2 P[#true <= k]; by brute force over the binomial pattern
        tot = 0.0
        for bits in product([0, 1], repeat=L):
            if sum(bits) <= k:
                tot += float(np.prod([p if b else 1 - p for p, b in zip(pt, bits)]))
        return 1 - 2 * tot
    raise ValueError


@pytest.mark.parametrize("kind", ["xor", "or", "nae", "card"])
def test_symmetric_closed_forms_all_paths(kind):
    rng = np.random.default_rng(hash(kind) % 1000)
    for L in (1, 2, 3, 5, 7):
        for _ in range(4):
            k = int(rng.integers(0, L + 1))
            neg = rng.random(L) < 0.5
            lits = " ".join(("-" if n else "+") + f"b{i}" for i, n in enumerate(neg))
            head = f"c card {k} 1" if kind == "card" else f"c {kind} 1"
            f, c = _c(f"p hsmt {L} 0\n{head} {lits}")
            v = rng.uniform(-1, 1, L)
            want = _closed_forms(kind, L, k, v, neg)
            t = semantics.truth_table(c)
            assert abs(expectation.enum_expectation(t, v) - want) < 1e-13
            assert abs(expectation.contract_expectation(t, v) - want) < 1e-13
            assert abs(expectation.wfe_expectation(expectation.wfe_coefficients(t), v) - want) < 1e-13
            E3, g3 = expectation.sym_expectation_and_gradient(c, v)
            assert abs(E3 - want) < 1e-13
            g1 = expectation.enum_gradient(t, v)
            assert np.allclose(g1, g3, atol=1e-13) and np.allclose(g1, expectation.contract_gradient(t, v), atol=1e-13)
            # central finite differences of the closed form
            h = 1e-6
            for s in range(L):
                vp, vm = v.copy(), v.copy()
                vp[s] += h
                vm[s] -= h
                fd = (_closed_forms(kind, L, k, vp, neg) - _closed_forms(kind, L, k, vm, neg)) / (2 * h)
                assert abs(fd - g1[s]) < 1e-8


def test_parseval_vertex_exactness_range():
    # S:134; range lemma P:1620-1626
    rng = np.random.default_rng(5)
    for _ in range(40):
        s = int(rng.integers(1, 9))
        ops = ["and", "or", "xor"]

        def rnd(depth):
            if depth == 0 or rng.random() < 0.3:
                i = int(rng.integers(0, s))
                leaf = f"b{i}" if i % 2 == 0 else f"a{i // 2}"
                return f"(not {leaf})" if rng.random() < 0.4 else leaf
            return "(" + ops[int(rng.integers(0, 3))] + " " + " ".join(rnd(depth - 1) for _ in range(int(rng.integers(2, 4)))) + ")"
        atoms = "\n".join(f"a {i} <= 0 0:1" for i in range(s))
        f = hsmt.parse(f"p hsmt {s} 1\n{atoms}\ne 1 {rnd(3)}")
        c = f.constraints[0]
        t = semantics.truth_table(c)
        coef = expectation.wfe_coefficients(t)
        assert abs(np.sum(coef ** 2) - 1.0) < 1e-12
        ns = len(semantics.slots(c))
        for z in product([-1.0, 1.0], repeat=ns):
            idx = sum((1 << p) for p, zz in enumerate(z) if zz == -1)
            fz = -1.0 if t[idx] else 1.0
            assert expectation.enum_expectation(t, list(z)) == fz
            assert abs(expectation.wfe_expectation(coef, list(z)) - fz) < 1e-12
        v = rng.uniform(-1, 1, ns)
        E = expectation.enum_expectation(t, v)
        assert -1.0 - 1e-15 <= E <= 1.0 + 1e-15


def test_multilinear_expectation_lemma():
    # Lemma P:802-828: E_{x~S_a} f(x) = f(a) -- the multilinear extension equals the
    # average over rounding outcomes; checked by sampling rounding outcomes.
    f, c = _c("p hsmt 4 0\ne 1 (or (xor b0 b1) (and b2 (not b3)) (xor b1 b3))")
    t = semantics.truth_table(c)
    rng = np.random.default_rng(3)
    a = rng.uniform(-1, 1, 4)
    x = np.where(rng.random((300000, 4)) < (1 - a) / 2, -1, 1)
    vals = np.array([-1.0 if semantics.constraint_sat(f, c, xi, []) else 1.0 for xi in x[:20000]])
    E = expectation.enum_expectation(t, a)
    assert abs(vals.mean() - E) < 4 * vals.std() / math.sqrt(len(vals))


# ----------------------------------------------------------------------------- objective (Eq.10)

def test_fig2_closed_form():
    g = load("fig2.json")
    f = hsmt.parse(g["hsmt"])
    for p in g["points"]:
        C, ga, gb = objective.objective_and_gradient(f, [p["a"]], [p["b"]], 1 / p["sigma"])
        assert abs(C - p["C"]) < 1e-8
        if "grad" in p:
            assert abs(ga[0] - p["grad"][0]) < 1e-8 and abs(gb[0] - p["grad"][1]) < 1e-8
    for v in g["vertices"]:
        assert semantics.eval_formula(f, [v["x"]], [v["y"]])[0] == v["F"]
    # Thm.3 / Cor.2: sigma = 0 recovers F_w at vertices
    for v in g["vertices"]:
        d = smoothing.atom_smooth(f.atoms[0], [v["y"]], math.inf)
        E = sum(expectation.enum_expectation(semantics.truth_table(c), [v["x"], d]) for c in f.constraints)
        assert E == v["F"]


def test_cfg1_values():
    g = load("cfg1_values.json")
    f = hsmt.parse(fsmt_gen.cfg1().text)
    for p in g["points"]:
        C, ga, gb, terms = objective.objective_and_gradient(f, p["a"], p["b"], 1 / p["sigma"], want_terms=True)
        assert abs(C - p["C"]) < 1e-8
        if "E" in p:
            assert np.allclose([terms[i] for i in range(6)], p["E"], atol=1e-6)
        if "grad_a" in p:
            assert np.allclose(ga, p["grad_a"], atol=1e-6) and np.allclose(gb, p["grad_b"], atol=1e-6)
    # hand re-derivation of E_0..E_2 at a=0,b=0,sigma=1: c0 = a*d = 0; c1 = 1-(1-a)(1+d)/2 = 0.5;
    # c2 = OR(b1,b2,a1): -1 + 2 (1/2)(1/2)(1+erf(-1/2))/2
    want2 = -1 + 2 * 0.5 * 0.5 * (1 + math.erf(-0.5)) / 2
    assert abs(g["points"][0]["E"][2] - want2) < 1e-6


def test_gradient_finite_differences():
    # analytic gradient vs central FD (h=1e-6) of the objective
    for name in ("cfg1", "cfg2s", "cfg4s"):
        inst = fsmt_gen.config(name)
        f = hsmt.parse(inst.text)
        rng = np.random.default_rng(7)
        a = rng.uniform(-0.9, 0.9, f.n_bool)
        b = rng.uniform(0.05, 0.95, f.n_real)
        kappa = 1.3
        w = rng.integers(1, 4, len(f.constraints)).astype(float)
        C, ga, gb = objective.objective_and_gradient(f, a, b, kappa, w)
        h = 1e-6
        for i in rng.choice(f.n_bool, size=min(4, f.n_bool), replace=False):
            ap, am = a.copy(), a.copy()
            ap[i] += h
            am[i] -= h
            fd = (objective.objective_and_gradient(f, ap, b, kappa, w)[0] - objective.objective_and_gradient(f, am, b, kappa, w)[0]) / (2 * h)
            assert abs(fd - ga[i]) <= 1e-6 * max(1.0, abs(fd))
        for j in rng.choice(f.n_real, size=min(4, f.n_real), replace=False):
            bp, bm = b.copy(), b.copy()
            bp[j] += h
            bm[j] -= h
            fd = (objective.objective_and_gradient(f, a, bp, kappa, w)[0] - objective.objective_and_gradient(f, a, bm, kappa, w)[0]) / (2 * h)
            assert abs(fd - gb[j]) <= 1e-6 * max(1.0, abs(fd))


def test_placement_template_closed_form():
    g = load("placement_template.json")
    # build the single non-overlap constraint between two modules (K = 7 bit pairs)
    K = 7
    text = (f"p hsmt {2 * K} 4\n"
            "a 0 >= 0.4 0:1 2:-1\na 1 >= 0.4 2:1 0:-1\na 2 >= 0.4 1:1 3:-1\na 3 >= 0.4 3:1 1:-1\n"
            "e 1 (or " + " ".join(f"(xor b{i} b{K + i})" for i in range(K)) + " a0 a1 a2 a3)\n")
    f = hsmt.parse(text)
    a = np.array(g["a_u"] + g["a_v"])
    b = np.array([g["xy"]["x"][0], g["xy"]["y"][0], g["xy"]["x"][1], g["xy"]["y"][1]])
    d = [smoothing.atom_smooth(at, b, g["kappa"]) for at in f.atoms]
    assert np.allclose(d, g["d_atoms"], atol=1e-9)
    C, ga, gb = objective.objective_and_gradient(f, a, b, g["kappa"])
    # closed form (independent of the oracle code path)
    au, av = np.array(g["a_u"]), np.array(g["a_v"])
    closed = -1 + 2 * np.prod((1 + au * av) / 2) * np.prod((1 + np.array(d)) / 2)
    assert abs(C - closed) < 1e-12 and abs(C - g["E"]) < 1e-9
    assert np.allclose(ga[:K], g["dE_da_u"], atol=1e-9) and np.allclose(ga[K:], g["dE_da_v"], atol=1e-9)
    assert np.allclose(gb[[0, 2]], g["dE_dx"], atol=1e-9) and np.allclose(gb[[1, 3]], g["dE_dy"], atol=1e-9)
    C10, _, _ = objective.objective_and_gradient(f, a, b, 10.0)
    assert abs(C10 - g["E_kappa10"]) < 1e-9


def test_sparse_wfe_matches_enumeration_on_template():
    inst = fsmt_gen.config("cfg4s")
    f = hsmt.parse(inst.text)
    c = f.constraints[0]
    t = semantics.truth_table(c)
    masks, vals = expectation.wfe_sparse(expectation.wfe_coefficients(t))
    s = len(semantics.slots(c))
    K = inst.meta["bits_per_module"]
    assert len(masks) == 2 ** (K + 4)          # 2^(#pairs + #atoms) nonzero terms
    rng = np.random.default_rng(2)
    V = rng.uniform(-1, 1, (5, s))
    E, dE = expectation.wfe_sparse_eval(masks, vals, s, V)
    for r in range(5):
        assert abs(E[r] - expectation.enum_expectation(t, V[r])) < 1e-13
        assert np.allclose(dE[r], expectation.enum_gradient(t, V[r]), atol=1e-13)


# ----------------------------------------------------------------------------- structure (Def.2, R7)

@pytest.mark.parametrize("L", [1, 2, 3, 5, 8])
def test_robdd_node_counts(L):
    lits = " ".join(f"+b{i}" for i in range(L))
    counts = {}
    for kind in ("xor", "or", "nae"):
        f = hsmt.parse(f"p hsmt {L} 0\nc {kind} 1 {lits}")
        _, nodes, root, _ = robdd.constraint_structure(f.constraints[0])
        counts[kind] = len(nodes)
    assert counts["xor"] == 2 * L - 1                   # S:226 (XOR_8 -> 15)
    assert counts["or"] == L                            # S:227 (OR_2 -> 2)
    assert counts["nae"] == (2 * L - 1 if L > 1 else 0)  # NAE_1 is constant False
    if L == 1:
        f = hsmt.parse("p hsmt 1 0\nc or 1 +b0")
        _, nodes, root, _ = robdd.constraint_structure(f.constraints[0])
        assert nodes == [(0, robdd.TRUE, robdd.FALSE)] and root == 0


def test_robdd_card_and_template_counts():
    def card_count(L, k):
        return sum(sum(1 for c in range(max(0, k - L + i + 1), min(i, k) + 1)) for i in range(L))
    f = hsmt.parse("p hsmt 8 0\nc card 4 1 " + " ".join(f"+b{i}" for i in range(8)))
    assert len(robdd.constraint_structure(f.constraints[0])[1]) == card_count(8, 4) == 20
    for k, t in ((4, 2), (7, 4)):
        atoms = "\n".join(f"a {i} <= 0 0:1" for i in range(t))
        body = " ".join(f"(xor b{i} b{k + i})" for i in range(k)) + " " + " ".join(f"a{i}" for i in range(t))
        f = hsmt.parse(f"p hsmt {2 * k} 1\n{atoms}\ne 1 (or {body})")
        assert len(robdd.constraint_structure(f.constraints[0])[1]) == 3 * k + t   # R6: 14 / 25


def test_robdd_semantics_and_canonical_numbering():
    inst = fsmt_gen.config("cfg2s")
    f = hsmt.parse(inst.text)
    for c in f.constraints[:25]:
        kinds, nodes, root, gids = robdd.constraint_structure(c)
        t = semantics.truth_table(c)
        s = len(gids)
        # evaluate the diagram on every vertex
        for idx in range(1 << s):
            v = root
            while v >= 0:
                lvl, hi, lo = nodes[v]
                v = hi if (idx >> lvl) & 1 else lo
            assert (v == robdd.TRUE) == bool(t[idx])
        # reduced + ordered + canonical order
        assert len(set(nodes)) == len(nodes) and all(n[1] != n[2] for n in nodes)
        assert all(n[0] < nodes[ch][0] for n in nodes for ch in (n[1], n[2]) if ch >= 0)
        assert [n[0] for n in nodes] == sorted(n[0] for n in nodes)


# ----------------------------------------------------------------------------- soundness / brute force (Thm.1)

def test_fourier_motzkin_spec():
    # S:168-170
    F = bruteforce.fm_feasible
    from fractions import Fraction as Fr
    assert F([({0: Fr(1)}, Fr(0), False), ({0: Fr(-1)}, Fr(-1), False)], 1) is None
    w = F([({0: Fr(1)}, Fr(1), False), ({0: Fr(-1)}, Fr(0), False)], 1)
    assert w is not None and 0 <= w[0] <= 1
    w = F([({0: Fr(1), 1: Fr(-1)}, Fr(-1), False), ({1: Fr(1)}, Fr(0), False)], 2)
    assert w is not None and w[0] - w[1] <= -1 and w[1] <= 0
    assert F([({0: Fr(1)}, Fr(0), True), ({0: Fr(-1)}, Fr(0), False)], 1) is None     # y<0 and y>=0


def test_brute_force_cfg1_and_toys():
    g = load("cfg1_values.json")["brute_force"]
    f = hsmt.parse(fsmt_gen.cfg1().text)
    assert bruteforce.brute_force_sat(f) is not None
    assert bruteforce.count_models(f) == g["n_models"]
    obj, sat = semantics.eval_formula(f, g["witness_x"], g["witness_y"])
    assert all(sat) and obj == -6.0                                          # Thm.1: F_w = -sum w
    assert bruteforce.brute_force_sat(hsmt.parse("p hsmt 1 0\nc or 1 +b0\nc or 1 -b0")) is None
    assert bruteforce.brute_force_sat(hsmt.parse("p hsmt 0 1\na 0 <= 0 0:1\nc or 1 +a0\nc or 1 -a0")) is None
    fig2 = hsmt.parse(load("fig2.json")["hsmt"])
    x, y = bruteforce.brute_force_sat(fig2)
    assert x == [-1] and y[0] > 0


def test_min_vertex_objective_iff_sat():
    # Thm.1: min over vertices of F_w = -sum w iff satisfiable, on random tiny formulas
    rng = np.random.default_rng(11)
    for trial in range(25):
        nb = 3
        lines = ["p hsmt 3 1", "a 0 <= 0 0:1", "a 1 <= 1 0:1"]
        for _ in range(int(rng.integers(2, 6))):
            L = int(rng.integers(1, 4))
            pool = rng.choice(5, size=L, replace=False)
            lits = " ".join(("-" if rng.random() < .5 else "+") + (f"b{p}" if p < 3 else f"a{p - 3}") for p in pool)
            lines.append(f"c {rng.choice(['or', 'xor', 'nae'])} 1 {lits}")
        f = hsmt.parse("\n".join(lines))
        model = bruteforce.brute_force_sat(f)
        best = min(semantics.eval_formula(f, list(x), [y])[0]
                   for x in product([-1, 1], repeat=nb) for y in (-0.5, 0.5, 1.5))
        sw = sum(c.weight for c in f.constraints)
        assert (model is not None) == (best == -sw)


@pytest.mark.parametrize("name", ["cfg1", "cfg2s", "cfg3s", "cfg4s", "cfg2", "cfg4m", "place9856s", "rand100", "rand300"])
def test_generator_witnesses_exact(name):
    inst = fsmt_gen.config(name)
    f = hsmt.parse(inst.text)
    assert (f.n_bool, f.n_real, len(f.constraints)) == (inst.n_bool, inst.n_real, inst.n_cons)
    obj, sat = semantics.eval_formula(f, inst.x_star, inst.y_star)
    assert all(sat) and obj == -sum(c.weight for c in f.constraints)


def test_paper_family_sizes():
    """The generators reproduce the paper's instance sizes: the placement family at n_m = 64, n_l = 8
    (896 modules, 9,856 variables; 400,960 non-overlap + 3,584 feasibility + 10,880 routing =
    415,424 constraints) and the random family's counts per n
    (n/5 card + n/5 nae + n/50 xor of lengths min(50, n/5) / 50)."""
    p = fsmt_gen.config("place9856")
    assert (p.n_bool + p.n_real, p.meta["modules"], p.n_cons, p.meta["routing"]) == (9856, 896, 415424, 10880)
    assert p.text.count("\ne 1 (or ") == 400960 and p.text.count("\ne 1 (not (xor ") == 1088 * 6
    for n in (100, 600, 1000):
        r = fsmt_gen.config(f"rand{n}")
        lines = r.text.splitlines()
        l = min(50, n // 5)
        assert (r.n_bool, r.n_real, r.n_cons) == (n, n, n // 5 * 2 + n // 50)
        assert sum(ln.startswith(f"c card {l // 2} ") and len(ln.split()) == 4 + l for ln in lines) == n // 5
        assert sum(ln.startswith("c nae ") and len(ln.split()) == 3 + l for ln in lines) == n // 5
        assert sum(ln.startswith("c xor ") and len(ln.split()) == 3 + 50 for ln in lines) == n // 50


# ----------------------------------------------------------------------------- Alg.2 / projection / rounding

def test_erwa_closed_form_matches_alg2_literal():
    # R18: Alg.2 verbatim (rho=.5, gamma=2, tau=1, h<-1) gives w during stage t = 2^(U_{t-1} + max(t-2,0)/2)
    rng = np.random.default_rng(4)
    for _ in range(2000):
        T = int(rng.integers(1, 25))
        u = rng.integers(0, 2, T)
        h, w = 0.0, 1.0
        U = 0
        for t in range(1, T + 1):
            assert w == 2.0 ** (U + max(t - 2, 0) / 2) or abs(w / 2.0 ** (U + max(t - 2, 0) / 2) - 1) < 1e-15
            h = solve.RHO * h + u[t - 1]
            w = w * solve.GAMMA ** h
            h = 1.0
            U += int(u[t - 1])
    # reset-to-0 reading: w during stage t = 2^(U_{t-1})
    for _ in range(200):
        T = int(rng.integers(1, 25))
        u = rng.integers(0, 2, T)
        h, w, U = 0.0, 1.0, 0
        for t in range(1, T + 1):
            assert w == 2.0 ** U
            h = solve.RHO * h + u[t - 1]
            w *= solve.GAMMA ** h
            h = 0.0
            U += int(u[t - 1])


def test_projection_and_bounds():
    # S:370-372
    lo = np.array([0.0], dtype=np.float32)
    hi = np.array([1.0], dtype=np.float32)
    a, b = solve.project(np.array([2.0, -3.0]), np.array([2.0]), lo, hi)
    assert list(a) == [1.0, -1.0] and list(b) == [1.0]
    f = hsmt.parse(fsmt_gen.cfg1().text)
    lo, hi = solve.bounds(f)
    assert lo[1] == np.float32(0.25) and np.isinf(lo[0]) and np.isinf(hi[0]) and np.isinf(hi[1])
    # placement bounds: 0 <= x <= 1 - w exactly (tightest fp32 satisfying the exact check)
    inst = fsmt_gen.config("cfg4s")
    f = hsmt.parse(inst.text)
    lo, hi = solve.bounds(f)
    for j in range(f.n_real):
        assert lo[j] == 0.0
        assert semantics.eval_atom(hsmt.parse(f"p hsmt 0 1\na 0 <= {1 - float(inst.meta['sizes'][j // 2][j % 2])!r} 0:1").atoms[0], [float(hi[j])])
        assert float(np.nextafter(hi[j], np.float32(2))) > 1 - float(inst.meta["sizes"][j // 2][j % 2])
    # negative and strict unit literals
    f = hsmt.parse("p hsmt 0 1\na 0 <= 0.1 0:1\nc or 1 -a0")
    lo, hi = solve.bounds(f)
    assert float(lo[0]) > 0.1 and float(np.nextafter(lo[0], np.float32(-1))) <= 0.1


def test_rounding_rules():
    a = np.array([-0.5, 0.0, -0.0, 0.3, -1.0, 1.0])
    assert list(solve.round_sign(a)) == [-1, 1, 1, 1, -1, 1]                      # sgn(0)=+1
    # randomised rounding frequency ~ (1-a)/2  (Eq.4)
    a = np.full(4000, 0.4)
    x = solve.round_philox(a, 99, 0, 1)
    assert abs(np.mean(x == -1) - 0.3) < 0.03


def test_init_point_reading():
    f = hsmt.parse(fsmt_gen.cfg1().text)
    lo, hi = solve.bounds(f)
    a, b = solve.init_point(f, 0x0123456789ABCDEF, 5, lo, hi)
    assert np.all(np.abs(a) < 1) and b[1] >= 0.25
    assert all(np.float32(v) == v for v in a) and all(np.float32(v) == v for v in b)


def test_oracle_solve_cfg1_sound():
    f = hsmt.parse(fsmt_gen.cfg1().text)
    p = solve.Params(steps=30, eta=0.1)
    verdict, r, res = solve.solve(f, 4, 1234, p)
    assert verdict == "SAT"
    obj, sat = semantics.eval_formula(f, res[r].x, res[r].y)
    assert all(sat)
    # unsatisfiable formula -> UNKNOWN
    g = hsmt.parse("p hsmt 1 0\nc or 1 +b0\nc or 1 -b0")
    verdict, _, _ = solve.solve(g, 2, 1, solve.Params(kappas=[1.0, 2.0], steps=5))
    assert verdict == "UNKNOWN"


@pytest.mark.parametrize("name", ["cfg1", "cfg2s", "cfg3s", "cfg4s"])
def test_grouped_sparse_path_matches_enumeration(name):
    inst = fsmt_gen.config(name)
    f = hsmt.parse(inst.text)
    rng = np.random.default_rng(21)
    a = rng.uniform(-1, 1, f.n_bool)
    b = rng.uniform(0, 1, f.n_real)
    w = rng.integers(1, 5, len(f.constraints)).astype(float)
    C1, ga1, gb1, t1 = objective.objective_and_gradient(f, a, b, 1.7, w, want_terms=True)
    C2, ga2, gb2, t2 = objective.objective_and_gradient_grouped(f, a, b, 1.7, w, want_terms=True)
    assert abs(C1 - C2) < 1e-10 * max(1, abs(C1))
    assert np.allclose(ga1, ga2, atol=1e-12) and np.allclose(gb1, gb2, atol=1e-12)
    assert all(abs(t1[i] - t2[i]) < 1e-13 for i in t1)


def test_multiple_roundings_reading_r34():
    """R34: with n_roundings = M the stage keeps the first of M Philox draws with the fewest
    violations; M = 1 is the single draw of R17 (draw m uses stage word t + (m << 16))."""
    inst = fsmt_gen.config("cfg1")
    f = hsmt.parse(inst.text)
    lo, hi = solve.bounds(f)
    base = solve.Params(rounding="philox", steps=3, kappas=[0.5, 1.0, 1.5])
    r1 = solve.solve_restart(f, 7, 3, base, lo, hi)
    base.n_roundings = 1
    assert solve.solve_restart(f, 7, 3, base, lo, hi).history == r1.history
    # the M-draw stage-1 choice equals the brute-force minimum over the M draws
    a, b = solve.init_point(f, 7, 3, lo, hi)
    w = [c.weight for c in f.constraints]
    for _ in range(3):
        a, b, _, _ = solve.pgd_step(f, a, b, 0.5, w, base.eta, lo, hi)
    y = np.asarray(b, dtype=np.float32)
    draws = [solve.violations(f, solve.round_philox(a, 7, 3, 1 + (m << 16)), y).sum() for m in range(6)]
    assert draws[0] == solve.violations(f, solve.round_philox(a, 7, 3, 1), y).sum()
    base.n_roundings = 6
    base.kappas = [0.5]
    res = solve.solve_restart(f, 7, 3, base, lo, hi)
    assert res.history[0][2] == min(draws)


# ----------------------------------------------------------------------------- Alg.2 loop / Eq.13 pins


@pytest.mark.parametrize("erwa_mode", [0, 1])
def test_solve_restart_loop_weights_match_r18_closed_form(erwa_mode, monkeypatch):
    """solve_restart runs Alg.2 literally: h <- rho h + u; w <- w gamma^h; h <- 1
    (verbatim) or 0 (reset reading).  With an injected violation sequence u_t, the weights it
    hands to each stage's PGD steps must equal R18's closed form, derived independently:
    w(t) = 2^(U_{t-1} + max(t-2, 0)/2) (verbatim) and 2^(U_{t-1}) (reset-to-0), U_{t-1} = the
    violations of stages 1..t-1."""
    f = hsmt.parse("p hsmt 3 0\nc or 1 +b0 +b1\nc xor 1 +b1 +b2\nc or 2 -b0\nc nae 1 +b0 +b1 +b2\n")
    T, C = 9, len(f.constraints)
    rng = np.random.default_rng(7)
    useq = (rng.random((T, C)) < 0.6).astype(np.int64)
    useq[:, 0] = 1                                   # never SAT: every stage reaches the weight update
    seen = []
    stage = {"t": 0}

    def fake_violations(ff, x, y):
        stage["t"] += 1
        return useq[stage["t"] - 1].copy()

    def fake_pgd(ff, a, b, kappa, w, eta, lo, hi, eta_b=None, H=None, proj_iters=0):
        seen.append(np.array(w, dtype=np.float64).copy())
        return np.asarray(a), np.asarray(b), 1.0, 0.0            # gm2 > eps^2: one step, no move

    monkeypatch.setattr(solve, "violations", fake_violations)
    monkeypatch.setattr(solve, "pgd_step", fake_pgd)
    p = solve.Params(kappas=[1.0] * T, steps=1, eps=1e-3, erwa_mode=erwa_mode)
    res = solve.solve_restart(f, 3, 0, p)
    assert res.sat_stage == 0 and len(seen) == T
    base = np.array([c.weight for c in f.constraints])
    U = np.zeros(C)
    for t in range(1, T + 1):
        e = 0.0 if erwa_mode == 1 else max(t - 2, 0) / 2.0
        want = base * 2.0 ** (U + e)
        np.testing.assert_allclose(seen[t - 1], want, rtol=1e-13, atol=0)
        U += useq[t - 1]


def test_pgd_step_eq13_blockwise_norm_hand_case():
    """Eq.11-13 with the block step reading (eta for a, eta_b for b): one step on
    {b0 or a0} (a0: y0 <= 0.5) at a = -0.99, b = 0.3, kappa = 1, eta = 0.1, eta_b = 0.05.
    By hand (Eq.8: E = -1 + 2 (1 + v)/2 (1 + d)/2 with v = a, d = erf((y0 - 0.5)/sqrt 2)):
    dE/da = (1 + d)/2, dE/db = (1 + a)/2 sqrt(2/pi) exp(-(y0 - 0.5)^2 / 2);
    a' = clip(a - eta dE/da, -1, 1) = -1 (the step crosses -1), b' = b - eta_b dE/db (no bound);
    ||gm||^2 = ((a - a')/eta)^2 + ((b - b')/eta_b)^2 = 0.1^2 + (dE/db)^2."""
    f = hsmt.parse("p hsmt 1 1\na 0 <= 0.5 0:1\nc or 1 +b0 +a0\n")
    lo, hi = solve.bounds(f)
    a, b, eta, eta_b = -0.99, 0.3, 0.1, 0.05
    d = math.erf((b - 0.5) / math.sqrt(2.0))
    ga = (1.0 + d) / 2.0
    gb = (1.0 + a) / 2.0 * math.sqrt(2.0 / math.pi) * math.exp(-((b - 0.5) ** 2) / 2.0)
    a2, b2, gm2, C = solve.pgd_step(f, np.array([a]), np.array([b]), 1.0, None, eta, lo, hi, eta_b=eta_b)
    assert a - eta * ga < -1.0
    assert a2[0] == -1.0
    assert abs(b2[0] - (b - eta_b * gb)) <= 1e-15
    assert abs(gm2 - (((a + 1.0) / eta) ** 2 + gb ** 2)) <= 1e-12
    assert abs(C - (-1.0 + (1.0 + a) * (1.0 + d) / 2.0)) <= 1e-15


def test_objective_default_weights_are_the_formula_weights():
    """Eq.3 / Eq.10 weight every constraint by its w_c: omitting `weights` must use the
    formula's weights, not 1."""
    f = hsmt.parse("p hsmt 2 0\nc or 3 +b0 +b1\nc xor 0.5 +b0 +b1\n")
    a, b = np.array([0.3, -0.6]), np.zeros(0)
    C, ga, gb = objective.objective_and_gradient(f, a, b, 1.0)
    # E_or = -1 + 2 (1+a0)/2 (1+a1)/2, E_xor = a0 a1 (SURVEY §8(c) O4 closed forms)
    e_or = -1.0 + (1 + a[0]) * (1 + a[1]) / 2.0
    e_xor = a[0] * a[1]
    assert abs(C - (3 * e_or + 0.5 * e_xor)) <= 1e-15
    np.testing.assert_allclose(ga, [3 * (1 + a[1]) / 2 + 0.5 * a[1], 3 * (1 + a[0]) / 2 + 0.5 * a[0]], atol=1e-15)
    Cg, gag, _ = objective.objective_and_gradient_grouped(f, a, b, 1.0)
    assert abs(Cg - C) <= 1e-15 and np.allclose(gag, ga, atol=1e-15)
