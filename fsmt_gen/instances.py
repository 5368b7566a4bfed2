"""HSMT instance generators (no method arithmetic; see package docstring).

Every generator is deterministic per seed and planted-SAT: it returns the
witness it planted (x in {+-1}^n with -1 = True, y as fp32 values).  Tests check
the witness with the oracle's exact verifier; the generator itself only does
the instance-construction arithmetic (positions, sizes, schedules).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

CFG1_TEXT = """\
# config 1 (tiny; SURVEY Appendix A). Truth encoding: -1 = True. Atoms are canonicalized at load.
p hsmt 4 2
# a0: y0 <= 0   ((y0 > 0) is the literal "not a0")
a 0 <= 0 0:1
# a1: y0 + y1 <= 1
a 1 <= 1 0:1 1:1
# a2: y0 - y1 >= -0.5   (canonical: -y0 + y1 <= 0.5)
a 2 >= -0.5 0:1 1:-1
# a3: y1 >= 0.25        (canonical: -y1 <= -0.25)
a 3 >= 0.25 1:1
# Fig.2 pair (P:307): c0 = (not x) XOR (y>0),  c1 = x AND (y>0)
e 1 (xor (not b0) (not a0))
e 1 (and b0 (not a0))
c or 1 +b1 +b2 +a1
c xor 1 +b1 +b3 +a2
c nae 1 +b1 +b2 +a3
# unit atom: becomes the bound y1 >= 0.25 in the projection, and stays an objective term (R15, R16)
c or 1 +a3
"""


@dataclass
class Instance:
    name: str
    text: str
    n_bool: int
    n_real: int
    n_cons: int
    x_star: np.ndarray          # planted Booleans, int8 +-1 (-1 = True)
    y_star: np.ndarray          # planted reals, float32
    meta: dict = field(default_factory=dict)


def cfg1() -> Instance:
    # witness: b0 = T, b1 = b2 = b3 = F, y = (0.25, 0.5)
    return Instance("cfg1", CFG1_TEXT, 4, 2, 6,
                    np.array([-1, 1, 1, 1], dtype=np.int8), np.array([0.25, 0.5], dtype=np.float32))


def _num(v: float) -> str:
    return repr(float(v))


# ----------------------------------------------------------------------------- cfg2 random hybrid


def random_hybrid(n_bool=100, n_real=100, n_atoms=100, n_card=952, n_nae=952, n_xor=96,
                  l_card=20, l_nae=20, l_xor=50, k_card=None, seed=2) -> Instance:
    """Random hybrid card/nae/xor family (SURVEY §8(d) cfg2 recipe).

    Atoms: sum over 3 distinct reals q_j y_j <= q0, q_j in {+-1,+-2,+-3};
    planted x*, y* ~ U(-1,1); q0 = q.y* +- U(0.05, 0.5) (atom True or False at
    y* with margin).  Literals are drawn distinct from the 2n-slot pool with
    random polarity, then polarity-repaired to hold at the planted point.
    """
    rng = np.random.default_rng(seed)
    if k_card is None:
        k_card = l_card // 2
    x_star = np.where(rng.random(n_bool) < 0.5, -1, 1).astype(np.int8)
    y_star = rng.uniform(-1.0, 1.0, n_real).astype(np.float32)
    lines = [f"p hsmt {n_bool} {n_real}"]
    atom_true = np.zeros(n_atoms, dtype=bool)
    for i in range(n_atoms):
        cols = rng.choice(n_real, size=3, replace=False)
        qs = rng.choice([-3, -2, -1, 1, 2, 3], size=3)
        s = 0.0
        for j, q in zip(cols, qs):
            s += float(q) * float(y_star[j])
        margin = float(rng.uniform(0.05, 0.5))
        truth = bool(rng.random() < 0.5)
        q0 = round(s + margin if truth else s - margin, 6)
        atom_true[i] = truth
        lines.append(f"a {i} <= {_num(q0)} " + " ".join(f"{j}:{q}" for j, q in zip(cols, qs)))
    # slot pool: 0..n_bool-1 Booleans, n_bool.. atoms
    pool_true = np.concatenate([x_star == -1, atom_true])

    def lit_tok(slot, neg):
        kind = "b" if slot < n_bool else "a"
        idx = slot if slot < n_bool else slot - n_bool
        return ("-" if neg else "+") + kind + str(idx)

    def draw(L):
        sl = rng.choice(n_bool + n_atoms, size=L, replace=False)
        neg = rng.random(L) < 0.5
        return sl, neg

    for _ in range(n_card):
        sl, neg = draw(l_card)
        lit_true = pool_true[sl] ^ neg
        # repair: flip true literals until #true <= k
        for p in np.nonzero(lit_true)[0][: max(0, int(lit_true.sum()) - k_card)]:
            neg[p] = ~neg[p]
        lines.append(f"c card {k_card} 1 " + " ".join(lit_tok(s, n) for s, n in zip(sl, neg)))
    for _ in range(n_nae):
        sl, neg = draw(l_nae)
        lit_true = pool_true[sl] ^ neg
        if lit_true.all() or (~lit_true).all():
            neg[0] = ~neg[0]
        lines.append("c nae 1 " + " ".join(lit_tok(s, n) for s, n in zip(sl, neg)))
    for _ in range(n_xor):
        sl, neg = draw(l_xor)
        lit_true = pool_true[sl] ^ neg
        if int(lit_true.sum()) % 2 == 0:
            neg[0] = ~neg[0]
        lines.append("c xor 1 " + " ".join(lit_tok(s, n) for s, n in zip(sl, neg)))
    return Instance("cfg2", "\n".join(lines) + "\n", n_bool, n_real, n_card + n_nae + n_xor, x_star, y_star,
                    {"seed": seed})


def paper_random(n: int, seed: int = 0) -> Instance:
    """The paper's random hybrid family (Results "random benchmark"): n
    Booleans, n reals, n LRA atoms; m_card = m_nae = n/5 and m_xor = n/50 constraints of lengths
    l_card = l_nae = min(50, n/5) and l_xor = 50, n in {100, ..., 1000}.  Readings (DESIGN.md §3
    R36): the card threshold is k = l/2 ("sum l_i <= k", k unstated); atoms and literals
    as cfg2 (3-real atoms; literals drawn from the 2n-slot pool with random polarity,
    planted-SAT repair)."""
    assert n % 50 == 0 and n >= 100
    l = min(50, n // 5)
    inst = random_hybrid(n_bool=n, n_real=n, n_atoms=n, n_card=n // 5, n_nae=n // 5, n_xor=n // 50,
                         l_card=l, l_nae=l, l_xor=50, k_card=l // 2, seed=1000 + n + 7919 * seed)
    inst.name = f"rand{n}"
    inst.meta.update({"n": n, "l": l, "k_card": l // 2, "family_seed": seed})
    return inst


# ----------------------------------------------------------------------------- cfg3 scheduling


def scheduling(n_w=16, n_j=448, seed=3, dep_prob=0.5, gap=1e-6) -> Instance:
    """Continuous-time scheduling with the R23 reading of the feasibility clause.

    Variables: job j has worker bits x_{i,j} = Boolean j*B + i (B = log2 n_w,
    X_j = sum_i 2^i [x_{i,j} True]) and start time y_j = real j.
    Constraints: non-overlap for every pair j < j' (B XOR pairs v two separation
    atoms), feasibility per (job, worker) as two clauses (R23), dependency unit
    atoms y_j - y_j' >= t_j' (soft, R15).  T = greedy list-schedule makespan.
    """
    rng = np.random.default_rng(seed)
    B = int(n_w).bit_length() - 1
    assert 1 << B == n_w
    d = np.round(rng.uniform(0.0, 1.0, n_w), 6)
    t = np.round(rng.uniform(0.0, 1.0, n_j), 6)
    deps = [None] * n_j
    for j in range(1, n_j):
        if rng.random() < dep_prob:
            deps[j] = int(rng.integers(0, j))
    # greedy: jobs in index order, worker that can start earliest
    free = d.copy()
    start = np.zeros(n_j)
    worker = np.zeros(n_j, dtype=np.int64)
    for j in range(n_j):
        ready = 0.0 if deps[j] is None else start[deps[j]] + t[deps[j]]
        cand = np.maximum(np.maximum(free, d), ready) + gap
        w = int(np.argmin(cand))
        worker[j] = w
        start[j] = cand[w]
        free[w] = start[j] + t[j]
    T = float(np.max(free - d)) + gap
    T = float(np.ceil(T * 1e6) / 1e6)
    lines = [f"p hsmt {n_j * B} {n_j}"]
    atoms = []
    cons = []

    def atom(rel, rhs, coeffs):
        atoms.append(f"a {len(atoms)} {rel} {_num(rhs)} " + " ".join(f"{j}:{q}" for j, q in coeffs))
        return len(atoms) - 1

    for j in range(n_j):
        for jp in range(j + 1, n_j):
            a0 = atom(">=", t[jp], [(j, 1), (jp, -1)])
            a1 = atom(">=", t[j], [(jp, 1), (j, -1)])
            pairs = " ".join(f"(xor b{j * B + i} b{jp * B + i})" for i in range(B))
            cons.append(f"e 1 (or {pairs} a{a0} a{a1})")
    for j in range(n_j):
        for w in range(n_w):
            neq = " ".join((("-" if (w >> i) & 1 else "+") + f"b{j * B + i}") for i in range(B))
            a_lo = atom(">=", d[w], [(j, 1)])
            cons.append(f"c or 1 {neq} +a{a_lo}")
            a_hi = atom("<=", round(float(d[w]) + T - float(t[j]), 9), [(j, 1)])
            cons.append(f"c or 1 {neq} +a{a_hi}")
    for j in range(n_j):
        if deps[j] is not None:
            jp = deps[j]
            a0 = atom(">=", t[jp], [(j, 1), (jp, -1)])
            cons.append(f"c or 1 +a{a0}")
    text = "\n".join(lines + atoms + cons) + "\n"
    x_star = np.ones(n_j * B, dtype=np.int8)
    for j in range(n_j):
        for i in range(B):
            if (worker[j] >> i) & 1:
                x_star[j * B + i] = -1
    return Instance("cfg3", text, n_j * B, n_j, len(cons), x_star, start.astype(np.float32),
                    {"seed": seed, "T": T, "n_w": n_w, "n_j": n_j, "bits": B, "n_dep": sum(x is not None for x in deps)})


# ----------------------------------------------------------------------------- cfg4 placement

_SIZES = {  # (w, d) as decimal literals
    "large_pe": ("0.4", "0.4"),
    "small_pe": ("0.2", "0.2"),
    "large_mem": ("0.1", "0.1"),
    "small_mem_x": ("0.1", "0.05"),
    "small_mem_y": ("0.05", "0.1"),
}
_ONE_MINUS = {"0.4": "0.6", "0.2": "0.8", "0.1": "0.9", "0.05": "0.95"}


def placement(n_m=32, n_l=4, counts=(148, 592, 148, 296), seed=4, gap=1e-6) -> Instance:
    """3D placement: non-overlap for every module pair + boundary bounds.

    Module j: macro bits m_{i,j} = Boolean j*K + i (i < log2 n_m), layer bits
    l_{i,j} = Boolean j*K + log2 n_m + i, K = log2 n_m + log2 n_l; x_j = real 2j,
    y_j = real 2j+1.  Non-overlap (reading R24): OR of all macro/layer bit XORs
    and the four separation atoms.  Feasibility: 0 <= x_j <= 1 - w_j,
    0 <= y_j <= 1 - d_j as single-variable unit atoms (-> projection bounds).
    Routing-aware constraints are excluded (R25).  Default counts are the paper's
    proportions x 4.625 (1,184 modules).
    """
    rng = np.random.default_rng(seed)
    bm = int(n_m).bit_length() - 1
    bl = int(n_l).bit_length() - 1
    K = bm + bl
    kinds = (["large_pe"] * counts[0] + ["small_pe"] * counts[1] + ["large_mem"] * counts[2]
             + ["small_mem"] * counts[3])
    kinds = [kinds[i] for i in rng.permutation(len(kinds))]
    sizes = []
    sm = 0
    for k in kinds:
        if k == "small_mem":             # alternate the axis of small memories
            k = "small_mem_x" if sm % 2 == 0 else "small_mem_y"
            sm += 1
        sizes.append(_SIZES[k])
    M = len(sizes)
    wf = np.array([float(w) for w, _ in sizes])
    df = np.array([float(h) for _, h in sizes])
    # planted witness: shelf-pack modules (decreasing height) into the n_m*n_l bins, round-robin
    nb = n_m * n_l
    bins_order = rng.permutation(nb)
    order = sorted(range(M), key=lambda j: (-df[j], -wf[j], j))
    shelves = [[] for _ in range(nb)]       # per bin: list of [y0, height, x_cursor]
    pos = np.zeros((M, 2))
    binof = np.zeros(M, dtype=np.int64)
    rr = 0
    for j in order:
        placed = False
        for attempt in range(nb):
            bidx = int(bins_order[(rr + attempt) % nb])
            sh = shelves[bidx]
            for s in sh:
                if s[2] + wf[j] <= 1.0 - gap and df[j] <= s[1]:
                    pos[j] = (s[2], s[0])
                    s[2] += wf[j] + gap
                    placed = True
                    break
            if not placed:
                y0 = 0.0 if not sh else sh[-1][0] + sh[-1][1] + gap
                if y0 + df[j] <= 1.0 - gap:
                    sh.append([y0, df[j], wf[j] + gap])
                    pos[j] = (0.0, y0)
                    placed = True
            if placed:
                binof[j] = bidx
                rr = (rr + attempt + 1) % nb
                break
        assert placed, "placement generator could not pack the planted witness"
    y_star = np.empty(2 * M, dtype=np.float32)
    y_star[0::2] = pos[:, 0]
    y_star[1::2] = pos[:, 1]
    x_star = np.ones(M * K, dtype=np.int8)
    for j in range(M):
        macro, layer = binof[j] // n_l, binof[j] % n_l
        for i in range(bm):
            if (macro >> i) & 1:
                x_star[j * K + i] = -1
        for i in range(bl):
            if (layer >> i) & 1:
                x_star[j * K + bm + i] = -1
    # emit
    out = [f"p hsmt {M * K} {2 * M}"]
    atoms = []
    cons = []
    na = 0
    for j in range(M):
        xj, yj = 2 * j, 2 * j + 1
        wj, dj = sizes[j]
        for jp in range(j + 1, M):
            xp, yp = 2 * jp, 2 * jp + 1
            wp, dp = sizes[jp]
            atoms.append(f"a {na} >= {wp} {xj}:1 {xp}:-1\n"
                         f"a {na + 1} >= {wj} {xp}:1 {xj}:-1\n"
                         f"a {na + 2} >= {dp} {yj}:1 {yp}:-1\n"
                         f"a {na + 3} >= {dj} {yp}:1 {yj}:-1")
            pairs = " ".join(f"(xor b{j * K + i} b{jp * K + i})" for i in range(K))
            cons.append(f"e 1 (or {pairs} a{na} a{na + 1} a{na + 2} a{na + 3})")
            na += 4
    for j in range(M):
        xj, yj = 2 * j, 2 * j + 1
        wj, dj = sizes[j]
        atoms.append(f"a {na} >= 0 {xj}:1\na {na + 1} <= {_ONE_MINUS[wj]} {xj}:1\n"
                     f"a {na + 2} >= 0 {yj}:1\na {na + 3} <= {_ONE_MINUS[dj]} {yj}:1")
        cons.append(f"c or 1 +a{na}\nc or 1 +a{na + 1}\nc or 1 +a{na + 2}\nc or 1 +a{na + 3}")
        na += 4
    text = "\n".join(out + atoms + cons) + "\n"
    n_cons = M * (M - 1) // 2 + 4 * M
    return Instance("cfg4", text, M * K, 2 * M, n_cons, x_star, y_star,
                    {"seed": seed, "modules": M, "bits_per_module": K, "n_m": n_m, "n_l": n_l, "n_atoms": na,
                     "sizes": sizes, "bins": binof})


def placement_routed(n_m=64, n_l=8, seed=5) -> Instance:
    """The paper's placement family itself, routing-aware constraints included.

    Modules: n_m large PEs (0.4 x 0.4), n_m*n_l small PEs (0.2 x 0.2), n_m large
    memories (0.1 x 0.1), n_m*n_l/2 small memories (0.1 x 0.05, axis alternating).
    Reading R25 (the paper's counts: 10,880 routing constraints at n_m = 64, n_l = 8 = 1,088
    associated pairs x (log2 n_m bit equalities + 4 adjacency atoms)): each large PE is paired with
    one large memory, and each small PE with two small memories; small PE (m, l) of macro m goes with
    small memories (m, 2 floor(l / 4)) and (m, 2 floor(l / 4) + 1), so every small memory serves four
    PEs.  Routing constraints per associated (j, j'): m_{i,j} = m_{i,j'} for every macro bit, and the
    adjacency unit atoms x_j - x_j' <= w_j', x_j' - x_j <= w_j, y_j - y_j' <= d_j', y_j' - y_j <= d_j
    (multi-variable unit atoms: halfspaces of the R33 projection, or soft terms).  Non-overlap and
    feasibility as `placement`.  Planted witness: per macro, small PEs of layers 0-3 at spot A and
    of layers 4-7 at spot B, their memories at the same spot in layers the spot's PEs do not use,
    large PE and memory stacked in layers 0 / 1 (>= 0.05 clearance wherever modules share a layer).
    n_m = 64, n_l = 8: 896 modules, 9,856 variables, 415,424 constraints.
    """
    assert n_l == 8, "the planted layout uses 8 layers (4 per spot)"
    rng = np.random.default_rng(seed)
    bm = int(n_m).bit_length() - 1
    bl = int(n_l).bit_length() - 1
    K = bm + bl
    mods = []              # (kind, macro, index-within-macro)
    for m in range(n_m):
        mods.append(("large_pe", m, 0))
        mods.extend(("small_pe", m, l) for l in range(n_l))
        mods.append(("large_mem", m, 0))
        mods.extend(("small_mem", m, k) for k in range(n_l // 2))
    perm = rng.permutation(len(mods))
    mods = [mods[i] for i in perm]
    M = len(mods)
    sizes, pos, layer = [], np.zeros((M, 2)), np.zeros(M, dtype=np.int64)
    at = {}
    sm = 0
    for j, (kind, m, i) in enumerate(mods):
        at[(kind, m, i)] = j
        if kind == "small_mem":
            sz = _SIZES["small_mem_x" if sm % 2 == 0 else "small_mem_y"]
            sm += 1
        else:
            sz = _SIZES[kind]
        sizes.append(sz)
        if kind == "small_pe":                     # spot A (layers 0-3) or spot B (layers 4-7)
            pos[j] = (0.05, 0.05) if i < 4 else (0.5, 0.05)
            layer[j] = i
        elif kind == "small_mem":                  # mems 0,1 at spot A in layers 4,5; mems 2,3 at B in 0,1
            pos[j] = (0.1, 0.1) if i < 2 else (0.55, 0.1)
            layer[j] = 4 + i if i < 2 else i - 2
        elif kind == "large_pe":
            pos[j] = (0.05, 0.5)
            layer[j] = 0
        else:                                      # large memory, adjacent to (inside the window of) its PE
            pos[j] = (0.2, 0.6)
            layer[j] = 1
    pairs = []
    for m in range(n_m):
        pairs.append((at[("large_pe", m, 0)], at[("large_mem", m, 0)]))
        for l in range(n_l):
            base = 2 * (l // 4)
            for k in (base, base + 1):
                pairs.append((at[("small_pe", m, l)], at[("small_mem", m, k)]))
    macro = np.array([m for _, m, _ in mods])
    x_star = np.ones(M * K, dtype=np.int8)
    for j in range(M):
        for i in range(bm):
            if (macro[j] >> i) & 1:
                x_star[j * K + i] = -1
        for i in range(bl):
            if (layer[j] >> i) & 1:
                x_star[j * K + bm + i] = -1
    y_star = np.empty(2 * M, dtype=np.float32)
    y_star[0::2] = pos[:, 0]
    y_star[1::2] = pos[:, 1]
    out = [f"p hsmt {M * K} {2 * M}"]
    atoms, cons = [], []
    na = 0
    for j in range(M):
        xj, yj = 2 * j, 2 * j + 1
        wj, dj = sizes[j]
        for jp in range(j + 1, M):
            xp, yp = 2 * jp, 2 * jp + 1
            wp, dp = sizes[jp]
            atoms.append(f"a {na} >= {wp} {xj}:1 {xp}:-1\n"
                         f"a {na + 1} >= {wj} {xp}:1 {xj}:-1\n"
                         f"a {na + 2} >= {dp} {yj}:1 {yp}:-1\n"
                         f"a {na + 3} >= {dj} {yp}:1 {yj}:-1")
            bits = " ".join(f"(xor b{j * K + i} b{jp * K + i})" for i in range(K))
            cons.append(f"e 1 (or {bits} a{na} a{na + 1} a{na + 2} a{na + 3})")
            na += 4
    for j in range(M):
        xj, yj = 2 * j, 2 * j + 1
        wj, dj = sizes[j]
        atoms.append(f"a {na} >= 0 {xj}:1\na {na + 1} <= {_ONE_MINUS[wj]} {xj}:1\n"
                     f"a {na + 2} >= 0 {yj}:1\na {na + 3} <= {_ONE_MINUS[dj]} {yj}:1")
        cons.append(f"c or 1 +a{na}\nc or 1 +a{na + 1}\nc or 1 +a{na + 2}\nc or 1 +a{na + 3}")
        na += 4
    for j, jp in pairs:                            # routing-aware (reading R25)
        xj, yj, xp, yp = 2 * j, 2 * j + 1, 2 * jp, 2 * jp + 1
        (wj, dj), (wp, dp) = sizes[j], sizes[jp]
        for i in range(bm):
            cons.append(f"e 1 (not (xor b{j * K + i} b{jp * K + i}))")
        atoms.append(f"a {na} <= {wp} {xj}:1 {xp}:-1\na {na + 1} <= {wj} {xp}:1 {xj}:-1\n"
                     f"a {na + 2} <= {dp} {yj}:1 {yp}:-1\na {na + 3} <= {dj} {yp}:1 {yj}:-1")
        cons.append(f"c or 1 +a{na}\nc or 1 +a{na + 1}\nc or 1 +a{na + 2}\nc or 1 +a{na + 3}")
        na += 4
    text = "\n".join(out + atoms + cons) + "\n"
    n_cons = M * (M - 1) // 2 + 4 * M + len(pairs) * (bm + 4)
    return Instance("place9856", text, M * K, 2 * M, n_cons, x_star, y_star,
                    {"seed": seed, "modules": M, "bits_per_module": K, "n_m": n_m, "n_l": n_l, "n_atoms": na,
                     "pairs": len(pairs), "routing": len(pairs) * (bm + 4)})


def config(name: str) -> Instance:
    return CONFIGS[name]()


CONFIGS = {
    "cfg1": cfg1,
    "cfg2": random_hybrid,
    "cfg3": scheduling,
    "cfg4": placement,
    # small versions of the structured families (parity at oracle-friendly sizes)
    "cfg3s": lambda: scheduling(n_w=4, n_j=24, seed=13),
    "cfg4s": lambda: placement(n_m=2, n_l=2, counts=(4, 12, 4, 6), seed=14),
    # mid-size placement with cfg4's real class (n_m = 32, n_l = 4: 7 bit pairs, 25 nodes, 18 slots)
    "cfg4m": lambda: placement(n_m=32, n_l=4, counts=(8, 32, 8, 12), seed=44),
    "cfg2s": lambda: random_hybrid(n_bool=20, n_real=20, n_atoms=20, n_card=30, n_nae=30, n_xor=6,
                                   l_card=8, l_nae=8, l_xor=12, seed=12),
}
# the paper's placement family with routing (R25): 9,856 variables / 415,424 constraints,
# and a small version (n_m = 4, n_l = 8: 56 modules) for oracle-sized parity
CONFIGS["place9856"] = placement_routed
CONFIGS["place9856s"] = lambda: placement_routed(n_m=4, n_l=8, seed=15)
# the paper's random family at every n: "rand100" ... "rand1000"
CONFIGS.update({f"rand{n}": (lambda n=n: paper_random(n)) for n in range(100, 1001, 100)})
