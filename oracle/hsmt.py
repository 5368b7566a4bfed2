"""Oracle HSMT parser (test infrastructure only; see oracle/__init__.py).

Grammar, line oriented, ``#`` comments:
    p hsmt <n_bool> <n_real>                   header, first non-comment line
    a <id> <rel> <rhs> <j>:<coeff> ...          atom  sum_j coeff*y_j <rel> rhs, rel in {<=,<,>=,>}
    c <kind> [<k>] <weight> <lit> ...           symmetric constraint, kind in {or,card,nae,xor}
    e <weight> <sexpr>                          expression constraint
    literal tokens  +b<i> | -b<i> | +a<id> | -a<id>
    sexpr           (and e..) | (or e..) | (xor e..) | (not e) | b<i> | a<id>

Atoms are canonicalised to ``q.y <= q0`` / ``q.y < q0`` by negating (q, q0) for
>= / >; ``=`` is rejected (P:135 vs P:230, reading R9).
Truth encoding: -1 = True, +1 = False.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Union


class HsmtError(ValueError):
    """Parse / validation error; message is ``line:col: msg``."""


@dataclass(frozen=True)
class Atom:
    coeffs: tuple      # ((j, q_ij), ...) in stored order, canonical (<=/<) sign
    rhs: float         # q_i0, canonical sign
    strict: bool       # True for '<'


# A literal is (kind, index, negated) with kind 'b' (Boolean var) or 'a' (atom).
# An expression is ('lit', kind, idx, neg) | (op, (children...)) for op in
# and/or/xor | ('not', child).
Expr = Union[tuple]


@dataclass(frozen=True)
class Constraint:
    kind: str          # 'or' | 'card' | 'nae' | 'xor' | 'expr'
    k: int             # CARD threshold (sat iff #true <= k); 0 otherwise
    lits: tuple        # symmetric kinds: ((kind, idx, neg), ...)
    expr: tuple        # kind == 'expr': expression tree; else None
    weight: float


@dataclass(frozen=True)
class Formula:
    n_bool: int
    n_real: int
    atoms: tuple       # (Atom, ...) indexed by atom id
    constraints: tuple  # (Constraint, ...) in file order


def _err(line, col, msg):
    raise HsmtError(f"{line}:{col}: {msg}")


def _parse_index(tok, prefix, line, col):
    if not tok.startswith(prefix) or not tok[len(prefix):].isdigit():
        _err(line, col, f"bad token {tok!r}")
    return int(tok[len(prefix):])


def _parse_sexpr(text, line, col0):
    toks = text.replace("(", " ( ").replace(")", " ) ").split()
    pos = 0

    def rec():
        nonlocal pos
        if pos >= len(toks):
            _err(line, col0, "unexpected end of expression")
        t = toks[pos]
        pos += 1
        if t == "(":
            if pos >= len(toks):
                _err(line, col0, "unexpected end of expression")
            op = toks[pos]
            pos += 1
            kids = []
            while pos < len(toks) and toks[pos] != ")":
                kids.append(rec())
            if pos >= len(toks):
                _err(line, col0, "missing ')'")
            pos += 1
            if op == "not":
                if len(kids) != 1:
                    _err(line, col0, "'not' takes one argument")
                return ("not", kids[0])
            if op not in ("and", "or", "xor"):
                _err(line, col0, f"unknown operator {op!r}")
            if not kids:
                _err(line, col0, f"empty ({op})")
            return (op, tuple(kids))
        if t == ")":
            _err(line, col0, "unexpected ')'")
        if t.startswith("b"):
            return ("lit", "b", _parse_index(t, "b", line, col0), False)
        if t.startswith("a"):
            return ("lit", "a", _parse_index(t, "a", line, col0), False)
        _err(line, col0, f"bad token {t!r}")

    e = rec()
    if pos != len(toks):
        _err(line, col0, "trailing tokens after expression")
    return e


def _parse_weight(tok, line, col):
    try:
        w = float(tok)
    except ValueError:
        _err(line, col, f"bad weight {tok!r}")
    if not (w > 0.0) or w == float("inf"):
        _err(line, col, "weight must be positive and finite")
    return w


def parse(text: str) -> Formula:
    """Parse HSMT text into a validated Formula."""
    n_bool = n_real = None
    atoms = {}
    cons = []
    for ln, raw in enumerate(text.splitlines(), start=1):
        s = raw.split("#", 1)[0].strip()
        if not s:
            continue
        f = s.split()
        tag = f[0]
        if n_bool is None:
            if tag != "p" or len(f) != 4 or f[1] != "hsmt":
                _err(ln, 1, "expected header 'p hsmt <n_bool> <n_real>'")
            try:
                n_bool, n_real = int(f[2]), int(f[3])
            except ValueError:
                _err(ln, 1, "bad header counts")
            if n_bool < 0 or n_real < 0:
                _err(ln, 1, "negative header counts")
            continue
        if tag == "p":
            _err(ln, 1, "duplicate header")
        if tag == "a":
            if len(f) < 5:
                _err(ln, 1, "atom needs id, relation, rhs and >= 1 coefficient")
            aid = _parse_index("a" + f[1], "a", ln, 3)
            rel = f[2]
            if rel == "=":
                _err(ln, 1, "equality atoms unsupported")
            if rel not in ("<=", "<", ">=", ">"):
                _err(ln, 1, f"bad relation {rel!r}")
            try:
                rhs = float(f[3])
            except ValueError:
                _err(ln, 1, f"bad rhs {f[3]!r}")
            coeffs = []
            seen = set()
            for t in f[4:]:
                if ":" not in t:
                    _err(ln, 1, f"bad coefficient {t!r}")
                js, qs = t.split(":", 1)
                if not js.isdigit():
                    _err(ln, 1, f"bad variable index {js!r}")
                j = int(js)
                try:
                    q = float(qs)
                except ValueError:
                    _err(ln, 1, f"bad coefficient {qs!r}")
                if j >= n_real:
                    _err(ln, 1, f"real index {j} out of range")
                if j in seen:
                    _err(ln, 1, f"duplicate variable {j} in atom")
                if q == 0.0 or q != q or abs(q) == float("inf"):
                    _err(ln, 1, "coefficients must be finite and nonzero")
                seen.add(j)
                coeffs.append((j, q))
            if aid in atoms:
                _err(ln, 1, f"duplicate atom id {aid}")
            if rel in (">=", ">"):      # canonicalise: q.y >= q0  <=>  -q.y <= -q0
                coeffs = [(j, -q) for j, q in coeffs]
                rhs = -rhs
            atoms[aid] = Atom(tuple(coeffs), rhs, rel in ("<", ">"))
            continue
        if tag == "c":
            if len(f) < 3:
                _err(ln, 1, "constraint too short")
            kind = f[1]
            if kind not in ("or", "card", "nae", "xor"):
                _err(ln, 3, f"unknown constraint kind {kind!r}")
            i = 2
            k = 0
            if kind == "card":
                if not f[2].isdigit():
                    _err(ln, 1, "card needs an integer threshold")
                k = int(f[2])
                i = 3
            if len(f) <= i:
                _err(ln, 1, "missing weight")
            w = _parse_weight(f[i], ln, 1)
            lits = []
            for t in f[i + 1:]:
                if len(t) < 3 or t[0] not in "+-" or t[1] not in "ab" or not t[2:].isdigit():
                    _err(ln, 1, f"bad literal {t!r}")
                lits.append((t[1], int(t[2:]), t[0] == "-"))
            if not lits:
                _err(ln, 1, "empty literal list")
            if kind == "card" and k > len(lits):
                _err(ln, 1, "card threshold exceeds literal count")
            cons.append((ln, Constraint(kind, k, tuple(lits), None, w)))
            continue
        if tag == "e":
            if len(f) < 3:
                _err(ln, 1, "expression constraint too short")
            w = _parse_weight(f[1], ln, 1)
            body = s.split(None, 2)[2]
            cons.append((ln, Constraint("expr", 0, (), _parse_sexpr(body, ln, 1), w)))
            continue
        _err(ln, 1, f"unknown line tag {tag!r}")
    if n_bool is None:
        _err(1, 1, "missing header")
    k_total = len(atoms)
    if sorted(atoms) != list(range(k_total)):
        _err(1, 1, "atom ids must be dense 0..k-1")

    def check_lit(ln, kind, idx):
        if kind == "b" and idx >= n_bool:
            _err(ln, 1, f"Boolean index {idx} out of range")
        if kind == "a" and idx >= k_total:
            _err(ln, 1, f"atom index {idx} out of range")

    def check_expr(ln, e):
        if e[0] == "lit":
            check_lit(ln, e[1], e[2])
        elif e[0] == "not":
            check_expr(ln, e[1])
        else:
            for kid in e[1]:
                check_expr(ln, kid)

    out = []
    for ln, c in cons:
        if c.kind == "expr":
            check_expr(ln, c.expr)
        else:
            for kind, idx, _ in c.lits:
                check_lit(ln, kind, idx)
        out.append(c)
    return Formula(n_bool, n_real, tuple(atoms[i] for i in range(k_total)), tuple(out))
