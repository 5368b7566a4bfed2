"""Structure-only ROBDD from a truth table — oracle-private builder, test infrastructure only.

Used solely to check the product's xBDD structure bit-exactly (parity row P1).
xBDD (Def.2): a DAG whose decision nodes test a Boolean variable or
an atom ("interpreting atomic constraints as propositional variables"),
with a true and a false out-edge.  Built here as the reduced ordered BDD of the
constraint's truth table over its slots (order = slot order, readings R5/R6):
no node with hi == lo, no duplicate (level, hi, lo) (canonical).

Canonical numbering (reading R7): node id = rank after a stable sort of the
nodes by (level ascending, pre-order index of a DFS from the root that visits
hi before lo).  Terminals: -1 = FALSE, -2 = TRUE.  hi = slot literal True.
"""
from __future__ import annotations

import json

import numpy as np

from .semantics import slots, truth_table

FALSE = -1
TRUE = -2


def build_from_table(table: np.ndarray, s: int):
    """Returns (nodes[(level, hi, lo)], root) in canonical numbering."""
    # tensor axis t <-> slot t ; index 1 on an axis = slot True
    t = table.reshape((2,) * s).transpose(tuple(range(s - 1, -1, -1))) if s else table.reshape(())
    unique = {}        # (level, hi, lo) -> provisional id
    raw = []
    memo = {}

    def rec(sub, level):
        if sub.all():
            return TRUE
        if not sub.any():
            return FALSE
        key = (level, sub.tobytes())
        if key in memo:
            return memo[key]
        # split on slot `level` (axis 0 of sub)
        hi = rec(sub[1], level + 1)
        lo = rec(sub[0], level + 1)
        if hi == lo:
            out = hi
        else:
            k = (level, hi, lo)
            out = unique.get(k)
            if out is None:
                out = len(raw)
                unique[k] = out
                raw.append(k)
        memo[key] = out
        return out

    root = rec(t, 0)
    if root < 0:
        return [], root
    # canonical renumbering: pre-order DFS from root visiting hi first
    pre = {}

    def dfs(v):
        if v < 0 or v in pre:
            return
        pre[v] = len(pre)
        _, hi, lo = raw[v]
        dfs(hi)
        dfs(lo)

    dfs(root)
    order = sorted(pre, key=lambda v: (raw[v][0], pre[v]))
    new = {v: i for i, v in enumerate(order)}
    ren = lambda v: v if v < 0 else new[v]
    nodes = [(raw[v][0], ren(raw[v][1]), ren(raw[v][2])) for v in order]
    return nodes, ren(root)


def constraint_structure(c):
    sl = slots(c)
    nodes, root = build_from_table(truth_table(c), len(sl))
    kinds = [0 if k == "b" else 1 for k, _ in sl]
    gids = [i for _, i in sl]
    return kinds, nodes, root, gids


def canonical_dump(f):
    """(templates_jsonl: str, constraints_bin: bytes) per the SURVEY §8(c) canonical dump.

    templates.jsonl: one line per template in first-occurrence order:
        {"slot_kinds":[..],"nodes":[[level,hi,lo],..],"root":r}
    constraints.bin: per constraint, little-endian u32: template_id, n_slots, slot global ids.
    """
    tids = {}
    lines = []
    out = bytearray()
    for c in f.constraints:
        kinds, nodes, root, gids = constraint_structure(c)
        key = (tuple(kinds), tuple(nodes), root)
        tid = tids.get(key)
        if tid is None:
            tid = len(tids)
            tids[key] = tid
            lines.append(json.dumps({"slot_kinds": kinds, "nodes": [list(n) for n in nodes], "root": root},
                                    separators=(",", ":")))
        out += np.array([tid, len(gids)] + gids, dtype="<u4").tobytes()
    return "".join(l + "\n" for l in lines), bytes(out)
