"""CPU tests of the C-ABI library: symbols, host-side logic (parser, xBDD builder, bounds,
host verifier) through a host-only context, compared with the independent oracle.

P1 (structure parity) is bit-exact: the product's canonical dump must equal the oracle's.
"""
import os
import re
import tempfile

import numpy as np
import pytest

from paper_2603_22877_b200 import native as N
from paper_2603_22877_b200 import Solver, FsmtError
from oracle import hsmt, robdd, semantics, solve as osolve
import fsmt_gen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "fsmt.h")).read()
    names = set(re.findall(r"\b(fsmt_[a-z_0-9]+)\s*\(", hdr))
    assert len(names) >= 25
    for n in sorted(names):
        assert hasattr(N.lib, n), f"libfsmt.so does not export {n}"


def _host(text):
    s = Solver(-1)
    s.load_formula(text)
    s.build_xbdd()
    return s


@pytest.mark.parametrize("name", ["cfg1", "cfg2s", "cfg3s", "cfg4s"])
def test_structure_dump_bit_exact_vs_oracle(name):
    inst = fsmt_gen.config(name)
    s = _host(inst.text)
    with tempfile.TemporaryDirectory() as d:
        s.dump_structure(d)
        tj = open(os.path.join(d, "templates.jsonl")).read()
        cb = open(os.path.join(d, "constraints.bin"), "rb").read()
    ot, ob = robdd.canonical_dump(hsmt.parse(inst.text))
    assert tj == ot
    assert cb == ob


def test_structure_symmetric_large_properties():
    # cfg2 has XOR50 (beyond the oracle's truth-table builder): check reduced/ordered/size
    inst = fsmt_gen.config("cfg2")
    s = _host(inst.text)
    d = s.get_dims()
    assert d["n_cons"] == 2000 and d["max_slots"] == 50
    with tempfile.TemporaryDirectory() as dd:
        s.dump_structure(dd)
        import json
        tmpls = [json.loads(l) for l in open(os.path.join(dd, "templates.jsonl"))]
        cons = np.fromfile(os.path.join(dd, "constraints.bin"), dtype="<u4")
    f = hsmt.parse(inst.text)
    pos = 0
    for ci, c in enumerate(f.constraints):
        tid, ns = int(cons[pos]), int(cons[pos + 1])
        gids = list(cons[pos + 2:pos + 2 + ns])
        pos += 2 + ns
        assert [i for _, i in semantics.slots(c)] == gids
        t = tmpls[tid]
        nodes = [tuple(n) for n in t["nodes"]]
        assert len(set(nodes)) == len(nodes) and all(n[1] != n[2] for n in nodes)
        if c.kind == "xor":
            assert len(nodes) == 2 * ns - 1
        if c.kind == "nae":
            assert len(nodes) == 2 * ns - 1
        # semantic spot-check on random vertices against the oracle's exact semantics
        rng = np.random.default_rng(ci)
        for _ in range(20):
            bits = rng.integers(0, 2, ns)
            v = t["root"]
            while v >= 0:
                lvl, hi, lo = nodes[v]
                v = hi if bits[lvl] else lo
            truth = {key: bool(bits[p]) for p, key in enumerate(semantics.slots(c))}
            assert (v == -2) == bool(semantics.constraint_sat_values(c, truth))
    assert pos == len(cons)


@pytest.mark.parametrize("name", ["cfg1", "cfg3s", "cfg4s"])
def test_bounds_match_oracle(name):
    inst = fsmt_gen.config(name)
    s = _host(inst.text)
    lo, hi = s.get_bounds()
    olo, ohi = osolve.bounds(hsmt.parse(inst.text))
    assert np.array_equal(lo, olo) and np.array_equal(hi, ohi)


def test_bounds_edge_cases_match_oracle():
    text = ("p hsmt 0 4\na 0 <= 0.1 0:1\na 1 < 0.3 1:3\na 2 >= -0.7 2:-2\na 3 > 1e-9 3:7\n"
            "c or 1 -a0\nc or 1 +a1\nc or 1 +a2\nc xor 1 -a3\ne 1 (not a1)\n")
    s = _host(text)
    lo, hi = s.get_bounds()
    olo, ohi = osolve.bounds(hsmt.parse(text))
    assert np.array_equal(lo, olo) and np.array_equal(hi, ohi)


@pytest.mark.parametrize("name", ["cfg1", "cfg2s", "cfg3s", "cfg4s"])
def test_host_verify_matches_oracle(name):
    inst = fsmt_gen.config(name)
    s = _host(inst.text)
    f = hsmt.parse(inst.text)
    rng = np.random.default_rng(3)
    n, pc = s.verify(inst.x_star, inst.y_star, per_con=True)
    assert n == 0 and not pc.any()
    for trial in range(6):
        x = inst.x_star.copy()
        y = inst.y_star.copy()
        flip = rng.random(len(x)) < 0.1 * trial
        x[flip] = -x[flip]
        y = (y + rng.normal(0, 0.05 * trial, len(y))).astype(np.float32)
        n, pc = s.verify(x, y, per_con=True)
        want = osolve.violations(f, x, y)
        assert np.array_equal(pc.astype(np.int64), want) and n == int(want.sum())


def test_parse_errors_and_state_machine():
    s = Solver(-1)
    with pytest.raises(FsmtError) as e:
        s.load_formula("p hsmt 0 1\na 0 = 0 0:1\n")
    assert e.value.status == N.ERR_UNSUPPORTED
    for bad in ["p hsmt 1 0\nc or 0 +b0", "p hsmt 1 0\nc or 1", "p hsmt 1 0\nc or 1 +b3", "c or 1 +b0",
                "p hsmt 1 1\na 0 <= 0 0:0", "p hsmt 1 1\na 1 <= 0 0:1", "p hsmt 1 0\ne 1 (foo b0)"]:
        with pytest.raises(FsmtError) as e:
            s.load_formula(bad)
        assert e.value.status in (N.ERR_PARSE, N.ERR_UNSUPPORTED)
    with pytest.raises(FsmtError) as e:
        s.load_formula("p hsmt 1 0\nc or 1 +b0 +q1\n")
    assert re.match(r"ERR_PARSE: 2:\d+: ", str(e.value))
    s2 = Solver(-1)
    with pytest.raises(FsmtError) as e:
        s2.build_xbdd()
    assert e.value.status == N.ERR_STATE
    s2.load_formula(fsmt_gen.cfg1().text)
    with pytest.raises(FsmtError) as e:       # fsmt_prepare needs a built formula
        s2.prepare(64)
    assert e.value.status == N.ERR_STATE
    s2.build_xbdd()
    s2.prepare(64)                            # host-only: OK, no effect
    assert "prepared" not in s2.jit_info()["status"]
    with pytest.raises(FsmtError) as e:
        s2.begin(4, 1)
    assert e.value.status == N.ERR_CUDA


def test_dims_cfg3_cfg4_shapes():
    inst = fsmt_gen.config("cfg3")
    d = _host(inst.text).get_dims()
    assert d["n_bool"] + d["n_real"] == 2240 and d["n_cons"] == inst.n_cons
    # 1 non-overlap template (14 nodes, 10 slots) + feasibility (5 nodes) + unit atom
    assert d["max_nodes"] == 14 and d["max_slots"] == 10


@pytest.mark.parametrize("name", ["cfg3s", "cfg4s"])
def test_jit_source_compiles_for_sm100a(tmp_path, name):
    """The specialised sweep emitted by the plan (tiles.cpp) is valid sm_100a CUDA without spills."""
    import subprocess
    s = _host(fsmt_gen.config(name).text)
    info = s.jit_info()
    assert info["jit_classes"] >= 1 and info["tiles"] >= 1 and info["status"] == "host-only"
    src = s.jit_source()
    assert "fsmt_k1_jit" in src
    cu = tmp_path / "k1.cu"
    cu.write_text(src)
    out = subprocess.run(["/usr/local/cuda/bin/nvcc", "-cubin", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                          "-Xptxas", "-v", str(cu), "-o", str(tmp_path / "k1.cubin")],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "0 bytes spill stores" in out.stderr, out.stderr[-2000:]


def test_host_verify_threaded_large_matches_oracle():
    """fsmt_verify on cfg3 (114,688 constraints: the multi-threaded host re-check) agrees with
    the oracle's exact semantics on a sample of constraints, and its count with its per-constraint
    verdicts."""
    from tests.helpers import subformula
    inst = fsmt_gen.config("cfg3")
    s = _host(inst.text)
    rng = np.random.default_rng(5)
    x = inst.x_star.copy()
    flip = rng.random(len(x)) < 0.05
    x[flip] = -x[flip]
    y = (inst.y_star + rng.normal(0, 0.02, len(inst.y_star))).astype(np.float32)
    n, pc = s.verify(x, y, per_con=True)
    assert n == int(pc.sum()) and 0 < n < len(pc)
    csel = np.sort(rng.choice(len(pc), 1500, replace=False))
    sub, keep = subformula(inst.text, extra_constraints=csel)
    fs = hsmt.parse(sub)
    want = np.array([0 if semantics.constraint_sat(fs, c, x, y) else 1 for c in fs.constraints])
    assert np.array_equal(pc[keep].astype(int), want)
