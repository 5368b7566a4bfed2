"""The JIT-specialised sweep compiles with NVRTC for sm_100a here (no GPU needed), without spills:
the generic module of fsmt_build_xbdd and the modules fsmt_prepare(R) builds (restart count
compiled in, U prefetch)."""
import os
import re

import pytest

import fsmt_gen
from paper_2603_22877_b200 import Solver

VARIANTS = [{}, {"FSMT_JIT_CHECK_RC": "1024"}, {"FSMT_JIT_CHECK_RC": "1000000", "FSMT_JIT_UPF": "3"}]


@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()) or "generic")
@pytest.mark.parametrize("name", ["cfg3s", "cfg4s"])
def test_nvrtc_compiles_specialised_sweep(name, env):
    s = Solver(-1)
    s.load_formula(fsmt_gen.config(name).text)
    s.build_xbdd()
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        nbytes, log = s.jit_check()
        src = s.jit_source()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    assert nbytes > 0
    m = re.findall(r"(\d+) bytes spill stores", log)
    assert m and all(int(x) == 0 for x in m), log[-2000:]
    if "FSMT_JIT_CHECK_RC" in env:
        assert src.startswith("#define FSMT_RC " + env["FSMT_JIT_CHECK_RC"] + "u")
    assert "fsmt_q(" in src and "fsmt_w(" in src          # on-grid flushes and shifted ERWA weights


@pytest.mark.parametrize("name,vmax", [("cfg4", 54), ("cfg3", 40)])
def test_stream_row_budget_from_typical_constraint(name, vmax):
    """The planner's stream-row budget is 3x the typical constraint's variables in [40, 56]
    (DESIGN.md §7 / §9: the measured optima of cfg4 and cfg3)."""
    if os.environ.get("FSMT_TILE_VMAX"):
        pytest.skip("FSMT_TILE_VMAX overrides the rule")
    s = Solver(-1)
    s.load_formula(fsmt_gen.config(name).text)
    s.build_xbdd()
    assert f"#define VMAX {vmax}\n" in s.jit_source()
