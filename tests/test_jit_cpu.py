"""The JIT-specialised sweep compiles with NVRTC for sm_100a here (no GPU needed), without spills."""
import re

import pytest

import fsmt_gen
from paper_2603_22877_b200 import Solver


@pytest.mark.parametrize("name", ["cfg3s", "cfg4s"])
def test_nvrtc_compiles_specialised_sweep(name):
    s = Solver(-1)
    s.load_formula(fsmt_gen.config(name).text)
    s.build_xbdd()
    nbytes, log = s.jit_check()
    assert nbytes > 0
    m = re.findall(r"(\d+) bytes spill stores", log)
    assert m and all(int(x) == 0 for x in m), log[-2000:]
