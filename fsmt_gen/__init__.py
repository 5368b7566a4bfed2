"""Seeded synthetic input generators shared by the tests, the oracle checks and bench.py.

This package holds NONE of FourierSMT's arithmetic (no smoothing, expectation,
message passing, rounding, verification or weight update): it only emits HSMT
text for the BASELINE.json configs, planted witnesses for them, and
seeded relaxed points.  Both the CUDA product and the oracle consume its output.

Configs (DESIGN.md §5 input recipe):
  cfg1  tiny hand-written formula
  cfg2  random hybrid 100 Booleans / 100 reals / 100 atoms / 2,000 card/nae/xor constraints
  cfg3  scheduling n_w = 16, n_j = 448: 2,240 vars / ~114,688 constraints (reading R23)
  cfg4  placement n_m = 32, n_l = 4, 1,184 modules: 10,656 vars / 705,072 constraints (R24-R26)
  randN the paper's random hybrid family at n = 100..1000 (reading R36)
"""
from .instances import (  # noqa: F401
    Instance, cfg1, random_hybrid, paper_random, scheduling, placement, config, CONFIGS,
)
from .points import random_points  # noqa: F401
