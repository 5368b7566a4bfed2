"""Which module fsmt_prepare builds for a config (restarts per lane, register cap of the hot sweep):
python scripts/diag_prepare.py cfg4 1024"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fsmt_gen  # noqa: E402
from paper_2603_22877_b200 import Solver  # noqa: E402

name, R = sys.argv[1], int(sys.argv[2])
s = Solver(0)
s.load_formula(fsmt_gen.config(name).text)
s.build_xbdd()
s.prepare(R)
print(name, R, s.jit_info()["status"])
