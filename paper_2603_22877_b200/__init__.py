"""B200-native FourierSMT hot path (arXiv 2603.22877): batched xBDD COP + gradient sweep,
projected gradient step, rounding and exact verification as sm_100a CUDA kernels behind
the C ABI of include/fsmt.h.  Importing this package loads libfsmt.so; there is no CPU
fallback.
"""
from .native import SAT, UNKNOWN, HOST, DEVICE, ROUND_SIGN, ROUND_PHILOX, ERWA_VERBATIM, ERWA_RESET0, FsmtError  # noqa: F401
from .solver import Solver, SolveResult  # noqa: F401

__all__ = ["Solver", "SolveResult", "FsmtError", "SAT", "UNKNOWN"]
