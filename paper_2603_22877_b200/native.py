"""ctypes binding of libfsmt.so (include/fsmt.h) — argument marshalling only.

Every computation happens in the library's CUDA kernels (or, for parse/build/host
verification, its C++ host code).  If the library is missing this module raises
ImportError: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfsmt.so")

OK, ERR_ARG, ERR_PARSE, ERR_UNSUPPORTED, ERR_STATE, ERR_NODE_BUDGET, ERR_OOM, ERR_CUDA, ERR_TIMEOUT, ERR_RANGE = range(10)
STATUS_NAMES = ["OK", "ERR_ARG", "ERR_PARSE", "ERR_UNSUPPORTED", "ERR_STATE", "ERR_NODE_BUDGET", "ERR_OOM",
                "ERR_CUDA", "ERR_TIMEOUT", "ERR_RANGE"]
UNKNOWN, SAT = 0, 10
HOST, DEVICE = 0, 1
ROUND_SIGN, ROUND_PHILOX = 0, 1
ERWA_VERBATIM, ERWA_RESET0 = 0, 1


class Dims(C.Structure):
    _fields_ = [("n_bool", C.c_uint32), ("n_real", C.c_uint32), ("n_atoms", C.c_uint32), ("n_cons", C.c_uint32),
                ("n_templates", C.c_uint32), ("max_slots", C.c_uint32), ("max_nodes", C.c_uint32),
                ("n_bounded", C.c_uint32), ("n_nodes", C.c_uint64), ("n_slot_refs", C.c_uint64),
                ("n_halfspaces", C.c_uint32), ("n_slot_rows", C.c_uint32)]


class Params(C.Structure):
    _fields_ = [("kappas", C.POINTER(C.c_float)), ("n_stages", C.c_uint32), ("eta", C.c_float), ("eps", C.c_float),
                ("rounding", C.c_uint32), ("erwa_mode", C.c_uint32), ("time_limit_s", C.c_double),
                ("eta_mode", C.c_uint32), ("proj_iters", C.c_uint32),
                ("n_roundings", C.c_uint32)]


class Stats(C.Structure):
    _fields_ = [("stages_run", C.c_uint32), ("steps_run", C.c_uint32), ("winner_restart", C.c_uint32),
                ("winner_stage", C.c_uint32), ("best_unsat", C.c_uint32), ("host_verified", C.c_uint32),
                ("solve_ms", C.c_double), ("evals", C.c_double)]


if not os.path.exists(LIB_PATH):
    # A fresh checkout: compile it (nvcc, sm_100a) rather than fall back to anything.
    import importlib.util as _ilu
    _spec = _ilu.spec_from_file_location("_fsmt_build", os.path.join(HERE, "build.py"))
    _b = _ilu.module_from_spec(_spec)
    _spec.loader.exec_module(_b)
    try:
        _b.build()
    except Exception as _e:  # noqa: BLE001
        raise ImportError(f"libfsmt.so could not be built: {_e}") from _e
if not os.path.exists(LIB_PATH):
    raise ImportError(f"libfsmt.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(there is no CPU fallback)")
lib = C.CDLL(LIB_PATH)

_vp = C.c_void_p
_u32, _u64, _i32, _f32, _f64 = C.c_uint32, C.c_uint64, C.c_int, C.c_float, C.c_double
_SIGS = {
    "fsmt_create": (_i32, [_i32, C.POINTER(_vp)]),
    "fsmt_destroy": (None, [_vp]),
    "fsmt_last_error": (C.c_char_p, [_vp]),
    "fsmt_bind_stream": (_i32, [_vp, _vp]),
    "fsmt_load_formula": (_i32, [_vp, C.c_char_p, C.c_size_t]),
    "fsmt_build_xbdd": (_i32, [_vp, _u64]),
    "fsmt_get_dims": (_i32, [_vp, C.POINTER(Dims)]),
    "fsmt_get_bounds": (_i32, [_vp, _vp, _vp]),
    "fsmt_dump_structure": (_i32, [_vp, C.c_char_p]),
    "fsmt_set_params": (_i32, [_vp, C.POINTER(Params)]),
    "fsmt_solve": (_i32, [_vp, _u32, _u32, _u64, C.POINTER(_i32), _vp, _vp, C.POINTER(Stats)]),
    "fsmt_begin": (_i32, [_vp, _u32, _u64, _u32]),
    "fsmt_set_state": (_i32, [_vp, _vp, _vp, _i32]),
    "fsmt_get_state": (_i32, [_vp, _vp, _vp, _i32]),
    "fsmt_set_counters": (_i32, [_vp, _vp, _i32]),
    "fsmt_get_counters": (_i32, [_vp, _vp, _i32]),
    "fsmt_sweep": (_i32, [_vp, _f32, _u32]),
    "fsmt_get_sweep": (_i32, [_vp, _vp, _vp, _vp, _i32]),
    "fsmt_constraint_terms": (_i32, [_vp, _f32, _u32, _vp]),
    "fsmt_update": (_i32, [_vp, _f32, _f32, _f32, _vp]),
    "fsmt_step_sizes": (_i32, [_vp, _f32, C.POINTER(_f32), C.POINTER(_f32)]),
    "fsmt_stage_end": (_i32, [_vp, _u32, _vp]),
    "fsmt_get_model": (_i32, [_vp, _u32, _vp, _vp]),
    "fsmt_get_rounded": (_i32, [_vp, _vp, _i32]),
    "fsmt_verify": (_i32, [_vp, _vp, _vp, C.POINTER(_u32), _vp]),
    "fsmt_verify_batch": (_i32, [_vp, _u32, _vp, _vp, _i32, _vp, _vp]),
    "fsmt_kernel_launches": (_u64, [_vp]),
    "fsmt_restarts": (_u32, [_vp]),
    "fsmt_device_buffers": (_i32, [_vp] + [C.POINTER(_vp)] * 7),
    "fsmt_time_sweep": (_i32, [_vp, _f32, _u32, _u32, C.POINTER(_f64)]),
    "fsmt_run_stage": (_i32, [_vp, _u32, _f32, _u32, _vp, C.POINTER(_u32)]),
    "fsmt_set_timing": (_i32, [_vp, _i32]),
    "fsmt_get_timing": (_i32, [_vp, _vp, _vp, _i32]),
    "fsmt_jit_info": (_i32, [_vp, C.POINTER(_u32), C.POINTER(_u32), C.POINTER(_u32), C.c_char_p, C.c_size_t]),
    "fsmt_jit_source": (C.c_size_t, [_vp, C.c_char_p, C.c_size_t]),
    "fsmt_mc_allreduce_f64": (_i32, [_vp, _vp, C.c_uint64, C.c_uint32, C.c_uint32]),
    "fsmt_prepare": (_i32, [_vp, _u32]),
    "fsmt_eval": (_i32, [_vp, _u32, _vp, _vp, _f32, _vp, _u32, _vp, _vp, _vp, _i32]),
    "fsmt_jit_check": (_i32, [_vp, C.POINTER(C.c_size_t), C.c_char_p, C.c_size_t]),
    "fsmt_shard": (_i32, [_vp, _u32, _u32, _u32]),
    "fsmt_bind_buffers": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "fsmt_bind_slot_grads": (_i32, [_vp, _vp]),
    "fsmt_sweep_finish": (_i32, [_vp]),
}
for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


class FsmtError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")
        self.status = status


def _ptr(arr, dtype=None):
    """(pointer, where) for a numpy array (host) or a torch tensor (device or host)."""
    if arr is None:
        return None, HOST
    if isinstance(arr, np.ndarray):
        if dtype is not None and arr.dtype != dtype:
            raise TypeError(f"expected {np.dtype(dtype)}, got {arr.dtype}")
        if not arr.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return arr.ctypes.data, HOST
    # torch tensor (duck-typed to avoid importing torch here)
    if not arr.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return arr.data_ptr(), (DEVICE if arr.is_cuda else HOST)
