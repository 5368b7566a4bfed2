"""Thin Python face of the C ABI (include/fsmt.h): same names, argument marshalling only."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import native as N


@dataclass
class SolveResult:
    verdict: int            # N.SAT (10) or N.UNKNOWN (0)
    x: np.ndarray           # int8 [n_bool], -1 = True
    y: np.ndarray           # float32 [n_real]
    stats: dict


class Solver:
    """One fsmt_ctx.  device=-1 gives a host-only context (parse / build / dump / host verify)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        s = N.lib.fsmt_create(int(device), C.byref(h))
        if s != N.OK:
            raise N.FsmtError(s, f"fsmt_create(device={device}) failed")
        self._h = h
        self.device = device
        self.dims = None

    # ---------------------------------------------------------------- plumbing
    def _check(self, s):
        if s != N.OK:
            raise N.FsmtError(s, N.lib.fsmt_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            N.lib.fsmt_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def bind_stream(self, stream_ptr: int | None):
        """Launch on this cudaStream_t handle (int); 0 (torch's default stream) means the legacy
        default stream (cudaStreamLegacy); None = the context's own non-blocking stream."""
        if stream_ptr is not None and int(stream_ptr) == 0:
            stream_ptr = 1                                   # cudaStreamLegacy
        self._check(N.lib.fsmt_bind_stream(self._h, stream_ptr))

    # ---------------------------------------------------------------- a0
    def load_formula(self, text: str | bytes):
        data = text.encode() if isinstance(text, str) else text
        self._check(N.lib.fsmt_load_formula(self._h, data, len(data)))
        self.dims = None

    def build_xbdd(self, node_budget: int = 0):
        self._check(N.lib.fsmt_build_xbdd(self._h, int(node_budget)))
        d = N.Dims()
        self._check(N.lib.fsmt_get_dims(self._h, C.byref(d)))
        self.dims = d

    def eval(self, a, b, kappa: float, U=None, stage_t: int = 1):
        """fsmt_eval: (obj[R], grad_a[n_bool][R], grad_b[n_real][R]) at host point a, b (float32)."""
        a = np.ascontiguousarray(a, dtype=np.float32)
        b = np.ascontiguousarray(b, dtype=np.float32)
        R = a.shape[1] if a.ndim == 2 and a.shape[0] else b.shape[1]
        u = None if U is None else np.ascontiguousarray(U, dtype=np.uint16)
        obj = np.empty(R, dtype=np.float64)
        ga = np.empty((self.dims.n_bool, R), dtype=np.float64)
        gb = np.empty((self.dims.n_real, R), dtype=np.float64)
        self._check(N.lib.fsmt_eval(self._h, R, a.ctypes.data, b.ctypes.data, kappa,
                                    None if u is None else u.ctypes.data, stage_t,
                                    obj.ctypes.data, ga.ctypes.data, gb.ctypes.data, N.HOST))
        self.R = R                        # fsmt_eval leaves its R-restart state in the context
        return obj, ga, gb

    def prepare(self, R: int):
        """Compile the specialised kernels once more with R restarts as a constant (fsmt_prepare);
        launches over exactly R restarts use that copy (bit-identical, fewer instructions)."""
        self._check(N.lib.fsmt_prepare(self._h, int(R)))

    def get_dims(self) -> dict:
        d = N.Dims()
        self._check(N.lib.fsmt_get_dims(self._h, C.byref(d)))
        return {k: getattr(d, k) for k, _ in d._fields_}

    def get_bounds(self):
        lo = np.empty(self.dims.n_real, dtype=np.float32)
        hi = np.empty(self.dims.n_real, dtype=np.float32)
        self._check(N.lib.fsmt_get_bounds(self._h, lo.ctypes.data, hi.ctypes.data))
        return lo, hi

    def dump_structure(self, directory: str):
        self._check(N.lib.fsmt_dump_structure(self._h, directory.encode()))

    # ---------------------------------------------------------------- solve
    def set_params(self, kappas=None, eta=0.0, eps=0.0, rounding=N.ROUND_SIGN, erwa_mode=N.ERWA_VERBATIM,
                   time_limit_s=0.0, eta_mode=0, proj_iters=0, n_roundings=1):
        p = N.Params()
        if kappas is not None:
            self._kappas = np.ascontiguousarray(kappas, dtype=np.float32)
            p.kappas = self._kappas.ctypes.data_as(C.POINTER(C.c_float))
            p.n_stages = len(self._kappas)
        p.eta, p.eps, p.rounding, p.erwa_mode, p.time_limit_s = eta, eps, rounding, erwa_mode, time_limit_s
        p.eta_mode = eta_mode
        p.proj_iters = proj_iters
        p.n_roundings = n_roundings
        self._check(N.lib.fsmt_set_params(self._h, C.byref(p)))

    def solve(self, restarts: int, steps: int, seed: int) -> SolveResult:
        v = C.c_int()
        x = np.empty(self.dims.n_bool, dtype=np.int8)
        y = np.empty(self.dims.n_real, dtype=np.float32)
        st = N.Stats()
        s = N.lib.fsmt_solve(self._h, restarts, steps, seed, C.byref(v), x.ctypes.data, y.ctypes.data, C.byref(st))
        if s not in (N.OK, N.ERR_TIMEOUT):
            self._check(s)
        self.R = restarts                 # fsmt_solve leaves its R-restart state in the context
        stats = {k: getattr(st, k) for k, _ in st._fields_}
        stats["timeout"] = s == N.ERR_TIMEOUT
        return SolveResult(v.value, x, y, stats)

    # ---------------------------------------------------------------- step API
    def begin(self, restarts: int, seed: int, restart_offset: int = 0):
        self._check(N.lib.fsmt_begin(self._h, restarts, seed, restart_offset))
        self.R = restarts

    def set_state(self, a, b):
        pa, wa = N._ptr(a, np.float32)
        pb, wb = N._ptr(b, np.float32)
        if a is not None and b is not None and wa != wb:
            raise ValueError("a and b must both be host or both be device arrays")
        self._check(N.lib.fsmt_set_state(self._h, pa, pb, wa if a is not None else wb))

    def get_state(self):
        a = np.empty((self.dims.n_bool, self.R), dtype=np.float32)
        b = np.empty((self.dims.n_real, self.R), dtype=np.float32)
        self._check(N.lib.fsmt_get_state(self._h, a.ctypes.data, b.ctypes.data, N.HOST))
        return a, b

    def set_counters(self, U):
        """U[n_cons][R] ERWA violation counts (u16; host arrays of any integer dtype are converted)."""
        if isinstance(U, np.ndarray):
            U = np.ascontiguousarray(U, dtype=np.uint16)
        p, w = N._ptr(U, np.uint16)
        self._check(N.lib.fsmt_set_counters(self._h, p, w))

    def get_counters(self):
        U = np.empty((self.dims.n_cons, self.R), dtype=np.uint16)
        self._check(N.lib.fsmt_get_counters(self._h, U.ctypes.data, N.HOST))
        return U

    def sweep(self, kappa: float, stage_t: int = 1):
        self._check(N.lib.fsmt_sweep(self._h, kappa, stage_t))

    def sweep_finish(self):
        """fsmt_sweep_finish: constraint-sharded mode chains the all-reduced slot-table rows into the
        gradients (no-op otherwise)."""
        self._check(N.lib.fsmt_sweep_finish(self._h))

    def bind_slot_grads(self, gu):
        """Bind a device float64 [n_slot_rows][R] tensor as the slot-table gradient rows."""
        self._check(N.lib.fsmt_bind_slot_grads(self._h, None if gu is None else gu.data_ptr()))

    def get_sweep(self):
        ga = np.empty((self.dims.n_bool, self.R), dtype=np.float64)
        gb = np.empty((self.dims.n_real, self.R), dtype=np.float64)
        obj = np.empty(self.R, dtype=np.float64)
        self._check(N.lib.fsmt_get_sweep(self._h, ga.ctypes.data, gb.ctypes.data, obj.ctypes.data, N.HOST))
        return obj, ga, gb

    def constraint_terms(self, kappa: float, restart: int):
        E = np.empty(self.dims.n_cons, dtype=np.float64)
        self._check(N.lib.fsmt_constraint_terms(self._h, kappa, restart, E.ctypes.data))
        return E

    def update(self, eta: float, eps: float, want_gm2: bool = False, eta_b: float = 0.0):
        """K3 with step eta for the Booleans and eta_b (<= 0: eta) for the reals (fsmt_update)."""
        gm2 = np.empty(self.R, dtype=np.float64) if want_gm2 else None
        self._check(N.lib.fsmt_update(self._h, eta, eta_b, eps, gm2.ctypes.data if want_gm2 else None))
        return gm2

    def step_sizes(self, kappa: float):
        """(eta_a, eta_b) of a stage at kappa under the params' eta / eta_mode (fsmt_step_sizes)."""
        ea, eb = C.c_float(), C.c_float()
        self._check(N.lib.fsmt_step_sizes(self._h, kappa, C.byref(ea), C.byref(eb)))
        return ea.value, eb.value

    def stage_end(self, stage_t: int, copy: bool = True):
        """K4 + K5; returns unsat[R] (host) or None when copy=False (the result stays in the
        device unsat buffer, e.g. a bound tensor to be all-reduced)."""
        if not copy:
            self._check(N.lib.fsmt_stage_end(self._h, stage_t, None))
            return None
        u = np.empty(self.R, dtype=np.uint32)
        self._check(N.lib.fsmt_stage_end(self._h, stage_t, u.ctypes.data))
        return u

    def run_stage(self, stage_t: int, kappa: float, steps: int, want_unsat: bool = True):
        """One annealing stage (steps x {K1, K3} + K4/K5); returns (unsat[R] or None, min_unsat)."""
        u = np.empty(self.R, dtype=np.uint32) if want_unsat else None
        m = C.c_uint32()
        self._check(N.lib.fsmt_run_stage(self._h, stage_t, kappa, steps, u.ctypes.data if want_unsat else None,
                                         C.byref(m)))
        return u, m.value

    def set_timing(self, enable: bool):
        self._check(N.lib.fsmt_set_timing(self._h, int(enable)))

    def get_timing(self, reset: bool = False):
        """{kernel class: (total device ms, launch groups)} for k1_sweep / k3_update / k45_stage_end."""
        ms = np.zeros(3, dtype=np.float64)
        cnt = np.zeros(3, dtype=np.uint64)
        self._check(N.lib.fsmt_get_timing(self._h, ms.ctypes.data, cnt.ctypes.data, int(reset)))
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(["k1_sweep", "k3_update", "k45_stage_end"])}

    def get_model(self, restart: int):
        x = np.empty(self.dims.n_bool, dtype=np.int8)
        y = np.empty(self.dims.n_real, dtype=np.float32)
        self._check(N.lib.fsmt_get_model(self._h, restart, x.ctypes.data, y.ctypes.data))
        return x, y

    def get_rounded(self):
        x = np.empty((self.dims.n_bool, self.R), dtype=np.int8)
        self._check(N.lib.fsmt_get_rounded(self._h, x.ctypes.data, N.HOST))
        return x

    def verify(self, x, y, per_con: bool = False):
        x = np.ascontiguousarray(x, dtype=np.int8)
        y = np.ascontiguousarray(y, dtype=np.float32)
        n = C.c_uint32()
        pc = np.empty(self.dims.n_cons, dtype=np.uint8) if per_con else None
        self._check(N.lib.fsmt_verify(self._h, x.ctypes.data, y.ctypes.data, C.byref(n),
                                      pc.ctypes.data if per_con else None))
        return (n.value, pc) if per_con else n.value

    def verify_batch(self, x, y, per_con: bool = False):
        """x[n_bool][R] int8, y[n_real][R] float32 (numpy or device tensors)."""
        px, wx = N._ptr(x, np.int8)
        py, _ = N._ptr(y, np.float32)
        R = x.shape[1] if x.ndim == 2 else y.shape[1]
        u = np.empty(R, dtype=np.uint32)
        pc = np.empty((self.dims.n_cons, R), dtype=np.uint8) if per_con else None
        self._check(N.lib.fsmt_verify_batch(self._h, R, px, py, wx, u.ctypes.data, pc.ctypes.data if per_con else None))
        return (u, pc) if per_con else u

    # ---------------------------------------------------------------- introspection
    def kernel_launches(self) -> int:
        return int(N.lib.fsmt_kernel_launches(self._h))

    def device_buffers(self) -> dict:
        ptrs = [C.c_void_p() for _ in range(7)]
        self._check(N.lib.fsmt_device_buffers(self._h, *[C.byref(p) for p in ptrs]))
        return dict(zip(["a", "b", "grad_a", "grad_b", "U", "obj", "unsat"], [p.value for p in ptrs]))

    def jit_info(self) -> dict:
        n1, n2, n3 = C.c_uint32(), C.c_uint32(), C.c_uint32()
        buf = C.create_string_buffer(4096)
        self._check(N.lib.fsmt_jit_info(self._h, C.byref(n1), C.byref(n2), C.byref(n3), buf, 4096))
        return {"jit_classes": n1.value, "tiles": n2.value, "jit_cons": n3.value, "status": buf.value.decode()}

    def shard(self, rank: int, world: int, mode: int):
        """mode 0: restart-sharded (all constraints); 1: constraint-sharded (partial sums)."""
        self._check(N.lib.fsmt_shard(self._h, rank, world, mode))

    def bind_buffers(self, grad_a=None, grad_b=None, obj=None, unsat=None, umax=None):
        """Bind caller-owned device tensors (float64 [n_bool][R], [n_real][R], [R]; int32 [R] unsat and
        umax); host tensors are rejected (FSMT_ERR_ARG)."""
        ptr = lambda t: None if t is None else t.data_ptr()
        self._check(N.lib.fsmt_bind_buffers(self._h, ptr(grad_a), ptr(grad_b), ptr(obj), ptr(unsat), ptr(umax)))

    def mc_allreduce_f64(self, mc_ptr: int, n: int, rank: int, world: int):
        """C4 in the NVSwitch: all-reduce SUM of n f64 of a multicast buffer (fsmt_mc_allreduce_f64;
        the caller barriers the ranks before and after)."""
        self._check(N.lib.fsmt_mc_allreduce_f64(self._h, C.c_void_p(mc_ptr), n, rank, world))

    def jit_check(self):
        """NVRTC-compile the specialised sweep (no device needed): (cubin bytes, compiler log)."""
        n = C.c_size_t()
        buf = C.create_string_buffer(1 << 16)
        self._check(N.lib.fsmt_jit_check(self._h, C.byref(n), buf, 1 << 16))
        return n.value, buf.value.decode(errors="replace")

    def jit_source(self) -> str:
        n = N.lib.fsmt_jit_source(self._h, None, 0)
        if n == 0:
            return ""
        buf = C.create_string_buffer(n)
        N.lib.fsmt_jit_source(self._h, buf, n)
        return buf.value.decode()

    def time_sweep(self, kappa: float, stage_t: int, iters: int) -> float:
        ms = C.c_double()
        self._check(N.lib.fsmt_time_sweep(self._h, kappa, stage_t, iters, C.byref(ms)))
        return ms.value
