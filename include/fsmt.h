/*
 * fsmt.h — C ABI of the B200-native FourierSMT hot path (arXiv 2603.22877).
 *
 * Citation convention: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
 * R<k> = reading k in DESIGN.md §3.  The library is one shared object
 * (paper_2603_22877_b200/libfsmt.so); every step of the path runs in its own
 * sm_100a CUDA kernels.  No C++ exception crosses this boundary; every call
 * returns an fsmt_status, and on failure fsmt_last_error() holds a message
 * (parse errors carry "line:col: msg").  Outputs are written only on FSMT_OK.
 *
 * Call order (enforced, FSMT_ERR_STATE otherwise):
 *     fsmt_create -> fsmt_load_formula -> fsmt_build_xbdd -> [fsmt_set_params]
 *       -> fsmt_solve                                   (whole Alg.2, one call)
 *       -> fsmt_begin -> {fsmt_sweep, fsmt_update, fsmt_stage_end}*   (step API)
 * A context is bound to one CUDA device, owns all its device memory and is not
 * thread-safe.  Pointer arguments marked "where" are host pointers when
 * where == FSMT_HOST and device pointers (on the ctx's device) when
 * where == FSMT_DEVICE; the library never keeps a caller pointer after return.
 *
 * Layouts: per-restart state is restart-minor, row = variable:
 *     a[n_bool][R] f32, b[n_real][R] f32, grad_a[n_bool][R] f64, grad_b[n_real][R] f64,
 *     U[n_cons][R] u16, x[n_bool][R] i8, obj[R] f64, unsat[R] u32, umax[R] u32.
 * Truth encoding: -1 = True, +1 = False.
 */
#ifndef FSMT_H
#define FSMT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fsmt_ctx fsmt_ctx;

typedef enum {
    FSMT_OK = 0,
    FSMT_ERR_ARG = 1,          /* NULL / out-of-range argument */
    FSMT_ERR_PARSE = 2,        /* HSMT syntax / validation error */
    FSMT_ERR_UNSUPPORTED = 3,  /* '=' atoms (R9), non-positive weights */
    FSMT_ERR_STATE = 4,        /* call out of order */
    FSMT_ERR_NODE_BUDGET = 5,  /* a constraint's xBDD exceeds the node budget / encoding limits */
    FSMT_ERR_OOM = 6,          /* device or host allocation failed */
    FSMT_ERR_CUDA = 7,         /* CUDA runtime error (no device, launch failure, ...) */
    FSMT_ERR_TIMEOUT = 8,      /* time limit hit inside fsmt_solve (verdict is still set) */
    FSMT_ERR_RANGE = 9         /* ERWA weights 2^(U[c][r] + e_t) (R18) beyond the fp64 range of the
                                  accumulation (U + e_t past ~900), or a u16 counter past 65535 */
} fsmt_status;

typedef enum { FSMT_UNKNOWN = 0, FSMT_SAT = 10 } fsmt_verdict;   /* S:514 exit codes */

enum { FSMT_HOST = 0, FSMT_DEVICE = 1 };
enum { FSMT_ROUND_SIGN = 0, FSMT_ROUND_PHILOX = 1 };             /* R17 */
enum { FSMT_ERWA_VERBATIM = 0, FSMT_ERWA_RESET0 = 1 };           /* R18 */

typedef struct {
    uint32_t n_bool, n_real, n_atoms, n_cons;
    uint32_t n_templates;      /* distinct canonical xBDDs (Def.2, R7) */
    uint32_t max_slots;        /* max distinct variables in one constraint (R5) */
    uint32_t max_nodes;        /* max decision nodes in one template */
    uint32_t n_bounded;        /* reals with a finite projection bound (R15) */
    uint64_t n_nodes;          /* sum over constraints of |V_c| */
    uint64_t n_slot_refs;      /* sum over constraints of slot count */
    uint32_t n_halfspaces;     /* multi-variable unit atom literals (projection halfspaces, R33) */
    uint32_t n_slot_rows;      /* rows of the symmetric classes' slot-table gradient gu[rows][R] (0: none) */
} fsmt_dims;

typedef struct {
    const float* kappas;       /* annealing schedule as kappa_t = 1/sigma_t >= 0 (Alg.2, R11/R12); NULL -> 0.1..2.0 */
    uint32_t n_stages;         /* length of kappas (ignored when kappas == NULL) */
    float eta;                 /* PGD step size (Eq.11, R13); <= 0 -> 0.05 */
    float eps;                 /* epsilon of Eq.14 (R14); <= 0 -> 1e-2 */
    uint32_t rounding;         /* FSMT_ROUND_SIGN (Alg.1 line 10) | FSMT_ROUND_PHILOX (Eq.4) */
    uint32_t erwa_mode;        /* FSMT_ERWA_VERBATIM (Alg.2 h<-1) | FSMT_ERWA_RESET0 */
    double time_limit_s;       /* <= 0: none (P:696 uses 1000 s) */
    uint32_t eta_mode;         /* step size in stage t (R13): 0 eta; 1 eta/kappa_t; 2 eta/kappa_t^2 (the
                                  kappa-scaling of 1/L); 3 block steps: eta for a, eta/kappa_t^2
                                  for b (only the real block's Lipschitz term grows with kappa)
                                  -- kappa_t < 1 counts as 1 */
    uint32_t proj_iters;       /* projection of the real block (Def.1/Prop.1): 0 = R15 (interval
                                  clamps from single-variable unit atoms; multi-variable unit atoms stay
                                  soft); N > 0 = R33: the QP with every unit atom, by N sweeps of Dykstra's
                                  algorithm over the halfspaces g.b <= h then the box, at init and after every
                                  gradient step (<= 100000; FSMT_ERR_ARG above; fsmt_begin fails with
                                  FSMT_ERR_ARG when the halfspace variables and corrections exceed the 227 KB
                                  of shared memory of one CTA) */
    uint32_t n_roundings;      /* R34 (FSMT_ROUND_PHILOX only): draws of R(a) per stage, the first with the
                                  fewest violated constraints kept per restart (0/1 = one draw; <= 4096);
                                  needs the unsharded mode (fsmt_stage_end fails with FSMT_ERR_STATE) */
} fsmt_params;

typedef struct {
    uint32_t stages_run;       /* annealing stages executed */
    uint32_t steps_run;        /* PGD steps executed (all stages) */
    uint32_t winner_restart;   /* restart whose model is returned */
    uint32_t winner_stage;     /* stage at which it was found (1-based) */
    uint32_t best_unsat;       /* unsat count of the returned model (0 iff SAT) */
    uint32_t host_verified;    /* 1 iff the returned model passed the host fp64 re-check */
    double solve_ms;           /* wall time of fsmt_solve after build */
    double evals;              /* constraint x restart COP+grad evaluations performed */
} fsmt_stats;

/* ---- lifecycle -------------------------------------------------------------------------- */

/* Create a context on CUDA device `cuda_device`. FSMT_ERR_CUDA if the device is unusable.
 * cuda_device == -1 creates a HOST-ONLY context: load / build / dims / bounds / dump /
 * fsmt_verify work (they are host code); every kernel-backed call returns FSMT_ERR_CUDA. */
fsmt_status fsmt_create(int cuda_device, fsmt_ctx** out);
void fsmt_destroy(fsmt_ctx* ctx);
/* Last error message of ctx (never NULL; "" when none). */
const char* fsmt_last_error(const fsmt_ctx* ctx);
/* Bind a cudaStream_t (as void*) for all subsequent launches; NULL = the ctx's own (non-blocking)
 * stream.  The legacy default stream is cudaStreamLegacy ((void*)1): a framework whose current
 * stream handle is 0 (e.g. torch's default stream) must pass 1, not NULL, to be ordered with it. */
fsmt_status fsmt_bind_stream(fsmt_ctx* ctx, void* cuda_stream);

/* ---- a0: formula -> xBDDs (Alg.1 lines 1-2) ---------------------------------- */

/* Parse HSMT text (grammar in DESIGN.md §2).  Atoms are canonicalised to
 * q.y <= q0 / < q0; '=' is rejected (FSMT_ERR_UNSUPPORTED, R9).  The text is
 * copied; a prior formula is replaced (and all derived state dropped). */
fsmt_status fsmt_load_formula(fsmt_ctx* ctx, const char* hsmt, size_t len);

/* Compile every constraint to its reduced ordered xBDD over its slots (Def.2
 * "atomic constraints as propositional variables"; slot order R6, numbering R7),
 * dedup into templates, derive the projection bounds (R15), flatten to SoA and upload.
 * node_budget: max decision nodes per constraint (0 -> 32767, also the encoding limit). */
fsmt_status fsmt_build_xbdd(fsmt_ctx* ctx, uint64_t node_budget);

/* Optional, after fsmt_build_xbdd: compile a second copy of the specialised sweep/check
 * kernels (K1, K5; DESIGN.md §7 items 11 and 13) for exactly R restarts: R as a compile-time
 * constant, U[c][r] loaded 3 constraints ahead when U exceeds the L2, and the hot sweep's
 * register cap chosen among 64 / 72 / none as the first whose kernel does not spill (NVRTC +
 * load, up to three candidate compiles, a few seconds).  Every later launch over a state of
 * exactly R restarts (fsmt_begin / fsmt_solve with restarts == R) uses it; other R keep the
 * generic kernels.  Per constraint and restart the arithmetic is the generic kernels'.  R == 0
 * drops the copy.  FSMT_ERR_STATE before build; FSMT_ERR_CUDA if no candidate compiles (the
 * generic kernels stay in use); OK and no effect for a host-only context or a formula
 * without specialised kernel classes. */
fsmt_status fsmt_prepare(fsmt_ctx* ctx, uint32_t R);

fsmt_status fsmt_get_dims(const fsmt_ctx* ctx, fsmt_dims* out);
/* Projection bounds lo[n_real], hi[n_real] (host, f32; +-inf when unbounded). */
fsmt_status fsmt_get_bounds(const fsmt_ctx* ctx, float* lo, float* hi);
/* Canonical structure dump: <dir>/templates.jsonl + <dir>/constraints.bin. */
fsmt_status fsmt_dump_structure(const fsmt_ctx* ctx, const char* dir);

/* ---- whole solve (Alg.2 around Alg.1) ----------------------------- */

fsmt_status fsmt_set_params(fsmt_ctx* ctx, const fsmt_params* params);   /* NULL -> defaults */

/* Run `restarts` lock-step restarts of Alg.2 with `steps` PGD steps per stage (R21),
 * seeded Philox init (R20).  verdict = FSMT_SAT only if a restart's rounded model passes
 * the device exact check (K5) AND the host fp64 re-check; the winner is the
 * lexicographically smallest (stage, restart).  Otherwise FSMT_UNKNOWN and the
 * outputs hold the model with the smallest (unsat, stage, restart).
 * x_out[n_bool] in {-1,+1}, y_out[n_real] (host, caller-allocated); stats may be NULL. */
fsmt_status fsmt_solve(fsmt_ctx* ctx, uint32_t restarts, uint32_t steps, uint64_t seed,
                       fsmt_verdict* verdict, int8_t* x_out, float* y_out, fsmt_stats* stats);

/* ---- step API (one stage = S x {sweep, update} + stage_end); the multi-GPU driver and
 *      the parity tests use it; it runs exactly the kernels fsmt_solve runs ------------- */

/* Allocate per-restart state for R restarts and run K0 (Philox init, R20) with global
 * restart ids restart_offset..restart_offset+R-1; U <- 0. */
fsmt_status fsmt_begin(fsmt_ctx* ctx, uint32_t restarts, uint64_t seed, uint32_t restart_offset);
/* Overwrite / read the relaxed point (a[n_bool][R], b[n_real][R]). set_state does NOT project. */
fsmt_status fsmt_set_state(fsmt_ctx* ctx, const float* a, const float* b, int where);
fsmt_status fsmt_get_state(fsmt_ctx* ctx, float* a, float* b, int where);
/* Overwrite / read the ERWA violation counters U[n_cons][R] u16 (R18), original constraint order. */
fsmt_status fsmt_set_counters(fsmt_ctx* ctx, const uint16_t* U, int where);
fsmt_status fsmt_get_counters(fsmt_ctx* ctx, uint16_t* U, int where);

/* K1: objective and gradient at the current point for all restarts (a1-a4 of SURVEY §8(a)):
 * obj[r] = sum_c w_cr E_c (Eq.10), grad = dC/d(a,b) (Alg.B with the sign of R1, chain rule
 * P:1326-1327), w_cr = w_c * 2^(U[c][r] + e_t), e_t = max(t-2,0)/2 (VERBATIM) or 0 (RESET0).
 * Per-term arithmetic is fp32; every fp64 partial sum is rounded to a per-restart power-of-two
 * grid before it is added, so obj and the gradients are exact sums of those values: bitwise
 * reproducible and independent of restart or constraint sharding (DESIGN.md §7 item 14; the
 * grid is <= 2^-48 of an a-priori bound of the restart's gradient).  FSMT_ERR_RANGE when
 * e_t > 600 (weights beyond fp64). */
fsmt_status fsmt_sweep(fsmt_ctx* ctx, float kappa, uint32_t stage_t);
/* Read the last sweep's outputs: grad_a[n_bool][R], grad_b[n_real][R] (f64), obj[R] (f64).
 * Any pointer may be NULL. */
fsmt_status fsmt_get_sweep(fsmt_ctx* ctx, double* grad_a, double* grad_b, double* obj, int where);
/* One call for the parity / bench hook of SURVEY §8(b): objective and gradient of R restarts at
 * the given point.  Allocates (fsmt_begin, seed 0) when no state of R restarts exists, then
 * overwrites a[n_bool][R], b[n_real][R] (not projected) and the ERWA counters (U[n_cons][R];
 * NULL = all 0), runs K1 (= fsmt_sweep(kappa, stage_t)) and writes obj[R], grad_a[n_bool][R],
 * grad_b[n_real][R] (f64; any output may be NULL).  All pointers are host (FSMT_HOST) or device
 * (FSMT_DEVICE) per `where`.  Replaces the context's current state. */
fsmt_status fsmt_eval(fsmt_ctx* ctx, uint32_t R, const float* a, const float* b, float kappa, const uint16_t* U,
                      uint32_t stage_t, double* obj, double* grad_a, double* grad_b, int where);
/* Per-constraint E_c for restart r from the last sweep's kernels (debug/parity hook, host E[n_cons]). */
fsmt_status fsmt_constraint_terms(fsmt_ctx* ctx, float kappa, uint32_t restart, double* E);

/* K3: projected gradient step (Eq.11-14): for every non-frozen restart,
 * (a',b') = proj(a - eta*grad_a, b - eta_b*grad_b); gm2[r] = ||(a-a')/eta||^2 + ||(b-b')/eta_b||^2
 * (Eq.13 blockwise); if gm2 <= eps^2 the restart is frozen for the rest of the stage (no update),
 * else (a,b) <- (a',b').  eta_b <= 0 means eta_b = eta (Eq.11's single step).  fsmt_step_sizes
 * gives the (eta, eta_b) of a stage under the ctx's eta_mode (what fsmt_run_stage uses).
 * gm2_out[R] (host, may be NULL) receives the squared gradient-mapping norms. */
fsmt_status fsmt_update(fsmt_ctx* ctx, float eta, float eta_b, float eps, double* gm2_out);
/* The step sizes of a stage at kappa under the ctx params (eta, eta_mode; R13): eta_a for the
 * Boolean block, eta_b for the real block. */
fsmt_status fsmt_step_sizes(const fsmt_ctx* ctx, float kappa, float* eta_a, float* eta_b);

/* K4+K5 (a6-a9): round x = sgn(a) or R(a) (R17), y = b; exact check of every constraint
 * (R22); U[c][r] += u_c; umax[r] = max_c U[c][r]; unsat[r] = #violated; clears the per-stage
 * frozen flags.  unsat_out[R] (host, may be NULL).  FSMT_ERR_RANGE when a stage's sweep took the
 * ERWA weights 2^(U + e_t) beyond the fp64 range (U + e_t past ~900) or a counter passed 65535
 * (never silently saturated). */
fsmt_status fsmt_stage_end(fsmt_ctx* ctx, uint32_t stage_t, uint32_t* unsat_out);
/* One whole annealing stage for all restarts, as fsmt_solve runs it (Alg.2 loop body,
 * P:513-528): `steps` x {K1 sweep at kappa, K3 update(fsmt_step_sizes(kappa), eps)} then K4+K5
 * stage_end.  The frozen flags are cleared first.  unsat_out[R] (host, may be NULL); *min_unsat
 * (may be NULL) receives min_r unsat[r].  Uses the ctx params (eta, eta_mode, eps, rounding,
 * erwa_mode).  FSMT_ERR_STATE on a constraint-sharded context with world > 1 (its steps need the
 * caller's all-reduces); FSMT_ERR_RANGE as fsmt_stage_end / fsmt_sweep. */
fsmt_status fsmt_run_stage(fsmt_ctx* ctx, uint32_t stage_t, float kappa, uint32_t steps, uint32_t* unsat_out,
                           uint32_t* min_unsat);

/* Multi-GPU sharding. mode 0 = restart-sharded: this context evaluates every
 * constraint (ranks differ only by fsmt_begin's restart_offset). mode 1 = constraint-sharded:
 * this context sweeps (K1) and checks (K5) only its contiguous share of the constraints
 * (tile range balanced by constraint count), so grad_a/grad_b/obj and unsat are PARTIAL sums
 * the caller must all-reduce (SUM) across ranks before fsmt_update / before reading unsat;
 * every rank then holds and updates all R restarts identically. Call after fsmt_build_xbdd. */
fsmt_status fsmt_shard(fsmt_ctx* ctx, uint32_t rank, uint32_t world, uint32_t mode);
/* Constraint-sharded mode with symmetric classes (n_slot_rows > 0): fsmt_sweep leaves the
 * slot-table gradient rows gu[n_slot_rows][R] f64 (grid units, partial) and does NOT chain them into
 * grad_a / grad_b; the caller all-reduces gu with the gradients, then calls fsmt_sweep_finish, which
 * chains the summed rows identically on every rank (the chain's rounding is not linear, so it must
 * see the full rows).  Unsharded / restart-sharded: fsmt_sweep chains them itself and
 * fsmt_sweep_finish is a no-op.  fsmt_bind_slot_grads binds caller device memory for gu. */
fsmt_status fsmt_sweep_finish(fsmt_ctx* ctx);
fsmt_status fsmt_bind_slot_grads(fsmt_ctx* ctx, void* gu);
/* Replace the ctx's grad_a[n_bool][R] f64, grad_b[n_real][R] f64, obj[R] f64, unsat[R] u32 and
 * umax[R] u32 (max_c U[c][r], the weight shift of the sweep; its current values are copied in)
 * device buffers with caller-owned device memory of the same shapes (NULL keeps the ctx's own),
 * e.g. torch tensors that torch.distributed all-reduces.  In constraint-sharded mode the caller
 * all-reduces grad/obj (SUM, after fsmt_sweep), unsat (SUM) and umax (MAX, after fsmt_stage_end);
 * the sums are exact (fsmt_sweep), so every rank holds the single-GPU values bit for bit.
 * FSMT_ERR_ARG for host memory.  Valid until the next fsmt_begin; the caller keeps ownership and
 * must keep them alive; the ctx's kernels run on its bound stream (fsmt_bind_stream). */
fsmt_status fsmt_bind_buffers(fsmt_ctx* ctx, void* grad_a, void* grad_b, void* obj, void* unsat, void* umax);

/* C4 through the NVSwitch (P:690-696 runs the method on 8 GPUs): an in-switch
 * all-reduce SUM of n f64 elements of a MULTICAST buffer (NVLS) -- the flat [grad_a | grad_b | obj |
 * slot rows] buffer of the constraint-sharded mode, allocated as symmetric memory on every rank
 * (e.g. torch.distributed._symmetric_memory) with mc_ptr its multicast address.  Rank k reduces the
 * elements [k n / world, (k+1) n / world) with multimem.ld_reduce.add.f64 (the switch adds the
 * world ranks' copies) and multimem.st's the sum back to every rank's copy.  The values are on-grid
 * integers (fsmt_sweep's exact sums), so the switch's fp64 adds are exact and the result is bit-for-
 * bit the NCCL all-reduce's.  The caller brackets the call with a device barrier across the ranks
 * (every rank's sweep finished before; every rank's stores landed after).  Runs on the ctx's bound
 * stream; FSMT_ERR_ARG for a null mc_ptr, world == 0 or rank >= world.  Needs >= 2 GPUs behind
 * NVSwitch with multicast support (not testable on one GPU). */
fsmt_status fsmt_mc_allreduce_f64(fsmt_ctx* ctx, void* mc_ptr, uint64_t n, uint32_t rank, uint32_t world);

/* Rounded model of one restart from the last stage_end: x[n_bool] (-1/+1), y[n_real] (host). */
fsmt_status fsmt_get_model(fsmt_ctx* ctx, uint32_t restart, int8_t* x_out, float* y_out);
/* Rounded Booleans of all restarts from the last stage_end: x[n_bool][R] int8 (where). */
fsmt_status fsmt_get_rounded(fsmt_ctx* ctx, int8_t* x, int where);

/* Host exact fp64 check of one model (Thm.1, R22): n_unsat, per_con[n_cons] (1 = violated,
 * may be NULL). Runs on the CPU (it is the re-verification step of fsmt_solve). */
fsmt_status fsmt_verify(fsmt_ctx* ctx, const int8_t* x, const float* y, uint32_t* n_unsat, uint8_t* per_con);

/* Device verification of arbitrary models: x[n_bool][R] i8, y[n_real][R] f32 (where),
 * unsat_out[R] (host), per_con[n_cons][R] u8 (host, may be NULL). Uses the K5 kernel. */
fsmt_status fsmt_verify_batch(fsmt_ctx* ctx, uint32_t R, const int8_t* x, const float* y, int where,
                              uint32_t* unsat_out, uint8_t* per_con);

/* ---- introspection ------------------------------------------------------------------------ */
/* Work plan of the sweep: number of JIT-specialised kernel classes, tiles, and
 * constraints the specialised kernel covers (0 when it is not active); msg receives
 * "active", "host-only", "no JIT classes" or the NVRTC / load error. Setting FSMT_JIT=0 in the
 * environment before fsmt_build_xbdd disables specialisation (every constraint then runs
 * through the generic interpreter kernel). */
fsmt_status fsmt_jit_info(const fsmt_ctx* ctx, uint32_t* n_jit_classes, uint32_t* n_tiles, uint32_t* jit_cons,
                          char* msg, size_t msg_len);
/* Copies the generated CUDA source of the specialised sweep into buf (NUL-terminated, truncated
 * to len); returns the full size including the NUL (0 if not built). Host-only contexts too. */
size_t fsmt_jit_source(const fsmt_ctx* ctx, char* buf, size_t len);
/* Compile the specialised sweep with NVRTC only (no device needed; host-only contexts too):
 * FSMT_OK and the cubin size, or FSMT_ERR_CUDA with the compiler log in fsmt_last_error. The
 * compiler log (ptxas register / spill report) is copied to log (may be NULL). */
fsmt_status fsmt_jit_check(fsmt_ctx* ctx, size_t* cubin_bytes, char* log, size_t log_len);
/* Number of this library's kernel launches since the ctx was created. */
uint64_t fsmt_kernel_launches(const fsmt_ctx* ctx);
/* Current restart count (0 before fsmt_begin). */
uint32_t fsmt_restarts(const fsmt_ctx* ctx);
/* Device pointers of the state buffers (for torch.distributed collectives); any may be NULL. */
fsmt_status fsmt_device_buffers(fsmt_ctx* ctx, void** a, void** b, void** grad_a, void** grad_b,
                                void** U, void** obj, void** unsat);
/* Time the sweep kernel alone: runs `iters` K1 launches on the ctx stream and returns the
 * average per-launch device time in ms measured with CUDA events on that stream. */
fsmt_status fsmt_time_sweep(fsmt_ctx* ctx, float kappa, uint32_t stage_t, uint32_t iters, double* ms_out);
/* Per-kernel device timing: when enabled, every K1 / K3 / K5 launch is bracketed by CUDA
 * events on the launch stream.  fsmt_get_timing synchronises and returns, per kernel class
 * k in {0: K1 sweep, 1: K3 update (3 launches), 2: K4+K5 stage end}, the summed device ms
 * and the launch-group count since the last reset.  ms[3], count[3]. */
fsmt_status fsmt_set_timing(fsmt_ctx* ctx, int enable);
fsmt_status fsmt_get_timing(fsmt_ctx* ctx, double* ms, uint64_t* count, int reset);

#ifdef __cplusplus
}
#endif
#endif /* FSMT_H */
