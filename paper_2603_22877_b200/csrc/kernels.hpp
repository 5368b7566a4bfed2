// Device-side data structures and kernel launchers (K0-K5) of the FourierSMT hot path.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fsmt {

// Per-restart scales of one sweep (k1_prologue; mirrored in the JIT source, DESIGN.md §7 item 14).
// The ERWA weight w_c 2^(U + e_t) (R18) enters the fp32 arithmetic as w_c 2^-wexp 2^(U - s_r)
// 2^frac(e_t) with s_r = max(0, max_c U[c][r] - kWeightWindow) (no fp32 weight overflows).  Every
// fp32 partial gradient sum v (reduced units) is flushed as the integer rint(v 2^-G_r) (fp32:
// exact scaling, values >= 2^23 are integers already) into grad_a / grad_b, which therefore hold
// integers in GRID UNITS whose sums stay below 2^51 (G_r from an a-priori bound): the fp64 sums
// are exact, whatever the order of the atomics or the sharding.  The true gradient is the
// stored value times gs = 2^(G_r + s_r + wexp + floor(e_t)) (K3 and fsmt_get_sweep apply it);
// ti = 1/gs.  The objective is flushed on its own grid in true units: rint(v oi) os.
struct FxScale {
    double gs, ti;
    double oi, os;
    float gif;                   // 2^frac(e_t) 2^-G_r (the flush scale into grid units)
    int32_t ebias;               // 127 - s_r (exponent bias of the fp32 weight 2^(U - s_r))
};
constexpr int kWeightWindow = 24;   // fp32 weights stay <= 2^24 w_c 2^-wexp

// The parameters of one annealing stage on the device (the device-side solve loop, DESIGN.md §7
// item 16): k_stage_begin copies entry t-1 of the schedule here at the top of every stage, and the
// stage's kernels read kappa / step sizes / stage number from it instead of their launch arguments
// when DevState::ds is set.
struct DevStage {
    float kappa, eta_a, eta_b;
    uint32_t t;                  // stage number (1-based): Philox rounding counter, ERWA e_t
    int32_t et_int;              // floor(e_t) (R18)
    float wfrac;                 // 2^frac(e_t)
    uint32_t pad[2];
};
// Progress of the device-side solve loop (one per solve).
struct DevSolve {
    uint32_t t;                  // the stage the next loop iteration runs (1-based)
    uint32_t t_end;              // last stage of this graph launch
    uint32_t best_unsat, best_stage, best_r;
    uint32_t done;               // 1: a restart is SAT, or t passed t_end
    uint32_t pad[2];
};

struct DevNode {          // = TNode (8 bytes): level, hi, lo (-1 FALSE, -2 TRUE), pad
    uint16_t level;
    int16_t hi;
    int16_t lo;
    uint16_t pad;
};

// Read-only formula structure in HBM (SoA).
struct DevFormula {
    uint32_t n_bool, n_real, n_cons, n_atoms;
    uint32_t max_slots, max_nodes;
    const uint32_t* cons_tmpl;      // [C]
    const uint32_t* cons_slot_off;  // [C+1]
    const uint32_t* slot_ids;       // [sum slots]
    const float* cons_w;            // [C]
    const uint32_t* tmpl_node_off;  // [T+1]
    const DevNode* nodes;           // [sum template nodes]
    const uint32_t* tmpl_kind_off;  // [T+1]
    const uint8_t* kinds;           // [sum template slots]
    const int32_t* tmpl_root;       // [T]
    const uint32_t* atom_rowptr;    // [K+1]
    const uint32_t* atom_col;       // [nnz]
    const float* atom_val;          // [nnz] f32 (smoothing)
    const double* atom_val64;       // [nnz] f64 (exact check, R22)
    const float* atom_rhs;          // [K]
    const double* atom_rhs64;       // [K]
    const uint8_t* atom_strict;     // [K]
    const float* atom_invnorm;      // [K] 1/||q_i||
    const float* lo;                // [n_real]
    const float* hi;                // [n_real]
    const uint32_t* orig;           // [C] internal -> original constraint id (constraint arrays and U
                                    //     are in the internal, tile-sorted order; see tiles.cpp)
    // Prop.1 projection with multi-variable unit atoms (R33): halfspaces g.b <= h, Dykstra sweeps
    uint32_t n_half = 0, n_hvars = 0, proj_iters = 0, n_hlevels = 0, h_nnz = 0;
    const uint32_t* h_rowptr = nullptr;  // [n_half+1], halfspaces in dependency-level order
    const uint32_t* h_col = nullptr;     // [nnz] index into hvars
    const float* h_g = nullptr;          // [nnz]
    const float* h_h = nullptr;          // [n_half]
    const float* h_inv2 = nullptr;       // [n_half] 1/||g||^2
    const uint32_t* hvars = nullptr;     // [n_hvars] reals in some halfspace (box corrections)
    const uint8_t* in_h = nullptr;       // [n_real] 1 if in some halfspace
    const uint32_t* h_level_off = nullptr;  // [n_hlevels+1] halfspace range of each level
    uint32_t generic_begin;         // internal [generic_begin, generic_end) run through the generic K1
    uint32_t generic_end;           //   (generic_end < n_cons only in constraint-sharded mode)
    // a-priori bounds of the on-grid accumulation (FxScale), over the whole formula with the
    // normalised weights w_c 2^-wexp: fx_fb = max over Booleans / slot-table rows of the summed
    // weights of their slots (|dE/dv| <= 1), fx_fa = max over reals j of sum w |q_ij| / ||q_i||
    // sqrt(2/pi) (times kappa: |dd/db_j| <= kappa sqrt(2/pi) |q_j| / ||q||),
    // fx_sw = sum of the weights (|E_c| <= 1)
    double fx_fb = 0.0, fx_fa = 0.0, fx_sw = 0.0;
    int32_t wexp = 0;
};

// Per-restart state, restart-minor (row = variable / constraint).
struct DevState {
    uint32_t R;
    float* a;          // [n_bool][R]
    float* b;          // [n_real][R]
    double* ga;        // [n_bool][R] gradient in grid units (times gsc[r]: FxScale)
    double* gb;        // [n_real][R] gradient in grid units
    uint16_t* U;       // [C][R] ERWA violation counts (R18)
    double* obj;       // [R]
    int8_t* x;         // [n_bool][R]
    uint32_t* unsat;   // [R]
    uint8_t* frozen;   // [R]
    double* gm2;       // [R]
    double* gm2_part;  // [n_parts][R]
    float* bn;         // [n_real][R] candidate b of the projected step (R33), or null
    int8_t* x_best;    // [n_bool][R] best rounding of the stage (R34), or null
    uint32_t* unsat_m; // [R]
    uint32_t* unsat_best;  // [R]
    uint8_t* better;   // [R]
    uint32_t* umax;    // [R] max_c U[c][r] (K5 keeps it; the sweep's weight shift)
    FxScale* fx;       // [R] per-restart scales of the current sweep (k1_prologue)
    const DevStage* ds = nullptr;   // device-side stage parameters (graph solve loop), or null
    double* gsc;       // [R] fx[r].gs (grid scale of the gradients, read by K3 / the output copy)
    uint32_t* flags;   // [4] flags[0]: bit 0 an ERWA counter reached 65535, bit 1 ERWA weights 2^(U + e_t)
                       //     beyond the fp64 range of the accumulation (FSMT_ERR_RANGE)
};

int sweep_smem_bytes(const DevFormula& F, int warps);

// K0: Philox init (R20) + projection.
void launch_init(const DevFormula& F, const DevState& S, uint64_t seed, uint32_t restart_offset, cudaStream_t st);
// K1 (generic interpreter): forward/backward xBDD sweep over internal constraints
// [F.generic_begin, n_cons), objective + gradient (fp64 accumulation).
void launch_sweep(const DevFormula& F, const DevState& S, float kappa, double* terms, uint32_t terms_r, cudaStream_t st);
// Before every sweep: zero grad_a, grad_b, obj (and the slot-table gradients gu[gu_rows][R] when
// non-null) and write S.fx / S.gsc for the stage exponent e_t = et_int + log2(wfrac) (wfrac = 1 or
// sqrt 2, applied in the flush).
void launch_prologue(const DevFormula& F, const DevState& S, float kappa, int et_int, float wfrac, double* gu,
                     uint64_t gu_rows, cudaStream_t st);
// umax[r] = max_c U[c][r] (after fsmt_set_counters).
void launch_umax(const DevFormula& F, const DevState& S, cudaStream_t st);
// C4 in the switch: multimem all-reduce SUM of this rank's slice of a multicast f64 buffer (NVLS)
void launch_mc_allreduce_f64(double* mc, uint64_t n, uint32_t rank, uint32_t world, cudaStream_t st);
// dst[i][r] = src[i][r] * gsc[r] (grid units -> gradient), rows x R doubles.
void launch_scale_rows(double* dst, const double* src, const double* gsc, uint64_t rows, uint32_t R, cudaStream_t st);
// K1 (JIT-specialised, tiles): see tiles.cpp / jit.cpp.
struct DevTiles {
    const void* tiles;           // TileDesc[n_tiles]
    uint32_t n_tiles;
    const void* recs;            // uint4 records
    const uint32_t* tile_vars;
    uint32_t vmax;               // stream variables (shared-memory accumulator rows) per tile (Plan::vmax)
    uint32_t rmax;               // run variables per tile (Plan::rmax)
    uint32_t ring_uint4;         // K1's per-warp shared-memory record ring, in uint4 (Plan::ring_uint4)
    uint32_t vid_bytes;          // K1's shared-memory variable-id width, 2 or 4 (Plan::vid_bytes)
    uint32_t cons_per_tile;      // mean constraints per tile (launch-time split rule)
    const void* vrecs;           // K5 records (atom ids), tile.pad1 = offset in uint4
    uint32_t first;              // global index of tiles[0] (constraint shards start mid-plan)
};
// Slot tables of the symmetric JIT classes (rows: Booleans [0, n_bool), table atom t at nv + t).
struct DevSlots {
    uint32_t n_sa = 0, nv = 0;          // table atoms; nv = n_bool + n_real
    const uint32_t* atoms = nullptr;    // [n_sa] atom ids
    float* PT = nullptr;                // [nv + n_sa][R] p_true of the row
    float* DD = nullptr;                // [n_sa][R] dd/dz factor
    double* GU = nullptr;               // [nv + n_sa][R] dE/dp_true of the row (weighted)
    uint8_t* TT = nullptr;              // [nv + n_sa][R] exact truth of the row (K5)
};
void launch_slot_prob(cudaKernel_t k, const DevFormula& F, const DevState& S, const DevSlots& D, float kappa, cudaStream_t st);
void launch_slot_chain(cudaKernel_t k, const DevFormula& F, const DevState& S, const DevSlots& D, cudaStream_t st);
void launch_slot_truth(cudaKernel_t k, const DevFormula& F, const DevState& S, const DevSlots& D, const int8_t* x,
                       const float* y, cudaStream_t st);
// K5 (JIT-specialised, tiles): exact check over the tiles of T (+ ERWA counters / per_con).
void launch_verify_jit(cudaKernel_t k, const DevFormula& F, const DevState& S, const DevTiles& T, const int8_t* x,
                       const float* y, uint16_t* U_update, uint8_t* per_con, cudaStream_t st, const uint8_t* TT = nullptr);
void launch_sweep_jit(cudaKernel_t k, const DevFormula& F, const DevState& S, const DevTiles& T, float kappa,
                      double* terms, uint32_t terms_r, cudaStream_t st, const DevSlots* D = nullptr);
// row gather for u16 matrices: dst[i][:] = src[idx[i]][:]  (U between original and internal order)
void launch_gather_rows_u16(uint16_t* dst, const uint16_t* src, const uint32_t* idx, uint32_t rows, uint32_t R,
                            cudaStream_t st);
// K3: projected step (three launches: partial norms, finalize, apply).
int update_parts(const DevFormula& F, uint32_t R);   // parts of the K3 norm (size of gm2_part / R)
// eta: step for a (Booleans); eta_b: step for b (reals), <= 0 -> eta (Eq.11 uses one eta; R13).
void launch_update(const DevFormula& F, const DevState& S, float eta, float eps, cudaStream_t st, float eta_b = 0.f);
// Dykstra projection (R33) of X [n_real][R] in place: F.proj_iters sweeps over the halfspaces then
// the box, per restart (skips frozen restarts when skip_frozen).
void launch_project(const DevFormula& F, const DevState& S, float* X, bool skip_frozen, cudaStream_t st);
size_t project_smem_bytes(const DevFormula& F, uint32_t nnz);   // k_dykstra shared memory (<= 227 KB)
// R34: keep, per restart, the rounding with the fewest violations: restarts whose unsat_m beats
// unsat_best (or m == 0) copy x into x_best.
void launch_keep_best(const DevFormula& F, const DevState& S, const uint32_t* unsat_m, uint32_t* unsat_best,
                      int8_t* x_best, uint8_t* flag, uint32_t m, cudaStream_t st);
// Device-side solve loop (DESIGN.md §7 item 16): stage parameters from the schedule, and the
// per-stage best-model / continue decision that drives the graph's WHILE node.
void launch_stage_begin(const DevSolve* sv, const DevStage* sched, DevStage* ds, cudaStream_t st);
void launch_stage_best(DevSolve* sv, const DevState& S, uint32_t n_bool, uint32_t n_real, int8_t* xk, float* yk,
                       cudaGraphConditionalHandle h, cudaStream_t st);
// K4: rounding (R17).
void launch_round(const DevFormula& F, const DevState& S, uint32_t rounding, uint64_t seed, uint32_t restart_offset,
                  uint32_t stage, cudaStream_t st);
// K5: exact verification + ERWA counter update (R18, R22).
// K5 over internal constraints [cb, ce) (ce = UINT32_MAX: to the end).
void launch_verify(const DevFormula& F, const DevState& S, const int8_t* x, const float* y, uint16_t* U_update,
                   uint8_t* per_con, cudaStream_t st, uint32_t cb = 0, uint32_t ce = UINT32_MAX);

}  // namespace fsmt
