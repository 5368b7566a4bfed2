// Internal data model of the FourierSMT core (host side).  See include/fsmt.h for the ABI.
// P:n = PAPER.md line n, S:n = SPEC.md line n, R<k> = DESIGN.md §3 reading k.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace fsmt {

// Truth encoding: -1 = True. Terminal ids in the canonical xBDD numbering (R7).
constexpr int kFalse = -1;
constexpr int kTrue = -2;

struct ParseError {
    int line, col;
    std::string msg;
    bool unsupported;  // maps to FSMT_ERR_UNSUPPORTED ('=' atoms, bad weights)
};

// Expression pool node: op in {LIT, AND, OR, XOR, NOT}; LIT: kind 0 = Boolean var, 1 = atom.
enum ExprOp : uint8_t { OP_LIT = 0, OP_AND = 1, OP_OR = 2, OP_XOR = 3, OP_NOT = 4 };
struct ExprNode {
    uint8_t op;
    uint8_t kind;     // LIT only
    uint32_t idx;     // LIT only
    uint32_t first;   // first child index in Formula::kids (AND/OR/XOR/NOT)
    uint32_t n;       // number of children
};

enum ConsKind : uint8_t { K_OR = 0, K_CARD = 1, K_NAE = 2, K_XOR = 3, K_EXPR = 4 };
struct Lit {
    uint8_t kind;     // 0 Boolean, 1 atom
    uint8_t neg;
    uint32_t idx;
};
struct Constraint {
    uint8_t kind;
    uint32_t k;           // CARD threshold: sat iff #true <= k
    uint32_t lit_first;   // symmetric: literals in Formula::lits
    uint32_t lit_n;
    uint32_t expr_root;   // K_EXPR: root node in Formula::expr
    double weight;
};

// Canonical atoms q.y <= q0 / q.y < q0, CSR over reals.
struct Formula {
    uint32_t n_bool = 0, n_real = 0;
    std::vector<uint32_t> atom_rowptr{0};
    std::vector<uint32_t> atom_col;
    std::vector<double> atom_val;
    std::vector<double> atom_rhs;
    std::vector<uint8_t> atom_strict;
    std::vector<Constraint> cons;
    std::vector<Lit> lits;
    std::vector<ExprNode> expr;
    std::vector<uint32_t> kids;
    uint32_t n_atoms() const { return (uint32_t)atom_rhs.size(); }
};

// Parses HSMT. Throws ParseError.
Formula parse_hsmt(const char* text, size_t len);

// Decision node of a template: level = slot position; hi = slot literal True.
struct TNode {
    uint16_t level;
    int16_t hi;
    int16_t lo;
    uint16_t pad;
};

struct Template {
    std::vector<uint8_t> kinds;   // per slot: 0 Boolean, 1 atom
    std::vector<TNode> nodes;     // canonical numbering (R7)
    int root;                     // node id, or kFalse / kTrue for constant constraints
};

struct Built {
    std::vector<Template> tmpls;
    std::vector<uint32_t> cons_tmpl;       // [C]
    std::vector<uint32_t> cons_slot_off;   // [C+1]
    std::vector<uint32_t> slot_ids;        // global var / atom ids, per constraint slot
    std::vector<float> cons_w;             // [C] base weights w_c (Alg.2 input)
    std::vector<float> lo, hi;             // projection bounds (R15), f32
    uint32_t max_slots = 0, max_nodes = 0, n_bounded = 0;
    uint64_t n_nodes = 0;
    // symmetric constraints over distinct variables (count-DP fast path):
    // cons_sym = 1 + kind (OR, CARD, NAE, XOR) or 0; slot_neg = literal polarity per slot
    std::vector<uint8_t> cons_sym;         // [C]
    std::vector<uint16_t> cons_k;          // [C] CARD threshold
    std::vector<uint8_t> slot_neg;         // parallel to slot_ids
    // multi-variable unit atom literals as halfspaces g.b <= h (Prop.1, reading R33)
    std::vector<uint32_t> h_rowptr{0}, h_col;
    std::vector<double> h_g, h_h;
};

// ---- device work plan (csrc/tiles.cpp) -----------------------------------------------------
// Constraints are permuted into an internal order grouped into tiles: a tile is a run of
// constraints of one kernel class (template + nnz of each atom slot) whose variables fit a
// small local table, so the JIT-specialised sweep accumulates their gradients on chip.
constexpr uint32_t kTileVmaxDefault = 48;    // stream variables (shared-memory rows) per tile (FSMT_TILE_VMAX)
constexpr uint32_t kTileRmaxDefault = 128;   // run variables per tile (FSMT_TILE_RMAX)
constexpr uint32_t kTileCmax = 64;        // constraints per tile
constexpr uint32_t kUPad = 16;            // spare constraint rows after U (the sweep's U prefetch, <= 12 ahead)
constexpr uint32_t kGroupVarsDefault = 64;   // variables per footprint group (VMAX/2)

struct KClass {
    uint32_t tmpl;
    std::vector<uint8_t> nnz;    // per atom slot (slot order)
    uint32_t n_refs;             // Boolean slots + sum nnz
    uint32_t words;              // record words before padding
    uint32_t stride4;            // record stride in uint4
    uint32_t vstride4;           // K5 record stride in uint4 (atom id per atom slot)
    bool jit;
    uint64_t n_cons;
    std::vector<uint8_t> stream;  // per reference: 1 = changes most constraints (no run register)
    // affine groups: reference r with aff_head[r] = q >= 0 reads, in every constraint of the
    // class, the variable of q plus aff_dg[r] at the local (tile) index of q plus aff_dl[r]
    // (e.g. the 7 bits and 2 coordinates of one placement module): q's check / lookup serves all
    std::vector<int32_t> aff_head, aff_dg, aff_dl;
    std::vector<int32_t> alias;   // per reference: earlier reference with the same variable in every
                                  // constraint of the class (one load, one accumulator), or -1
    // record compression: logical word w is stored at position wpos[w] of the compressed record,
    // or (wpos[w] < 0) is the same for every constraint of the class and is emitted as the
    // literal wconst[w] in the generated code (e.g. unit weights, +-1 coefficients, 1/||q||)
    std::vector<int32_t> wpos;
    std::vector<uint32_t> wconst;
    // symmetric class: every OR/CARD/NAE/XOR constraint of one (kind, L, k) over
    // distinct variables shares the all-positive diagram stmpl; slots read shared probability
    // tables (Booleans and the symmetric classes' atoms), literal polarities are record sign bits
    bool sym = false;
    uint32_t sym_kind = 0, sym_L = 0, sym_k = 0;
    Template stmpl;
    // count class (CARD only): the sweep evaluates the constraint by its count distribution
    // (O(L^2)) instead of the xBDD's messages, and K5 counts true literals
    bool count = false;
    // product class (OR / NAE / XOR): the COP is a closed form in leave-one-out products of the literal
    // probabilities (OR 1 - prod pf, NAE 1 - prod pt - prod pf, XOR (1 - prod (pf - pt)) / 2; Cor.1),
    // evaluated in O(L) with prefix / suffix products (no division, R28b)
    bool prod = false;
    // K5 record folding: every constraint of the class has the same coefficients and strictness
    // at each atom slot (kept here, emitted as exact fp64 literals); the K5 record then holds only
    // the atoms' fp64 right-hand sides
    bool vfold = false;
    std::vector<std::vector<double>> vcoef;   // per atom slot
    std::vector<uint8_t> vstrict;             // per atom slot
};

// n_vars = n_stream | n_run << 16; tile_vars[var_off ..) holds the stream variables then the run
// variables; pad0 = record uint4s, pad1 = K5 record offset (uint4)
struct TileDesc {                // mirrored in the JIT source (32 bytes)
    uint32_t kclass, cons_begin, n_cons, var_off, n_vars, rec_off, pad0, pad1;
};

struct Plan {
    std::vector<uint32_t> order;      // internal -> original constraint id
    std::vector<uint32_t> pos;        // original -> internal
    std::vector<KClass> kclasses;
    std::vector<uint32_t> cons_kclass;  // internal order
    std::vector<TileDesc> tiles;      // JIT tiles only, in internal order
    std::vector<uint32_t> tile_vars;  // unified var ids: Boolean i -> i, real j -> n_bool + j
    std::vector<uint32_t> recs;       // JIT records (uint32 words, stride4*4 per constraint)
    std::vector<uint32_t> vrecs;      // K5 JIT records (atom ids, vstride4*4 per constraint); tile.pad1 = offset
    uint32_t jit_cons_end = 0;        // internal [0, jit_cons_end) are JIT constraints
    uint32_t n_jit_kclasses = 0;
    int wexp = 0;                     // base weights enter the records as w_c 2^-wexp (max <= 1, exact;
                                      // k1_prologue multiplies 2^wexp back in the fp64 flush)
    uint32_t vmax = kTileVmaxDefault; // stream variables per tile = shared-memory accumulator rows
    uint32_t rmax = kTileRmaxDefault; // run variables per tile (register accumulators, flushed to HBM)
    uint32_t group = kTileVmaxDefault;  // footprint group size in variables (FSMT_TILE_GROUP)
    uint32_t cmax = kTileCmax;        // constraints per tile (FSMT_TILE_CMAX)
    // atoms read through the slot tables by symmetric JIT classes; table row of atom sym_atoms[t]
    // is n_bool + n_real + t (rows [0, n_bool) are the Booleans, the real rows are unused)
    std::vector<uint32_t> sym_atoms;
    bool has_sym = false;
    uint32_t vmax_sym = 128;          // stream rows of symmetric-class tiles (FSMT_TILE_VMAX_SYM)
    // shared-memory rows per warp of the JIT sweep: the largest tile limit in use
    uint32_t kernel_vmax() const { return has_sym ? std::max(vmax, vmax_sym) : vmax; }
    // bytes per variable id in the sweep's shared-memory id table: u16 when every tile variable id fits
    bool vid32 = false;   // FSMT_JIT_VID32=1: 4-byte ids even when they fit 2 (parity matrix)
    uint32_t vid_bytes() const {
        if (vid32) return 4;
        for (uint32_t v : tile_vars)
            if (v > 0xFFFFu) return 4;
        return 2;
    }
    // the sweep's per-warp shared-memory record ring (two records of the widest JIT class, 16 B units)
    uint32_t ring_uint4() const {
        uint32_t ms = 1;
        for (uint32_t k = 0; k < n_jit_kclasses && k < kclasses.size(); ++k) ms = std::max(ms, kclasses[k].stride4);
        return 2 * ms;
    }
    std::vector<uint32_t> class_tile_begin;   // [n_jit_kclasses + 1]: class k's tiles are [begin[k], begin[k+1])
};

Plan make_plan(const Formula& f, const Built& b, bool enable_jit);
// CUDA source of the specialised sweep kernel for the plan's JIT classes.
// u_prefetch_default: how many constraints ahead the sweep loads U (FSMT_JIT_UPF overrides)
// k1_min_ctas > 0: __launch_bounds__(32, k1_min_ctas) on the hot sweep kernel (register cap);
// class_caps (optional, one per JIT class): the caps of the per-class hot kernels fsmt_k1_c<k>
std::string jit_source(const Formula& f, const Built& b, const Plan& p, int u_prefetch_default = 0, int k1_min_ctas = 0,
                       const std::vector<int>* class_caps = nullptr);
// Exponent k with max_c w_c 2^-k in (1/2, 1] (0 for no constraints): the weight normalisation of
// the sweep (DESIGN.md §7 item 14).
int weight_exponent(const Built& b);

struct BuildError {
    std::string msg;
    bool budget;
};

// Canonical xBDD of the all-positive symmetric constraint kind (OR/CARD/NAE/XOR) over L slots
// (slot kinds 2 = "table slot", see tiles.cpp); a constraint's literal polarities act on it as
// per-slot swaps of p_true / p_false.
Template symmetric_template(uint32_t kind, uint32_t L, uint32_t k);

// Compiles every constraint (a0 of SURVEY §8(a)). Throws BuildError.
Built build_xbdds(const Formula& f, uint64_t node_budget);

// Exact fp64 check of one atom at y (R22): s = 0; s += q_j*y_j in stored order; s <= q0 (< q0 strict).
bool eval_atom_exact(const Formula& f, uint32_t atom, const float* y, size_t stride);

// Host exact check of a full model (used as the host re-verification of fsmt_solve).
uint32_t verify_host(const Formula& f, const Built& b, const int8_t* x, const float* y, uint8_t* per_con);

std::string dump_templates_jsonl(const Built& b);
std::vector<uint8_t> dump_constraints_bin(const Built& b);

}  // namespace fsmt
