// C-ABI implementation (include/fsmt.h): context, call-order state machine, device buffers,
// and the Alg.2 / Alg.1 driver loop around the sm_100a kernels.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/fsmt.h"
#include "fsmt_internal.hpp"
#include "jit.hpp"
#include "kernels.hpp"

using namespace fsmt;

struct fsmt_ctx {
    int device = 0;
    bool host_only = false;     // cuda_device == -1: parse/build/dump/host-verify only
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    std::string err;
    int stage = 0;              // 0 created, 1 loaded, 2 built, 3 begun
    Formula f;
    Built b;
    DevFormula F{};
    std::vector<void*> fallocs;
    DevState S{};
    std::vector<void*> sallocs;
    double* terms = nullptr;    // [C] debug hook buffer
    double* scratch = nullptr;  // [max(n_bool, n_real)][R] gradients scaled out of grid units (fsmt_get_sweep)
    // device work plan (tiles.cpp) + JIT-specialised sweep (jit.cpp)
    bool jit_enabled = true;
    Plan plan;
    std::string jit_src, jit_error;
    JitKernel jit;
    JitKernel jit_r;            // fsmt_prepare(R): the same module with R a compile-time constant
    uint32_t jit_r_R = 0;
    int jit_r_cap = 0;          // the prepared hot sweep's register cap (min CTAs/SM; 0 = none)
    bool ext_bound = false;     // fsmt_bind_buffers / fsmt_bind_slot_grads replaced state buffers
    std::vector<int> jit_r_caps;   // the per-class sweep kernels' caps (fsmt_k1_c<k>)
    DevTiles T{};
    DevSlots slots{};                  // slot tables of the symmetric JIT classes (has_sym)
    cudaGraphExec_t gexec = nullptr;   // fsmt_run_stage's PGD steps as one CUDA graph (re-used, updated)
    bool has_sym = false;
    const uint32_t* d_pos = nullptr;   // original -> internal constraint index (device)
    // constraint sharding (fsmt_shard): this context's part of the sweep and of the check
    DevTiles T_all{};                  // every JIT tile
    uint32_t vrange[2][2] = {{0, 0}, {0, 0}};   // internal constraint ranges verified by K5
    uint32_t shard_mode = 0, shard_rank = 0, shard_world = 1;
    // params
    std::vector<float> kappas;
    float eta = 0.05f, eps = 1e-2f;
    uint32_t rounding = FSMT_ROUND_SIGN, erwa_mode = FSMT_ERWA_VERBATIM, eta_mode = 0;
    uint32_t n_roundings = 1;          // R34
    double time_limit = 0.0;
    // run
    uint64_t seed = 0;
    uint32_t restart_offset = 0;
    bool rounded = false;
    uint64_t launches = 0;
    uint32_t* hflags = nullptr;        // pinned host copy of S.flags[0] (read at every stage end)
    // auxiliary streams for the concurrent per-class sweep launches (fork / join by events)
    static constexpr size_t kAux = 4;
    cudaStream_t aux[kAux] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t ev_fork = nullptr, ev_join[kAux] = {nullptr, nullptr, nullptr, nullptr};
    // per-kernel-class device timing (fsmt_set_timing)
    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_open[3];
    double t_ms[3] = {0, 0, 0};
    uint64_t t_cnt[3] = {0, 0, 0};
};

namespace {
cudaEvent_t ev_get(fsmt_ctx* ctx) {
    if (!ctx->ev_pool.empty()) {
        cudaEvent_t e = ctx->ev_pool.back();
        ctx->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}
// Brackets a launch group of kernel class k with events on the launch stream.
struct Timed {
    fsmt_ctx* ctx;
    int k;
    cudaEvent_t e0 = nullptr;
    Timed(fsmt_ctx* c, int kk) : ctx(c), k(kk) {
        if (ctx->timing) {
            e0 = ev_get(ctx);
            cudaEventRecord(e0, ctx->stream);
        }
    }
    ~Timed() {
        if (ctx->timing) {
            cudaEvent_t e1 = ev_get(ctx);
            cudaEventRecord(e1, ctx->stream);
            ctx->ev_open[k].emplace_back(e0, e1);
        }
    }
};
void timing_collect(fsmt_ctx* ctx) {
    for (int k = 0; k < 3; ++k) {
        for (auto& pr : ctx->ev_open[k]) {
            cudaEventSynchronize(pr.second);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, pr.first, pr.second);
            ctx->t_ms[k] += ms;
            ctx->t_cnt[k] += 1;
            ctx->ev_pool.push_back(pr.first);
            ctx->ev_pool.push_back(pr.second);
        }
        ctx->ev_open[k].clear();
    }
}
}  // namespace

namespace {

void default_kappas(std::vector<float>& k) {
    k.clear();
    for (int i = 1; i <= 20; ++i) k.push_back((float)(0.1 * i));   // 1/sigma = 0.1..2.0 (R12)
}

fsmt_status fail(fsmt_ctx* c, fsmt_status s, const std::string& msg) {
    if (c) c->err = msg;
    return s;
}

#define CK(call)                                                                             \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess) return fail(ctx, FSMT_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
    } while (0)

template <typename T>
fsmt_status upload(fsmt_ctx* ctx, const std::vector<T>& v, const T*& dst, std::vector<void*>& allocs) {
    void* p = nullptr;
    size_t bytes = std::max<size_t>(v.size() * sizeof(T), sizeof(T));
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) return fail(ctx, FSMT_ERR_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    allocs.push_back(p);
    if (!v.empty()) CK(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    dst = (const T*)p;
    return FSMT_OK;
}

void free_list(std::vector<void*>& v) {
    for (void* p : v) cudaFree(p);
    v.clear();
}

void drop_state(fsmt_ctx* ctx) {
    if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; }
    free_list(ctx->sallocs);
    ctx->S = DevState{};
    ctx->slots.PT = ctx->slots.DD = nullptr;
    ctx->slots.GU = nullptr;
    ctx->slots.TT = nullptr;
    ctx->scratch = nullptr;     // freed with the state allocations
    ctx->rounded = false;
    ctx->ext_bound = false;
    if (ctx->terms) { cudaFree(ctx->terms); ctx->terms = nullptr; }
}

void drop_formula(fsmt_ctx* ctx) {
    drop_state(ctx);
    free_list(ctx->fallocs);
    ctx->F = DevFormula{};
    jit_release(ctx->jit);
    jit_release(ctx->jit_r);
    ctx->jit_r_R = 0;
    ctx->T = DevTiles{};
    ctx->T_all = DevTiles{};
    ctx->slots = DevSlots{};
    ctx->has_sym = false;
    ctx->d_pos = nullptr;
}

fsmt_status upload_bytes(fsmt_ctx* ctx, const void* src, size_t bytes, const void*& dst) {
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(bytes, 16));
    if (e != cudaSuccess) return fail(ctx, FSMT_ERR_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    ctx->fallocs.push_back(p);
    if (bytes) CK(cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice));
    dst = p;
    return FSMT_OK;
}

// R18: weight during stage t = w_c * 2^(U + e_t), e_t = max(t-2,0)/2 (Alg.2 verbatim) or 0
// (reset-to-0): the integer part of e_t is applied exactly in the fp64 flush (FxScale), the
// fractional part 2^(1/2) in the fp32 weight.
int et_int_of(uint32_t stage_t, uint32_t mode) {
    if (mode == FSMT_ERWA_RESET0 || stage_t <= 2) return 0;
    return (int)((stage_t - 2) / 2);
}
float wfrac_of(uint32_t stage_t, uint32_t mode) {
    if (mode == FSMT_ERWA_RESET0 || stage_t <= 2 || (stage_t - 2) % 2 == 0) return 1.0f;
    return 1.41421356237309505f;
}


// after a stage end and a sync: the K5 overflow flag (an ERWA counter passed 255; R18 needs the
// exact count, so the u8 counter is never silently saturated)
fsmt_status check_flags(fsmt_ctx* ctx) {
    if (ctx->hflags && (*ctx->hflags & 1u))
        return fail(ctx, FSMT_ERR_RANGE, "ERWA counter overflow: a constraint was violated more than 65535 times in one "
                                         "restart (u16 U[c][r], R18)");
    if (ctx->hflags && (*ctx->hflags & 2u))
        return fail(ctx, FSMT_ERR_RANGE, "ERWA weights 2^(U + e_t) beyond the fp64 range of the accumulation (U + e_t > "
                                         "~900, R18)");
    return FSMT_OK;
}

fsmt_status need(fsmt_ctx* ctx, int stage, const char* what) {
    if (!ctx) return FSMT_ERR_ARG;
    if (stage >= 3 && ctx->host_only) return fail(ctx, FSMT_ERR_CUDA, std::string(what) + ": host-only context has no device");
    if (ctx->stage < stage) return fail(ctx, FSMT_ERR_STATE, std::string(what) + ": called out of order");
    return FSMT_OK;
}

template <typename T>
fsmt_status copy_in(fsmt_ctx* ctx, T* dst, const T* src, size_t n, int where) {
    if (n == 0) return FSMT_OK;
    if (!src) return fail(ctx, FSMT_ERR_ARG, "null input pointer");
    CK(cudaMemcpyAsync(dst, src, n * sizeof(T), where == FSMT_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return FSMT_OK;
}

template <typename T>
fsmt_status copy_out(fsmt_ctx* ctx, T* dst, const T* src, size_t n, int where) {
    if (n == 0 || !dst) return FSMT_OK;
    CK(cudaMemcpyAsync(dst, src, n * sizeof(T), where == FSMT_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return FSMT_OK;
}

fsmt_status check_launch(fsmt_ctx* ctx) {
    CK(cudaGetLastError());
    return FSMT_OK;
}

}  // namespace

extern "C" {

fsmt_status fsmt_create(int cuda_device, fsmt_ctx** out) {
    if (!out) return FSMT_ERR_ARG;
    *out = nullptr;
    if (cuda_device == -1) {
        fsmt_ctx* h = new (std::nothrow) fsmt_ctx();
        if (!h) return FSMT_ERR_OOM;
        h->host_only = true;
        default_kappas(h->kappas);
        *out = h;
        return FSMT_OK;
    }
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return FSMT_ERR_CUDA;
    if (cuda_device < 0 || cuda_device >= n) return FSMT_ERR_ARG;
    if (cudaSetDevice(cuda_device) != cudaSuccess) return FSMT_ERR_CUDA;
    fsmt_ctx* ctx = new (std::nothrow) fsmt_ctx();
    if (!ctx) return FSMT_ERR_OOM;
    ctx->device = cuda_device;
    if (cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete ctx;
        return FSMT_ERR_CUDA;
    }
    ctx->stream = ctx->own_stream;
    if (cudaMallocHost((void**)&ctx->hflags, 16) != cudaSuccess) {
        cudaStreamDestroy(ctx->own_stream);
        delete ctx;
        return FSMT_ERR_OOM;
    }
    *ctx->hflags = 0;
    for (size_t i = 0; i < fsmt_ctx::kAux; ++i)
        if (cudaStreamCreateWithFlags(&ctx->aux[i], cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&ctx->ev_join[i], cudaEventDisableTiming) != cudaSuccess) {
            fsmt_destroy(ctx);
            return FSMT_ERR_CUDA;
        }
    if (cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess) {
        fsmt_destroy(ctx);
        return FSMT_ERR_CUDA;
    }
    default_kappas(ctx->kappas);
    *out = ctx;
    return FSMT_OK;
}

void fsmt_destroy(fsmt_ctx* ctx) {
    if (!ctx) return;
    if (ctx->host_only) {
        delete ctx;
        return;
    }
    cudaSetDevice(ctx->device);
    drop_formula(ctx);
    timing_collect(ctx);
    for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    if (ctx->hflags) cudaFreeHost(ctx->hflags);
    for (size_t i = 0; i < fsmt_ctx::kAux; ++i) {
        if (ctx->aux[i]) cudaStreamDestroy(ctx->aux[i]);
        if (ctx->ev_join[i]) cudaEventDestroy(ctx->ev_join[i]);
    }
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    delete ctx;
}

const char* fsmt_last_error(const fsmt_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

fsmt_status fsmt_bind_stream(fsmt_ctx* ctx, void* s) {
    if (!ctx) return FSMT_ERR_ARG;
    ctx->stream = s ? (cudaStream_t)s : ctx->own_stream;
    return FSMT_OK;
}

fsmt_status fsmt_load_formula(fsmt_ctx* ctx, const char* text, size_t len) {
    if (!ctx || (!text && len)) return FSMT_ERR_ARG;
    if (!ctx->host_only) {
        cudaSetDevice(ctx->device);
        drop_formula(ctx);
    }
    ctx->stage = 0;
    try {
        ctx->f = parse_hsmt(text, len);
    } catch (const ParseError& e) {
        return fail(ctx, e.unsupported ? FSMT_ERR_UNSUPPORTED : FSMT_ERR_PARSE,
                    std::to_string(e.line) + ":" + std::to_string(e.col) + ": " + e.msg);
    } catch (const std::bad_alloc&) {
        return fail(ctx, FSMT_ERR_OOM, "host allocation failed while parsing");
    }
    ctx->b = Built{};
    ctx->stage = 1;
    ctx->err.clear();
    return FSMT_OK;
}

fsmt_status fsmt_build_xbdd(fsmt_ctx* ctx, uint64_t node_budget) {
    fsmt_status s = need(ctx, 1, "fsmt_build_xbdd");
    if (s) return s;
    if (!ctx->host_only) {
        cudaSetDevice(ctx->device);
        drop_formula(ctx);
    }
    ctx->stage = 1;
    try {
        ctx->b = build_xbdds(ctx->f, node_budget);
    } catch (const BuildError& e) {
        return fail(ctx, e.budget ? FSMT_ERR_NODE_BUDGET : FSMT_ERR_ARG, e.msg);
    } catch (const std::bad_alloc&) {
        return fail(ctx, FSMT_ERR_OOM, "host allocation failed while building xBDDs");
    }
    {
        const char* env = getenv("FSMT_JIT");
        ctx->jit_enabled = !(env && env[0] == '0');
        ctx->plan = make_plan(ctx->f, ctx->b, ctx->jit_enabled);
        ctx->jit_src = ctx->plan.n_jit_kclasses ? jit_source(ctx->f, ctx->b, ctx->plan) : std::string();
    }
    if (ctx->host_only) {
        ctx->stage = 2;
        ctx->err.clear();
        return FSMT_OK;
    }
    const Formula& f = ctx->f;
    const Built& b = ctx->b;
    const Plan& P = ctx->plan;
    // constraint arrays in the internal (tile-sorted) order
    const size_t C = f.cons.size();
    std::vector<uint32_t> c_tmpl(C), c_off(C + 1), c_ids;
    std::vector<float> c_w(C);
    c_ids.reserve(b.slot_ids.size());
    c_off[0] = 0;
    for (size_t i = 0; i < C; ++i) {
        const uint32_t o = P.order[i];
        c_tmpl[i] = b.cons_tmpl[o];
        c_w[i] = std::ldexp(b.cons_w[o], -P.wexp);   // normalised base weight (FxScale; exact)
        c_ids.insert(c_ids.end(), b.slot_ids.begin() + b.cons_slot_off[o], b.slot_ids.begin() + b.cons_slot_off[o + 1]);
        c_off[i + 1] = (uint32_t)c_ids.size();
    }
    // flatten templates
    std::vector<uint32_t> node_off{0}, kind_off{0};
    std::vector<DevNode> nodes;
    std::vector<uint8_t> kinds;
    std::vector<int32_t> roots;
    for (const Template& t : b.tmpls) {
        for (const TNode& n : t.nodes) nodes.push_back(DevNode{n.level, n.hi, n.lo, 0});
        kinds.insert(kinds.end(), t.kinds.begin(), t.kinds.end());
        node_off.push_back((uint32_t)nodes.size());
        kind_off.push_back((uint32_t)kinds.size());
        roots.push_back(t.root);
    }
    std::vector<float> aval(f.atom_val.size()), arhs(f.n_atoms()), ainv(f.n_atoms());
    for (size_t i = 0; i < f.atom_val.size(); ++i) aval[i] = (float)f.atom_val[i];
    for (uint32_t i = 0; i < f.n_atoms(); ++i) {
        arhs[i] = (float)f.atom_rhs[i];
        double n2 = 0.0;
        for (uint32_t t = f.atom_rowptr[i]; t < f.atom_rowptr[i + 1]; ++t) n2 += f.atom_val[t] * f.atom_val[t];
        ainv[i] = (float)(1.0 / std::sqrt(n2));
    }
    DevFormula& F = ctx->F;
    F.n_bool = f.n_bool;
    F.n_real = f.n_real;
    F.n_cons = (uint32_t)f.cons.size();
    F.n_atoms = f.n_atoms();
    F.max_slots = b.max_slots;
    F.max_nodes = b.max_nodes;
    {   // a-priori bounds of the on-grid fp64 accumulation (kernels.hpp FxScale, DevFormula::fx_*)
        std::vector<double> fbool(f.n_bool, 0.0), fatom(f.n_atoms(), 0.0), freal(f.n_real, 0.0), inv(f.n_atoms(), 0.0);
        for (uint32_t i = 0; i < f.n_atoms(); ++i) {
            double n2 = 0.0;
            for (uint32_t t = f.atom_rowptr[i]; t < f.atom_rowptr[i + 1]; ++t) n2 += f.atom_val[t] * f.atom_val[t];
            inv[i] = n2 > 0 ? 1.0 / std::sqrt(n2) : 0.0;
        }
        double sw = 0.0;
        for (size_t c = 0; c < C; ++c) {
            const double w = std::ldexp((double)b.cons_w[c], -P.wexp);
            sw += w;
            const Template& t = b.tmpls[b.cons_tmpl[c]];
            for (size_t sl = 0; sl < t.kinds.size(); ++sl) {
                const uint32_t id = b.slot_ids[b.cons_slot_off[c] + sl];
                if (t.kinds[sl] == 0) {
                    fbool[id] += w;
                } else {
                    fatom[id] += w;
                    for (uint32_t k = f.atom_rowptr[id]; k < f.atom_rowptr[id + 1]; ++k)
                        freal[f.atom_col[k]] += w * std::fabs(f.atom_val[k]) * inv[id] * 0.7978845608028654;
                }
            }
        }
        F.fx_fb = 0.0;
        for (double v : fbool) F.fx_fb = std::max(F.fx_fb, v);
        for (double v : fatom) F.fx_fb = std::max(F.fx_fb, v);
        F.fx_fa = 0.0;
        for (double v : freal) F.fx_fa = std::max(F.fx_fa, v);
        F.fx_sw = sw;
        F.wexp = P.wexp;
    }
#define UP(vec, field) do { s = upload(ctx, vec, F.field, ctx->fallocs); if (s) return s; } while (0)
    UP(c_tmpl, cons_tmpl);
    UP(c_off, cons_slot_off);
    UP(c_ids, slot_ids);
    UP(c_w, cons_w);
    UP(P.order, orig);
    UP(node_off, tmpl_node_off);
    UP(nodes, nodes);
    UP(kind_off, tmpl_kind_off);
    UP(kinds, kinds);
    UP(roots, tmpl_root);
    UP(f.atom_rowptr, atom_rowptr);
    UP(f.atom_col, atom_col);
    UP(aval, atom_val);
    UP(f.atom_val, atom_val64);
    UP(arhs, atom_rhs);
    UP(f.atom_rhs, atom_rhs64);
    UP(f.atom_strict, atom_strict);
    UP(ainv, atom_invnorm);
    UP(b.lo, lo);
    UP(b.hi, hi);
    {   // R33 halfspaces (multi-variable unit atoms), reordered by dependency level: a halfspace's
        // level is one more than the last earlier halfspace sharing a variable, so one level's
        // halfspaces touch disjoint variables and the level-by-level sweep performs exactly the
        // sequential Dykstra sweep of constraint order (k_dykstra)
        const size_t K = b.h_rowptr.size() - 1;
        std::vector<uint8_t> in_h(f.n_real, 0);
        std::vector<uint32_t> hv, lidx(f.n_real, 0);
        for (uint32_t j : b.h_col) in_h[j] = 1;
        for (uint32_t j = 0; j < f.n_real; ++j)
            if (in_h[j]) { lidx[j] = (uint32_t)hv.size(); hv.push_back(j); }
        std::vector<uint32_t> level(K, 0), last(f.n_real, 0);
        uint32_t n_levels = 0;
        for (size_t k = 0; k < K; ++k) {
            uint32_t l = 0;
            for (uint32_t t = b.h_rowptr[k]; t < b.h_rowptr[k + 1]; ++t) l = std::max(l, last[b.h_col[t]]);
            level[k] = l;
            for (uint32_t t = b.h_rowptr[k]; t < b.h_rowptr[k + 1]; ++t) last[b.h_col[t]] = l + 1;
            n_levels = std::max(n_levels, l + 1);
        }
        std::vector<uint32_t> order(K);
        for (size_t k = 0; k < K; ++k) order[k] = (uint32_t)k;
        std::stable_sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) { return level[x] < level[y]; });
        std::vector<uint32_t> rowptr{0}, lcol, loff(n_levels + 1, 0);
        std::vector<float> hg, hh, inv2;
        for (uint32_t k : order) {
            double n2 = 0.0;
            for (uint32_t t = b.h_rowptr[k]; t < b.h_rowptr[k + 1]; ++t) {
                lcol.push_back(lidx[b.h_col[t]]);
                hg.push_back((float)b.h_g[t]);
                n2 += (double)(float)b.h_g[t] * (double)(float)b.h_g[t];
            }
            rowptr.push_back((uint32_t)lcol.size());
            hh.push_back((float)b.h_h[k]);
            inv2.push_back((float)(1.0 / n2));
            ++loff[level[k] + 1];
        }
        for (uint32_t l = 0; l < n_levels; ++l) loff[l + 1] += loff[l];
        F.n_half = (uint32_t)K;
        F.n_hvars = (uint32_t)hv.size();
        F.n_hlevels = n_levels;
        F.h_nnz = (uint32_t)lcol.size();
        UP(rowptr, h_rowptr);
        UP(lcol, h_col);
        UP(hg, h_g);
        UP(hh, h_h);
        UP(inv2, h_inv2);
        UP(hv, hvars);
        UP(in_h, in_h);
        UP(loff, h_level_off);
    }
#undef UP
    s = upload(ctx, P.pos, ctx->d_pos, ctx->fallocs);
    if (s) return s;
    // JIT-specialised sweep for the hot kernel classes (tiles.cpp); on failure everything runs
    // through the generic kernel and the reason is kept in jit_error.
    F.generic_begin = 0;
    ctx->jit_error.clear();
    if (!P.tiles.empty()) {
        std::string err;
        if (jit_compile(ctx->jit_src, ctx->jit, err)) {
            const void* tp = nullptr;
            s = upload_bytes(ctx, P.tiles.data(), P.tiles.size() * sizeof(TileDesc), tp);
            if (s) return s;
            const uint32_t* rp = nullptr;
            s = upload(ctx, P.recs, rp, ctx->fallocs);
            if (s) return s;
            const uint32_t* vp = nullptr;
            s = upload(ctx, P.tile_vars, vp, ctx->fallocs);
            if (s) return s;
            ctx->T.tiles = tp;
            ctx->T.n_tiles = (uint32_t)P.tiles.size();
            ctx->T.recs = rp;
            ctx->T.tile_vars = vp;
            ctx->T.vmax = P.kernel_vmax();
            ctx->T.ring_uint4 = P.ring_uint4();
            ctx->T.vid_bytes = P.vid_bytes();
            ctx->T.cons_per_tile = P.tiles.empty() ? 0u : (uint32_t)(P.jit_cons_end / P.tiles.size());
            // run-variable id slots the tiles actually use (<= Plan::rmax): the sweep's shared memory
            // is sized by it, so more one-warp CTAs fit per SM
            uint32_t rmax_used = 1;
            for (const TileDesc& td : P.tiles) rmax_used = std::max(rmax_used, td.n_vars >> 16);
            ctx->T.rmax = rmax_used;
            const uint32_t* vr = nullptr;
            s = upload(ctx, P.vrecs, vr, ctx->fallocs);
            if (s) return s;
            ctx->T.vrecs = vr;
            F.generic_begin = P.jit_cons_end;
            if (P.has_sym) {
                const uint32_t* sa = nullptr;
                s = upload(ctx, P.sym_atoms, sa, ctx->fallocs);
                if (s) return s;
                ctx->slots = DevSlots{};
                ctx->slots.atoms = sa;
                ctx->slots.n_sa = (uint32_t)P.sym_atoms.size();
                ctx->slots.nv = f.n_bool + f.n_real;
                ctx->has_sym = true;
            }
        } else {
            ctx->jit_error = err;
        }
    }
    F.generic_end = F.n_cons;
    ctx->T_all = ctx->T;
    ctx->vrange[0][0] = 0;
    ctx->vrange[0][1] = F.n_cons;
    ctx->vrange[1][0] = ctx->vrange[1][1] = 0;
    ctx->shard_mode = 0;
    ctx->stage = 2;
    ctx->err.clear();
    return FSMT_OK;
}

fsmt_status fsmt_get_dims(const fsmt_ctx* ctx, fsmt_dims* out) {
    if (!ctx || !out) return FSMT_ERR_ARG;
    if (ctx->stage < 1) return FSMT_ERR_STATE;
    fsmt_dims d{};
    d.n_bool = ctx->f.n_bool;
    d.n_real = ctx->f.n_real;
    d.n_atoms = ctx->f.n_atoms();
    d.n_cons = (uint32_t)ctx->f.cons.size();
    if (ctx->stage >= 2) {
        d.n_templates = (uint32_t)ctx->b.tmpls.size();
        d.max_slots = ctx->b.max_slots;
        d.max_nodes = ctx->b.max_nodes;
        d.n_bounded = ctx->b.n_bounded;
        d.n_nodes = ctx->b.n_nodes;
        d.n_slot_refs = ctx->b.slot_ids.size();
        d.n_halfspaces = (uint32_t)(ctx->b.h_rowptr.size() - 1);
        d.n_slot_rows = ctx->has_sym ? ctx->slots.nv + ctx->slots.n_sa : 0;
    }
    *out = d;
    return FSMT_OK;
}

fsmt_status fsmt_get_bounds(const fsmt_ctx* ctx, float* lo, float* hi) {
    if (!ctx) return FSMT_ERR_ARG;
    if (ctx->stage < 2) return FSMT_ERR_STATE;
    if (lo) std::copy(ctx->b.lo.begin(), ctx->b.lo.end(), lo);
    if (hi) std::copy(ctx->b.hi.begin(), ctx->b.hi.end(), hi);
    return FSMT_OK;
}

fsmt_status fsmt_dump_structure(const fsmt_ctx* cctx, const char* dir) {
    fsmt_ctx* ctx = const_cast<fsmt_ctx*>(cctx);
    if (!ctx || !dir) return FSMT_ERR_ARG;
    if (ctx->stage < 2) return fail(ctx, FSMT_ERR_STATE, "fsmt_dump_structure: build first");
    std::string p1 = std::string(dir) + "/templates.jsonl", p2 = std::string(dir) + "/constraints.bin";
    FILE* fp = fopen(p1.c_str(), "wb");
    if (!fp) return fail(ctx, FSMT_ERR_ARG, "cannot write " + p1);
    std::string t = dump_templates_jsonl(ctx->b);
    fwrite(t.data(), 1, t.size(), fp);
    fclose(fp);
    fp = fopen(p2.c_str(), "wb");
    if (!fp) return fail(ctx, FSMT_ERR_ARG, "cannot write " + p2);
    std::vector<uint8_t> c = dump_constraints_bin(ctx->b);
    fwrite(c.data(), 1, c.size(), fp);
    fclose(fp);
    return FSMT_OK;
}

fsmt_status fsmt_set_params(fsmt_ctx* ctx, const fsmt_params* p) {
    if (!ctx) return FSMT_ERR_ARG;
    if (!p) {
        default_kappas(ctx->kappas);
        ctx->eta = 0.05f;
        ctx->eps = 1e-2f;
        ctx->rounding = FSMT_ROUND_SIGN;
        ctx->n_roundings = 1;
        ctx->erwa_mode = FSMT_ERWA_VERBATIM;
        ctx->eta_mode = 0;
        ctx->F.proj_iters = 0;
        ctx->time_limit = 0;
        return FSMT_OK;
    }
    if (p->kappas) {
        if (p->n_stages == 0) return fail(ctx, FSMT_ERR_ARG, "empty kappa schedule");
        for (uint32_t i = 0; i < p->n_stages; ++i)
            if (!(p->kappas[i] >= 0.f) || !std::isfinite(p->kappas[i])) return fail(ctx, FSMT_ERR_ARG, "kappa must be finite and >= 0");
        ctx->kappas.assign(p->kappas, p->kappas + p->n_stages);
    } else {
        default_kappas(ctx->kappas);
    }
    if (p->rounding > 1 || p->erwa_mode > 1 || p->eta_mode > 3 || p->proj_iters > 100000 || p->n_roundings > 4096)
        return fail(ctx, FSMT_ERR_ARG, "bad rounding / erwa_mode / eta_mode / proj_iters / n_roundings");
    ctx->n_roundings = std::max<uint32_t>(1, p->n_roundings);
    ctx->F.proj_iters = p->proj_iters;
    ctx->eta = p->eta > 0 ? p->eta : 0.05f;
    ctx->eps = p->eps > 0 ? p->eps : 1e-2f;
    ctx->rounding = p->rounding;
    ctx->erwa_mode = p->erwa_mode;
    ctx->eta_mode = p->eta_mode;
    ctx->time_limit = p->time_limit_s;
    return FSMT_OK;
}

fsmt_status fsmt_begin(fsmt_ctx* ctx, uint32_t R, uint64_t seed, uint32_t restart_offset) {
    fsmt_status s = need(ctx, 2, "fsmt_begin");
    if (s) return s;
    if (ctx->host_only) return fail(ctx, FSMT_ERR_CUDA, "fsmt_begin: host-only context has no device");
    if (R == 0) return fail(ctx, FSMT_ERR_ARG, "restarts must be > 0");
    if (ctx->F.proj_iters && ctx->F.n_half && project_smem_bytes(ctx->F, ctx->F.h_nnz) > 227 * 1024)
        return fail(ctx, FSMT_ERR_ARG, "too many multi-variable unit atoms for the on-chip Dykstra projection (R33)");
    cudaSetDevice(ctx->device);
    // the state of a previous begin with the same restart count is reused (no cudaFree / cudaMalloc:
    // they cost 40-50 ms at R = 32, i.e. most of a time-to-SAT run) unless buffers were bound
    const bool reuse = ctx->S.a && ctx->S.R == R && !ctx->ext_bound;
    if (reuse) {
        if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; }
        ctx->rounded = false;
        if (ctx->terms) { cudaFree(ctx->terms); ctx->terms = nullptr; }
    } else {
        drop_state(ctx);
    }
    const DevFormula& F = ctx->F;
    DevState& S = ctx->S;
    S.R = R;
    auto alloc = [&](void** p, size_t bytes) -> fsmt_status {
        cudaError_t e = cudaMalloc(p, std::max<size_t>(bytes, 16));
        if (e != cudaSuccess) return fail(ctx, FSMT_ERR_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
        ctx->sallocs.push_back(*p);
        return FSMT_OK;
    };
    const size_t nb = (size_t)F.n_bool * R, nr = (size_t)F.n_real * R, nc = (size_t)F.n_cons * R;
    if (!reuse) {
        const size_t parts = (size_t)update_parts(F, R);
        // grad_a and grad_b are one allocation ([var][R] over the unified variable id: gb = ga + nb), so
        // a stream row flushes to ga + g*R whatever the variable's kind; U has kUPad spare constraint
        // rows so the sweep's U prefetch may read past the last tile without a bounds test
        if ((s = alloc((void**)&S.a, nb * 4)) || (s = alloc((void**)&S.b, nr * 4)) || (s = alloc((void**)&S.ga, (nb + nr) * 8)) ||
            (s = alloc((void**)&S.U, (nc + (size_t)kUPad * R) * 2)) || (s = alloc((void**)&S.obj, (size_t)R * 8)) ||
            (s = alloc((void**)&S.x, nb)) || (s = alloc((void**)&S.unsat, (size_t)R * 4)) ||
            (s = alloc((void**)&S.frozen, R)) || (s = alloc((void**)&S.gm2, (size_t)R * 8)) ||
            (s = alloc((void**)&S.gm2_part, std::max<size_t>(parts, 1) * R * 8))) {
            drop_state(ctx);
            return s;
        }
        S.gb = S.ga + nb;
        if (ctx->has_sym) {   // slot tables (rows: Booleans, reals (unused), table atoms)
            DevSlots& D = ctx->slots;
            const size_t rows = (size_t)D.nv + D.n_sa;
            if ((s = alloc((void**)&D.PT, rows * R * 4)) ||
                (s = alloc((void**)&D.DD, (size_t)D.n_sa * R * 4)) || (s = alloc((void**)&D.GU, rows * R * 8)) ||
                (s = alloc((void**)&D.TT, rows * R))) {
                drop_state(ctx);
                return s;
            }
        }
        if ((s = alloc((void**)&S.x_best, nb)) || (s = alloc((void**)&S.unsat_m, (size_t)R * 4)) ||
            (s = alloc((void**)&S.unsat_best, (size_t)R * 4)) || (s = alloc((void**)&S.better, R)) ||
            (s = alloc((void**)&S.umax, (size_t)R * 4)) || (s = alloc((void**)&S.fx, (size_t)R * sizeof(FxScale))) ||
            (s = alloc((void**)&S.gsc, (size_t)R * 8)) || (s = alloc((void**)&S.flags, 16)) ||
            (s = alloc((void**)&ctx->scratch, (size_t)std::max(F.n_bool, F.n_real) * R * 8))) {
            drop_state(ctx);
            return s;
        }
        S.bn = nullptr;
        if (F.n_half) {   // R33: the candidate b of the projected step
            if ((s = alloc((void**)&S.bn, nr * 4))) {
                drop_state(ctx);
                return s;
            }
        }
    }
    CK(cudaMemsetAsync(S.U, 0, (nc + (size_t)kUPad * R) * 2, ctx->stream));
    CK(cudaMemsetAsync(S.umax, 0, (size_t)R * 4, ctx->stream));
    CK(cudaMemsetAsync(S.flags, 0, 16, ctx->stream));
    CK(cudaMemsetAsync(S.frozen, 0, R, ctx->stream));
    CK(cudaMemsetAsync(S.ga, 0, nb * 8, ctx->stream));
    CK(cudaMemsetAsync(S.gb, 0, nr * 8, ctx->stream));
    CK(cudaMemsetAsync(S.obj, 0, (size_t)R * 8, ctx->stream));
    launch_init(F, S, seed, restart_offset, ctx->stream);
    launch_project(F, S, S.b, false, ctx->stream);     // R33: init is projected like every step
    ctx->launches += 1 + (F.proj_iters && F.n_half ? 1 : 0);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->seed = seed;
    ctx->restart_offset = restart_offset;
    ctx->stage = 3;
    return FSMT_OK;
}

fsmt_status fsmt_set_state(fsmt_ctx* ctx, const float* a, const float* b, int where) {
    fsmt_status s = need(ctx, 3, "fsmt_set_state");
    if (s) return s;
    if ((s = copy_in(ctx, ctx->S.a, a, (size_t)ctx->F.n_bool * ctx->S.R, where))) return s;
    return copy_in(ctx, ctx->S.b, b, (size_t)ctx->F.n_real * ctx->S.R, where);
}

fsmt_status fsmt_get_state(fsmt_ctx* ctx, float* a, float* b, int where) {
    fsmt_status s = need(ctx, 3, "fsmt_get_state");
    if (s) return s;
    if ((s = copy_out(ctx, a, ctx->S.a, (size_t)ctx->F.n_bool * ctx->S.R, where))) return s;
    return copy_out(ctx, b, ctx->S.b, (size_t)ctx->F.n_real * ctx->S.R, where);
}

// U is kept in the internal constraint order; the ABI speaks the original order.
fsmt_status fsmt_set_counters(fsmt_ctx* ctx, const uint16_t* U, int where) {
    fsmt_status s = need(ctx, 3, "fsmt_set_counters");
    if (s) return s;
    const size_t n = (size_t)ctx->F.n_cons * ctx->S.R;
    if (n == 0) return FSMT_OK;
    if (!U) return fail(ctx, FSMT_ERR_ARG, "null input pointer");
    uint16_t* tmp = nullptr;
    CK(cudaMalloc((void**)&tmp, n * 2));
    cudaError_t e = cudaMemcpyAsync(tmp, U, n * 2, where == FSMT_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                    ctx->stream);
    if (e == cudaSuccess) {
        launch_gather_rows_u16(ctx->S.U, tmp, ctx->F.orig, ctx->F.n_cons, ctx->S.R, ctx->stream);
        launch_umax(ctx->F, ctx->S, ctx->stream);      // the weight shift follows the new counters
        ctx->launches += 2;
        e = cudaStreamSynchronize(ctx->stream);
    }
    cudaFree(tmp);
    if (e != cudaSuccess) return fail(ctx, FSMT_ERR_CUDA, std::string("fsmt_set_counters: ") + cudaGetErrorString(e));
    return check_launch(ctx);
}

fsmt_status fsmt_get_counters(fsmt_ctx* ctx, uint16_t* U, int where) {
    fsmt_status s = need(ctx, 3, "fsmt_get_counters");
    if (s) return s;
    const size_t n = (size_t)ctx->F.n_cons * ctx->S.R;
    if (n == 0 || !U) return FSMT_OK;
    uint16_t* tmp = nullptr;
    CK(cudaMalloc((void**)&tmp, n * 2));
    launch_gather_rows_u16(tmp, ctx->S.U, ctx->d_pos, ctx->F.n_cons, ctx->S.R, ctx->stream);
    ctx->launches += 1;
    cudaError_t e = cudaMemcpyAsync(U, tmp, n * 2, where == FSMT_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                    ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    cudaFree(tmp);
    if (e != cudaSuccess) return fail(ctx, FSMT_ERR_CUDA, std::string("fsmt_get_counters: ") + cudaGetErrorString(e));
    return check_launch(ctx);
}

fsmt_status fsmt_jit_info(const fsmt_ctx* ctx, uint32_t* n_jit_classes, uint32_t* n_tiles, uint32_t* jit_cons,
                          char* msg, size_t msg_len) {
    if (!ctx) return FSMT_ERR_ARG;
    if (ctx->stage < 2) return FSMT_ERR_STATE;
    const bool active = !ctx->host_only && ctx->T.n_tiles > 0;
    if (n_jit_classes) *n_jit_classes = ctx->plan.n_jit_kclasses;
    if (n_tiles) *n_tiles = (uint32_t)ctx->plan.tiles.size();
    if (jit_cons) *jit_cons = active ? ctx->plan.jit_cons_end : 0;
    if (msg && msg_len) {
        std::string m = ctx->host_only ? "host-only" : (active ? "active" : (ctx->plan.tiles.empty() ? "no JIT classes" : ctx->jit_error));
        if (active && ctx->jit_r.kernel)
        {
            m += "; prepared R=" + std::to_string(ctx->jit_r_R) + " k1 cap=" + std::to_string(ctx->jit_r_cap) + " class caps=";
            for (size_t k = 0; k < ctx->jit_r_caps.size(); ++k) m += (k ? "," : "") + std::to_string(ctx->jit_r_caps[k]);
        }
        snprintf(msg, msg_len, "%s", m.c_str());
    }
    return FSMT_OK;
}

static std::string prepared_source_tuned(const fsmt_ctx* ctx, uint32_t R, int* cap);

fsmt_status fsmt_jit_check(fsmt_ctx* ctx, size_t* cubin_bytes, char* log, size_t log_len) {
    if (!ctx) return FSMT_ERR_ARG;
    if (ctx->stage < 2) return fail(ctx, FSMT_ERR_STATE, "fsmt_jit_check: build first");
    if (ctx->jit_src.empty()) return fail(ctx, FSMT_ERR_STATE, "fsmt_jit_check: no JIT classes");
    std::vector<char> cubin;
    std::string lg, err;
    // FSMT_JIT_CHECK_RC=R: check the module fsmt_prepare(R) would build (register counts)
    std::string src = ctx->jit_src;
    if (const char* rc = getenv("FSMT_JIT_CHECK_RC")) src = prepared_source_tuned(ctx, (uint32_t)atoi(rc), nullptr);
    bool ok = jit_cubin(src, cubin, lg, err);
    if (log && log_len) snprintf(log, log_len, "%s", lg.c_str());
    if (!ok) return fail(ctx, FSMT_ERR_CUDA, err);
    if (cubin_bytes) *cubin_bytes = cubin.size();
    return FSMT_OK;
}

// The source fsmt_prepare(R) compiles: the restart count as a constant (FSMT_RC); U loaded 3
// constraints ahead when U[c][r] exceeds ~1.5x the 126 MB L2 and so comes from HBM every sweep
// (cfg4 9.78 -> 8.85 ms), else 2 ahead.
static std::string prepared_source(const fsmt_ctx* ctx, uint32_t R, int min_ctas, const std::vector<int>* caps = nullptr) {
    // (v25: also for an L2-resident U -- its ~600-cycle L2 latency was cfg3's top stall: cfg3 K1
    // 0.694 -> 0.637 ms with 2 ahead)
    const int upf = (double)ctx->plan.jit_cons_end * R > 192e6 ? 3 : 2;
    std::vector<int> all(ctx->plan.n_jit_kclasses, min_ctas);
    const std::string src = (upf || min_ctas || caps) ? jit_source(ctx->f, ctx->b, ctx->plan, upf, min_ctas, caps ? caps : &all)
                                                       : ctx->jit_src;
    return "#define FSMT_RC " + std::to_string(R) + "u\n" + src;
}

// spill-store bytes ptxas reports for one kernel of an NVRTC log (-1 if not found)
static long spill_stores(const std::string& log, const std::string& kernel) {
    const std::string key = "Function properties for " + kernel + "\n";
    const size_t at = log.find(key);
    if (at == std::string::npos) return -1;
    const size_t sp = log.find(" bytes spill stores", at + key.size());
    if (sp == std::string::npos) return -1;
    size_t b = sp;
    while (b > 0 && isdigit((unsigned char)log[b - 1])) --b;
    return atol(log.substr(b, sp - b).c_str());
}

// The prepared module's source with the hot kernel's register cap: the highest residency (32,
// then 28 one-warp CTAs per SM: 64 / 72 registers) whose compile has no spills, else no cap
// (cfg3 best at 64, cfg4 at 72, cfg2 uncapped)
static std::string prepared_source_tuned(const fsmt_ctx* ctx, uint32_t R, int* cap) {
    for (int mc : {32, 28, 24, 20}) {
        const std::string src = prepared_source(ctx, R, mc);
        std::vector<char> cubin;
        std::string log, err;
        if (jit_cubin(src, cubin, log, err) && spill_stores(log, "fsmt_k1_jit") == 0) {
            if (cap) *cap = mc;
            return src;
        }
    }
    if (cap) *cap = 0;
    return prepared_source(ctx, R, 0);
}

fsmt_status fsmt_prepare(fsmt_ctx* ctx, uint32_t R) {
    fsmt_status s = need(ctx, 2, "fsmt_prepare");
    if (s) return s;
    if (R == 0 || !ctx->jit.kernel || ctx->host_only) {
        if (!ctx->host_only) cudaStreamSynchronize(ctx->stream);
        if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; }
        jit_release(ctx->jit_r);
        ctx->jit_r_R = 0;
        return FSMT_OK;
    }
    if (ctx->jit_r.kernel && ctx->jit_r_R == R) return FSMT_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);   // the previous copy may still be in flight
    if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; }   // may hold its kernels
    jit_release(ctx->jit_r);
    ctx->jit_r_R = 0;
    // register cap of the hot sweep: the highest residency (32, then 28 one-warp CTAs per SM:
    // 64 / 72 registers) whose kernel needs no local memory (no spills), else none (DESIGN.md
    // §7 item 13) -- chosen for the all-class kernel and for each per-class kernel fsmt_k1_c<k>
    // separately (§7 item 17).  Judged from the loaded kernels' attributes, not the compiler log.
    const uint32_t nk = ctx->plan.n_jit_kclasses;
    int cap = 0;
    bool cap_found = false;
    std::vector<int> caps(nk, 0);
    std::vector<char> found(nk, 0);
    std::string err;
    // (the last candidate, 12 CTAs = 168 registers, is for the very wide symmetric classes: taken when
    // it needs at most 64 bytes of local memory -- the random family's count-CARD(50) class, 186 registers uncapped:
    // 10,000 points at n = 1,000 2.40 -> 2.02 ms)
    auto spills = [](cudaKernel_t k, size_t tol) {
        cudaFuncAttributes fa{};
        return cudaFuncGetAttributes(&fa, (const void*)k) != cudaSuccess || fa.localSizeBytes > tol;
    };
    auto regs = [](cudaKernel_t k) {
        cudaFuncAttributes fa{};
        return cudaFuncGetAttributes(&fa, (const void*)k) == cudaSuccess ? fa.numRegs : 0;
    };
    std::vector<int> free_regs(nk, 0);   // registers of the uncapped per-class kernels (filled lazily)
    for (int mc : {32, 28, 24, 20, 12}) {
        const size_t tol = mc == 12 ? 64 : 0;
        JitKernel cand;
        if (!jit_compile(prepared_source(ctx, R, mc), cand, err)) continue;
        if (!cap_found && mc != 12 && !spills(cand.kernel, 0)) {
            cap = mc;
            cap_found = true;
        }
        for (uint32_t k = 0; k < nk && k < cand.kclass.size(); ++k)
            if (!found[k] && !spills(cand.kclass[k], tol) && (mc != 12 || regs(cand.kclass[k]) > 0)) {
                if (mc == 12) {   // only where it binds: the uncapped kernel needs more than 168 registers
                    if (!free_regs[k]) {
                        std::vector<int> none(nk, 0);
                        JitKernel un;
                        if (jit_compile(prepared_source(ctx, R, 0, &none), un, err)) {
                            for (uint32_t j = 0; j < nk && j < un.kclass.size(); ++j) free_regs[j] = regs(un.kclass[j]);
                            jit_release(un);
                        }
                    }
                    if (free_regs[k] <= 168) continue;
                }
                caps[k] = mc;
                found[k] = 1;
            }
        jit_release(cand);
    }
    if (!jit_compile(prepared_source(ctx, R, cap, &caps), ctx->jit_r, err)) return fail(ctx, FSMT_ERR_CUDA, "fsmt_prepare: " + err);
    ctx->jit_r_cap = cap;
    ctx->jit_r_caps = caps;
    ctx->jit_r_R = R;
    return FSMT_OK;
}

size_t fsmt_jit_source(const fsmt_ctx* ctx, char* buf, size_t len) {
    if (!ctx || ctx->stage < 2) return 0;
    std::string src = ctx->jit_src;
    if (const char* rc = getenv("FSMT_JIT_CHECK_RC"))   // the source fsmt_prepare(R) would compile
        if (!src.empty()) src = prepared_source_tuned(ctx, (uint32_t)atoi(rc), nullptr);
    if (buf && len) snprintf(buf, len, "%s", src.c_str());
    return src.size() + 1;
}

// the JIT module for a launch over R restarts: the R-specialised copy when fsmt_prepare(R)
// built one, else the generic module
static const JitKernel& jk(const fsmt_ctx* ctx, uint32_t R) {
    return (ctx->jit_r.kernel && ctx->jit_r_R == R) ? ctx->jit_r : ctx->jit;
}

static fsmt_status sweep_impl(fsmt_ctx* ctx, float kappa, uint32_t stage_t, double* terms, uint32_t terms_r) {
    const DevFormula& F = ctx->F;
    const DevState& S = ctx->S;
    const int et = et_int_of(stage_t, ctx->erwa_mode);
    {
        Timed tm(ctx, 0);
        const float ws = wfrac_of(stage_t, ctx->erwa_mode);
        const bool sym = ctx->has_sym && ctx->T.n_tiles;
        // zero grad_a / grad_b / obj (+ the slot-table gradients) and write the per-restart scales
        launch_prologue(F, S, kappa, et, ws, ctx->has_sym ? ctx->slots.GU : nullptr,
                        ctx->has_sym ? (uint64_t)ctx->slots.nv + ctx->slots.n_sa : 0, ctx->stream);
        ctx->launches += 1;
        if (sym) {   // shared slot probabilities for the symmetric classes
            launch_slot_prob(jk(ctx, S.R).kprob, F, S, ctx->slots, kappa, ctx->stream);
            ctx->launches += 1;
        }
        if (ctx->T.n_tiles) {
            const JitKernel& J = jk(ctx, S.R);
            const bool dbg = S.U == nullptr || terms != nullptr;
            const char* pc = getenv("FSMT_JIT_PERCLASS");
            const std::vector<uint32_t>& cb = ctx->plan.class_tile_begin;
            if (!dbg && !(pc && pc[0] == '0') && J.kclass.size() == ctx->plan.n_jit_kclasses && cb.size() == J.kclass.size() + 1) {
                // classes that gain from their own register allocation launch their own kernel; runs of
                // the others share one all-class launch (DESIGN.md §7 item 17); the launches run
                // concurrently on the auxiliary streams (their atomics add exact grid units)
                const uint32_t lo = ctx->T.first, hi = ctx->T.first + ctx->T.n_tiles;
                std::vector<std::pair<cudaKernel_t, std::pair<uint32_t, uint32_t>>> L;
                for (size_t k = 0; k < J.kclass.size(); ++k) {
                    const uint32_t b0 = std::max(lo, cb[k]), b1 = std::min(hi, cb[k + 1]);
                    if (b1 <= b0) continue;
                    const cudaKernel_t kk = J.kclass_sep[k] ? J.kclass[k] : J.kernel;
                    if (!L.empty() && kk == J.kernel && L.back().first == J.kernel && L.back().second.second == b0)
                        L.back().second.second = b1;
                    else
                        L.push_back({kk, {b0, b1}});
                }
                const bool fork = L.size() > 1;
                if (fork) CK(cudaEventRecord(ctx->ev_fork, ctx->stream));
                for (size_t i = 0; i < L.size(); ++i) {
                    const uint32_t b0 = L[i].second.first, b1 = L[i].second.second;
                    DevTiles Tk = ctx->T;
                    Tk.tiles = (const char*)ctx->T.tiles + (size_t)(b0 - lo) * sizeof(TileDesc);
                    Tk.n_tiles = b1 - b0;
                    Tk.first = b0;
                    cudaStream_t st = fork ? ctx->aux[i % fsmt_ctx::kAux] : ctx->stream;
                    if (fork && i < fsmt_ctx::kAux) CK(cudaStreamWaitEvent(st, ctx->ev_fork, 0));
                    launch_sweep_jit(L[i].first, F, S, Tk, kappa, terms, terms_r, st, &ctx->slots);
                    ctx->launches += 1;
                }
                if (fork)
                    for (size_t i = 0; i < std::min(L.size(), (size_t)fsmt_ctx::kAux); ++i) {
                        CK(cudaEventRecord(ctx->ev_join[i], ctx->aux[i]));
                        CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_join[i], 0));
                    }
            } else {
                launch_sweep_jit(dbg ? J.kernel_dbg : J.kernel, F, S, ctx->T, kappa, terms, terms_r, ctx->stream, &ctx->slots);
                ctx->launches += 1;
            }
        }
        if (F.generic_begin < F.generic_end) {
            launch_sweep(F, S, kappa, terms, terms_r, ctx->stream);
            ctx->launches += 1;
        }
        // constraint-sharded: the rows are partial; the chain waits for their all-reduce
        if (ctx->has_sym && !(ctx->shard_mode == 1 && ctx->shard_world > 1)) {
            launch_slot_chain(jk(ctx, S.R).kchain, F, S, ctx->slots, ctx->stream);
            ctx->launches += 1;
        }
    }
    return check_launch(ctx);
}

static fsmt_status update_impl(fsmt_ctx* ctx, float eta, float eps, float eta_b = 0.f) {
    {
        Timed tm(ctx, 1);
        launch_update(ctx->F, ctx->S, eta, eps, ctx->stream, eta_b);
    }
    ctx->launches += 3 + (ctx->F.proj_iters && ctx->F.n_half && ctx->S.bn ? 2 : 0);
    return check_launch(ctx);
}

// K5 over this context's constraints for the rounded model in S2.x (unsat into S2.unsat)
static void verify_rounded(fsmt_ctx* ctx, const DevState& S2, uint16_t* U_update) {
    if (ctx->T.n_tiles && ctx->jit.kernel5) {    // specialised check of this context's tiles
        if (ctx->has_sym) {
            launch_slot_truth(jk(ctx, S2.R).ktruth, ctx->F, S2, ctx->slots, S2.x, S2.b, ctx->stream);
            ctx->launches += 1;
        }
        launch_verify_jit(jk(ctx, S2.R).kernel5, ctx->F, S2, ctx->T, S2.x, S2.b, U_update, nullptr, ctx->stream, ctx->slots.TT);
        launch_verify(ctx->F, S2, S2.x, S2.b, U_update, nullptr, ctx->stream, ctx->F.generic_begin, ctx->F.generic_end);
        ctx->launches += 2;
    } else {
        for (int k = 0; k < 2; ++k)             // the constraint ranges this context owns
            if (ctx->vrange[k][1] > ctx->vrange[k][0]) {
                launch_verify(ctx->F, S2, S2.x, S2.b, U_update, nullptr, ctx->stream, ctx->vrange[k][0], ctx->vrange[k][1]);
                ctx->launches += 1;
            }
    }
}

static fsmt_status stage_end_impl(fsmt_ctx* ctx, uint32_t stage_t) {
    const DevState& S = ctx->S;
    const uint32_t M = ctx->rounding == FSMT_ROUND_PHILOX ? ctx->n_roundings : 1;
    if (M > 1 && ctx->shard_mode != 0)
        return fail(ctx, FSMT_ERR_STATE, "n_roundings > 1 needs the unsharded mode (the choice needs global counts)");
    {
        Timed tm(ctx, 2);
        if (M > 1) {   // R34: M draws of R(a), keep the one with the fewest violations per restart
            DevState S2 = S;
            S2.unsat = S.unsat_m;
            for (uint32_t m = 0; m < M; ++m) {
                CK(cudaMemsetAsync(S.unsat_m, 0, (size_t)S.R * 4, ctx->stream));
                launch_round(ctx->F, S, ctx->rounding, ctx->seed, ctx->restart_offset, stage_t + (m << 16), ctx->stream);
                verify_rounded(ctx, S2, nullptr);
                launch_keep_best(ctx->F, S, S.unsat_m, S.unsat_best, S.x_best, S.better, m, ctx->stream);
                ctx->launches += 3;
            }
            CK(cudaMemcpyAsync(S.x, S.x_best, (size_t)ctx->F.n_bool * S.R, cudaMemcpyDeviceToDevice, ctx->stream));
        } else {
            launch_round(ctx->F, S, ctx->rounding, ctx->seed, ctx->restart_offset, stage_t, ctx->stream);
            ctx->launches += 1;
        }
        CK(cudaMemsetAsync(S.unsat, 0, (size_t)S.R * 4, ctx->stream));
        verify_rounded(ctx, S, S.U);
        if (!S.ds) CK(cudaMemcpyAsync(ctx->hflags, S.flags, 4, cudaMemcpyDeviceToHost, ctx->stream));   // read after the sync
    }
    CK(cudaMemsetAsync(S.frozen, 0, S.R, ctx->stream));
    fsmt_status s = check_launch(ctx);
    if (s) return s;
    ctx->rounded = true;
    return FSMT_OK;
}

fsmt_status fsmt_sweep(fsmt_ctx* ctx, float kappa, uint32_t stage_t) {
    fsmt_status s = need(ctx, 3, "fsmt_sweep");
    if (s) return s;
    if (!(kappa >= 0.f) || !std::isfinite(kappa)) return fail(ctx, FSMT_ERR_ARG, "kappa must be finite and >= 0");
    if (stage_t == 0) stage_t = 1;
    return sweep_impl(ctx, kappa, stage_t, nullptr, 0);
}

fsmt_status fsmt_sweep_finish(fsmt_ctx* ctx) {
    fsmt_status s = need(ctx, 3, "fsmt_sweep_finish");
    if (s) return s;
    if (ctx->has_sym && ctx->shard_mode == 1 && ctx->shard_world > 1) {
        launch_slot_chain(jk(ctx, ctx->S.R).kchain, ctx->F, ctx->S, ctx->slots, ctx->stream);
        ctx->launches += 1;
    }
    return check_launch(ctx);
}

fsmt_status fsmt_bind_slot_grads(fsmt_ctx* ctx, void* gu) {
    fsmt_status s = need(ctx, 3, "fsmt_bind_slot_grads");
    if (s) return s;
    if (!ctx->has_sym) return gu ? fail(ctx, FSMT_ERR_ARG, "fsmt_bind_slot_grads: no slot-table rows") : FSMT_OK;
    cudaPointerAttributes at{};
    if (gu && (cudaPointerGetAttributes(&at, gu) != cudaSuccess || at.type != cudaMemoryTypeDevice)) {
        cudaGetLastError();
        return fail(ctx, FSMT_ERR_ARG, "fsmt_bind_slot_grads: device memory only");
    }
    if (gu) {
        ctx->slots.GU = (double*)gu;
        ctx->ext_bound = true;
    }
    return FSMT_OK;
}

fsmt_status fsmt_get_sweep(fsmt_ctx* ctx, double* ga, double* gb, double* obj, int where) {
    fsmt_status s = need(ctx, 3, "fsmt_get_sweep");
    if (s) return s;
    const DevState& S = ctx->S;
    // the sweep leaves the gradients in grid units (kernels.hpp FxScale): scale them by gsc[r]
    auto grad_out = [&](double* dst, const double* src, uint32_t rows) -> fsmt_status {
        if (!dst || rows == 0) return FSMT_OK;
        double* to = where == FSMT_DEVICE ? dst : ctx->scratch;
        launch_scale_rows(to, src, S.gsc, rows, S.R, ctx->stream);
        ctx->launches += 1;
        if (where == FSMT_DEVICE) {
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(ctx->stream));
            return FSMT_OK;
        }
        return copy_out(ctx, dst, (const double*)ctx->scratch, (size_t)rows * S.R, FSMT_HOST);
    };
    if ((s = grad_out(ga, S.ga, ctx->F.n_bool))) return s;
    if ((s = grad_out(gb, S.gb, ctx->F.n_real))) return s;
    if ((s = copy_out(ctx, obj, S.obj, (size_t)S.R, where))) return s;
    CK(cudaMemcpy(ctx->hflags, S.flags, 4, cudaMemcpyDeviceToHost));    // a sweep past the fp64 weight range
    return check_flags(ctx);
}

fsmt_status fsmt_eval(fsmt_ctx* ctx, uint32_t R, const float* a, const float* b, float kappa, const uint16_t* U,
                      uint32_t stage_t, double* obj, double* grad_a, double* grad_b, int where) {
    fsmt_status s = need(ctx, 2, "fsmt_eval");
    if (s) return s;
    if (R == 0 || !a || !b) return fail(ctx, FSMT_ERR_ARG, "fsmt_eval: R > 0 and the point a, b are required");
    if (ctx->stage < 3 || ctx->S.R != R) {
        if ((s = fsmt_begin(ctx, R, 0, 0))) return s;
    } else if (!U) {
        CK(cudaMemsetAsync(ctx->S.U, 0, (size_t)ctx->F.n_cons * R * 2, ctx->stream));
        CK(cudaMemsetAsync(ctx->S.umax, 0, (size_t)R * 4, ctx->stream));
    }
    if ((s = fsmt_set_state(ctx, a, b, where))) return s;
    if (U && (s = fsmt_set_counters(ctx, U, where))) return s;
    if ((s = fsmt_sweep(ctx, kappa, stage_t))) return s;
    return fsmt_get_sweep(ctx, grad_a, grad_b, obj, where);
}

fsmt_status fsmt_constraint_terms(fsmt_ctx* ctx, float kappa, uint32_t restart, double* E) {
    fsmt_status s = need(ctx, 3, "fsmt_constraint_terms");
    if (s) return s;
    if (restart >= ctx->S.R || !E) return fail(ctx, FSMT_ERR_ARG, "bad restart / output");
    if (!ctx->terms) CK(cudaMalloc((void**)&ctx->terms, std::max<size_t>((size_t)ctx->F.n_cons * 8, 8)));
    if ((s = sweep_impl(ctx, kappa, 1, ctx->terms, restart))) return s;
    return copy_out(ctx, E, ctx->terms, ctx->F.n_cons, FSMT_HOST);
}

fsmt_status fsmt_update(fsmt_ctx* ctx, float eta, float eta_b, float eps, double* gm2_out) {
    fsmt_status s = need(ctx, 3, "fsmt_update");
    if (s) return s;
    if (!(eta > 0.f) || !(eps >= 0.f)) return fail(ctx, FSMT_ERR_ARG, "eta must be > 0 and eps >= 0");
    if ((s = update_impl(ctx, eta, eps, eta_b > 0.f ? eta_b : eta))) return s;
    if (gm2_out) return copy_out(ctx, gm2_out, ctx->S.gm2, ctx->S.R, FSMT_HOST);
    return FSMT_OK;
}

fsmt_status fsmt_stage_end(fsmt_ctx* ctx, uint32_t stage_t, uint32_t* unsat_out) {
    fsmt_status s = need(ctx, 3, "fsmt_stage_end");
    if (s) return s;
    if (stage_t == 0) stage_t = 1;
    if ((s = stage_end_impl(ctx, stage_t))) return s;
    if (unsat_out) {
        if ((s = copy_out(ctx, unsat_out, ctx->S.unsat, ctx->S.R, FSMT_HOST))) return s;
    } else {
        CK(cudaStreamSynchronize(ctx->stream));
    }
    return check_flags(ctx);
}

fsmt_status fsmt_shard(fsmt_ctx* ctx, uint32_t rank, uint32_t world, uint32_t mode) {
    fsmt_status s = need(ctx, 2, "fsmt_shard");
    if (s) return s;
    if (ctx->host_only) return fail(ctx, FSMT_ERR_CUDA, "fsmt_shard: host-only context has no device");
    if (world == 0 || rank >= world || mode > 1) return fail(ctx, FSMT_ERR_ARG, "bad rank / world / mode");
    const Plan& P = ctx->plan;
    DevFormula& F = ctx->F;
    const uint32_t C = F.n_cons;
    const uint32_t jit_end = ctx->T_all.n_tiles ? P.jit_cons_end : 0;
    ctx->shard_mode = mode;
    ctx->shard_rank = rank;
    ctx->shard_world = world;
    if (mode == 0 || world == 1) {         // restart sharding: every constraint here
        ctx->T = ctx->T_all;
        F.generic_begin = jit_end;
        F.generic_end = C;
        ctx->vrange[0][0] = 0;
        ctx->vrange[0][1] = C;
        ctx->vrange[1][0] = ctx->vrange[1][1] = 0;
        return FSMT_OK;
    }
    // constraint sharding: contiguous tile range balanced by constraint count,
    // plus an even split of the generic tail
    const uint32_t nt = ctx->T_all.n_tiles;
    uint32_t t0 = 0, t1 = 0;
    if (nt) {
        const uint64_t lo_target = (uint64_t)jit_end * rank / world, hi_target = (uint64_t)jit_end * (rank + 1) / world;
        uint64_t acc = 0;
        t0 = nt;
        t1 = nt;
        for (uint32_t t = 0; t < nt; ++t) {
            if (acc >= lo_target && t0 == nt) t0 = t;
            if (acc >= hi_target) {
                t1 = t;
                break;
            }
            acc += P.tiles[t].n_cons;
        }
        if (t0 > t1) t0 = t1;
    }
    ctx->T = ctx->T_all;
    ctx->T.tiles = (const char*)ctx->T_all.tiles + (size_t)t0 * sizeof(TileDesc);
    ctx->T.first = t0;
    ctx->T.n_tiles = t1 - t0;
    const uint32_t gn = C - jit_end;
    // split on the generic sweep's 16-constraint chunk boundaries (kernels.cu kChunk): each chunk's
    // objective partial is then the unsharded one, so the shards' sums are bit-identical
    auto cut = [&](uint32_t k) { return std::min<uint32_t>(gn, (uint32_t)(((uint64_t)gn * k / world + 15) / 16 * 16)); };
    F.generic_begin = jit_end + cut(rank);
    F.generic_end = jit_end + cut(rank + 1);
    if (t1 > t0) {
        ctx->vrange[0][0] = P.tiles[t0].cons_begin;
        ctx->vrange[0][1] = P.tiles[t1 - 1].cons_begin + P.tiles[t1 - 1].n_cons;
    } else {
        ctx->vrange[0][0] = ctx->vrange[0][1] = 0;
    }
    ctx->vrange[1][0] = F.generic_begin;
    ctx->vrange[1][1] = F.generic_end;
    return FSMT_OK;
}

fsmt_status fsmt_bind_buffers(fsmt_ctx* ctx, void* grad_a, void* grad_b, void* obj, void* unsat, void* umax) {
    fsmt_status s = need(ctx, 3, "fsmt_bind_buffers");
    if (s) return s;
    for (void* p : {grad_a, grad_b, obj, unsat, umax}) {   // device memory only (the kernels write them)
        cudaPointerAttributes at{};
        if (p && (cudaPointerGetAttributes(&at, p) != cudaSuccess || at.type != cudaMemoryTypeDevice)) {
            cudaGetLastError();
            return fail(ctx, FSMT_ERR_ARG, "fsmt_bind_buffers: buffers must be device memory");
        }
    }
    if (umax && ctx->S.umax) CK(cudaMemcpyAsync(umax, ctx->S.umax, (size_t)ctx->S.R * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    if (grad_a || grad_b || obj || unsat || umax) ctx->ext_bound = true;
    if (grad_a) ctx->S.ga = (double*)grad_a;
    if (grad_b) ctx->S.gb = (double*)grad_b;
    if (obj) ctx->S.obj = (double*)obj;
    if (unsat) ctx->S.unsat = (uint32_t*)unsat;
    if (umax) ctx->S.umax = (uint32_t*)umax;
    CK(cudaStreamSynchronize(ctx->stream));
    return FSMT_OK;
}

fsmt_status fsmt_mc_allreduce_f64(fsmt_ctx* ctx, void* mc_ptr, uint64_t n, uint32_t rank, uint32_t world) {
    if (!ctx) return FSMT_ERR_ARG;
    if (ctx->host_only) return fail(ctx, FSMT_ERR_CUDA, "fsmt_mc_allreduce_f64: host-only context has no device");
    if (!mc_ptr || world == 0 || rank >= world) return fail(ctx, FSMT_ERR_ARG, "fsmt_mc_allreduce_f64: null multicast pointer or bad rank");
    if (n == 0) return FSMT_OK;
    cudaSetDevice(ctx->device);
    launch_mc_allreduce_f64((double*)mc_ptr, n, rank, world, ctx->stream);
    ctx->launches += 1;
    return check_launch(ctx);
}

fsmt_status fsmt_run_stage(fsmt_ctx* ctx, uint32_t stage_t, float kappa, uint32_t steps, uint32_t* unsat_out,
                           uint32_t* min_unsat) {
    fsmt_status s = need(ctx, 3, "fsmt_run_stage");
    if (s) return s;
    if (!(kappa >= 0.f) || !std::isfinite(kappa)) return fail(ctx, FSMT_ERR_ARG, "kappa must be finite and >= 0");
    if (stage_t == 0) stage_t = 1;
    if (ctx->shard_mode == 1 && ctx->shard_world > 1)
        return fail(ctx, FSMT_ERR_STATE, "fsmt_run_stage: constraint-sharded contexts need the caller's all-reduce per step "
                                         "(use fsmt_sweep / fsmt_update / fsmt_stage_end)");
    CK(cudaMemsetAsync(ctx->S.frozen, 0, ctx->S.R, ctx->stream));
    float eta_t = 0.f, eta_b = 0.f;
    fsmt_step_sizes(ctx, kappa, &eta_t, &eta_b);
    // FSMT_GRAPH=1: the S PGD steps are captured into one CUDA graph (one graph launch instead of
    // ~5 S kernel launches); the executable graph is kept and updated in place with the next
    // stage's parameters.  Opt-in: capture + update cost about what the launches cost on the
    // configs measured; never with per-kernel timing (events).
    const char* ge = getenv("FSMT_GRAPH");
    if (ge && ge[0] == '1' && !ctx->timing && steps >= 2) {
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        fsmt_status s2 = FSMT_OK;
        for (uint32_t k = 0; k < steps && !s2; ++k) {
            s2 = sweep_impl(ctx, kappa, stage_t, nullptr, 0);
            if (!s2) s2 = update_impl(ctx, eta_t, ctx->eps, eta_b);
        }
        const cudaError_t ee = cudaStreamEndCapture(ctx->stream, &g);
        if (s2 || ee != cudaSuccess) {
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            if (s2) return s2;
            CK(ee);
        }
        if (ctx->gexec) {
            cudaGraphExecUpdateResultInfo info;
            if (cudaGraphExecUpdate(ctx->gexec, g, &info) != cudaSuccess) {
                cudaGetLastError();
                cudaGraphExecDestroy(ctx->gexec);
                ctx->gexec = nullptr;
            }
        }
        cudaError_t ei = cudaSuccess;
        if (!ctx->gexec) ei = cudaGraphInstantiate(&ctx->gexec, g, 0);
        cudaGraphDestroy(g);
        CK(ei);
        CK(cudaGraphLaunch(ctx->gexec, ctx->stream));
    } else {
        for (uint32_t k = 0; k < steps; ++k) {
            if ((s = sweep_impl(ctx, kappa, stage_t, nullptr, 0))) return s;
            if ((s = update_impl(ctx, eta_t, ctx->eps, eta_b))) return s;
        }
    }
    if ((s = stage_end_impl(ctx, stage_t))) return s;
    if (unsat_out || min_unsat) {
        std::vector<uint32_t> tmp;
        uint32_t* u = unsat_out;
        if (!u) {
            tmp.resize(ctx->S.R);
            u = tmp.data();
        }
        if ((s = copy_out(ctx, u, ctx->S.unsat, ctx->S.R, FSMT_HOST))) return s;
        if (min_unsat) *min_unsat = *std::min_element(u, u + ctx->S.R);
    } else {
        CK(cudaStreamSynchronize(ctx->stream));
    }
    return check_flags(ctx);
}

fsmt_status fsmt_step_sizes(const fsmt_ctx* ctx, float kappa, float* eta_a, float* eta_b) {
    if (!ctx || !eta_a || !eta_b) return FSMT_ERR_ARG;
    const float kk = std::max(kappa, 1.0f);
    float ea = ctx->eta, eb = ctx->eta;                    // eta_mode 0
    if (ctx->eta_mode == 1) ea = eb = ctx->eta / kk;
    if (ctx->eta_mode == 2) ea = eb = ctx->eta / (kk * kk);
    if (ctx->eta_mode == 3) eb = ctx->eta / (kk * kk);     // block steps: a keeps eta, b gets eta/kappa^2
    *eta_a = ea;
    *eta_b = eb;
    return FSMT_OK;
}

fsmt_status fsmt_set_timing(fsmt_ctx* ctx, int enable) {
    if (!ctx) return FSMT_ERR_ARG;
    if (ctx->host_only) return fail(ctx, FSMT_ERR_CUDA, "host-only context has no device");
    ctx->timing = enable != 0;
    return FSMT_OK;
}

fsmt_status fsmt_get_timing(fsmt_ctx* ctx, double* ms, uint64_t* count, int reset) {
    if (!ctx) return FSMT_ERR_ARG;
    if (ctx->host_only) return fail(ctx, FSMT_ERR_CUDA, "host-only context has no device");
    timing_collect(ctx);
    for (int k = 0; k < 3; ++k) {
        if (ms) ms[k] = ctx->t_ms[k];
        if (count) count[k] = ctx->t_cnt[k];
        if (reset) {
            ctx->t_ms[k] = 0;
            ctx->t_cnt[k] = 0;
        }
    }
    return FSMT_OK;
}

fsmt_status fsmt_get_model(fsmt_ctx* ctx, uint32_t r, int8_t* x_out, float* y_out) {
    fsmt_status s = need(ctx, 3, "fsmt_get_model");
    if (s) return s;
    if (!ctx->rounded) return fail(ctx, FSMT_ERR_STATE, "fsmt_get_model: no stage_end yet");
    const DevState& S = ctx->S;
    if (r >= S.R) return fail(ctx, FSMT_ERR_ARG, "restart out of range");
    if (x_out && ctx->F.n_bool)
        CK(cudaMemcpy2DAsync(x_out, 1, S.x + r, S.R, 1, ctx->F.n_bool, cudaMemcpyDeviceToHost, ctx->stream));
    if (y_out && ctx->F.n_real)
        CK(cudaMemcpy2DAsync(y_out, 4, S.b + r, (size_t)S.R * 4, 4, ctx->F.n_real, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return FSMT_OK;
}

fsmt_status fsmt_get_rounded(fsmt_ctx* ctx, int8_t* x, int where) {
    fsmt_status s = need(ctx, 3, "fsmt_get_rounded");
    if (s) return s;
    if (!ctx->rounded) return fail(ctx, FSMT_ERR_STATE, "fsmt_get_rounded: no stage_end yet");
    return copy_out(ctx, x, ctx->S.x, (size_t)ctx->F.n_bool * ctx->S.R, where);
}

fsmt_status fsmt_verify(fsmt_ctx* ctx, const int8_t* x, const float* y, uint32_t* n_unsat, uint8_t* per_con) {
    fsmt_status s = need(ctx, 2, "fsmt_verify");
    if (s) return s;
    if ((!x && ctx->f.n_bool) || (!y && ctx->f.n_real) || !n_unsat) return fail(ctx, FSMT_ERR_ARG, "null argument");
    *n_unsat = verify_host(ctx->f, ctx->b, x, y, per_con);
    return FSMT_OK;
}

fsmt_status fsmt_verify_batch(fsmt_ctx* ctx, uint32_t R, const int8_t* x, const float* y, int where,
                              uint32_t* unsat_out, uint8_t* per_con) {
    fsmt_status s = need(ctx, 2, "fsmt_verify_batch");
    if (s) return s;
    if (ctx->host_only) return fail(ctx, FSMT_ERR_CUDA, "fsmt_verify_batch: host-only context has no device");
    if (R == 0 || !unsat_out) return fail(ctx, FSMT_ERR_ARG, "bad arguments");
    cudaSetDevice(ctx->device);
    const DevFormula& F = ctx->F;
    DevState T{};
    T.R = R;
    int8_t* dx = nullptr;
    float* dy = nullptr;
    uint8_t* dpc = nullptr;
    std::vector<void*> tmp;
    auto alloc = [&](void** p, size_t bytes) -> bool {
        if (cudaMalloc(p, std::max<size_t>(bytes, 16)) != cudaSuccess) return false;
        tmp.push_back(*p);
        return true;
    };
    const size_t nb = (size_t)F.n_bool * R, nr = (size_t)F.n_real * R, nc = (size_t)F.n_cons * R;
    uint8_t* dtt = nullptr;
    const size_t tt_rows = ctx->has_sym ? (size_t)ctx->slots.nv + ctx->slots.n_sa : 0;
    if (!alloc((void**)&dx, nb) || !alloc((void**)&dy, nr * 4) || !alloc((void**)&T.unsat, (size_t)R * 4) ||
        (per_con && !alloc((void**)&dpc, nc)) || (tt_rows && !alloc((void**)&dtt, tt_rows * R))) {
        free_list(tmp);
        return fail(ctx, FSMT_ERR_OOM, "cudaMalloc failed in fsmt_verify_batch");
    }
    cudaMemcpyKind k = where == FSMT_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    cudaError_t e = cudaSuccess;
    if (nb) e = cudaMemcpyAsync(dx, x, nb, k, ctx->stream);
    if (e == cudaSuccess && nr) e = cudaMemcpyAsync(dy, y, nr * 4, k, ctx->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(T.unsat, 0, (size_t)R * 4, ctx->stream);
    if (e == cudaSuccess) {
        if (ctx->T_all.n_tiles && ctx->jit.kernel5) {
            if (dtt) {
                DevSlots D2 = ctx->slots;
                D2.TT = dtt;
                launch_slot_truth(jk(ctx, R).ktruth, F, T, D2, dx, dy, ctx->stream);
                ctx->launches += 1;
            }
            launch_verify_jit(jk(ctx, R).kernel5, F, T, ctx->T_all, dx, dy, nullptr, dpc, ctx->stream, dtt);
            launch_verify(F, T, dx, dy, nullptr, dpc, ctx->stream, ctx->plan.jit_cons_end, F.n_cons);
            ctx->launches += 2;
        } else {
            launch_verify(F, T, dx, dy, nullptr, dpc, ctx->stream);
            ctx->launches += 1;
        }
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(unsat_out, T.unsat, (size_t)R * 4, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess && per_con) e = cudaMemcpyAsync(per_con, dpc, nc, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    free_list(tmp);
    if (e != cudaSuccess) return fail(ctx, FSMT_ERR_CUDA, std::string("fsmt_verify_batch: ") + cudaGetErrorString(e));
    return FSMT_OK;
}

// The device-side solve loop (DESIGN.md §7 item 16): the whole Alg.2 loop as ONE
// CUDA graph whose WHILE node runs a stage per iteration -- k_stage_begin (the stage's kappa, steps,
// e_t from the schedule), S x {sweep, update}, stage end (K4, K5), k_stage_best (best model kept on
// the device; continue while nothing is SAT and stages remain) -- so there is no host round trip per
// stage.  The host relaunches the same executable graph every `chunk` stages only to honour the
// time limit.  Same kernels and arithmetic as the host loop: identical results (tests).
static fsmt_status solve_graph(fsmt_ctx* ctx, uint32_t steps, std::chrono::steady_clock::time_point t0, uint32_t& stages,
                               uint32_t& best_unsat, uint32_t& best_stage, uint32_t& best_r, std::vector<int8_t>& bx,
                               std::vector<float>& by, bool& timeout) {
    const uint32_t T = (uint32_t)ctx->kappas.size();
    const uint32_t nbool = ctx->F.n_bool, nreal = ctx->F.n_real;
    std::vector<DevStage> sched(T);
    for (uint32_t t = 1; t <= T; ++t) {
        DevStage& d = sched[t - 1];
        d = DevStage{};
        d.kappa = ctx->kappas[t - 1];
        fsmt_step_sizes(ctx, d.kappa, &d.eta_a, &d.eta_b);
        d.t = t;
        d.et_int = et_int_of(t, ctx->erwa_mode);
        d.wfrac = wfrac_of(t, ctx->erwa_mode);

    }
    const uint32_t chunk = ctx->time_limit > 0 ? 16u : T;
    DevStage* d_sched = nullptr;
    DevStage* d_ds = nullptr;
    DevSolve* d_sv = nullptr;
    int8_t* d_xk = nullptr;
    float* d_yk = nullptr;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ex = nullptr;
    fsmt_status st = FSMT_OK;
    auto cleanup = [&]() {
        if (ex) cudaGraphExecDestroy(ex);
        if (g) cudaGraphDestroy(g);
        for (void* p : {(void*)d_sched, (void*)d_ds, (void*)d_sv, (void*)d_xk, (void*)d_yk})
            if (p) cudaFree(p);
        ctx->S.ds = nullptr;
    };
#define CKG(call)                                                                                            \
    do {                                                                                                     \
        cudaError_t e_ = (call);                                                                             \
        if (e_ != cudaSuccess) {                                                                             \
            cudaStreamCaptureStatus cs_;                                                                     \
            if (cudaStreamIsCapturing(ctx->stream, &cs_) == cudaSuccess && cs_ != cudaStreamCaptureStatusNone) { \
                cudaGraph_t junk_ = nullptr;                                                                 \
                cudaStreamEndCapture(ctx->stream, &junk_);                                                   \
                if (junk_) cudaGraphDestroy(junk_);                                                          \
            }                                                                                                \
            cudaGetLastError();                                                                              \
            cleanup();                                                                                       \
            return fail(ctx, FSMT_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e_));                \
        }                                                                                                    \
    } while (0)
    CKG(cudaMalloc((void**)&d_sched, sizeof(DevStage) * std::max<uint32_t>(T, 1)));
    CKG(cudaMalloc((void**)&d_ds, sizeof(DevStage)));
    CKG(cudaMalloc((void**)&d_sv, sizeof(DevSolve)));
    CKG(cudaMalloc((void**)&d_xk, std::max<uint32_t>(nbool, 1)));
    CKG(cudaMalloc((void**)&d_yk, 4 * std::max<uint32_t>(nreal, 1)));
    CKG(cudaMemcpyAsync(d_sched, sched.data(), sizeof(DevStage) * T, cudaMemcpyHostToDevice, ctx->stream));
    DevSolve sv{};
    sv.t = 1;
    sv.t_end = std::min(T, chunk);
    sv.best_unsat = UINT32_MAX;
    CKG(cudaMemcpyAsync(d_sv, &sv, sizeof(sv), cudaMemcpyHostToDevice, ctx->stream));
    CKG(cudaStreamSynchronize(ctx->stream));
    // the graph: one WHILE node whose body is one stage
    CKG(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    CKG(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    CKG(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    ctx->S.ds = d_ds;
    const uint64_t l0 = ctx->launches;
    CKG(cudaStreamBeginCaptureToGraph(ctx->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    launch_stage_begin(d_sv, d_sched, d_ds, ctx->stream);
    CKG(cudaMemsetAsync(ctx->S.frozen, 0, ctx->S.R, ctx->stream));
    for (uint32_t k = 0; k < steps && !st; ++k) {
        st = sweep_impl(ctx, 0.f, 1, nullptr, 0);              // kappa / e_t from the DevStage
        if (!st) st = update_impl(ctx, 1.f, ctx->eps, 1.f);   // eta / eta_b from the DevStage
    }
    if (!st) st = stage_end_impl(ctx, 0);                      // Philox stage word from the DevStage
    launch_stage_best(d_sv, ctx->S, nbool, nreal, d_xk, d_yk, h, ctx->stream);
    cudaGraph_t cap = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(ctx->stream, &cap);
    ctx->S.ds = nullptr;
    const uint64_t per_stage = ctx->launches - l0 + 2;
    ctx->launches = l0;
    if (st) {
        cleanup();
        return st;
    }
    CKG(ec);
    CKG(cudaGraphInstantiate(&ex, g, 0));
    for (;;) {
        CKG(cudaGraphLaunch(ex, ctx->stream));
        CKG(cudaMemcpyAsync(&sv, d_sv, sizeof(sv), cudaMemcpyDeviceToHost, ctx->stream));
        CKG(cudaMemcpyAsync(ctx->hflags, ctx->S.flags, 4, cudaMemcpyDeviceToHost, ctx->stream));
        CKG(cudaStreamSynchronize(ctx->stream));
        if ((st = check_flags(ctx))) break;
        if (sv.best_unsat == 0 || sv.t > T) break;
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (ctx->time_limit > 0 && el > ctx->time_limit) {
            timeout = true;
            break;
        }
        const uint32_t t_end = std::min(T, sv.t + chunk - 1);
        CKG(cudaMemcpyAsync(&d_sv->t_end, &t_end, 4, cudaMemcpyHostToDevice, ctx->stream));
    }
    stages = sv.t - 1;
    ctx->launches += per_stage * stages;
    best_unsat = sv.best_unsat;
    best_stage = sv.best_stage;
    best_r = sv.best_r;
    if (!st && best_unsat != UINT32_MAX) {
        if (nbool) CKG(cudaMemcpyAsync(bx.data(), d_xk, nbool, cudaMemcpyDeviceToHost, ctx->stream));
        if (nreal) CKG(cudaMemcpyAsync(by.data(), d_yk, 4 * (size_t)nreal, cudaMemcpyDeviceToHost, ctx->stream));
        CKG(cudaStreamSynchronize(ctx->stream));
        ctx->rounded = true;
    }
#undef CKG
    cleanup();
    return st;
}

fsmt_status fsmt_solve(fsmt_ctx* ctx, uint32_t restarts, uint32_t steps, uint64_t seed, fsmt_verdict* verdict,
                       int8_t* x_out, float* y_out, fsmt_stats* stats) {
    fsmt_status s = need(ctx, 2, "fsmt_solve");
    if (s) return s;
    if (ctx->host_only) return fail(ctx, FSMT_ERR_CUDA, "fsmt_solve: host-only context has no device");
    if (!verdict || restarts == 0) return fail(ctx, FSMT_ERR_ARG, "bad arguments");
    if (ctx->shard_mode == 1 && ctx->shard_world > 1)
        return fail(ctx, FSMT_ERR_STATE, "fsmt_solve: constraint-sharded context (use the step API with all-reduces)");
    auto t0 = std::chrono::steady_clock::now();
    if ((s = fsmt_begin(ctx, restarts, seed, 0))) return s;
    const uint32_t nbool = ctx->F.n_bool, nreal = ctx->F.n_real;
    std::vector<uint32_t> unsat(restarts);
    std::vector<int8_t> bx(nbool);
    std::vector<float> by(nreal);
    uint32_t best_unsat = UINT32_MAX, best_stage = 0, best_r = 0;
    uint32_t stages = 0, steps_run = 0;
    bool sat = false, timeout = false;
    fsmt_stats st{};
    // the device-side loop (one CUDA graph, no per-stage host round trip) unless FSMT_SOLVE_GRAPH=0,
    // per-kernel timing is on (events) or the stage graph of FSMT_GRAPH is requested
    const char* sg = getenv("FSMT_SOLVE_GRAPH");
    const char* og = getenv("FSMT_GRAPH");
    const bool graph = !(sg && sg[0] == '0') && !ctx->timing && !(og && og[0] == '1');
    if (graph) {
        if ((s = solve_graph(ctx, steps, t0, stages, best_unsat, best_stage, best_r, bx, by, timeout))) return s;
        steps_run = stages * steps;
        sat = best_unsat == 0;
    }
    for (uint32_t t = 1; !graph && t <= ctx->kappas.size(); ++t) {
        const float kappa = ctx->kappas[t - 1];
        if ((s = fsmt_run_stage(ctx, t, kappa, steps, unsat.data(), nullptr))) return s;
        steps_run += steps;
        ++stages;
        // lowest restart with unsat == 0 wins (smallest (t, r)); else track min (unsat, t, r)
        uint32_t r_min = 0;
        for (uint32_t r = 1; r < restarts; ++r)
            if (unsat[r] < unsat[r_min]) r_min = r;
        if (unsat[r_min] < best_unsat) {   // keep the model; the host re-check runs once, on the returned one
            if ((s = fsmt_get_model(ctx, r_min, bx.data(), by.data()))) return s;
            best_unsat = unsat[r_min];
            best_stage = t;
            best_r = r_min;
        }
        if (best_unsat == 0) {
            sat = true;
            break;
        }
        double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (ctx->time_limit > 0 && el > ctx->time_limit) {
            timeout = true;
            break;
        }
    }
    // host fp64 re-verification of the returned model ("never SAT without verify")
    if (best_unsat != UINT32_MAX) {
        const uint32_t host_unsat = verify_host(ctx->f, ctx->b, bx.data(), by.data(), nullptr);
        if (sat && host_unsat != 0)
            return fail(ctx, FSMT_ERR_CUDA, "device verdict SAT contradicted by host re-verification");
        st.host_verified = host_unsat == best_unsat;
    }
    *verdict = sat ? FSMT_SAT : FSMT_UNKNOWN;
    if (x_out) std::copy(bx.begin(), bx.end(), x_out);
    if (y_out) std::copy(by.begin(), by.end(), y_out);
    if (stats) {
        st.stages_run = stages;
        st.steps_run = steps_run;
        st.winner_restart = best_r;
        st.winner_stage = best_stage;
        st.best_unsat = best_unsat;
        st.solve_ms = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() * 1e3;
        st.evals = (double)steps_run * (double)ctx->F.n_cons * (double)restarts;
        *stats = st;
    }
    return timeout ? FSMT_ERR_TIMEOUT : FSMT_OK;
}

uint64_t fsmt_kernel_launches(const fsmt_ctx* ctx) { return ctx ? ctx->launches : 0; }
uint32_t fsmt_restarts(const fsmt_ctx* ctx) { return ctx && ctx->stage >= 3 ? ctx->S.R : 0; }

fsmt_status fsmt_device_buffers(fsmt_ctx* ctx, void** a, void** b, void** ga, void** gb, void** U, void** obj,
                                void** unsat) {
    fsmt_status s = need(ctx, 3, "fsmt_device_buffers");
    if (s) return s;
    if (a) *a = ctx->S.a;
    if (b) *b = ctx->S.b;
    if (ga) *ga = ctx->S.ga;
    if (gb) *gb = ctx->S.gb;
    if (U) *U = ctx->S.U;
    if (obj) *obj = ctx->S.obj;
    if (unsat) *unsat = ctx->S.unsat;
    return FSMT_OK;
}

fsmt_status fsmt_time_sweep(fsmt_ctx* ctx, float kappa, uint32_t stage_t, uint32_t iters, double* ms_out) {
    fsmt_status s = need(ctx, 3, "fsmt_time_sweep");
    if (s) return s;
    if (!ms_out || iters == 0) return fail(ctx, FSMT_ERR_ARG, "bad arguments");
    const bool was = ctx->timing;
    timing_collect(ctx);
    const double ms0 = ctx->t_ms[0];
    const uint64_t n0 = ctx->t_cnt[0];
    ctx->timing = true;
    for (uint32_t i = 0; i < iters; ++i)
        if ((s = sweep_impl(ctx, kappa, stage_t ? stage_t : 1, nullptr, 0))) break;
    timing_collect(ctx);
    ctx->timing = was;
    if (s) return s;
    *ms_out = (ctx->t_ms[0] - ms0) / (double)std::max<uint64_t>(ctx->t_cnt[0] - n0, 1);
    return FSMT_OK;
}

}  // extern "C"
