#include <cstdlib>
// sm_100a kernels of the FourierSMT hot path.
//
//   K0 k0_init    Philox init of (a, b) + projection            (R20; Def.1)
//   K1 k1_sweep   slot probabilities + Gaussian smoothing (Eq.4, Eq.7), forward xBDD pass
//                 (Alg.F), backward pass (Alg.B, sign R1), chain rule
//                 (P:1326-1327), weighted objective and gradient accumulation (Eq.10)
//   K3 k3_*       projected gradient step, gradient mapping, eps-freeze (Eq.11-14)
//   K4 k4_round   x = sgn(a) | R(a) (Alg.1 line 10; Eq.4; R17)
//   K5 k5_verify  exact check of every constraint (R22) + ERWA violation counters (R18)
//
// Layout: restart-minor; a warp's 32 lanes are 32 restarts of the same constraint, so every
// structure load is warp-uniform (one transaction, broadcast) and every state load/store is
// a coalesced 128 B row segment.  No tensor cores: nothing here is a dense contraction.
#include <cmath>
#include <cstdio>

#include "kernels.hpp"

namespace fsmt {
namespace {

constexpr int kFalseT = -1;
constexpr int kTrueT = -2;
constexpr int kChunk = 16;        // constraints per warp in K1 / K5

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

__device__ __forceinline__ uint32_t draw24(uint64_t seed, uint32_t r, uint32_t var, uint32_t stage, uint32_t tag) {
    const uint4 o = philox4x32_10(make_uint4(r, var, stage, tag), make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
    return o.x >> 8;
}

// ---------------------------------------------------------------------------------------- K0

// w0 * 2^(u + ebias - 127): the fp32 ERWA weight with the restart's shift (FxScale; exact, 0 below
// 2^-126, never inf since u + ebias <= 127 + kWeightWindow)
__device__ __forceinline__ float weight_of(float w0, uint32_t u, int ebias) {
    return w0 * __uint_as_float((uint32_t)max((int)u + ebias, 0) << 23);
}

// v on the restart's grid, in grid units (FxScale): rintf(v 2^-G), exact scaling; fp32 values of
// magnitude >= 2^23 are integers already
__device__ __forceinline__ double grid_units(float v, float gif) { return (double)rintf(v * gif); }

__device__ __forceinline__ int ceil_log2(double x) {
    if (!(x > 0.0)) return 0;
    int e = 0;
    const double f = frexp(x, &e);    // x = f 2^e, f in [1/2, 1)
    return f == 0.5 ? e - 1 : e;
}

__global__ void k0_init(DevFormula F, DevState S, uint64_t seed, uint32_t off) {
    const uint64_t n = (uint64_t)(F.n_bool + F.n_real) * S.R;
    for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = (uint32_t)(idx / S.R), r = (uint32_t)(idx % S.R);
        if (v < F.n_bool) {
            const uint32_t k = draw24(seed, off + r, v, 0, 0);
            const float a = (float)((int32_t)(2u * k + 1u) - (1 << 24)) * 0x1p-24f;   // exact (R20)
            S.a[(size_t)v * S.R + r] = fminf(fmaxf(a, -1.f), 1.f);
        } else {
            const uint32_t j = v - F.n_bool;
            const uint32_t k = draw24(seed, off + r, j, 0, 1);
            const double u = (double)(2u * k + 1u) * 0x1p-25;
            const float lo = F.lo[j], hi = F.hi[j];
            double val;
            if (isfinite(lo) && isfinite(hi))
                val = __dadd_rn((double)lo, __dmul_rn(__dsub_rn((double)hi, (double)lo), u));
            else
                val = __dsub_rn(__dmul_rn(2.0, u), 1.0);
            const float bv = __double2float_rn(val);
            // with the R33 projection the halfspace variables start unclamped (Dykstra owns their box)
            S.b[(size_t)j * S.R + r] = (F.proj_iters && F.in_h[j]) ? bv : fminf(fmaxf(bv, lo), hi);
        }
    }
}

// ---------------------------------------------------------------------------------------- K1

__global__ void __launch_bounds__(256) k1_sweep(DevFormula F, DevState S, float kappa,
                                                double* __restrict__ terms, uint32_t terms_r, int smax, int nmax) {
    extern __shared__ float smem[];
    if (S.ds) kappa = S.ds->kappa;                               // device-side solve loop (DevStage)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t R = S.R;
    const uint32_t rtiles = (R + 31) / 32;
    const uint64_t gw = (uint64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    const uint32_t rt = (uint32_t)(gw % rtiles);
    const uint64_t c0 = F.generic_begin + (gw / rtiles) * kChunk;
    if (c0 >= F.generic_end) return;
    const uint64_t c1 = min(c0 + (uint64_t)kChunk, (uint64_t)F.generic_end);
    const uint32_t r = rt * 32 + lane;
    const bool live = r < R;
    const size_t rr = live ? r : 0;
    float* PT = smem + (size_t)warp * (4 * smax + nmax) * 32;   // P[slot True]   (Eq.4 / Eq.7)
    float* PF = PT + smax * 32;                                   // P[slot False]
    float* DD = PF + smax * 32;                                   // dd/dz' factor for atom slots
    float* G = DD + smax * 32;                                    // dE/dv per slot
    float* M = G + smax * 32;                                     // m_td, then m_bu (in place)
    const float kq = kappa * 0.70710678118654752f;               // kappa / sqrt(2)
    const float dcoef = kappa * 0.79788456080286536f;            // kappa * sqrt(2/pi)
    double objacc = 0.0;
    const FxScale fx = S.fx[rr];
    for (uint64_t c = c0; c < c1; ++c) {
        const uint32_t tid = F.cons_tmpl[c];
        const uint32_t so = F.cons_slot_off[c];
        const uint32_t ns = F.cons_slot_off[c + 1] - so;
        const uint32_t ko = F.tmpl_kind_off[tid];
        const uint32_t no = F.tmpl_node_off[tid];
        const uint32_t nn = F.tmpl_node_off[tid + 1] - no;
        const int root = F.tmpl_root[tid];
        // w_cr = w_c 2^(U + e_t) (R18) in the restart's reduced units (FxScale)
        const float w = weight_of(F.cons_w[c], S.U ? S.U[(size_t)c * R + rr] : 0u, fx.ebias);   // 2^frac(e_t): fx.gif
        // a1: slot probabilities (Eq.4 for Booleans, Eq.7 for atoms; erfc form, R28b)
        for (uint32_t s = 0; s < ns; ++s) {
            const uint32_t gid = F.slot_ids[so + s];
            float pt, pf, dd = 0.f;
            if (F.kinds[ko + s] == 0) {
                const float v = S.a[(size_t)gid * R + rr];
                pt = 0.5f * (1.f - v);
                pf = 0.5f * (1.f + v);
            } else {
                const uint32_t k0 = F.atom_rowptr[gid], k1 = F.atom_rowptr[gid + 1];
                float z = -F.atom_rhs[gid];
                for (uint32_t k = k0; k < k1; ++k) z = fmaf(F.atom_val[k], S.b[(size_t)F.atom_col[k] * R + rr], z);
                const float inv = F.atom_invnorm[gid];
                const float u = kq * z * inv;                           // z / (sqrt2 ||q|| sigma)
                pt = 0.5f * erfcf(u);                                   // (1 - d)/2, d = erf(u)
                pf = 0.5f * erfcf(-u);                                  // (1 + d)/2
                dd = dcoef * inv * expf(-u * u);                        // dd/db_j = dd * q_j
            }
            PT[s * 32 + lane] = pt;
            PF[s * 32 + lane] = pf;
            DD[s * 32 + lane] = dd;
            G[s * 32 + lane] = 0.f;
        }
        // a2: forward pass, Alg.F: m_td[root] = 1; m_td[v.t] += p m_td[v]; m_td[v.f] += (1-p) m_td[v]
        for (uint32_t v = 0; v < nn; ++v) M[v * 32 + lane] = 0.f;
        float pT = (root == kTrueT) ? 1.f : 0.f;
        if (root >= 0) M[root * 32 + lane] = 1.f;
        for (uint32_t v = 0; v < nn; ++v) {
            const DevNode nd = F.nodes[no + v];
            const float m = M[v * 32 + lane];
            const float th = PT[nd.level * 32 + lane] * m;
            const float tl = PF[nd.level * 32 + lane] * m;
            if (nd.hi >= 0) M[nd.hi * 32 + lane] += th; else if (nd.hi == kTrueT) pT += th;
            if (nd.lo >= 0) M[nd.lo * 32 + lane] += tl; else if (nd.lo == kTrueT) pT += tl;
        }
        const float E = 1.f - 2.f * pT;                               // Alg.F line P:1170
        // a3: backward pass, Alg.B: m_bu[T]=1, m_bu[F]=0, m_bu[v] = p m_bu[v.t] + (1-p) m_bu[v.f];
        //     dE/dv_s = sum_{v: slot s} m_td[v] (m_bu[v.t] - m_bu[v.f])     (R1)
        for (int v = (int)nn - 1; v >= 0; --v) {
            const DevNode nd = F.nodes[no + v];
            const float bh = nd.hi >= 0 ? M[nd.hi * 32 + lane] : (nd.hi == kTrueT ? 1.f : 0.f);
            const float bl = nd.lo >= 0 ? M[nd.lo * 32 + lane] : (nd.lo == kTrueT ? 1.f : 0.f);
            const float mt = M[v * 32 + lane];
            G[nd.level * 32 + lane] += mt * (bh - bl);
            M[v * 32 + lane] = PT[nd.level * 32 + lane] * bh + PF[nd.level * 32 + lane] * bl;
        }
        // a4: chain rule + accumulate (fp64, R28; every term on the restart's grid: exact sums)
        if (live) {
            for (uint32_t s = 0; s < ns; ++s) {
                const uint32_t gid = F.slot_ids[so + s];
                const float g = w * G[s * 32 + lane];
                if (F.kinds[ko + s] == 0) {
                    atomicAdd(&S.ga[(size_t)gid * R + r], grid_units(g, fx.gif));
                } else {
                    const float gd = g * DD[s * 32 + lane];
                    for (uint32_t k = F.atom_rowptr[gid]; k < F.atom_rowptr[gid + 1]; ++k)
                        atomicAdd(&S.gb[(size_t)F.atom_col[k] * R + r], grid_units(gd * F.atom_val[k], fx.gif));
                }
            }
            objacc += (double)w * (double)E;
            if (terms != nullptr && r == terms_r) terms[F.orig[c]] = (double)E;
        }
    }
    if (live) atomicAdd(&S.obj[r], rint(objacc * fx.oi) * fx.os);
}

// Before every sweep (DESIGN.md §7 item 14): zero the fp64 outputs and write the restart's FxScale.
// With m = umax[r], s_r = max(0, m - W), wm = min(m, W): fp32 weights are <= 2^wm (normalised
// w_c <= 1, times 2^frac(e_t) <= sqrt 2), so every partial gradient sum in reduced units is
// bounded by B_g = 2^wm max(fx_fb, kappa fx_fa) times 2 (sqrt 2) times 2 (margin); the grid 2^G,
// G = ceil(log2 B_g) - 48, keeps every sum below 2^50 grid units (exact integers in fp64).
__global__ void k1_prologue(DevFormula F, DevState S, float kappa, int et_int, float wfrac, double* __restrict__ gu,
                            uint64_t gu_rows) {
    if (S.ds) {                                                   // device-side solve loop (DevStage)
        kappa = S.ds->kappa;
        et_int = S.ds->et_int;
        wfrac = S.ds->wfrac;
    }
    const uint64_t R = S.R;
    const uint64_t nb = (uint64_t)F.n_bool * R, nr = (uint64_t)F.n_real * R, ng = gu ? gu_rows * R : 0;
    const uint64_t n = nb + nr + R + ng;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        if (i < nb) S.ga[i] = 0.0;
        else if (i < nb + nr) S.gb[i - nb] = 0.0;
        else if (i < nb + nr + R) {
            const uint32_t r = (uint32_t)(i - nb - nr);
            S.obj[r] = 0.0;
            const int m = (int)S.umax[r];
            const int sh = max(0, m - kWeightWindow), wm = min(m, kWeightWindow);
            // G in [-100, 120]: 2^-G is a normal fp32 (bounds >= 2^-52 for any non-empty formula)
            const int G = min(120, max(-100, ceil_log2(ldexp(fmax(F.fx_fb, (double)kappa * F.fx_fa), wm)) - 48));
            const int O = ceil_log2(ldexp(F.fx_sw, wm)) - 48;
            const int tail = sh + F.wexp + et_int;
            // the largest value a sum can reach is 2^(G or O + tail + 50): beyond fp64, report
            if (max(G, O) + tail > 960) atomicOr(S.flags, 2u);
            FxScale fx;
            fx.gs = ldexp(1.0, G + tail);
            fx.ti = ldexp(1.0, -(G + tail));
            fx.oi = (double)wfrac * ldexp(1.0, -O);   // 2^frac(e_t) applied at the flush (x wfrac: one fp64 rounding)
            fx.os = ldexp(1.0, O + tail);
            fx.gif = wfrac * ldexpf(1.f, -G);         // 2^frac(e_t) times 2^-G (exact scaling by 2^-G)
            fx.ebias = 127 - sh;
            S.fx[r] = fx;
            S.gsc[r] = fx.gs;
        } else {
            gu[i - nb - nr - R] = 0.0;
        }
    }
}

__global__ void k_scale_rows(double* __restrict__ dst, const double* __restrict__ src, const double* __restrict__ gsc,
                             uint64_t n, uint32_t R) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        dst[i] = src[i] * gsc[i % R];
}

__global__ void k_umax(const uint16_t* __restrict__ U, uint32_t C, uint32_t R, uint32_t* __restrict__ umax) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R) return;
    uint32_t m = 0;
    for (uint32_t c = 0; c < C; ++c) m = max(m, (uint32_t)U[(size_t)c * R + r]);
    umax[r] = m;
}

// ---------------------------------------------------------------------------------------- K3

constexpr int kVarsPerPart = 64;

__device__ __forceinline__ float step_value(float x, double g, float eta, float lo, float hi) {
    double t = (double)x - (double)eta * g;
    t = fmin(fmax(t, (double)lo), (double)hi);
    return __double2float_rn(t);
}

// candidate b' of the projected step (R33): halfspace variables unclamped (Dykstra projects
// them), the others clamped to their interval (their exact projection)
__global__ void k3_cand(DevFormula F, DevState S, float eta_b) {
    if (S.ds) eta_b = S.ds->eta_b;
    const uint64_t n = (uint64_t)F.n_real * S.R;
    for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t j = (uint32_t)(idx / S.R);
        const bool h = F.in_h[j];
        S.bn[idx] = step_value(S.b[idx], S.gb[idx] * S.gsc[idx % S.R], eta_b, h ? -INFINITY : F.lo[j], h ? INFINITY : F.hi[j]);
    }
}

// Dykstra's algorithm (R33), one CTA per restart, the restart's halfspace variables and all
// corrections in shared memory: sets C_1..C_K = halfspaces g_k.b <= h_k in constraint order,
// then C_0 = the box of the halfspace variables, F.proj_iters sweeps.  The halfspaces are
// stored by dependency level (api.cpp): within a level they touch disjoint variables, so the
// threads of the CTA project them concurrently and the level barrier reproduces the sequential
// sweep exactly.
__global__ void __launch_bounds__(128) k_dykstra(DevFormula F, DevState S, float* __restrict__ X, bool skip_frozen) {
    extern __shared__ float sh[];
    const uint32_t r = blockIdx.x, R = S.R;
    if (skip_frozen && S.frozen[r]) return;
    const uint32_t nv = F.n_hvars, nnz = F.h_rowptr[F.n_half];
    float* xs = sh;                 // [nv] iterate
    float* pb = xs + nv;            // [nv] box corrections
    float* ph = pb + nv;            // [nnz] halfspace corrections
    for (uint32_t v = threadIdx.x; v < nv; v += blockDim.x) {
        xs[v] = X[(size_t)F.hvars[v] * R + r];
        pb[v] = 0.f;
    }
    for (uint32_t k = threadIdx.x; k < nnz; k += blockDim.x) ph[k] = 0.f;
    __syncthreads();
    for (uint32_t it = 0; it < F.proj_iters; ++it) {
        for (uint32_t l = 0; l < F.n_hlevels; ++l) {
            for (uint32_t h = F.h_level_off[l] + threadIdx.x; h < F.h_level_off[l + 1]; h += blockDim.x) {
                const uint32_t k0 = F.h_rowptr[h], k1 = F.h_rowptr[h + 1];
                float v = -F.h_h[h];
                for (uint32_t k = k0; k < k1; ++k) v = fmaf(F.h_g[k], xs[F.h_col[k]] + ph[k], v);
                const float t = fmaxf(v, 0.f) * F.h_inv2[h];
                for (uint32_t k = k0; k < k1; ++k) {
                    const float y = xs[F.h_col[k]] + ph[k];
                    const float xn = fmaf(-t, F.h_g[k], y);
                    ph[k] = y - xn;
                    xs[F.h_col[k]] = xn;
                }
            }
            __syncthreads();
        }
        for (uint32_t v = threadIdx.x; v < nv; v += blockDim.x) {
            const uint32_t j = F.hvars[v];
            const float y = xs[v] + pb[v];
            const float xn = fminf(fmaxf(y, F.lo[j]), F.hi[j]);
            pb[v] = y - xn;
            xs[v] = xn;
        }
        __syncthreads();
    }
    for (uint32_t v = threadIdx.x; v < nv; v += blockDim.x) X[(size_t)F.hvars[v] * R + r] = xs[v];
}

__global__ void k3_norm(DevFormula F, DevState S, float eta, float eta_b, uint32_t vpp) {
    if (S.ds) { eta = S.ds->eta_a; eta_b = S.ds->eta_b; }
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= S.R) return;
    const uint32_t part = blockIdx.y;
    const uint32_t nv = F.n_bool + F.n_real;
    const uint32_t v0 = part * vpp, v1 = min(v0 + vpp, nv);
    const double gs = S.gsc[r];                 // grid units -> gradient (FxScale)
    double acc = 0.0;
    for (uint32_t v = v0; v < v1; ++v) {
        float x, xn;
        if (v < F.n_bool) {
            x = S.a[(size_t)v * S.R + r];
            xn = step_value(x, S.ga[(size_t)v * S.R + r] * gs, eta, -1.f, 1.f);
        } else {
            const uint32_t j = v - F.n_bool;
            x = S.b[(size_t)j * S.R + r];
            xn = S.bn ? S.bn[(size_t)j * S.R + r] : step_value(x, S.gb[(size_t)j * S.R + r] * gs, eta_b, F.lo[j], F.hi[j]);
        }
        const double d = ((double)x - (double)xn) / (double)(v < F.n_bool ? eta : eta_b);
        acc += d * d;
    }
    S.gm2_part[(size_t)part * S.R + r] = acc;
}

// few restarts (R < 512): many short parts, summed per restart by one block (fixed order)
__global__ void k3_final_block(DevState S, uint32_t n_parts, float eps) {
    __shared__ double red[8];
    const uint32_t r = blockIdx.x;
    double acc = 0.0;
    for (uint32_t p = threadIdx.x; p < n_parts; p += blockDim.x) acc += S.gm2_part[(size_t)p * S.R + r];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (uint32_t w = 0; w < blockDim.x / 32; ++w) t += red[w];
        S.gm2[r] = t;
        if (!S.frozen[r] && t <= (double)eps * (double)eps) S.frozen[r] = 1;   // Eq.14
    }
}

__global__ void k3_final(DevState S, uint32_t n_parts, float eps) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= S.R) return;
    double acc = 0.0;
    for (uint32_t p = 0; p < n_parts; ++p) acc += S.gm2_part[(size_t)p * S.R + r];
    S.gm2[r] = acc;
    if (!S.frozen[r] && acc <= (double)eps * (double)eps) S.frozen[r] = 1;   // Eq.14
}

__global__ void k3_apply(DevFormula F, DevState S, float eta, float eta_b) {
    if (S.ds) { eta = S.ds->eta_a; eta_b = S.ds->eta_b; }
    const uint64_t n = (uint64_t)(F.n_bool + F.n_real) * S.R;
    for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = (uint32_t)(idx / S.R), r = (uint32_t)(idx % S.R);
        if (S.frozen[r]) continue;
        const double gs = S.gsc[r];
        if (v < F.n_bool) {
            float& x = S.a[(size_t)v * S.R + r];
            x = step_value(x, S.ga[(size_t)v * S.R + r] * gs, eta, -1.f, 1.f);
        } else {
            const uint32_t j = v - F.n_bool;
            float& x = S.b[(size_t)j * S.R + r];
            x = S.bn ? S.bn[(size_t)j * S.R + r] : step_value(x, S.gb[(size_t)j * S.R + r] * gs, eta_b, F.lo[j], F.hi[j]);
        }
    }
}

// ---------------------------------------------------------------------------------------- K4

__global__ void k4_round(DevFormula F, DevState S, uint32_t rounding, uint64_t seed, uint32_t off, uint32_t stage) {
    if (S.ds) stage += S.ds->t;            // device-side solve loop: the launch passes only the R34 draw (m << 16)
    const uint64_t n = (uint64_t)F.n_bool * S.R;
    for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t i = (uint32_t)(idx / S.R), r = (uint32_t)(idx % S.R);
        const float a = S.a[idx];
        bool is_true;
        if (rounding == 0) {
            is_true = a < 0.f;                                    // sgn(0) = +1
        } else {
            const uint32_t k = draw24(seed, off + r, i, stage, 2);
            is_true = a < 1.f - (float)k * 0x1p-23f;              // P[x=-1] = (1-a)/2 (Eq.4)
        }
        S.x[idx] = is_true ? (int8_t)-1 : (int8_t)1;
    }
}

// ---------------------------------------------------------------------------------------- K5

__global__ void __launch_bounds__(256) k5_verify(DevFormula F, DevState S, const int8_t* __restrict__ x,
                                                 const float* __restrict__ y, uint16_t* __restrict__ Uupd,
                                                 uint8_t* __restrict__ per_con, uint32_t cb, uint32_t ce) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t R = S.R;
    const uint32_t rtiles = (R + 31) / 32;
    const uint64_t gw = (uint64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    const uint32_t rt = (uint32_t)(gw % rtiles);
    const uint64_t c0 = cb + (gw / rtiles) * kChunk;
    if (c0 >= ce) return;
    const uint64_t c1 = min(c0 + (uint64_t)kChunk, (uint64_t)ce);
    const uint32_t r = rt * 32 + lane;
    if (r >= R) return;
    uint32_t cnt = 0, umx = 0, ovf = 0;
    for (uint64_t c = c0; c < c1; ++c) {
        const uint32_t tid = F.cons_tmpl[c];
        const uint32_t so = F.cons_slot_off[c];
        const uint32_t ko = F.tmpl_kind_off[tid];
        const uint32_t no = F.tmpl_node_off[tid];
        int v = F.tmpl_root[tid];
        while (v >= 0) {
            const DevNode nd = F.nodes[no + v];
            const uint32_t gid = F.slot_ids[so + nd.level];
            bool truth;
            if (F.kinds[ko + nd.level] == 0) {
                truth = x[(size_t)gid * R + r] == -1;
            } else {                                          // exact fp64, stored order, no FMA (R22)
                double s = 0.0;
                for (uint32_t k = F.atom_rowptr[gid]; k < F.atom_rowptr[gid + 1]; ++k)
                    s = __dadd_rn(s, __dmul_rn(F.atom_val64[k], (double)y[(size_t)F.atom_col[k] * R + r]));
                truth = F.atom_strict[gid] ? (s < F.atom_rhs64[gid]) : (s <= F.atom_rhs64[gid]);
            }
            v = truth ? nd.hi : nd.lo;
        }
        const uint32_t u = (v == kFalseT) ? 1u : 0u;            // u_c = f_c/2 + 1/2 (Alg.2 line 7)
        cnt += u;
        if (Uupd && u) {                                      // U += u: only violated constraints touch memory
            uint16_t& cell = Uupd[(size_t)c * R + r];
            const uint32_t nv = (uint32_t)cell + 1u;
            ovf |= nv > 65535u;                               // reported (FSMT_ERR_RANGE), never silent
            const uint32_t nc = min(65535u, nv);
            cell = (uint16_t)nc;
            umx = max(umx, nc);
        }
        if (per_con) per_con[(size_t)F.orig[c] * R + r] = (uint8_t)u;
    }
    atomicAdd(&S.unsat[r], cnt);
    if (umx) atomicMax(&S.umax[r], umx);
    if (ovf) atomicOr(S.flags, 1u);
}


}  // namespace

int sweep_smem_bytes(const DevFormula& F, int warps) {
    const int smax = (int)F.max_slots > 0 ? (int)F.max_slots : 1;
    const int nmax = (int)F.max_nodes > 0 ? (int)F.max_nodes : 1;
    return warps * (4 * smax + nmax) * 32 * (int)sizeof(float);
}

static int sweep_warps(const DevFormula& F) {
    for (int w = 8; w >= 1; w >>= 1)
        if (sweep_smem_bytes(F, w) <= 110 * 1024) return w;
    return 1;
}

void launch_init(const DevFormula& F, const DevState& S, uint64_t seed, uint32_t off, cudaStream_t st) {
    const uint64_t n = (uint64_t)(F.n_bool + F.n_real) * S.R;
    const int threads = 256;
    const uint64_t blocks = std::min<uint64_t>((n + threads - 1) / threads, 148ull * 16);
    if (n) k0_init<<<(unsigned)std::max<uint64_t>(blocks, 1), threads, 0, st>>>(F, S, seed, off);
}

__global__ void k_gather_rows_u16(uint16_t* __restrict__ dst, const uint16_t* __restrict__ src,
                                  const uint32_t* __restrict__ idx, uint32_t rows, uint32_t R, int scatter) {
    const uint64_t n = (uint64_t)rows * R;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t i = (uint32_t)(t / R), r = (uint32_t)(t % R);
        if (scatter) dst[(size_t)idx[i] * R + r] = src[t];
        else dst[t] = src[(size_t)idx[i] * R + r];
    }
}

void launch_gather_rows_u16(uint16_t* dst, const uint16_t* src, const uint32_t* idx, uint32_t rows, uint32_t R,
                            cudaStream_t st) {
    if (!rows || !R) return;
    k_gather_rows_u16<<<148 * 8, 256, 0, st>>>(dst, src, idx, rows, R, 0);
}

// Tiles are split into constraint ranges at launch when (tiles x restart tiles) would leave the
// GPU short of one-warp CTAs (few restarts, e.g. R = 32): ~16 K CTAs fill 148 SMs x 28 slots four
// times over; at most 8 ranges per tile.
// Each range re-runs the tile's start and flushes all its stream rows, so a range keeps >= 32
// constraints (cfg2's 8-constraint symmetric tiles: 0.13 -> 0.30 ms split 3 ways).
static uint32_t tile_split(uint64_t ctas, uint64_t cons_per_tile) {
    const char* fe = getenv("FSMT_TILE_SPLIT");   // A/B and the parity matrix (read per launch)
    const int forced = fe ? atoi(fe) : 0;
    if (forced > 0) return (uint32_t)std::min(forced, 64);
    const uint64_t target = 148ull * 28 * 4;
    if (ctas == 0 || ctas >= target) return 1;
    const uint64_t by_size = std::max<uint64_t>(1, cons_per_tile / 32);
    return (uint32_t)std::min<uint64_t>(std::min<uint64_t>(8, by_size), (target + ctas - 1) / ctas);
}

void launch_sweep_jit(cudaKernel_t k, const DevFormula& F, const DevState& S, const DevTiles& T, float kappa,
                      double* terms, uint32_t terms_r, cudaStream_t st, const DevSlots* D) {
    if (T.n_tiles == 0 || S.R == 0) return;
    const int kVmax = (int)T.vmax, kVtot = (int)(T.vmax + T.rmax);    // Plan::vmax, Plan::rmax
    // one one-warp CTA per (tile, 32 restarts)
    const uint64_t rtiles = (S.R + 31) / 32;
    uint32_t nsplit = tile_split((uint64_t)T.n_tiles * rtiles, T.cons_per_tile);
    const unsigned blocks = (unsigned)((uint64_t)T.n_tiles * rtiles * nsplit);
    const size_t smem = (size_t)T.ring_uint4 * 16 + (size_t)kVmax * 32 * 4 + (size_t)kVtot * T.vid_bytes;   // ring | rows | ids
    if (smem > 48 * 1024) cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    uint32_t n_tiles = T.n_tiles, R = S.R, n_bool = F.n_bool;
    const float* kdev = S.ds ? &S.ds->kappa : nullptr;
    const uint16_t* U = S.U;
    const float* PT = D ? D->PT : nullptr;
    double* GU = D ? D->GU : nullptr;
    void* args[] = {(void*)&T.tiles, &n_tiles, (void*)&T.recs, (void*)&T.tile_vars, (void*)&S.a, (void*)&S.b,
                    (void*)&S.ga, (void*)&S.gb, (void*)&U, (void*)&S.obj, &R, &n_bool, &kappa,
                    &terms, &terms_r, (void*)&F.orig, (void*)&PT, (void*)&GU, (void*)&S.fx, (void*)&kdev, &nsplit};
    cudaLaunchKernel((const void*)k, dim3(blocks), dim3(32), args, smem, st);
}

void launch_slot_prob(cudaKernel_t k, const DevFormula& F, const DevState& S, const DevSlots& D, float kappa, cudaStream_t st) {
    uint32_t n_bool = F.n_bool, nv = D.nv, n_sa = D.n_sa, R = S.R;
    const uint64_t n = (uint64_t)(n_bool + n_sa) * R;
    if (!n) return;
    const float* kdev = S.ds ? &S.ds->kappa : nullptr;
    void* args[] = {&n_bool, &nv, &n_sa, (void*)&D.atoms, (void*)&S.a, (void*)&S.b, (void*)&F.atom_rowptr,
                    (void*)&F.atom_col, (void*)&F.atom_val, (void*)&F.atom_rhs, (void*)&F.atom_invnorm, &R, &kappa,
                    (void*)&D.PT, (void*)&D.DD, (void*)&kdev};
    cudaLaunchKernel((const void*)k, dim3((unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16)), dim3(256), args, 0, st);
}

void launch_slot_chain(cudaKernel_t k, const DevFormula& F, const DevState& S, const DevSlots& D, cudaStream_t st) {
    uint32_t n_bool = F.n_bool, nv = D.nv, n_sa = D.n_sa, R = S.R;
    if (!R) return;
    void* args[] = {&n_bool, &nv, &n_sa, (void*)&D.atoms, (void*)&F.atom_rowptr, (void*)&F.atom_col, (void*)&F.atom_val,
                    &R, (void*)&D.GU, (void*)&D.DD, (void*)&S.ga, (void*)&S.gb};
    const uint64_t n = ((uint64_t)n_bool + n_sa) * R;
    cudaLaunchKernel((const void*)k, dim3((unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148ull * 16))), dim3(256),
                     args, 0, st);
}

void launch_slot_truth(cudaKernel_t k, const DevFormula& F, const DevState& S, const DevSlots& D, const int8_t* x,
                       const float* y, cudaStream_t st) {
    uint32_t n_bool = F.n_bool, nv = D.nv, n_sa = D.n_sa, R = S.R;
    const uint64_t n = (uint64_t)(n_bool + n_sa) * R;
    if (!n) return;
    void* args[] = {&n_bool, &nv, &n_sa, (void*)&D.atoms, (void*)&x, (void*)&y, (void*)&F.atom_rowptr, (void*)&F.atom_col,
                    (void*)&F.atom_val64, (void*)&F.atom_rhs64, (void*)&F.atom_strict, &R, (void*)&D.TT};
    cudaLaunchKernel((const void*)k, dim3((unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16)), dim3(256), args, 0, st);
}

void launch_verify_jit(cudaKernel_t k, const DevFormula& F, const DevState& S, const DevTiles& T, const int8_t* x,
                       const float* y, uint16_t* U_update, uint8_t* per_con, cudaStream_t st, const uint8_t* TT) {
    if (T.n_tiles == 0 || S.R == 0) return;
    const int vtot = (int)(T.vmax + T.rmax);
    uint32_t nsplit = tile_split((uint64_t)T.n_tiles * ((S.R + 31) / 32), T.cons_per_tile);
    const unsigned blocks = (unsigned)((uint64_t)T.n_tiles * ((S.R + 31) / 32) * nsplit);   // one warp per (tile range, 32 restarts)
    const size_t smem = (size_t)vtot * 4;
    uint32_t n_tiles = T.n_tiles, R = S.R, n_bool = F.n_bool;
    uint32_t* unsat = S.unsat;
    void* args[] = {(void*)&T.tiles, &n_tiles, (void*)&T.recs, (void*)&T.vrecs, (void*)&T.tile_vars, (void*)&x,
                    (void*)&y, (void*)&U_update, (void*)&unsat, (void*)&per_con, (void*)&F.orig, &R, &n_bool,
                    (void*)&F.atom_rowptr, (void*)&F.atom_val64, (void*)&F.atom_rhs64, (void*)&F.atom_strict, (void*)&TT,
                    (void*)&S.umax, (void*)&S.flags, &nsplit};
    cudaLaunchKernel((const void*)k, dim3(blocks), dim3(32), args, smem, st);
}

void launch_prologue(const DevFormula& F, const DevState& S, float kappa, int et_int, float wfrac, double* gu, uint64_t gu_rows,
                     cudaStream_t st) {
    if (S.R == 0) return;
    const uint64_t n = ((uint64_t)F.n_bool + F.n_real + 1 + (gu ? gu_rows : 0)) * S.R;
    const unsigned blocks = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
    k1_prologue<<<blocks, 256, 0, st>>>(F, S, kappa, et_int, wfrac, gu, gu_rows);
}

void launch_scale_rows(double* dst, const double* src, const double* gsc, uint64_t rows, uint32_t R, cudaStream_t st) {
    const uint64_t n = rows * R;
    if (!n) return;
    k_scale_rows<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16), 256, 0, st>>>(dst, src, gsc, n, R);
}

void launch_umax(const DevFormula& F, const DevState& S, cudaStream_t st) {
    if (S.R == 0) return;
    k_umax<<<(S.R + 127) / 128, 128, 0, st>>>(S.U, F.n_cons, S.R, S.umax);
}

void launch_sweep(const DevFormula& F, const DevState& S, float kappa, double* terms, uint32_t terms_r, cudaStream_t st) {
    if (F.generic_end <= F.generic_begin || S.R == 0) return;
    const int warps = sweep_warps(F);
    const int smem = sweep_smem_bytes(F, warps);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k1_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    const uint64_t chunks = (F.generic_end - F.generic_begin + kChunk - 1) / kChunk;
    const uint64_t nw = chunks * ((S.R + 31) / 32);
    const uint64_t blocks = (nw + warps - 1) / warps;
    k1_sweep<<<(unsigned)blocks, warps * 32, smem, st>>>(F, S, kappa, terms, terms_r,
                                                         std::max<int>(1, F.max_slots), std::max<int>(1, F.max_nodes));
}

// variables per part of the gradient-mapping norm: at most 64, and few enough that the grid of
// (restart blocks x parts) has >= 8 blocks per SM (cfg4 at R = 1,024: 72 -> 64; cfg2: 2)
static uint32_t vars_per_part(const DevFormula& F, uint32_t R) {
    const uint32_t nv = F.n_bool + F.n_real;
    const uint32_t rblocks = R >= 128 ? (R + 127) / 128 : 1;
    const uint32_t want_parts = std::max<uint32_t>(1, (148u * 8u + rblocks - 1) / rblocks);
    return std::max<uint32_t>(1, std::min<uint32_t>((uint32_t)kVarsPerPart, (nv + want_parts - 1) / want_parts));
}
int update_parts(const DevFormula& F, uint32_t R) {
    const uint32_t vpp = vars_per_part(F, R);
    return (int)((F.n_bool + F.n_real + vpp - 1) / vpp);
}

void launch_update(const DevFormula& F, const DevState& S, float eta, float eps, cudaStream_t st, float eta_b) {
    if (!(eta_b > 0.f)) eta_b = eta;
    const uint32_t parts = (uint32_t)update_parts(F, S.R);
    if (parts == 0 || S.R == 0) return;
    DevState Sp = S;
    if (F.proj_iters && F.n_half && S.bn) {       // Prop.1 with halfspaces (R33): candidate + Dykstra
        const uint64_t n = (uint64_t)F.n_real * S.R;
        k3_cand<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16), 256, 0, st>>>(F, S, eta_b);
        launch_project(F, S, S.bn, true, st);
    } else {
        Sp.bn = nullptr;
    }
    const uint32_t tpb = S.R >= 128 ? 128u : 32u * ((S.R + 31) / 32);
    dim3 g1((S.R + tpb - 1) / tpb, parts);
    k3_norm<<<g1, tpb, 0, st>>>(F, Sp, eta, eta_b, vars_per_part(F, S.R));
    if (S.R >= 512 && parts <= 256) k3_final<<<(S.R + 127) / 128, 128, 0, st>>>(S, parts, eps);
    else k3_final_block<<<S.R, 256, 0, st>>>(S, parts, eps);   // few restarts or many parts: a block per restart
    const uint64_t n = (uint64_t)(F.n_bool + F.n_real) * S.R;
    const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, 148ull * 16);
    k3_apply<<<(unsigned)blocks, 256, 0, st>>>(F, Sp, eta, eta_b);
}

size_t project_smem_bytes(const DevFormula& F, uint32_t nnz) { return ((size_t)2 * F.n_hvars + nnz) * 4; }

void launch_project(const DevFormula& F, const DevState& S, float* X, bool skip_frozen, cudaStream_t st) {
    if (!F.proj_iters || !F.n_half || S.R == 0) return;
    const size_t smem = project_smem_bytes(F, F.h_nnz);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_dykstra, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_dykstra<<<S.R, 128, smem, st>>>(F, S, X, skip_frozen);
}

__global__ void k_best_flag(uint32_t R, const uint32_t* __restrict__ um, uint32_t* __restrict__ ub, uint8_t* __restrict__ flag,
                            uint32_t m) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R) return;
    const bool better = m == 0 || um[r] < ub[r];
    flag[r] = better;
    if (better) ub[r] = um[r];
}

__global__ void k_copy_cols(uint64_t n, uint32_t R, const int8_t* __restrict__ x, int8_t* __restrict__ xb,
                            const uint8_t* __restrict__ flag) {
    for (uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (uint64_t)gridDim.x * blockDim.x)
        if (flag[idx % R]) xb[idx] = x[idx];
}

// ---------------------------------------------------------------- device-side solve loop (Alg.2)

// Top of a stage: its parameters from the schedule (entry t - 1).
__global__ void k_stage_begin(const DevSolve* __restrict__ sv, const DevStage* __restrict__ sched, DevStage* __restrict__ ds) {
    if (threadIdx.x == 0) *ds = sched[sv->t - 1];
}

// End of a stage (Alg.2 P:526-528 and the lock-step winner rule of fsmt_solve): the restart with the
// fewest violated constraints (the lowest index among equals); when it beats the best so far its
// rounded model (x[:, r], y = b[:, r]) is kept; the loop continues while no restart is SAT and
// stages remain in this launch.  One block.
__global__ void __launch_bounds__(1024) k_stage_best(DevSolve* __restrict__ sv, DevState S, uint32_t n_bool, uint32_t n_real,
                                                     int8_t* __restrict__ xk, float* __restrict__ yk,
                                                     cudaGraphConditionalHandle h) {
    __shared__ unsigned long long red[32];
    __shared__ int improved;
    unsigned long long key = ~0ull;
    for (uint32_t r = threadIdx.x; r < S.R; r += blockDim.x) {
        const unsigned long long k = ((unsigned long long)S.unsat[r] << 32) | r;
        key = k < key ? k : key;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long v = __shfl_down_sync(0xffffffffu, key, o);
        key = v < key ? v : key;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = key;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (uint32_t w = 1; w < (blockDim.x + 31) / 32; ++w) key = red[w] < key ? red[w] : key;
        red[0] = key;
        const uint32_t u = (uint32_t)(key >> 32);
        improved = u < sv->best_unsat;
        if (improved) {
            sv->best_unsat = u;
            sv->best_stage = sv->t;
            sv->best_r = (uint32_t)(key & 0xffffffffu);
        }
    }
    __syncthreads();
    if (improved) {
        const uint32_t r = (uint32_t)(red[0] & 0xffffffffu);
        for (uint32_t i = threadIdx.x; i < n_bool; i += blockDim.x) xk[i] = S.x[(size_t)i * S.R + r];
        for (uint32_t j = threadIdx.x; j < n_real; j += blockDim.x) yk[j] = S.b[(size_t)j * S.R + r];
    }
    if (threadIdx.x == 0) {
        const uint32_t t = sv->t + 1;
        sv->t = t;
        sv->done = sv->best_unsat == 0 || t > sv->t_end;
        cudaGraphSetConditional(h, sv->done ? 0u : 1u);
    }
}

void launch_stage_begin(const DevSolve* sv, const DevStage* sched, DevStage* ds, cudaStream_t st) {
    k_stage_begin<<<1, 32, 0, st>>>(sv, sched, ds);
}

void launch_stage_best(DevSolve* sv, const DevState& S, uint32_t n_bool, uint32_t n_real, int8_t* xk, float* yk,
                       cudaGraphConditionalHandle h, cudaStream_t st) {
    k_stage_best<<<1, 1024, 0, st>>>(sv, S, n_bool, n_real, xk, yk, h);
}

void launch_keep_best(const DevFormula& F, const DevState& S, const uint32_t* unsat_m, uint32_t* unsat_best,
                      int8_t* x_best, uint8_t* flag, uint32_t m, cudaStream_t st) {
    if (!S.R) return;
    k_best_flag<<<(S.R + 255) / 256, 256, 0, st>>>(S.R, unsat_m, unsat_best, flag, m);
    const uint64_t n = (uint64_t)F.n_bool * S.R;
    if (n) k_copy_cols<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 16), 256, 0, st>>>(n, S.R, S.x, x_best, flag);
}

void launch_round(const DevFormula& F, const DevState& S, uint32_t rounding, uint64_t seed, uint32_t off,
                  uint32_t stage, cudaStream_t st) {
    const uint64_t n = (uint64_t)F.n_bool * S.R;
    if (!n) return;
    const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, 148ull * 16);
    k4_round<<<(unsigned)blocks, 256, 0, st>>>(F, S, rounding, seed, off, stage);
}

void launch_verify(const DevFormula& F, const DevState& S, const int8_t* x, const float* y, uint16_t* U_update,
                   uint8_t* per_con, cudaStream_t st, uint32_t cb, uint32_t ce) {
    if (ce == UINT32_MAX) ce = F.n_cons;
    if (ce <= cb || S.R == 0) return;
    const uint64_t chunks = (ce - cb + kChunk - 1) / kChunk;
    const uint64_t nw = chunks * ((S.R + 31) / 32);
    const uint64_t blocks = (nw + 7) / 8;
    k5_verify<<<(unsigned)blocks, 256, 0, st>>>(F, S, x, y, U_update, per_con, cb, ce);
}

// ------------------------------------------------------------------------- C4 through the NVSwitch
// One-shot in-switch all-reduce of a multicast f64 buffer (fsmt_mc_allreduce_f64): each rank owns a
// contiguous slice; multimem.ld_reduce returns the sum over the ranks' copies (computed in the
// switch), multimem.st writes it to every rank's copy.  sm_90+ PTX; f64 has no vector form.
namespace {
__global__ void k_mc_allreduce_f64(double* __restrict__ mc, uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += (uint64_t)gridDim.x * blockDim.x) {
        double v;
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f64 %0, [%1];" : "=d"(v) : "l"(mc + i) : "memory");
        asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" ::"l"(mc + i), "d"(v) : "memory");
    }
}
}  // namespace

void launch_mc_allreduce_f64(double* mc, uint64_t n, uint32_t rank, uint32_t world, cudaStream_t st) {
    const uint64_t lo = n * rank / world, hi = n * (rank + 1) / world;
    if (hi <= lo) return;
    const uint64_t blocks = std::min<uint64_t>((hi - lo + 255) / 256, 148ull * 8);
    k_mc_allreduce_f64<<<(unsigned)blocks, 256, 0, st>>>(mc, lo, hi);
}

}  // namespace fsmt
