// Device work plan and the JIT-specialised sweep source (K1).
//
// Plan: every constraint gets a kernel class (template + nnz of each atom slot).  Variables
// are grouped by first appearance (a constraint's newly seen variables form one batch; a
// batch never straddles a group), each constraint is keyed by (kernel class, footprint
// groups) and the stable sort of these keys is the internal constraint order.  Each
// reference position of a class is "stream" (its variable changes from one constraint to
// the next most of the time) or "run".  Runs of one key become tiles of <= cmax constraints
// with <= vmax stream variables (one shared-memory accumulator row each, flushed once per
// tile) and <= rmax run variables (register accumulators, flushed once per run).
//
// JIT: for each hot kernel class the forward pass (Alg.F) and backward pass
// (Alg.B, sign R1) are emitted as straight-line code over the class's
// canonical xBDD, with messages in registers; slot probabilities follow Eq.4 / Eq.7 and the
// chain rule P:1326-1327.  Constraints of other classes run through the generic kernel.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <sstream>
#include <unordered_map>

#include "fsmt_internal.hpp"

namespace fsmt {

namespace {
constexpr uint32_t kJitMaxNodes = 96;
constexpr uint32_t kJitMaxRefs = 64;
constexpr uint32_t kJitMaxClasses = 32;
constexpr uint64_t kJitMinCons = 32;      // specialise only classes with enough constraints
constexpr uint64_t kJitMinConsSym = 1;    // symmetric classes: few (kind, L, k) classes, each worth specialising
constexpr uint32_t kCountMaxL = 64;       // count classes: q[0..L] in registers
constexpr uint32_t kJitMaxNodesSym = 160; // symmetric classes (messages only, no inline atom math)
constexpr uint32_t kSymMark = 0xFFFFFFF0u;
}  // namespace

int weight_exponent(const Built& b) {
    float m = 0.f;
    for (float w : b.cons_w) m = std::max(m, w);
    if (!(m > 0.f)) return 0;
    int e = 0;
    const float fr = std::frexp(m, &e);   // m = fr 2^e, fr in [1/2, 1)
    return fr == 0.5f ? e - 1 : e;
}

Plan make_plan(const Formula& f, const Built& b, bool enable_jit) {
    Plan p;
    p.wexp = weight_exponent(b);
    if (const char* v = getenv("FSMT_JIT_VID32")) p.vid32 = v[0] == '1';
    if (const char* v = getenv("FSMT_TILE_VMAX")) p.vmax = (uint32_t)std::max(16, std::min(256, atoi(v)));
    if (const char* v = getenv("FSMT_TILE_CMAX")) p.cmax = (uint32_t)std::max(1, std::min(1024, atoi(v)));
    if (const char* v = getenv("FSMT_TILE_RMAX")) p.rmax = (uint32_t)std::max(16, std::min(1024, atoi(v)));
    p.group = p.vmax;
    if (const char* v = getenv("FSMT_TILE_VMAX_SYM")) p.vmax_sym = (uint32_t)std::max(16, std::min(512, atoi(v)));
    if (const char* v = getenv("FSMT_TILE_GROUP")) p.group = (uint32_t)std::max(8, std::min(1024, atoi(v)));
    const uint32_t C = (uint32_t)b.cons_tmpl.size();
    // 1. kernel classes
    std::map<std::vector<uint32_t>, uint32_t> kc_of;
    std::vector<uint32_t> kcl(C);
    const char* sym_env = getenv("FSMT_JIT_SYM");        // "0": symmetric classes off (A/B)
    const bool sym_on = !(sym_env && sym_env[0] == '0');
    // a symmetric constraint reads its atoms through the slot tables only when they are shared
    // (each referenced by >= 2 constraints): unique atoms are cheaper inline
    std::vector<uint32_t> atom_refs(f.n_atoms(), 0);
    for (uint32_t c = 0; c < C; ++c) {
        const Template& t = b.tmpls[b.cons_tmpl[c]];
        for (size_t s = 0; s < t.kinds.size(); ++s)
            if (t.kinds[s] == 1) ++atom_refs[b.slot_ids[b.cons_slot_off[c] + s]];
    }
    auto sym_ok = [&](uint32_t c) {
        const Template& t = b.tmpls[b.cons_tmpl[c]];
        for (size_t s = 0; s < t.kinds.size(); ++s)
            if (t.kinds[s] == 1 && atom_refs[b.slot_ids[b.cons_slot_off[c] + s]] < 2) return false;
        return true;
    };
    for (uint32_t c = 0; c < C; ++c) {
        const Template& t = b.tmpls[b.cons_tmpl[c]];
        const uint32_t Ls = b.cons_slot_off[c + 1] - b.cons_slot_off[c];
        if (sym_on && b.cons_sym[c] && Ls >= 2 && sym_ok(c)) {
            const uint32_t kind = b.cons_sym[c] - 1u, kk = kind == 1 ? b.cons_k[c] : 0u;
            std::vector<uint32_t> key{kSymMark, kind, Ls, kk};
            auto it = kc_of.find(key);
            uint32_t k;
            if (it == kc_of.end()) {
                k = (uint32_t)p.kclasses.size();
                kc_of.emplace(key, k);
                KClass kc;
                kc.sym = true;
                kc.sym_kind = kind;
                kc.sym_L = Ls;
                kc.sym_k = kk;
                kc.stmpl = symmetric_template(kind, Ls, kk);
                kc.tmpl = UINT32_MAX;
                kc.n_refs = Ls;
                kc.words = 1 + (Ls + 1) / 2 + (Ls + 31) / 32;   // weight, slot refs, sign bits
                kc.stride4 = (kc.words + 3) / 4;
                kc.vstride4 = 1;
                // CARD over many literals (CARD(50, 25): 650 nodes) cannot keep its messages in registers:
                // its count distribution q[0..L] can (FSMT_JIT_COUNT=1: every CARD class, =0: none)
                const char* ce = getenv("FSMT_JIT_COUNT");
                const bool big = kc.stmpl.nodes.size() > kJitMaxNodesSym;
                kc.count = kind == K_CARD && Ls <= kCountMaxL && kc.stmpl.root >= 0 && kk < Ls &&
                           (ce ? ce[0] == '1' : big);
                const char* pe = getenv("FSMT_JIT_PROD");
                kc.prod = kind != K_CARD && Ls <= kCountMaxL && kc.stmpl.root >= 0 && !(pe && pe[0] == '0');
                kc.jit = enable_jit && (!big || kc.count || kc.prod) && Ls <= kJitMaxRefs && kc.stmpl.root >= 0;
                kc.n_cons = 0;
                p.kclasses.push_back(kc);
            } else {
                k = it->second;
            }
            kcl[c] = k;
            p.kclasses[k].n_cons++;
            continue;
        }
        std::vector<uint32_t> key{b.cons_tmpl[c]};
        const uint32_t* ids = b.slot_ids.data() + b.cons_slot_off[c];
        uint32_t refs = 0;
        for (size_t s = 0; s < t.kinds.size(); ++s) {
            if (t.kinds[s] == 0) {
                ++refs;
            } else {
                uint32_t nnz = f.atom_rowptr[ids[s] + 1] - f.atom_rowptr[ids[s]];
                key.push_back(nnz);
                refs += nnz;
            }
        }
        auto it = kc_of.find(key);
        uint32_t k;
        if (it == kc_of.end()) {
            k = (uint32_t)p.kclasses.size();
            kc_of.emplace(key, k);
            KClass kc;
            kc.tmpl = b.cons_tmpl[c];
            for (size_t i = 1; i < key.size(); ++i) kc.nnz.push_back((uint8_t)std::min<uint32_t>(key[i], 255));
            kc.n_refs = refs;
            uint32_t atom_words = 0;
            bool small_nnz = true;
            for (size_t i = 1; i < key.size(); ++i) {
                atom_words += 2 + key[i];
                small_nnz &= key[i] <= 8;
            }
            kc.words = 1 + (refs + 1) / 2 + atom_words;
            kc.stride4 = (kc.words + 3) / 4;
            kc.vstride4 = std::max<uint32_t>(1, ((uint32_t)(key.size() - 1) + 3) / 4);
            kc.jit = enable_jit && small_nnz && t.nodes.size() <= kJitMaxNodes && refs <= kJitMaxRefs && t.root >= 0;
            kc.n_cons = 0;
            p.kclasses.push_back(kc);
        } else {
            k = it->second;
        }
        kcl[c] = k;
        p.kclasses[k].n_cons++;
    }
    // keep the kJitMaxClasses heaviest JIT-able classes; renumber so JIT classes come first
    std::vector<uint32_t> idx(p.kclasses.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = (uint32_t)i;
    auto work = [&](uint32_t k) {
        const KClass& K = p.kclasses[k];
        return K.n_cons * (uint64_t)((K.sym ? K.stmpl : b.tmpls[K.tmpl]).nodes.size() + K.n_refs);
    };
    std::stable_sort(idx.begin(), idx.end(), [&](uint32_t x, uint32_t y) {
        if (p.kclasses[x].jit != p.kclasses[y].jit) return p.kclasses[x].jit;
        return work(x) > work(y);
    });
    uint32_t njit = 0;
    for (uint32_t k : idx)
        if (p.kclasses[k].jit && p.kclasses[k].n_cons < (p.kclasses[k].sym ? kJitMinConsSym : kJitMinCons))
            p.kclasses[k].jit = false;
    for (uint32_t k : idx)
        if (p.kclasses[k].jit) {
            if (njit < kJitMaxClasses) ++njit;
            else p.kclasses[k].jit = false;
        }
    std::stable_sort(idx.begin(), idx.end(), [&](uint32_t x, uint32_t y) {
        if (p.kclasses[x].jit != p.kclasses[y].jit) return p.kclasses[x].jit;
        return work(x) > work(y);
    });
    std::vector<uint32_t> ren(p.kclasses.size());
    std::vector<KClass> sorted;
    for (size_t i = 0; i < idx.size(); ++i) {
        ren[idx[i]] = (uint32_t)i;
        sorted.push_back(p.kclasses[idx[i]]);
    }
    p.kclasses.swap(sorted);
    for (uint32_t& k : kcl) k = ren[k];
    p.n_jit_kclasses = njit;

    // 1b. atoms read through the slot tables (symmetric JIT classes), by first appearance
    std::vector<int32_t> sym_row(f.n_atoms(), -1);
    for (uint32_t c = 0; c < C; ++c) {
        const KClass& K = p.kclasses[kcl[c]];
        if (!(K.sym && K.jit)) continue;
        p.has_sym = true;
        const Template& t = b.tmpls[b.cons_tmpl[c]];
        const uint32_t* ids = b.slot_ids.data() + b.cons_slot_off[c];
        for (size_t s = 0; s < t.kinds.size(); ++s)
            if (t.kinds[s] == 1 && sym_row[ids[s]] < 0) {
                sym_row[ids[s]] = (int32_t)p.sym_atoms.size();
                p.sym_atoms.push_back(ids[s]);
            }
    }

    // 2. footprint groups by first-appearance batches
    const uint32_t NV = f.n_bool + f.n_real;
    std::vector<uint32_t> group(NV + p.sym_atoms.size(), UINT32_MAX);
    uint32_t cur_group = 0, cur_size = 0;
    std::vector<uint32_t> batch;
    // variables of constraint c in reference order; a symmetric JIT class's references are its
    // slots' table rows (Boolean i -> i, table atom t -> NV + t)
    auto cons_vars = [&](uint32_t c, std::vector<uint32_t>& out) {
        out.clear();
        const Template& t = b.tmpls[b.cons_tmpl[c]];
        const uint32_t* ids = b.slot_ids.data() + b.cons_slot_off[c];
        const KClass& K = p.kclasses[kcl[c]];
        if (K.sym && K.jit) {
            for (size_t s = 0; s < t.kinds.size(); ++s) out.push_back(t.kinds[s] == 0 ? ids[s] : NV + (uint32_t)sym_row[ids[s]]);
            return;
        }
        for (size_t s = 0; s < t.kinds.size(); ++s) {
            if (t.kinds[s] == 0) out.push_back(ids[s]);
            else
                for (uint32_t k = f.atom_rowptr[ids[s]]; k < f.atom_rowptr[ids[s] + 1]; ++k)
                    out.push_back(f.n_bool + f.atom_col[k]);
        }
    };
    std::vector<uint32_t> vars;
    // stream-row budget from the typical constraint: 3x its distinct variables, in [40, 56]
    // (cfg4, 18 variables, best at 54; cfg3, 10 variables, best at 40), unless
    // FSMT_TILE_VMAX / FSMT_TILE_GROUP set it
    size_t typical_vars = 0;   // distinct variables of the most common (non-symmetric JIT) constraint
    if (!getenv("FSMT_TILE_VMAX") || !getenv("FSMT_TILE_MERGE")) {
        std::map<size_t, uint32_t> nvars;
        for (uint32_t c = 0; c < C; ++c) {
            const KClass& K = p.kclasses[kcl[c]];
            if (!K.jit || K.sym) continue;
            cons_vars(c, vars);
            std::sort(vars.begin(), vars.end());
            ++nvars[(size_t)(std::unique(vars.begin(), vars.end()) - vars.begin())];
        }
        size_t mode = 0;
        uint32_t best = 0;
        for (const auto& kv : nvars)
            if (kv.second > best) { best = kv.second; mode = kv.first; }
        typical_vars = mode;
        if (best && !getenv("FSMT_TILE_VMAX")) {
            p.vmax = (uint32_t)std::max<size_t>(40, std::min<size_t>(56, 3 * mode));
            if (!getenv("FSMT_TILE_GROUP")) p.group = p.vmax;
        }
    }
    for (uint32_t c = 0; c < C; ++c) {
        cons_vars(c, vars);
        batch.clear();
        for (uint32_t u : vars)
            if (group[u] == UINT32_MAX && std::find(batch.begin(), batch.end(), u) == batch.end()) batch.push_back(u);
        if (batch.empty()) continue;
        if (cur_size > 0 && cur_size + batch.size() > p.group) {
            ++cur_group;
            cur_size = 0;
        }
        for (uint32_t u : batch) group[u] = cur_group;
        cur_size += (uint32_t)batch.size();
    }
    // Tile merging (FSMT_TILE_MERGE=0/1 overrides): the stream side's group leads the sort key, and a
    // tile may span several keys that share it, within the row / run / constraint budgets (up to 256
    // run variables and 256 constraints), so the per-tile start and stream-row flush are amortised
    // over more constraints.  Default for formulas whose typical constraint has >= 16 variables
    // (cfg4 7.08 -> 6.58 ms, place9856 6.03 -> 4.98 ms; cfg3, 10 variables, 0.711 ->
    // 0.735 ms merged).
    const char* tm_env = getenv("FSMT_TILE_MERGE");
    const bool tile_merge = tm_env ? tm_env[0] == '1' : typical_vars >= 16;
    if (tile_merge && !getenv("FSMT_TILE_CMAX")) p.cmax = 256;
    if (tile_merge && !getenv("FSMT_TILE_RMAX")) p.rmax = 256;   // run ids are 2 B of shared memory each
    // 3. sort keys
    struct Key {
        uint32_t kc;
        uint32_t g[4];
    };
    std::vector<Key> keys(C);
    std::vector<uint32_t> gs;
    for (uint32_t c = 0; c < C; ++c) {
        cons_vars(c, vars);
        gs.clear();
        for (uint32_t u : vars) gs.push_back(group[u]);
        std::sort(gs.begin(), gs.end());
        gs.erase(std::unique(gs.begin(), gs.end()), gs.end());
        Key k{kcl[c], {UINT32_MAX, UINT32_MAX, UINT32_MAX, UINT32_MAX}};
        if (gs.size() <= 4) {
            for (size_t i = 0; i < gs.size(); ++i) k.g[i] = gs[i];
            // merge mode: the newest group (whose variables change fastest in first-appearance order:
            // the stream side) leads the key, so the blocks sharing a stream group are adjacent
            if (tile_merge && gs.size() > 1) std::rotate(k.g, k.g + gs.size() - 1, k.g + gs.size());
        } else {
            k.g[0] = UINT32_MAX - 1;          // wide footprint: keep original order
        }
        keys[c] = k;
    }
    p.order.resize(C);
    for (uint32_t c = 0; c < C; ++c) p.order[c] = c;
    std::stable_sort(p.order.begin(), p.order.end(), [&](uint32_t x, uint32_t y) {
        const Key &a = keys[x], &bb = keys[y];
        if (a.kc != bb.kc) return a.kc < bb.kc;
        return std::lexicographical_compare(a.g, a.g + 4, bb.g, bb.g + 4);
    });
    p.pos.resize(C);
    p.cons_kclass.resize(C);
    for (uint32_t i = 0; i < C; ++i) {
        p.pos[p.order[i]] = i;
        p.cons_kclass[i] = kcl[p.order[i]];
    }
    // 4. per JIT class and reference position (SURVEY §8(a) a4 accumulation):
    //    "stream" if the variable changes from one constraint to the next of the class in the
    //    internal order most of the time (accumulated straight into a shared-memory row),
    //    "run" otherwise (register accumulator, flushed with one fp64 atomic per run);
    //    aliases: reference r reads the same variable as an earlier reference in every
    //    constraint of the class (e.g. x_j in both separation atoms of a placement pair)
    std::vector<uint32_t> rv, pv;
    {
        std::vector<std::vector<uint64_t>> changes(p.n_jit_kclasses);
        std::vector<std::vector<uint8_t>> same(p.n_jit_kclasses);
        std::vector<uint64_t> seen(p.n_jit_kclasses, 0);
        for (uint32_t k = 0; k < p.n_jit_kclasses; ++k) {
            changes[k].assign(p.kclasses[k].n_refs, 0);
            same[k].assign((size_t)p.kclasses[k].n_refs * p.kclasses[k].n_refs, 1);
        }
        for (uint32_t i = 0; i < C && p.kclasses[p.cons_kclass[i]].jit; ++i) {
            const uint32_t k = p.cons_kclass[i];
            const uint32_t nr = p.kclasses[k].n_refs;
            cons_vars(p.order[i], rv);
            const bool has_prev = i > 0 && p.cons_kclass[i - 1] == k;
            if (has_prev) cons_vars(p.order[i - 1], pv);
            for (uint32_t r = 0; r < nr; ++r) changes[k][r] += !has_prev || rv[r] != pv[r];
            ++seen[k];
            std::vector<uint8_t>& sm = same[k];
            for (uint32_t r = 1; r < nr; ++r)
                for (uint32_t q = 0; q < r; ++q) sm[(size_t)r * nr + q] &= (uint8_t)(rv[r] == rv[q]);
        }
        const bool use_stream = true;   // stream-off (every reference in run mode) lost 32.8 vs 22.6 ms
        const char* ae = getenv("FSMT_JIT_ALIAS");
        const bool use_alias = !(ae && ae[0] == '0');
        for (uint32_t k = 0; k < p.n_jit_kclasses; ++k) {
            KClass& K = p.kclasses[k];
            K.stream.assign(K.n_refs, 0);
            K.alias.assign(K.n_refs, -1);
            for (uint32_t r = 0; r < K.n_refs; ++r) K.stream[r] = use_stream && seen[k] && 2 * changes[k][r] > seen[k];
            if (!use_alias || !seen[k]) continue;
            for (uint32_t r = 1; r < K.n_refs; ++r)
                for (uint32_t q = 0; q < r; ++q)
                    if (same[k][(size_t)r * K.n_refs + q] && K.alias[q] < 0) {
                        K.alias[r] = (int32_t)q;
                        K.stream[r] = K.stream[q];
                        break;
                    }
        }
    }

    // 4b. K5 record folding (see KClass::vfold)
    {
        const char* ve = getenv("FSMT_JIT_VFOLD");
        const bool von = !(ve && ve[0] == '0');
        std::vector<uint8_t> seen_k(p.n_jit_kclasses, 0);
        for (uint32_t k = 0; k < p.n_jit_kclasses; ++k) p.kclasses[k].vfold = von && !p.kclasses[k].sym;
        for (uint32_t i2 = 0; i2 < C && p.kclasses[p.cons_kclass[i2]].jit; ++i2) {
            KClass& K = p.kclasses[p.cons_kclass[i2]];
            if (!K.vfold) continue;
            const uint32_t c = p.order[i2];
            const Template& t = b.tmpls[K.tmpl];
            const uint32_t* ids = b.slot_ids.data() + b.cons_slot_off[c];
            std::vector<std::vector<double>> co;
            std::vector<uint8_t> st;
            for (size_t sl = 0; sl < t.kinds.size(); ++sl)
                if (t.kinds[sl] == 1) {
                    const uint32_t at = ids[sl];
                    co.emplace_back(f.atom_val.begin() + f.atom_rowptr[at], f.atom_val.begin() + f.atom_rowptr[at + 1]);
                    st.push_back(f.atom_strict[at]);
                }
            if (!seen_k[p.cons_kclass[i2]]) {
                seen_k[p.cons_kclass[i2]] = 1;
                K.vcoef = co;
                K.vstrict = st;
            } else if (co != K.vcoef || st != K.vstrict) {
                K.vfold = false;
            }
        }
        for (uint32_t k = 0; k < p.n_jit_kclasses; ++k) {
            KClass& K = p.kclasses[k];
            if (K.vfold) K.vstride4 = std::max<uint32_t>(1, (2 * (uint32_t)K.vcoef.size() + 3) / 4);
        }
    }

    // 5. tiles + records over the JIT prefix: a tile is a run of one sort key with <= cmax
    //    constraints, <= vmax stream variables (shared-memory rows) and <= rmax run variables;
    //    a reference's record field is its variable's index among the tile's stream or run
    //    variables
    uint32_t i = 0;
    std::vector<uint32_t> sloc, rloc, adds, addr;
    auto index_of = [](const std::vector<uint32_t>& v, uint32_t u) {
        return (uint32_t)(std::find(v.begin(), v.end(), u) - v.begin());
    };
    while (i < C && p.kclasses[p.cons_kclass[i]].jit) {
        const uint32_t kc = p.cons_kclass[i];
        const KClass& K = p.kclasses[kc];
        TileDesc T{kc, i, 0, (uint32_t)p.tile_vars.size(), 0, (uint32_t)(p.recs.size() / 4), 0,
                   (uint32_t)(p.vrecs.size() / 4)};
        sloc.clear();
        rloc.clear();
        const Key& k0 = keys[p.order[i]];
        while (i < C && p.cons_kclass[i] == kc && T.n_cons < p.cmax) {
            const Key& ki = keys[p.order[i]];
            if (T.n_cons > 0 && !tile_merge && (memcmp(ki.g, k0.g, sizeof(k0.g)) != 0)) break;
            cons_vars(p.order[i], vars);
            adds.clear();
            addr.clear();
            for (uint32_t r = 0; r < K.n_refs; ++r) {
                if (K.alias[r] >= 0) continue;
                const uint32_t u = vars[r];
                if (K.stream[r]) {
                    if (index_of(sloc, u) == sloc.size() && index_of(adds, u) == adds.size()) adds.push_back(u);
                } else if (index_of(rloc, u) == rloc.size() && index_of(addr, u) == addr.size()) {
                    addr.push_back(u);
                }
            }
            if (sloc.size() + adds.size() > (K.sym ? p.vmax_sym : p.vmax) || rloc.size() + addr.size() > p.rmax) break;
            sloc.insert(sloc.end(), adds.begin(), adds.end());
            rloc.insert(rloc.end(), addr.begin(), addr.end());
            // record
            const uint32_t c = p.order[i];
            if (K.sym) {
                // weight, one table-row ref per slot, then the slots' literal signs (1 = negated)
                std::vector<uint32_t> rec(K.stride4 * 4, 0);
                float w = std::ldexp(b.cons_w[c], -p.wexp);
                memcpy(&rec[0], &w, 4);
                const uint32_t L = K.n_refs, so = b.cons_slot_off[c];
                for (uint32_t r = 0; r < L; ++r) {
                    const uint32_t l = K.stream[r] ? index_of(sloc, vars[r]) : index_of(rloc, vars[r]);
                    rec[1 + r / 2] |= (l & 0xFFFFu) << (16 * (r % 2));
                    rec[1 + (L + 1) / 2 + r / 32] |= (uint32_t)(b.slot_neg[so + r] != 0) << (r % 32);
                }
                p.recs.insert(p.recs.end(), rec.begin(), rec.end());
                p.vrecs.insert(p.vrecs.end(), (size_t)K.vstride4 * 4, 0u);
                ++T.n_cons;
                ++i;
                continue;
            }
            const Template& t = b.tmpls[K.tmpl];
            const uint32_t* ids = b.slot_ids.data() + b.cons_slot_off[c];
            std::vector<uint32_t> rec(K.stride4 * 4, 0);
            float w = std::ldexp(b.cons_w[c], -p.wexp);
            memcpy(&rec[0], &w, 4);
            uint32_t ref = 0;
            auto put_ref = [&](uint32_t u) {
                const uint32_t tr = K.alias[ref] >= 0 ? (uint32_t)K.alias[ref] : ref;
                const uint32_t l = K.stream[tr] ? index_of(sloc, u) : index_of(rloc, u);
                rec[1 + ref / 2] |= (l & 0xFFFFu) << (16 * (ref % 2));
                ++ref;
            };
            uint32_t aw = 1 + (K.n_refs + 1) / 2;
            std::vector<uint32_t> vrec(K.vstride4 * 4, 0);   // K5 record: atom id per atom slot
            uint32_t va = 0;
            for (size_t s = 0; s < t.kinds.size(); ++s) {
                if (t.kinds[s] == 0) {
                    put_ref(ids[s]);
                } else {
                    uint32_t atom = ids[s];
                    if (K.vfold) {   // the atom's fp64 right-hand side (lo, hi words)
                        uint64_t bits;
                        memcpy(&bits, &f.atom_rhs[atom], 8);
                        vrec[va++] = (uint32_t)bits;
                        vrec[va++] = (uint32_t)(bits >> 32);
                    } else {
                        vrec[va++] = atom;
                    }
                    float rhs = (float)f.atom_rhs[atom];
                    double n2 = 0.0;
                    for (uint32_t kk = f.atom_rowptr[atom]; kk < f.atom_rowptr[atom + 1]; ++kk)
                        n2 += f.atom_val[kk] * f.atom_val[kk];
                    float inv = (float)(1.0 / std::sqrt(n2));
                    memcpy(&rec[aw], &rhs, 4);
                    memcpy(&rec[aw + 1], &inv, 4);
                    aw += 2;
                    for (uint32_t kk = f.atom_rowptr[atom]; kk < f.atom_rowptr[atom + 1]; ++kk) {
                        put_ref(f.n_bool + f.atom_col[kk]);
                        float q = (float)f.atom_val[kk];
                        memcpy(&rec[aw++], &q, 4);
                    }
                }
            }
            p.recs.insert(p.recs.end(), rec.begin(), rec.end());
            p.vrecs.insert(p.vrecs.end(), vrec.begin(), vrec.end());
            ++T.n_cons;
            ++i;
        }
        if (T.n_cons == 0) break;   // a single constraint over too many variables: rest is generic
        T.n_vars = (uint32_t)sloc.size() | ((uint32_t)rloc.size() << 16);
        T.pad0 = T.n_cons * K.stride4;
        p.tile_vars.insert(p.tile_vars.end(), sloc.begin(), sloc.end());
        p.tile_vars.insert(p.tile_vars.end(), rloc.begin(), rloc.end());
        p.tiles.push_back(T);
    }
    p.jit_cons_end = i;
    // any JIT-class constraints after the cut run through the generic kernel

    // 5c. affine reference groups (KClass::aff_head): from the tile records (local indices) and
    //     the constraints' variables, per class; a group's members must share the head's kind
    //     (Boolean / real / table row) and stream flag.  FSMT_JIT_AFFINE=0 disables.
    {
        const char* ae = getenv("FSMT_JIT_AFFINE");
        const bool on = !(ae && ae[0] == '0');
        std::vector<std::vector<uint8_t>> ok(p.n_jit_kclasses);
        std::vector<std::vector<int32_t>> dg(p.n_jit_kclasses), dl(p.n_jit_kclasses);
        std::vector<uint8_t> init(p.n_jit_kclasses, 0);
        std::vector<int> rkind;
        for (const TileDesc& T : p.tiles) {
            const KClass& K = p.kclasses[T.kclass];
            const uint32_t nr = K.n_refs;
            std::vector<uint8_t>& okk = ok[T.kclass];
            for (uint32_t c = 0; c < T.n_cons; ++c) {
                const uint32_t* rec = p.recs.data() + ((size_t)T.rec_off + (size_t)c * K.stride4) * 4;
                cons_vars(p.order[T.cons_begin + c], vars);
                auto lref = [&](uint32_t r) { return (int32_t)((rec[1 + r / 2] >> (16 * (r % 2))) & 0xFFFFu); };
                if (!init[T.kclass]) {
                    init[T.kclass] = 1;
                    okk.assign((size_t)nr * nr, 0);
                    dg[T.kclass].assign((size_t)nr * nr, 0);
                    dl[T.kclass].assign((size_t)nr * nr, 0);
                    for (uint32_t r = 1; r < nr; ++r)
                        for (uint32_t q = 0; q < r; ++q) {
                            okk[(size_t)r * nr + q] = 1;
                            dg[T.kclass][(size_t)r * nr + q] = (int32_t)vars[r] - (int32_t)vars[q];
                            dl[T.kclass][(size_t)r * nr + q] = lref(r) - lref(q);
                        }
                    continue;
                }
                for (uint32_t r = 1; r < nr; ++r)
                    for (uint32_t q = 0; q < r; ++q) {
                        const size_t ix = (size_t)r * nr + q;
                        if (okk[ix] && ((int32_t)vars[r] - (int32_t)vars[q] != dg[T.kclass][ix] || lref(r) - lref(q) != dl[T.kclass][ix]))
                            okk[ix] = 0;
                    }
            }
        }
        for (uint32_t k = 0; k < p.n_jit_kclasses; ++k) {
            KClass& K = p.kclasses[k];
            const uint32_t nr = K.n_refs;
            K.aff_head.assign(nr, -1);
            K.aff_dg.assign(nr, 0);
            K.aff_dl.assign(nr, 0);
            if (!on || !init[k]) continue;
            // reference kinds in reference order
            rkind.clear();
            const Template& t = K.sym ? K.stmpl : b.tmpls[K.tmpl];
            for (size_t sl = 0, ai = 0; sl < t.kinds.size(); ++sl) {
                if (t.kinds[sl] == 1) {
                    for (uint32_t z = 0; z < K.nnz[ai]; ++z) rkind.push_back(1);
                    ++ai;
                } else {
                    rkind.push_back(t.kinds[sl]);
                }
            }
            for (uint32_t r = 1; r < nr; ++r) {
                if (K.alias[r] >= 0) continue;
                for (uint32_t q = 0; q < r; ++q) {
                    if (K.alias[q] >= 0 || K.aff_head[q] >= 0) continue;
                    if (rkind[q] != rkind[r] || K.stream[q] != K.stream[r]) continue;
                    const size_t ix = (size_t)r * nr + q;
                    if (!ok[k][ix] || dl[k][ix] == 0) continue;
                    K.aff_head[r] = (int32_t)q;
                    K.aff_dg[r] = dg[k][ix];
                    K.aff_dl[r] = dl[k][ix];
                    break;
                }
            }
        }
    }

    // 6. record compression: words equal across a whole class become literals in the code
    // (FSMT_JIT_FOLD=0 disables; cfg4: 7 -> 4 uint4 per record, 13.7 vs 14.0 ms at vmax 48)
    const char* cz = getenv("FSMT_JIT_FOLD");
    const bool fold = !(cz && cz[0] == '0');
    std::vector<std::vector<uint8_t>> varies(p.n_jit_kclasses);
    std::vector<std::vector<uint32_t>> first(p.n_jit_kclasses);
    for (uint32_t k = 0; k < p.n_jit_kclasses; ++k) {
        varies[k].assign(p.kclasses[k].words, fold ? 0 : 1);
        first[k].assign(p.kclasses[k].words, 0);
    }
    // a reference word whose two references are both aliases or affine-group members is never read
    // (K1 and K5 address those from their target / group head): dropped like a constant word
    // (cfg4: 16 -> 8 words per record, half the record loads)
    std::vector<std::vector<uint8_t>> unread(p.n_jit_kclasses);
    for (uint32_t k = 0; k < p.n_jit_kclasses; ++k) {
        const KClass& K = p.kclasses[k];
        unread[k].assign(K.words, 0);
        if (!fold) continue;
        auto skipped = [&](uint32_t r) {
            return r >= K.n_refs || (r < K.alias.size() && K.alias[r] >= 0) || (r < K.aff_head.size() && K.aff_head[r] >= 0);
        };
        for (uint32_t r = 0; r < K.n_refs; r += 2)
            if (1 + r / 2 < K.words && skipped(r) && skipped(r + 1)) unread[k][1 + r / 2] = 1;
    }
    std::vector<uint8_t> have(p.n_jit_kclasses, 0);
    for (const TileDesc& T : p.tiles) {
        const KClass& K = p.kclasses[T.kclass];
        for (uint32_t c = 0; c < T.n_cons; ++c) {
            const uint32_t* rec = p.recs.data() + ((size_t)T.rec_off + (size_t)c * K.stride4) * 4;
            if (!have[T.kclass]) {
                for (uint32_t w = 0; w < K.words; ++w) first[T.kclass][w] = rec[w];
                have[T.kclass] = 1;
            }
            for (uint32_t w = 0; w < K.words; ++w) varies[T.kclass][w] |= rec[w] != first[T.kclass][w];
        }
    }
    std::vector<uint32_t> old_stride(p.n_jit_kclasses);
    for (uint32_t k = 0; k < p.n_jit_kclasses; ++k) {
        KClass& K = p.kclasses[k];
        old_stride[k] = K.stride4;
        K.wpos.assign(K.words, -1);
        K.wconst = first[k];
        int32_t n = 0;
        for (uint32_t w = 0; w < K.words; ++w)
            if (varies[k][w] && !unread[k][w]) K.wpos[w] = n++;
        K.stride4 = std::max<uint32_t>(1, ((uint32_t)n + 3) / 4);
    }
    std::vector<uint32_t> packed;
    packed.reserve(p.recs.size());
    for (TileDesc& T : p.tiles) {
        const KClass& K = p.kclasses[T.kclass];
        const uint32_t os = old_stride[T.kclass];
        const uint32_t new_off = (uint32_t)(packed.size() / 4);
        for (uint32_t c = 0; c < T.n_cons; ++c) {
            const uint32_t* rec = p.recs.data() + ((size_t)T.rec_off + (size_t)c * os) * 4;
            std::vector<uint32_t> out(K.stride4 * 4, 0);
            for (uint32_t w = 0; w < K.words; ++w)
                if (K.wpos[w] >= 0) out[(size_t)K.wpos[w]] = rec[w];
            packed.insert(packed.end(), out.begin(), out.end());
        }
        T.rec_off = new_off;
        T.pad0 = T.n_cons * K.stride4;
    }
    p.recs.swap(packed);
    // two spare records (of the widest class) after the last: the sweep copies the records two
    // constraints ahead without a bounds test (the values read past a tile are never used)
    p.recs.insert(p.recs.end(), (size_t)p.ring_uint4() * 4, 0u);
    // each JIT class's tiles are contiguous (the internal order sorts by class first)
    p.class_tile_begin.assign(p.n_jit_kclasses + 1, (uint32_t)p.tiles.size());
    for (uint32_t t = (uint32_t)p.tiles.size(); t-- > 0;) p.class_tile_begin[p.tiles[t].kclass] = t;
    for (uint32_t k = p.n_jit_kclasses; k-- > 0;) p.class_tile_begin[k] = std::min(p.class_tile_begin[k], p.class_tile_begin[k + 1]);
    return p;
}

// ------------------------------------------------------------------------------ codegen

namespace {

std::string fnum(float v) {
    char buf[64];
    snprintf(buf, sizeof(buf), "%.9gf", v);
    return buf;
}

// FSMT_JIT_PAIR=0: atoms one at a time on the scalar FP32 pipe instead of in pairs on the
// packed f32x2 pipe (A/B; both bit-identical).
bool jit_pair() {
    const char* e = getenv("FSMT_JIT_PAIR");
    return !(e && e[0] == '0');
}

// FSMT_JIT_UPF=d: the sweep loads U[c][r] d constraints ahead (0: in the iteration, plain load).
// Without the variable: g_upf (jit_source's argument; fsmt_prepare picks it from the size of U).
thread_local int g_upf = 0;   // per thread: contexts may build concurrently
thread_local bool g_all_small = false;   // every JIT class non-symmetric with <= 16 references (loop unroll)
int u_prefetch() {
    const char* e = getenv("FSMT_JIT_UPF");
    return e ? std::max(0, std::min(12, atoi(e))) : g_upf;
}

const char* kErfcPrelude =
    "// Per-restart scales of the sweep (kernels.hpp FxScale, written by k1_prologue; DESIGN.md §7\n"
    "// item 14): the ERWA weight w_c 2^(U + e_t) (R18) is applied as fp32 w_c' 2^(U - s_r) (s_r =\n"
    "// max(0, max_c U - 24), so no fp32 weight overflows), and every fp32 partial sum is flushed as\n"
    "// the integer rint(v 2^frac(e_t) 2^-G_r) into the fp64 gradient: integer sums below 2^53 are exact, so the\n"
    "// atomics' order does not matter (deterministic, sharding-invariant); the consumers multiply by\n"
    "// the restart's grid scale 2^(G_r + s_r + weight and stage exponents).\n"
    "struct FxScale { double gs, ti, oi, os; float gif; int ebias; };\n"
    "// v on the grid, in grid units: rintf(v gif), gif = 2^frac(e_t) 2^-G (fp32 values >= 2^23 are integers)\n"
    "__device__ __forceinline__ double fsmt_q(float v, float gif) { return (double)rintf(v * gif); }\n"
    "// w0 * 2^(u + ebias - 127) exactly (a power of two times w0; 0 below 2^-126, never inf: u + ebias <= 151)\n"
    "__device__ __forceinline__ float fsmt_w(float w0, u32 u, int ebias) {\n"
    "  return w0 * __uint_as_float((u32)max((int)u + ebias, 0) << 23);\n"
    "}\n"
    "// fsmt_prepare(R): the module compiled with FSMT_RC = R takes the restart count as a constant,\n"
    "// so every [var][R] row offset (k * 4R bytes) folds into the load's immediate offset.  The\n"
    "// launcher uses that module only for a state of exactly R restarts.\n"
    "#ifdef FSMT_RC\n"
    "#define FSMT_SPECIALISE_R R = FSMT_RC;\n"
    "#else\n"
    "#define FSMT_SPECIALISE_R\n"
    "#endif\n"
    "#define FSMT_AT(base, off) (*(const float*)((const char*)(base) + (off)))\n"
    "// 16-byte asynchronous global -> shared copy (the sweep's record ring)\n"
    "__device__ __forceinline__ void fsmt_cpa16(uint4* dst, const uint4* src) {\n"
    "  asm volatile(\"cp.async.ca.shared.global [%0], [%1], 16;\" :: \"r\"((u32)__cvta_generic_to_shared(dst)), \"l\"(__cvta_generic_to_global(src)) : \"memory\");\n"
    "}\n"
    "__device__ __forceinline__ void fsmt_cpa_commit() { asm volatile(\"cp.async.commit_group;\" ::: \"memory\"); }\n"
    "template <int N> __device__ __forceinline__ void fsmt_cpa_wait() { asm volatile(\"cp.async.wait_group %0;\" :: \"n\"(N) : \"memory\"); }\n"
    "__device__ __forceinline__ float fsmt_rcp(float x) { float r; asm(\"rcp.approx.ftz.f32 %0, %1;\" : \"=f\"(r) : \"f\"(x)); return r; }\n"
    "__device__ __forceinline__ float fsmt_ex2(float x) { float r; asm(\"ex2.approx.ftz.f32 %0, %1;\" : \"=f\"(r) : \"f\"(x)); return r; }\n"
    "// 0.5*erfc(z) for z >= 0 and ez = exp(-z^2) (dd/db factor, P:1326-1327).  Coefficients from\n"
    "// scripts/fit_erfc.py: z < 0.75: 0.5 (1 - z P(z^2)), P ~ erf(z)/z (degree 5);\n"
    "// z >= 0.75: t Q(t) ez, t = 1/(1 + z/2), Q ~ 0.5 erfcx(z)/t (degree 7), reusing ez.\n"
    "// Max abs error 5.3e-8 in fp32 (with exact exp).\n"
    "__device__ __forceinline__ float fsmt_half_erfc(float z, float& ez) {\n"
    "  const float z2 = z * z;\n"
    "  ez = fsmt_ex2(-1.44269504088896341f * z2);\n"
    "  float p = -3.380429407e-04f;   // 0.5 P (exact halving of the fitted coefficients)\n"
    "  p = fmaf(p, z2, 2.5579733775e-03f); p = fmaf(p, z2, -1.3417707755e-02f); p = fmaf(p, z2, 5.64169623e-02f);\n"
    "  p = fmaf(p, z2, -1.880631e-01f); p = fmaf(p, z2, 5.641895535e-01f);\n"
    "  const float small = fmaf(-z, p, 0.5f);\n"
    "  float t;   // 1/(1 + z/2) with 1 + z/2 >= 1: rcp.approx needs no denormal range fix-up\n"
    "  asm(\"rcp.approx.ftz.f32 %0, %1;\" : \"=f\"(t) : \"f\"(fmaf(0.5f, z, 1.f)));\n"
    "  float q = 4.469624162e-02f;\n"
    "  q = fmaf(q, t, -1.088827997e-01f); q = fmaf(q, t, 3.824992850e-02f); q = fmaf(q, t, 3.101851977e-02f);\n"
    "  q = fmaf(q, t, 8.971593529e-02f); q = fmaf(q, t, 1.233071312e-01f); q = fmaf(q, t, 1.410502791e-01f);\n"
    "  q = fmaf(q, t, 1.410473883e-01f);\n"
    "  const float tail = t * q * ez;\n"
    "  return z < 0.75f ? small : tail;\n"
    "}\n"
    "// Two atoms at once on the packed fp32x2 pipe (FFMA2/FMUL2, sm_100): per component exactly\n"
    "// the operations of fsmt_half_erfc (each f32x2 lane rounds like the scalar op), so the\n"
    "// result is bit-identical while the issue count of the polynomial halves.\n"
    "#define FSMT_C2(v) make_float2(v, v)\n"
    "__device__ __forceinline__ float2 fsmt_half_erfc2(float2 z, float2& ez) {\n"
    "  const float2 z2 = __fmul2_rn(z, z);\n"
    "  const float2 ea = __fmul2_rn(FSMT_C2(-1.44269504088896341f), z2);\n"
    "  ez = make_float2(fsmt_ex2(ea.x), fsmt_ex2(ea.y));\n"
    "  float2 p = FSMT_C2(-3.380429407e-04f);\n"
    "  p = __ffma2_rn(p, z2, FSMT_C2(2.5579733775e-03f)); p = __ffma2_rn(p, z2, FSMT_C2(-1.3417707755e-02f));\n"
    "  p = __ffma2_rn(p, z2, FSMT_C2(5.64169623e-02f)); p = __ffma2_rn(p, z2, FSMT_C2(-1.880631e-01f));\n"
    "  p = __ffma2_rn(p, z2, FSMT_C2(5.641895535e-01f));\n"
    "  const float2 small = __ffma2_rn(make_float2(-z.x, -z.y), p, FSMT_C2(0.5f));\n"
    "  const float2 den = __ffma2_rn(FSMT_C2(0.5f), z, FSMT_C2(1.f));\n"
    "  float2 t;\n"
    "  asm(\"rcp.approx.ftz.f32 %0, %1;\" : \"=f\"(t.x) : \"f\"(den.x));\n"
    "  asm(\"rcp.approx.ftz.f32 %0, %1;\" : \"=f\"(t.y) : \"f\"(den.y));\n"
    "  float2 q = FSMT_C2(4.469624162e-02f);\n"
    "  q = __ffma2_rn(q, t, FSMT_C2(-1.088827997e-01f)); q = __ffma2_rn(q, t, FSMT_C2(3.824992850e-02f));\n"
    "  q = __ffma2_rn(q, t, FSMT_C2(3.101851977e-02f)); q = __ffma2_rn(q, t, FSMT_C2(8.971593529e-02f));\n"
    "  q = __ffma2_rn(q, t, FSMT_C2(1.233071312e-01f)); q = __ffma2_rn(q, t, FSMT_C2(1.410502791e-01f));\n"
    "  q = __ffma2_rn(q, t, FSMT_C2(1.410473883e-01f));\n"
    "  const float2 tail = __fmul2_rn(__fmul2_rn(t, q), ez);\n"
    "  return make_float2(z.x < 0.75f ? small.x : tail.x, z.y < 0.75f ? small.y : tail.y);\n"
    "}\n\n";

const char* comp(uint32_t w) {
    static const char* c[] = {"x", "y", "z", "w"};
    return c[w % 4];
}

// Record word w of the class being emitted (g_wk): a register of the loaded (compressed)
// record, or a literal when the word is constant over the class (record compression).
thread_local const KClass* g_wk = nullptr;
std::string word(uint32_t w) {
    if (g_wk && w < g_wk->wpos.size()) {
        const int32_t p = g_wk->wpos[w];
        if (p < 0) return "(" + std::to_string(g_wk->wconst[w]) + "u)";
        return "q" + std::to_string(p / 4) + "." + comp((uint32_t)p);
    }
    return "q" + std::to_string(w / 4) + "." + comp(w);
}

void emit_class(std::ostringstream& o, uint32_t kid, const KClass& K, const Template& t) {
    g_wk = &K;
    const std::string TY = "float", ZR = "0.f", AT = "FSMT_AT";
    const size_t ns = t.kinds.size();
    // DBG = false (the hot instantiation): U present, no per-constraint E_c debug output, so
    // neither test is in the loop
    o << "template <bool DBG> __device__ __forceinline__ void kc" << kid
      << "(const TileDesc& T, const uint4* __restrict__ rp, const VID* __restrict__ vs, const VID* __restrict__ vr,\n"
         "    " << TY << "* __restrict__ accs, const float* __restrict__ ab, const float* __restrict__ bb,\n"
         "    double* __restrict__ ga, double* __restrict__ gb, const unsigned short* __restrict__ U,\n"
         "    u32 R, u32 R4, u64 rr, u32 r, bool live, u32 n_bool, float kq, float dcoef, int ebias,\n"
         "    float gif, float& objacc,\n"
         "    double* __restrict__ terms, u32 terms_r, const u32* __restrict__ orig,\n"
         "    const float* __restrict__ PTl, double* __restrict__ gu,\n"
         "    uint4* __restrict__ rring, u32 lane) {\n"
         "  const bool hasU = !DBG || U != nullptr, hasT = DBG && terms != nullptr;\n";
    // refs
    std::vector<int> ref_kind;      // 0 Boolean, 1 real, 2 slot-table row (symmetric classes)
    std::vector<int> slot_ref0(ns);
    for (size_t s = 0, ai = 0; s < ns; ++s) {
        slot_ref0[s] = (int)ref_kind.size();
        if (t.kinds[s] == 0 || t.kinds[s] == 2) {
            ref_kind.push_back(t.kinds[s]);
        } else {
            const uint32_t nz = K.nnz[ai++];
            for (uint32_t k = 0; k < nz; ++k) ref_kind.push_back(1);
        }
    }
    const size_t nr = ref_kind.size();
    auto is_stream = [&](size_t i) { return i < K.stream.size() && K.stream[i]; };
    auto alias_of = [&](size_t i) -> int {   // target reference of an alias, -1 if i is its own
        return i < K.alias.size() ? K.alias[i] : -1;
    };
    auto head_of = [&](size_t i) -> int {   // affine group head (-1: i is a head or ungrouped)
        return i < K.aff_head.size() ? K.aff_head[i] : -1;
    };
    std::vector<std::vector<size_t>> members(nr);
    for (size_t i = 0; i < nr; ++i)
        if (alias_of(i) < 0 && head_of(i) >= 0) members[(size_t)head_of(i)].push_back(i);
    const std::string I = "";
    for (size_t i = 0; i < nr; ++i) {
        if (is_stream(i) || alias_of(i) >= 0) continue;
        if (head_of(i) < 0) o << "  u32 cur" << i << " = 0xffffffffu, gcur" << i << " = 0u;";
        o << " " << TY << " val" << i << " = " << ZR << ", acc" << i << " = " << ZR
          << ";\n";
    }
    // value of reference i at byte offset `off` of its column base: Booleans in a (ab), reals
    // by unified id in b (bb), table rows in PT / PF (PTl / PFl)
    auto ld_at = [&](size_t i, const std::string& off, const std::string& px = "") {
        const std::string is = std::to_string(i);
        if (ref_kind[i] == 2) return px + "val" + is + " = FSMT_AT(PTl, " + off + ");";   // p_true of the row; p_false = 1 - p_true
        return px + "val" + is + " = " + AT + "(" + (ref_kind[i] == 0 ? "ab" : "bb") + ", " + off + ");";
    };
    auto dgoff = [&](size_t m) { return "(u64)(" + std::to_string(K.aff_dg[m]) + " * (long long)R4)"; };
    // a run group's flush: one address for the head, the members at constant row offsets from it
    // (dg * R elements: an immediate in the R-specialised module)
    auto flush_group = [&](size_t i) {
        const std::string g = "gcur" + std::to_string(i);
        const std::string base = ref_kind[i] == 0 ? "ga + (u64)" + g + " * R + r"
                               : ref_kind[i] == 2 ? "gu + (u64)" + g + " * R + r"
                                                  : "gb + (u64)(" + g + " - n_bool) * R + r";
        std::string c = "if (live) { double* gp = " + base + "; atomicAdd(gp, fsmt_q(acc" + std::to_string(i) + ", gif));";
        for (size_t m : members[i])
            c += " atomicAdd(gp + (long long)(" + std::to_string(K.aff_dg[m]) + ") * R, fsmt_q(acc" + std::to_string(m) + ", gif));";
        return c + " }";
    };
    // ERWA counters: a byte load per constraint, issued u_prefetch() constraints ahead so its
    // DRAM latency overlaps the passes of the current constraints
    const int upf = u_prefetch();
    const char* uld = "__ldg";
    const std::string ucast = "";
    // (U has kUPad spare rows after the last constraint, so the look-ahead loads need no bounds
    // test; the values read past the tile are never used; one running pointer, no index math)
    if (upf > 0) {
        o << "  const unsigned short* Up = hasU ? U + (u64)T.cons_begin * R + rr : nullptr;\n";
        for (int k = 0; k < upf; ++k)
            o << "  u32 un" << k << " = hasU ? (u32)" << uld << "(" << ucast << "(Up + (u64)" << k << "u * R)) : 0u;\n";
        o << "  const unsigned short* Upf = hasU ? Up + (u64)" << upf << "u * R : nullptr;\n";
    }
    // Software pipeline over the constraints (FSMT_JIT_VPF=0 disables; DESIGN.md §7 item 18): the
    // record is loaded one constraint ahead, and from it the stream references' values of the NEXT
    // constraint are loaded during this one, so their L2 latency hides behind a whole iteration
    // (ncu v18: the record load and then the value loads were the top long-scoreboard stalls; the
    // record look-ahead alone measured neutral).  The plan keeps a spare record after the last, so
    // the look-ahead load needs no bounds test; past a tile's end the look-ahead row is the current one.
    const char* vpf_env = getenv("FSMT_JIT_VPF");
    size_t n_stream_vals = 0;   // registers the value look-ahead holds (stream heads + members)
    for (size_t i = 0; i < nr; ++i) n_stream_vals += is_stream(i) && alias_of(i) < 0;
    const char* vmx_env = getenv("FSMT_JIT_VPF_MAX");
    // (classes with more look-ahead values than this keep the in-iteration loads: their registers are
    // scarcer than the latency; random family n = 500 1.52 -> 1.43 ms, cfg2 0.138 -> 0.134)
    const size_t vpf_max = vmx_env ? (size_t)std::max(0, atoi(vmx_env)) : 32;
    const bool vpf = !(vpf_env && vpf_env[0] == '0') && n_stream_vals <= vpf_max;
    const bool rpf = vpf;
    auto nword = [&](uint32_t w) { const std::string x = word(w); return x[0] == 'q' ? "n" + x : x; };
    // next-constraint stream values: psl (local index) and pval per stream head and member
    auto stream_prefetch = [&](const std::string& ind, bool decl, bool guarded) {
        for (size_t i = 0; i < nr; ++i) {
            if (!is_stream(i) || alias_of(i) >= 0 || head_of(i) >= 0) continue;
            const std::string is = std::to_string(i);
            const std::string ext = "(" + nword(1 + (uint32_t)i / 2) + " >> " + std::to_string(16 * (i % 2)) + ") & 0xffffu";
            // past the tile's last constraint the look-ahead record is another tile's: the current row
            // again (a row of this reference's kind, so the address stays inside its array)
            o << ind << (decl ? "u32 " : "") << "psl" << is << " = " << (guarded ? "c + 1u < T.n_cons ? " : "") << "(" << ext << ")"
              << (guarded ? " : psl" + is : std::string()) << ";\n";
            o << ind << "{ const u64 pso = (u64)vs[psl" << is << "] * R4; " << ld_at(i, "pso", "p");
            for (size_t m : members[i]) o << " " << ld_at(m, "pso + " + dgoff(m), "p");
            o << " }\n";
        }
    };
    // The records travel through a two-slot shared-memory ring (cp.async by lanes < stride, record
    // c + 2 issued in iteration c, waited for at the top of iteration c + 1): the wait is explicit, so
    // the compiler cannot hoist the record's move into the uniform datapath right behind its load
    // (ncu v19: with the look-ahead in registers, 27 % of the stall samples sat on that R2UR).
    const uint32_t S4 = K.stride4;
    // FSMT_JIT_RALL=1: every lane copies every chunk (identical bytes to the same address), so its own
    // wait suffices and no __syncwarp is needed (A/B)
    const char* rall_env = getenv("FSMT_JIT_RALL");
    const bool rall = rall_env && rall_env[0] == '1';
    auto cpy = [&](const std::string& ind, const std::string& dst, const std::string& src) {
        if (rall)
            for (uint32_t q = 0; q < S4; ++q) o << ind << "fsmt_cpa16(" << dst << " + " << q << "u, " << src << " + " << q << "u);\n";
        else
            o << ind << "if (lane < " << S4 << "u) fsmt_cpa16(" << dst << " + lane, " << src << " + lane);\n";
    };
    if (rpf) {
        cpy("  ", "rring", "rp");
        o << "  fsmt_cpa_commit();\n";
        cpy("  ", "rring + " + std::to_string(S4) + "u", "rp + " + std::to_string(S4) + "u");
        o << "  fsmt_cpa_commit();\n  fsmt_cpa_wait<1>();\n" << (rall ? "" : "  __syncwarp();\n");
        for (uint32_t q = 0; q < S4; ++q) o << "  uint4 nq" << q << " = rring[" << q << "];\n";
    }
    if (vpf) {
        for (size_t i = 0; i < nr; ++i)
            if (is_stream(i) && alias_of(i) < 0)
                o << "  " << TY << " pval" << i << ";\n";
        stream_prefetch("  ", true, false);
    }
    // the constraint loop unrolled twice for small classes (FSMT_JIT_UNROLL overrides; DESIGN.md §9:
    // round 1 cfg3 0.884 -> 0.849 ms, cfg4 8.36 -> 8.33 ms; 4 is slower on cfg4); emitted right
    // before the loop (after the look-ahead prologue)
    std::string unroll_pragma;
    {
        // round 2: with the exact flush, the 22-reference placement class is faster not unrolled (cfg4
        // 8.08 vs 8.42 ms) while the 12-reference scheduling class keeps unroll 2 (cfg3 0.774 vs 0.864 ms)
        const char* ur = getenv("FSMT_JIT_UNROLL");
        // v21: with the value look-ahead, unroll 2 also for the placement class (no register-rotation
        // moves: cfg4 7.41 -> 7.12 ms at 80 registers); symmetric classes and classes without it keep
        // the round-2 rule (cfg2 0.133 vs 0.157 ms, random family n = 100 0.121 vs 0.131 ms unrolled)
        // v24: when every class is small and non-symmetric (<= 16 references: they share the all-class
        // kernel's registers), unroll 4 (cfg3 0.733 -> 0.694 ms; a heavy class beside an unrolled small
        // one lost its register cap on cfg4, 6.54 -> 6.72 ms)
        const int def_unroll = K.n_refs <= 16 ? (g_all_small ? 4 : 2) : (vpf && !K.sym ? 2 : 1);
        unroll_pragma = "#pragma unroll " + std::to_string(ur ? std::max(1, atoi(ur)) : def_unroll) + "\n";
    }
    o << unroll_pragma << "  for (u32 c = 0; c < T.n_cons; ++c, rp += " << K.stride4 << ") {\n";
    if (rpf) {
        for (uint32_t q = 0; q < S4; ++q) o << "    const uint4 q" << q << " = nq" << q << ";\n";
        o << "    fsmt_cpa_wait<0>();\n" << (rall ? "" : "    __syncwarp();\n");   // record c + 1 has landed in slot (c + 1) & 1
        for (uint32_t q = 0; q < S4; ++q) o << "    nq" << q << " = rring[((c + 1u) & 1u) * " << S4 << "u + " << q << "u];\n";
        cpy("    ", "rring + (c & 1u) * " + std::to_string(S4) + "u", "rp + " + std::to_string(2 * S4) + "u");
        o << "    fsmt_cpa_commit();\n";
    } else {
        for (uint32_t q = 0; q < S4; ++q) o << "    const uint4 q" << q << " = __ldg(rp + " << q << ");\n";
    }
    if (upf > 0) {
        o << "    const u32 uc = un0;\n";
        for (int k = 0; k + 1 < upf; ++k) o << "    un" << k << " = un" << k + 1 << ";\n";
        o << "    if (hasU) { un" << upf - 1 << " = (u32)" << uld << "(" << ucast << "Upf); Upf += R; }\n";
    } else {
        o << "    const u32 uc = hasU ? (u32)U[(u64)(T.cons_begin + c) * R + rr] : 0u;\n";
    }
    // w_c' 2^(U - s_r) (R18 with the restart's shift; 2^frac(e_t) is applied in the flush: FxScale)
    o << "    const float w = fsmt_w(__uint_as_float(" << word(0) << "), uc, ebias);\n";
    for (size_t i = 0; i < nr; ++i) {
        uint32_t wd = 1 + (uint32_t)i / 2;
        const std::string ext = "(" + word(wd) + " >> " + std::to_string(16 * (i % 2)) + ") & 0xffffu";
        if (alias_of(i) >= 0) {
            o << "    const " << TY << " val" << i << " = val" << alias_of(i) << ";   // alias\n";
            continue;
        }
        if (head_of(i) >= 0) continue;   // loaded with its group head
        if (is_stream(i) && vpf) {   // loaded during the previous constraint
            o << "    const u32 sl" << i << " = psl" << i << ";\n    const " << TY << " val" << i << " = pval" << i
              << ";\n";
            for (size_t m : members[i])
                o << "    const " << TY << " val" << m << " = pval" << m
                  << ";\n";
        } else if (is_stream(i)) {
            // stream reference: new variable (almost) every constraint; no run register
            o << "    const u32 sl" << i << " = " << ext << ";\n"
              << "    const u64 so" << i << " = (u64)vs[sl" << i << "] * R4;\n";
            o << "    " << TY << " val" << i << "; " << ld_at(i, "so" + std::to_string(i)) << "\n";
            for (size_t m : members[i])
                o << "    " << TY << " val" << m << "; "
                  << ld_at(m, "so" + std::to_string(i) + " + " + dgoff(m)) << "   // affine\n";
        } else {
            o << "    { const u32 l = " << ext << "; if (l != cur" << i << ") { if (cur" << i << " != 0xffffffffu) { "
              << flush_group(i);
            o << " } cur" << i << " = l; gcur" << i << " = vr[l]; acc" << i << " = " << ZR << "; ";
            o << ld_at(i, "(u64)gcur" + std::to_string(i) + " * R4");
            for (size_t m : members[i]) o << " acc" << m << " = " << ZR << "; " << ld_at(m, "(u64)gcur" + std::to_string(i) + " * R4 + " + dgoff(m));
            o << " } }\n";
        }
    }
    if (vpf) stream_prefetch("    ", false, true);
    // slot probabilities
    uint32_t aw = 1 + ((uint32_t)nr + 1) / 2;
    std::vector<uint32_t> coef_word(nr, 0);
    const uint32_t sign_word = 1 + ((uint32_t)nr + 1) / 2;   // symmetric classes: literal signs
    // atom pairs for the packed f32x2 pipe: consecutive atom slots with equal nnz and equal
    // class-constant status of 1/||q|| (their words are consecutive in the record)
    std::vector<int> pair_with(ns, -1), pair_second(ns, 0);
    if (jit_pair()) {
        int pend = -1;
        uint32_t awp = 1 + ((uint32_t)nr + 1) / 2, pend_aw = 0;
        for (size_t s = 0, ai = 0; s < ns; ++s) {
            if (t.kinds[s] != 1) continue;
            const uint32_t nz = K.nnz[ai];
            const bool ic = K.wpos[awp + 1] < 0;
            if (pend >= 0 && K.nnz[ai - 1] == nz && (K.wpos[pend_aw + 1] < 0) == ic) {
                pair_with[(size_t)pend] = (int)s;
                pair_second[s] = 1;
                pend = -1;
            } else {
                pend = (int)s;
                pend_aw = awp;
            }
            awp += 2 + nz;
            ++ai;
        }
    }
    for (size_t s = 0, ai = 0; s < ns; ++s) {
        if (t.kinds[s] == 1 && pair_second[s]) {   // emitted with its partner
            aw += 2 + K.nnz[ai++];
            continue;
        }
        if (t.kinds[s] == 1 && pair_with[s] >= 0) {
            const size_t b = (size_t)pair_with[s];
            const uint32_t nnz = K.nnz[ai++], awb = aw + 2 + nnz;
            const std::string sa = std::to_string(s), sb = std::to_string(b);
            o << "    float2 zp" << sa << " = make_float2(-__uint_as_float(" << word(aw) << "), -__uint_as_float(" << word(awb) << "));\n";
            o << "    const float inv" << sa << " = __uint_as_float(" << word(aw + 1) << "), inv" << sb << " = __uint_as_float("
              << word(awb + 1) << ");\n";
            for (uint32_t k = 0; k < nnz; ++k) {
                coef_word[slot_ref0[s] + k] = aw + 2 + k;
                coef_word[slot_ref0[b] + k] = awb + 2 + k;
                o << "    zp" << sa << " = __ffma2_rn(make_float2(__uint_as_float(" << word(aw + 2 + k) << "), __uint_as_float("
                  << word(awb + 2 + k) << ")), make_float2(val" << slot_ref0[s] + k << ", val" << slot_ref0[b] + k << "), zp" << sa << ");\n";
            }
            if (K.wpos[aw + 1] < 0)
                o << "    const float2 up" << sa << " = __fmul2_rn(zp" << sa << ", make_float2(kq * inv" << sa << ", kq * inv" << sb << "));\n";
            else
                o << "    const float2 up" << sa << " = __fmul2_rn(__fmul2_rn(FSMT_C2(kq), zp" << sa << "), make_float2(inv" << sa
                  << ", inv" << sb << "));\n";
            o << "    const float u" << sa << " = up" << sa << ".x, u" << sb << " = up" << sa << ".y;\n"
              << "    float2 ezp" << sa << ";\n"
              << "    const float2 ep" << sa << " = fsmt_half_erfc2(make_float2(fabsf(u" << sa << "), fabsf(u" << sb << ")), ezp" << sa << ");\n"
              << "    const float2 omp" << sa << " = __fadd2_rn(FSMT_C2(1.f), make_float2(-ep" << sa << ".x, -ep" << sa << ".y));\n"
              << "    const float pt" << sa << " = u" << sa << " >= 0.f ? ep" << sa << ".x : omp" << sa << ".x;\n"
              << "    const float pf" << sa << " = u" << sa << " >= 0.f ? omp" << sa << ".x : ep" << sa << ".x;\n"
              << "    const float pt" << sb << " = u" << sb << " >= 0.f ? ep" << sa << ".y : omp" << sa << ".y;\n"
              << "    const float pf" << sb << " = u" << sb << " >= 0.f ? omp" << sa << ".y : ep" << sa << ".y;\n"
              << "    const float2 ddp" << sa << " = __fmul2_rn(make_float2(dcoef * inv" << sa << ", dcoef * inv" << sb << "), ezp" << sa << ");\n";
            aw += 2 + nnz;
            continue;
        }
        if (t.kinds[s] == 0) {
            o << "    const " << TY << " pt" << s << " = 0.5f * (1.f - val" << slot_ref0[s] << "), pf" << s << " = 0.5f * (1.f + val"
              << slot_ref0[s] << ");\n";
        } else if (t.kinds[s] == 2) {
            // negated literal: p_true and p_false of its row swap (Eq.4 / Eq.7 of the literal); the
            // tables hold p_true only, p_false = 1 - p_true (one load and one register per literal)
            const int ri = slot_ref0[s];
            o << "    const bool sg" << s << " = (" << word(sign_word + (uint32_t)s / 32) << " >> " << s % 32 << ") & 1u;\n"
              << "    const float qf" << s << " = 1.f - val" << ri << ";\n"
              << "    const float pt" << s << " = sg" << s << " ? qf" << s << " : val" << ri << ", pf" << s << " = sg" << s
              << " ? val" << ri << " : qf" << s << ";\n";
        } else {
            const uint32_t nnz = K.nnz[ai++];
            o << "    float z" << s << " = -__uint_as_float(" << word(aw) << ");\n";
            o << "    const float inv" << s << " = __uint_as_float(" << word(aw + 1) << ");\n";
            for (uint32_t k = 0; k < nnz; ++k) {
                coef_word[slot_ref0[s] + k] = aw + 2 + k;
                o << "    z" << s << " = fmaf(__uint_as_float(" << word(aw + 2 + k) << "), val" << slot_ref0[s] + k << ", z" << s << ");\n";
            }
            aw += 2 + nnz;
            // inv class-constant (folded): kappa/sqrt2 * inv and the dd factor are loop-invariant
            const bool inv_const = K.wpos[aw - 2 - nnz + 1] < 0;
            if (inv_const)
                o << "    const " << TY << " u" << s << " = z" << s << " * (kq * inv" << s << ");\n";
            else
                o << "    const " << TY << " u" << s << " = kq * z" << s << " * inv" << s << ";\n";
            o << "    float ez" << s << ";\n    const float e" << s << " = fsmt_half_erfc(fabsf(u" << s << "), ez" << s << ");\n";
            o << "    const float pt" << s << " = u" << s << " >= 0.f ? e" << s << " : 1.f - e" << s << ";\n"
              << "    const float pf" << s << " = u" << s << " >= 0.f ? 1.f - e" << s << " : e" << s << ";\n"
              << "    const float dd" << s << " = (dcoef * inv" << s << ") * ez" << s << ";\n";
        }
    }
    // XOR diamonds (peephole, FSMT_JIT_DIAMOND=0 disables): node n at slot s whose children h, l
    // sit at one slot s', have n as their only parent, and cross (hi(h) = lo(l) = X, lo(h) =
    // hi(l) = Y).  Then n reaches X with P_X = pt_s pt_s' + pf_s pf_s' (s, s' equal) and Y with
    // 1 - P_X, so h and l need no messages of their own:
    //   forward  m[X] += P_X m[n], m[Y] += (1 - P_X) m[n]
    //   backward d = m_bu[X] - m_bu[Y], m_bu[n] = m_bu[Y] + P_X d,
    //            dCOP/dpt_s += m[n] d (pt_s' - pf_s'), dCOP/dpt_s' += m[n] d (pt_s - pf_s)
    // which is Alg.F/Alg.B over n, h, l regrouped (P_X + P_Y = 1).  For two Boolean slots
    // P_X = (1 + v_s v_s')/2 and pt - pf = -v.
    // (A count class has no node passes: nn = 0 and the count DP below sets pT and G.)
    const size_t nn = (K.count || K.prod) ? 0 : t.nodes.size();
    std::vector<int> indeg(nn, 0);
    for (size_t v = 0; v < nn; ++v) {
        if (t.nodes[v].hi >= 0) ++indeg[t.nodes[v].hi];
        if (t.nodes[v].lo >= 0) ++indeg[t.nodes[v].lo];
    }
    if (t.root >= 0 && nn) ++indeg[t.root];
    std::vector<char> dhead(nn, 0), dskip(nn, 0);
    const char* dm_env = getenv("FSMT_JIT_DIAMOND");
    if (!(dm_env && dm_env[0] == '0')) {
        for (size_t v = 0; v < nn; ++v) {
            const TNode& nd = t.nodes[v];
            if (dskip[v] || nd.hi < 0 || nd.lo < 0 || nd.hi == nd.lo) continue;
            const TNode& h = t.nodes[nd.hi];
            const TNode& l = t.nodes[nd.lo];
            if (h.level != l.level || indeg[nd.hi] != 1 || indeg[nd.lo] != 1) continue;
            if (h.hi != l.lo || h.lo != l.hi || h.hi == h.lo) continue;
            dhead[v] = 1;
            dskip[nd.hi] = dskip[nd.lo] = 1;
        }
    }
    auto is_bool = [&](uint32_t lv) { return t.kinds[lv] == 0; };
    auto vref = [&](uint32_t lv) { return "val" + std::to_string(slot_ref0[lv]); };
    // Boolean x Boolean diamonds' P_X / P_Y two at a time on the f32x2 pipe (FSMT_JIT_PAIR=0:
    // one at a time inside the forward pass); per component the same operations
    std::vector<char> dpre(nn, 0);
    if (jit_pair()) {
        std::vector<size_t> bb;
        for (size_t v = 0; v < nn; ++v)
            if (dhead[v] && is_bool(t.nodes[v].level) && is_bool(t.nodes[t.nodes[v].hi].level)) bb.push_back(v);
        for (size_t k = 0; k + 1 < bb.size(); k += 2) {
            const size_t va = bb[k], vb = bb[k + 1];
            const std::string a = std::to_string(va), b2 = std::to_string(vb);
            const uint32_t a1 = t.nodes[va].level, a2 = t.nodes[t.nodes[va].hi].level;
            const uint32_t b1 = t.nodes[vb].level, b22 = t.nodes[t.nodes[vb].hi].level;
            o << "    const float2 vvp" << a << " = __fmul2_rn(make_float2(" << vref(a1) << ", " << vref(b1) << "), make_float2("
              << vref(a2) << ", " << vref(b22) << "));\n"
              << "    const float2 PXp" << a << " = __ffma2_rn(FSMT_C2(0.5f), vvp" << a << ", FSMT_C2(0.5f));\n"
              << "    const float2 PYp" << a << " = __ffma2_rn(FSMT_C2(-0.5f), vvp" << a << ", FSMT_C2(0.5f));\n"
              << "    const " << TY << " PX" << a << " = PXp" << a << ".x, PY" << a << " = PYp" << a << ".x, PX" << b2 << " = PXp" << a
              << ".y, PY" << b2 << " = PYp" << a << ".y;\n";
            dpre[va] = dpre[vb] = 1;
        }
    }
    // forward pass (Alg.F): m_td in registers.  Mass conservation: every node's outgoing
    // probabilities sum to 1 (pt + pf = 1, P_X + P_Y = 1), so the two terminals' masses sum to
    // m_root = 1 and only the terminal with fewer incoming edges is accumulated; when that is
    // FALSE, E = 1 - 2 P(TRUE) = 2 P(FALSE) - 1 (cfg4: 11 of 12 edges reach TRUE).  A message's
    // first contribution is a plain product (no fmaf with a zero addend).
    size_t f_true = 0, f_false = 0;
    for (size_t v = 0; v < nn; ++v) {
        if (dskip[v]) continue;
        const TNode& nd = t.nodes[v];
        const int c1 = dhead[v] ? t.nodes[nd.hi].hi : nd.hi, c2 = dhead[v] ? t.nodes[nd.hi].lo : nd.lo;
        for (int ch : {c1, c2}) {
            f_true += ch == kTrue;
            f_false += ch == kFalse;
        }
    }
    const bool massF = nn > 0 && f_false < f_true;
    const std::string PTERM = massF ? "pF" : "pT";
    const int ptgt = massF ? kFalse : kTrue;
    for (size_t v = 0; v < nn; ++v)
        if (!dskip[v]) o << "    " << TY << " m" << v << " = " << ((int)v == t.root ? "1.f" : ZR) << ";\n";
    o << "    " << TY << " pT = " << ZR << (massF ? ", pF = 0.f" : "") << ";\n";
    std::vector<char> mset(nn + 1, 0);   // message (or, at index nn, the terminal sum) already assigned
    if (t.root >= 0 && (size_t)t.root < nn) mset[(size_t)t.root] = 1;
    for (size_t v = 0; v < nn; ++v) {
        if (dskip[v]) continue;
        const TNode& nd = t.nodes[v];
        auto push = [&](int child, const std::string& pn) {
            if (child < 0 && child != ptgt) return;
            const size_t slot = child >= 0 ? (size_t)child : nn;
            const std::string dst = child >= 0 ? "m" + std::to_string(child) : PTERM;
            const std::string src = (int)v == t.root ? std::string() : " * m" + std::to_string(v);
            if (!mset[slot]) o << "    " << dst << " = " << pn << src << ";\n";
            else o << "    " << dst << " = fmaf(" << pn << ", m" << v << ", " << dst << ");\n";
            mset[slot] = 1;
        };
        if (dhead[v]) {
            const TNode& h = t.nodes[nd.hi];
            const uint32_t s1 = nd.level, s2 = h.level;
            const std::string P = "PX" + std::to_string(v), Q = "PY" + std::to_string(v);
            if (dpre[v]) {
                // P_X / P_Y computed in pairs above
            } else if (is_bool(s1) && is_bool(s2)) {
                o << "    const " << TY << " vv" << v << " = " << vref(s1) << " * " << vref(s2) << ";\n"
                  << "    const " << TY << " " << P << " = fmaf(0.5f, vv" << v << ", 0.5f), " << Q << " = fmaf(-0.5f, vv" << v
                  << ", 0.5f);\n";
            } else {
                o << "    const " << TY << " " << P << " = fmaf(pt" << s1 << ", pt" << s2 << ", pf" << s1 << " * pf" << s2 << "), " << Q
                  << " = fmaf(pt" << s1 << ", pf" << s2 << ", pf" << s1 << " * pt" << s2 << ");\n";
            }
            push(h.hi, P);   // X: s, s' equal
            push(h.lo, Q);   // Y
            continue;
        }
        push(nd.hi, "pt" + std::to_string(nd.level));
        push(nd.lo, "pf" + std::to_string(nd.level));
    }
    // backward pass (Alg.B, sign R1): m_bu in registers, dE/dv per slot.  Complement form
    // (FSMT_JIT_CMP=0 disables): when more edges reach TRUE than FALSE, the pass
    // carries
    // c[v] = 1 - m_bu[v] (the same linear recurrence with the terminal values swapped,
    // using p + (1 - p) = 1), so the OR-chains' "1 - m_bu" subtractions vanish; then
    // G_s = -dCOP/dp_s and every use of G takes the sign back (gref).
    size_t e_true = 0, e_false = 0;
    for (size_t v = 0; v < nn; ++v) {
        if (dskip[v]) continue;
        for (int ch : {t.nodes[v].hi, t.nodes[v].lo}) {
            e_true += ch == kTrue;
            e_false += ch == kFalse;
        }
    }
    const char* cmp_env = getenv("FSMT_JIT_CMP");
    const bool cmp = !(cmp_env && cmp_env[0] == '0') && e_true > e_false;
    // Weight-seeded backward pass (xBDD classes): Alg.B is linear in the terminal values, so
    // seeding the non-zero terminal with the constraint weight w instead of 1 yields w m_bu and
    // w dCOP/dp directly; a Boolean slot's product terms then add straight into its accumulator
    // (one FFMA each) instead of G = a b followed by acc += w G (DESIGN.md §7 item 18).
    const bool wseed = nn > 0;
    const std::string ONE = wseed ? "w" : "1.f";
    for (size_t s = 0; s < ns; ++s) o << "    " << TY << " G" << s << " = " << ZR << ";\n";
    // G_s = sum of product terms a * b, collected here and emitted after the pass (first term a
    // plain product, then fmaf in the pass's order) unless folded into the accumulation
    std::vector<std::vector<std::pair<std::string, std::string>>> gt(ns);
    auto gfma = [&](size_t s, const std::string& a, const std::string& b) { gt[s].emplace_back(a, b); };
    auto gadd = [&](size_t s, const std::string& a, bool neg) { gt[s].emplace_back(neg ? "(-" + a + ")" : a, "1.f"); };
    auto bu = [&](int child) -> std::string {
        if (child >= 0) return "bu" + std::to_string(child);
        return (child == kTrue) != cmp ? ONE : "0.f";
    };
    for (size_t vv = nn; vv-- > 0;) {
        if (dskip[vv]) continue;
        const TNode& nd = t.nodes[vv];
        if (dhead[vv]) {
            const TNode& h = t.nodes[nd.hi];
            const uint32_t s1 = nd.level, s2 = h.level;
            const std::string X = bu(h.hi), Y = bu(h.lo), sv = std::to_string(vv);
            if (Y == "0.f")
                o << "    const " << TY << " d" << sv << " = " << X << ";\n"
                  << "    const " << TY << " bu" << sv << " = PX" << sv << " * d" << sv << ";\n";
            else
                o << "    const " << TY << " d" << sv << " = " << X << " - " << Y << ";\n"
                  << "    const " << TY << " bu" << sv << " = fmaf(PX" << sv << ", d" << sv << ", " << Y << ");\n";
            o << "    const " << TY << " md" << sv << " = m" << sv << " * d" << sv << ";\n";
            if (is_bool(s1) && is_bool(s2)) {
                gfma(s1, "-md" + sv, vref(s2));
                gfma(s2, "-md" + sv, vref(s1));
            } else {
                gfma(s1, "md" + sv, "(pt" + std::to_string(s2) + " - pf" + std::to_string(s2) + ")");
                gfma(s2, "md" + sv, "(pt" + std::to_string(s1) + " - pf" + std::to_string(s1) + ")");
            }
            continue;
        }
        std::string bh = bu(nd.hi), bl = bu(nd.lo);
        std::string lv = std::to_string(nd.level);
        // m_bu[v] = p m_bu[hi] + (1-p) m_bu[lo]
        std::string val;
        const std::string wpt = wseed ? "w * pt" + lv : "pt" + lv, wpf = wseed ? "w * pf" + lv : "pf" + lv;
        if (bh == ONE && bl == "0.f") val = wpt;
        else if (bh == "0.f" && bl == ONE) val = wpf;
        else if (bh == ONE) val = "fmaf(pf" + lv + ", " + bl + ", " + wpt + ")";
        else if (bl == ONE) val = "fmaf(pt" + lv + ", " + bh + ", " + wpf + ")";
        else if (bh == "0.f") val = "pf" + lv + " * " + bl;
        else if (bl == "0.f") val = "pt" + lv + " * " + bh;
        else {
            // both children internal: d = m_bu[hi] - m_bu[lo]; m_bu[v] = m_bu[lo] + p d (p + (1-p) = 1),
            // and d is reused by the gradient term below
            o << "    const " << TY << " d" << vv << " = " << bh << " - " << bl << ";\n";
            o << "    const " << TY << " bu" << vv << " = fmaf(pt" << lv << ", d" << vv << ", " << bl << ");\n";
            gfma(nd.level, "m" + std::to_string(vv), "d" + std::to_string(vv));
            continue;
        }
        o << "    const " << TY << " bu" << vv << " = " << val << ";\n";
        const std::string mv = "m" + std::to_string(vv);
        if (bh == ONE && bl == "0.f") wseed ? gfma(nd.level, mv, "w") : gadd(nd.level, mv, false);
        else if (bh == "0.f" && bl == ONE) wseed ? gfma(nd.level, mv, "(-w)") : gadd(nd.level, mv, true);
        else if (bl == "0.f") gfma(nd.level, mv, bh);
        else if (bh == "0.f") gfma(nd.level, mv, "(-" + bl + ")");
        else gfma(nd.level, mv, "(" + bh + " - " + bl + ")");
    }
    // symmetric (count / product) classes add each slot's gradient into its accumulator as soon as
    // it is formed, so the L gradients are never live together (registers: DESIGN.md §7 item 15)
    auto acc_dst = [&](size_t ri) -> std::string {
        if (!is_stream(ri)) return "acc" + std::to_string(ri);
        return head_of(ri) >= 0 ? "accs[(sl" + std::to_string(head_of(ri)) + " + " + std::to_string(K.aff_dl[ri]) + ") * 32]"
                                : "accs[sl" + std::to_string(ri) + " * 32]";
    };
    std::vector<char> g_inline(ns, 0);
    auto emit_inline_acc = [&](size_t s2, const std::string& ind) {
        const int ri0 = slot_ref0[s2];
        const size_t ri = (size_t)(alias_of((size_t)ri0) >= 0 ? alias_of((size_t)ri0) : ri0);
        const std::string d = acc_dst(ri), gs = "G" + std::to_string(s2), sg = "sg" + std::to_string(s2);
        o << ind << d << " = fmaf(w, " << sg << " ? -" << gs << " : " << gs << ", " << d << ");\n";
        g_inline[s2] = 1;
    };
    const bool sym_inline = (K.count || K.prod) && std::all_of(t.kinds.begin(), t.kinds.end(), [](int k) { return k == 2; });
    if (K.prod) {
        // OR / NAE / XOR over the L literals (pt_s = P(literal s true)): the COP in closed form and
        // dCOP/dpt_s from leave-one-out products, prefix products in registers times a running suffix:
        //   OR:  COP = 1 - prod pf,              G_s = prod_{j != s} pf_j
        //   NAE: COP = 1 - prod pt - prod pf,    G_s = prod_{j != s} pf_j - prod_{j != s} pt_j
        //   XOR: COP = (1 - prod d) / 2, d = pf - pt (E[(-1)^count]),  G_s = prod_{j != s} d_j
        // (pf_s = 1 - pt_s in the derivative; Eq.8 / Cor.1 for symmetric constraints)
        const uint32_t L = (uint32_t)ns, kind = K.sym_kind;
        auto S = [](uint32_t s) { return std::to_string(s); };
        if (kind == K_XOR)
            for (uint32_t s2 = 0; s2 < L; ++s2) o << "    const float xd" << s2 << " = pf" << s2 << " - pt" << s2 << ";\n";
        const std::string f1 = kind == K_XOR ? "xd" : "pf";          // the product every kind uses
        o << "    float ua0 = 1.f;";
        for (uint32_t s2 = 1; s2 <= L; ++s2) o << " const float ua" << s2 << " = ua" << s2 - 1 << (s2 == 1 ? "" : "") << " * " << f1 << S(s2 - 1) << ";";
        o << "\n";
        if (kind == K_NAE) {
            o << "    float va0 = 1.f;";
            for (uint32_t s2 = 1; s2 <= L; ++s2) o << " const float va" << s2 << " = va" << s2 - 1 << " * pt" << S(s2 - 1) << ";";
            o << "\n    pT = 1.f - ua" << L << " - va" << L << ";\n";
        } else if (kind == K_XOR) {
            o << "    pT = 0.5f * (1.f - ua" << L << ");\n";
        } else {
            o << "    pT = 1.f - ua" << L << ";\n";
        }
        o << "    { float ub = 1.f" << (kind == K_NAE ? ", vb = 1.f" : "") << ";\n";
        for (uint32_t s2 = L; s2-- > 0;) {
            if (kind == K_NAE)
                o << "      G" << s2 << " = fmaf(ua" << s2 << ", ub, -(va" << s2 << " * vb)); ub *= pf" << s2 << "; vb *= pt" << s2 << ";\n";
            else
                o << "      G" << s2 << " = ua" << s2 << " * ub; ub *= " << f1 << s2 << ";\n";
            if (sym_inline) emit_inline_acc(s2, "      ");
        }
        o << "    }\n";
    }
    if (K.count) {
        // CARD(L, k) by its count distribution ("O((n+k)^2)" for symmetric literals): with
        // pt_s = P(literal s true), q_c = P(c of the literals true) by the DP q'_c = q_c pf + q_{c-1} pt
        // (full q_0..q_L, in registers); COP = q_0 + ... + q_k.  dCOP/dpt_s = -r_k with r the
        // distribution of the OTHER literals (moving mass from count k to k+1), taken out of q by the
        // recursion q_c = r_c pf_s + r_{c-1} pt_s: upward (r_c = (q_c - pt_s r_{c-1}) / pf_s) when
        // pt_s <= 1/2, downward from r_{L-1} = q_L / pt_s when pt_s > 1/2 -- the direction whose
        // ratio pt/pf (pf/pt) is <= 1, so rounding errors do not grow.
        // Both passes on the packed f32x2 pipe (each component rounds like the scalar code, so the
        // values are those of the scalar DP): the forward update treats q_{-1} = q_{i+1} = 0, which
        // makes every literal update the fixed pairs (q_{2m+1}, q_{2m}); the backward runs the two
        // directions (cf, cb) as one pair for min(k, L-1-k) steps.
        const uint32_t L = (uint32_t)ns, kk = K.sym_k;
        auto cq = [](uint32_t c) { return "cq" + std::to_string(c); };
        o << "    float cq0 = pf0, cq1 = pt0";
        for (uint32_t c = 2; c <= L + 1; ++c) o << ", " << cq(c) << " = 0.f";
        o << ";\n";
        for (uint32_t i = 1; i < L; ++i) {
            const std::string is = std::to_string(i);
            o << "    { const float2 P2 = FSMT_C2(pt" << is << "), F2 = FSMT_C2(pf" << is << ");\n";
            for (int m = (int)(i + 1) / 2; m >= 0; --m) {
                const uint32_t hi = 2 * (uint32_t)m + 1, lo = 2 * (uint32_t)m;
                if (lo > i + 1) continue;
                const std::string lm1 = m == 0 ? std::string("0.f") : cq(lo - 1);
                o << "      { const float2 nw = __ffma2_rn(make_float2(" << cq(lo) << ", " << lm1 << "), P2, __fmul2_rn(make_float2("
                  << cq(hi) << ", " << cq(lo) << "), F2)); " << cq(hi) << " = nw.x; " << cq(lo) << " = nw.y; }\n";
            }
            o << "    }\n";
        }
        o << "    pT = cq0;";
        for (uint32_t c = 1; c <= kk; ++c) o << " pT += " << cq(c) << ";";
        o << "\n";
        const uint32_t nf = kk, nb = L - 1 - kk, np = std::min(nf, nb);
        for (uint32_t s2 = 0; s2 < L; ++s2) {
            const std::string ss = std::to_string(s2);
            // (rcp.approx: the divisor of the direction kept is >= 1/2, where MUFU.RCP is within 1 ulp;
            // the discarded direction may divide by ~0, its inf / NaN never reaches G)
            o << "    { const float rf = fsmt_rcp(pf" << ss << "), rb = fsmt_rcp(pt" << ss << ");\n"
              << "      const float2 NP = make_float2(-pt" << ss << ", -pf" << ss << "), RR = make_float2(rf, rb);\n"
              << "      float2 cc = __fmul2_rn(make_float2(cq0, " << cq(L) << "), RR);";
            for (uint32_t j = 1; j <= np; ++j) o << " cc = __fmul2_rn(__ffma2_rn(NP, cc, make_float2(" << cq(j) << ", " << cq(L - j) << ")), RR);";
            for (uint32_t j = np + 1; j <= nf; ++j) o << " cc.x = fmaf(-pt" << ss << ", cc.x, " << cq(j) << ") * rf;";
            for (uint32_t j = np + 1; j <= nb; ++j) o << " cc.y = fmaf(-pf" << ss << ", cc.y, " << cq(L - j) << ") * rb;";
            o << "\n      G" << ss << " = pt" << ss << " <= 0.5f ? -cc.x : -cc.y;\n";
            if (sym_inline) emit_inline_acc(s2, "      ");
            o << "    }\n";
        }
    }
    // a Boolean slot of a weight-seeded class whose G is only accumulated: its terms go straight
    // into the accumulator (signs taken back for the complement form); every other G is emitted
    auto is_ident = [](const std::string& x) {
        if (x.empty()) return false;
        for (char ch : x)
            if (!(isalnum((unsigned char)ch) || ch == '_')) return false;
        return true;
    };
    auto negate = [&](const std::string& a) -> std::string {
        if (a.size() > 1 && a[0] == '-' && is_ident(a.substr(1))) return a.substr(1);
        if (a.size() > 3 && a.compare(0, 2, "(-") == 0 && a.back() == ')' && is_ident(a.substr(2, a.size() - 3)))
            return a.substr(2, a.size() - 3);
        return "(-(" + a + "))";
    };
    auto folded = [&](size_t s) { return wseed && t.kinds[s] == 0 && !gt[s].empty(); };
    for (size_t s = 0; s < ns; ++s) {
        if (folded(s)) continue;
        for (size_t k = 0; k < gt[s].size(); ++k) {
            const auto& ab = gt[s][k];
            if (k == 0) o << "    G" << s << " = " << ab.first << " * " << ab.second << ";\n";
            else o << "    G" << s << " = fmaf(" << ab.first << ", " << ab.second << ", G" << s << ");\n";
        }
    }
    auto gref = [&](size_t s) { return cmp ? "(-G" + std::to_string(s) + ")" : "G" + std::to_string(s); };
    if (massF) o << "    const " << TY << " E = fmaf(2.f, pF, -1.f);\n";
    else o << "    const " << TY << " E = 1.f - 2.f * pT;\n";
    // the objective's first level in fp32 over the tile's <= 256 constraints, flushed once per tile into
    // the fp64 objective (two-level accumulation, R28: the per-tile fp32 sum of <= 256 terms adds
    // <= 256 x 2^-24 relative; across tiles the sum is exact on the objective's grid)
    o << "    objacc = fmaf(w, E, objacc);\n"
         "    if (hasT && live && r == terms_r) terms[orig[T.cons_begin + c]] = (double)E;\n";
    // gradient terms per target reference (aliases fold into their target: one read-modify-write)
    std::vector<std::vector<std::pair<std::string, std::string>>> terms_of(nr);
    auto accum = [&](int ri, const std::string& a, const std::string& b) {
        const int tgt = alias_of((size_t)ri) >= 0 ? alias_of((size_t)ri) : ri;
        terms_of[(size_t)tgt].emplace_back(a, b);
    };
    const std::string WG = wseed ? "1.f" : "w";   // weight factor still to apply to a G
    for (size_t s = 0; s < ns; ++s) {
        if (t.kinds[s] == 0) {
            if (folded(s))
                for (const auto& ab : gt[s]) accum(slot_ref0[s], cmp ? negate(ab.first) : ab.first, ab.second);
            else
                accum(slot_ref0[s], WG, gref(s));
        } else if (t.kinds[s] == 2) {
            // dCOP/dp_true of the row = -dCOP/dp_true of a negated literal
            if (!g_inline[s]) accum(slot_ref0[s], WG, "(sg" + std::to_string(s) + " ? -" + gref(s) + " : " + gref(s) + ")");
        } else {
            if (pair_with[s] >= 0) {
                const std::string sa = std::to_string(s), sb = std::to_string(pair_with[s]);
                const std::string gg = "make_float2(" + gref(s) + ", " + gref((size_t)pair_with[s]) + ")";
                o << "    const float2 gdp" << sa << " = __fmul2_rn(" << (wseed ? gg : "__fmul2_rn(FSMT_C2(w), " + gg + ")") << ", ddp" << sa << ");\n"
                  << "    const float gd" << sa << " = gdp" << sa << ".x, gd" << sb << " = gdp" << sa << ".y;\n";
            } else if (!pair_second[s]) {
                o << "    const " << TY << " gd" << s << " = " << (wseed ? std::string() : "w * ") << gref(s) << " * dd" << s << ";\n";
            }
            size_t ai = 0;
            for (size_t s2 = 0; s2 < s; ++s2) ai += t.kinds[s2] == 1;
            for (uint32_t k = 0; k < K.nnz[ai]; ++k) {
                int ri = slot_ref0[s] + (int)k;
                accum(ri, "gd" + std::to_string(s), "__uint_as_float(" + word(coef_word[ri]) + ")");
            }
        }
    }
    for (size_t ri = 0; ri < nr; ++ri) {
        if (terms_of[ri].empty()) continue;
        std::string dst = "acc" + std::to_string(ri);
        if (is_stream(ri))
            dst = head_of(ri) >= 0 ? "accs[(sl" + std::to_string(head_of(ri)) + " + " + std::to_string(K.aff_dl[ri]) + ") * 32]"
                                   : "accs[sl" + std::to_string(ri) + " * 32]";
        std::string e = dst;
        for (const auto& ab : terms_of[ri]) e = "fmaf(" + ab.first + ", " + ab.second + ", " + e + ")";
        o << "    " << dst << " = " << e << ";\n";
    }
    o << "  }\n";
    for (size_t i = 0; i < nr; ++i)
        if (!is_stream(i) && alias_of(i) < 0 && head_of(i) < 0) {
            o << "  if (cur" << i << " != 0xffffffffu) { " << flush_group(i) << " }\n";
        }
    o << "}\n\n";
}

// K5 specialised: exact check of the rounded model (R22) for one kernel class.  Every slot's
// truth value is computed, then the canonical xBDD is evaluated bottom-up with selects
// (branch-free: lanes = restarts take different paths).  Atoms: s = 0; s += q_j y_j in stored
// order in fp64 without FMA; s <= q0 (< q0 when strict).
void emit_verify_class(std::ostringstream& o, uint32_t kid, const KClass& K, const Template& t) {
    g_wk = &K;
    const size_t ns = t.kinds.size();
    o << "__device__ __forceinline__ u32 kv" << kid
      << "(const TileDesc& T, const uint4* __restrict__ rp, const uint4* __restrict__ vp, const u32* __restrict__ vs,\n"
         "    const u32* __restrict__ vr, const signed char* __restrict__ x, const float* __restrict__ y, unsigned short* __restrict__ U,\n"
         "    unsigned char* __restrict__ per_con, const u32* __restrict__ orig, u32 R, u64 rr, u32 r, bool live,\n"
         "    u32 n_bool, const u32* __restrict__ arow, const double* __restrict__ aval,\n"
         "    const double* __restrict__ arhs, const unsigned char* __restrict__ astrict,\n"
         "    const unsigned char* __restrict__ TT, u32& umx, u32& ovf) {\n"
         "  u32 cnt = 0u;\n"
         "  const u32 R4 = R * 4u;\n"
         "  const signed char* xb = x + rr;                          // the lane's column bases\n"
         "  const float* yb = y + (rr - (u64)n_bool * R);             // reals by their unified id\n"
         "  const unsigned char* TTl = TT ? TT + rr : nullptr;\n";
    // words 1.. hold the refs (symmetric classes: then the sign words)
    const uint32_t ref_words = 1 + (K.n_refs + 1) / 2 + (K.sym ? (K.n_refs + 31) / 32 : 0);
    uint32_t q_needed = 0;                                          // compressed uint4s holding them
    for (uint32_t w = 1; w < ref_words; ++w)
        if (K.wpos[w] >= 0) q_needed = std::max(q_needed, (uint32_t)K.wpos[w] / 4 + 1);
    // reference kinds in reference order (0 Boolean, 1 real, 2 table row)
    const uint32_t nref = K.n_refs;
    std::vector<int> rk;
    for (size_t sl = 0, a2 = 0; sl < ns; ++sl) {
        if (t.kinds[sl] == 1) {
            for (uint32_t z = 0; z < K.nnz[a2]; ++z) rk.push_back(1);
            ++a2;
        } else {
            rk.push_back(t.kinds[sl]);
        }
    }
    auto is_alias = [&](uint32_t i) { return i < K.alias.size() && K.alias[i] >= 0; };
    auto head_of = [&](uint32_t i) -> int { return i < K.aff_head.size() ? K.aff_head[i] : -1; };
    auto is_stream = [&](uint32_t i) { return i < K.stream.size() && K.stream[i]; };
    std::vector<std::vector<uint32_t>> members(nref);
    for (uint32_t i = 0; i < nref; ++i)
        if (!is_alias(i) && head_of(i) >= 0) members[(uint32_t)head_of(i)].push_back(i);
    auto ty = [&](uint32_t i) { return std::string(rk[i] == 1 ? "double" : "bool"); };
    // reference i at element offset `e` (u64) of its column: a group member sits at its head's
    // offset plus the constant dg * R, which folds into the load's immediate when R is a
    // compile-time constant (fsmt_prepare)
    auto load_e = [&](uint32_t i, const std::string& e) {
        if (rk[i] == 0) return "xb[" + e + "] == (signed char)-1";
        if (rk[i] == 1) return "(double)FSMT_AT(yb, (" + e + ") * 4u)";
        return "TTl[" + e + "] != 0";
    };
    auto moff = [&](const std::string& base, uint32_t m) {
        return base + " + (u64)((long long)(" + std::to_string(K.aff_dg[m]) + ") * R)";
    };
    // run groups keep their values while the head's variable does not change (one check per
    // group); stream groups load every constraint (one lookup per group)
    for (uint32_t i = 0; i < nref; ++i)
        if (!is_alias(i) && head_of(i) < 0 && !is_stream(i)) {
            o << "  u32 kc" << i << " = 0xffffffffu; " << ty(i) << " kv" << i << " = 0;";
            for (uint32_t m : members[i]) o << " " << ty(m) << " kv" << m << " = 0;";
            o << "\n";
        }
    // the check loop unrolled 4 times for non-symmetric classes, so the compiler issues the next
    // constraints' loads before this one's selects (FSMT_JIT_K5UNROLL overrides; cfg4
    // stage end 3.26 -> 3.06 ms)
    {
        const char* ku = getenv("FSMT_JIT_K5UNROLL");
        o << "#pragma unroll " << (ku ? std::max(1, atoi(ku)) : (K.sym ? 1 : 4)) << "\n";
    }
    o << "  for (u32 c = 0; c < T.n_cons; ++c, rp += " << K.stride4 << ", vp += " << K.vstride4 << ") {\n";
    for (uint32_t q = 0; q < q_needed; ++q) o << "    const uint4 q" << q << " = __ldg(rp + " << q << ");\n";
    for (uint32_t q = 0; q < K.vstride4; ++q) o << "    const uint4 v" << q << " = __ldg(vp + " << q << ");\n";
    uint32_t ref = 0, ai = 0;
    for (uint32_t i = 0; i < nref; ++i) {
        if (is_alias(i) || head_of(i) >= 0) continue;
        const std::string ext = "((" + word(1 + i / 2) + " >> " + std::to_string(16 * (i % 2)) + ") & 0xffffu)";
        if (is_stream(i)) {
            const std::string ob = "ob" + std::to_string(i);
            o << "    const u64 " << ob << " = (u64)vs[" << ext << "] * R;\n";
            o << "    const " << ty(i) << " kv" << i << " = " << load_e(i, ob) << ";\n";
            for (uint32_t m : members[i])
                o << "    const " << ty(m) << " kv" << m << " = " << load_e(m, moff(ob, m)) << ";\n";
        } else {
            o << "    { const u32 l = " << ext << "; if (l != kc" << i << ") { kc" << i << " = l; const u64 ob = (u64)vr[l] * R; kv" << i
              << " = " << load_e(i, "ob") << ";";
            for (uint32_t m : members[i]) o << " kv" << m << " = " << load_e(m, moff("ob", m)) << ";";
            o << " } }\n";
        }
    }
    for (uint32_t i = 0; i < nref; ++i)
        if (is_alias(i)) o << "    const " << ty(i) << " kv" << i << " = kv" << K.alias[i] << ";\n";
    for (size_t s = 0; s < ns; ++s) {
        if (t.kinds[s] == 2) {   // table slot: truth of the row (fsmt_kt_jit) xor the literal's sign
            o << "    const bool t" << s << " = kv" << ref << " != (bool)((" << word(1 + ((uint32_t)ns + 1) / 2 + (uint32_t)s / 32)
              << " >> " << s % 32 << ") & 1u);\n";
            ++ref;
            continue;
        }
        if (t.kinds[s] == 0) {
            o << "    const bool t" << s << " = kv" << ref << ";\n";
            ++ref;
        } else {
            const uint32_t nnz = K.nnz[ai];
            if (K.vfold) {   // class-constant coefficients / strictness as exact literals, rhs from the record
                auto vw = [&](uint32_t w) { return "v" + std::to_string(w / 4) + "." + comp(w); };
                // s = 0; s += q_j y_j in stored order (R22).  A class-constant q_j = +-1 makes q_j y_j = +-y_j
                // exactly, and 0 + x = x (up to the sign of a zero, which no comparison sees): the same
                // values without the multiplications and the leading add
                o << "    bool t" << s << ";\n    { double sacc = 0.0;\n";
                for (uint32_t k = 0; k < nnz; ++k) {
                    const double q = K.vcoef[ai][k];
                    uint64_t bits;
                    memcpy(&bits, &q, 8);
                    const std::string kv = "kv" + std::to_string(ref);
                    const std::string term = q == 1.0 ? kv : q == -1.0 ? "(-" + kv + ")"
                                                     : "__dmul_rn(__longlong_as_double(" + std::to_string((long long)bits) + "LL), " + kv + ")";
                    if (k == 0) o << "      sacc = " << term << ";\n";
                    else o << "      sacc = __dadd_rn(sacc, " << term << ");\n";
                    ++ref;
                }
                o << "      const double rhs = __hiloint2double((int)" << vw(2 * ai + 1) << ", (int)" << vw(2 * ai) << ");\n"
                  << "      t" << s << " = " << (K.vstrict[ai] ? "sacc < rhs" : "sacc <= rhs") << "; }\n";
                ++ai;
                continue;
            }
            const std::string aid = "v" + std::to_string(ai / 4) + "." + comp(ai);
            o << "    bool t" << s << ";\n    { const u32 aid = " << aid << "; const u32 k0 = arow[aid]; double sacc = 0.0;\n";
            for (uint32_t k = 0; k < nnz; ++k) {
                o << "      sacc = __dadd_rn(sacc, __dmul_rn(aval[k0 + " << k << "], kv" << ref << "));\n";
                ++ref;
            }
            o << "      const double rhs = arhs[aid];\n      t" << s << " = astrict[aid] ? (sacc < rhs) : (sacc <= rhs); }\n";
            ++ai;
        }
    }
    auto sat = [&](int child) -> std::string {
        if (child >= 0) return "s" + std::to_string(child);
        return child == kTrue ? "true" : "false";
    };
    if (K.count || K.prod) {   // symmetric: satisfied by the number of true literals
        o << "    u32 nt = 0u;";
        for (size_t s = 0; s < ns; ++s) o << " nt += (u32)t" << s << ";";
        const std::string sat = K.sym_kind == K_CARD ? "nt <= " + std::to_string(K.sym_k) + "u"
                              : K.sym_kind == K_OR   ? std::string("nt >= 1u")
                              : K.sym_kind == K_NAE  ? "(nt >= 1u && nt < " + std::to_string(ns) + "u)"
                                                     : std::string("(nt & 1u)");
        o << "\n    const u32 u = " << sat << " ? 0u : 1u;\n";
    } else {
        for (size_t vv = t.nodes.size(); vv-- > 0;) {
            const TNode& nd = t.nodes[vv];
            o << "    const bool s" << vv << " = t" << nd.level << " ? " << sat(nd.hi) << " : " << sat(nd.lo) << ";\n";
        }
        o << "    const u32 u = " << (t.root >= 0 ? "s" + std::to_string(t.root) : std::string(t.root == kTrue ? "true" : "false"))
          << " ? 0u : 1u;\n";
    }
    o << ""
         "    if (live) {\n"
         "      if (U && u) {   // U += u (R18): only violated constraints touch memory; past 65535 is reported\n"
         "        unsigned short* cell = U + (u64)(T.cons_begin + c) * R + rr;\n"
         "        const u32 nv = (u32)*cell + 1u;\n"
         "        ovf |= nv > 65535u;\n"
         "        const u32 nc = nv > 65535u ? 65535u : nv;\n"
         "        *cell = (unsigned short)nc;\n"
         "        umx = umx > nc ? umx : nc;\n"
         "      }\n"
         "      if (per_con) per_con[(u64)orig[T.cons_begin + c] * R + rr] = (unsigned char)u;\n"
         "    }\n"
         "    cnt += u;\n  }\n  return cnt;\n}\n\n";
}

}  // namespace

std::string jit_source(const Formula& f, const Built& b, const Plan& p, int u_prefetch_default, int k1_min_ctas,
                       const std::vector<int>* class_caps) {
    g_upf = u_prefetch_default;
    g_all_small = p.n_jit_kclasses > 0;
    for (uint32_t k = 0; k < p.n_jit_kclasses; ++k) g_all_small = g_all_small && !p.kclasses[k].sym && p.kclasses[k].n_refs <= 16;
    std::ostringstream o;
    o << "// generated by fsmt tiles.cpp: specialised K1 sweep for " << p.n_jit_kclasses << " kernel classes\n"
         "typedef unsigned int u32;\ntypedef unsigned long long u64;\n"
         "struct TileDesc { u32 kclass, cons_begin, n_cons, var_off, n_vars, rec_off, pad0, pad1; };\n"
      << "#define VMAX " << p.kernel_vmax() << "\n#define VTOT " << p.kernel_vmax() + p.rmax << "\n#define RING " << p.ring_uint4() << "\ntypedef " << (p.vid_bytes() == 2 ? "unsigned short" : "u32") << " VID;   // sweep id-table entry"
      << "\n\n" << kErfcPrelude;
    auto tmpl_of = [&](const KClass& K) -> const Template& { return K.sym ? K.stmpl : b.tmpls[K.tmpl]; };
    for (uint32_t k = 0; k < p.n_jit_kclasses; ++k) emit_class(o, k, p.kclasses[k], tmpl_of(p.kclasses[k]));
    const char* minb = getenv("FSMT_JIT_MINB");      // optional min CTAs/SM (register cap), A/B tuning
    // fsmt_k1_jit: the hot kernel (U present, no E_c output); fsmt_k1_jit_dbg: U may be NULL and
    // the per-constraint E_c debug hook is live.  Separate kernels, so the hot one keeps its own
    // register allocation.  One warp per CTA (CTA-uniform control flow, DESIGN.md §7 item 5).
    // fsmt_k1_c<k>: the hot kernel of class k alone, launched over that class's tiles, so each class
    // gets its own register allocation and cap (DESIGN.md §7 item 17).
    for (int kv = -2; kv < (int)p.n_jit_kclasses; ++kv) {
    const int dbgk = kv == -1;
    // hot kernel: k1_min_ctas resident warps per SM as a register cap (fsmt_prepare picks
    // the largest of 32 / 28 that compiles without spills; 0 = none); FSMT_JIT_MINB overrides
    const int cap = kv >= 0 && class_caps ? (*class_caps)[(size_t)kv] : k1_min_ctas;
    const std::string mb = minb ? std::string(minb) : (dbgk || cap <= 0 ? std::string() : std::to_string(cap));
    o << "extern \"C\" __global__ void __launch_bounds__(32" << (atoi(mb.c_str()) > 0 ? ", " + mb : std::string())
      << ") " << (kv >= 0 ? "fsmt_k1_c" + std::to_string(kv) : std::string(dbgk ? "fsmt_k1_jit_dbg" : "fsmt_k1_jit")) << "(\n"
         "    const TileDesc* __restrict__ tiles, u32 n_tiles, const uint4* __restrict__ recs,\n"
         "    const u32* __restrict__ tile_vars, const float* __restrict__ a, const float* __restrict__ b,\n"
         "    double* __restrict__ ga, double* __restrict__ gb, const unsigned short* __restrict__ U,\n"
         "    double* __restrict__ obj, u32 R, u32 n_bool, float kappa,\n"
         "    double* __restrict__ terms, u32 terms_r, const u32* __restrict__ orig,\n"
         "    const float* __restrict__ PT, double* __restrict__ gu,\n"
         "    const FxScale* __restrict__ fxs, const float* __restrict__ kdev, u32 nsplit) {\n"
         "  FSMT_SPECIALISE_R\n"
         "  if (kdev) kappa = *kdev;   // the device-side solve loop's stage kappa (DevStage)\n"
         "  extern __shared__ float smem[];\n"
         "  const int lane = threadIdx.x & 31;\n"
         "  uint4* ring = (uint4*)smem;                           // record ring (RING uint4)\n"
         "  float* acc = smem + RING * 4;                         // stream-variable rows\n"
         "  VID* vs = (VID*)(acc + VMAX * 32);                    // stream then run variable ids\n"
         "  const u32 rtiles = (R + 31) / 32;\n"
      << "  const u64 tsub = blockIdx.x / rtiles;                // tile-major: a tile's restart tiles together\n"
         "  const u64 ti = tsub / nsplit;\n"
         "  const u32 rt = (u32)(blockIdx.x % rtiles);\n"
         "  if (ti >= n_tiles) return;\n"
         "  TileDesc T = tiles[ti];\n"
         "  // launch-time split of a tile into nsplit constraint ranges (few restarts: enough CTAs to fill\n"
         "  // the GPU); each range flushes its own stream rows (exact on-grid adds, any order)\n"
         "  u32 cb = 0u;\n"
         "  if (nsplit > 1u) {\n"
         "    const u32 sub = (u32)(tsub % nsplit);\n"
         "    cb = (u32)((u64)T.n_cons * sub / nsplit);\n"
         "    const u32 ce = (u32)((u64)T.n_cons * (sub + 1u) / nsplit);\n"
         "    if (ce <= cb) return;\n"
         "    T.cons_begin += cb;\n"
         "    T.n_cons = ce - cb;\n"
         "  }\n"
         "  const u32 n_s = T.n_vars & 0xffffu, n_v = n_s + (T.n_vars >> 16);\n"
         "  const u32 r = rt * 32 + lane;\n"
         "  const bool live = r < R;\n"
         "  const u64 rr = live ? r : 0;\n"
         "  for (u32 l = lane; l < n_v; l += 32) vs[l] = tile_vars[T.var_off + l];\n"
         "  for (u32 l = lane; l < n_s * 8u; l += 32u) ((float4*)acc)[l] = make_float4(0.f, 0.f, 0.f, 0.f);   // rows, 16 B stores\n"
         "  __syncwarp();\n"
         "  const VID* vr = vs + n_s;\n"
         "  const float kq = kappa * 0.70710678118654752f;\n"
         "  const float dcoef = kappa * 0.79788456080286536f;\n"
         "  const float gif = fxs[rr].gif;\n"
         "  const int ebias = fxs[rr].ebias;\n"
         "  float objacc = 0.f;\n"
         "  const uint4* rp = recs + T.rec_off;\n"
         "  // the lane's column bases: element (v, restart rr) of a [var][R] array at base + v * 4R bytes\n"
         "  const u32 R4 = R * 4u;\n"
         "  const float* ab = a + rr;\n"
         "  const float* bb = b + (rr - (u64)n_bool * R);   // reals are addressed by their unified id\n"
         "  const float* PTl = PT ? PT + rr : nullptr;\n"

         "  bool symt = false;   // symmetric class: the tile's variables are slot-table rows\n"
         "  switch (T.kclass) {\n";
    for (uint32_t k = 0; k < p.n_jit_kclasses; ++k) {
        if (kv >= 0 && (int)k != kv) continue;
        const std::string args = "(T, rp + (u64)cb * " + std::to_string(p.kclasses[k].stride4) +
                                 "u, vs, vr, acc + lane, ab, bb, ga, gb, U, R, R4, rr, r, live, n_bool, kq, dcoef, ebias, "
                                 "gif, objacc, terms, terms_r, orig, PTl, gu, ring, (u32)lane); ";
        o << "    case " << k << ": kc" << k << (dbgk ? "<true>" : "<false>") << args
          << (p.kclasses[k].sym ? "symt = true; " : "") << "break;\n";
    }
    o << "    default: break;\n  }\n"
         "  __syncwarp();\n"
         "  if (!live) return;\n"
         "  for (u32 l = 0; l < n_s; ++l) {   // stream rows: one on-grid fp64 add per row and tile\n"
         "    const u32 g = vs[l];\n"
         "    const double v = fsmt_q(acc[l * 32 + lane], gif);\n"
         "    if (symt) atomicAdd(gu + (u64)g * R + r, v);\n"
         "    else if (g < n_bool) atomicAdd(ga + (u64)g * R + r, v); else atomicAdd(gb + (u64)(g - n_bool) * R + r, v);\n"
         "  }\n"
         "  atomicAdd(obj + r, rint((double)objacc * fxs[r].oi) * fxs[r].os);   // on the objective's grid, true units\n"
         "}\n\n";
    }
    // K5: exact verification of the rounded models + ERWA counters over the same tiles
    for (uint32_t k = 0; k < p.n_jit_kclasses; ++k) emit_verify_class(o, k, p.kclasses[k], tmpl_of(p.kclasses[k]));
    o << "extern \"C\" __global__ void __launch_bounds__(32) fsmt_k5_jit(\n"
         "    const TileDesc* __restrict__ tiles, u32 n_tiles, const uint4* __restrict__ recs,\n"
         "    const uint4* __restrict__ vrecs, const u32* __restrict__ tile_vars, const signed char* __restrict__ x,\n"
         "    const float* __restrict__ y, unsigned short* __restrict__ U, u32* __restrict__ unsat,\n"
         "    unsigned char* __restrict__ per_con, const u32* __restrict__ orig, u32 R, u32 n_bool,\n"
         "    const u32* __restrict__ arow, const double* __restrict__ aval, const double* __restrict__ arhs,\n"
         "    const unsigned char* __restrict__ astrict, const unsigned char* __restrict__ TT,\n"
         "    u32* __restrict__ umax, u32* __restrict__ flags, u32 nsplit) {\n"
         "  FSMT_SPECIALISE_R\n"
         "  extern __shared__ float smem[];\n"
         "  const int lane = threadIdx.x & 31;\n"
         "  u32* vs = (u32*)smem;\n"
         "  const u32 rtiles = (R + 31) / 32;\n"
         "  const u64 gw = (u64)blockIdx.x;\n"
         "  const u32 rt = (u32)(gw % rtiles);\n"
         "  const u64 tsub = gw / rtiles;\n"
         "  const u64 ti = tsub / nsplit;\n"
         "  if (ti >= n_tiles) return;\n"
         "  TileDesc T = tiles[ti];\n"
         "  u32 cb = 0u;   // launch-time split (as the sweep)\n"
         "  if (nsplit > 1u) {\n"
         "    const u32 sub = (u32)(tsub % nsplit);\n"
         "    cb = (u32)((u64)T.n_cons * sub / nsplit);\n"
         "    const u32 ce = (u32)((u64)T.n_cons * (sub + 1u) / nsplit);\n"
         "    if (ce <= cb) return;\n"
         "    T.cons_begin += cb;\n"
         "    T.n_cons = ce - cb;\n"
         "  }\n"
         "  const u32 r = rt * 32 + lane;\n"
         "  const bool live = r < R;\n"
         "  const u64 rr = live ? r : 0;\n"
         "  const u32 n_s = T.n_vars & 0xffffu, n_v = n_s + (T.n_vars >> 16);\n"
         "  for (u32 l = lane; l < n_v; l += 32) vs[l] = tile_vars[T.var_off + l];\n"
         "  __syncwarp();\n"
         "  const u32* vr = vs + n_s;\n"
         "  const uint4* rp = recs + T.rec_off;\n"
         "  const uint4* vp = vrecs + T.pad1;\n"
         "  u32 cnt = 0u, umx = 0u, ovf = 0u;\n"
         "  switch (T.kclass) {\n";
    for (uint32_t k = 0; k < p.n_jit_kclasses; ++k)
        o << "    case " << k << ": cnt = kv" << k << "(T, rp + (u64)cb * " << p.kclasses[k].stride4 << "u, vp + (u64)cb * "
          << p.kclasses[k].vstride4 << "u, vs, vr, x, y, U, per_con, orig, R, rr, r, live, n_bool, arow, aval, arhs, astrict, TT, umx, ovf); break;\n";
    o << "    default: break;\n  }\n"
         "  if (live && cnt) atomicAdd(unsat + r, cnt);\n"
         "  if (live && umx) atomicMax(umax + r, umx);   // the restart's largest counter (k1_prologue's shift)\n"
         "  if (ovf) atomicOr(flags, 1u);                 // a counter passed 65535: fsmt_stage_end fails (FSMT_ERR_RANGE)\n"
         "}\n";
    // slot tables for the symmetric classes: probabilities of every Boolean and
    // table atom once per sweep, the row gradients chained back to grad_a / grad_b, and the rows'
    // exact truth values for K5
    o << "extern \"C\" __global__ void fsmt_kp_jit(u32 n_bool, u32 nv, u32 n_sa, const u32* __restrict__ satoms,\n"
         "    const float* __restrict__ a, const float* __restrict__ b, const u32* __restrict__ arow,\n"
         "    const u32* __restrict__ acol, const float* __restrict__ aval, const float* __restrict__ arhs,\n"
         "    const float* __restrict__ ainv, u32 R, float kappa, float* __restrict__ PT,\n"
         "    float* __restrict__ DD, const float* __restrict__ kdev) {\n"
         "  if (kdev) kappa = *kdev;\n"
         "  const u64 n = (u64)(n_bool + n_sa) * R;\n"
         "  const float kq = kappa * 0.70710678118654752f, dcoef = kappa * 0.79788456080286536f;\n"
         "  for (u64 idx = (u64)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (u64)gridDim.x * blockDim.x) {\n"
         "    const u32 row = (u32)(idx / R), r = (u32)(idx % R);\n"
         "    if (row < n_bool) {                       // Eq.4: p_true = (1 - a)/2\n"
         "      const float v = a[idx];\n"
         "      PT[idx] = 0.5f * (1.f - v);\n"
         "    } else {                                  // Eq.7 with the erfc form (R28b)\n"
         "      const u32 t = row - n_bool, at = satoms[t];\n"
         "      float z = -arhs[at];\n"
         "      for (u32 k = arow[at]; k < arow[at + 1]; ++k) z = fmaf(aval[k], b[(u64)acol[k] * R + r], z);\n"
         "      const float inv = ainv[at], u = kq * z * inv;\n"
         "      float ez;\n"
         "      const float e = fsmt_half_erfc(fabsf(u), ez);\n"
         "      const u64 o = (u64)(nv + t) * R + r;\n"
         "      PT[o] = u >= 0.f ? e : 1.f - e;\n"
         "      DD[(u64)t * R + r] = dcoef * inv * ez;\n"
         "    }\n"
         "  }\n"
         "}\n\n"
         "extern \"C\" __global__ void fsmt_kc_jit(u32 n_bool, u32 nv, u32 n_sa, const u32* __restrict__ satoms,\n"
         "    const u32* __restrict__ arow, const u32* __restrict__ acol, const float* __restrict__ aval, u32 R,\n"
         "    const double* __restrict__ gu, const float* __restrict__ DD, double* __restrict__ ga, double* __restrict__ gb) {\n"
         "  // one thread per (row, restart); grid units throughout (the rows are exact integer sums, the b\n"
         "  // terms are rounded to the grid), so the atomics' sums are exact and their order is immaterial\n"
         "  const u64 nb = (u64)n_bool * R, n = nb + (u64)n_sa * R;\n"
         "  for (u64 idx = (u64)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (u64)gridDim.x * blockDim.x) {\n"
         "    if (idx < nb) { ga[idx] += gu[idx]; continue; }          // Boolean rows: dE/da_i\n"
         "    const u32 t = (u32)((idx - nb) / R), r = (u32)((idx - nb) % R);\n"
         "    const double g = gu[(u64)(nv + t) * R + r] * (double)DD[(u64)t * R + r];   // dE/db_j = sum G dd q_j (P:1326-1327)\n"
         "    const u32 at = satoms[t];\n"
         "    for (u32 k = arow[at]; k < arow[at + 1]; ++k) atomicAdd(gb + (u64)acol[k] * R + r, rint(g * (double)aval[k]));\n"
         "  }\n"
         "}\n\n"
         "extern \"C\" __global__ void fsmt_kt_jit(u32 n_bool, u32 nv, u32 n_sa, const u32* __restrict__ satoms,\n"
         "    const signed char* __restrict__ x, const float* __restrict__ y, const u32* __restrict__ arow,\n"
         "    const u32* __restrict__ acol, const double* __restrict__ aval, const double* __restrict__ arhs,\n"
         "    const unsigned char* __restrict__ astrict, u32 R, unsigned char* __restrict__ TT) {\n"
         "  const u64 n = (u64)(n_bool + n_sa) * R;\n"
         "  for (u64 idx = (u64)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (u64)gridDim.x * blockDim.x) {\n"
         "    const u32 row = (u32)(idx / R), r = (u32)(idx % R);\n"
         "    if (row < n_bool) { TT[idx] = x[idx] == (signed char)-1; continue; }\n"
         "    const u32 t = row - n_bool, at = satoms[t];\n"
         "    double s = 0.0;                           // exact check (R22): fp64, stored order, no FMA\n"
         "    for (u32 k = arow[at]; k < arow[at + 1]; ++k) s = __dadd_rn(s, __dmul_rn(aval[k], (double)y[(u64)acol[k] * R + r]));\n"
         "    TT[(u64)(nv + t) * R + r] = astrict[at] ? (s < arhs[at]) : (s <= arhs[at]);\n"
         "  }\n"
         "}\n";
    (void)f;
    return o.str();
}

}  // namespace fsmt
