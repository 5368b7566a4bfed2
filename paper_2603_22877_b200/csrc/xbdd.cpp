// xBDD builder (a0 of SURVEY §8(a)): Alg.1 lines 1-2, Def.2.
//
// Each constraint is compiled to the reduced ordered BDD of its truth function over its
// slots, "interpreting atomic constraints as propositional variables"; no LP
// pruning.  Slots (R5/R6): one per distinct variable/atom, ordered by first
// appearance in a left-to-right DFS (literal order for symmetric kinds).  Construction is
// a small BDD package of our own (unique table + apply cache; CUDD is only suggested at
// P:292).  Canonical numbering (R7): stable sort by (level, pre-order index of a DFS from
// the root visiting hi first); terminals -1 FALSE, -2 TRUE.  Identical canonical diagrams
// share one template.  Projection bounds come from single-variable unit atoms (R15).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <unordered_map>

#include "fsmt_internal.hpp"

namespace fsmt {
namespace {

constexpr uint32_t kTermLevel = 0xFFFFFFFFu;

struct Mgr {
    std::vector<uint32_t> lvl{kTermLevel, kTermLevel};
    std::vector<int> hi{0, 1}, lo{0, 1};   // id 0 = FALSE, 1 = TRUE
    std::unordered_map<uint64_t, int> uniq;
    std::unordered_map<uint64_t, int> cache;
    uint64_t budget;

    explicit Mgr(uint64_t b) : budget(b) {}

    int mk(uint32_t l, int h, int lw) {
        if (h == lw) return h;
        uint64_t key = ((uint64_t)l << 44) | ((uint64_t)h << 22) | (uint64_t)lw;
        auto it = uniq.find(key);
        if (it != uniq.end()) return it->second;
        if (lvl.size() - 2 >= budget || lvl.size() >= (1u << 22) - 1) throw BuildError{"node budget exceeded", true};
        int id = (int)lvl.size();
        lvl.push_back(l);
        hi.push_back(h);
        lo.push_back(lw);
        uniq.emplace(key, id);
        return id;
    }
    int var(uint32_t level, bool neg) { return neg ? mk(level, 0, 1) : mk(level, 1, 0); }

    enum { AND = 0, OR = 1, XOR = 2 };
    int apply(int op, int f, int g) {
        if (f > g) std::swap(f, g);                   // all three ops commute
        switch (op) {
            case AND:
                if (f == 0) return 0;
                if (f == 1) return g;
                if (f == g) return f;
                break;
            case OR:
                if (f == 1 || g == 1) return 1;
                if (f == 0) return g;
                if (f == g) return f;
                break;
            default:
                if (f == 0) return g;
                if (f == g) return 0;
                break;
        }
        if (op == XOR && f == 1 && g == 1) return 0;
        uint64_t key = ((uint64_t)op << 60) | ((uint64_t)f << 30) | (uint64_t)g;
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
        uint32_t lf = lvl[f], lg = lvl[g];
        uint32_t top = std::min(lf, lg);
        int f1 = (lf == top) ? hi[f] : f, f0 = (lf == top) ? lo[f] : f;
        int g1 = (lg == top) ? hi[g] : g, g0 = (lg == top) ? lo[g] : g;
        int h = apply(op, f1, g1);
        int l = apply(op, f0, g0);
        int r = mk(top, h, l);
        cache.emplace(key, r);
        return r;
    }
    int neg(int f) { return apply(XOR, f, 1); }
};

struct SlotMap {
    std::vector<uint8_t> kinds;
    std::vector<uint32_t> ids;
    std::unordered_map<uint64_t, uint32_t> pos;
    uint32_t get(uint8_t kind, uint32_t idx) {
        uint64_t key = ((uint64_t)kind << 32) | idx;
        auto it = pos.find(key);
        if (it != pos.end()) return it->second;
        uint32_t p = (uint32_t)kinds.size();
        kinds.push_back(kind);
        ids.push_back(idx);
        pos.emplace(key, p);
        return p;
    }
    void clear() {
        kinds.clear();
        ids.clear();
        pos.clear();
    }
};

// Collect slots by first appearance (left-to-right DFS) and the shape key (slot-renamed text).
void collect_expr(const Formula& f, uint32_t v, SlotMap& sm, std::string& key) {
    const ExprNode& nd = f.expr[v];
    if (nd.op == OP_LIT) {
        uint32_t p = sm.get(nd.kind, nd.idx);
        key += 's';
        key += std::to_string(p);
        key += ' ';
        return;
    }
    static const char* names[] = {"", "(and ", "(or ", "(xor ", "(not "};
    key += names[nd.op];
    for (uint32_t t = 0; t < nd.n; ++t) collect_expr(f, f.kids[nd.first + t], sm, key);
    key += ')';
}

int compile_expr(const Formula& f, uint32_t v, const SlotMap& sm, Mgr& m) {
    const ExprNode& nd = f.expr[v];
    if (nd.op == OP_LIT) {
        uint64_t key = ((uint64_t)nd.kind << 32) | nd.idx;
        return m.var(sm.pos.at(key), false);
    }
    if (nd.op == OP_NOT) return m.neg(compile_expr(f, f.kids[nd.first], sm, m));
    int op = nd.op == OP_AND ? Mgr::AND : nd.op == OP_OR ? Mgr::OR : Mgr::XOR;
    int acc = compile_expr(f, f.kids[nd.first], sm, m);
    for (uint32_t t = 1; t < nd.n; ++t) acc = m.apply(op, acc, compile_expr(f, f.kids[nd.first + t], sm, m));
    return acc;
}

// Symmetric constraint over literal diagrams lit[0..L) (slot order): OR, CARD (#true <= k), NAE, XOR.
int combine_symmetric(Mgr& m, uint32_t kind, uint32_t k, const std::vector<int>& lit) {
    switch (kind) {
        case K_OR: {
            int acc = 0;
            for (int x : lit) acc = m.apply(Mgr::OR, acc, x);
            return acc;
        }
        case K_XOR: {                                  // odd number of true literals
            int acc = 0;
            for (int x : lit) acc = m.apply(Mgr::XOR, acc, x);
            return acc;
        }
        case K_NAE: {                                  // not (all true or all false)
            int all_t = 1, all_f = 1;
            for (int x : lit) {
                all_t = m.apply(Mgr::AND, all_t, x);
                all_f = m.apply(Mgr::AND, all_f, m.neg(x));
            }
            return m.neg(m.apply(Mgr::OR, all_t, all_f));
        }
        default: {                                     // CARD: #true <= k (count DP, saturating at k+1)
            std::vector<int> S(k + 2, 0);
            S[0] = 1;
            for (int x : lit) {
                int nx = m.neg(x);
                std::vector<int> T(k + 2, 0);
                T[k + 1] = m.apply(Mgr::OR, S[k + 1], m.apply(Mgr::AND, x, S[k]));
                for (uint32_t cc = k + 1; cc-- > 0;) {
                    int stay = m.apply(Mgr::AND, nx, S[cc]);
                    int move = cc > 0 ? m.apply(Mgr::AND, x, S[cc - 1]) : 0;
                    T[cc] = m.apply(Mgr::OR, stay, move);
                }
                S.swap(T);
            }
            return m.neg(S[k + 1]);
        }
    }
}

int compile_symmetric(const Formula& f, const Constraint& c, const SlotMap& sm, Mgr& m) {
    std::vector<int> lit(c.lit_n);
    for (uint32_t t = 0; t < c.lit_n; ++t) {
        const Lit& l = f.lits[c.lit_first + t];
        lit[t] = m.var(sm.pos.at(((uint64_t)l.kind << 32) | l.idx), l.neg != 0);
    }
    return combine_symmetric(m, c.kind, c.k, lit);
}

// Canonical numbering (R7) of the diagram rooted at `root` (manager ids).
Template canonicalise(const Mgr& m, int root, const std::vector<uint8_t>& kinds) {
    Template t;
    t.kinds = kinds;
    if (root <= 1) {
        t.root = root == 1 ? kTrue : kFalse;
        return t;
    }
    std::unordered_map<int, int> pre;
    std::vector<int> order;
    std::vector<int> st{root};
    while (!st.empty()) {                      // iterative pre-order, hi before lo
        int v = st.back();
        st.pop_back();
        if (v <= 1 || pre.count(v)) continue;
        pre.emplace(v, (int)order.size());
        order.push_back(v);
        st.push_back(m.lo[v]);
        st.push_back(m.hi[v]);
    }
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        if (m.lvl[a] != m.lvl[b]) return m.lvl[a] < m.lvl[b];
        return pre.at(a) < pre.at(b);
    });
    std::unordered_map<int, int> rank;
    for (size_t i = 0; i < order.size(); ++i) rank.emplace(order[i], (int)i);
    auto ren = [&](int v) { return v == 0 ? kFalse : v == 1 ? kTrue : rank.at(v); };
    if (order.size() > 32767) throw BuildError{"template exceeds 32767 nodes (encoding limit)", true};
    for (int v : order) t.nodes.push_back(TNode{(uint16_t)m.lvl[v], (int16_t)ren(m.hi[v]), (int16_t)ren(m.lo[v]), 0});
    t.root = ren(root);
    return t;
}

std::string template_key(const Template& t) {
    std::string k;
    k.append((const char*)t.kinds.data(), t.kinds.size());
    k += '|';
    k.append((const char*)t.nodes.data(), t.nodes.size() * sizeof(TNode));
    k += '|';
    k += std::to_string(t.root);
    return k;
}

}  // namespace

Template symmetric_template(uint32_t kind, uint32_t L, uint32_t k) {
    Mgr m(1u << 21);
    std::vector<int> lit(L);
    for (uint32_t t = 0; t < L; ++t) lit[t] = m.var(t, false);
    return canonicalise(m, combine_symmetric(m, kind, k, lit), std::vector<uint8_t>(L, 2));
}

namespace {

bool unit_holds(const Formula& f, uint32_t atom, bool positive, float y) {
    uint32_t r0 = f.atom_rowptr[atom];
    double s = 0.0;
    s = s + f.atom_val[r0] * (double)y;
    bool truth = f.atom_strict[atom] ? (s < f.atom_rhs[atom]) : (s <= f.atom_rhs[atom]);
    return positive ? truth : !truth;
}

}  // namespace

bool eval_atom_exact(const Formula& f, uint32_t atom, const float* y, size_t stride) {
    double s = 0.0;
    for (uint32_t t = f.atom_rowptr[atom]; t < f.atom_rowptr[atom + 1]; ++t)
        s = s + f.atom_val[t] * (double)y[(size_t)f.atom_col[t] * stride];
    return f.atom_strict[atom] ? (s < f.atom_rhs[atom]) : (s <= f.atom_rhs[atom]);
}

Built build_xbdds(const Formula& f, uint64_t node_budget) {
    if (node_budget == 0 || node_budget > 32767) node_budget = 32767;
    Built b;
    size_t C = f.cons.size();
    b.cons_tmpl.resize(C);
    b.cons_slot_off.resize(C + 1);
    b.cons_w.resize(C);
    b.cons_sym.assign(C, 0);
    b.cons_k.assign(C, 0);
    b.lo.assign(f.n_real, -INFINITY);
    b.hi.assign(f.n_real, INFINITY);
    std::unordered_map<std::string, uint32_t> shape_to_tid;
    std::unordered_map<std::string, uint32_t> key_to_tid;
    SlotMap sm;
    std::string shape;
    b.cons_slot_off[0] = 0;
    for (size_t ci = 0; ci < C; ++ci) {
        const Constraint& c = f.cons[ci];
        sm.clear();
        shape.clear();
        if (c.kind == K_EXPR) {
            shape = "e:";
            collect_expr(f, c.expr_root, sm, shape);
        } else {
            static const char* kn[] = {"or", "card", "nae", "xor"};
            shape = std::string(kn[c.kind]) + std::to_string(c.k) + ":";
            for (uint32_t t = 0; t < c.lit_n; ++t) {
                const Lit& l = f.lits[c.lit_first + t];
                uint32_t p = sm.get(l.kind, l.idx);
                shape += l.neg ? '-' : '+';
                shape += std::to_string(p);
                shape += ',';
            }
        }
        shape += '#';
        shape.append((const char*)sm.kinds.data(), sm.kinds.size());
        if (sm.kinds.size() > 65535) throw BuildError{"constraint has more than 65535 slots", true};
        uint32_t tid;
        auto hit = shape_to_tid.find(shape);
        if (hit != shape_to_tid.end()) {
            tid = hit->second;
        } else {
            // the manager also holds the intermediate diagrams of the construction (a CARD count DP
            // builds far more than it keeps): its cap is a memory guard; the budget binds the result
            Mgr m(std::max<uint64_t>(node_budget, 1u << 21));
            int root = c.kind == K_EXPR ? compile_expr(f, c.expr_root, sm, m) : compile_symmetric(f, c, sm, m);
            Template t = canonicalise(m, root, sm.kinds);
            if (t.nodes.size() > node_budget) throw BuildError{"node budget exceeded", true};
            std::string key = template_key(t);
            auto kh = key_to_tid.find(key);
            if (kh != key_to_tid.end()) {
                tid = kh->second;
            } else {
                tid = (uint32_t)b.tmpls.size();
                key_to_tid.emplace(key, tid);
                b.tmpls.push_back(std::move(t));
            }
            shape_to_tid.emplace(shape, tid);
        }
        const Template& t = b.tmpls[tid];
        b.cons_tmpl[ci] = tid;
        b.cons_w[ci] = (float)c.weight;
        const bool sym = c.kind != K_EXPR && sm.ids.size() == c.lit_n;   // distinct variables: slot i = literal i
        b.cons_sym[ci] = sym ? (uint8_t)(1 + c.kind) : 0;
        b.cons_k[ci] = (uint16_t)std::min<uint32_t>(c.k, 65535);
        for (size_t s = 0; s < sm.ids.size(); ++s) b.slot_neg.push_back(sym ? f.lits[c.lit_first + s].neg : 0);
        b.slot_ids.insert(b.slot_ids.end(), sm.ids.begin(), sm.ids.end());
        b.cons_slot_off[ci + 1] = (uint32_t)b.slot_ids.size();
        b.max_slots = std::max<uint32_t>(b.max_slots, (uint32_t)t.kinds.size());
        b.max_nodes = std::max<uint32_t>(b.max_nodes, (uint32_t)t.nodes.size());
        b.n_nodes += t.nodes.size();
        // projection bounds from single-variable unit atoms (Prop.1, R15)
        if (t.kinds.size() == 1 && t.kinds[0] == 1 && t.nodes.size() == 1) {
            uint32_t atom = sm.ids[0];
            const TNode& nd = t.nodes[0];
            bool positive = (nd.hi == kTrue && nd.lo == kFalse);
            bool negative = (nd.hi == kFalse && nd.lo == kTrue);
            uint32_t r0 = f.atom_rowptr[atom];
            const uint32_t nnz = f.atom_rowptr[atom + 1] - r0;
            if ((positive || negative) && nnz >= 2) {
                // R33: g = +-q, h = +-q0 - delta, delta = 2^-17 (|q0| + ||q||_1)
                double l1 = 0.0;
                for (uint32_t k = r0; k < r0 + nnz; ++k) l1 += std::fabs(f.atom_val[k]);
                const double delta = std::ldexp(std::fabs(f.atom_rhs[atom]) + l1, -17);
                const double sg = positive ? 1.0 : -1.0;
                for (uint32_t k = r0; k < r0 + nnz; ++k) {
                    b.h_col.push_back(f.atom_col[k]);
                    b.h_g.push_back(sg * f.atom_val[k]);
                }
                b.h_h.push_back(sg * f.atom_rhs[atom] - delta);
                b.h_rowptr.push_back((uint32_t)b.h_col.size());
            }
            if ((positive || negative) && nnz == 1) {
                uint32_t j = f.atom_col[r0];
                double q = f.atom_val[r0];
                bool upper = (q > 0) == positive;
                float y = (float)(f.atom_rhs[atom] / q);
                if (upper) {
                    while (unit_holds(f, atom, positive, std::nextafterf(y, INFINITY))) y = std::nextafterf(y, INFINITY);
                    while (!unit_holds(f, atom, positive, y)) y = std::nextafterf(y, -INFINITY);
                    b.hi[j] = std::min(b.hi[j], y);
                } else {
                    while (unit_holds(f, atom, positive, std::nextafterf(y, -INFINITY))) y = std::nextafterf(y, -INFINITY);
                    while (!unit_holds(f, atom, positive, y)) y = std::nextafterf(y, INFINITY);
                    b.lo[j] = std::max(b.lo[j], y);
                }
            }
        }
    }
    for (uint32_t j = 0; j < f.n_real; ++j) b.n_bounded += (std::isfinite(b.lo[j]) || std::isfinite(b.hi[j]));
    return b;
}

// Exact check of one model (R22) over constraints [c0, c1): the number violated.
static uint32_t verify_range(const Formula& f, const Built& b, const int8_t* x, const float* y, uint8_t* per_con,
                             size_t c0, size_t c1) {
    uint32_t n = 0;
    for (size_t ci = c0; ci < c1; ++ci) {
        const Template& t = b.tmpls[b.cons_tmpl[ci]];
        const uint32_t* ids = b.slot_ids.data() + b.cons_slot_off[ci];
        int v = t.root;
        while (v >= 0) {
            const TNode& nd = t.nodes[(size_t)v];
            bool truth = t.kinds[nd.level] == 0 ? (x[ids[nd.level]] == -1) : eval_atom_exact(f, ids[nd.level], y, 1);
            v = truth ? nd.hi : nd.lo;
        }
        uint8_t u = (v == kFalse);
        n += u;
        if (per_con) per_con[ci] = u;
    }
    return n;
}

// The host re-verification: constraint ranges on the host's cores (each constraint's
// verdict is independent, so the count does not depend on the split).
uint32_t verify_host(const Formula& f, const Built& b, const int8_t* x, const float* y, uint8_t* per_con) {
    const size_t C = f.cons.size();
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t nt = C < 20000 ? 1 : std::min<size_t>(hw, 16);
    if (nt == 1) return verify_range(f, b, x, y, per_con, 0, C);
    std::vector<uint32_t> part(nt, 0);
    std::vector<std::thread> th;
    for (size_t k = 0; k < nt; ++k)
        th.emplace_back([&, k] { part[k] = verify_range(f, b, x, y, per_con, C * k / nt, C * (k + 1) / nt); });
    for (auto& t : th) t.join();
    uint32_t n = 0;
    for (uint32_t v : part) n += v;
    return n;
}

std::string dump_templates_jsonl(const Built& b) {
    std::string s;
    for (const Template& t : b.tmpls) {
        s += "{\"slot_kinds\":[";
        for (size_t i = 0; i < t.kinds.size(); ++i) {
            if (i) s += ',';
            s += std::to_string(t.kinds[i]);
        }
        s += "],\"nodes\":[";
        for (size_t i = 0; i < t.nodes.size(); ++i) {
            if (i) s += ',';
            s += '[' + std::to_string(t.nodes[i].level) + ',' + std::to_string(t.nodes[i].hi) + ',' +
                 std::to_string(t.nodes[i].lo) + ']';
        }
        s += "],\"root\":" + std::to_string(t.root) + "}\n";
    }
    return s;
}

std::vector<uint8_t> dump_constraints_bin(const Built& b) {
    std::vector<uint8_t> out;
    auto put = [&](uint32_t v) {
        uint8_t w[4] = {(uint8_t)v, (uint8_t)(v >> 8), (uint8_t)(v >> 16), (uint8_t)(v >> 24)};
        out.insert(out.end(), w, w + 4);
    };
    for (size_t ci = 0; ci < b.cons_tmpl.size(); ++ci) {
        uint32_t n = b.cons_slot_off[ci + 1] - b.cons_slot_off[ci];
        put(b.cons_tmpl[ci]);
        put(n);
        for (uint32_t t = 0; t < n; ++t) put(b.slot_ids[b.cons_slot_off[ci] + t]);
    }
    return out;
}

}  // namespace fsmt
