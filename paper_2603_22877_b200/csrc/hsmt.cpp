// HSMT parser for the product path.  Own implementation; the oracle's
// Python parser (oracle/hsmt.py) shares no code with it.
//   p hsmt <n_bool> <n_real>
//   a <id> <rel> <rhs> <j>:<coeff> ...      rel in {<=,<,>=,>}  ('=' rejected, R9)
//   c <kind> [<k>] <weight> <lit>...        kind in {or,card,nae,xor}; lit = [+-][ab]<i>
//   e <weight> <sexpr>                      (and ..)|(or ..)|(xor ..)|(not e)|b<i>|a<i>
// Atoms canonicalised to q.y <= q0 / < q0 by negating (q, q0) for >= / >.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <unordered_set>

#include "fsmt_internal.hpp"

namespace fsmt {
namespace {

struct Cursor {
    const char* p;
    const char* end;
    int line;
    const char* line_start;
};

[[noreturn]] void fail(const Cursor& c, const char* at, const std::string& msg, bool unsupported = false) {
    throw ParseError{c.line, (int)(at - c.line_start) + 1, msg, unsupported};
}

bool is_space(char ch) { return ch == ' ' || ch == '\t' || ch == '\r'; }

// Token within the current line (stops at '#' or newline).
bool next_token(Cursor& c, const char*& b, const char*& e) {
    while (c.p < c.end && is_space(*c.p)) ++c.p;
    if (c.p >= c.end || *c.p == '\n' || *c.p == '#') return false;
    b = c.p;
    while (c.p < c.end && !is_space(*c.p) && *c.p != '\n' && *c.p != '#') ++c.p;
    e = c.p;
    return true;
}

bool parse_u32(const char* b, const char* e, uint32_t& out) {
    if (b == e || e - b > 10) return false;
    uint64_t v = 0;
    for (const char* q = b; q < e; ++q) {
        if (*q < '0' || *q > '9') return false;
        v = v * 10 + (uint64_t)(*q - '0');
    }
    if (v > 0xFFFFFFFFull) return false;
    out = (uint32_t)v;
    return true;
}

bool parse_double(const char* b, const char* e, double& out) {
    char buf[128];
    size_t n = (size_t)(e - b);
    if (n == 0 || n >= sizeof(buf)) return false;
    memcpy(buf, b, n);
    buf[n] = 0;
    char* endp = nullptr;
    out = strtod(buf, &endp);   // correctly rounded, same value as Python float()
    return endp == buf + n;
}

struct SexprParser {
    Formula& f;
    Cursor& cur;
    const char* p;
    const char* end;

    void skip() {
        while (p < end && (is_space(*p))) ++p;
    }
    uint32_t parse() {
        skip();
        if (p >= end) fail(cur, p, "unexpected end of expression");
        if (*p == '(') {
            ++p;
            skip();
            const char* ob = p;
            while (p < end && !is_space(*p) && *p != '(' && *p != ')') ++p;
            std::string op(ob, p);
            uint8_t code;
            if (op == "and") code = OP_AND;
            else if (op == "or") code = OP_OR;
            else if (op == "xor") code = OP_XOR;
            else if (op == "not") code = OP_NOT;
            else fail(cur, ob, "unknown operator '" + op + "'");
            std::vector<uint32_t> kids;
            for (;;) {
                skip();
                if (p >= end) fail(cur, p, "missing ')'");
                if (*p == ')') { ++p; break; }
                kids.push_back(parse());
            }
            if (code == OP_NOT && kids.size() != 1) fail(cur, ob, "'not' takes one argument");
            if (kids.empty()) fail(cur, ob, "empty (" + op + ")");
            ExprNode nd{code, 0, 0, (uint32_t)f.kids.size(), (uint32_t)kids.size()};
            f.kids.insert(f.kids.end(), kids.begin(), kids.end());
            f.expr.push_back(nd);
            return (uint32_t)f.expr.size() - 1;
        }
        if (*p == ')') fail(cur, p, "unexpected ')'");
        const char* tb = p;
        while (p < end && !is_space(*p) && *p != '(' && *p != ')') ++p;
        if (p - tb < 2 || (*tb != 'b' && *tb != 'a')) fail(cur, tb, "bad token");
        uint32_t idx;
        if (!parse_u32(tb + 1, p, idx)) fail(cur, tb, "bad token");
        ExprNode nd{OP_LIT, (uint8_t)(*tb == 'a'), idx, 0, 0};
        f.expr.push_back(nd);
        return (uint32_t)f.expr.size() - 1;
    }
};

}  // namespace

Formula parse_hsmt(const char* text, size_t len) {
    Formula f;
    Cursor c{text, text + len, 1, text};
    bool have_header = false;
    std::vector<int64_t> atom_slot;          // atom id -> row in CSR (dense check at end)
    struct PendingAtom { uint32_t first, n; double rhs; uint8_t strict; };
    std::vector<PendingAtom> pend;           // in file order
    std::vector<uint32_t> pend_col;
    std::vector<double> pend_val;
    std::vector<uint32_t> pend_id;
    std::vector<int> cons_line;
    std::vector<int> expr_line_of_cons;

    while (c.p < c.end) {
        const char *b, *e;
        if (!next_token(c, b, e)) {
            while (c.p < c.end && *c.p != '\n') ++c.p;  // comment / empty
            if (c.p < c.end) { ++c.p; ++c.line; c.line_start = c.p; }
            continue;
        }
        std::string tag(b, e);
        if (!have_header) {
            const char *b1, *e1, *b2, *e2, *b3, *e3;
            uint32_t nb, nr;
            if (tag != "p" || !next_token(c, b1, e1) || std::string(b1, e1) != "hsmt" || !next_token(c, b2, e2) ||
                !next_token(c, b3, e3) || !parse_u32(b2, e2, nb) || !parse_u32(b3, e3, nr))
                fail(c, b, "expected header 'p hsmt <n_bool> <n_real>'");
            f.n_bool = nb;
            f.n_real = nr;
            have_header = true;
        } else if (tag == "p") {
            fail(c, b, "duplicate header");
        } else if (tag == "a") {
            const char *bi, *ei, *br, *er, *bq, *eq;
            uint32_t id;
            if (!next_token(c, bi, ei) || !parse_u32(bi, ei, id)) fail(c, b, "bad atom id");
            if (!next_token(c, br, er)) fail(c, b, "missing relation");
            std::string rel(br, er);
            if (rel == "=") fail(c, br, "equality atoms unsupported", true);
            if (rel != "<=" && rel != "<" && rel != ">=" && rel != ">") fail(c, br, "bad relation '" + rel + "'");
            double rhs;
            if (!next_token(c, bq, eq) || !parse_double(bq, eq, rhs)) fail(c, b, "bad rhs");
            bool negate = (rel == ">=" || rel == ">");
            uint32_t first = (uint32_t)pend_col.size();
            std::unordered_set<uint32_t> seen;
            const char *bt, *et;
            while (next_token(c, bt, et)) {
                const char* colon = (const char*)memchr(bt, ':', (size_t)(et - bt));
                if (!colon) fail(c, bt, "bad coefficient");
                uint32_t j;
                double q;
                if (!parse_u32(bt, colon, j)) fail(c, bt, "bad variable index");
                if (!parse_double(colon + 1, et, q)) fail(c, bt, "bad coefficient");
                if (j >= f.n_real) fail(c, bt, "real index out of range");
                if (!seen.insert(j).second) fail(c, bt, "duplicate variable in atom");
                if (q == 0.0 || !std::isfinite(q)) fail(c, bt, "coefficients must be finite and nonzero");
                pend_col.push_back(j);
                pend_val.push_back(negate ? -q : q);
            }
            uint32_t n = (uint32_t)pend_col.size() - first;
            if (n == 0) fail(c, b, "atom needs >= 1 coefficient");
            pend.push_back({first, n, negate ? -rhs : rhs, (uint8_t)(rel == "<" || rel == ">")});
            pend_id.push_back(id);
        } else if (tag == "c") {
            const char *bk, *ek;
            if (!next_token(c, bk, ek)) fail(c, b, "constraint too short");
            std::string kind(bk, ek);
            Constraint cs{};
            if (kind == "or") cs.kind = K_OR;
            else if (kind == "card") cs.kind = K_CARD;
            else if (kind == "nae") cs.kind = K_NAE;
            else if (kind == "xor") cs.kind = K_XOR;
            else fail(c, bk, "unknown constraint kind '" + kind + "'");
            const char *bw, *ew;
            if (cs.kind == K_CARD) {
                const char *bt, *et;
                if (!next_token(c, bt, et) || !parse_u32(bt, et, cs.k)) fail(c, b, "card needs an integer threshold");
            }
            if (!next_token(c, bw, ew)) fail(c, b, "missing weight");
            if (!parse_double(bw, ew, cs.weight)) fail(c, bw, "bad weight");
            if (!(cs.weight > 0.0) || !std::isfinite(cs.weight)) fail(c, bw, "weight must be positive and finite", true);
            cs.lit_first = (uint32_t)f.lits.size();
            const char *bt, *et;
            while (next_token(c, bt, et)) {
                if (et - bt < 3 || (bt[0] != '+' && bt[0] != '-') || (bt[1] != 'a' && bt[1] != 'b')) fail(c, bt, "bad literal");
                Lit l{(uint8_t)(bt[1] == 'a'), (uint8_t)(bt[0] == '-'), 0};
                if (!parse_u32(bt + 2, et, l.idx)) fail(c, bt, "bad literal");
                f.lits.push_back(l);
            }
            cs.lit_n = (uint32_t)f.lits.size() - cs.lit_first;
            if (cs.lit_n == 0) fail(c, b, "empty literal list");
            if (cs.kind == K_CARD && cs.k > cs.lit_n) fail(c, b, "card threshold exceeds literal count");
            f.cons.push_back(cs);
            cons_line.push_back(c.line);
        } else if (tag == "e") {
            const char *bw, *ew;
            Constraint cs{};
            cs.kind = K_EXPR;
            if (!next_token(c, bw, ew)) fail(c, b, "expression constraint too short");
            if (!parse_double(bw, ew, cs.weight)) fail(c, bw, "bad weight");
            if (!(cs.weight > 0.0) || !std::isfinite(cs.weight)) fail(c, bw, "weight must be positive and finite", true);
            const char* lb = c.p;
            const char* le = lb;
            while (le < c.end && *le != '\n' && *le != '#') ++le;
            SexprParser sp{f, c, lb, le};
            cs.expr_root = sp.parse();
            sp.skip();
            if (sp.p != le) fail(c, sp.p, "trailing tokens after expression");
            c.p = le;
            f.cons.push_back(cs);
            cons_line.push_back(c.line);
        } else {
            fail(c, b, "unknown line tag '" + tag + "'");
        }
        // the rest of the line must be empty or a comment
        const char *bx, *ex;
        if (next_token(c, bx, ex)) fail(c, bx, "unexpected token");
        while (c.p < c.end && *c.p != '\n') ++c.p;
        if (c.p < c.end) { ++c.p; ++c.line; c.line_start = c.p; }
    }
    if (!have_header) throw ParseError{1, 1, "missing header", false};
    // dense atom ids 0..k-1, stored by id
    size_t k = pend.size();
    std::vector<int64_t> row_of(k, -1);
    for (size_t i = 0; i < k; ++i) {
        if (pend_id[i] >= k || row_of[pend_id[i]] != -1) throw ParseError{1, 1, "atom ids must be dense 0..k-1", false};
        row_of[pend_id[i]] = (int64_t)i;
    }
    f.atom_rowptr.assign(1, 0);
    f.atom_col.reserve(pend_col.size());
    f.atom_val.reserve(pend_val.size());
    f.atom_rhs.resize(k);
    f.atom_strict.resize(k);
    for (size_t id = 0; id < k; ++id) {
        const PendingAtom& pa = pend[(size_t)row_of[id]];
        for (uint32_t t = 0; t < pa.n; ++t) {
            f.atom_col.push_back(pend_col[pa.first + t]);
            f.atom_val.push_back(pend_val[pa.first + t]);
        }
        f.atom_rowptr.push_back((uint32_t)f.atom_col.size());
        f.atom_rhs[id] = pa.rhs;
        f.atom_strict[id] = pa.strict;
    }
    // index ranges of literals / expression leaves
    for (size_t ci = 0; ci < f.cons.size(); ++ci) {
        const Constraint& cs = f.cons[ci];
        auto check = [&](uint8_t kind, uint32_t idx) {
            if (kind == 0 && idx >= f.n_bool) throw ParseError{cons_line[ci], 1, "Boolean index out of range", false};
            if (kind == 1 && idx >= k) throw ParseError{cons_line[ci], 1, "atom index out of range", false};
        };
        if (cs.kind == K_EXPR) {
            std::vector<uint32_t> st{cs.expr_root};
            while (!st.empty()) {
                uint32_t v = st.back();
                st.pop_back();
                const ExprNode& nd = f.expr[v];
                if (nd.op == OP_LIT) check(nd.kind, nd.idx);
                else for (uint32_t t = 0; t < nd.n; ++t) st.push_back(f.kids[nd.first + t]);
            }
        } else {
            for (uint32_t t = 0; t < cs.lit_n; ++t) check(f.lits[cs.lit_first + t].kind, f.lits[cs.lit_first + t].idx);
        }
    }
    return f;
}

}  // namespace fsmt
