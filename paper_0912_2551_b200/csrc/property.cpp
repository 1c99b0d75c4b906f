// property.cpp -- property compiler: BLTLc text (reading R15)
// -> tokens -> AST -> monitor program (leaves + Kleene root, reading R16).
#include <cctype>
#include <cmath>
#include <limits>
#include <sstream>

#include "smc_internal.hpp"

namespace smc {

bool Interval::finite() const { return std::isfinite(hi); }

namespace {

const double INF = std::numeric_limits<double>::infinity();

struct Tok {
    enum T { ID, INT, NUM, OP, END } t;
    std::string s;
    size_t pos;
};

std::vector<Tok> tokenize(const std::string& src) {
    std::vector<Tok> out;
    size_t i = 0;
    while (i < src.size()) {
        char c = src[i];
        if (std::isspace((unsigned char)c)) { ++i; continue; }
        size_t st = i;
        if (std::isalpha((unsigned char)c) || c == '_') {
            while (i < src.size() && (std::isalnum((unsigned char)src[i]) || src[i] == '_')) ++i;
            out.push_back({Tok::ID, src.substr(st, i - st), st});
            continue;
        }
        if (std::isdigit((unsigned char)c) || (c == '.' && i + 1 < src.size() && std::isdigit((unsigned char)src[i + 1]))) {
            bool real = false;
            while (i < src.size() && std::isdigit((unsigned char)src[i])) ++i;
            if (i < src.size() && src[i] == '.') { real = true; ++i; while (i < src.size() && std::isdigit((unsigned char)src[i])) ++i; }
            if (i < src.size() && (src[i] == 'e' || src[i] == 'E')) {
                size_t j = i + 1;
                if (j < src.size() && (src[j] == '+' || src[j] == '-')) ++j;
                if (j < src.size() && std::isdigit((unsigned char)src[j])) {
                    real = true;
                    i = j;
                    while (i < src.size() && std::isdigit((unsigned char)src[i])) ++i;
                }
            }
            out.push_back({real ? Tok::NUM : Tok::INT, src.substr(st, i - st), st});
            continue;
        }
        static const char* two[] = {"<=", ">=", "==", "!="};
        bool matched = false;
        for (const char* op : two)
            if (src.compare(i, 2, op) == 0) { out.push_back({Tok::OP, op, st}); i += 2; matched = true; break; }
        if (matched) continue;
        if (std::string("()[],!&|<>=+-*/").find(c) != std::string::npos) {
            out.push_back({Tok::OP, std::string(1, c), st});
            ++i;
            continue;
        }
        fail(SMC_E_PARSE, "col " + std::to_string(st) + ": unexpected character '" + std::string(1, c) + "'");
    }
    out.push_back({Tok::END, "", src.size()});
    return out;
}

struct Lin {   // sum coef * x + cst
    std::map<int, int64_t> coef;
    int64_t cst = 0;
    bool is_const() const {
        for (auto& kv : coef) if (kv.second != 0) return false;
        return true;
    }
};

enum class NK { ATOM, TRUE_, FALSE_, NOT, AND, OR, X, U, F, G };
struct Node {
    NK k;
    Interval I;
    int a = -1, b = -1;
    int atom = -1;
};

struct Parser {
    std::vector<Tok> tk;
    size_t p = 0;
    const std::vector<std::string>& names;
    std::vector<Node>& nodes;
    std::vector<Atom>& atoms;
    Parser(const std::string& s, const std::vector<std::string>& n, std::vector<Node>& nd, std::vector<Atom>& at)
        : tk(tokenize(s)), names(n), nodes(nd), atoms(at) {}

    const Tok& cur() const { return tk[p]; }
    [[noreturn]] void err(const std::string& what) {
        fail(SMC_E_PARSE, "col " + std::to_string(cur().pos) + ": " + what +
                              (cur().t == Tok::END ? " (at end of input)" : " (at '" + cur().s + "')"));
    }
    bool is_op(const char* s) const { return cur().t == Tok::OP && cur().s == s; }
    bool is_kw(const char* s) const { return cur().t == Tok::ID && cur().s == s; }
    bool accept(const char* s) { if (is_op(s)) { ++p; return true; } return false; }
    void expect(const char* s) { if (!accept(s)) err(std::string("expected '") + s + "'"); }
    int node(Node n) { nodes.push_back(n); return (int)nodes.size() - 1; }

    double number() {
        if (is_kw("inf")) { ++p; return INF; }
        if (cur().t == Tok::INT || cur().t == Tok::NUM) {
            double v = std::strtod(cur().s.c_str(), nullptr);
            ++p;
            return v;
        }
        err("number expected");
    }
    bool interval_ahead() const {
        if (!(is_op("[") || is_op("("))) return false;
        if (is_op("[")) return true;
        // '(' number ','  -> interval, else a parenthesised operand
        return p + 2 < tk.size() && (tk[p + 1].t == Tok::INT || tk[p + 1].t == Tok::NUM ||
                                     (tk[p + 1].t == Tok::ID && tk[p + 1].s == "inf")) &&
               tk[p + 2].t == Tok::OP && tk[p + 2].s == ",";
    }
    Interval interval() {
        Interval I;
        I.lo = 0.0;
        I.hi = INF;
        if (!interval_ahead()) return I;
        I.lo_open = is_op("(");
        ++p;
        I.lo = number();
        expect(",");
        I.hi = number();
        if (is_op("]")) I.hi_open = false;
        else if (is_op(")")) I.hi_open = true;
        else err("expected ']' or ')'");
        ++p;
        if (std::isinf(I.hi)) I.hi_open = false;
        if (!(I.lo >= 0.0) || std::isinf(I.lo) || !(I.hi >= I.lo)) err("interval needs 0 <= a <= b");
        return I;
    }
    // ---- integer-linear forms
    static void add(Lin& l, const Lin& r, int64_t s) {
        for (auto& kv : r.coef) l.coef[kv.first] += s * kv.second;
        l.cst += s * r.cst;
    }
    static void scale(Lin& l, int64_t s) {
        for (auto& kv : l.coef) kv.second *= s;
        l.cst *= s;
    }
    // ---- general val: expr := term (('+'|'-') term)*, term := factor (('*'|'/') factor)*,
    // factor := '-' factor | '(' expr ')' | Int | Real | species | func '(' args ')'
    std::vector<VNode>* vn = nullptr;
    int vadd(VNode n) { vn->push_back(n); return (int)vn->size() - 1; }
    int val_expr() {
        int l = val_term();
        for (;;) {
            VNode n;
            if (accept("+")) n.k = VNode::ADD;
            else if (accept("-")) n.k = VNode::SUB;
            else return l;
            n.a = l;
            n.b = val_term();
            l = vadd(n);
        }
    }
    int val_term() {
        int l = val_factor();
        for (;;) {
            VNode n;
            if (accept("*")) n.k = VNode::MUL;
            else if (accept("/")) n.k = VNode::DIV;
            else return l;
            n.a = l;
            n.b = val_factor();
            l = vadd(n);
        }
    }
    int val_factor() {
        if (accept("-")) { VNode n; n.k = VNode::NEG; n.a = val_factor(); return vadd(n); }
        if (accept("(")) { int e = val_expr(); expect(")"); return e; }
        if (cur().t == Tok::INT) { VNode n; n.k = VNode::INT; n.i = std::stoll(cur().s); ++p; return vadd(n); }
        if (cur().t == Tok::NUM) { VNode n; n.k = VNode::REAL; n.d = std::strtod(cur().s.c_str(), nullptr); ++p; return vadd(n); }
        if (cur().t == Tok::ID) {
            const std::string id = cur().s;
            if (p + 1 < tk.size() && tk[p + 1].t == Tok::OP && tk[p + 1].s == "(") {
                VNode n;
                if (id == "sqrt") n.k = VNode::SQRT;
                else if (id == "abs") n.k = VNode::ABS;
                else if (id == "min") n.k = VNode::MIN;
                else if (id == "max") n.k = VNode::MAX;
                else if (id == "pow") n.k = VNode::POW;
                else err("unknown function '" + id + "'");
                p += 2;
                n.a = val_expr();
                if (n.k == VNode::MIN || n.k == VNode::MAX) { expect(","); n.b = val_expr(); }
                if (n.k == VNode::POW) {
                    expect(",");
                    if (cur().t != Tok::INT) err("integer exponent expected");
                    n.i = std::stoll(cur().s);
                    ++p;
                }
                expect(")");
                return vadd(n);
            }
            for (size_t i = 0; i < names.size(); ++i)
                if (names[i] == id) { VNode n; n.k = VNode::SPECIES; n.s = (int)i; ++p; return vadd(n); }
            err("unknown species '" + id + "'");
        }
        err("expression expected");
    }
    static bool needs_real(const std::vector<VNode>& v, int i) {
        const VNode& n = v[(size_t)i];
        if (n.k == VNode::REAL || n.k == VNode::DIV || n.k >= VNode::SQRT) return true;
        return (n.a >= 0 && needs_real(v, n.a)) || (n.b >= 0 && needs_real(v, n.b));
    }
    // integer tree -> linear form, false when a product of two species terms occurs
    static bool to_lin(const std::vector<VNode>& v, int i, Lin& out) {
        const VNode& n = v[(size_t)i];
        Lin l, r;
        switch (n.k) {
            case VNode::INT: out = Lin(); out.cst = n.i; return true;
            case VNode::SPECIES: out = Lin(); out.coef[n.s] = 1; return true;
            case VNode::NEG: if (!to_lin(v, n.a, out)) return false; scale(out, -1); return true;
            case VNode::ADD: case VNode::SUB:
                if (!to_lin(v, n.a, l) || !to_lin(v, n.b, r)) return false;
                add(l, r, n.k == VNode::ADD ? 1 : -1);
                out = l;
                return true;
            case VNode::MUL:
                if (!to_lin(v, n.a, l) || !to_lin(v, n.b, r)) return false;
                if (l.is_const()) { scale(r, l.cst); out = r; return true; }
                if (r.is_const()) { scale(l, r.cst); out = l; return true; }
                return false;
            default: return false;
        }
    }
    bool cmp(Cmp* c) {
        if (accept("<=")) { *c = Cmp::LE; return true; }
        if (accept(">=")) { *c = Cmp::GE; return true; }
        if (accept("==") || accept("=")) { *c = Cmp::EQ; return true; }
        if (accept("!=")) { *c = Cmp::NE; return true; }
        if (accept("<")) { *c = Cmp::LT; return true; }
        if (accept(">")) { *c = Cmp::GT; return true; }
        return false;
    }
    // ---- formulas: temporal unary > ! > & > U (right assoc) > |
    int disj() {
        int l = until();
        while (accept("|")) { Node n{NK::OR}; n.a = l; n.b = until(); l = node(n); }
        return l;
    }
    int until() {
        int l = conj();
        if (is_kw("U")) {
            ++p;
            Node n{NK::U};
            n.I = interval();
            n.a = l;
            n.b = until();
            return node(n);
        }
        return l;
    }
    int conj() {
        int l = unary();
        while (accept("&")) { Node n{NK::AND}; n.a = l; n.b = unary(); l = node(n); }
        return l;
    }
    int unary() {
        if (accept("!")) { Node n{NK::NOT}; n.a = unary(); return node(n); }
        if (is_kw("F") || is_kw("G") || is_kw("X")) {
            NK k = cur().s == "F" ? NK::F : (cur().s == "G" ? NK::G : NK::X);
            ++p;
            Node n{k};
            n.I = interval();
            n.a = unary();
            return node(n);
        }
        return primary();
    }
    int primary() {
        if (is_kw("true")) { ++p; return node(Node{NK::TRUE_}); }
        if (is_kw("false")) { ++p; return node(Node{NK::FALSE_}); }
        // an atom "lin cmp lin", else "(" formula ")": try the atom, rewind on failure
        size_t save = p;
        Error atom_err{0, ""};
        try {
            std::vector<VNode> v;
            vn = &v;
            const int lv = val_expr();
            Cmp c;
            if (cmp(&c)) {
                const int rv = val_expr();
                Atom at;
                at.op = c;
                Lin l, r;
                if (!needs_real(v, lv) && !needs_real(v, rv) && to_lin(v, lv, l) && to_lin(v, rv, r)) {
                    add(l, r, -1);                       // integer-linear: exact int64 form
                    for (auto& kv : l.coef)
                        if (kv.second != 0) at.coef.push_back(kv);
                    at.cst = l.cst;
                } else {                                 // general val
                    at.general = true;
                    at.real = needs_real(v, lv) || needs_real(v, rv);
                    at.v = v;
                    at.lhs = lv;
                    at.rhs = rv;
                }
                atoms.push_back(at);
                Node n{NK::ATOM};
                n.atom = (int)atoms.size() - 1;
                return node(n);
            }
        } catch (const Error& e) {
            if (e.code == SMC_E_UNSUPPORTED) throw;
            atom_err = e;
        }
        p = save;
        if (accept("(")) {
            int f = disj();
            expect(")");
            return f;
        }
        if (atom_err.code) throw atom_err;
        err("formula expected");
    }
};

// ------------------------------------------------------------ classifier ---
struct Classifier {
    const std::vector<Node>& nodes;
    Property& P;
    Classifier(const std::vector<Node>& n, Property& p) : nodes(n), P(p) {}

    bool boolean(int i) const {
        const Node& n = nodes[(size_t)i];
        switch (n.k) {
            case NK::ATOM: case NK::TRUE_: case NK::FALSE_: return true;
            case NK::NOT: return boolean(n.a);
            case NK::AND: case NK::OR: return boolean(n.a) && boolean(n.b);
            default: return false;
        }
    }
    int bexpr(int i) {
        const Node& n = nodes[(size_t)i];
        BExpr e;
        switch (n.k) {
            case NK::ATOM: e.k = BExpr::ATOM; e.atom = n.atom; break;
            case NK::TRUE_: e.k = BExpr::TRUE_; break;
            case NK::FALSE_: e.k = BExpr::FALSE_; break;
            case NK::NOT: e.k = BExpr::NOT; e.a = bexpr(n.a); break;
            case NK::AND: e.k = BExpr::AND; e.a = bexpr(n.a); e.b = bexpr(n.b); break;
            case NK::OR: e.k = BExpr::OR; e.a = bexpr(n.a); e.b = bexpr(n.b); break;
            default: fail(SMC_E_UNSUPPORTED, "internal: temporal operator in a state formula");
        }
        P.bexprs.push_back(e);
        return (int)P.bexprs.size() - 1;
    }
    static bool zc(const Interval& I) { return I.lo == 0.0 && !I.lo_open && !I.hi_open && I.finite(); }
    int leaf(Leaf L) {
        P.leaves.push_back(L);
        RootExpr r{RootExpr::LEAF};
        r.leaf = (int)P.leaves.size() - 1;
        P.root.push_back(r);
        return (int)P.root.size() - 1;
    }
    int root(int i) {
        const Node& n = nodes[(size_t)i];
        if (boolean(i)) {
            Leaf L{LeafKind::ATOM0};
            L.b1 = bexpr(i);
            return leaf(L);
        }
        switch (n.k) {
            case NK::NOT: { RootExpr r{RootExpr::NOT}; r.a = root(n.a); P.root.push_back(r); return (int)P.root.size() - 1; }
            case NK::AND:
            case NK::OR: {
                RootExpr r{n.k == NK::AND ? RootExpr::AND : RootExpr::OR};
                r.a = root(n.a);
                r.b = root(n.b);
                P.root.push_back(r);
                return (int)P.root.size() - 1;
            }
            case NK::F:
            case NK::G: {
                const Node& in = nodes[(size_t)n.a];
                if (boolean(n.a)) {
                    Leaf L{n.k == NK::F ? LeafKind::F : LeafKind::G};
                    L.I = n.I;
                    L.b1 = bexpr(n.a);
                    return leaf(L);
                }
                if (zc(n.I) && zc(in.I) && boolean(in.a) &&
                    ((n.k == NK::F && in.k == NK::G) || (n.k == NK::G && in.k == NK::F))) {
                    Leaf L{n.k == NK::F ? LeafKind::FG : LeafKind::GF};
                    L.I = n.I;
                    L.J = in.I;
                    L.b1 = bexpr(in.a);
                    return leaf(L);
                }
                break;
            }
            case NK::U: {
                if (boolean(n.a) && boolean(n.b)) {
                    Leaf L{LeafKind::U};
                    L.I = n.I;
                    L.b1 = bexpr(n.a);
                    L.b2 = bexpr(n.b);
                    return leaf(L);
                }
                const Node& l = nodes[(size_t)n.a];
                if (l.k == NK::G && boolean(l.a) && boolean(n.b) && zc(n.I) && zc(l.I)) {
                    Leaf L{LeafKind::GU};
                    L.I = n.I;
                    L.J = l.I;
                    L.b1 = bexpr(l.a);
                    L.b2 = bexpr(n.b);
                    return leaf(L);
                }
                break;
            }
            case NK::X:
                if (boolean(n.a)) {
                    Leaf L{LeafKind::X};
                    L.I = n.I;
                    L.b1 = bexpr(n.a);
                    return leaf(L);
                }
                break;
            default: break;
        }
        fail(SMC_E_UNSUPPORTED, "formula outside the compiled fragment (DESIGN.md §5): nested temporal operators "
                                "other than F[0,a]G[0,b], G[0,a]F[0,b], (G[0,b] .) U[0,c] .");
    }
};

double reach(const std::vector<Node>& nodes, int i, double t_max) {
    const Node& n = nodes[(size_t)i];
    auto hi = [&](const Interval& I) { return std::isfinite(I.hi) ? I.hi : t_max; };
    switch (n.k) {
        case NK::ATOM: case NK::TRUE_: case NK::FALSE_: return 0.0;
        case NK::NOT: return reach(nodes, n.a, t_max);
        case NK::AND: case NK::OR: return std::max(reach(nodes, n.a, t_max), reach(nodes, n.b, t_max));
        case NK::X: case NK::F: case NK::G: return hi(n.I) + reach(nodes, n.a, t_max);
        case NK::U: return hi(n.I) + std::max(reach(nodes, n.a, t_max), reach(nodes, n.b, t_max));
    }
    return 0.0;
}

bool has_unbounded(const std::vector<Node>& nodes, int i) {
    const Node& n = nodes[(size_t)i];
    bool self = (n.k == NK::X || n.k == NK::F || n.k == NK::G || n.k == NK::U) && !std::isfinite(n.I.hi);
    bool ca = n.a >= 0 && has_unbounded(nodes, n.a);
    bool cb = n.b >= 0 && has_unbounded(nodes, n.b);
    return self || ca || cb;
}

uint64_t next_id() {
    static std::mutex mu;
    static uint64_t id = 0;
    std::lock_guard<std::mutex> lk(mu);
    return ++id;
}

}  // namespace

std::unique_ptr<Property> compile_property(const Model& m, const std::string& text,
                                           const std::vector<std::string>& names, double t_max) {
    auto P = std::make_unique<Property>();
    P->id = next_id();
    P->text = text;
    P->N = m.N;
    P->t_max = t_max;
    std::vector<Node> nodes;
    Parser ps(text, names, nodes, P->atoms);
    if (ps.cur().t == Tok::END) ps.err("empty formula");
    int top = ps.disj();
    if (ps.cur().t != Tok::END) ps.err("unexpected trailing input");
    if (has_unbounded(nodes, top) && !(t_max > 0.0))
        fail(SMC_E_UNSUPPORTED, "unbounded temporal operator needs t_max > 0 (pessimistic cut-off, P:314-317)");
    Classifier cl(nodes, *P);
    try {
        P->root_idx = cl.root(top);
    } catch (const Error& e) {
        // outside the streaming templates: literal |= on buffered traces (NEXT-2, reading R23)
        if (e.code != SMC_E_UNSUPPORTED || e.msg.rfind("formula outside the compiled fragment", 0) != 0) throw;
        if (P->atoms.size() > 32) fail(SMC_E_UNSUPPORTED, "nested formula with more than 32 atoms");
        P->literal = true;
        P->leaves.clear();
        P->root.clear();
        P->bexprs.clear();
        P->root_idx = -1;
        for (const Node& n : nodes) {
            LNode l;
            l.k = (LNode::K)(int)n.k;
            l.I = n.I;
            l.a = n.a;
            l.b = n.b;
            l.atom = n.atom;
            P->lnodes.push_back(l);
        }
        P->lroot = top;
    }
    P->horizon = reach(nodes, top, t_max > 0 ? t_max : 0.0);
    if (t_max > 0.0 && t_max < P->horizon) P->horizon = t_max;
    return P;
}

}  // namespace smc

using namespace smc;

extern "C" {

int smc_property_compile(const smc_model* mh, const char* formula, const char* const* species_names, double t_max,
                         smc_property** out) {
    if (!mh || !formula || !out || !(t_max >= 0.0) || std::isinf(t_max)) {
        set_error("smc_property_compile: need model, formula, out and finite t_max >= 0");
        return SMC_E_ARG;
    }
    *out = nullptr;
    try {
        std::vector<std::string> names;
        for (int s = 0; s < mh->m.N; ++s)
            names.push_back(species_names ? std::string(species_names[s]) : "S" + std::to_string(s));
        auto* h = new smc_property();
        try {
            h->p = compile_property(mh->m, formula, names, t_max);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
        return SMC_OK;
    } catch (const Error& e) {
        set_error(e.msg);
        return e.code;
    } catch (const std::exception& e) {
        set_error(e.what());
        return SMC_E_ARG;
    }
}

void smc_property_destroy(smc_property* p) { delete p; }

}  // extern "C"
