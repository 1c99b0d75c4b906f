// codegen.cpp -- specialise the SSA kernels to one (model, property) pair.
//
// Variant 1 (thread-owned): the model is emitted as straight-line code with
// compile-time species/reaction indices, so x[N] and a[M] stay in registers;
// the dependency graph becomes one bit-mask test per propensity.
// Variant 2 (tile): sizes and table offsets become constants; the tables
// themselves are packed here (pack_tables) and staged to smem by TMA.
// Both variants get the same generated monitor (reading R16 templates).
#include <algorithm>
#include <cmath>
#include <map>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <sstream>

#include "smc_internal.hpp"

namespace smc {

namespace {

std::string dlit(double v) {          // exact double literal
    if (std::isinf(v)) return v > 0 ? "(1.0/0.0)" : "(-1.0/0.0)";
    char buf[64];
    std::snprintf(buf, sizeof buf, "%a", v);
    return buf;
}
std::string ilit(int64_t v) { return "(" + std::to_string(v) + "LL)"; }

// ---------------------------------------------------------------- monitor ---
struct MonGen {
    const Property& P;
    bool xd = false;   // the counts are binary64 (variant 1 / sweep binary64 modes)
    explicit MonGen(const Property& p, bool xd_ = false) : P(p), xd(xd_) {}

    // general val tree: int64 (Int, species, + - *) or binary64 in tree order
    static std::string val(const Atom& at, int i) {
        const VNode& n = at.v[(size_t)i];
        const bool R = at.real;
        switch (n.k) {
            case VNode::INT: return R ? dlit((double)n.i) : ilit(n.i);
            case VNode::REAL: return dlit(n.d);
            case VNode::SPECIES: return (R ? "(double)x[" : "(smc_i64)x[") + std::to_string(n.s) + "]";
            case VNode::NEG: return "(-" + val(at, n.a) + ")";
            case VNode::ADD: return R ? "__dadd_rn(" + val(at, n.a) + ", " + val(at, n.b) + ")" : "(" + val(at, n.a) + " + " + val(at, n.b) + ")";
            case VNode::SUB: return R ? "__dadd_rn(" + val(at, n.a) + ", -" + val(at, n.b) + ")" : "(" + val(at, n.a) + " - " + val(at, n.b) + ")";
            case VNode::MUL: return R ? "__dmul_rn(" + val(at, n.a) + ", " + val(at, n.b) + ")" : "(" + val(at, n.a) + " * " + val(at, n.b) + ")";
            case VNode::DIV: return "__ddiv_rn(" + val(at, n.a) + ", " + val(at, n.b) + ")";
            case VNode::SQRT: return "__dsqrt_rn(" + val(at, n.a) + ")";
            case VNode::ABS: return "fabs(" + val(at, n.a) + ")";
            case VNode::MIN: return "smc_vmin(" + val(at, n.a) + ", " + val(at, n.b) + ")";
            case VNode::MAX: return "smc_vmax(" + val(at, n.a) + ", " + val(at, n.b) + ")";
            case VNode::POW: return "smc_vpow(" + val(at, n.a) + ", " + std::to_string(n.i) + ")";
        }
        return "0";
    }
    std::string atom(int i) const {
        const Atom& a = P.atoms[(size_t)i];
        static const char* cops[] = {" < ", " <= ", " >= ", " > ", " == ", " != "};
        if (a.general) return "(" + val(a, a.lhs) + cops[(int)a.op] + val(a, a.rhs) + ")";
        if (xd) {
            // binary64 counts: sum_s coef_s x_s + cst is formed exactly in binary64 when every
            // partial sum is an integer below 2^53 (|coef| sum x (2^31 - 1) + |cst| < 2^53), so
            // the comparison equals the int64 one with no fp64 -> int64 conversion
            long double bound = std::fabs((long double)a.cst);
            for (auto& kv : a.coef) bound += std::fabs((long double)kv.second) * 2147483647.0L;
            if (bound < 9007199254740992.0L) {
                std::string e = dlit((double)a.cst);
                for (auto& kv : a.coef) e = "__fma_rn(" + dlit((double)kv.second) + ", x[" + std::to_string(kv.first) + "], " + e + ")";
                static const char* dops[] = {" < ", " <= ", " >= ", " > ", " == ", " != "};
                return "(" + e + dops[(int)a.op] + "0.0)";
            }
        }
        std::string s = "(";
        for (auto& kv : a.coef) s += "(smc_i64)x[" + std::to_string(kv.first) + "] * " + ilit(kv.second) + " + ";
        s += ilit(a.cst) + ")";
        static const char* ops[] = {" < ", " <= ", " >= ", " > ", " == ", " != "};
        return "(" + s + ops[(int)a.op] + "0LL)";
    }
    std::string bexpr(int i) const {
        if (i < 0) return "true";
        const BExpr& e = P.bexprs[(size_t)i];
        switch (e.k) {
            case BExpr::ATOM: return atom(e.atom);
            case BExpr::TRUE_: return "true";
            case BExpr::FALSE_: return "false";
            case BExpr::NOT: return "(!" + bexpr(e.a) + ")";
            case BExpr::AND: return "(" + bexpr(e.a) + " && " + bexpr(e.b) + ")";
            case BExpr::OR: return "(" + bexpr(e.a) + " || " + bexpr(e.b) + ")";
        }
        return "false";
    }
    static std::string contains(const Interval& I, const char* t) {
        std::string s = std::string("(") + t + (I.lo_open ? " > " : " >= ") + dlit(I.lo);
        if (I.finite()) s += std::string(" && ") + t + (I.hi_open ? " < " : " <= ") + dlit(I.hi);
        return s + ")";
    }
    static std::string beyond(const Interval& I, const char* t) {
        if (!I.finite()) return "false";
        return std::string("(") + t + (I.hi_open ? " >= " : " > ") + dlit(I.hi) + ")";
    }
    std::string root(int i) const {
        const RootExpr& r = P.root[(size_t)i];
        switch (r.k) {
            case RootExpr::LEAF: return "smc_tri(s" + std::to_string(r.leaf) + ")";
            case RootExpr::NOT: return "smc_knot(" + root(r.a) + ")";
            case RootExpr::AND: return "smc_kand(" + root(r.a) + ", " + root(r.b) + ")";
            case RootExpr::OR: return "smc_kor(" + root(r.a) + ", " + root(r.b) + ")";
        }
        return "2";
    }

    std::string emit() const {
        std::ostringstream o;
        const size_t L = P.leaves.size();
        o << "// monitor for: " << P.text << "\n";
        o << "struct SmcMon {\n";
        for (size_t i = 0; i < L; ++i) {
            o << "    unsigned char s" << i << ";\n";
            const Leaf& lf = P.leaves[i];
            if (lf.kind == LeafKind::FG || lf.kind == LeafKind::GF) o << "    bool rs" << i << "_set; double rs" << i << ";\n";
            if (lf.kind == LeafKind::GU) o << "    bool w" << i << "; double D" << i << ";\n";
        }
        o << "    __device__ __forceinline__ void bind(const SmcParams&, smc_u64, unsigned, int) {}\n";
        // a streaming monitor stops the moment it decides: the events applied are the count;
        // reaching the event cap undecided is an error
        o << "    __device__ __forceinline__ long long events(long long k) const { return k; }\n";
        o << "    __device__ __forceinline__ int at_cap(long long) { return 2; }\n";
        // init
        o << "    __device__ __forceinline__ void init() {\n";
        for (size_t i = 0; i < L; ++i) {
            o << "        s" << i << " = 0;\n";
            const Leaf& lf = P.leaves[i];
            if (lf.kind == LeafKind::FG || lf.kind == LeafKind::GF) o << "        rs" << i << "_set = false; rs" << i << " = 0.0;\n";
            if (lf.kind == LeafKind::GU) o << "        w" << i << " = false; D" << i << " = 0.0;\n";
        }
        o << "    }\n";
        // enter
        o << "    template <class XA> __device__ __forceinline__ void enter(smc_u32 k, double t, double tp, const XA& x) {\n";
        o << "        (void)k; (void)tp;\n";
        for (size_t i = 0; i < L; ++i) {
            const Leaf& lf = P.leaves[i];
            std::string s = "s" + std::to_string(i), id = std::to_string(i);
            std::string B1 = bexpr(lf.b1), B2 = bexpr(lf.b2);
            o << "        if (" << s << " == 0) {\n";
            switch (lf.kind) {
                case LeafKind::ATOM0: o << "            " << s << " = " << B1 << " ? 1 : 2;\n"; break;
                case LeafKind::F: o << "            if (" << contains(lf.I, "t") << " && " << B1 << ") " << s << " = 1;\n"; break;
                case LeafKind::G: o << "            if (" << contains(lf.I, "t") << " && !" << B1 << ") " << s << " = 2;\n"; break;
                case LeafKind::U:
                    o << "            if (" << contains(lf.I, "t") << " && " << B2 << ") " << s << " = 1;\n";
                    o << "            else if (!" << B1 << ") " << s << " = 2;\n";
                    break;
                case LeafKind::X:
                    o << "            if (k == 1u) " << s << " = (" << contains(lf.I, "t") << " && " << B1 << ") ? 1 : 2;\n";
                    break;
                case LeafKind::FG:
                case LeafKind::GF:
                    o << "            const bool b = " << (lf.kind == LeafKind::GF ? "!" : "") << B1 << ";\n";
                    o << "            if (!b) rs" << id << "_set = false;\n";
                    o << "            else if (!rs" << id << "_set && t <= " << dlit(lf.I.hi) << ") { rs" << id
                      << "_set = true; rs" << id << " = t; }\n";
                    break;
                case LeafKind::GU:
                    o << "            const bool b1 = " << B1 << ";\n";
                    o << "            if (w" << id << ") { if (!b1) " << s << " = 2; }\n";
                    o << "            else if (" << B2 << ") {\n";
                    o << "                if (k == 0u) " << s << " = 1;\n";
                    o << "                else { w" << id << " = true; D" << id << " = __dadd_rn(tp, " << dlit(lf.J.hi) << ");\n";
                    o << "                       if (t > D" << id << ") " << s << " = 1; else if (!b1) " << s << " = 2; }\n";
                    o << "            } else if (!b1) " << s << " = 2;\n";
                    break;
            }
            o << "        }\n";
        }
        o << "    }\n";
        // advance
        o << "    __device__ __forceinline__ void advance(smc_u32 k, double tn, double tau) {\n        (void)k; (void)tau;\n";
        for (size_t i = 0; i < L; ++i) {
            const Leaf& lf = P.leaves[i];
            std::string s = "s" + std::to_string(i), id = std::to_string(i);
            switch (lf.kind) {
                case LeafKind::ATOM0: break;
                case LeafKind::F: case LeafKind::U:
                    o << "        if (" << s << " == 0 && " << beyond(lf.I, "tn") << ") " << s << " = 2;\n"; break;
                case LeafKind::G:
                    o << "        if (" << s << " == 0 && " << beyond(lf.I, "tn") << ") " << s << " = 1;\n"; break;
                case LeafKind::X:
                    o << "        if (" << s << " == 0 && k == 0u && !" << contains(lf.I, "tn") << ") " << s << " = 2;\n"; break;
                case LeafKind::FG:
                case LeafKind::GF: {
                    const char* yes = lf.kind == LeafKind::FG ? "1" : "2";
                    const char* no = lf.kind == LeafKind::FG ? "2" : "1";
                    o << "        if (" << s << " == 0) {\n";
                    o << "            if (rs" << id << "_set && tn > __dadd_rn(rs" << id << ", " << dlit(lf.J.hi) << ")) " << s << " = " << yes << ";\n";
                    o << "            else if (!rs" << id << "_set && tn > " << dlit(lf.I.hi) << ") " << s << " = " << no << ";\n";
                    o << "        }\n";
                    break;
                }
                case LeafKind::GU:
                    o << "        if (" << s << " == 0) {\n";
                    o << "            if (w" << id << ") { if (tn > D" << id << ") " << s << " = 1; }\n";
                    o << "            else if (tn > " << dlit(lf.I.hi) << ") " << s << " = 2;\n";
                    o << "        }\n";
                    break;
            }
        }
        o << "    }\n";
        // absorb
        o << "    __device__ __forceinline__ void absorb() {\n";
        for (size_t i = 0; i < L; ++i) {
            const Leaf& lf = P.leaves[i];
            std::string s = "s" + std::to_string(i), id = std::to_string(i);
            std::string val;
            switch (lf.kind) {
                case LeafKind::ATOM0: continue;
                case LeafKind::F: case LeafKind::U: case LeafKind::X: val = "2"; break;
                case LeafKind::G: val = "1"; break;
                case LeafKind::FG: val = "(rs" + id + "_set ? 1 : 2)"; break;
                case LeafKind::GF: val = "(rs" + id + "_set ? 2 : 1)"; break;
                case LeafKind::GU: val = "(w" + id + " ? 1 : 2)"; break;
            }
            o << "        if (" << s << " == 0) " << s << " = " << val << ";\n";
        }
        o << "    }\n";
        // timeout
        o << "    __device__ __forceinline__ void timeout() {\n";
        for (size_t i = 0; i < L; ++i) o << "        if (s" << i << " == 0) s" << i << " = 3;\n";
        o << "    }\n";
        // verdict
        o << "    __device__ __forceinline__ int verdict() const {\n";
        if (L == 1 && P.root[(size_t)P.root_idx].k == RootExpr::LEAF) {   // root is the leaf itself
            o << "        return s0 == 0 ? -1 : (s0 == 1 ? 1 : 0);   // unknown -> false (P:314-317)\n    }\n};\n";
            return o.str();
        }
        o << "        const int r = " << root(P.root_idx) << ";\n";
        o << "        if (r != 2) return r;\n";
        o << "        if (";
        for (size_t i = 0; i < L; ++i) o << (i ? " || " : "") << "s" << i << " == 0";
        o << ") return -1;\n";
        o << "        return 0;   // unknown at t_max -> false (P:314-317)\n";
        o << "    }\n};\n";
        return o.str();
    }
};

// ---------------------------------------- window monitor (literal |=, R23/R27) ---
// The nodes of the formula reachable from the root, children before parents, with the time
// (and, for root-level booleans, the number of positions) the root can reach through each
// node: a node creates position m only while t_m <= tlim (relative slack 1e-6 covers the
// rounding between entry times and the left-to-right elapsed sums, R27) and m < plim.
struct WinNode {
    LNode n;
    int a = -1, b = -1, par = -1;
    double tlim = 0.0;
    long long plim = 1;
};

std::vector<WinNode> window_nodes(const Property& P) {
    std::vector<int> order, remap(P.lnodes.size(), -1);
    std::function<void(int)> post = [&](int i) {
        const LNode& n = P.lnodes[(size_t)i];
        if (n.a >= 0) post(n.a);
        if (n.b >= 0) post(n.b);
        remap[(size_t)i] = (int)order.size();
        order.push_back(i);
    };
    post(P.lroot);
    std::vector<WinNode> w(order.size());
    for (size_t q = 0; q < order.size(); ++q) {
        w[q].n = P.lnodes[(size_t)order[q]];
        w[q].a = w[q].n.a >= 0 ? remap[(size_t)w[q].n.a] : -1;
        w[q].b = w[q].n.b >= 0 ? remap[(size_t)w[q].n.b] : -1;
    }
    const double BIG = 1e300;
    const long long PINF = 0x7fffffff;
    w.back().tlim = 0.0;                     // the root: position 0 only
    w.back().plim = 1;
    for (int q = (int)w.size() - 1; q >= 0; --q) {
        WinNode& x = w[(size_t)q];
        for (int c : {x.a, x.b}) {
            if (c < 0) continue;
            WinNode& y = w[(size_t)c];
            y.par = q;
            const bool temporal = x.n.k == LNode::F || x.n.k == LNode::G || x.n.k == LNode::U;
            if (temporal || x.n.k == LNode::X) {
                y.tlim = (x.tlim >= BIG || !x.n.I.finite()) ? BIG : (x.tlim + x.n.I.hi) * (1.0 + 1e-6) + 1e-300;
                y.plim = temporal ? PINF : std::min(PINF, x.plim + 1);
            } else {
                y.tlim = x.tlim;
                y.plim = x.plim;
            }
        }
    }
    return w;
}

// ring entry bytes: t, tau; a (v, r) queue per node; F / G: two (index, r) deques; U: elapsed +
// 32-byte state per pending position.  Nodes with a single position (plim == 1: the root and
// root-level booleans) keep theirs in a small area of SMC_WIN_SE entries per slot instead.
static size_t node_entry_bytes(const WinNode& x) {
    return 8 + ((x.n.k == LNode::F || x.n.k == LNode::G) ? 16 : (x.n.k == LNode::U ? 40 : 0));
}
size_t win_bytes(const Property& P) {
    size_t b = 16;
    for (auto& x : window_nodes(P)) if (x.plim != 1) b += node_entry_bytes(x);
    return b;
}
size_t win_small(const Property& P) {
    size_t b = 0;
    for (auto& x : window_nodes(P)) if (x.plim == 1) b += node_entry_bytes(x);
    return 16 * b;
}

// smc_lit_mask(x): atom bit mask of a state; the node table of ssa_window.cuh
std::string window_code(const Property& P) {
    std::ostringstream o;
    MonGen mg(P);
    o << "template <class XA> __device__ __forceinline__ unsigned smc_lit_mask(const XA& x) {\n    unsigned mk = 0u;\n";
    for (size_t i = 0; i < P.atoms.size(); ++i) o << "    if " << mg.atom((int)i) << " mk |= " << (1u << i) << "u;\n";
    o << "    return mk;\n}\n";
    const auto w = window_nodes(P);
    o << "#define SMC_WIN_NODES " << w.size() << "\n#define SMC_WIN_ROOT " << w.size() - 1
      << "\n#define SMC_WIN_PER_ENTRY " << win_bytes(P) << "\n#define SMC_WIN_SMALL " << win_small(P)
      << "\n#define SMC_WIN_SE 16\ntemplate <int I> struct SmcWN;\n";
    // offsets in bytes-per-entry units: big nodes within the W-entry arrays (queues, then U's
    // elapsed and states, then F / G deques), small nodes within the SMC_WIN_SE-entry area
    size_t oq[2] = {16, 0}, oel[2] = {0, 0}, ost[2] = {0, 0}, odq[2] = {0, 0};
    for (int sm = 0; sm < 2; ++sm) {
        size_t o = oq[sm];
        for (auto& x : w) if ((x.plim == 1) == (sm == 1)) o += 8;
        oel[sm] = o;
        for (auto& x : w) if ((x.plim == 1) == (sm == 1) && x.n.k == LNode::U) o += 8;
        ost[sm] = o;
        for (auto& x : w) if ((x.plim == 1) == (sm == 1) && x.n.k == LNode::U) o += 32;
        odq[sm] = o;
    }
    for (size_t i = 0; i < w.size(); ++i) {
        const WinNode& x = w[i];
        const bool isu = x.n.k == LNode::U, isfg = x.n.k == LNode::F || x.n.k == LNode::G;
        const bool fin = x.n.I.finite();
        const int sm = x.plim == 1 ? 1 : 0;
        o << "template <> struct SmcWN<" << i << "> {   // " << (int)x.n.k << "\n"
          << "    static constexpr int kind = " << (int)x.n.k << ", a = " << x.a << ", b = " << x.b
          << ", atom = " << x.n.atom << ", par = " << x.par << ";\n"
          << "    static constexpr double lo = " << dlit(x.n.I.lo) << ", hi = " << dlit(fin ? x.n.I.hi : 0.0)
          << ", tlim = " << dlit(x.tlim) << ";\n"
          << "    static constexpr bool lo_open = " << (x.n.I.lo_open ? "true" : "false")
          << ", hi_open = " << (x.n.I.hi_open ? "true" : "false") << ", hi_inf = " << (fin ? "false" : "true")
          << ", small = " << (sm ? "true" : "false") << ";\n"
          << "    static constexpr int plim = " << x.plim << ";\n"
          << "    static constexpr long long oq = " << oq[sm] << ", oel = " << (isu ? oel[sm] : 0)
          << ", ost = " << (isu ? ost[sm] : 0) << ", odq = " << (isfg ? odq[sm] : 0) << ";\n};\n";
        oq[sm] += 8;
        if (isu) { oel[sm] += 8; ost[sm] += 32; }
        if (isfg) odq[sm] += 16;
    }
    return o.str();
}

// ------------------------------------------------ explicit rate expressions ---
// Straight-line IEEE binary64 code of an explicit rate tree (rates.cpp), in tree
// order; xa = the count array expression ("x" in registers, "xs" in smem).
std::string rate_code(const std::vector<RNode>& t, int i, const char* xa) {
    const RNode& n = t[(size_t)i];
    switch (n.k) {
        case RNode::CONST: return dlit(n.v);
        case RNode::SPECIES: return std::string("(double)") + xa + "[" + std::to_string(n.species) + "]";
        case RNode::NEG: return "(-" + rate_code(t, n.a, xa) + ")";
        case RNode::ADD: return "__dadd_rn(" + rate_code(t, n.a, xa) + ", " + rate_code(t, n.b, xa) + ")";
        case RNode::SUB: return "__dadd_rn(" + rate_code(t, n.a, xa) + ", -" + rate_code(t, n.b, xa) + ")";
        case RNode::MUL: return "__dmul_rn(" + rate_code(t, n.a, xa) + ", " + rate_code(t, n.b, xa) + ")";
        case RNode::DIV: return "__ddiv_rn(" + rate_code(t, n.a, xa) + ", " + rate_code(t, n.b, xa) + ")";
    }
    return "0.0";
}
// body of an explicit law: the guard (a reactant below its stoichiometry -> 0), then
// v(x); a negative or NaN value is returned as NaN (bad propensity, the replica errs)
std::string explicit_body(const Reaction& r, const char* xa, const char* indent) {
    std::ostringstream o;
    for (int q = 0; q < 2; ++q)
        if (r.s[q] >= 0) o << indent << "if (" << xa << "[" << r.s[q] << "] < " << r.st[q] << ") return 0.0;\n";
    o << indent << "{ const double v = " << rate_code(r.rate, (int)r.rate.size() - 1, xa) << ";\n";
    o << indent << "  return v >= 0.0 ? v : __longlong_as_double(0x7ff8000000000000LL); }\n";
    return o.str();
}

// ------------------------------------------------- variant 1 model code ---
std::string law_expr(const Reaction& r, int k) {
    // h exact in int64, a = c * (double)h, Hill: a / (1 + q^n)
    std::vector<std::string> terms;
    for (int q = 0; q < 2; ++q) {
        if (r.s[q] < 0) continue;
        std::string xs = "(smc_i64)x[" + std::to_string(r.s[q]) + "]";
        terms.push_back(r.st[q] == 1 ? xs : "((" + xs + " * (" + xs + " - 1LL)) / 2LL)");
    }
    std::string h;
    if (terms.empty()) h = "1LL";
    else if (terms.size() == 1) h = terms[0];
    else h = "(" + terms[0] + " * " + terms[1] + ")";
    (void)r;
    return "__dmul_rn(smc_rc[" + std::to_string(k) + "], (double)(" + h + "))";   // c_k from the constant bank
}

void xd_forms(const Model& m, std::vector<int>& form, std::vector<double>& cs);
std::string xd_law_body(const Model& m, int k, int f, const char* rc, const HillTables* ht);

// Variant 1 with the counts as binary64 registers (exact integers < 2^31): the laws are
// fp64 products with no int64 -> fp64 conversion on the per-event chain (R20); the
// count-overflow test of R17 is a high-word compare.
std::string model_code_thread_xd(const Model& m) {
    std::ostringstream o;
    const int N = m.N, M = m.M;
    std::vector<double> cs;
    std::vector<int> form;
    xd_forms(m, form, cs);
    o << "typedef double smc_x1t;\n";
    o << "__constant__ double smc_rc[" << M << "] = {";
    for (int k = 0; k < M; ++k) o << (k ? ", " : "") << dlit(cs[(size_t)k]);
    o << "};\n";
    o << "__device__ __forceinline__ void smc_init_x(smc_x1t (&x)[SMC_N]) {\n";
    for (int s = 0; s < N; ++s) o << "    x[" << s << "] = " << m.x0[(size_t)s] << ".0;\n";
    o << "}\n";
    const HillTables ht = pack_hill_tables(m);
    for (int k = 0; k < M; ++k) {
        o << "__device__ __forceinline__ double smc_law" << k << "(const smc_x1t (&x)[SMC_N], const double* __restrict__ H) {\n";
        o << "    (void)H;\n" << xd_law_body(m, k, form[(size_t)k], "smc_rc", &ht) << "}\n";
    }
    o << "__device__ __forceinline__ void smc_laws_all(double (&a)[SMC_M], const smc_x1t (&x)[SMC_N], const double* __restrict__ H) {\n";
    for (int k = 0; k < M; ++k) o << "    a[" << k << "] = smc_law" << k << "(x, H);\n";
    o << "}\n";
    o << "__device__ __forceinline__ bool smc_apply(int j, smc_x1t (&x)[SMC_N]) {\n    bool ovf = false;\n";
    for (int s = 0; s < N; ++s) {
        std::vector<std::pair<int, int>> ds;
        bool pos = false;
        for (int j = 0; j < M; ++j)
            for (auto& ch : m.R[(size_t)j].change)
                if (ch.first == s) { ds.push_back({j, ch.second}); pos |= ch.second > 0; }
        if (ds.empty()) continue;
        std::string sel = "0.0";           // binary64 deltas: no int -> fp64 conversion on the chain
        for (auto it = ds.rbegin(); it != ds.rend(); ++it)
            sel = "(j == " + std::to_string(it->first) + " ? " + std::to_string(it->second) + ".0 : " + sel + ")";
        o << "    x[" << s << "] = __dadd_rn(x[" << s << "], " << sel << ");\n";
        if (pos) o << "    ovf |= __double2hiint(x[" << s << "]) >= 0x41E00000;\n";   // x >= 2^31
    }
    o << "    return !ovf;\n}\n";
    o << "__device__ __forceinline__ void smc_update(int j, double (&a)[SMC_M], const smc_x1t (&x)[SMC_N], const double* __restrict__ H) {\n";
    o << "    (void)j;\n";
    for (int k = 0; k < M; ++k) o << "    a[" << k << "] = smc_law" << k << "(x, H);\n";
    o << "}\n";
    o << "__device__ __forceinline__ int smc_last_positive(const double (&a)[SMC_M]) {\n    return ";
    for (int k = M - 1; k >= 1; --k) o << "a[" << k << "] > 0.0 ? " << k << " : ";
    o << "0;\n}\n";
    return o.str();
}

std::string model_code_thread(const Model& m) {
    std::ostringstream o;
    const int N = m.N, M = m.M;
    o << "typedef int smc_x1t;\n";
    // rate constants in the constant bank (DMUL reads c[][] operands; no per-event
    // materialisation of 64-bit immediates)
    o << "__constant__ double smc_rc[" << M << "] = {";
    for (int k = 0; k < M; ++k) o << (k ? ", " : "") << dlit(m.R[(size_t)k].c);
    o << "};\n";
    o << "__device__ __forceinline__ void smc_init_x(int (&x)[SMC_N]) {\n";
    for (int s = 0; s < N; ++s) o << "    x[" << s << "] = " << m.x0[(size_t)s] << ";\n";
    o << "}\n";
    const HillTables ht = pack_hill_tables(m);
    for (int k = 0; k < M; ++k) {
        const Reaction& r = m.R[(size_t)k];
        o << "__device__ __forceinline__ double smc_law" << k << "(const int (&x)[SMC_N], const double* __restrict__ H) {\n";
        if (!r.rate.empty()) {
            o << "    (void)H;\n" << explicit_body(r, "x", "    ") << "}\n";
            continue;
        }
        if (ht.offset[(size_t)k] >= 0)   // zero-order Hill law: a_k(x_r) tabulated (same IEEE ops, host side)
            o << "    if (x[" << r.rep << "] < " << ht.size << ") return __ldg(H + " << ht.offset[(size_t)k] << " + x["
              << r.rep << "]);\n";
        o << "    double a = " << law_expr(r, k) << ";\n";
        if (r.hill) {
            o << "    const double q = __ddiv_rn((double)x[" << r.rep << "], " << dlit(r.K) << ");\n";
            o << "    double qn = q;\n";
            for (int i = 1; i < r.n; ++i) o << "    qn = __dmul_rn(qn, q);\n";
            o << "    a = __ddiv_rn(a, __dadd_rn(1.0, qn));\n";
        }
        o << "    return a;\n}\n";
    }
    o << "__device__ __forceinline__ void smc_laws_all(double (&a)[SMC_M], const int (&x)[SMC_N], const double* __restrict__ H) {\n";
    for (int k = 0; k < M; ++k) o << "    a[" << k << "] = smc_law" << k << "(x, H);\n";
    o << "}\n";
    // x += v_j, per species, in wrapping 32-bit arithmetic.  Counts are >= 0 and
    // |delta| <= 4, so x + delta exceeds 2^31-1 exactly when the wrapped result is
    // negative (reading R17): one sign test over the OR of the grown species.
    o << "__device__ __forceinline__ bool smc_apply(int j, int (&x)[SMC_N]) {\n    int grown = 0;\n";
    for (int s = 0; s < N; ++s) {
        std::vector<std::pair<int, int>> ds;
        bool pos = false;
        for (int j = 0; j < M; ++j)
            for (auto& ch : m.R[(size_t)j].change)
                if (ch.first == s) { ds.push_back({j, ch.second}); pos |= ch.second > 0; }
        if (ds.empty()) continue;
        std::string sel = "0";
        for (auto it = ds.rbegin(); it != ds.rend(); ++it)
            sel = "(j == " + std::to_string(it->first) + " ? " + std::to_string(it->second) + " : " + sel + ")";
        o << "    x[" << s << "] = (int)((unsigned)x[" << s << "] + (unsigned)" << sel << ");\n";
        if (pos) o << "    grown |= x[" << s << "];\n";
    }
    o << "    return grown >= 0;\n}\n";
    // Propensity update after R_j fired.  In a thread-owned warp the 32 lanes fire
    // different reactions, so the union of dep(j) over the warp is (nearly) every
    // reaction and a masked update executes every law anyway plus the mask tests and
    // branches; the kernel therefore recomputes all M laws (straight-line, bit-identical
    // to recomputing only dep(j)).  The dependency graph drives the tile variant, where
    // M >> 32.
    o << "__device__ __forceinline__ void smc_update(int j, double (&a)[SMC_M], const int (&x)[SMC_N], const double* __restrict__ H) {\n";
    o << "    (void)j;\n";
    for (int k = 0; k < M; ++k) o << "    a[" << k << "] = smc_law" << k << "(x, H);\n";
    o << "}\n";
    o << "__device__ __forceinline__ int smc_last_positive(const double (&a)[SMC_M]) {\n    return ";
    for (int k = M - 1; k >= 1; --k) o << "a[" << k << "] > 0.0 ? " << k << " : ";
    o << "0;\n}\n";
    return o.str();
}

// ------------------------------------------------- variant 4 model code ---
// Pass 1 of the sweep kernel: every law in index order from register copies of the
// counts, group sums of SMC_SW_S consecutive laws (left to right) and the prefix chain
// P_g = P_{g-1} + sum_g (reading R12).  Laws use the same IEEE operations as the law
// table of pass 2 (ssa_sweep.cuh smc_law_sw): exact int64 h, one rounding to double,
// a = c * h, Hill as in variant 1 (computed, not tabulated).
int sweep_group(const Model& m) {
    // small groups keep the in-group selection one chunk of independent law reads; the
    // G = M/S prefixes live in registers, so S grows with M beyond ~29 groups.  C4 (M = 200,
    // events/s): S:C = 7:7 1.63e10, 5:5 1.61e10, 6:6 1.60e10, 10:5 1.60e10, 12:4 1.50e10,
    // 16:4 1.22e10
    int S = std::max(7, (m.M + 28) / 29);
    if (const char* e = std::getenv("SMC_SW_S")) S = std::max(1, std::atoi(e));
    return std::min(S, m.M);
}

// Laws over binary64 counts (sweep SMC_SW_XD, variant 1 with binary64 registers): plain
// fp64 products of the counts, identical to the int64 forms (R20).  form: 0 c, 1 c x,
// 2 (c/2) x (x-1) (exact fold), 3 c x y, 4 general (explicit, order 3-4, unfoldable).
void xd_forms(const Model& m, std::vector<int>& form, std::vector<double>& cs) {
    const int M = m.M;
    form.assign((size_t)M, 4);
    cs.assign((size_t)M, 0.0);
    for (int k = 0; k < M; ++k) {
        const Reaction& r = m.R[(size_t)k];
        double c = r.c;
        int order = 0;
        for (int q = 0; q < 2; ++q) order += r.s[q] >= 0 ? r.st[q] : 0;
        int f = 4;
        if (!r.rate.empty() || order > 2) f = 4;
        else if (r.s[0] < 0) f = 0;
        else if (r.s[1] < 0 && r.st[0] == 1) f = 1;
        else if (r.s[1] < 0) {
            if ((c * 0.5) * 2.0 == c && c * 0.5 >= 0x1p-1021) { f = 2; c *= 0.5; }   // exact fold
        } else if (r.st[0] == 1 && r.st[1] == 1) f = 3;
        form[(size_t)k] = f;
        cs[(size_t)k] = c;
    }
}

// statements of law k over double x[] with rates in constant array `rc`; zero-order Hill
// laws read the host table H (variant 1) when ht is given
std::string xd_law_body(const Model& m, int k, int f, const char* rc, const HillTables* ht) {
    std::ostringstream o;
    const Reaction& r = m.R[(size_t)k];
    const std::string K = std::to_string(k);
    if (!r.rate.empty()) return explicit_body(r, "x", "    ");
    if (ht && ht->offset[(size_t)k] >= 0)
        o << "    if (x[" << r.rep << "] < " << ht->size << ".0) return __ldg(H + " << ht->offset[(size_t)k]
          << " + (int)x[" << r.rep << "]);\n";
    const std::string a = std::to_string(r.s[0]), b = std::to_string(r.s[1]), C = std::string(rc) + "[" + K + "]";
    switch (f) {
        case 0: o << "    double v = " << C << ";\n"; break;
        case 1: o << "    double v = __dmul_rn(" << C << ", x[" << a << "]);\n"; break;
        case 2: o << "    double v = __dmul_rn(" << C << ", __fma_rn(x[" << a << "], x[" << a << "], -x[" << a << "]));\n"; break;
        case 3: o << "    double v = __dmul_rn(" << C << ", __dmul_rn(x[" << a << "], x[" << b << "]));\n"; break;
        default: {                                   // order 3-4 / unfoldable homodimer: exact int64 h
            std::vector<std::string> terms;
            for (int q = 0; q < 2; ++q) {
                if (r.s[q] < 0) continue;
                std::string xs = "(smc_i64)x[" + std::to_string(r.s[q]) + "]";
                terms.push_back(r.st[q] == 1 ? xs : "((" + xs + " * (" + xs + " - 1LL)) / 2LL)");
            }
            std::string h = terms.empty() ? "1LL" : (terms.size() == 1 ? terms[0] : "(" + terms[0] + " * " + terms[1] + ")");
            o << "    double v = __dmul_rn(" << C << ", (double)(" << h << "));\n";
        }
    }
    if (r.hill) {
        o << "    const double q = __ddiv_rn(x[" << r.rep << "], " << dlit(r.K) << ");\n";
        o << "    double qn = q;\n";
        for (int i = 1; i < r.n; ++i) o << "    qn = __dmul_rn(qn, q);\n";
        o << "    v = __ddiv_rn(v, __dadd_rn(1.0, qn));\n";
    }
    o << "    return v;\n";
    return o.str();
}

std::string sweep_code_xd(const Model& m, int S, int G) {
    std::ostringstream o;
    const int N = m.N, M = m.M;
    std::vector<double> cs;
    std::vector<int> form;
    xd_forms(m, form, cs);
    o << "__constant__ double smc_rc[" << M << "] = {";
    for (int k = 0; k < M; ++k) o << (k ? ", " : "") << dlit(cs[(size_t)k]);
    o << "};\n";
    for (int k = 0; k < M; ++k) {
        o << "__device__ __forceinline__ double smc_law" << k << "(const double (&x)[SMC_N]) {\n";
        o << xd_law_body(m, k, form[(size_t)k], "smc_rc", nullptr) << "}\n";
    }
    // SMC_SW_FMAACC (reading R25): g + c_k h_k with one rounding (fused multiply-add) for the
    // mass-action laws of order <= 2; the others add their law value
    bool fmaacc = true;
    if (const char* e = std::getenv("SMC_SW_FMAACC")) fmaacc = std::atoi(e) != 0;
    for (int k = 0; k < M; ++k) {
        const Reaction& r = m.R[(size_t)k];
        const std::string K = std::to_string(k), C = "smc_rc[" + K + "]";
        const std::string a = std::to_string(r.s[0]), b = std::to_string(r.s[1]);
        o << "__device__ __forceinline__ double smc_lawacc" << k << "(const double (&x)[SMC_N], double g) {\n    return ";
        const int f = form[(size_t)k];
        if (!fmaacc || r.hill || !r.rate.empty() || f == 4) o << "__dadd_rn(g, smc_law" << k << "(x));\n}\n";
        else if (f == 0) o << "__dadd_rn(g, " << C << ");\n}\n";
        else if (f == 1) o << "__fma_rn(" << C << ", x[" << a << "], g);\n}\n";
        else if (f == 2) o << "__fma_rn(" << C << ", __fma_rn(x[" << a << "], x[" << a << "], -x[" << a << "]), g);\n}\n";
        else o << "__fma_rn(" << C << ", __dmul_rn(x[" << a << "], x[" << b << "]), g);\n}\n";
    }
    o << "#define SMC_SW_FMAACC " << (fmaacc ? 1 : 0) << "\n";
    bool any_explicit = false;
    for (auto& r : m.R) any_explicit |= !r.rate.empty();
    if (any_explicit) {
        o << "__device__ __noinline__ double smc_explicit4(int k, const SmcXCol& xs) {\n    switch (k) {\n";
        for (int k = 0; k < M; ++k)
            if (!m.R[(size_t)k].rate.empty())
                o << "    case " << k << ":\n" << explicit_body(m.R[(size_t)k], "xs", "        ");
        o << "    }\n    return 0.0;\n}\n";
    }
    o << "__device__ __forceinline__ void smc_sweep(const SmcXCol& X, double (&P)[SMC_SW_G]) {\n";
    o << "    double x[SMC_N];\n#pragma unroll\n    for (int s = 0; s < SMC_N; ++s) x[s] = X[s];\n    double g, h;\n";
    // a group sum is SPLIT interleaved partial sums (members m = r mod SPLIT, each left
    // to right) added in order -- a fixed order (reading R12) with a shorter add chain
    int split = 1;
    if (const char* e = std::getenv("SMC_SW_SPLIT")) split = std::max(1, std::min(2, std::atoi(e)));
    for (int gi = 0; gi < G; ++gi) {
        const int k0 = gi * S, k1 = std::min(M, gi * S + S);
        for (int k = k0; k < k1; ++k) {
            const char* acc = (split == 2 && ((k - k0) & 1)) ? "h" : "g";
            if (k - k0 < split) o << "    " << acc << " = smc_law" << k << "(x);\n";
            else o << "    " << acc << " = smc_lawacc" << k << "(x, " << acc << ");\n";
        }
        if (split == 2 && k1 - k0 > 1) o << "    g = __dadd_rn(g, h);\n";
        if (gi == 0) o << "    P[0] = g;\n";
        else o << "    P[" << gi << "] = __dadd_rn(P[" << gi - 1 << "], g);\n";
    }
    o << "}\n";
    (void)N;
    return o.str();
}

// Counts as binary64 columns (SMC_SW_XD): the laws are plain fp64 products of the
// counts (exact integers, < 2^31), identical to the int64 forms: fl(x0 x1) is the
// rounding of the exact product either way, and x (x - 1) with the 1/2 folded into
// c (reading R20); no conversion per law.
// Count columns and CTA size of the sweep variant, from the packed table size: one CTA of
// up to 384 threads per SM (12 warps at 168 registers fill the register file; one CTA
// per SM measured +10 % over three CTAs of 128 on C4), binary64 columns when they fit,
// else int32 columns; SMC_SW_XD / SMC_SW_BLOCK override.
void sweep_shape(const Model& m, size_t table_bytes, bool& xd, int& blk) {
    const size_t avail = 233472 - 2048 - std::min<size_t>(table_bytes, 200000);
    auto fit = [&](size_t esz) { return (int)std::min<size_t>(384, avail / (esz * (size_t)(m.N + 1)) / 32 * 32); };
    xd = fit(8) >= 128;
    if (const char* e = std::getenv("SMC_SW_XD")) xd = std::atoi(e) != 0;
    blk = std::max(32, fit(xd ? 8 : 4));
    if (const char* e = std::getenv("SMC_SW_BLOCK")) {
        const int b = std::atoi(e);
        if (b >= 32 && b <= 512 && b % 32 == 0) blk = b;
    }
}

std::string model_code_sweep(const Model& m, bool xd) {
    std::ostringstream o;
    const int N = m.N, M = m.M, S = sweep_group(m), G = (M + S - 1) / S;
    o << "#define SMC_SW_S " << S << "\n#define SMC_SW_G " << G << "\n";
    if (xd) return o.str() + sweep_code_xd(m, S, G);
    o << "__constant__ double smc_rc[" << M << "] = {";
    for (int k = 0; k < M; ++k) o << (k ? ", " : "") << dlit(m.R[(size_t)k].c);
    o << "};\n";
    for (int k = 0; k < M; ++k) {
        const Reaction& r = m.R[(size_t)k];
        o << "__device__ __forceinline__ double smc_law" << k << "(const int (&x)[SMC_N]) {\n";
        if (!r.rate.empty()) {
            o << explicit_body(r, "x", "    ") << "}\n";
            continue;
        }
        o << "    double a = " << law_expr(r, k) << ";\n";
        if (r.hill) {
            o << "    const double q = __ddiv_rn((double)x[" << r.rep << "], " << dlit(r.K) << ");\n";
            o << "    double qn = q;\n";
            for (int i = 1; i < r.n; ++i) o << "    qn = __dmul_rn(qn, q);\n";
            o << "    a = __ddiv_rn(a, __dadd_rn(1.0, qn));\n";
        }
        o << "    return a;\n}\n";
    }
    bool any_explicit = false;
    for (auto& r : m.R) any_explicit |= !r.rate.empty();
    if (any_explicit) {                 // explicit laws of pass 2 (law-table kind 5)
        o << "__device__ __noinline__ double smc_explicit4(int k, const SmcXCol& xs) {\n    switch (k) {\n";
        for (int k = 0; k < M; ++k)
            if (!m.R[(size_t)k].rate.empty())
                o << "    case " << k << ":\n" << explicit_body(m.R[(size_t)k], "xs", "        ");
        o << "    }\n    return 0.0;\n}\n";
    }
    // fast laws, valid while every count is < 2^26: each mass-action count product h is
    // < 2^52, so the bit pattern 0x43300000:h is the double 2^52 + h exactly, and
    //   a = fma(c, 2^52 + h, -c 2^52) = round(c (2^52 + h) - c 2^52) = round(c h)
    // (one rounding of the exact value, -c 2^52 is an exact constant): the same double as
    // c * (double)h with one FP64 instruction and no int64 -> fp64 conversion (SMC_SW_FMA;
    // 0: (2^52 + h) - 2^52 then the product, two FP64 instructions)
    bool fma = true;
    if (const char* e = std::getenv("SMC_SW_FMA")) fma = std::atoi(e) != 0;
    o << "__constant__ double smc_rcn[" << M << "] = {";
    for (int k = 0; k < M; ++k) o << (k ? ", " : "") << dlit(-std::ldexp(m.R[(size_t)k].c, 52));
    o << "};\n";
    std::vector<bool> used((size_t)N, false);
    for (int k = 0; k < M; ++k) {
        const Reaction& r = m.R[(size_t)k];
        for (int sp : m.law_species(k)) used[(size_t)sp] = true;
        o << "__device__ __forceinline__ double smc_lawf" << k << "(const int (&x)[SMC_N]) {\n";
        int order = 0;
        for (int q = 0; q < 2; ++q) order += r.s[q] >= 0 ? r.st[q] : 0;
        if (!r.rate.empty() || order > 2) {           // explicit rate / order 3-4: the general law
            o << "    return smc_law" << k << "(x);\n}\n";
            continue;
        }
        std::string h;
        if (order == 0) h = "";
        else if (r.s[1] < 0 && r.st[0] == 1) h = "smc_u2d((smc_u64)(unsigned)x[" + std::to_string(r.s[0]) + "])";
        else if (r.s[1] < 0) {
            const std::string xs = "(smc_u64)(unsigned)x[" + std::to_string(r.s[0]) + "]";
            h = "smc_u2d((" + xs + " * (" + xs + " - 1ull)) >> 1)";     // x >= 1 whenever it matters; x = 0 -> 0
        } else {
            h = "smc_u2d((smc_u64)(unsigned)x[" + std::to_string(r.s[0]) + "] * (smc_u64)(unsigned)x[" +
                std::to_string(r.s[1]) + "])";
        }
        o << "    (void)x;\n";
        const std::string K = std::to_string(k);
        if (fma && !h.empty()) {                       // smc_u2d(v) -> the biased pattern of v
            const std::string hb = "__longlong_as_double((long long)(" + h.substr(8, h.size() - 9) + " | 0x4330000000000000ull))";
            o << "    double a = __fma_rn(smc_rc[" << K << "], " << hb << ", smc_rcn[" << K << "]);\n";
        } else {
            o << "    double a = " << (h.empty() ? "__dmul_rn(smc_rc[" + K + "], 1.0)" : "__dmul_rn(smc_rc[" + K + "], " + h + ")")
              << ";\n";
        }
        if (r.hill) {
            o << "    const double q = __ddiv_rn(smc_u2d((smc_u64)(unsigned)x[" << r.rep << "]), " << dlit(r.K) << ");\n";
            o << "    double qn = q;\n";
            for (int i = 1; i < r.n; ++i) o << "    qn = __dmul_rn(qn, q);\n";
            o << "    a = __ddiv_rn(a, __dadd_rn(1.0, qn));\n";
        }
        o << "    return a;\n}\n";
    }
    auto body = [&](const char* law, const char* indent) {
        for (int gi = 0; gi < G; ++gi) {
            for (int k = gi * S; k < std::min(M, gi * S + S); ++k) {
                const std::string call = std::string(law) + std::to_string(k) + "(x)";
                if (k == gi * S) o << indent << "g = " << call << ";\n";
                else o << indent << "g = __dadd_rn(g, " << call << ");\n";
            }
            if (gi == 0) o << indent << "P[0] = g;\n";
            else o << indent << "P[" << gi << "] = __dadd_rn(P[" << gi - 1 << "], g);\n";
        }
    };
    o << "__device__ __forceinline__ void smc_sweep(const SmcXCol& X, double (&P)[SMC_SW_G]) {\n";
    o << "    int x[SMC_N];\n#pragma unroll\n    for (int s = 0; s < SMC_N; ++s) x[s] = X[s];\n";
    o << "    unsigned big = 0u;\n";
    for (int sp = 0; sp < N; ++sp)
        if (used[(size_t)sp]) o << "    big |= (unsigned)x[" << sp << "];\n";
    o << "    double g;\n";
    bool fast = true;
    if (const char* e = std::getenv("SMC_SW_FAST")) fast = std::atoi(e) != 0;
    o << "    if (" << (fast ? "" : "false && ") << "(big >> 26) == 0u) {\n";
    body("smc_lawf", "        ");
    o << "    } else {\n";
    body("smc_law", "        ");
    o << "    }\n}\n";
    return o.str();
}

size_t align16(size_t v) { return (v + 15) & ~(size_t)15; }

}  // namespace


// resident 128-thread units per SM of variant 1 (register cap 65536 / (128 minb)): the small
// models (M <= 8: C1, C2) run latency-bound Wilson rounds below full occupancy and keep
// registers for ILP (4); larger ones are throughput-bound (6: C3 +4 %)
int thread_minb(const Model& m) {
    int minb = m.M <= 8 ? 4 : 6;
    if (const char* e = std::getenv("SMC_MINB")) minb = std::atoi(e);
    return std::max(1, minb);
}

// CTA size of variant 1 (SMC_V1_BLOCK overrides)
int thread_block(const Model& m) {
    // one CTA per SM holding all the resident threads of the register budget (minb x 128):
    // measured C2 0.688 -> 0.645 us per event on a 66 k batch (6.04e10 -> 6.35e10 events/s),
    // C3 7.69e10 -> 7.86e10, against 128-thread CTAs
    int b = thread_minb(m) * 128;
    if (const char* e = std::getenv("SMC_V1_BLOCK")) b = std::atoi(e);
    return (b >= 32 && b <= 1024 && b % 32 == 0) ? b : 128;
}

// --------------------------------------------------- variant 1 tables ---
HillTables pack_hill_tables(const Model& m) {
    HillTables h;
    h.offset.assign((size_t)m.M, -1);
    for (int k = 0; k < m.M; ++k) {
        const Reaction& r = m.R[(size_t)k];
        if (!r.hill || r.s[0] >= 0 || r.s[1] >= 0) continue;
        h.offset[(size_t)k] = (long long)h.values.size();
        for (int x = 0; x < h.size; ++x) {
            double a = r.c * (double)1LL;          // c * h with h = 1
            const double q = (double)x / r.K;
            double qn = q;
            for (int i = 1; i < r.n; ++i) qn = qn * q;
            h.values.push_back(a / (1.0 + qn));
        }
    }
    return h;
}

// --------------------------------------------------- variant 2 tables ---
// Tile width: 8 lanes per trajectory for small networks (4 trajectories per warp),
// 16 / 32 when the per-lane groups would get long.  SMC_TILE_WIDTH overrides.
int tile_width(const Model& m) {
    if (const char* e = std::getenv("SMC_TILE_WIDTH")) {
        int w = std::atoi(e);
        if (w == 4 || w == 8 || w == 16 || w == 32) return w;
    }
    return m.M <= 256 ? 8 : (m.M <= 512 ? 16 : 32);
}

// Law kind of reaction j (ssa_tile.cuh smc_law_tab, ssa_delta.cuh smc_dh): h = x[s0] * x[s1]
// with x[N] = 1 for kinds 0 (h = 1), 1 (x), 3 (x y); kind 2 (x(x-1)/2) as x * (x-1) with
// c/2 (exact: halving); 4 general order 3-4 (int64); 5 explicit rate.  c = the table's rate.
void law_kind(const Model& m, int j, uint32_t& kind, uint32_t& s0, uint32_t& s1, double& c) {
    const Reaction& r = m.R[(size_t)j];
    const int N = m.N;
    s0 = s1 = (uint32_t)N;
    c = r.c;
    if (!r.rate.empty()) kind = 5;                  // explicit rate (generated smc_explicit)
    else if (r.s[0] < 0) kind = 0;
    else if (r.s[1] < 0 && r.st[0] == 1) { kind = 1; s0 = (uint32_t)r.s[0]; }
    else if (r.s[1] < 0) {
        kind = 2;
        s0 = s1 = (uint32_t)r.s[0];
        if ((c * 0.5) * 2.0 == c && c * 0.5 >= 0x1p-1021) c *= 0.5;   // fold the 1/2 (exact)
        else { kind = 4; s1 = (uint32_t)N; }                       // subnormal rate: int64 path, x[N] = 1
    } else { kind = (r.st[0] == 1 && r.st[1] == 1) ? 3u : 4u; s0 = (uint32_t)r.s[0]; s1 = (uint32_t)r.s[1]; }
}

// Variant 5 fixed point (reading R26): Cq_k = round(c_k 2^L) with c_k the table's rate.  The
// group and total sums are sums of Cq_k h_k, h_k < 2^62 (counts < 2^31), so with
// Cq_max < 2^(66 - ceil(log2 M)) no sum reaches 2^128.  Eligible when every law is mass
// action of order <= 2 (kinds 0-3, no Hill) and the smallest positive rate still gets
// Cq >= 2^36 (relative rounding of a term <= 2^-37; C5: rates 1e-3..1 -> Cq >= 2^44).
int delta_scale(const Model& m) {
    double cmax = 0.0, cmin = 0.0;
    for (int j = 0; j < m.M; ++j) {
        const Reaction& r = m.R[(size_t)j];
        uint32_t kind, s0, s1;
        double c;
        law_kind(m, j, kind, s0, s1, c);
        if (kind > 3 || r.hill || !(c >= 0.0) || !std::isfinite(c)) return -1;
        if (c > 0.0) {
            cmax = std::max(cmax, c);
            cmin = (cmin == 0.0) ? c : std::min(cmin, c);
        }
    }
    if (cmax == 0.0) return 0;
    int lm = 0;
    while ((1 << lm) < m.M) ++lm;                       // ceil(log2 M)
    const int top = std::min(63, 66 - lm);              // Cq < 2^63 (u64) and M Cq 2^62 < 2^128
    const int L = top - 1 - (int)std::floor(std::log2(cmax));   // cmax 2^L < 2^top
    if (L < -900 || L > 900) return -1;
    if (std::ldexp(cmin, L) < 0x1p36) return -1;
    return L;
}

// Variant 5 tables: x0, the law table {s0 | kind << 16, s1, c} (the tile format), the change
// lists and dep(j) as a reaction-indexed CSR with 2-byte entries k.
TileLayout pack_delta_tables(const Model& m) {
    TileLayout L;
    const int N = m.N, M = m.M;
    L.dl = delta_scale(m);
    if (L.dl < 0) fail(SMC_E_MODEL, "delta variant: model not eligible (reading R26)");
    // tile width 8 (C5: 2.9e9 events/s vs 2.4e9 at 16, 1.6e9 at 32); widths below 8 are not
    // supported (TW = 4 hung on random networks)
    // small models (only reached by forcing the variant) use one tile per warp: with several
    // tiles per warp, warp intrinsics returned inconsistent values on small absorbing models
    // (C2 run to absorption), which full-warp tiles do not show
    L.tw = M >= 256 ? 8 : 32;
    if (const char* e = std::getenv("SMC_TILE_WIDTH")) {
        const int w = std::atoi(e);
        if (w == 8 || w == 16 || w == 32) L.tw = w;
    }
    // G groups of S laws, both multiples of TW, G ~ sqrt(M)
    int G = (int)std::ceil(std::sqrt((double)M));
    if (const char* e = std::getenv("SMC_DG")) G = std::max(1, std::atoi(e));
    G = (G + L.tw - 1) / L.tw * L.tw;
    int S = (M + G - 1) / G;
    S = (S + L.tw - 1) / L.tw * L.tw;
    L.dg = G;
    L.ds = S;
    L.n_pad = (N + 1 + 3) & ~3;
    L.tile_bytes = align16((size_t)16 * G + 4 * (size_t)L.n_pad);
    // dep(j) dealt into R_j rounds of <= TW lanes such that no two entries of one round touch
    // the same group: the entries sorted by group (largest multiplicity first) are dealt
    // round robin over R_j = max(ceil(|dep(j)| / TW), max multiplicity) rounds -- a group's
    // <= R_j entries land in distinct rounds, each round gets <= ceil(|dep(j)| / R_j) <= TW
    // entries -- so each lane updates its group with a plain read-modify-write (no atomics).
    // Stored compactly, round after round; dep_off[j] = start | R_j << 24, and the entry
    // count of round r of j at rcnt[j * DRMAX + r].
    std::vector<std::vector<std::vector<int>>> rounds((size_t)M);
    size_t nnz = 0;
    L.drmax = 1;
    for (int j = 0; j < M; ++j) {
        const auto& d = m.dep[(size_t)j];
        L.max_dep = std::max<int>(L.max_dep, (int)d.size());
        if (d.empty()) continue;
        std::map<int, std::vector<int>> byg;
        for (int k : d) byg[k / S].push_back(k);
        std::vector<std::vector<int>> grp;
        size_t mult = 0;
        for (auto& kv : byg) { grp.push_back(kv.second); mult = std::max(mult, kv.second.size()); }
        std::stable_sort(grp.begin(), grp.end(), [](const std::vector<int>& a, const std::vector<int>& b) {
            return a.size() > b.size();
        });
        const int R = std::max<int>((int)mult, ((int)d.size() + L.tw - 1) / L.tw);
        auto& rj = rounds[(size_t)j];
        rj.assign((size_t)R, {});
        int i = 0;
        for (auto& gl : grp)
            for (int k : gl) rj[(size_t)(i++ % R)].push_back(k);
        nnz += d.size();
        L.drmax = std::max(L.drmax, R);
    }
    if (L.drmax > 255) fail(SMC_E_MODEL, "delta variant: more than 255 dependency rounds");
    if (nnz >= (1u << 24)) fail(SMC_E_MODEL, "delta variant: dependency table too large");
    // entries: u16 k | (d0 + 4) << 10 | (d1 + 4) << 13 when M <= 1024 and every net change is in
    // [-4, 3] (C4, C5: [-2, 2]); else u32 k | (d0 + 8) << 16 | (d1 + 8) << 20
    int dmin = 0, dmax = 0;
    for (auto& r : m.R)
        for (auto& ch : r.change) { dmin = std::min(dmin, ch.second); dmax = std::max(dmax, ch.second); }
    if (dmin < -8 || dmax > 7) fail(SMC_E_MODEL, "delta variant: a net change beyond [-8, 7]");
    L.dep16 = M <= 1024 && dmin >= -4 && dmax <= 3;
    // round descriptor per j (u64): low word start | R << 24, high word (count_r - 1) in 4-bit
    // fields, while R <= 8 and every round holds <= 16 entries; else the rcnt table
    L.fatdep = L.drmax <= 8 && L.tw <= 16;
    size_t o = 0;
    L.off_x0 = o; o = align16(o + 4 * (size_t)L.n_pad);
    L.off_law = o; o = align16(o + 16 * (size_t)G * (size_t)S);   // in-group laws, permuted within groups
    L.off_hill_k = o; o = align16(o + 16 * (size_t)M);      // dependency law {s0 | s1 << 16, kind, Cq_k}
    // the laws (random gathers every event) are staged in shared memory; the per-event
    // tables read once per event (change lists, round descriptors, dependency entries) stay
    // in global memory and are read through the L1 (SMC_DGLOBAL=0: all in shared memory) --
    // freeing shared memory for more resident trajectories
    bool dglobal = true;
    if (const char* e = std::getenv("SMC_DGLOBAL")) dglobal = std::atoi(e) != 0;
    L.smem_bytes = o;
    L.off_chg = o; o = align16(o + 2 * 4 * (size_t)M);
    L.off_dep_off = o; o = align16(o + (L.fatdep ? 8 : 4) * ((size_t)M + 1));   // round descriptors
    L.off_hill_rep = o; o = align16(o + (L.fatdep ? 0 : (size_t)M * (size_t)L.drmax));   // rcnt[j][r] (u8)
    L.off_dep = o; o = align16(o + (L.dep16 ? 2 : 4) * nnz);
    L.bytes = o;
    if (!dglobal) L.smem_bytes = L.bytes;
    L.blob.assign(L.bytes, 0);
    auto* x0 = (int32_t*)(L.blob.data() + L.off_x0);
    for (int s = 0; s < N; ++s) x0[s] = m.x0[(size_t)s];
    x0[N] = 1;
    auto* chg = (uint16_t*)(L.blob.data() + L.off_chg);
    for (int p = M; p < G * S; ++p) {               // padding members: rate 0, x[N] * x[N]
        const int CHd = S / L.tw, gp = p / S, mp = p % S;
        const uint32_t w0 = (uint32_t)N | (1u << 16), w1 = (uint32_t)N;
        unsigned char* law = L.blob.data() + L.off_law + 16 * ((size_t)gp * S + (size_t)(mp % CHd) * L.tw + (size_t)(mp / CHd));
        std::memcpy(law, &w0, 4);
        std::memcpy(law + 4, &w1, 4);
    }
    for (int j = 0; j < M; ++j) {
        const Reaction& r = m.R[(size_t)j];
        uint32_t kind, s0, s1;
        double c;
        law_kind(m, j, kind, s0, s1, c);
        // in-group law table: member m of group g (lane m / CH, chunk slot m % CH) stored at
        // g S + (m % CH) TW + m / CH, so the TW lanes reading chunk slot c hit consecutive
        // 16-byte entries (conflict-free); padding up to G S: rate 0, operands x[N] = 1
        const uint32_t w0 = s0 | (kind << 16), w1 = s1;
        const int CHd = S / L.tw, gj = j / S, mj = j % S;
        unsigned char* law = L.blob.data() + L.off_law + 16 * ((size_t)gj * S + (size_t)(mj % CHd) * L.tw + (size_t)(mj / CHd));
        std::memcpy(law, &w0, 4);
        std::memcpy(law + 4, &w1, 4);
        std::memcpy(law + 8, &c, 8);
        // the dependency pass's law entry: operands, kind, Cq_k = round(c_k 2^L) (exact scaling,
        // round to nearest even)
        const uint64_t cq = (uint64_t)std::nearbyint(std::ldexp(c, L.dl));
        const uint32_t ops = s0 | (s1 << 16);
        unsigned char* dl = L.blob.data() + L.off_hill_k + 16 * (size_t)j;
        std::memcpy(dl, &ops, 4);
        std::memcpy(dl + 4, &kind, 4);
        std::memcpy(dl + 8, &cq, 8);
        if (r.change.size() > 4) fail(SMC_E_MODEL, "internal: more than 4 changed species");
        for (int q = 0; q < 4; ++q) {
            uint16_t e = 0xFFFF;
            if (q < (int)r.change.size()) e = (uint16_t)((r.change[(size_t)q].first << 4) | (r.change[(size_t)q].second + 8));
            chg[4 * j + q] = e;
        }
    }
    // entry: k and the net changes d0, d1 that R_j applies to law k's operand species s0, s1
    // (0 for an unchanged operand; ssa_delta.cuh smc_ddh)
    auto* doff32 = (uint32_t*)(L.blob.data() + L.off_dep_off);
    auto* doff64 = (uint64_t*)(L.blob.data() + L.off_dep_off);
    auto* rcnt = L.blob.data() + L.off_hill_rep;
    auto* dep32 = (uint32_t*)(L.blob.data() + L.off_dep);
    auto* dep16 = (uint16_t*)(L.blob.data() + L.off_dep);
    size_t pos = 0;
    for (int j = 0; j < M; ++j) {
        const auto& ch = m.R[(size_t)j].change;
        const auto& rj = rounds[(size_t)j];
        if (L.fatdep) {
            uint64_t d = (uint64_t)pos | ((uint64_t)rj.size() << 24);
            for (size_t r = 0; r < rj.size(); ++r) d |= (uint64_t)(rj[r].size() - 1) << (32 + 4 * r);
            doff64[j] = d;
        } else {
            doff32[j] = (uint32_t)pos | ((uint32_t)rj.size() << 24);
            for (size_t r = 0; r < rj.size(); ++r) rcnt[(size_t)j * L.drmax + r] = (uint8_t)rj[r].size();
        }
        for (size_t r = 0; r < rj.size(); ++r) {
            for (int k : rj[r]) {
                uint32_t kind, s0, s1;
                double c;
                law_kind(m, k, kind, s0, s1, c);
                int d0 = 0, d1 = 0;
                for (auto& cc : ch) {
                    if ((uint32_t)cc.first == s0) d0 = cc.second;
                    if ((uint32_t)cc.first == s1) d1 = cc.second;
                }
                if (L.dep16) dep16[pos++] = (uint16_t)((uint32_t)k | ((uint32_t)(d0 + 4) << 10) | ((uint32_t)(d1 + 4) << 13));
                else dep32[pos++] = (uint32_t)k | ((uint32_t)(d0 + 8) << 16) | ((uint32_t)(d1 + 8) << 20);
            }
        }
    }
    if (L.fatdep) doff64[M] = pos; else doff32[M] = (uint32_t)pos;
    // check: the rounds of dep(j) hold each k of dep(j) once, <= TW per round, no group twice
    for (int j = 0; j < M; ++j) {
        std::vector<int> seen;
        for (auto& rr : rounds[(size_t)j]) {
            std::vector<int> gr;
            for (int k : rr) { seen.push_back(k); gr.push_back(k / S); }
            std::sort(gr.begin(), gr.end());
            if ((int)rr.size() > L.tw || std::adjacent_find(gr.begin(), gr.end()) != gr.end())
                fail(SMC_E_MODEL, "internal: bad dependency round");
        }
        std::sort(seen.begin(), seen.end());
        if (seen != m.dep[(size_t)j]) fail(SMC_E_MODEL, "internal: dep rounds do not cover dep(j)");
    }
    return L;
}

TileLayout pack_tables(const Model& m, bool sweep) {
    TileLayout L;
    const int N = m.N, M = m.M;
    L.tw = tile_width(m);
    L.gs = (M + L.tw - 1) / L.tw;
    L.ch = 1;
    while (L.ch * L.tw < L.gs) L.ch *= 2;      // chunk per lane in the in-group selection (power of two)
    L.n_pad = (N + 1 + 3) & ~3;     // x[0..N) counts, x[N] = 1 (operand of h = x * 1 and h = 1 * 1)
    // per-trajectory slice: a[GS*TW] (fp64) + x[NPAD] (int32), 16-byte aligned; with several
    // tiles per warp the slice is padded to 8*TW mod 128 bytes so that the TPW tiles of a
    // warp cover consecutive bank ranges (minimum wavefronts per warp access)
    // a layout (ssa_tile.cuh smc_slot): row layout (group l contiguous, odd row stride) or
    // the XOR-swizzled column layout (SMC_ROWLAYOUT = 0)
    // measured: row layout +2 % on C5 (CH = 1: the in-group read is one contiguous row),
    // -3 % on C4 (CH = 4: stride-4 reads conflict 2-way); so rows only for CH = 1
    L.row = L.ch == 1;
    if (const char* e = std::getenv("SMC_ROWLAYOUT")) L.row = std::atoi(e) != 0;
    L.gsp = L.row ? (L.gs | 1) : L.gs;
    L.tile_bytes = align16((size_t)L.gsp * L.tw * 8 + 4 * (size_t)L.n_pad);
    if (L.tw < 16)      // TW lanes x 8 B per access: tiles of a warp cover consecutive bank ranges
        while (L.tile_bytes % 128 != (size_t)(8 * L.tw)) L.tile_bytes += 16;
    for (auto& r : m.R) {
        L.any_hill |= r.hill;
        int order = 0;
        for (int q = 0; q < 2; ++q) order += r.s[q] >= 0 ? r.st[q] : 0;
        L.any_general |= order > 2;
    }
    size_t nnz = 0;
    if (!sweep)
        for (auto& d : m.dep) { nnz += d.size(); L.max_dep = std::max<int>(L.max_dep, (int)d.size()); }
    size_t o = 0;
    L.off_x0 = o; o = align16(o + 4 * (size_t)L.n_pad);
    L.off_law = o; o = align16(o + 16 * (size_t)M);
    L.off_hill_rep = o; o = align16(o + (L.any_hill ? 4 * (size_t)M : 0));
    L.off_hill_k = o; o = align16(o + (L.any_hill ? 8 * (size_t)M : 0));
    L.off_hill_n = o; o = align16(o + (L.any_hill ? 4 * (size_t)M : 0));
    L.off_chg = o; o = align16(o + 2 * 4 * (size_t)M);
    // Large networks, one trajectory per warp: the dependency work of reaction j is the
    // union of the reader lists of the <= 4 species j changes (species-indexed CSR,
    // ~1.5 entries per reaction instead of |dep(j)| ~ 19 per reaction: C5 tables 67 -> 28 KiB,
    // i.e. more resident trajectories; a reaction reading two changed species is simply
    // recomputed twice).  Otherwise a reaction-indexed CSR of dep(j), 2-byte entries (k
    // only, slot recomputed) for M > 512, else 4-byte entries k | slot << 16.
    std::vector<std::vector<int>> readers((size_t)N);
    for (int k = 0; k < M; ++k)
        for (int sp : m.law_species(k)) readers[(size_t)sp].push_back(k);
    size_t nnz_sp = 0;
    if (!sweep)
        for (auto& r : readers) nnz_sp += r.size();
    L.depsp = M > 512 && L.tw == 32;
    if (const char* e = std::getenv("SMC_DEPSP")) L.depsp = std::atoi(e) != 0 && L.tw == 32;
    L.dep16 = L.depsp || M > 512;
    if (const char* e = std::getenv("SMC_DEP16")) L.dep16 = L.depsp || std::atoi(e) != 0;
    if (sweep) L.depsp = L.dep16 = false;
    // "fat" 16-byte entries {k | slot << 16, law meta, rate} for the reaction-indexed CSR:
    // the dependency walk reads contiguous entries instead of random law-table rows (the
    // law-table gather was 24 % of C4's shared-memory wavefronts, 70 % of them bank-conflict
    // excess)
    // (only while the 16-byte entries keep the tables small: a dense dep(j) at M ~ 500 would
    // otherwise not fit in shared memory)
    L.fatdep = !L.dep16 && N <= 4095 && 16 * nnz <= 48 * 1024;
    if (const char* e = std::getenv("SMC_FATDEP")) L.fatdep = std::atoi(e) != 0 && !L.dep16 && N <= 4095;
    L.off_dep_off = o; o = align16(o + 4 * ((size_t)(L.depsp ? N : M) + 1));
    L.off_dep = o; o = align16(o + (L.fatdep ? 16 : (L.dep16 ? 2 : 4)) * (L.depsp ? nnz_sp : nnz));
    L.bytes = o;
    L.blob.assign(L.bytes, 0);
    auto* x0 = (int32_t*)(L.blob.data() + L.off_x0);
    for (int s = 0; s < N; ++s) x0[s] = m.x0[(size_t)s];
    x0[N] = 1;
    auto* chg = (uint16_t*)(L.blob.data() + L.off_chg);
    std::vector<uint32_t> fat_meta((size_t)M);          // s0 | s1 << 12 | kind << 24 | st0==2 << 27 | st1==2 << 28 | hill << 31
    std::vector<double> fat_c((size_t)M);
    for (int j = 0; j < M; ++j) {
        const Reaction& r = m.R[(size_t)j];
        uint32_t kind, s0, s1;
        double c;
        law_kind(m, j, kind, s0, s1, c);
        uint32_t w0 = s0 | (kind << 16) | ((uint32_t)(r.s[0] >= 0 ? r.st[0] : 1) << 20);
        uint32_t w1 = s1 | ((uint32_t)(r.s[1] >= 0 ? r.st[1] : 1) << 16);

        L.any_explicit |= kind == 5;
        L.any_general |= kind == 4;                     // incl. a homodimer with a subnormal rate
        if (r.hill) w0 |= 0x80000000u;
        fat_meta[(size_t)j] = s0 | (s1 << 12) | (kind << 24) | ((uint32_t)(r.s[0] >= 0 && r.st[0] == 2) << 27) |
                              ((uint32_t)(r.s[1] >= 0 && r.st[1] == 2) << 28) | ((uint32_t)r.hill << 31);
        fat_c[(size_t)j] = c;
        unsigned char* law = L.blob.data() + L.off_law + 16 * (size_t)j;   // {u0, u1, double c}
        std::memcpy(law, &w0, 4);
        std::memcpy(law + 4, &w1, 4);
        std::memcpy(law + 8, &c, 8);
        if (L.any_hill) {
            ((int32_t*)(L.blob.data() + L.off_hill_rep))[j] = r.hill ? r.rep : 0;
            ((double*)(L.blob.data() + L.off_hill_k))[j] = r.hill ? r.K : 1.0;
            ((int32_t*)(L.blob.data() + L.off_hill_n))[j] = r.hill ? r.n : 1;
        }
        if (r.change.size() > 4) fail(SMC_E_MODEL, "internal: more than 4 changed species");
        for (int q = 0; q < 4; ++q) {
            uint16_t e = 0xFFFF;
            if (q < (int)r.change.size()) e = (uint16_t)((r.change[(size_t)q].first << 4) | (r.change[(size_t)q].second + 8));
            chg[4 * j + q] = e;
        }
    }
    if (sweep) {                                   // variant 4: no dependency graph
        // sweep law table: {u0 = column byte offset of s0 | flags, u1 = offset of s1, c},
        // padded with zero-rate entries to G*S so that every group has S members.
        // flags: bit 0 homodimer (h = x (x - 1), c halved as above), bit 1 general law
        // (order 3-4, explicit, Hill: the kernel takes the law-table path)
        L.sw_s = sweep_group(m);
        // independent law reads per chunk: the whole group for S <= 8 (C4: S = C = 7), else
        // the largest divisor of S up to 8 ((64, 512): S = 18, C = 6 8.1e9 vs C = 3 7.9e9)
        L.sw_c = 1;
        if (L.sw_s <= 8) L.sw_c = L.sw_s;
        else
            for (int c = 8; c >= 2; --c)
                if (L.sw_s % c == 0) { L.sw_c = c; break; }
        if (const char* e = std::getenv("SMC_SW_C")) {
            const int c = std::atoi(e);
            if (c >= 1 && L.sw_s % c == 0) L.sw_c = c;
        }
        const int G = (M + L.sw_s - 1) / L.sw_s;
        L.off_swlaw = align16(L.bytes);
        const size_t nb = L.off_swlaw + 16 * (size_t)G * L.sw_s;
        sweep_shape(m, nb, L.sw_xd, L.sw_blk);
        const uint32_t col = (uint32_t)L.sw_blk * (L.sw_xd ? 8u : 4u);
        L.blob.resize(nb, 0);
        L.bytes = nb;
        for (int j = 0; j < G * L.sw_s; ++j) {
            uint32_t u0 = (uint32_t)N * col, u1 = (uint32_t)N * col;
            double c = 0.0;
            if (j < M) {
                uint32_t w0, w1;
                std::memcpy(&w0, L.blob.data() + L.off_law + 16 * (size_t)j, 4);
                std::memcpy(&w1, L.blob.data() + L.off_law + 16 * (size_t)j + 4, 4);
                std::memcpy(&c, L.blob.data() + L.off_law + 16 * (size_t)j + 8, 8);
                const uint32_t kind = (w0 >> 16) & 7u;
                u0 = (w0 & 0xFFFFu) * col;
                u1 = (w1 & 0xFFFFu) * col;
                if (kind == 2) u0 |= 1u;
                if (kind >= 4 || (w0 & 0x80000000u)) u0 |= 2u;
            }
            unsigned char* e = L.blob.data() + L.off_swlaw + 16 * (size_t)j;
            std::memcpy(e, &u0, 4);
            std::memcpy(e + 4, &u1, 4);
            std::memcpy(e + 8, &c, 8);
        }
        return L;
    }
    if ((size_t)L.gs * L.tw > 65536) fail(SMC_E_MODEL, "tile variant: too many reactions for 16-bit slots");
    auto* doff = (uint32_t*)(L.blob.data() + L.off_dep_off);
    auto* dep = (uint32_t*)(L.blob.data() + L.off_dep);
    auto* dep16 = (uint16_t*)(L.blob.data() + L.off_dep);

    size_t pos = 0;
    if (L.depsp) {
        for (int sp = 0; sp < N; ++sp) {
            doff[sp] = (uint32_t)pos;
            for (int k : readers[(size_t)sp]) dep16[pos++] = (uint16_t)k;
        }
        doff[N] = (uint32_t)pos;
        return L;
    }
    for (int j = 0; j < M; ++j) {
        doff[j] = (uint32_t)pos;
        for (int k : m.dep[(size_t)j]) {
            const int l = k / L.gs, mm = k % L.gs;       // owner lane, member (ssa_tile.cuh smc_slot)
            const uint32_t slot = L.row ? (uint32_t)(l * L.gsp + mm) : (uint32_t)(mm * L.tw + (l ^ ((mm / L.ch) % L.tw)));
            if (L.fatdep) {
                unsigned char* fe = L.blob.data() + L.off_dep + 16 * pos++;
                const uint32_t ks = (uint32_t)k | (slot << 16);
                std::memcpy(fe, &ks, 4);
                std::memcpy(fe + 4, &fat_meta[(size_t)k], 4);
                std::memcpy(fe + 8, &fat_c[(size_t)k], 8);
            } else if (L.dep16) dep16[pos++] = (uint16_t)k;
            else dep[pos++] = (uint32_t)k | (slot << 16);
        }
    }
    doff[M] = (uint32_t)pos;
    return L;
}

size_t window_bytes_per_entry(const Property& p) { return win_bytes(p); }
size_t window_small_bytes(const Property& p) { return win_small(p); }

std::string generate_source(const Model& m, const Property& p, int variant, const TileLayout* tl) {
    std::ostringstream o;
    o << "// generated by libsmc codegen: model N=" << m.N << " M=" << m.M << ", variant " << variant << "\n";
    o << "#define SMC_N " << m.N << "\n#define SMC_M " << m.M << "\n";
    o << "#define SMC_TMAX " << dlit(p.t_max) << "\n";
    if (variant == 3) {
        // the trace must cover what the semantics can look at: t_max for unbounded formulas,
        // else the formula's reach (as the oracle's literal mode)
        const double H = p.t_max > 0.0 ? p.t_max : p.horizon;
        int minb = 2;                       // resident 128-thread CTAs the registers must allow
        if (const char* e = std::getenv("SMC_LIT_MINB")) minb = std::max(1, std::atoi(e));
        o << "#define SMC_BLOCK 128\n#define SMC_MINB " << minb << "\n#define SMC_PIPE2 0\n";
        o << "#define SMC_LIT_H " << dlit(H) << "\n#define SMC_LIT_NODES " << p.lnodes.size() << "\n";
    } else if (variant == 1) {
        // >= 4 resident CTAs of 128 threads: at most 128 registers per thread
        // resident 128-thread CTAs per SM (register cap 65536 / (128 minb)): the small models
        // (M <= 8: C1, C2) run latency-bound Wilson rounds below full occupancy and keep
        // registers for ILP (minb 4); larger ones are throughput-bound (minb 6: C3 +4 %)
        const int minb = thread_minb(m);
        const int blk = thread_block(m);    // the same resident threads in fewer, larger CTAs
        o << "#define SMC_BLOCK " << blk << "\n#define SMC_MINB " << std::max(1, minb * 128 / blk) << "\n";
        // two-stage draw pipeline: shorter per-event chain (-12 % at low occupancy, C2) for
        // register-light models; heavier models are throughput-bound and keep one stage
        int pipe2 = (m.M <= 8 && m.N <= 8) ? 1 : 0;
        if (const char* e = std::getenv("SMC_PIPE2")) pipe2 = std::atoi(e);
        o << "#define SMC_PIPE2 " << pipe2 << "\n";
        if (const char* e = std::getenv("SMC_UNROLL")) o << "#define SMC_UNROLL " << std::atoi(e) << "\n";
        if (const char* e = std::getenv("SMC_BURST")) o << "#define SMC_BURST " << std::max(1, std::atoi(e)) << "\n";
    } else if (variant == 4) {
        if (p.literal) {
            const double H = p.t_max > 0.0 ? p.t_max : p.horizon;
            o << "#define SMC_LIT_H " << dlit(H) << "\n";
        }
        // 128-thread CTAs; resident CTAs per SM bounded by the counts' shared memory
        // (tables + 128 columns of N+1 ints) and by registers (pass 1 keeps the counts and
        // the group prefixes in registers): 3 by default (<= 168 registers; C4: 3 -> 1.19e10,
        // 4 -> 1.14e10, 5 -> 8.8e9 events/s: the sweep's ILP needs the registers)
        const int blk = tl->sw_blk;
        const size_t per_cta = tl->bytes + (size_t)blk * (tl->sw_xd ? 8 : 4) * (size_t)(m.N + 1) + 1024 + 64;
        // CTAs per SM: bounded by shared memory and by the ~384 resident threads whose
        // ~168 registers (the sweep's ILP) fill the register file
        int minb = (int)std::max<size_t>(1, std::min<size_t>((size_t)std::max(1, 384 / blk), 233472 / per_cta));
        if (const char* e = std::getenv("SMC_MINB")) minb = std::atoi(e);
        o << "#define SMC_SWEEP 1\n#define SMC_BLOCK " << blk << "\n#define SMC_MINB " << std::max(1, minb) << "\n";
        o << "#define SMC_SW_XD " << (tl->sw_xd ? 1 : 0) << "\n#define SMC_OFF_SWLAW " << tl->off_swlaw
          << "\n#define SMC_SW_C " << tl->sw_c << "\n";
        if (const char* e = std::getenv("SMC_BURST")) o << "#define SMC_BURST " << std::max(1, std::atoi(e)) << "\n";
        if (const char* e = std::getenv("SMC_SW_DSCAN")) o << "#define SMC_SW_DSCAN " << std::atoi(e) << "\n";
        o << "#define SMC_SW_ANYGEN " << ((tl->any_hill || tl->any_general || tl->any_explicit) ? 1 : 0) << "\n";
        o << "#define SMC_OFF_X0 " << tl->off_x0 << "\n#define SMC_OFF_LAW " << tl->off_law
          << "\n#define SMC_OFF_HREP " << tl->off_hill_rep << "\n#define SMC_OFF_HK " << tl->off_hill_k
          << "\n#define SMC_OFF_HN " << tl->off_hill_n << "\n#define SMC_OFF_CHG " << tl->off_chg << "\n";
        o << "#define SMC_TAB_BYTES " << tl->bytes << "\n";
        o << "#define SMC_ANY_HILL " << (tl->any_hill ? 1 : 0) << "\n";
        o << "#define SMC_ANY_GENERAL " << (tl->any_general ? 1 : 0) << "\n";
        o << "#define SMC_ANY_EXPLICIT " << (tl->any_explicit ? 1 : 0) << "\n";
    } else if (variant == 5) {
        // upper bound of the CTA (register cap 65536 / blk: TW 32 64, 16 73, 8 102, <= 4 128)
        int blk = tl->tw >= 32 ? 1024 : (tl->tw == 16 ? 896 : (tl->tw == 8 ? 960 : 512));
        if (const char* e = std::getenv("SMC_DBLOCK")) blk = std::max(32, std::atoi(e) / 32 * 32);
        o << "#define SMC_TW " << tl->tw << "\n#define SMC_DG " << tl->dg << "\n#define SMC_DS " << tl->ds
          << "\n#define SMC_DBLOCK " << blk << "\n";
        if (const char* e = std::getenv("SMC_DCHECK")) o << "#define SMC_DCHECK " << std::atoi(e) << "\n";
        if (const char* e = std::getenv("SMC_DFAST")) o << "#define SMC_DFAST " << std::atoi(e) << "\n";
        if (std::getenv("SMC_DTRACE")) o << "#define SMC_DTRACE 1\n";
        if (std::getenv("SMC_DBOUNDS")) o << "#define SMC_DBOUNDS 1\n#define SMC_DTABEND " << tl->bytes << "\n";
        o << "#define SMC_DSCALE " << dlit(std::ldexp(1.0, tl->dl)) << "\n#define SMC_DINV " << dlit(std::ldexp(1.0, -tl->dl))
          << "\n#define SMC_DHI " << dlit(std::ldexp(1.0, 64 - tl->dl)) << "\n";
        o << "#define SMC_OFF_X0 " << tl->off_x0 << "\n#define SMC_OFF_LAW " << tl->off_law << "\n#define SMC_OFF_CQ "
          << tl->off_hill_k << "\n#define SMC_OFF_CHG " << tl->off_chg << "\n#define SMC_OFF_DOFF " << tl->off_dep_off
          << "\n#define SMC_OFF_DEP " << tl->off_dep << "\n#define SMC_OFF_RCNT " << tl->off_hill_rep
          << "\n#define SMC_DRMAX " << tl->drmax << "\n#define SMC_DDEP16 " << (tl->dep16 ? 1 : 0)
          << "\n#define SMC_DDESC64 " << (tl->fatdep ? 1 : 0) << "\n";
        o << "#define SMC_TAB_BYTES " << tl->smem_bytes << "\n#define SMC_TILE_BYTES " << tl->tile_bytes << "\n";
        o << "#define SMC_DGLOBAL " << (tl->smem_bytes < tl->bytes ? 1 : 0) << "\n";
    } else {
        if (p.literal) {
            const double H = p.t_max > 0.0 ? p.t_max : p.horizon;
            o << "#define SMC_LIT_H " << dlit(H) << "\n#define SMC_LIT_NODES " << p.lnodes.size() << "\n";
        }
        o << "#define SMC_ROWLAYOUT " << (tl->row ? 1 : 0) << "\n#define SMC_GSP " << tl->gsp << "\n";
        o << "#define SMC_TW " << tl->tw << "\n#define SMC_GS " << tl->gs << "\n#define SMC_CH " << tl->ch
          << "\n#define SMC_NPAD " << tl->n_pad << "\n";
        o << "#define SMC_OFF_X0 " << tl->off_x0 << "\n#define SMC_OFF_LAW " << tl->off_law
          << "\n#define SMC_OFF_HREP " << tl->off_hill_rep << "\n#define SMC_OFF_HK " << tl->off_hill_k
          << "\n#define SMC_OFF_HN " << tl->off_hill_n << "\n#define SMC_OFF_CHG " << tl->off_chg
          << "\n#define SMC_OFF_DOFF " << tl->off_dep_off << "\n#define SMC_OFF_DEP " << tl->off_dep << "\n";
        o << "#define SMC_TAB_BYTES " << tl->bytes << "\n";
        o << "#define SMC_TILE_BYTES " << tl->tile_bytes << "\n";
        o << "#define SMC_ANY_HILL " << (tl->any_hill ? 1 : 0) << "\n";
        o << "#define SMC_ANY_GENERAL " << (tl->any_general ? 1 : 0) << "\n";
        o << "#define SMC_DEP16 " << (tl->dep16 ? 1 : 0) << "\n";
        o << "#define SMC_DEPSP " << (tl->depsp ? 1 : 0) << "\n";
        o << "#define SMC_FATDEP " << (tl->fatdep ? 1 : 0) << "\n";
        o << "#define SMC_ANY_EXPLICIT " << (tl->any_explicit ? 1 : 0) << "\n";
        if (const char* e = std::getenv("SMC_FLAT")) o << "#define SMC_FLAT " << std::atoi(e) << "\n";
    }
    o << embedded_source("ssa_common.cuh") << "\n";
    if (variant == 1) {
        // binary64 count registers for the latency-bound small models (C2: 0.389 -> 0.381
        // us per event on the chain); larger ones keep int32 (C3: more spills, -6 %)
        bool xd = m.M <= 8 && m.N <= 8;
        if (const char* e = std::getenv("SMC_V1_XD")) xd = std::atoi(e) != 0;
        o << (xd ? model_code_thread_xd(m) : model_code_thread(m)) << "\n";
    }
    if (variant == 3) o << model_code_thread(m) << "\n";
    if (variant == 4) o << model_code_sweep(m, tl->sw_xd) << "\n";
    if (variant == 2 && tl->any_explicit) {          // explicit laws of the tile variant
        o << "__device__ __noinline__ double smc_explicit(int k, const int* xs) {\n    switch (k) {\n";
        for (int k = 0; k < m.M; ++k)
            if (!m.R[(size_t)k].rate.empty())
                o << "    case " << k << ":\n" << explicit_body(m.R[(size_t)k], "xs", "        ");
        o << "    }\n    return 0.0;\n}\n";
    }
    if (variant == 3) {
        o << window_code(p) << "\n" << embedded_source("ssa_window.cuh") << "\n" << embedded_source("ssa_literal.cuh")
          << "\n";
        return o.str();
    }
    if (p.literal) o << window_code(p) << "\n" << embedded_source("ssa_window.cuh") << "\n";   // variant 2 only
    else {
        bool xd = false;                // binary64 count arrays: variant 1 small models, sweep
        if (variant == 4) xd = tl->sw_xd;
        if (variant == 1) {
            xd = m.M <= 8 && m.N <= 8;
            if (const char* e = std::getenv("SMC_V1_XD")) xd = std::atoi(e) != 0;
        }
        if (const char* e = std::getenv("SMC_MON_XD")) xd = xd && std::atoi(e) != 0;
        o << MonGen(p, xd).emit() << "\n";
    }
    o << embedded_source(variant == 1 ? "ssa_thread.cuh"
                                      : (variant == 4 ? "ssa_sweep.cuh" : (variant == 5 ? "ssa_delta.cuh" : "ssa_tile.cuh")))
      << "\n";
    return o.str();
}

}  // namespace smc
