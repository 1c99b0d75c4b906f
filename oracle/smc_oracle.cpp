// =============================================================================
// smc_oracle.cpp -- plain, slow, single-threaded CPU ORACLE for the statistical
// model checker of arXiv:0912.2551 (Ballarini, Forlin, Mazza, Prandi,
// "Efficient parallel statistical model checking of biochemical networks").
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load this library.
// It shares NO code, header, table or constant generator with the CUDA path
// under paper_0912_2551_b200/ and it never imports from it.
//
// Every function cites the passage of /root/reference/PAPER.md ("P:<line>")
// it transcribes.  Where the paper is silent the reading of DESIGN.md §3
// ("Readings of the paper") is used and cited as "R<n>".
//
// Build (see oracle/oracle.py):  g++ -O2 -std=c++17 -ffp-contract=off -fPIC -shared
// -ffp-contract=off: no FMA contraction, every double op is one IEEE-754
// round-to-nearest operation (reading R14).
//
// What is pinned, and by what (tests/test_oracle_*.py):
//   philox      -- cuRAND's curand_Philox4x32_10 compiled for the host and the
//                  Random123 known-answer vectors (library routine, bit-exact).
//   SSA         -- closed forms (pure decay, pure death, pure birth,
//                  immigration-death), brute-force uniformisation of tiny
//                  CTMCs (scipy expm), exact event counts (early termination).
//   literal |=  -- hand traces with known verdicts (SPEC examples), duality
//                  G == !F!, monotonicity in the bound; streaming monitor ==
//                  literal |= on >= 10^4 random traces per template.
//   streaming   -- pinned to the literal semantics (above).
// Nothing in this file is "parity unpinned".
// =============================================================================
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace orc {

static const double INF = std::numeric_limits<double>::infinity();

// -----------------------------------------------------------------------------
// 1. Random numbers.  The paper scatters one seed per replica "to tackle the
//    problem of avoiding correlation".  Reading R10: a counter-based
//    Philox4x32-10 stream, key = seed, counter = (k_lo, k_hi, i_lo, i_hi) with
//    k = number of events applied so far and i = trajectory index.
// -----------------------------------------------------------------------------
void philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {            // key schedule: Weyl increments between rounds
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c[0];
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c[2];
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c[1] ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c[3] ^ k1;
        uint32_t n3 = lo0;
        c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

// The two uniforms of one SSA step ("standard Monte Carlo methods"):
//   u1 = ((((r0<<32)|r1) >> 11) + 1) * 2^-53  in (0,1]   -> tau   (Eq. 2a)
//   u2 = ( ((r2<<32)|r3) >> 11)      * 2^-53  in [0,1)   -> j     (Eq. 2b)
void step_uniforms(uint64_t seed, uint64_t traj, uint64_t step, double* u1, double* u2) {
    uint32_t ctr[4] = {(uint32_t)step, (uint32_t)(step >> 32), (uint32_t)traj, (uint32_t)(traj >> 32)};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t r[4];
    philox4x32_10(ctr, key, r);
    uint64_t w1 = ((uint64_t)r[0] << 32) | r[1];
    uint64_t w2 = ((uint64_t)r[2] << 32) | r[3];
    const double two_m53 = 1.0 / 9007199254740992.0;  // 2^-53, exact
    *u1 = (double)((w1 >> 11) + 1) * two_m53;
    *u2 = (double)(w2 >> 11) * two_m53;
}

// -----------------------------------------------------------------------------
// 2. The model: species counts x and reaction channels
//    R_j with propensity a_j(x) and change vector v_j.
// -----------------------------------------------------------------------------
// Explicit rate expression (Table 2): a tree over
// species counts (promoted to binary64) and decimal constants with + - * / and
// unary minus, evaluated recursively in IEEE binary64 (left-associative).
struct RateNode {
    char op;            // 'c' constant, 'x' species, '+', '-', '*', '/', 'n' (negate)
    double value = 0.0; // 'c'
    int species = -1;   // 'x'
    int a = -1, b = -1; // children
};

struct Reaction {
    std::vector<std::pair<int, int>> reactants;  // (species, stoichiometry), merged
    std::vector<std::pair<int, int>> change;     // (species, delta), delta != 0
    double c = 0.0;                              // rate constant c_j
    bool hill = false;                           // reading R9
    int repressor = -1;
    double K = 0.0;
    int n = 0;
    std::vector<RateNode> rate;                  // explicit rate (root = back()), empty = mass action
};

double rate_eval(const std::vector<RateNode>& t, int i, const int64_t* x) {
    const RateNode& n = t[(size_t)i];
    switch (n.op) {
        case 'c': return n.value;
        case 'x': return (double)x[n.species];
        case 'n': return -rate_eval(t, n.a, x);
        case '+': return rate_eval(t, n.a, x) + rate_eval(t, n.b, x);
        case '-': return rate_eval(t, n.a, x) - rate_eval(t, n.b, x);
        case '*': return rate_eval(t, n.a, x) * rate_eval(t, n.b, x);
        default: return rate_eval(t, n.a, x) / rate_eval(t, n.b, x);
    }
}

// Recursive-descent parser: expr := term (('+'|'-') term)*, term := unary (('*'|'/') unary)*,
// unary := '-' unary | primary, primary := number | name | '(' expr ')'.
struct RateParser {
    const std::string& s;
    const std::vector<std::string>& names;
    std::vector<RateNode>& out;
    size_t p = 0;
    [[noreturn]] void fail(const std::string& m) {
        throw std::runtime_error("rate expression: " + m + " at " + std::to_string(p));
    }
    void ws() { while (p < s.size() && std::isspace((unsigned char)s[p])) ++p; }
    int push(RateNode n) { out.push_back(n); return (int)out.size() - 1; }
    int expr() {
        int l = term();
        for (;;) {
            ws();
            if (p < s.size() && (s[p] == '+' || s[p] == '-')) {
                char o = s[p++];
                int r = term();
                RateNode n; n.op = o; n.a = l; n.b = r; l = push(n);
            } else return l;
        }
    }
    int term() {
        int l = unary();
        for (;;) {
            ws();
            if (p < s.size() && (s[p] == '*' || s[p] == '/')) {
                char o = s[p++];
                int r = unary();
                RateNode n; n.op = o; n.a = l; n.b = r; l = push(n);
            } else return l;
        }
    }
    int unary() {
        ws();
        if (p < s.size() && s[p] == '-') { ++p; RateNode n; n.op = 'n'; n.a = unary(); return push(n); }
        return primary();
    }
    int primary() {
        ws();
        if (p >= s.size()) fail("unexpected end");
        if (s[p] == '(') {
            ++p;
            int e = expr();
            ws();
            if (p >= s.size() || s[p] != ')') fail("')' expected");
            ++p;
            return e;
        }
        if (std::isdigit((unsigned char)s[p]) || s[p] == '.') {
            char* end = nullptr;
            double v = std::strtod(s.c_str() + p, &end);
            if (end == s.c_str() + p) fail("bad number");
            p = (size_t)(end - s.c_str());
            RateNode n; n.op = 'c'; n.value = v; return push(n);
        }
        if (std::isalpha((unsigned char)s[p]) || s[p] == '_') {
            size_t q = p;
            while (p < s.size() && (std::isalnum((unsigned char)s[p]) || s[p] == '_')) ++p;
            std::string id = s.substr(q, p - q);
            for (size_t i = 0; i < names.size(); ++i)
                if (names[i] == id) { RateNode n; n.op = 'x'; n.species = (int)i; return push(n); }
            fail("unknown species '" + id + "'");
        }
        fail("unexpected character");
    }
};

struct Model {
    int N = 0;
    std::vector<int64_t> x0;
    std::vector<Reaction> R;
};

// Mass action a_j = c_j * h_j(x), h_j = number of distinct reactant
// combinations: x for stoichiometry 1 ("a_1 = c_1 x_1 x_2") and
// x(x-1)/2 for a homodimer (reading R8); zero when a reactant is missing.
// Hill repression (reading R9): a_j = c_j h_j / (1 + (x_r/K)^n).
// Explicit rate: a_j = v(x), the propensity guard still applies (zero when a
// reactant count is below its stoichiometry); a negative or NaN v is a bad
// propensity (returned as NaN, the replica ends in error).
double propensity(const Reaction& r, const int64_t* x) {
    int64_t h = 1;
    for (const auto& rs : r.reactants) {
        int64_t xs = x[rs.first];
        if (xs < rs.second) return 0.0;
        if (rs.second == 1) h = h * xs;
        else h = h * (xs * (xs - 1) / 2);
    }
    if (!r.rate.empty()) {
        double v = rate_eval(r.rate, (int)r.rate.size() - 1, x);
        return (v >= 0.0) ? v : std::nan("");
    }
    double a = r.c * (double)h;
    if (r.hill) {
        double q = (double)x[r.repressor] / r.K;
        double qn = q;
        for (int i = 1; i < r.n; ++i) qn = qn * q;   // left-to-right product
        a = a / (1.0 + qn);
    }
    return a;
}

// -----------------------------------------------------------------------------
// 3. BLTLc formulas and their evaluation function Eval.
//    Atoms compare integer expressions over species counts, evaluated exactly
//    in int64.
// -----------------------------------------------------------------------------
//    The general val of P:209 (val ~ val with ~ in {+,-,*,/}, func, Int, Real):
//    an atom built only from Int constants, species, +, -, * is evaluated
//    exactly in int64; an atom with '/', a Real constant or a function
//    (sqrt, abs, min, max, pow(val, k) with an Int k >= 0) is evaluated in IEEE
//    binary64, recursively in tree order, counts promoted to double.
enum ExprKind { E_CONST, E_VAR, E_ADD, E_SUB, E_MUL, E_NEG, E_DIV, E_REAL, E_SQRT, E_ABS, E_MIN, E_MAX, E_POW };
struct Expr {
    ExprKind kind;
    int64_t value = 0;   // E_CONST; E_POW exponent
    double real = 0.0;   // E_REAL
    int var = -1;
    int lhs = -1, rhs = -1;
};

enum CmpOp { C_LT, C_LE, C_GE, C_GT, C_EQ, C_NE };
struct Atom {
    int lhs, rhs;
    CmpOp op;
    bool real = false;   // binary64 evaluation (see above)
};

struct Interval {  // I subset of R>=0; [0,inf) when omitted
    double lo = 0.0, hi = INF;
    bool lo_open = false, hi_open = false;
    bool contains(double e) const {
        bool a = lo_open ? (e > lo) : (e >= lo);
        bool b = hi_open ? (e < hi) : (e <= hi);
        return a && b;
    }
    bool beyond(double e) const { return hi_open ? (e >= hi) : (e > hi); }
};

enum NodeKind { N_ATOM, N_TRUE, N_FALSE, N_NOT, N_AND, N_OR, N_X, N_U, N_F, N_G };
struct Node {
    NodeKind kind;
    Interval I;
    int a = -1, b = -1;   // children (U: a = phi', b = phi'')
    int atom = -1;
};

struct Formula {
    std::vector<Expr> exprs;
    std::vector<Atom> atoms;
    std::vector<Node> nodes;
    int root = -1;
    double t_max = 0.0;   // reading R5: cap for unbounded formulas (0 = bounded only)
    std::vector<int> species_used;
};

int64_t eval_expr(const Formula& f, int e, const int64_t* x) {
    const Expr& ex = f.exprs[e];
    switch (ex.kind) {
        case E_CONST: return ex.value;
        case E_VAR: return x[ex.var];
        case E_ADD: return eval_expr(f, ex.lhs, x) + eval_expr(f, ex.rhs, x);
        case E_SUB: return eval_expr(f, ex.lhs, x) - eval_expr(f, ex.rhs, x);
        case E_MUL: return eval_expr(f, ex.lhs, x) * eval_expr(f, ex.rhs, x);
        case E_NEG: return -eval_expr(f, ex.lhs, x);
    }
    return 0;
}

double eval_real(const Formula& f, int e, const int64_t* x) {
    const Expr& ex = f.exprs[e];
    switch (ex.kind) {
        case E_CONST: return (double)ex.value;
        case E_REAL: return ex.real;
        case E_VAR: return (double)x[ex.var];
        case E_ADD: return eval_real(f, ex.lhs, x) + eval_real(f, ex.rhs, x);
        case E_SUB: return eval_real(f, ex.lhs, x) - eval_real(f, ex.rhs, x);
        case E_MUL: return eval_real(f, ex.lhs, x) * eval_real(f, ex.rhs, x);
        case E_DIV: return eval_real(f, ex.lhs, x) / eval_real(f, ex.rhs, x);
        case E_NEG: return -eval_real(f, ex.lhs, x);
        case E_SQRT: return std::sqrt(eval_real(f, ex.lhs, x));
        case E_ABS: return std::fabs(eval_real(f, ex.lhs, x));
        case E_MIN: { double a = eval_real(f, ex.lhs, x), b = eval_real(f, ex.rhs, x); return a < b ? a : b; }
        case E_MAX: { double a = eval_real(f, ex.lhs, x), b = eval_real(f, ex.rhs, x); return a > b ? a : b; }
        case E_POW: {
            double b = eval_real(f, ex.lhs, x), r = 1.0;
            for (int64_t i = 0; i < ex.value; ++i) r = (i == 0) ? b : r * b;   // left-to-right product
            return r;
        }
    }
    return 0.0;
}

template <class T>
bool compare(T l, T r, CmpOp op) {
    switch (op) {
        case C_LT: return l < r;
        case C_LE: return l <= r;
        case C_GE: return l >= r;
        case C_GT: return l > r;
        case C_EQ: return l == r;
        case C_NE: return l != r;
    }
    return false;
}

// sigma |= (val' <| val'') iff Eval(sigma[0],val') <| Eval(sigma[0],val'')
bool eval_atom(const Formula& f, int a, const int64_t* x) {
    const Atom& at = f.atoms[a];
    if (at.real) return compare(eval_real(f, at.lhs, x), eval_real(f, at.rhs, x), at.op);
    int64_t l = eval_expr(f, at.lhs, x), r = eval_expr(f, at.rhs, x);
    switch (at.op) {
        case C_LT: return l < r;
        case C_LE: return l <= r;
        case C_GE: return l >= r;
        case C_GT: return l > r;
        case C_EQ: return l == r;
        case C_NE: return l != r;
    }
    return false;
}

// ---- parser: concrete syntax of reading R15 (after S:207) -------------------
struct Parser {
    const std::string& s;
    size_t p = 0;
    const std::vector<std::string>& names;
    Formula& f;
    Parser(const std::string& s_, const std::vector<std::string>& n_, Formula& f_) : s(s_), names(n_), f(f_) {}

    [[noreturn]] void fail(const std::string& msg) {
        throw std::runtime_error("parse error at " + std::to_string(p) + ": " + msg);
    }
    void ws() { while (p < s.size() && std::isspace((unsigned char)s[p])) ++p; }
    bool peek(const char* t) { ws(); return s.compare(p, std::strlen(t), t) == 0; }
    bool eat(const char* t) { if (peek(t)) { p += std::strlen(t); return true; } return false; }
    bool is_ident_char(char c) { return std::isalnum((unsigned char)c) || c == '_'; }
    // keyword = whole identifier token
    bool peek_kw(const char* kw) {
        ws();
        size_t n = std::strlen(kw);
        if (s.compare(p, n, kw) != 0) return false;
        return p + n >= s.size() || !is_ident_char(s[p + n]);
    }
    bool eat_kw(const char* kw) { if (peek_kw(kw)) { p += std::strlen(kw); return true; } return false; }

    int add_node(Node n) { f.nodes.push_back(n); return (int)f.nodes.size() - 1; }
    int add_expr(Expr e) { f.exprs.push_back(e); return (int)f.exprs.size() - 1; }

    double number() {
        ws();
        if (eat_kw("inf")) return INF;
        size_t q = p;
        while (q < s.size() && (std::isdigit((unsigned char)s[q]) || s[q] == '.' || s[q] == 'e' || s[q] == 'E' ||
                                ((s[q] == '-' || s[q] == '+') && q > p && (s[q - 1] == 'e' || s[q - 1] == 'E'))))
            ++q;
        if (q == p) fail("number expected");
        double v = std::strtod(s.substr(p, q - p).c_str(), nullptr);
        p = q;
        return v;
    }
    // optional interval suffix: [a,b] (a,b] [a,b) (a,b) [a,inf)
    Interval interval() {
        Interval I;
        ws();
        if (p < s.size() && (s[p] == '[' || (s[p] == '(' && looks_like_interval()))) {
            I.lo_open = (s[p] == '(');
            ++p;
            I.lo = number();
            if (!eat(",")) fail("',' expected in interval");
            I.hi = number();
            ws();
            if (p >= s.size() || (s[p] != ']' && s[p] != ')')) fail("']' or ')' expected");
            I.hi_open = (s[p] == ')');
            ++p;
            if (std::isinf(I.hi)) I.hi_open = false;
            if (!(I.lo >= 0.0) || !(I.hi >= I.lo)) fail("bad interval");
        }
        return I;
    }
    // '(' number ',' ... : an interval, not a parenthesised subformula
    bool looks_like_interval() {
        size_t q = p + 1;
        while (q < s.size() && std::isspace((unsigned char)s[q])) ++q;
        size_t r = q;
        while (r < s.size() && (std::isdigit((unsigned char)s[r]) || s[r] == '.' || s[r] == 'e')) ++r;
        if (r == q) return false;
        while (r < s.size() && std::isspace((unsigned char)s[r])) ++r;
        return r < s.size() && s[r] == ',';
    }

    // arithmetic: expr := term (('+'|'-') term)* ; term := factor ('*' factor)* ;
    // factor := int | species | '-' factor | '(' expr ')'
    int expr() {
        int l = term();
        for (;;) {
            if (eat("+")) { Expr e{E_ADD}; e.lhs = l; e.rhs = term(); l = add_expr(e); }
            else if (peek("-") ) { ++p; Expr e{E_SUB}; e.lhs = l; e.rhs = term(); l = add_expr(e); }
            else return l;
        }
    }
    int term() {
        int l = factor();
        for (;;) {
            if (eat("*")) { Expr e{E_MUL}; e.lhs = l; e.rhs = factor(); l = add_expr(e); }
            else if (eat("/")) { Expr e{E_DIV}; e.lhs = l; e.rhs = factor(); l = add_expr(e); }
            else return l;
        }
    }
    int factor() {
        ws();
        if (eat("-")) { Expr e{E_NEG}; e.lhs = factor(); return add_expr(e); }
        if (eat("(")) { int e = expr(); if (!eat(")")) fail("')' expected"); return e; }
        if (p < s.size() && (std::isdigit((unsigned char)s[p]) || s[p] == '.')) {
            size_t q = p;
            while (q < s.size() && std::isdigit((unsigned char)s[q])) ++q;
            if (q < s.size() && (s[q] == '.' || s[q] == 'e' || s[q] == 'E')) {   // Real constant
                char* end = nullptr;
                Expr e{E_REAL};
                e.real = std::strtod(s.c_str() + p, &end);
                if (end == s.c_str() + p) fail("number expected");
                p = (size_t)(end - s.c_str());
                return add_expr(e);
            }
            Expr e{E_CONST};
            e.value = std::stoll(s.substr(p, q - p));
            p = q;
            return add_expr(e);
        }
        if (p < s.size() && (std::isalpha((unsigned char)s[p]) || s[p] == '_')) {
            size_t q = p;
            while (q < s.size() && is_ident_char(s[q])) ++q;
            std::string id = s.substr(p, q - p);
            size_t r = q;
            while (r < s.size() && std::isspace((unsigned char)s[r])) ++r;
            if (r < s.size() && s[r] == '(') {                                 // func(...)
                ExprKind k;
                if (id == "sqrt") k = E_SQRT;
                else if (id == "abs") k = E_ABS;
                else if (id == "min") k = E_MIN;
                else if (id == "max") k = E_MAX;
                else if (id == "pow") k = E_POW;
                else fail("unknown function '" + id + "'");
                p = r + 1;
                Expr e{k};
                e.lhs = expr();
                if (k == E_MIN || k == E_MAX) {
                    if (!eat(",")) fail("',' expected");
                    e.rhs = expr();
                } else if (k == E_POW) {
                    if (!eat(",")) fail("',' expected");
                    ws();
                    size_t t = p;
                    while (t < s.size() && std::isdigit((unsigned char)s[t])) ++t;
                    if (t == p) fail("integer exponent expected");
                    e.value = std::stoll(s.substr(p, t - p));
                    p = t;
                }
                if (!eat(")")) fail("')' expected");
                return add_expr(e);
            }
            for (size_t i = 0; i < names.size(); ++i)
                if (names[i] == id) {
                    p = q;
                    Expr e{E_VAR};
                    e.var = (int)i;
                    return add_expr(e);
                }
            fail("unknown species '" + id + "'");
        }
        fail("expression expected");
    }
    // an atom needs binary64 when it contains '/', a Real constant or a function
    bool has_real(int e) {
        const Expr& ex = f.exprs[(size_t)e];
        if (ex.kind == E_DIV || ex.kind == E_REAL || ex.kind == E_SQRT || ex.kind == E_ABS || ex.kind == E_MIN ||
            ex.kind == E_MAX || ex.kind == E_POW)
            return true;
        return (ex.lhs >= 0 && has_real(ex.lhs)) || (ex.rhs >= 0 && has_real(ex.rhs));
    }
    bool cmp_op(CmpOp* op) {
        ws();
        if (eat("<=")) { *op = C_LE; return true; }
        if (eat(">=")) { *op = C_GE; return true; }
        if (eat("==")) { *op = C_EQ; return true; }
        if (eat("!=")) { *op = C_NE; return true; }
        if (eat("<")) { *op = C_LT; return true; }
        if (eat(">")) { *op = C_GT; return true; }
        if (eat("=")) { *op = C_EQ; return true; }
        return false;
    }
    // precedence: temporal unary > ! > & > U (right assoc.) > |
    int formula() { return disj(); }
    int disj() {
        int l = until();
        while (eat("|")) { Node n{N_OR}; n.a = l; n.b = until(); l = add_node(n); }
        return l;
    }
    int until() {
        int l = conj();
        if (peek_kw("U")) {
            p += 1;
            Node n{N_U};
            n.I = interval();
            n.a = l;
            n.b = until();
            return add_node(n);
        }
        return l;
    }
    int conj() {
        int l = unary();
        while (eat("&")) { Node n{N_AND}; n.a = l; n.b = unary(); l = add_node(n); }
        return l;
    }
    int unary() {
        ws();
        if (eat("!")) { Node n{N_NOT}; n.a = unary(); return add_node(n); }
        if (peek_kw("F") || peek_kw("G") || peek_kw("X")) {
            char c = s[p];
            ++p;
            Node n{c == 'F' ? N_F : (c == 'G' ? N_G : N_X)};
            n.I = interval();
            n.a = unary();
            return add_node(n);
        }
        return primary();
    }
    int primary() {
        ws();
        if (eat_kw("true")) return add_node(Node{N_TRUE});
        if (eat_kw("false")) return add_node(Node{N_FALSE});
        // try an atom first (expr cmp expr); on failure rewind to '(' formula ')'
        size_t save = p;
        size_t ne = f.exprs.size();
        try {
            int l = expr();
            CmpOp op;
            if (!cmp_op(&op)) throw std::runtime_error("no comparison");
            int r = expr();
            f.atoms.push_back(Atom{l, r, op, has_real(l) || has_real(r)});
            Node n{N_ATOM};
            n.atom = (int)f.atoms.size() - 1;
            return add_node(n);
        } catch (const std::runtime_error&) {
            p = save;
            f.exprs.resize(ne);
        }
        if (eat("(")) {
            int x = formula();
            if (!eat(")")) fail("')' expected");
            return x;
        }
        fail("formula expected");
    }
};

void collect_species(const Formula& f, int e, std::vector<char>& used) {
    const Expr& ex = f.exprs[e];
    if (ex.kind == E_VAR) used[ex.var] = 1;
    if (ex.lhs >= 0) collect_species(f, ex.lhs, used);
    if (ex.rhs >= 0) collect_species(f, ex.rhs, used);
}

// Time reach of a formula: how far past sigma[0] the semantics
// can look.  Unbounded operators reach t_max (reading R5).
double reach(const Formula& f, int n) {
    const Node& nd = f.nodes[n];
    switch (nd.kind) {
        case N_ATOM: case N_TRUE: case N_FALSE: return 0.0;
        case N_NOT: return reach(f, nd.a);
        case N_AND: case N_OR: return std::max(reach(f, nd.a), reach(f, nd.b));
        case N_X: case N_F: case N_G: return nd.I.hi + reach(f, nd.a);
        case N_U: return nd.I.hi + std::max(reach(f, nd.a), reach(f, nd.b));
    }
    return 0.0;
}

// -----------------------------------------------------------------------------
// 4. Literal semantics |= on a finite trace, three-valued
//    (reading R4: "unknown" only when the trace ends before the verdict is
//    fixed; the root maps unknown -> false).
//
//    Trace: entries (s_k, t_k), k = 0..n, with t_k the ENTRY time (reading R2),
//    sojourns delta(sigma,k) = tau[k] (the drawn waiting times);
//    either the chain is absorbed in s_n (delta(sigma,n) = inf, reading R7) or
//    the next entry happens at t_end = t_n + tau[n] in an unknown state.
// -----------------------------------------------------------------------------
enum Tri : int8_t { T_FALSE = 0, T_TRUE = 1, T_UNKNOWN = 2 };
static Tri t_not(Tri a) { return a == T_UNKNOWN ? T_UNKNOWN : (a == T_TRUE ? T_FALSE : T_TRUE); }
static Tri t_and(Tri a, Tri b) {
    if (a == T_FALSE || b == T_FALSE) return T_FALSE;
    if (a == T_TRUE && b == T_TRUE) return T_TRUE;
    return T_UNKNOWN;
}
static Tri t_or(Tri a, Tri b) { return t_not(t_and(t_not(a), t_not(b))); }

struct Trace {
    int N = 0;                      // species stored per entry
    std::vector<double> t;          // entry times t_0..t_n
    std::vector<double> tau;        // sojourns; tau.size() == n+1 unless absorbed
    std::vector<int64_t> x;         // (n+1) x N states
    bool absorbed = false;
    int64_t n() const { return (int64_t)t.size() - 1; }
    const int64_t* state(int64_t k) const { return &x[(size_t)k * N]; }
};

struct LiteralChecker {
    const Formula& f;
    const Trace& tr;
    std::vector<std::vector<int8_t>> memo;
    LiteralChecker(const Formula& f_, const Trace& tr_) : f(f_), tr(tr_) {
        memo.assign(f.nodes.size(), std::vector<int8_t>((size_t)tr.n() + 1, -1));
    }
    // Start from the DEFINITE values of a checker on a shorter prefix of the same trace: the
    // three-valued semantics is monotone in the observed prefix (observing more never revokes
    // a definite value), so those values hold on this prefix too; unknown ones are recomputed.
    void seed(const LiteralChecker& shorter) {
        for (size_t n = 0; n < memo.size(); ++n) {
            const auto& src = shorter.memo[n];
            for (size_t m = 0; m < src.size() && m < memo[n].size(); ++m)
                if (src[m] == T_FALSE || src[m] == T_TRUE) memo[n][m] = src[m];
        }
    }

    // phi' U^I phi'' at sigma^m:  exists i: sigma^i |= phi'',
    // sum_{j<i} delta(sigma^m, j) in I, and sigma^j |= phi' for all j < i.
    // F^I phi == tt U^I phi is passed with phi' = -1 (tt).
    Tri until(int m, const Interval& I, int phi1, int phi2) {
        Tri res = T_FALSE, pre = T_TRUE;
        double elapsed = 0.0;
        const int64_t n = tr.n();
        for (int64_t k = m; k <= n; ++k) {
            if (k > m) elapsed = elapsed + tr.tau[(size_t)k - 1];
            if (I.beyond(elapsed)) return res;          // later i only larger sums
            if (I.contains(elapsed)) res = t_or(res, t_and(pre, value(phi2, k)));
            if (res == T_TRUE) return T_TRUE;
            Tri p1 = (phi1 < 0) ? T_TRUE : value(phi1, k);
            pre = t_and(pre, p1);
            if (pre == T_FALSE) return res;
        }
        if (tr.absorbed) return res;                    // no further suffixes
        double tail = elapsed + tr.tau[(size_t)n];      // elapsed at the next (unknown) entry
        if (I.beyond(tail)) return res;
        return t_or(res, t_and(pre, T_UNKNOWN));
    }

    Tri value(int node, int64_t m) {
        int8_t& slot = memo[node][(size_t)m];
        if (slot >= 0) return (Tri)slot;
        const Node& nd = f.nodes[node];
        Tri r = T_UNKNOWN;
        switch (nd.kind) {
            case N_TRUE: r = T_TRUE; break;
            case N_FALSE: r = T_FALSE; break;
            case N_ATOM: r = eval_atom(f, nd.atom, tr.state(m)) ? T_TRUE : T_FALSE; break;
            case N_NOT: r = t_not(value(nd.a, m)); break;
            case N_OR: r = t_or(value(nd.a, m), value(nd.b, m)); break;
            case N_AND: r = t_and(value(nd.a, m), value(nd.b, m)); break;
            case N_X: {  // sigma |= X^I phi iff sigma^1 |= phi and delta(sigma,0) in I
                if (m < tr.n()) {
                    r = nd.I.contains(tr.tau[(size_t)m]) ? value(nd.a, m + 1) : T_FALSE;
                } else if (tr.absorbed) {
                    r = T_FALSE;                        // no successor exists
                } else {
                    r = nd.I.contains(tr.tau[(size_t)m]) ? T_UNKNOWN : T_FALSE;
                }
                break;
            }
            case N_U: r = until((int)m, nd.I, nd.a, nd.b); break;
            case N_F: r = until((int)m, nd.I, -1, nd.a); break;            // F == tt U
            case N_G: {                                                     // G == !F!
                // !F^I !phi : evaluate F^I over the negation of phi
                Tri res = T_FALSE, pre = T_TRUE;
                double elapsed = 0.0;
                const int64_t n = tr.n();
                bool done = false;
                for (int64_t k = m; k <= n && !done; ++k) {
                    if (k > m) elapsed = elapsed + tr.tau[(size_t)k - 1];
                    if (nd.I.beyond(elapsed)) { done = true; break; }
                    if (nd.I.contains(elapsed)) res = t_or(res, t_and(pre, t_not(value(nd.a, k))));
                    if (res == T_TRUE) { done = true; break; }
                }
                if (!done && !tr.absorbed) {
                    double tail = elapsed + tr.tau[(size_t)n];
                    if (!nd.I.beyond(tail)) res = t_or(res, T_UNKNOWN);
                }
                r = t_not(res);
                break;
            }
        }
        slot = (int8_t)r;
        return r;
    }
};

// -----------------------------------------------------------------------------
// 5. Streaming monitor: the on-the-fly principle of P:291-294 ("simulation
//    proceeds with the generation of the next state only if phi is neither
//    satisfied nor falsified") for the template fragment of reading R16.
//    Each leaf keeps O(1) state; the root combines leaves with Kleene logic.
//    It is pinned to the literal |= above by tests on random traces.
// -----------------------------------------------------------------------------
enum LeafKind { L_ATOM0, L_F, L_G, L_U, L_X, L_FG, L_GF, L_GU };
struct Leaf {
    LeafKind kind;
    Interval I, J;      // outer / inner intervals
    int beta1 = -1, beta2 = -1;   // boolean (non-temporal) subformulas; -1 = tt
    // state
    Tri status = T_UNKNOWN;
    bool pending = true;
    bool rs_set = false;
    double rs = 0.0;
    bool witness = false;
    double D = 0.0;
};

struct Monitor {
    const Formula& f;
    std::vector<Leaf> leaves;
    std::vector<int> leaf_of_node;   // node -> leaf index, -1 if boolean connective
    double t_prev = 0.0;
    int64_t k = 0;

    explicit Monitor(const Formula& f_) : f(f_) {
        leaf_of_node.assign(f.nodes.size(), -1);
        classify(f.root);
    }

    bool is_boolean(int n) const {
        const Node& nd = f.nodes[n];
        switch (nd.kind) {
            case N_ATOM: case N_TRUE: case N_FALSE: return true;
            case N_NOT: return is_boolean(nd.a);
            case N_AND: case N_OR: return is_boolean(nd.a) && is_boolean(nd.b);
            default: return false;
        }
    }
    static bool zero_closed(const Interval& I) { return I.lo == 0.0 && !I.lo_open && !I.hi_open; }

    int add_leaf(int node, Leaf L) {
        leaves.push_back(L);
        leaf_of_node[node] = (int)leaves.size() - 1;
        return leaf_of_node[node];
    }
    // Root := boolean combination of leaves; anything else is unsupported.
    void classify(int n) {
        const Node& nd = f.nodes[n];
        if (is_boolean(n)) {                  // atoms at sigma[0]
            Leaf L{L_ATOM0};
            L.beta1 = n;
            add_leaf(n, L);
            return;
        }
        switch (nd.kind) {
            case N_NOT: classify(nd.a); return;
            case N_AND: case N_OR: classify(nd.a); classify(nd.b); return;
            case N_F: case N_G: {
                const Node& in = f.nodes[nd.a];
                if (is_boolean(nd.a)) {
                    Leaf L{nd.kind == N_F ? L_F : L_G};
                    L.I = nd.I;
                    L.beta1 = nd.a;
                    add_leaf(n, L);
                    return;
                }
                // F[0,a] G[0,b] beta  and  G[0,a] F[0,b] beta
                if (zero_closed(nd.I) && ((nd.kind == N_F && in.kind == N_G) || (nd.kind == N_G && in.kind == N_F)) &&
                    zero_closed(in.I) && is_boolean(in.a) && std::isfinite(nd.I.hi) && std::isfinite(in.I.hi)) {
                    Leaf L{nd.kind == N_F ? L_FG : L_GF};
                    L.I = nd.I;
                    L.J = in.I;
                    L.beta1 = in.a;
                    add_leaf(n, L);
                    return;
                }
                break;
            }
            case N_U: {
                if (is_boolean(nd.a) && is_boolean(nd.b)) {
                    Leaf L{L_U};
                    L.I = nd.I;
                    L.beta1 = nd.a;
                    L.beta2 = nd.b;
                    add_leaf(n, L);
                    return;
                }
                const Node& l = f.nodes[nd.a];
                if (l.kind == N_G && is_boolean(l.a) && is_boolean(nd.b) && zero_closed(nd.I) && zero_closed(l.I) &&
                    std::isfinite(nd.I.hi) && std::isfinite(l.I.hi)) {
                    Leaf L{L_GU};
                    L.I = nd.I;
                    L.J = l.I;
                    L.beta1 = l.a;
                    L.beta2 = nd.b;
                    add_leaf(n, L);
                    return;
                }
                break;
            }
            case N_X:
                if (is_boolean(nd.a)) {
                    Leaf L{L_X};
                    L.I = nd.I;
                    L.beta1 = nd.a;
                    add_leaf(n, L);
                    return;
                }
                break;
            default: break;
        }
        throw std::runtime_error("formula outside the streaming fragment (literal mode only)");
    }

    bool beta(int node, const int64_t* x) {   // boolean subformula at the current state
        if (node < 0) return true;
        const Node& nd = f.nodes[node];
        switch (nd.kind) {
            case N_TRUE: return true;
            case N_FALSE: return false;
            case N_ATOM: return eval_atom(f, nd.atom, x);
            case N_NOT: return !beta(nd.a, x);
            case N_AND: return beta(nd.a, x) && beta(nd.b, x);
            case N_OR: return beta(nd.a, x) || beta(nd.b, x);
            default: throw std::runtime_error("not boolean");
        }
    }
    static void decide(Leaf& L, bool v) {
        L.pending = false;
        L.status = v ? T_TRUE : T_FALSE;
    }

    // entry of state x at time t (entry index k)
    void enter(double t, const int64_t* x) {
        for (Leaf& L : leaves) {
            if (!L.pending) continue;
            switch (L.kind) {
                case L_ATOM0:
                    decide(L, beta(L.beta1, x));
                    break;
                case L_F:
                    if (L.I.contains(t) && beta(L.beta1, x)) decide(L, true);
                    break;
                case L_G:
                    if (L.I.contains(t) && !beta(L.beta1, x)) decide(L, false);
                    break;
                case L_U:
                    if (L.I.contains(t) && beta(L.beta2, x)) decide(L, true);
                    else if (!beta(L.beta1, x)) decide(L, false);
                    break;
                case L_X:
                    if (k == 1) decide(L, L.I.contains(t) && beta(L.beta1, x));
                    break;
                case L_FG:
                case L_GF: {
                    bool b = beta(L.beta1, x);
                    if (L.kind == L_GF) b = !b;            // G F beta == !(F G !beta)
                    if (!b) L.rs_set = false;
                    else if (!L.rs_set && t <= L.I.hi) { L.rs_set = true; L.rs = t; }
                    break;
                }
                case L_GU: {
                    bool b1 = beta(L.beta1, x);
                    if (L.witness) {
                        if (!b1) decide(L, false);
                    } else if (beta(L.beta2, x)) {
                        if (k == 0) decide(L, true);
                        else {
                            L.witness = true;
                            L.D = t_prev + L.J.hi;
                            if (t > L.D) decide(L, true);
                            else if (!b1) decide(L, false);
                        }
                    } else if (!b1) {
                        decide(L, false);
                    }
                    break;
                }
            }
        }
    }
    // the next entry would happen at time tn (checked BEFORE the state changes)
    void advance(double tn) {
        for (Leaf& L : leaves) {
            if (!L.pending) continue;
            switch (L.kind) {
                case L_ATOM0: break;
                case L_F: if (L.I.beyond(tn)) decide(L, false); break;
                case L_G: if (L.I.beyond(tn)) decide(L, true); break;
                case L_U: if (L.I.beyond(tn)) decide(L, false); break;
                case L_X: if (k == 0 && !L.I.contains(tn)) decide(L, false); break;   // t_1 = tn not in I
                case L_FG:
                case L_GF: {
                    bool v;
                    bool dec = false;
                    if (L.rs_set && tn > L.rs + L.J.hi) { v = true; dec = true; }
                    else if (!L.rs_set && tn > L.I.hi) { v = false; dec = true; }
                    if (dec) decide(L, L.kind == L_FG ? v : !v);
                    break;
                }
                case L_GU:
                    if (L.witness) { if (tn > L.D) decide(L, true); }
                    else if (tn > L.I.hi) decide(L, false);
                    break;
            }
        }
    }
    // a0 == 0: the current state is absorbing, no further entries (reading R7)
    void absorb() {
        for (Leaf& L : leaves) {
            if (!L.pending) continue;
            switch (L.kind) {
                case L_ATOM0: break;
                case L_F: case L_U: case L_X: decide(L, false); break;
                case L_G: decide(L, true); break;
                case L_FG: decide(L, L.rs_set); break;
                case L_GF: decide(L, !L.rs_set); break;
                case L_GU: decide(L, L.witness); break;
            }
        }
    }
    // t_max passed (reading R5): pending leaves become unknown
    void timeout() {
        for (Leaf& L : leaves)
            if (L.pending) { L.pending = false; L.status = T_UNKNOWN; }
    }
    Tri root_value(int n) const {
        int li = leaf_of_node[n];
        if (li >= 0) {
            const Leaf& L = leaves[li];
            return L.pending ? T_UNKNOWN : L.status;
        }
        const Node& nd = f.nodes[n];
        switch (nd.kind) {
            case N_NOT: return t_not(root_value(nd.a));
            case N_AND: return t_and(root_value(nd.a), root_value(nd.b));
            case N_OR: return t_or(root_value(nd.a), root_value(nd.b));
            default: return T_UNKNOWN;
        }
    }
    // decided: the root is T/F, or nothing is pending any more
    bool decided(Tri* out) const {
        Tri r = root_value(f.root);
        if (r != T_UNKNOWN) { *out = r; return true; }
        for (const Leaf& L : leaves) if (L.pending) return false;
        *out = T_UNKNOWN;
        return true;
    }
};

// -----------------------------------------------------------------------------
// 6. One replica: SSA direct method (template steps 1-5; Eq. 2a/2b,
//    P:156-165) driven by the streaming monitor (on-the-fly).
//    Full recompute of all a_j every event (the dependency graph
//    only reproduces this faster).
// -----------------------------------------------------------------------------
enum Verdict { V_FALSE = 0, V_TRUE = 1, V_ERROR = 2 };
static const int64_t COUNT_LIMIT = 2147483647LL;   // int32 counts (reading R17)

struct RunResult { int verdict; int64_t events; };

RunResult run_streaming(const Model& M, const Formula& f, uint64_t seed, uint64_t traj, int64_t event_cap) {
    std::vector<int64_t> x = M.x0;
    std::vector<double> a(M.R.size());
    Monitor mon(f);
    double t = 0.0;
    int64_t k = 0;
    mon.k = 0;
    mon.t_prev = 0.0;
    mon.enter(0.0, x.data());                  // sigma_buff = {(s0,t0)}
    Tri v;
    while (!mon.decided(&v)) {
        // step 1: a_0 = sum_j a_j, left to right in reaction order (reading R12)
        double a0 = 0.0;
        for (size_t j = 0; j < M.R.size(); ++j) {
            a[j] = propensity(M.R[j], x.data());
            a0 = (j == 0) ? a[j] : a0 + a[j];
        }
        if (!(a0 >= 0.0) || std::isinf(a0)) return {V_ERROR, k};   // bad propensity
        if (a0 == 0.0) {                           // template step 5 "Terminate" (R7)
            mon.absorb();
            continue;
        }
        double u1, u2;
        step_uniforms(seed, traj, (uint64_t)k, &u1, &u2);
        double e = -std::log(u1);
        double tau = e / a0;                       // step 3, Eq. 2a
        double tn = t + tau;
        mon.advance(tn);                           // close windows that tn passes
        if (mon.decided(&v)) break;
        if (f.t_max > 0.0 && tn > f.t_max) {       // pessimistic cut-off
            mon.timeout();
            continue;
        }
        // step 2: j = min{ j : sum_{i<=j} a_i > u2 a_0 }, Eq. 2b
        double target = u2 * a0;
        double acc = 0.0;
        int j = -1;
        for (size_t i = 0; i < M.R.size(); ++i) {
            acc = (i == 0) ? a[i] : acc + a[i];
            if (acc > target) { j = (int)i; break; }
        }
        if (j < 0)                                 // rounding: last j with a_j > 0 (R11)
            for (int i = (int)M.R.size() - 1; i >= 0; --i)
                if (a[(size_t)i] > 0.0) { j = i; break; }
        // step 4: x <- x + v_j, t <- t + tau
        for (const auto& ch : M.R[(size_t)j].change) {
            int64_t nv = x[(size_t)ch.first] + ch.second;
            if (nv > COUNT_LIMIT) return {V_ERROR, k};
            x[(size_t)ch.first] = nv;
        }
        mon.t_prev = t;
        t = tn;
        ++k;
        mon.k = k;
        mon.enter(t, x.data());
        if (k >= event_cap) {
            if (!mon.decided(&v)) return {V_ERROR, k};
        }
    }
    return {v == T_TRUE ? V_TRUE : V_FALSE, k};   // unknown -> false at the root
}

// Simulate WITHOUT on-the-fly halting up to horizon H (first entry time > H
// is recorded as the overshoot), storing the trace; used by literal mode.
bool simulate_trace(const Model& M, uint64_t seed, uint64_t traj, double H, int64_t event_cap,
                    const std::vector<int>& keep, Trace* tr, bool* error, bool cap_is_error = true) {
    std::vector<int64_t> x = M.x0;
    std::vector<double> a(M.R.size());
    tr->N = (int)keep.size();
    tr->t.assign(1, 0.0);
    tr->tau.clear();
    tr->x.clear();
    for (int s : keep) tr->x.push_back(x[(size_t)s]);
    tr->absorbed = false;
    *error = false;
    double t = 0.0;
    int64_t k = 0;
    for (;;) {
        double a0 = 0.0;
        for (size_t j = 0; j < M.R.size(); ++j) {
            a[j] = propensity(M.R[j], x.data());
            a0 = (j == 0) ? a[j] : a0 + a[j];
        }
        if (!(a0 >= 0.0) || std::isinf(a0)) { *error = true; return false; }
        if (a0 == 0.0) { tr->absorbed = true; return true; }
        double u1, u2;
        step_uniforms(seed, traj, (uint64_t)k, &u1, &u2);
        double e = -std::log(u1);
        double tau = e / a0;
        double tn = t + tau;
        tr->tau.push_back(tau);
        if (tn > H) return true;                   // overshoot: next entry unknown
        double target = u2 * a0;
        double acc = 0.0;
        int j = -1;
        for (size_t i = 0; i < M.R.size(); ++i) {
            acc = (i == 0) ? a[i] : acc + a[i];
            if (acc > target) { j = (int)i; break; }
        }
        if (j < 0)
            for (int i = (int)M.R.size() - 1; i >= 0; --i)
                if (a[(size_t)i] > 0.0) { j = i; break; }
        for (const auto& ch : M.R[(size_t)j].change) {
            int64_t nv = x[(size_t)ch.first] + ch.second;
            if (nv > COUNT_LIMIT) { *error = true; return false; }
            x[(size_t)ch.first] = nv;
        }
        t = tn;
        ++k;
        tr->t.push_back(t);
        for (int s : keep) tr->x.push_back(x[(size_t)s]);
        if (k >= event_cap) {
            if (cap_is_error) { *error = true; return false; }
            return true;                           // truncated (tests only): tau has n entries
        }
    }
}

}  // namespace orc

// =============================================================================
// C interface for ctypes (tests / bench cpu_baseline only)
// =============================================================================
using namespace orc;

static thread_local std::string g_err;

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

void orc_philox(uint64_t seed, uint64_t traj, uint64_t step, uint32_t* out4) {
    uint32_t ctr[4] = {(uint32_t)step, (uint32_t)(step >> 32), (uint32_t)traj, (uint32_t)(traj >> 32)};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    philox4x32_10(ctr, key, out4);
}
void orc_philox_raw(const uint32_t* ctr4, const uint32_t* key2, uint32_t* out4) { philox4x32_10(ctr4, key2, out4); }
void orc_uniforms(uint64_t seed, uint64_t traj, uint64_t step, double* u1, double* u2) {
    step_uniforms(seed, traj, step, u1, u2);
}

// reactants/products: [M][2] species index (-1 none) and stoichiometry
void* orc_model_new(int32_t N, const int64_t* x0, int32_t M, const int32_t* r_idx, const int32_t* r_st,
                    const int32_t* p_idx, const int32_t* p_st, const double* rate) {
    try {
        auto* m = new Model();
        m->N = N;
        m->x0.assign(x0, x0 + N);
        for (int j = 0; j < M; ++j) {
            Reaction r;
            r.c = rate[j];
            std::vector<int64_t> delta((size_t)N, 0);
            for (int q = 0; q < 2; ++q) {
                int s = r_idx[2 * j + q];
                if (s < 0) continue;
                bool merged = false;
                for (auto& rs : r.reactants)
                    if (rs.first == s) { rs.second += r_st[2 * j + q]; merged = true; }
                if (!merged) r.reactants.push_back({s, r_st[2 * j + q]});
                delta[(size_t)s] -= r_st[2 * j + q];
            }
            for (int q = 0; q < 2; ++q) {
                int s = p_idx[2 * j + q];
                if (s < 0) continue;
                delta[(size_t)s] += p_st[2 * j + q];
            }
            for (auto& rs : r.reactants)
                if (rs.second > 2) throw std::runtime_error("stoichiometry > 2");
            for (int s = 0; s < N; ++s)
                if (delta[(size_t)s] != 0) r.change.push_back({s, (int)delta[(size_t)s]});
            m->R.push_back(r);
        }
        return m;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
int orc_model_set_hill(void* mp, int32_t j, int32_t repressor, double K, int32_t n) {
    auto* m = (Model*)mp;
    if (j < 0 || j >= (int)m->R.size() || repressor < 0 || repressor >= m->N || !(K > 0) || n < 1) return -1;
    m->R[(size_t)j].hill = true;
    m->R[(size_t)j].repressor = repressor;
    m->R[(size_t)j].K = K;
    m->R[(size_t)j].n = n;
    return 0;
}
// explicit rate expression for reaction j over species names[0..N) (replaces mass action)
int orc_model_set_rate(void* mp, int32_t j, const char* expr, const char* const* names) {
    auto* m = (Model*)mp;
    if (j < 0 || j >= (int)m->R.size() || !expr || !names) return -1;
    try {
        std::vector<std::string> nm;
        for (int i = 0; i < m->N; ++i) nm.push_back(names[i]);
        std::vector<RateNode> t;
        std::string text(expr);
        RateParser P{text, nm, t};
        P.expr();
        P.ws();
        if (P.p != text.size()) P.fail("trailing input");
        m->R[(size_t)j].rate = t;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}
void orc_model_free(void* m) { delete (Model*)m; }

double orc_propensity(void* mp, int32_t j, const int64_t* x) { return propensity(((Model*)mp)->R[(size_t)j], x); }

void* orc_formula_new(const char* text, const char* const* names, int32_t n_names, double t_max) {
    try {
        std::vector<std::string> nm;
        for (int i = 0; i < n_names; ++i) nm.push_back(names[i]);
        auto* f = new Formula();
        f->t_max = t_max;
        std::string s(text);
        Parser P(s, nm, *f);
        f->root = P.formula();
        P.ws();
        if (P.p != s.size()) P.fail("trailing input");
        std::vector<char> used((size_t)n_names, 0);
        for (const Atom& a : f->atoms) { collect_species(*f, a.lhs, used); collect_species(*f, a.rhs, used); }
        for (int i = 0; i < n_names; ++i) if (used[(size_t)i]) f->species_used.push_back(i);
        return f;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void orc_formula_free(void* f) { delete (Formula*)f; }
double orc_formula_reach(void* fp) { auto* f = (Formula*)fp; return reach(*f, f->root); }
int orc_formula_streamable(void* fp) {
    try { Monitor m(*(Formula*)fp); return 1; } catch (...) { return 0; }
}

// Literal |= and the streaming monitor on a caller-supplied trace.
// t[n+1] entry times, tau[n+1 or n] sojourns, x[(n+1)*N_all] states.
// Returns 0/1/2 (false/true/unknown); *decided_at = entry index at which the
// streaming monitor decided (streaming only).
int orc_check_literal(void* fp, int64_t n_entries, const double* t, const double* tau, const int64_t* x,
                      int32_t N, int32_t absorbed) {
    auto* f = (Formula*)fp;
    Trace tr;
    tr.N = N;
    tr.t.assign(t, t + n_entries);
    tr.tau.assign(tau, tau + (absorbed ? n_entries - 1 : n_entries));
    tr.x.assign(x, x + n_entries * N);
    tr.absorbed = absorbed != 0;
    LiteralChecker lc(*f, tr);
    return (int)lc.value(f->root, 0);
}
int orc_check_streaming(void* fp, int64_t n_entries, const double* t, const double* tau, const int64_t* x,
                        int32_t N, int32_t absorbed, int64_t* decided_at) {
    auto* f = (Formula*)fp;
    try {
        Monitor mon(*f);
        Tri v;
        mon.k = 0;
        mon.enter(t[0], x);
        *decided_at = 0;
        if (mon.decided(&v)) return (int)v;
        for (int64_t k = 1; k < n_entries; ++k) {
            mon.advance(t[k]);
            if (mon.decided(&v)) { *decided_at = k; return (int)v; }
            mon.t_prev = t[k - 1];
            mon.k = k;
            mon.enter(t[k], x + k * N);
            if (mon.decided(&v)) { *decided_at = k; return (int)v; }
        }
        *decided_at = n_entries;
        if (absorbed) {
            mon.absorb();
        } else {
            mon.advance(t[n_entries - 1] + tau[n_entries - 1]);
        }
        if (mon.decided(&v)) return (int)v;
        return (int)T_UNKNOWN;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// One batch of replicas [first, first+n): mode 0 = streaming (on-the-fly),
// 1 = literal (simulate to the horizon, evaluate |=; the event count is the first
// index at which the observed prefix decides |=).  verdicts/events may be
// NULL.  counts[4] = {n_true, n_false, events, errors}.
int orc_run(void* mp, void* fp, uint64_t seed, uint64_t first, uint64_t n, int32_t mode, int64_t event_cap,
            uint8_t* verdicts, int64_t* events, int64_t* counts) {
    auto* M = (Model*)mp;
    auto* f = (Formula*)fp;
    counts[0] = counts[1] = counts[2] = counts[3] = 0;
    try {
        double H = 0.0;
        if (mode == 1) {
            H = (f->t_max > 0.0) ? f->t_max : reach(*f, f->root);
            if (!std::isfinite(H)) throw std::runtime_error("unbounded formula needs t_max > 0");
        } else {
            Monitor probe(*f);   // throws when outside the streaming fragment
            if (f->t_max <= 0.0 && !std::isfinite(reach(*f, f->root)))
                throw std::runtime_error("unbounded formula needs t_max > 0");
        }
        for (uint64_t q = 0; q < n; ++q) {
            uint64_t i = first + q;
            RunResult rr;
            if (mode == 0) {
                rr = run_streaming(*M, *f, seed, i, event_cap);
            } else {
                Trace tr;
                bool err = false;
                // the literal checker evaluates atoms on stored states: keep all species
                std::vector<int> keep;
                for (int s = 0; s < M->N; ++s) keep.push_back(s);
                // the event cap truncates the stored trace (the replica is an error only if
                // no prefix with fewer than event_cap events decides |=, below)
                simulate_trace(*M, seed, i, H, event_cap, keep, &tr, &err, false);
                const bool truncated = !err && !tr.absorbed && (int64_t)tr.tau.size() == tr.n();
                if (err) rr = {V_ERROR, tr.n()};
                else {
                    // On-the-fly halting (the replica stops as soon as the formula
                    // is decided): the event count is the FIRST k at which the three-valued |=
                    // of the observed prefix -- entries 0..k and the sojourn of entry k, the
                    // unobserved future unknown -- is definite.  The prefix of the stored trace
                    // is exactly what the simulation had observed after drawing step k (the
                    // streams are keyed by step).  Definiteness is monotone in k (observing
                    // more never revokes a definite value), so the first such k is found by
                    // bisection over [0, n); if no proper prefix decides, the whole trace
                    // (horizon overshoot or absorption) does, with all n events.
                    // prefix k's checker, seeded with the definite values of the longest prefix
                    // known to be undecided (`base`); bisection over [0, n) by monotonicity
                    std::unique_ptr<LiteralChecker> base;
                    auto prefix_check = [&](int64_t k, std::unique_ptr<Trace>& keep) {
                        keep.reset(new Trace());
                        Trace& p = *keep;
                        p.N = tr.N;
                        p.t.assign(tr.t.begin(), tr.t.begin() + k + 1);
                        p.tau.assign(tr.tau.begin(), tr.tau.begin() + k + 1);
                        p.x.assign(tr.x.begin(), tr.x.begin() + (k + 1) * tr.N);
                        p.absorbed = false;
                        std::unique_ptr<LiteralChecker> pc(new LiteralChecker(*f, p));
                        if (base) pc->seed(*base);
                        return pc;
                    };
                    const int64_t n_ev = tr.n();
                    const int64_t last = n_ev - 1;
                    std::unique_ptr<Trace> base_tr, hi_tr;
                    int64_t lo = -1, hi = -1;                    // lo undecided, hi definite
                    Tri hv = T_UNKNOWN;
                    // gallop: prefixes 63, 127, 255, ... (each seeded from the previous one)
                    for (int64_t k = std::min<int64_t>(63, last); k >= 0 && hi < 0;
                         k = (k == last) ? -1 : std::min<int64_t>(2 * k + 1, last)) {
                        std::unique_ptr<Trace> kt;
                        auto pc = prefix_check(k, kt);
                        const Tri v = pc->value(f->root, 0);
                        if (v != T_UNKNOWN) { hi = k; hv = v; }
                        else { lo = k; base = std::move(pc); base_tr = std::move(kt); }
                    }
                    if (hi >= 0) {
                        while (hi - lo > 1) {
                            const int64_t mid = lo + (hi - lo) / 2;
                            std::unique_ptr<Trace> kt;
                            auto pc = prefix_check(mid, kt);
                            const Tri v = pc->value(f->root, 0);
                            if (v != T_UNKNOWN) { hi = mid; hv = v; }
                            else { lo = mid; base = std::move(pc); base_tr = std::move(kt); }
                        }
                    }
                    const Tri pv = hv;
                    if (pv != T_UNKNOWN) {
                        rr = {pv == T_TRUE ? V_TRUE : V_FALSE, hi};
                    } else if (truncated) {
                        rr = {V_ERROR, n_ev};             // event cap reached undecided
                    } else {
                        LiteralChecker lc(*f, tr);
                        if (base) lc.seed(*base);
                        Tri v = lc.value(f->root, 0);
                        rr = {v == T_TRUE ? V_TRUE : V_FALSE, n_ev};
                    }
                }
            }
            if (verdicts) verdicts[q] = (uint8_t)rr.verdict;
            if (events) events[q] = rr.events;
            if (rr.verdict == V_TRUE) counts[0]++;
            else if (rr.verdict == V_FALSE) counts[1]++;
            else counts[3]++;
            counts[2] += rr.events;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Full trace to horizon H (all species), for SSA statistics tests.
// Returns number of entries written (<= cap_entries), -1 on error.
// Truncated at cap_entries entries if the horizon is not reached first.
int64_t orc_simulate(void* mp, uint64_t seed, uint64_t traj, double H, int64_t cap_entries, double* t_out,
                     double* tau_out, int64_t* x_out, int32_t* absorbed, int64_t* n_tau) {
    auto* M = (Model*)mp;
    Trace tr;
    bool err = false;
    std::vector<int> keep;
    for (int s = 0; s < M->N; ++s) keep.push_back(s);
    simulate_trace(*M, seed, traj, H, cap_entries - 1 > 0 ? cap_entries - 1 : 1, keep, &tr, &err, false);
    *n_tau = (int64_t)tr.tau.size();
    if (err) return -1;
    int64_t ne = (int64_t)tr.t.size();
    if (ne > cap_entries) return -1;
    std::memcpy(t_out, tr.t.data(), sizeof(double) * (size_t)ne);
    std::memcpy(tau_out, tr.tau.data(), sizeof(double) * tr.tau.size());
    std::memcpy(x_out, tr.x.data(), sizeof(int64_t) * tr.x.size());
    *absorbed = tr.absorbed ? 1 : 0;
    return ne;
}

}  // extern "C"
