// rates.cpp -- explicit (non-mass-action) propensity expressions (Table 2,
// P:513-538) for smc_model_set_rate_expr.  Tokenised, then
// parsed by precedence climbing into a postfix-free node list; codegen.cpp turns
// the tree into straight-line IEEE binary64 code (__dadd_rn / __dmul_rn /
// __ddiv_rn in tree order, left-associative), so every evaluation of a_j is
// reproducible bit for bit.
#include <cctype>
#include <cstdlib>
#include <cstring>

#include "smc_internal.hpp"

namespace smc {

namespace {

struct Tok {
    enum K { NUM, ID, OP, LP, RP, END } k;
    double v = 0.0;
    std::string s;
    char op = 0;
    size_t pos = 0;
};

std::vector<Tok> tokenize(const std::string& e) {
    std::vector<Tok> out;
    size_t i = 0;
    while (i < e.size()) {
        const char ch = e[i];
        if (std::isspace((unsigned char)ch)) { ++i; continue; }
        Tok t;
        t.pos = i;
        if (std::isdigit((unsigned char)ch) || ch == '.') {
            char* end = nullptr;
            t.k = Tok::NUM;
            t.v = std::strtod(e.c_str() + i, &end);
            if (end == e.c_str() + i) fail(SMC_E_PARSE, "rate expression: bad number at " + std::to_string(i));
            i = (size_t)(end - e.c_str());
        } else if (std::isalpha((unsigned char)ch) || ch == '_') {
            t.k = Tok::ID;
            while (i < e.size() && (std::isalnum((unsigned char)e[i]) || e[i] == '_')) t.s += e[i++];
        } else if (std::strchr("+-*/", ch)) {
            t.k = Tok::OP;
            t.op = ch;
            ++i;
        } else if (ch == '(') {
            t.k = Tok::LP;
            ++i;
        } else if (ch == ')') {
            t.k = Tok::RP;
            ++i;
        } else {
            fail(SMC_E_PARSE, std::string("rate expression: unexpected '") + ch + "' at " + std::to_string(i));
        }
        out.push_back(t);
    }
    Tok end;
    end.k = Tok::END;
    end.pos = e.size();
    out.push_back(end);
    return out;
}

struct Climber {
    const std::vector<Tok>& t;
    const std::vector<std::string>& names;
    std::vector<RNode>& nodes;
    size_t i = 0;

    [[noreturn]] void err(const std::string& m) {
        fail(SMC_E_PARSE, "rate expression: " + m + " at " + std::to_string(t[i].pos));
    }
    int add(const RNode& n) {
        nodes.push_back(n);
        return (int)nodes.size() - 1;
    }
    static int prec(char op) { return (op == '+' || op == '-') ? 1 : 2; }
    int atom() {
        const Tok& k = t[i];
        if (k.k == Tok::OP && k.op == '-') {          // unary minus binds tighter than * and /
            ++i;
            RNode n;
            n.k = RNode::NEG;
            n.a = atom();
            return add(n);
        }
        if (k.k == Tok::NUM) { ++i; RNode n; n.k = RNode::CONST; n.v = k.v; return add(n); }
        if (k.k == Tok::ID) {
            for (size_t s = 0; s < names.size(); ++s)
                if (names[s] == k.s) { ++i; RNode n; n.k = RNode::SPECIES; n.species = (int)s; return add(n); }
            err("unknown species '" + k.s + "'");
        }
        if (k.k == Tok::LP) {
            ++i;
            const int e = climb(1);
            if (t[i].k != Tok::RP) err("')' expected");
            ++i;
            return e;
        }
        err(k.k == Tok::END ? "unexpected end" : "operand expected");
    }
    int climb(int min_prec) {
        int lhs = atom();
        while (t[i].k == Tok::OP && prec(t[i].op) >= min_prec) {
            const char op = t[i].op;
            ++i;
            const int rhs = climb(prec(op) + 1);         // left-associative
            RNode n;
            n.k = op == '+' ? RNode::ADD : op == '-' ? RNode::SUB : op == '*' ? RNode::MUL : RNode::DIV;
            n.a = lhs;
            n.b = rhs;
            lhs = add(n);
        }
        return lhs;
    }
};

}  // namespace

std::vector<RNode> parse_rate(const std::string& expr, const std::vector<std::string>& names) {
    const std::vector<Tok> toks = tokenize(expr);
    std::vector<RNode> nodes;
    Climber c{toks, names, nodes};
    const int root = c.climb(1);
    if (toks[c.i].k != Tok::END) c.err("trailing input");
    if (root != (int)nodes.size() - 1) fail(SMC_E_PARSE, "rate expression: internal root order");
    return nodes;
}

void rate_species(const std::vector<RNode>& t, std::vector<int>& out) {
    for (const RNode& n : t)
        if (n.k == RNode::SPECIES) out.push_back(n.species);
}

}  // namespace smc
