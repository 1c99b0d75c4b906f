// smc_internal.hpp -- host-side data structures of libsmc (B200 path).
// Independent of oracle/: nothing here is shared with the CPU oracle.
#pragma once
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/smc.h"

namespace smc {

// ---------------------------------------------------------------- errors ---
void set_error(const std::string& msg);
struct Error {
    int code;
    std::string msg;
};
[[noreturn]] void fail(int code, const std::string& msg);

// ----------------------------------------------------------------- model ---
// Explicit rate expression node (rates.cpp); the root is the last node.
struct RNode {
    enum K { CONST, SPECIES, ADD, SUB, MUL, DIV, NEG } k = CONST;
    double v = 0.0;
    int species = -1;
    int a = -1, b = -1;
};
std::vector<RNode> parse_rate(const std::string& expr, const std::vector<std::string>& names);
void rate_species(const std::vector<RNode>& t, std::vector<int>& out);

// One reaction channel R_j after normalisation.
struct Reaction {
    int s[2] = {-1, -1};     // reactant species (merged), -1 = none
    int st[2] = {0, 0};      // stoichiometry 1..2
    std::vector<std::pair<int, int>> change;   // (species, delta != 0), species ascending
    double c = 0.0;
    bool hill = false;
    int rep = -1;
    double K = 0.0;
    int n = 0;
    std::vector<RNode> rate;   // explicit propensity (replaces c * h), empty = mass action
};

struct Kernel;        // compiled + loaded module (jit.cpp)
struct DeviceState;   // device buffers (runtime.cpp)
struct DeviceStateDeleter { void operator()(DeviceState* d) const; };

struct Model {
    int N = 0, M = 0;
    std::vector<int32_t> x0;
    std::vector<Reaction> R;
    int variant_forced = 0;
    uint64_t event_cap = 2147483647ull;
    bool speculate = true;           // prefix-exact speculative rounds in smc_estimate
    // dependency graph: dep[j] = { k : species(law_k) intersects changed(j) }
    std::vector<std::vector<int>> dep;
    bool deps_built = false;
    // run state
    uint64_t cursor = 0;
    uint64_t last_seed = 0;
    bool has_seed = false;
    std::unique_ptr<DeviceState, DeviceStateDeleter> dev;
    std::mutex mu;
    void build_deps();
    std::vector<int> law_species(int k) const;   // species read by a_k
    int variant() const;                          // 1 thread-owned, 2 tile, 4 sweep, 5 delta
    bool sweep_fits() const;
    bool delta_fits() const;                      // variant 5 can hold the model
};

// -------------------------------------------------------------- property ---
enum class Cmp { LT, LE, GE, GT, EQ, NE };
// general val of P:209 (val ~ val, func, Int, Real)
struct VNode {
    enum K { INT, REAL, SPECIES, ADD, SUB, MUL, DIV, NEG, SQRT, ABS, MIN, MAX, POW } k = INT;
    int64_t i = 0;      // INT value, POW exponent
    double d = 0.0;     // REAL value
    int s = -1;         // SPECIES
    int a = -1, b = -1;
};
struct Atom {
    // integer-linear atoms: sum_s coef[s] x_s + cst  (cmp)  0, exact int64
    std::vector<std::pair<int, int64_t>> coef;
    int64_t cst = 0;
    Cmp op = Cmp::GT;
    // general atoms: lhs (cmp) rhs over the trees in v; int64 when only Int constants,
    // species, + - * occur (non-linear products), binary64 otherwise ('/', Real, func)
    bool general = false;
    bool real = false;
    std::vector<VNode> v;
    int lhs = -1, rhs = -1;
};
struct Interval {
    double lo = 0.0, hi = 0.0;      // hi = +inf when unbounded
    bool lo_open = false, hi_open = false;
    bool finite() const;
};
// boolean expression over atoms: postfix-free tree
struct BExpr {
    enum K { ATOM, TRUE_, FALSE_, NOT, AND, OR } k;
    int atom = -1;
    int a = -1, b = -1;
};
enum class LeafKind { ATOM0, F, G, U, X, FG, GF, GU };
struct Leaf {
    LeafKind kind;
    Interval I, J;       // outer / inner interval
    int b1 = -1, b2 = -1;   // BExpr roots (-1 = tt)
};
struct RootExpr {        // Kleene combination of leaves
    enum K { LEAF, NOT, AND, OR } k;
    int leaf = -1;
    int a = -1, b = -1;
};
// AST node of a formula outside the streaming fragment (kept for the literal variant)
struct LNode {
    enum K { ATOM, TRUE_, FALSE_, NOT, AND, OR, X, U, F, G } k = TRUE_;
    Interval I;
    int a = -1, b = -1;
    int atom = -1;
};
struct Property {
    uint64_t id = 0;
    // formulas outside the streaming fragment of reading R16: each replica's trace is
    // buffered to the horizon and |= is evaluated literally on it (variant 3)
    bool literal = false;
    std::vector<LNode> lnodes;   // children before parents
    int lroot = -1;
    std::string text;
    int N = 0;
    double t_max = 0.0;
    std::vector<Atom> atoms;
    std::vector<BExpr> bexprs;
    std::vector<Leaf> leaves;
    std::vector<RootExpr> root;
    int root_idx = -1;
    double horizon = 0.0;
};
std::unique_ptr<Property> compile_property(const Model& m, const std::string& text,
                                           const std::vector<std::string>& names, double t_max);

// --------------------------------------------------------------- codegen ---
struct TileLayout {               // packed model tables (variant 2), byte offsets
    int tw = 32;                  // lanes per trajectory tile
    int gs = 0;                   // reactions per lane group
    int gsp = 0;                  // row stride of a group in the row layout (odd), else gs
    bool row = true;              // row layout of a (ssa_tile.cuh smc_slot)
    int ch = 0;                   // level-2 chunk per lane
    int n_pad = 0;
    size_t tile_bytes = 0;        // smem per trajectory
    size_t off_x0 = 0, off_law = 0, off_hill_rep = 0, off_hill_k = 0, off_hill_n = 0;
    size_t off_chg = 0, off_dep_off = 0, off_dep = 0, bytes = 0;
    bool any_hill = false;
    bool any_general = false;     // a reaction of order 3-4 (int64 law path)
    bool dep16 = false;           // 2-byte dependency entries (k only)
    bool depsp = false;           // species-indexed reader CSR instead of dep(j) (TW = 32)
    bool fatdep = false;          // 16-byte dependency entries carrying the law (meta, rate)
    bool any_explicit = false;    // an explicit rate expression (generated smc_explicit)
    // variant 4 (sweep): law table in the sweep format, padded to G*S entries
    size_t off_swlaw = 0;
    int sw_s = 0, sw_c = 0;       // laws per group, independent law reads per chunk
    bool sw_xd = false;           // counts as binary64 columns
    int sw_blk = 128;             // CTA size = stride of the count columns
    int max_dep = 0;
    // variant 5 (delta): G exact fixed-point group sums of S laws, Cq = round(c 2^L)
    int dg = 0, ds = 0, drmax = 0, dl = 0;
    size_t smem_bytes = 0;        // variant 5: the TMA-staged prefix (the rest is read through L1)
    std::vector<uint8_t> blob;    // host copy
};
TileLayout pack_tables(const Model& m, bool sweep = false);   // sweep: law/change tables only (variant 4)
TileLayout pack_delta_tables(const Model& m);                 // variant 5
int delta_scale(const Model& m);  // L of variant 5, or -1 if the model is not eligible
int thread_minb(const Model& m);    // resident 128-thread units per SM of variant 1 (codegen.cpp)
int thread_block(const Model& m);   // CTA size of variant 1
// variant 1: zero-order Hill propensities a_k(x_r), x_r < size, tabulated on the host with
// the same IEEE operations as the law (one __ldg instead of two divisions per update)
struct HillTables {
    int size = 2048;
    std::vector<long long> offset;   // per reaction, -1 = not tabulated
    std::vector<double> values;
};
HillTables pack_hill_tables(const Model& m);
std::string generate_source(const Model& m, const Property& p, int variant, const TileLayout* tl);
// bytes per ring entry of one replica slot of the window monitor (ssa_window.cuh, R27)
size_t window_bytes_per_entry(const Property& p);
// bytes per replica slot of the single-position nodes' small area
size_t window_small_bytes(const Property& p);
std::string embedded_source(const char* name);   // kernels/*.cuh embedded at build time

// -------------------------------------------------------------------- jit ---
struct Kernel {
    void* library = nullptr;      // cudaLibrary_t
    void* kernel = nullptr;       // cudaKernel_t
    int regs = 0;
    float compile_ms = 0.f;
    std::string name;
};
std::shared_ptr<Kernel> get_kernel(const std::string& source, const char* entry);

// --------------------------------------------------------------- runtime ---
struct Hooks {
    void* (*alloc)(size_t, void*) = nullptr;
    void (*free_)(void*, void*) = nullptr;
    void* alloc_user = nullptr;
    void* stream = nullptr;
    int rank = 0, world = 1;
    int (*allreduce)(int64_t*, int32_t, void*) = nullptr;
    void* allreduce_user = nullptr;
};
Hooks& hooks();

// global counts of round range [base, base+n): shard + allreduce
int run_round(Model& m, const Property& p, uint64_t seed, uint64_t base, uint64_t n, smc_counts* out);

// ---------------------------------------------------------------- wilson ---
double normal_quantile(double c);
void wilson_interval(double p_hat, double n, double z, double* lo, double* hi);
int64_t wilson_sample_size(double p, double eps, double z);
double round_estimate(double p_hat, double eps);

}  // namespace smc

struct smc_model {
    smc::Model m;
};
struct smc_property {
    std::unique_ptr<smc::Property> p;
};
