// model.cpp -- model packer: validation, reactant merging, change vectors and
// the reaction dependency graph.
#include <cstdlib>
#include <algorithm>
#include <cmath>
#include <set>
#include <sstream>

#include "smc_internal.hpp"

namespace smc {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
const char* last_error() { return g_err.c_str(); }
[[noreturn]] void fail(int code, const std::string& msg) { throw Error{code, msg}; }

// species whose counts a_k reads (reactants, Hill repressor)
std::vector<int> Model::law_species(int k) const {
    std::vector<int> s;
    const Reaction& r = R[(size_t)k];
    for (int q = 0; q < 2; ++q)
        if (r.s[q] >= 0) s.push_back(r.s[q]);
    if (r.hill) s.push_back(r.rep);
    rate_species(r.rate, s);
    std::sort(s.begin(), s.end());
    s.erase(std::unique(s.begin(), s.end()), s.end());
    return s;
}

// dep(j) = { k : law_species(k) intersects changed(j) } (ascending k).
// Only these a_k can change when R_j fires; recomputing exactly them gives the
// same propensity vector as a full recompute.
void Model::build_deps() {
    if (deps_built) return;
    std::vector<std::vector<int>> readers((size_t)N);
    for (int k = 0; k < M; ++k)
        for (int s : law_species(k)) readers[(size_t)s].push_back(k);
    dep.assign((size_t)M, {});
    for (int j = 0; j < M; ++j) {
        std::set<int> d;
        for (auto& ch : R[(size_t)j].change)
            for (int k : readers[(size_t)ch.first]) d.insert(k);
        dep[(size_t)j].assign(d.begin(), d.end());
    }
    deps_built = true;
}

// variant 4 (sweep) holds the counts of 128 trajectories per CTA in shared memory
bool Model::sweep_fits() const { return N <= 4095 && 128 * 4 * (size_t)(N + 1) + 24 * (size_t)M + 4096 <= 200 * 1024; }

// variant 5 (exact fixed-point group sums, dependency deltas): mass action of order <= 2
// only, rates within the fixed-point range (delta_scale), 16-bit reaction indices
bool Model::delta_fits() const { return M <= 65535 && N <= 65534 && delta_scale(*this) >= 0; }

int Model::variant() const {
    if (variant_forced) return variant_forced;
    if (N <= 32 && M <= 32) return 1;
    // sweep for mid-size networks (pass 1 is straight-line code over all M laws with the
    // counts in registers): the register copy of the counts decides -- measured faster than
    // the tile kernel for N <= 160 up to M = 1000 (scripts/variant_boundary.py: 1.3-3.4x),
    // slower at N = 200 (M 512: 0.54x, C5's M 1000: 0.56x).  SMC_SWEEP=0/1 forces the
    // automatic choice off / on
    bool sweep = N <= 160 && M <= 1024;
    if (const char* e = std::getenv("SMC_SWEEP")) sweep = std::atoi(e) != 0;
    if (sweep && sweep_fits()) return 4;
    // larger mass-action networks (C5): the delta kernel (no stored propensities);
    // SMC_DELTA=0 keeps the tile kernel
    bool delta = true;
    if (const char* e = std::getenv("SMC_DELTA")) delta = std::atoi(e) != 0;
    return (delta && delta_fits()) ? 5 : 2;
}

}  // namespace smc

using namespace smc;

extern "C" {

const char* smc_last_error(void) { return smc::last_error(); }

int smc_model_create(int32_t n_species, const int32_t* init_counts, int32_t n_reactions,
                     const int32_t* reactant_idx, const int32_t* reactant_st, const int32_t* product_idx,
                     const int32_t* product_st, const double* rate, smc_model** out) {
    if (!out) { set_error("smc_model_create: out is NULL"); return SMC_E_ARG; }
    *out = nullptr;
    if (n_species < 1 || n_reactions < 1 || !init_counts || !reactant_idx || !reactant_st || !product_idx ||
        !product_st || !rate) {
        set_error("smc_model_create: need n_species >= 1, n_reactions >= 1 and non-NULL arrays");
        return SMC_E_ARG;
    }
    if (n_species > 4095 || n_reactions > 65535) {
        set_error("smc_model_create: at most 4095 species and 65535 reactions");
        return SMC_E_ARG;
    }
    std::ostringstream viol;
    int nviol = 0;
    auto bad = [&](const std::string& s) { viol << (nviol++ ? "; " : "") << s; };
    auto* h = new smc_model();
    Model& m = h->m;
    m.N = n_species;
    m.M = n_reactions;
    m.x0.assign(init_counts, init_counts + n_species);
    for (int s = 0; s < n_species; ++s)
        if (init_counts[s] < 0) bad("init_counts[" + std::to_string(s) + "] < 0");
    m.R.resize((size_t)n_reactions);
    for (int j = 0; j < n_reactions; ++j) {
        Reaction& r = m.R[(size_t)j];
        std::vector<long long> delta((size_t)n_species, 0);
        std::string tag = "reaction " + std::to_string(j);
        if (!(rate[j] > 0.0) || !std::isfinite(rate[j])) bad(tag + ": rate must be finite and > 0");
        r.c = rate[j];
        int nr = 0;
        for (int q = 0; q < 2; ++q) {
            int s = reactant_idx[2 * j + q], st = reactant_st[2 * j + q];
            if (s < 0) continue;
            if (s >= n_species) { bad(tag + ": reactant species out of range"); continue; }
            if (st < 1 || st > 2) { bad(tag + ": reactant stoichiometry must be 1..2"); continue; }
            delta[(size_t)s] -= st;
            if (nr == 1 && r.s[0] == s) { r.st[0] += st; continue; }   // A + A == 2A
            r.s[nr] = s;
            r.st[nr] = st;
            ++nr;
        }
        for (int q = 0; q < nr; ++q)
            if (r.st[q] > 2) bad(tag + ": merged stoichiometry > 2");
        for (int q = 0; q < 2; ++q) {
            int s = product_idx[2 * j + q], st = product_st[2 * j + q];
            if (s < 0) continue;
            if (s >= n_species) { bad(tag + ": product species out of range"); continue; }
            if (st < 1 || st > 2) { bad(tag + ": product stoichiometry must be 1..2"); continue; }
            delta[(size_t)s] += st;
        }
        for (int s = 0; s < n_species; ++s)
            if (delta[(size_t)s] != 0) r.change.push_back({s, (int)delta[(size_t)s]});
        // keep reactant slots ordered by species for a canonical law
        if (nr == 2 && r.s[1] < r.s[0]) { std::swap(r.s[0], r.s[1]); std::swap(r.st[0], r.st[1]); }
    }
    if (nviol) {
        delete h;
        set_error("model validation failed: " + viol.str());
        return SMC_E_MODEL;
    }
    *out = h;
    return SMC_OK;
}

int smc_model_set_hill(smc_model* h, int32_t reaction, int32_t repressor, double K, int32_t n) {
    if (!h) { set_error("smc_model_set_hill: NULL model"); return SMC_E_ARG; }
    Model& m = h->m;
    std::lock_guard<std::mutex> lk(m.mu);
    if (reaction < 0 || reaction >= m.M || repressor < 0 || repressor >= m.N || !(K > 0) || !std::isfinite(K) ||
        n < 1 || n > 8) {
        set_error("smc_model_set_hill: need valid reaction/repressor, K > 0, 1 <= n <= 8");
        return SMC_E_ARG;
    }
    if (m.dev) { set_error("smc_model_set_hill: model already used by a run"); return SMC_E_ARG; }
    if (!m.R[(size_t)reaction].rate.empty()) { set_error("smc_model_set_hill: reaction has an explicit rate"); return SMC_E_ARG; }
    Reaction& r = m.R[(size_t)reaction];
    r.hill = true;
    r.rep = repressor;
    r.K = K;
    r.n = n;
    m.deps_built = false;
    return SMC_OK;
}

int smc_model_set_rate_expr(smc_model* h, int32_t reaction, const char* expr, const char* const* species_names) {
    if (!h || !expr) { set_error("smc_model_set_rate_expr: NULL argument"); return SMC_E_ARG; }
    Model& m = h->m;
    std::lock_guard<std::mutex> lk(m.mu);
    if (reaction < 0 || reaction >= m.M) { set_error("smc_model_set_rate_expr: reaction out of range"); return SMC_E_ARG; }
    if (m.dev) { set_error("smc_model_set_rate_expr: model already used by a run"); return SMC_E_ARG; }
    if (m.R[(size_t)reaction].hill) { set_error("smc_model_set_rate_expr: reaction has Hill repression"); return SMC_E_ARG; }
    std::vector<std::string> names;
    for (int s = 0; s < m.N; ++s) names.push_back(species_names ? std::string(species_names[s]) : "S" + std::to_string(s));
    try {
        m.R[(size_t)reaction].rate = parse_rate(expr, names);
    } catch (const Error& e) {
        set_error(e.msg);
        return e.code;
    }
    m.deps_built = false;
    return SMC_OK;
}

int smc_model_set_variant(smc_model* h, int32_t variant) {
    if (!h || variant < 0 || variant > 5 || variant == 3) {
        set_error("smc_model_set_variant: variant 0 (automatic), 1, 2, 4 or 5");
        return SMC_E_ARG;
    }
    Model& m = h->m;
    if (variant == 5 && !m.delta_fits()) {
        set_error("smc_model_set_variant: delta variant needs mass action of order <= 2 with rates within 2^20 of "
                  "each other (fixed-point group sums, reading R26)");
        return SMC_E_ARG;
    }
    if (variant == 4 && !m.sweep_fits()) {
        set_error("smc_model_set_variant: sweep variant needs the counts of 128 trajectories in shared memory");
        return SMC_E_ARG;
    }
    if (variant == 1 && (m.N > 32 || m.M > 32)) {
        set_error("smc_model_set_variant: thread-owned variant needs N <= 32 and M <= 32");
        return SMC_E_ARG;
    }
    std::lock_guard<std::mutex> lk(m.mu);
    if (m.dev && variant != m.variant_forced) {
        set_error("smc_model_set_variant: model already used by a run");
        return SMC_E_ARG;
    }
    m.variant_forced = variant;
    return SMC_OK;
}

int smc_model_set_event_cap(smc_model* h, uint64_t cap) {
    // per-replica event counts are int32 on the device (events_out, spec_e)
    if (!h || cap < 1 || cap > 0x7FFFFFFFull) { set_error("smc_model_set_event_cap: 1 <= cap <= 2^31 - 1"); return SMC_E_ARG; }
    Model& m = h->m;
    std::lock_guard<std::mutex> lk(m.mu);
    if (m.dev && cap != m.event_cap) { set_error("smc_model_set_event_cap: model already used by a run"); return SMC_E_ARG; }
    m.event_cap = cap;
    return SMC_OK;
}

int smc_model_set_speculation(smc_model* h, int32_t on) {
    if (!h) { set_error("smc_model_set_speculation: NULL model"); return SMC_E_ARG; }
    Model& m = h->m;
    std::lock_guard<std::mutex> lk(m.mu);
    m.speculate = on != 0;
    return SMC_OK;
}

void smc_model_destroy(smc_model* h) { delete h; }

}  // extern "C"
