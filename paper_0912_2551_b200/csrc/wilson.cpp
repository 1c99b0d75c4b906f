// wilson.cpp -- host statistics of §3.3: z_{1-alpha/2}, Eq. 3,
// Eq. 4 and the iterative Wilson procedure of Fig. 2.
// Compiled with -ffp-contract=off: every double operation below is one IEEE
// binary64 round-to-nearest operation, in the order written (reading W8), so
// the results are bit-identical to any other correct evaluation of the same
// expression text (the oracle's is plain Python floats).
#include <cfloat>
#include <cmath>
#include <cstring>

#include "smc_internal.hpp"

namespace smc {

// z = Phi^{-1}((1 + c)/2) = sqrt(2) * w, erf(w) = c  (reading W1).
// Solved in x87 long double (64-bit mantissa): bisection to a 2^-70 bracket,
// then Newton steps, then one rounding to binary64.  For c >= 0.5 the
// complementary form erfc(w) = 1 - c keeps full relative accuracy in the tail.
double normal_quantile(double c) {
    if (!(c > 0.0 && c < 1.0)) return NAN;
    const bool tail = c >= 0.5;
    const long double target = tail ? (1.0L - (long double)c) : (long double)c;   // both exact
    auto F = [&](long double w) { return tail ? erfcl(w) : erfl(w); };           // tail: decreasing
    long double lo = 0.0L, hi = 28.0L;
    for (int it = 0; it < 200 && hi - lo > 1e-21L * (hi > 1 ? hi : 1); ++it) {
        long double mid = 0.5L * (lo + hi);
        long double f = F(mid);
        bool below = tail ? (f > target) : (f < target);   // mid < root
        if (below) lo = mid; else hi = mid;
    }
    long double w = 0.5L * (lo + hi);
    const long double two_over_sqrt_pi = 1.1283791670955125738961589031215452L;
    for (int it = 0; it < 4; ++it) {
        long double d = two_over_sqrt_pi * expl(-w * w);
        long double f = F(w) - target;
        long double step = tail ? (-f / d) : (f / d);   // d/dw erfc = -d
        long double w2 = w - step;
        if (!(w2 > lo - 1e-18L && w2 < hi + 1e-18L)) break;
        w = w2;
    }
    const long double sqrt2 = 1.4142135623730950488016887242096981L;
    return (double)(sqrt2 * w);
}

// Eq. 3, clamped to [0,1].  Evaluation order (W8):
//   zz = z*z; c = p + zz/(2n); r = z*sqrt(p*(1-p)/n + zz/((4n)*n)); den = 1 + zz/n
void wilson_interval(double p, double n, double z, double* lo, double* hi) {
    double zz = z * z;
    double c = p + zz / (2.0 * n);
    double r = z * std::sqrt(p * (1.0 - p) / n + zz / ((4.0 * n) * n));
    double den = 1.0 + zz / n;
    double L = (c - r) / den;
    double U = (c + r) / den;
    *lo = L > 0.0 ? L : 0.0;
    *hi = U < 1.0 ? U : 1.0;
}

// Eq. 4, ceiling, N >= 1 (W3).  A = p(1-p), d = p - 0.5, e2 = eps^2:
//   N = ceil( zz * ((A - 2 e2) + sqrt(A*A + (4 e2)*(d*d))) / (2 e2) )
int64_t wilson_sample_size(double p, double eps, double z) {
    double zz = z * z;
    double A = p * (1.0 - p);
    double d = p - 0.5;
    double e2 = eps * eps;
    double val = zz * (A - 2.0 * e2 + std::sqrt(A * A + 4.0 * e2 * (d * d))) / (2.0 * e2);
    double cv = std::ceil(val);
    int64_t N = (int64_t)cv;
    return N < 1 ? 1 : N;
}

// Fig. 2: round the estimate by eps toward 0.5.
double round_estimate(double p_hat, double eps) { return p_hat <= 0.5 ? p_hat + eps : p_hat - eps; }

}  // namespace smc

using namespace smc;

extern "C" {

double smc_normal_quantile(double confidence) { return normal_quantile(confidence); }

int smc_wilson_interval(int64_t n_true, int64_t n, double confidence, double* lower, double* upper) {
    if (n < 1 || n_true < 0 || n_true > n || !lower || !upper || !(confidence > 0 && confidence < 1)) {
        set_error("smc_wilson_interval: need n >= 1, 0 <= n_true <= n, confidence in (0,1)");
        return SMC_E_ARG;
    }
    double z = normal_quantile(confidence);
    wilson_interval((double)n_true / (double)n, (double)n, z, lower, upper);
    return SMC_OK;
}

int64_t smc_wilson_sample_size(double p, double half_width, double confidence) {
    if (!(p >= 0 && p <= 1) || !(half_width > 0 && half_width < 0.5) || !(confidence > 0 && confidence < 1)) {
        set_error("smc_wilson_sample_size: need p in [0,1], half_width in (0,0.5), confidence in (0,1)");
        return -1;
    }
    return wilson_sample_size(p, half_width, normal_quantile(confidence));
}

int smc_shard_range(uint64_t base, uint64_t n, int32_t rank, int32_t world, uint64_t* lo, uint64_t* hi) {
    if (world < 1 || rank < 0 || rank >= world || !lo || !hi) {
        set_error("smc_shard_range: need 0 <= rank < world");
        return SMC_E_ARG;
    }
    // floor(r n / world) without 128-bit overflow for n < 2^63
    auto part = [&](uint64_t r) -> uint64_t {
        unsigned __int128 v = (unsigned __int128)r * n / (unsigned)world;
        return (uint64_t)v;
    };
    *lo = base + part((uint64_t)rank);
    *hi = base + part((uint64_t)rank + 1);
    return SMC_OK;
}

}  // extern "C"
