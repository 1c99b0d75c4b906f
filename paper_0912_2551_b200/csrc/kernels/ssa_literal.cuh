// ssa_literal.cuh -- variant 3: thread-owned SSA with a BUFFERED trace and the
// literal |= for formulas outside the streaming templates of reading
// R16 (arbitrary nesting, non-zero inner lower bounds).
//
// Each thread owns one trajectory at a time (x[N], a[M] in registers, exactly as
// variant 1) and records its entries in a private slice of a global buffer:
//   t_k (entry time), tau_k (sojourn; tau_n = the overshoot draw), atom mask_k,
// until the first draw whose time exceeds the formula's horizon H (reach or
// t_max) or absorption.  Then the generated smc_lit_eval() evaluates every
// subformula bottom-up over the buffer, in the order and arithmetic of the
// semantics (elapsed = tau_m + tau_{m+1} + ... left to right), three-valued,
// and the root at sigma[0] gives the verdict (unknown -> false).
// On-the-fly halting (reading R24): after the sojourn of entry k is drawn, at the
// checkpoints k = 64, 128, 256, ..., the three-valued |= of the prefix (entries 0..k,
// the unobserved future unknown) is evaluated; a definite value is final (the
// semantics is monotone in the observed prefix) and the replica stops -- its event
// count is the FIRST decision index k* (P:291-294), found by bisection over the
// buffered prefixes between the last undecided checkpoint and k (smc_lit_first), the
// same count the oracle's literal mode returns.  Otherwise the replica runs to the
// horizon (and k* is searched among its proper prefixes).  A trace longer than the
// buffer capacity ends the replica as an error.
//
// Generated hooks (codegen.cpp): as variant 1, plus SMC_LIT_H, SMC_LIT_NODES,
//   smc_lit_mask(x), smc_lit_eval(t, tau, mask, val, n, absorbed, cap), smc_lit_first.

extern "C" __global__ void __launch_bounds__(SMC_BLOCK, 2) smc_ssa_literal(SmcParams P) {
    const smc_u64 gtid = (smc_u64)blockIdx.x * blockDim.x + threadIdx.x;
    const double* __restrict__ H = (const double*)P.tables;
    const smc_u64 cap = P.lit_cap;                      // entries per thread slice
    double* tb = P.lit_t + gtid * cap;
    double* ub = P.lit_tau + gtid * cap;
    unsigned* mb = P.lit_mask + gtid * cap;
    unsigned char* vb = P.lit_val + gtid * cap * SMC_LIT_NODES;
    int x[SMC_N];
    double a[SMC_M];
    smc_u32 c_true = 0, c_false = 0, c_err = 0;
    smc_i64 c_ev = 0;

    for (;;) {
        const smc_u64 rel = atomicAdd(P.cursor, 1ull);
        if (rel >= P.count) break;
        const smc_u64 traj = P.first + rel;
        smc_init_x(x);
        smc_laws_all(a, x, H);
        double t = 0.0;
        smc_u64 k = 0;
        tb[0] = 0.0;
        mb[0] = smc_lit_mask(x);
        bool absorbed = false, err = false;
        int decided = -1;
        long long und = -1, kev = -1;                      // longest prefix undecided; first decision index
        for (;;) {
            double A = a[0];
#pragma unroll
            for (int m = 1; m < SMC_M; ++m) A = __dadd_rn(A, a[m]);
            if (!(A >= SMC_A_MIN) || A > SMC_A_MAX) {
                if (A == 0.0) absorbed = true;            // no further entries (reading R7)
                else err = true;                          // bad propensity (R19)
                break;
            }
            double e, u2;
            smc_draw(P.seed, traj, k, e, u2);
            const double tau = smc_tau(e, A);
            const double tn = __dadd_rn(t, tau);
            ub[k] = tau;
            if (tn > SMC_LIT_H) break;                    // overshoot: the trace covers the horizon
            if (k >= 64 && (k & (k - 1)) == 0) {          // checkpoint k = 64 * 2^i (R24): halt once the
                int r = smc_lit_eval(tb, ub, mb, vb, (long long)k, false, (long long)cap);
                if (r != 2) {                             // prefix decides |=; its first decision index
                    kev = smc_lit_first(tb, ub, mb, vb, und, (long long)k, (long long)cap, r);
                    decided = r;
                    break;
                }
                und = (long long)k;
            }
            if (k + 1 >= P.event_cap) {                   // the next event would reach the cap: the
                int r = smc_lit_eval(tb, ub, mb, vb, (long long)k, false, (long long)cap);
                if (r != 2) {                             // prefix decides now, else an error
                    kev = smc_lit_first(tb, ub, mb, vb, und, (long long)k, (long long)cap, r);
                    decided = r;
                } else {
                    err = true;
                }
                break;
            }
            if (k + 1 >= cap) { err = true; break; }      // trace buffer full (reading R23)
            // selection (Eq. 2b): first j with sum_{i<=j} a_i > u2 a0 (left to right)
            const double target = __dmul_rn(u2, A);
            double acc = 0.0;
            int j = -1;
#pragma unroll
            for (int m = 0; m < SMC_M; ++m) {
                acc = (m == 0) ? a[0] : __dadd_rn(acc, a[m]);
                if (j < 0 && acc > target) j = m;
            }
            if (j < 0) j = smc_last_positive(a);          // rounding (reading R11)
            if (!smc_apply(j, x)) { err = true; break; }  // count overflow (R17)
            smc_update(j, a, x, H);
            t = tn;
            ++k;
            tb[k] = t;
            mb[k] = smc_lit_mask(x);
        }
        int v = 2;
        if (decided >= 0) {
            v = decided;
        } else if (!err) {
            // end of the trace (horizon overshoot after entry k, or absorption at k): the first
            // definite proper prefix if any, else the whole trace with k events
            if ((long long)k - 1 > und) {
                int r = smc_lit_eval(tb, ub, mb, vb, (long long)k - 1, false, (long long)cap);
                if (r != 2) { kev = smc_lit_first(tb, ub, mb, vb, und, (long long)k - 1, (long long)cap, r); v = r; }
            }
            if (v == 2) v = smc_lit_eval(tb, ub, mb, vb, (long long)k, absorbed, (long long)cap) == 1 ? 1 : 0;
        }
        if (kev >= 0) k = (smc_u64)kev;                    // events: the first decision index
        if (v == 1) ++c_true;
        else if (v == 0) ++c_false;
        else ++c_err;
        c_ev += (smc_i64)k;
        if (P.verdicts) { P.verdicts[rel] = (unsigned char)v; P.events_out[rel] = (int)k; }
    }
    smc_flush_counts(c_true, c_false, c_ev, c_err, P.counters);
}
