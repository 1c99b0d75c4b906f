// ssa_literal.cuh -- variant 3: thread-owned SSA for formulas outside the streaming
// templates of reading R16 (arbitrary nesting, non-zero inner lower bounds; SURVEY §8(f)
// NEXT-2), checked on the fly by the window monitor (ssa_window.cuh, readings R23/R24/R27).
//
// Each thread owns one trajectory at a time (x[N], a[M] in registers, exactly as variant
// 1) and one slot of window-monitor rings.  The monitor sees every entry (enter), every
// sojourn (advance), the absorption and the event cap; the replica stops as soon as the
// root's value and its first decision index are known, and at the horizon H
// (the formula's reach, or t_max) the trace ends: unknown -> false (R4).
//
// Generated hooks (codegen.cpp): as variant 1, plus smc_lit_mask, the SmcWN node table
// and SMC_LIT_H.

extern "C" __global__ void __launch_bounds__(SMC_BLOCK, SMC_MINB) smc_ssa_literal(SmcParams P) {
    const smc_u64 gtid = (smc_u64)blockIdx.x * blockDim.x + threadIdx.x;
    const double* __restrict__ H = (const double*)P.tables;
    const unsigned me = 1u << (threadIdx.x & 31u);
    SmcMon mon;
    mon.bind(P, gtid, me, (int)(threadIdx.x & 31u));
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
        double t = 0.0, tp = 0.0;
        smc_u32 k = 0;
        mon.init();
        mon.enter(0u, 0.0, 0.0, x);                       // sigma_buff = {(s0, t0)}
        int v = -1;
        for (;;) {
            double A = a[0];
#pragma unroll
            for (int m = 1; m < SMC_M; ++m) A = __dadd_rn(A, a[m]);
            if (!(A >= SMC_A_MIN) || A > SMC_A_MAX) {
                if (A == 0.0) { mon.absorb(); v = mon.verdict(); }   // no further entries (reading R7)
                else v = 2;                                          // bad propensity (R19)
                break;
            }
            double e, u2;
            smc_draw(P.seed, traj, k, e, u2);
            const double tau = smc_tau(e, A);
            const double tn = __dadd_rn(t, tau);
            mon.advance(k, tn, tau);                      // prefix k; the horizon ends the trace
            v = mon.verdict();
            if (v >= 0) break;
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
            if (!smc_apply(j, x)) { v = 2; break; }       // count overflow (R17)
            smc_update(j, a, x, H);
            tp = t;
            t = tn;
            ++k;
            mon.enter(k, t, tp, x);
            if ((smc_u64)k >= P.event_cap) {              // the prefix up to entry k - 1 decides, else error
                v = mon.at_cap((long long)k);
                break;
            }
        }
        const long long ke = (v == 0 || v == 1) ? mon.events((long long)k) : (long long)k;
        if (v == 1) ++c_true;
        else if (v == 0) ++c_false;
        else ++c_err;
        c_ev += (smc_i64)ke;
        if (P.verdicts) { P.verdicts[rel] = (unsigned char)v; P.events_out[rel] = (int)ke; }
    }
    smc_flush_counts(c_true, c_false, c_ev, c_err, P.counters);
}
