// ssa_thread.cuh -- variant 1: persistent THREAD-OWNED SSA + monitor kernel.
//
// Each lane owns one trajectory; species counts x[N] and propensities a[M]
// live in registers (every index below is a compile-time constant after the
// generated model code is inlined).  Lanes whose trajectory is decided are
// refilled by warp ballot + one warp-aggregated 64-bit atomic on the work
// cursor (compaction of the finished lanes onto new indices), so a warp keeps
// all of its lanes busy while paths of different lengths end at different
// times (P:291-294 on-the-fly halting makes them diverge).  The refill runs
// once per SMC_BURST events; a lane that finishes inside a burst idles for the
// rest of it (at most SMC_BURST-1 event slots per trajectory).
//
// The random draw of step k+1 (Philox + log) does not depend on the state, so
// it is issued at the top of step k, in the same basic block as the a0 sum,
// and overlaps the state-dependent chain of step k (SMC_PIPE2: the Philox block
// of step k+2 and the u53 + log of step k+1 as two independent chains).
// After a reaction all M <= 32 laws are recomputed straight-line: the lanes of a
// warp fire different reactions, so a masked dependency update would execute
// (nearly) every law anyway; the values are identical.
//
// Generated hooks (codegen.cpp): SMC_N, SMC_M, SMC_BLOCK, SMC_MINB, SMC_TMAX, SMC_PIPE2,
//   smc_init_x(x), smc_laws_all(a, x, H), smc_apply(j, x) -> ok,
//   smc_update(j, a, x, H), smc_last_positive(a), struct SmcMon.
//   H = P.tables: tabulated Hill propensities (zero-order Hill laws).
//
// One event (SSA template P:173-179 with the monitor of P:291-294):
//   a0 = sum a (fixed order)          step 1
//   a0 == 0 -> absorbed               step 5 "Terminate", reading R7
//   tau = -log(u1)/a0, t' = t + tau   step 3, Eq. 2a
//   monitor.advance(t')               close windows t' passes (may decide)
//   j = min{j : sum_{i<=j} a_i > u2 a0}  step 2, Eq. 2b
//   x += v_j; a_k = law_k(x) (all k); t = t'          step 4
//   monitor.enter(t, x)               (may decide)

#ifndef SMC_PIPE2
#define SMC_PIPE2 0
#endif
#ifndef SMC_UNROLL
#define SMC_UNROLL 1
#endif
#ifndef SMC_BURST
#define SMC_BURST 32      // refill every 32 events: C2 6.35e10 (8) -> 6.48e10, C3 7.87e10 -> 7.91e10
#endif

extern "C" __global__ void __launch_bounds__(SMC_BLOCK, SMC_MINB) smc_ssa_thread(SmcParams P) {
    const smc_u32 lane = threadIdx.x & 31u;
    const double* __restrict__ H = (const double*)P.tables;
    const smc_u32 cap = (smc_u32)(P.event_cap < 0xFFFFFFFFull ? P.event_cap : 0xFFFFFFFFull);
    smc_x1t x[SMC_N];                     // int32, or binary64 (codegen SMC_V1_XD)
    double a[SMC_M];
    double t = 0.0, tp = 0.0;
    double e_cur = 0.0, u_cur = 0.0;      // draw of the current step k
#if SMC_PIPE2
    smc_u32 r_nx[4] = {0u, 0u, 0u, 0u};   // Philox block of step k+1 (its u53 + log run in step k)
#endif
    smc_u32 k = 0;
    smc_u64 rel = 0, traj = 0;
    SmcMon mon;
    bool busy = false, exhausted = false;
    smc_u32 c_true = 0, c_false = 0, c_err = 0;
    smc_i64 c_ev = 0;

    for (;;) {
        // ---- refill: compact the idle lanes onto fresh trajectory indices
        for (;;) {
            const bool want = !busy && !exhausted;
            const smc_u32 wm = __ballot_sync(SMC_FULL, want);
            if (wm == 0u) break;
            const int leader = __ffs(wm) - 1;
            smc_u64 base = 0;
            if ((int)lane == leader) base = atomicAdd(P.cursor, (smc_u64)__popc(wm));
            base = __shfl_sync(SMC_FULL, base, leader);
            if (want) {
                rel = base + (smc_u64)__popc(wm & ((1u << lane) - 1u));
                if (rel >= P.count) {
                    exhausted = true;
                } else {
                    traj = P.first + rel;
                    smc_init_x(x);
                    smc_laws_all(a, x, H);
                    t = 0.0;
                    tp = 0.0;
                    k = 0;
                    mon.init();
                    mon.enter(0u, 0.0, 0.0, x);          // sigma_buff = {(s0, t0)}
                    const int v = mon.verdict();
                    if (v >= 0) {
                        if (v == 1) ++c_true; else ++c_false;
                        if (P.verdicts) { P.verdicts[rel] = (unsigned char)v; P.events_out[rel] = 0; }
                    } else {
                        busy = true;
                        smc_draw(P.seed, traj, 0ull, e_cur, u_cur);
#if SMC_PIPE2
                        smc_draw_words(P.seed, traj, 1ull, r_nx);
#endif
                    }
                }
            }
        }
        if (!__any_sync(SMC_FULL, busy)) break;

#pragma unroll SMC_UNROLL
        for (int burst = 0; burst < SMC_BURST; ++burst) {
            if (!busy) continue;
            // ---- one SSA event of this lane's trajectory
            double e_nx, u_nx;                            // step k+1's draw, off the critical path
#if SMC_PIPE2
            // two independent chains: fp64 half of step k+1's draw, integer half of step k+2's
            smc_draw_from(r_nx, e_nx, u_nx);
            smc_u32 r_nx2[4];
            smc_draw_words(P.seed, traj, (smc_u64)k + 2ull, r_nx2);
#else
            smc_draw(P.seed, traj, (smc_u64)k + 1ull, e_nx, u_nx);
#endif
            double c[SMC_M];
            c[0] = a[0];
#pragma unroll
            for (int m = 1; m < SMC_M; ++m) c[m] = __dadd_rn(c[m - 1], a[m]);
            const double A = c[SMC_M - 1];
            const double tau = smc_tau(e_cur, A);
            const double tn = __dadd_rn(t, tau);
            int v = -1;
            if (!(A >= SMC_A_MIN) || A > SMC_A_MAX) {            // A == 0: absorbed; else error (R19)
                if (A == 0.0) {                           // absorbed (reading R7)
                    mon.absorb();
                    v = mon.verdict();
                } else {
                    v = 2;                                // bad propensity
                }
            } else {
                mon.advance(k, tn, tau);
                v = mon.verdict();
                if (v < 0 && SMC_TMAX > 0.0 && tn > SMC_TMAX) {
                    mon.timeout();
                    v = mon.verdict();
                }
                if (v < 0) {
                    const double target = __dmul_rn(u_cur, A);
                    int j = 0;
#pragma unroll
                    for (int m = 0; m < SMC_M; ++m) j += (c[m] <= target) ? 1 : 0;   // c is non-decreasing
                    if (j == SMC_M) j = smc_last_positive(a);                      // rounding (reading R11)
                    if (!smc_apply(j, x)) {
                        v = 2;                                                     // count overflow
                    } else {
                        smc_update(j, a, x, H);
                        tp = t;
                        t = tn;
                        ++k;
                        e_cur = e_nx;
                        u_cur = u_nx;
#if SMC_PIPE2
                        for (int q = 0; q < 4; ++q) r_nx[q] = r_nx2[q];
#endif
                        mon.enter(k, t, tp, x);
                        v = mon.verdict();
                        if (v < 0 && k >= cap) v = 2;
                    }
                }
            }
            if (v >= 0) {
                if (v == 1) ++c_true;
                else if (v == 0) ++c_false;
                else ++c_err;
                c_ev += k;
                if (P.verdicts) { P.verdicts[rel] = (unsigned char)v; P.events_out[rel] = (int)k; }
                busy = false;
            }
        }
    }
    smc_flush_counts(c_true, c_false, c_ev, c_err, P.counters);
}
