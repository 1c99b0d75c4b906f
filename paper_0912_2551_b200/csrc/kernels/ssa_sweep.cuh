// ssa_sweep.cuh -- variant 4: persistent THREAD-OWNED SSA + monitor kernel for
// networks too large for registers (C4: 50 x 200), with a full propensity SWEEP
// per event instead of stored propensities.
//
// * Each lane owns one trajectory (refill, burst and verdict logic as variant 1).
//   Its counts live in shared memory as a column: x[s] at s*SMC_BLOCK + tid, so
//   every access -- uniform s in the sweep, per-lane s in the selection and the
//   update -- hits bank (tid mod 32): conflict-free whatever the species.
//   x[N] = 1 is a constant column (operand of h = x * 1 in the law table).
//   SMC_SW_XD: the counts are stored as binary64 (exact integers < 2^31; the
//   count-overflow test of R17 is x > 2^31 - 1), so the laws are fp64 products
//   with no int -> fp64 conversion; otherwise int32 columns.
// * Model tables (law table, change lists, Hill parameters) are staged once per CTA
//   by a TMA bulk copy (cp.async.bulk + mbarrier), as in the tile variant.
// * Per event, pass 1 (generated straight-line code, smc_sweep): every law a_k(x)
//   in index order, summed per group of SMC_SW_S consecutive reactions, and the
//   group prefix P_g = P_{g-1} + (group g sum) kept in registers; a0 = P_{G-1}
//   (reading R12: a fixed order).  All lanes of a warp run the same law at the
//   same time: rates come from the constant bank, species loads are uniform
//   offsets.  The propensities are not stored: a dependency-driven update would
//   touch, over the 32 lanes' different reactions, nearly every law anyway (the
//   argument of variant 1), and not storing a[M] frees the 1.6 KB per trajectory
//   that would cap residency.
// * Selection (Eq. 2b), pass 2: the group g = #{P_i <= u2 a0} by integer compares
//   of the non-negative doubles' bit patterns (P_{g-1} by a select tree), then the
//   member inside g by a running sum from P_{g-1} over the group's laws re-evaluated
//   from the sweep-format law table (pre-scaled column offsets; all reads of a chunk
//   of SMC_SW_C laws independent; one dependent add chain).
// * x += v_j from the change table; the monitor reads its atoms from the column.
// * One CTA of up to 384 threads per SM (12 warps at ~168 registers fill the
//   register file); a slice smaller than the resident capacity launches smaller CTAs
//   (the column stride stays SMC_BLOCK).
//
// Generated hooks (codegen.cpp): SMC_N, SMC_M, SMC_BLOCK, SMC_MINB, SMC_SW_S, SMC_SW_G,
//   SMC_SW_C, SMC_SW_XD, SMC_SW_ANYGEN, SMC_OFF_X0/LAW/SWLAW/HREP/HK/HN/CHG,
//   SMC_TAB_BYTES, SMC_ANY_HILL, SMC_ANY_GENERAL, SMC_ANY_EXPLICIT (+ smc_explicit4),
//   smc_sweep(X, P), SMC_TMAX, SmcMon.

#ifndef SMC_BURST
#define SMC_BURST 8
#endif
#ifndef SMC_SW_DSCAN
#define SMC_SW_DSCAN 1     // 1: prefix scan by DSETP; 2: also the in-group count
#endif

struct SmcSwTabs {
    const int* x0;
    const SmcLaw* law;               // tile-format law table (general laws)
    const SmcLaw* swlaw;             // sweep-format law table, G*S entries
    const int* hill_rep;
    const double* hill_k;
    const int* hill_n;
    const unsigned short* chg;       // [M][4]: species << 4 | (delta + 8), 0xFFFF = none
};

// a_k(x) from the law table (readings R8/R9/R20) -- the same IEEE
// operations as the generated pass-1 law, so both passes see identical values:
// order <= 2: h = fl(x0 * x1) (x[N] = 1 for the missing operand), kind 2 as
// fl(x (x-1)) with the 1/2 folded into c; order 3-4: exact int64 binomials.
// General path (order 3-4, explicit rates, Hill): the tile-format law table.
__device__ __noinline__ double smc_law_gen(int k, const SmcXCol& X, const SmcSwTabs& T) {
    const SmcLaw L = T.law[k];
    const int kind = (int)((L.u0 >> 16) & 7u);
#if SMC_ANY_EXPLICIT
    if (kind == 5) return smc_explicit4(k, X);
#endif
#if SMC_SW_XD
    const double v0 = X[(int)(L.u0 & 0xFFFFu)];
    const double v1 = X[(int)(L.u1 & 0xFFFFu)];
#else
    const int v0 = X[(int)(L.u0 & 0xFFFFu)];
    const int v1 = X[(int)(L.u1 & 0xFFFFu)];
#endif
    double h;
    if (kind == 4) {
        const smc_i64 y0 = (smc_i64)v0, y1 = (smc_i64)v1;
        const smc_i64 h0 = ((L.u0 >> 20) & 3u) == 1u ? y0 : (y0 * (y0 - 1)) / 2;
        const smc_i64 h1 = ((L.u1 >> 16) & 3u) == 1u ? y1 : (y1 * (y1 - 1)) / 2;
        h = (double)(h0 * h1);
    } else {
#if SMC_SW_XD
        const double xb = (kind == 2) ? __dadd_rn(v0, -1.0) : v1;
        h = __dmul_rn(v0, xb);
#else
        const int xb = (kind == 2) ? max(v0 - 1, 0) : v1;
        h = (double)((smc_i64)v0 * (smc_i64)xb);
#endif
    }
    double a = __dmul_rn(L.c, h);
#if SMC_ANY_HILL
    if ((int)L.u0 < 0) {
        const double q = __ddiv_rn((double)X[T.hill_rep[k]], T.hill_k[k]);
        double qn = q;
        for (int i = 1; i < T.hill_n[k]; ++i) qn = __dmul_rn(qn, q);
        a = __ddiv_rn(a, __dadd_rn(1.0, qn));
    }
#endif
    return a;
}

// Sweep-format entry: u0 = byte offset of the column of s0 (a multiple of 4) | flags (bit 0 homodimer,
// bit 1 general law), u1 = byte offset of the column of s1, c = rate (halved for a
// homodimer); entries past M are zero-rate padding (a = 0).
__device__ __forceinline__ double smc_law_sw(int k, const SmcXCol& X, const SmcSwTabs& T) {
    const SmcLaw L = T.swlaw[k];
#if SMC_SW_ANYGEN
    if (L.u0 & 2u) return smc_law_gen(k, X, T);
#endif
    const char* xb = (const char*)X.p;
    const smc_xt v0 = *(const smc_xt*)(xb + (L.u0 & ~3u));
    const smc_xt v1 = *(const smc_xt*)(xb + L.u1);
#if SMC_SW_XD
    // x0 (x1 - d), d = 1 for a homodimer: one rounding of the exact x0 x1 - d x0
    const double h = __fma_rn(v0, v1, (L.u0 & 1u) ? -v0 : 0.0);
#else
    const double h = (double)((smc_i64)v0 * (smc_i64)(v1 - (int)(L.u0 & 1u)));
#endif
    return __dmul_rn(L.c, h);
}

// acc + a_k for pass 2, in the arithmetic of pass 1's accumulation: with SMC_SW_FMAACC
// (reading R25) fma(c, h, acc) -- one rounding -- for the sweep-format laws, acc + a_k for
// the general ones
#ifndef SMC_SW_FMAACC
#define SMC_SW_FMAACC 0
#endif
__device__ __forceinline__ double smc_acc_sw(int k, double acc, const SmcXCol& X, const SmcSwTabs& T) {
#if SMC_SW_FMAACC && SMC_SW_XD
    const SmcLaw L = T.swlaw[k];
#if SMC_SW_ANYGEN
    if (L.u0 & 2u) return __dadd_rn(acc, smc_law_gen(k, X, T));
#endif
    const char* xb = (const char*)X.p;
    const double v0 = *(const double*)(xb + (L.u0 & ~3u));
    const double v1 = *(const double*)(xb + L.u1);
    return __fma_rn(L.c, __fma_rn(v0, v1, (L.u0 & 1u) ? -v0 : 0.0), acc);
#else
    return __dadd_rn(acc, smc_law_sw(k, X, T));
#endif
}

// non-negative doubles (and -0) order like their bit patterns as signed int64
__device__ __forceinline__ smc_i64 smc_ord(double v) { return __double_as_longlong(v); }

// member of group gi: first j with base + a_{j0} + ... + a_j > target (left to right).
// Chunks of SMC_SW_C laws: the reads of a chunk are independent (one load latency per
// chunk), the running sum is the only chain; inside a chunk the member is the count of
// prefixes <= target (the prefixes are non-decreasing).  Rounding (no prefix exceeds the
// target although P_gi does): the last a_j > 0 of the group (R11), re-evaluated.
#if SMC_SW_S % SMC_SW_C != 0
#error "SMC_SW_C must divide SMC_SW_S"
#endif
__device__ __forceinline__ int smc_pick(int gi, double base, double target, const SmcXCol& X, const SmcSwTabs& T) {
    const int j0 = gi * SMC_SW_S;
    const smc_i64 tb = smc_ord(target);
    double acc = base;
#pragma unroll 1
    for (int c0 = j0; c0 < j0 + SMC_SW_S; c0 += SMC_SW_C) {
        int cnt = 0;
#pragma unroll
        for (int m = 0; m < SMC_SW_C; ++m) {
            acc = smc_acc_sw(c0 + m, acc, X, T);      // the law reads do not depend on acc
#if SMC_SW_DSCAN >= 2
            cnt += (acc <= target) ? 1 : 0;
#else
            cnt += (smc_ord(acc) <= tb) ? 1 : 0;
#endif
        }
        if (cnt < SMC_SW_C) return c0 + cnt;
    }
#pragma unroll 1
    for (int j = j0 + SMC_SW_S - 1; j > j0; --j)
        if (smc_law_sw(j, X, T) > 0.0) return j;
    return j0;
}

// P at the last index i in [LO, HI) with le[i] (le is a prefix of trues: the prefixes are
// non-decreasing), else fb -- a select tree of depth log2(G) instead of a G-long chain
template <int LO, int HI> struct SmcLastLe {
    static __device__ __forceinline__ double pick(const double (&P)[SMC_SW_G], const bool (&le)[SMC_SW_G], double fb) {
        if constexpr (HI <= LO) {
            return fb;
        } else if constexpr (HI - LO == 1) {
            return le[LO] ? P[LO] : fb;
        } else {
            // le[MID]: the answer is P[MID] or later; else it lies in [LO, MID) (or is fb)
            constexpr int MID = (LO + HI) / 2;
            const double right = SmcLastLe<MID + 1, HI>::pick(P, le, P[MID]);
            const double left = SmcLastLe<LO, MID>::pick(P, le, fb);
            return le[MID] ? right : left;
        }
    }
};

// rounding with u2 a0 >= every prefix: the last reaction with a_j > 0 (reading R11)
__device__ __noinline__ int smc_last_positive_sw(const SmcXCol& X, const SmcSwTabs& T) {
    for (int j = SMC_M - 1; j > 0; --j)
        if (smc_law_sw(j, X, T) > 0.0) return j;
    return 0;
}

extern "C" __global__ void __launch_bounds__(SMC_BLOCK, SMC_MINB) smc_ssa_sweep(SmcParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ __align__(8) unsigned long long bar;
    const smc_u32 lane = threadIdx.x & 31u;

    // ---- stage the model tables: one TMA bulk copy per 32 KB chunk
    if (threadIdx.x == 0) smc_mbar_init(&bar, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        smc_mbar_expect_tx(&bar, (unsigned)SMC_TAB_BYTES);
        for (unsigned off = 0; off < (unsigned)SMC_TAB_BYTES; off += 32768u) {
            const unsigned n = ((unsigned)SMC_TAB_BYTES - off) < 32768u ? ((unsigned)SMC_TAB_BYTES - off) : 32768u;
            smc_bulk_g2s(smem + off, (const unsigned char*)P.tables + off, n, &bar);
        }
    }
    smc_mbar_wait(&bar, 0);
    SmcSwTabs T;
    T.x0 = (const int*)(smem + SMC_OFF_X0);
    T.law = (const SmcLaw*)(smem + SMC_OFF_LAW);
    T.swlaw = (const SmcLaw*)(smem + SMC_OFF_SWLAW);
    T.hill_rep = (const int*)(smem + SMC_OFF_HREP);
    T.hill_k = (const double*)(smem + SMC_OFF_HK);
    T.hill_n = (const int*)(smem + SMC_OFF_HN);
    T.chg = (const unsigned short*)(smem + SMC_OFF_CHG);
    smc_xt* const xcol = (smc_xt*)(smem + SMC_TAB_BYTES) + threadIdx.x;
    const SmcXCol X{xcol};
    xcol[SMC_N * SMC_BLOCK] = (smc_xt)1;                // x[N] = 1

    const smc_u32 cap = (smc_u32)(P.event_cap < 0xFFFFFFFFull ? P.event_cap : 0xFFFFFFFFull);
    double t = 0.0, tp = 0.0;
    double e_cur = 0.0, u_cur = 0.0;      // draw of the current step k
    smc_u32 k = 0;
    smc_u64 rel = 0, traj = 0;
    SmcMon mon;                            // a template monitor, or the window monitor (R27)
    mon.bind(P, (smc_u64)blockIdx.x * blockDim.x + threadIdx.x, 1u << lane, (int)lane);
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
                    for (int s = 0; s < SMC_N; ++s) xcol[s * SMC_BLOCK] = (smc_xt)T.x0[s];
                    t = 0.0;
                    tp = 0.0;
                    k = 0;
                    mon.init();
                    mon.enter(0u, 0.0, 0.0, X);          // sigma_buff = {(s0, t0)}
                    const int v = mon.verdict();
                    if (v >= 0) {
                        if (v == 1) ++c_true; else ++c_false;
                        if (P.verdicts) { P.verdicts[rel] = (unsigned char)v; P.events_out[rel] = 0; }
                    } else {
                        busy = true;
                        smc_draw(P.seed, traj, 0ull, e_cur, u_cur);
                    }
                }
            }
        }
        if (!__any_sync(SMC_FULL, busy)) break;

#pragma unroll 1
        for (int burst = 0; burst < SMC_BURST; ++burst) {
            if (!busy) continue;
            double e_nx, u_nx;                            // step k+1's draw, off the critical path
            smc_draw(P.seed, traj, (smc_u64)k + 1ull, e_nx, u_nx);
            double Pg[SMC_SW_G];
            smc_sweep(X, Pg);                             // pass 1: a0 and the group prefixes
            const double A = Pg[SMC_SW_G - 1];
            const double tau = smc_tau(e_cur, A);
            const double tn = __dadd_rn(t, tau);
            int v = -1;
            if (!(A >= SMC_A_MIN) || A > SMC_A_MAX) {      // A == 0: absorbed; else error (R19)
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
                    // ---- selection (Eq. 2b): group by the prefixes, member by pass 2
                    const double target = __dmul_rn(u_cur, A);
                    const smc_i64 tb = smc_ord(target);
                    int gi = 0;
                    bool le[SMC_SW_G];
#pragma unroll
                    for (int i = 0; i < SMC_SW_G; ++i) {
#if SMC_SW_DSCAN
                        le[i] = Pg[i] <= target;                // one DSETP on the FP64 pipe
#else
                        le[i] = smc_ord(Pg[i]) <= tb;           // two ISETP on the integer pipe
#endif
                        gi += le[i] ? 1 : 0;
                    }
                    const double base = SmcLastLe<0, SMC_SW_G>::pick(Pg, le, 0.0);   // P_{gi-1} (0 if gi = 0)
                    const int j = (gi < SMC_SW_G) ? smc_pick(gi, base, target, X, T) : smc_last_positive_sw(X, T);
                    // ---- x += v_j (wrapping add; a negative result is a count overflow, R17)
                    const uint2 ce = *(const uint2*)(T.chg + 4 * j);
                    bool ovf = false;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const unsigned e = ((q < 2 ? ce.x : ce.y) >> (16 * (q & 1))) & 0xFFFFu;
                        if (e != 0xFFFFu) {
                            smc_xt* xp = xcol + (int)(e >> 4) * SMC_BLOCK;
#if SMC_SW_XD
                            const double nv = __dadd_rn(*xp, (double)((int)(e & 15u) - 8));   // exact
                            // nv > 2^31 - 1 for an integer nv >= 0 <=> its high word >= that of 2^31
                            ovf |= __double2hiint(nv) >= 0x41E00000;
#else
                            const int nv = (int)((unsigned)*xp + (unsigned)((int)(e & 15u) - 8));
                            ovf |= nv < 0;
#endif
                            *xp = nv;
                        }
                    }
                    if (ovf) {
                        v = 2;
                    } else {
                        tp = t;
                        t = tn;
                        ++k;
                        e_cur = e_nx;
                        u_cur = u_nx;
                        mon.enter(k, t, tp, X);
                        v = mon.verdict();
                        if (v < 0 && k >= cap) v = mon.at_cap((long long)k);
                    }
                }
            }
            if (v >= 0) {
                const smc_u32 ke = (v == 0 || v == 1) ? (smc_u32)mon.events((long long)k) : k;   // window monitor:
                if (v == 1) ++c_true;                                                    // the first decision
                else if (v == 0) ++c_false;                                              // index
                else ++c_err;
                c_ev += ke;
                if (P.verdicts) { P.verdicts[rel] = (unsigned char)v; P.events_out[rel] = (int)ke; }
                busy = false;
            }
        }
    }
    smc_flush_counts(c_true, c_false, c_ev, c_err, P.counters);
}
