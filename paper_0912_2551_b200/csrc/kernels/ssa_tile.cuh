// ssa_tile.cuh -- variant 2: persistent WARP-OWNED (tile) SSA + monitor kernel
// for networks whose state does not fit in registers (C4: 50 x 200, C5:
// 200 x 1000).
//
// * Model tables (reactant/law table, change lists, dependency CSR) are staged
//   ONCE per CTA from HBM into shared memory by a TMA bulk copy
//   (cp.async.bulk ... mbarrier::complete_tx), then read from smem only.
// * One warp owns one trajectory: species counts x[N] and propensities a[M]
//   live in the warp's shared-memory slice; lane l owns the contiguous
//   reaction group [l*GS, (l+1)*GS) and keeps its group sum S_l in a register.
//   a is stored XOR-swizzled, a(l, m) at m*32 + (l ^ m), so both the per-lane
//   group walk (fixed m, all l) and the level-2 scan (fixed l, all m) are
//   bank-conflict free.
// * Per event: a0 = inclusive warp scan of S (fixed order), reaction selection
//   in two levels (group by ballot on the scan, member by a scan inside the
//   group), x += v_j by <= 4 lanes, the dependency list dep(j) evaluated one
//   reaction per lane, and only the touched groups re-summed (fixed order,
//   never incremental deltas: reading R12).
// * Philox + log for 32 future steps are computed by the 32 lanes at once and
//   handed out by shuffle (state-independent, so batching them is exact).
//
// Generated hooks (codegen.cpp): SMC_N, SMC_M, SMC_GS, SMC_GS2, SMC_NPAD,
//   SMC_OFF_*, SMC_TAB_BYTES, SMC_WARP_BYTES, SMC_ANY_HILL, SMC_TMAX, SmcMon.

__device__ __forceinline__ void smc_mbar_init(unsigned long long* bar, unsigned count) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void smc_mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void smc_bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(d), "l"(src), "r"(bytes), "r"(b) : "memory");
}
__device__ __forceinline__ void smc_mbar_wait(unsigned long long* bar, unsigned parity) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    unsigned done = 0;
    while (!done) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done) : "r"(a), "r"(parity) : "memory");
    }
}

struct SmcTabs {
    const int* x0;
    const int2* sp;       // .x = s0 | st0 << 16 | hill << 31, .y = s1 | st1 << 16 (0xFFFF = none)
    const double* c;
    const int* hill_rep;
    const double* hill_k;
    const int* hill_n;
    const unsigned short* chg;       // [M][4]: species << 4 | (delta + 8), 0xFFFF = none
    const unsigned* dep_off;         // [M+1]
    const unsigned short* dep_idx;   // [nnz]
};

// a_j(x) from the shared-memory law table (readings R8/R9);
// h_j is exact in int64, then one conversion and one multiply.
__device__ __forceinline__ double smc_law_tab(int j, const int* xs, const SmcTabs& T) {
    const int2 sp = T.sp[j];
    smc_i64 h = 1;
    const int s0 = sp.x & 0xFFFF, s1 = sp.y & 0xFFFF;
    if (s0 != 0xFFFF) {
        const smc_i64 v = xs[s0];
        h = (((sp.x >> 16) & 3) == 1) ? v : (v * (v - 1)) / 2;
    }
    if (s1 != 0xFFFF) {
        const smc_i64 v = xs[s1];
        h = h * ((((sp.y >> 16) & 3) == 1) ? v : (v * (v - 1)) / 2);
    }
    double a = __dmul_rn(T.c[j], (double)h);
#if SMC_ANY_HILL
    if (sp.x < 0) {
        const double q = __ddiv_rn((double)xs[T.hill_rep[j]], T.hill_k[j]);
        double qn = q;
        for (int i = 1; i < T.hill_n[j]; ++i) qn = __dmul_rn(qn, q);
        a = __ddiv_rn(a, __dadd_rn(1.0, qn));
    }
#endif
    return a;
}

__device__ __forceinline__ int smc_aidx(int j) {     // swizzled slot of reaction j
    const int l = j / SMC_GS, m = j - l * SMC_GS;
    return m * 32 + (l ^ m);
}

extern "C" __global__ void __launch_bounds__(512, 1) smc_ssa_tile(SmcParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ __align__(8) unsigned long long bar;
    const smc_u32 lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;

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

    SmcTabs T;
    T.x0 = (const int*)(smem + SMC_OFF_X0);
    T.sp = (const int2*)(smem + SMC_OFF_SP);
    T.c = (const double*)(smem + SMC_OFF_C);
    T.hill_rep = (const int*)(smem + SMC_OFF_HREP);
    T.hill_k = (const double*)(smem + SMC_OFF_HK);
    T.hill_n = (const int*)(smem + SMC_OFF_HN);
    T.chg = (const unsigned short*)(smem + SMC_OFF_CHG);
    T.dep_off = (const unsigned*)(smem + SMC_OFF_DOFF);
    T.dep_idx = (const unsigned short*)(smem + SMC_OFF_DIDX);
    double* at = (double*)(smem + SMC_TAB_BYTES + (size_t)warp * SMC_WARP_BYTES);
    int* xs = (int*)(at + SMC_GS * 32);

    smc_i64 c_true = 0, c_false = 0, c_ev = 0, c_err = 0;   // lane 0 of each warp
    for (;;) {
        smc_u64 rel = 0;
        if (lane == 0) rel = atomicAdd(P.cursor, 1ull);
        rel = __shfl_sync(SMC_FULL, rel, 0);
        if (rel >= P.count) break;
        const smc_u64 traj = P.first + rel;

        // ---- init: x = x0, all a_j, group sums, monitor at sigma[0]
        for (int s = lane; s < SMC_N; s += 32) xs[s] = T.x0[s];
        __syncwarp();
        double S = 0.0;
#pragma unroll 4
        for (int m = 0; m < SMC_GS; ++m) {
            const int j = (int)lane * SMC_GS + m;
            const double val = (j < SMC_M) ? smc_law_tab(j, xs, T) : 0.0;
            at[m * 32 + ((int)lane ^ m)] = val;
            S = (m == 0) ? val : __dadd_rn(S, val);
        }
        __syncwarp();
        SmcMon mon;
        mon.init();
        double t = 0.0, tp = 0.0;
        smc_u32 k = 0, k0 = 0, kend = 0;
        double Eb = 0.0, Ub = 0.0;
        mon.enter(0u, 0.0, 0.0, xs);
        int v = mon.verdict();
        while (v < 0) {
            // a0 = inclusive scan of the group sums (fixed association per lane)
            double Pp = S;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double y = __shfl_up_sync(SMC_FULL, Pp, o);
                if ((int)lane >= o) Pp = __dadd_rn(y, Pp);
            }
            const double A = __shfl_sync(SMC_FULL, Pp, 31);
            if (!(A >= 0.0) || A > 1.7976931348623157e308) { v = 2; break; }
            if (A == 0.0) { mon.absorb(); v = mon.verdict(); break; }
            if (k >= kend) {                       // 32 future draws, one per lane
                k0 = k;
                kend = k + 32u;
                smc_draw(P.seed, traj, (smc_u64)(k0 + lane), Eb, Ub);
            }
            const double E = __shfl_sync(SMC_FULL, Eb, (int)(k - k0));
            const double U = __shfl_sync(SMC_FULL, Ub, (int)(k - k0));
            const double tn = __dadd_rn(t, __ddiv_rn(E, A));
            mon.advance(k, tn);
            v = mon.verdict();
            if (v >= 0) break;
            if (SMC_TMAX > 0.0 && tn > SMC_TMAX) { mon.timeout(); v = mon.verdict(); break; }

            // ---- two-level selection: group g, then member m  (Eq. 2b)
            const double target = __dmul_rn(U, A);
            const smc_u32 bg = __ballot_sync(SMC_FULL, Pp > target);
            int j;
            if (bg) {
                const int g = __ffs(bg) - 1;
                double base = __shfl_sync(SMC_FULL, Pp, (g + 31) & 31);
                if (g == 0) base = 0.0;
                const double val = ((int)lane < SMC_GS) ? at[lane * 32 + (g ^ (int)lane)] : 0.0;
                double q = (lane == 0) ? __dadd_rn(base, val) : val;
#pragma unroll
                for (int o = 1; o < SMC_GS2; o <<= 1) {
                    const double y = __shfl_up_sync(SMC_FULL, q, o);
                    if ((int)lane >= o) q = __dadd_rn(y, q);
                }
                const smc_u32 bm = __ballot_sync(SMC_FULL, (int)lane < SMC_GS && q > target);
                if (bm) {
                    j = g * SMC_GS + __ffs(bm) - 1;
                } else {                               // ulp tie: last positive member
                    const smc_u32 bp = __ballot_sync(SMC_FULL, (int)lane < SMC_GS && val > 0.0);
                    j = g * SMC_GS + 31 - __clz(bp);
                }
            } else {                                   // rounding: last a_j > 0 (reading R11)
                const smc_u32 bs = __ballot_sync(SMC_FULL, S > 0.0);
                const int g = 31 - __clz(bs);
                const double val = ((int)lane < SMC_GS) ? at[lane * 32 + (g ^ (int)lane)] : 0.0;
                const smc_u32 bp = __ballot_sync(SMC_FULL, (int)lane < SMC_GS && val > 0.0);
                j = g * SMC_GS + 31 - __clz(bp);
            }

            // ---- x += v_j  (<= 4 distinct species, one lane each)
            bool ovf = false;
            if (lane < 4u) {
                const unsigned e = T.chg[j * 4 + (int)lane];
                if (e != 0xFFFFu) {
                    const int s = (int)(e >> 4);
                    const smc_i64 nv = (smc_i64)xs[s] + (smc_i64)((int)(e & 15u) - 8);
                    if (nv > 2147483647ll) ovf = true;
                    else xs[s] = (int)nv;
                }
            }
            if (__any_sync(SMC_FULL, ovf)) { v = 2; break; }
            __syncwarp();

            // ---- a_k = law_k(x) for k in dep(j), one reaction per lane
            const unsigned d0 = T.dep_off[j], d1 = T.dep_off[j + 1];
            smc_u32 touched = 0;
            for (unsigned b = d0; b < d1; b += 32u) {
                if (b + lane < d1) {
                    const int kk = T.dep_idx[b + lane];
                    const double an = smc_law_tab(kk, xs, T);
                    at[smc_aidx(kk)] = an;
                    touched |= 1u << (kk / SMC_GS);
                }
            }
            touched = __reduce_or_sync(SMC_FULL, touched);
            __syncwarp();
            // ---- re-sum only the touched groups, left to right
            if ((touched >> lane) & 1u) {
                double s2 = at[lane];
#pragma unroll 8
                for (int m = 1; m < SMC_GS; ++m) s2 = __dadd_rn(s2, at[m * 32 + ((int)lane ^ m)]);
                S = s2;
            }
            tp = t;
            t = tn;
            ++k;
            mon.enter(k, t, tp, xs);
            v = mon.verdict();
            if (v < 0 && (smc_u64)k >= P.event_cap) v = 2;
        }
        if (lane == 0) {
            if (v == 1) ++c_true;
            else if (v == 0) ++c_false;
            else ++c_err;
            c_ev += k;
            if (P.verdicts) { P.verdicts[rel] = (unsigned char)v; P.events_out[rel] = (int)k; }
        }
        __syncwarp();
    }
    smc_flush_counts(c_true, c_false, c_ev, c_err, P.counters);
}
