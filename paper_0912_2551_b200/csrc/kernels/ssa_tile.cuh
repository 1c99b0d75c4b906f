// ssa_tile.cuh -- variant 2: persistent TILE-OWNED SSA + monitor kernel for
// networks whose state does not fit in registers (C4: 50 x 200, C5: 200 x 1000).
//
// * Model tables (law table, change lists, dependency CSR) are staged ONCE per
//   CTA from HBM into shared memory by a TMA bulk copy (cp.async.bulk ...
//   mbarrier::complete_tx) and then read from smem only.
// * A tile of SMC_TW lanes (4, 8, 16 or 32) owns one trajectory; a warp runs
//   TPW = 32/SMC_TW trajectories in lock step.  x[N] and a[M] live in the tile's
//   shared-memory slice; lane l of a tile owns the contiguous reaction group
//   [l*GS, (l+1)*GS) and keeps its group sum S_l in a register.
//   For CH > 1, a(l, m) is stored at m*TW + (l ^ ((m / CH) % TW)): the group walk
//   of the resum (all lanes at the same m) and the chunked in-group selection
//   (lane c reads m = c*CH + i) are both bank-conflict free; for CH = 1 in rows
//   l*GSP + m (odd GSP: SMC_ROWLAYOUT).  Tile slices are padded so the TPW tiles of
//   a warp cover consecutive bank ranges; x[N] = 1 is a constant count slot.
// * Per event: a0 = inclusive tile scan of the TW group sums (fixed order),
//   two-level selection (group by ballot on the scan, member by chunked scan
//   inside the group), x += v_j by <= 4 lanes, then the dependency work of ALL
//   tiles of the warp is flattened over the 32 lanes (a_k = law_k(x), k in
//   dep(j)), and only the touched groups are re-summed (reading R12: a fixed
//   order, never incremental deltas).
// * Propensity laws are evaluated in fp64 on integer-valued doubles; for
//   reaction order <= 2 this is exactly (double)h with h the int64 combinatorial
//   count (see smc_law_tab), order 3-4 takes the int64 path.
// * Formulas outside the streaming templates use the window monitor (ssa_window.cuh:
//   the literal |= on the fly with memory bounded by the formula's windows, readings
//   R23/R27; the tile's lanes share its rings) through the same SmcMon interface
//   (bind / init / enter / advance / absorb / timeout / verdict / at_cap / events).
// * The Philox + log draws of the next SMC_TW steps of every tile are computed
//   together at the start of each burst of SMC_TW events, one draw per lane
//   (state-independent, so batching them is exact).
//
// Generated hooks (codegen.cpp): SMC_N, SMC_M, SMC_TW, SMC_GS, SMC_CH, SMC_NPAD,
//   SMC_OFF_*, SMC_TAB_BYTES, SMC_TILE_BYTES, SMC_ANY_HILL, SMC_ANY_GENERAL, SMC_DEP16,
//   SMC_ANY_EXPLICIT (+ smc_explicit), SMC_DEPSP, SMC_FATDEP, SMC_ROWLAYOUT, SMC_GSP,
//   SMC_TMAX, SmcMon (+ SMC_LIT_H, the SmcWN node table, smc_lit_mask for the window monitor).

struct SmcTabs {
    const int* x0;
    const SmcLaw* law;
    const int* hill_rep;
    const double* hill_k;
    const int* hill_n;
    const unsigned short* chg;       // [M][4]: species << 4 | (delta + 8), 0xFFFF = none
    const unsigned* dep_off;         // [M+1]
#if SMC_DEP16
    const unsigned short* dep;       // [nnz]: k (slot computed: halves the largest table)
#else
    const unsigned* dep;             // [nnz]: k | slot(k) << 16
#endif
};

// a_k(x) (readings R8/R9).  For order <= 2 the combinatorial count h is
// formed in fp64 from the integer counts: x0, x0*x1 and x0*(x0-1) are single roundings
// of the exact integer products (counts < 2^31, so the int64 product is exact), and
// halving is exact, hence h equals (double)(int64 h) bit for bit; a = c * h, and for a
// homodimer (c/2) * fl(x(x-1)) = c * (fl(x(x-1))/2) as real numbers, so the fold of the
// 1/2 into the table's rate gives the same double (reading R20).
__device__ __forceinline__ double smc_law_tab(int k, const int* xs, const SmcTabs& T) {
    const SmcLaw L = T.law[k];
    const int kind = (int)((L.u0 >> 16) & 7u);
#if SMC_ANY_EXPLICIT
    if (kind == 5) return smc_explicit(k, xs);           // explicit rate (codegen.cpp)
#endif
    const int v0 = xs[L.u0 & 0xFFFFu];
    const int v1 = xs[L.u1 & 0xFFFFu];
    double h;
#if SMC_ANY_GENERAL
    if (kind == 4) {
        const smc_i64 y0 = v0, y1 = v1;
        const smc_i64 h0 = ((L.u0 >> 20) & 3u) == 1u ? y0 : (y0 * (y0 - 1)) / 2;
        const smc_i64 h1 = ((L.u1 >> 16) & 3u) == 1u ? y1 : (y1 * (y1 - 1)) / 2;
        h = (double)(h0 * h1);
    } else
#endif
    {
        // x[s0] * x[s1] with x[N] = 1 (kinds 0, 1, 3); kind 2: x * (x-1), the 1/2 folded into c
        const int xb = (kind == 2) ? max(v0 - 1, 0) : v1;
        h = __dmul_rn((double)v0, (double)xb);
    }
    double a = __dmul_rn(L.c, h);
#if SMC_ANY_HILL
    if ((int)L.u0 < 0) {
        const double q = __ddiv_rn((double)xs[T.hill_rep[k]], T.hill_k[k]);
        double qn = q;
        for (int i = 1; i < T.hill_n[k]; ++i) qn = __dmul_rn(qn, q);
        a = __ddiv_rn(a, __dadd_rn(1.0, qn));
    }
#endif
    return a;
}

// a_k(x) from a fat dependency entry: meta = s0 | s1 << 12 | kind << 24 | (st0 == 2) << 27 |
// (st1 == 2) << 28 | hill << 31, c the (folded) rate -- the same arithmetic as smc_law_tab
__device__ __forceinline__ double smc_law_meta(unsigned meta, double c, int k, const int* xs, const SmcTabs& T) {
    const int kind = (int)((meta >> 24) & 7u);
#if SMC_ANY_EXPLICIT
    if (kind == 5) return smc_explicit(k, xs);
#endif
    const int v0 = xs[meta & 0xFFFu];
    const int v1 = xs[(meta >> 12) & 0xFFFu];
    double h;
#if SMC_ANY_GENERAL
    if (kind == 4) {
        const smc_i64 y0 = v0, y1 = v1;
        const smc_i64 h0 = ((meta >> 27) & 1u) ? (y0 * (y0 - 1)) / 2 : y0;
        const smc_i64 h1 = ((meta >> 28) & 1u) ? (y1 * (y1 - 1)) / 2 : y1;
        h = (double)(h0 * h1);
    } else
#endif
    {
        const int xb = (kind == 2) ? max(v0 - 1, 0) : v1;
        h = __dmul_rn((double)v0, (double)xb);
    }
    double a = __dmul_rn(c, h);
#if SMC_ANY_HILL
    if ((int)meta < 0) {
        const double q = __ddiv_rn((double)xs[T.hill_rep[k]], T.hill_k[k]);
        double qn = q;
        for (int i = 1; i < T.hill_n[k]; ++i) qn = __dmul_rn(qn, q);
        a = __ddiv_rn(a, __dadd_rn(1.0, qn));
    }
#endif
    (void)k;
    return a;
}
struct __align__(16) SmcDepFat {
    unsigned ks;      // k | slot << 16
    unsigned meta;
    double c;
};

#ifndef SMC_FLAT
#define SMC_FLAT 1      // dependency work of all tiles of a warp flattened over the 32 lanes
#endif

// smem slot of a(l, m), l = group (owner lane), m = member (SMC_CH is a power of two)
#if SMC_ROWLAYOUT
// row layout: group l is a contiguous row of SMC_GSP (odd) doubles, so the lanes of a tile
// at the same member fall on distinct bank pairs and the group walk is immediate offsets
__device__ __forceinline__ int smc_slot(int l, int m) { return l * SMC_GSP + m; }
#else
__device__ __forceinline__ int smc_slot(int l, int m) { return m * SMC_TW + (l ^ ((m / SMC_CH) % SMC_TW)); }
#endif
// dependency entry -> (reaction k, smem slot of a_k)
__device__ __forceinline__ void smc_dep_entry(unsigned e, int& k, int& slot) {
#if SMC_DEP16
    k = (int)e;
    const int l = k / SMC_GS, m = k - l * SMC_GS;
    slot = smc_slot(l, m);
#else
    k = (int)(e & 0xFFFFu);
    slot = (int)(e >> 16);
#endif
}
// owner lane of a slot (inverse of smc_slot)
#if SMC_ROWLAYOUT
__device__ __forceinline__ int smc_owner(int slot) { return slot / SMC_GSP; }
#else
__device__ __forceinline__ int smc_owner(int slot) { return (slot % SMC_TW) ^ ((slot / SMC_TW / SMC_CH) % SMC_TW); }
#endif

// Group sum of lane l: two interleaved partial sums (even / odd members, each left to
// right), then added -- a fixed order (reading R12) with half the dependent-add chain.
__device__ __forceinline__ double smc_group_sum(const double* at, int l) {
#if SMC_ROWLAYOUT
    at += l * SMC_GSP;                        // row of group l: members at immediate offsets
    l = 0;
#endif
    double se = at[smc_slot(l, 0)];
    if (SMC_GS == 1) return se;
    double so = at[smc_slot(l, 1)];
#pragma unroll
    for (int m = 2; m + 1 < SMC_GS; m += 2) {
        se = __dadd_rn(se, at[smc_slot(l, m)]);
        so = __dadd_rn(so, at[smc_slot(l, m + 1)]);
    }
    if (SMC_GS & 1) se = __dadd_rn(se, at[smc_slot(l, SMC_GS - 1)]);
    return __dadd_rn(se, so);
}

extern "C" __global__ void __launch_bounds__(768, 1) smc_ssa_tile(SmcParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ __align__(8) unsigned long long bar;
    const int lane = (int)(threadIdx.x & 31u), warp = (int)(threadIdx.x >> 5);
    constexpr int TW = SMC_TW, TPW = 32 / SMC_TW;
    const int tl = lane % TW, tile = lane / TW;
    const smc_u32 tbits = (TW == 32) ? SMC_FULL : (((1u << TW) - 1u) << (tile * TW));

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
    T.law = (const SmcLaw*)(smem + SMC_OFF_LAW);
    T.hill_rep = (const int*)(smem + SMC_OFF_HREP);
    T.hill_k = (const double*)(smem + SMC_OFF_HK);
    T.hill_n = (const int*)(smem + SMC_OFF_HN);
    T.chg = (const unsigned short*)(smem + SMC_OFF_CHG);
    T.dep_off = (const unsigned*)(smem + SMC_OFF_DOFF);
#if SMC_DEP16
    T.dep = (const unsigned short*)(smem + SMC_OFF_DEP);
#else
    T.dep = (const unsigned*)(smem + SMC_OFF_DEP);
#endif
    unsigned char* const warp_base = smem + SMC_TAB_BYTES + (size_t)warp * TPW * SMC_TILE_BYTES;
    double* at = (double*)(warp_base + (size_t)tile * SMC_TILE_BYTES);
    int* xs = (int*)(at + SMC_GSP * TW);

    // ---- per-tile trajectory state (replicated in the tile's lanes)
    bool act = false, exhausted = false;
    smc_u64 rel = 0, traj = 0;
    double t = 0.0, tp = 0.0, S = 0.0;
    smc_u32 k = 0, kb = 0;
    double Eb = 0.0, Ub = 0.0;          // draw of step kb + tl
    SmcMon mon;
    mon.bind(P, ((smc_u64)blockIdx.x * (blockDim.x >> 5) + (smc_u64)warp) * TPW + (smc_u64)tile, tbits,
             tile * TW);                                   // trace slot, lanes, leader (R23)
    smc_u32 c_true = 0, c_false = 0, c_err = 0;   // tile leader
    smc_i64 c_ev = 0;

    for (;;) {
        // ---- refill: tiles without a trajectory claim fresh indices (one atomic per warp)
        for (;;) {
            const bool want = !act && !exhausted;
            const smc_u32 wm = __ballot_sync(SMC_FULL, want && tl == 0);
            if (wm == 0u) break;
            const int leader = __ffs(wm) - 1;
            smc_u64 base = 0;
            if (lane == leader) base = atomicAdd(P.cursor, (smc_u64)__popc(wm));
            base = __shfl_sync(SMC_FULL, base, leader);
            if (want) {
                rel = base + (smc_u64)__popc(wm & ((1u << (tile * TW)) - 1u));
                if (rel >= P.count) exhausted = true;
            }
            const bool init = want && !exhausted;
            if (init) {
                traj = P.first + rel;
                for (int s = tl; s <= SMC_N; s += TW) xs[s] = T.x0[s];   // x[N] = 1
            }
            __syncwarp();
            if (init) {
                for (int m = 0; m < SMC_GS; ++m) {
                    const int j = tl * SMC_GS + m;
                    at[smc_slot(tl, m)] = (j < SMC_M) ? smc_law_tab(j, xs, T) : 0.0;
                }
            }
            __syncwarp();
            if (init) {
                S = smc_group_sum(at, tl);
                t = 0.0;
                tp = 0.0;
                k = 0;
                mon.init();
                mon.enter(0u, 0.0, 0.0, xs);        // sigma_buff = {(s0, t0)}
                const int v = mon.verdict();
                if (v >= 0) {
                    if (tl == 0) {
                        if (v == 1) ++c_true; else ++c_false;
                        if (P.verdicts) { P.verdicts[rel] = (unsigned char)v; P.events_out[rel] = 0; }
                    }
                } else {
                    act = true;
                }
            }
        }
        if (!__any_sync(SMC_FULL, act)) break;

        // ---- burst of TW events: draws of steps k .. k+TW-1, one per lane
        if (act) smc_draw(P.seed, traj, (smc_u64)(k + (smc_u32)tl), Eb, Ub);
        kb = k;
#pragma unroll 1
        for (int s = 0; s < TW; ++s) {
            if (!__any_sync(SMC_FULL, act)) break;
            // a0 = inclusive scan of the group sums, fixed association per lane
            double Pp = S;
#pragma unroll
            for (int o = 1; o < TW; o <<= 1) {
                const double y = __shfl_up_sync(SMC_FULL, Pp, o, TW);
                if (tl >= o) Pp = __dadd_rn(y, Pp);
            }
            const double A = __shfl_sync(SMC_FULL, Pp, TW - 1, TW);
            const int q = (int)(k - kb) & (TW - 1);
            const double E = __shfl_sync(SMC_FULL, Eb, q, TW);
            const double U = __shfl_sync(SMC_FULL, Ub, q, TW);
            const double tau = smc_tau(E, A);
            const double tn = __dadd_rn(t, tau);
            int v = -1;
            if (act) {
                if (!(A >= SMC_A_MIN) || A > SMC_A_MAX) {            // A == 0: absorbed; else error (R19)
                    if (A == 0.0) { mon.absorb(); v = mon.verdict(); }     // absorbed (reading R7)
                    else v = 2;                                            // bad propensity
                } else {
                    mon.advance(k, tn, tau);
                    v = mon.verdict();
                    if (v < 0 && SMC_TMAX > 0.0 && tn > SMC_TMAX) { mon.timeout(); v = mon.verdict(); }
                }
            }
            const bool go = act && v < 0;              // this tile applies a reaction
            // ---- two-level selection (Eq. 2b): group g by ballot on the scan ...
            const double target = __dmul_rn(U, A);
            const smc_u32 bg = (__ballot_sync(SMC_FULL, Pp > target) & tbits) >> (tile * TW);
            int g = __ffs(bg) - 1;
            if (__any_sync(SMC_FULL, bg == 0u)) {          // rounding: last group with a_j > 0 (R11)
                const smc_u32 bp = (__ballot_sync(SMC_FULL, S > 0.0) & tbits) >> (tile * TW);
                if (bg == 0u) g = bp ? 31 - __clz(bp) : 0;
            }
            double base = __shfl_sync(SMC_FULL, Pp, (g + TW - 1) & (TW - 1), TW);
            if (g == 0) base = 0.0;
            // ... then the member inside group g: lane tl scans its chunk of SMC_CH elements
            double cs = 0.0;
            double av[SMC_CH];
#pragma unroll
            for (int c = 0; c < SMC_CH; ++c) {
                const int m = tl * SMC_CH + c;
                av[c] = (m < SMC_GS) ? at[smc_slot(g, m)] : 0.0;
                cs = (c == 0) ? av[c] : __dadd_rn(cs, av[c]);
            }
            double ps = cs;                              // inclusive scan of the chunk sums
#pragma unroll
            for (int o = 1; o < TW; o <<= 1) {
                const double y = __shfl_up_sync(SMC_FULL, ps, o, TW);
                if (tl >= o) ps = __dadd_rn(y, ps);
            }
            double acc = __shfl_up_sync(SMC_FULL, ps, 1, TW);
            acc = (tl == 0) ? base : __dadd_rn(base, acc);
            int hit = -1;
#pragma unroll
            for (int c = 0; c < SMC_CH; ++c) {
                acc = __dadd_rn(acc, av[c]);
                if (hit < 0 && acc > target) hit = c;
            }
            const smc_u32 bh = (__ballot_sync(SMC_FULL, bg != 0 && hit >= 0) & tbits) >> (tile * TW);
            int jm = __shfl_sync(SMC_FULL, ((__ffs(bh) - 1) & (TW - 1)) * SMC_CH + hit, (__ffs(bh) - 1) & (TW - 1), TW);
            if (__any_sync(SMC_FULL, bh == 0u)) {          // rounding: last a_j > 0 (reading R11)
                int lastpos = -1;
#pragma unroll
                for (int c = 0; c < SMC_CH; ++c)
                    if (av[c] > 0.0) lastpos = c;
                const smc_u32 bl = (__ballot_sync(SMC_FULL, lastpos >= 0) & tbits) >> (tile * TW);
                const int src = bl ? 31 - __clz(bl) : 0;
                const int jl = __shfl_sync(SMC_FULL, src * SMC_CH + lastpos, src, TW);
                if (bh == 0u) jm = jl;
            }
            const int j = go ? g * SMC_GS + jm : 0;

            // ---- x += v_j (<= 4 distinct species, one lane each; wrapping add, sign = overflow)
            bool ovf = false;
            if (go && tl < 4) {
                const unsigned e = T.chg[j * 4 + tl];
                if (e != 0xFFFFu) {
                    const int sp = (int)(e >> 4);
                    const int nv = (int)((unsigned)xs[sp] + (unsigned)((int)(e & 15u) - 8));
                    ovf = nv < 0;
                    xs[sp] = nv;
                }
            }
            const bool tile_ovf = ((__ballot_sync(SMC_FULL, ovf) & tbits) != 0u);
            __syncwarp();
            // ---- a_k = law_k(x) for k in dep(j) of every tile, flattened over the 32 lanes
            smc_u32 touched = 0;                         // bit (tile' * TW + owner lane)
            {
                const unsigned d0 = go ? T.dep_off[j] : 0u;
                const unsigned nd = go ? T.dep_off[j + 1] - d0 : 0u;
#if SMC_DEPSP
                if (TPW == 1) {                           // union of the reader lists of the changed species
                    unsigned st[4], pre[4], tot = 0;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const unsigned ce = go ? T.chg[j * 4 + q] : 0xFFFFu;
                        const unsigned sp = ce >> 4;
                        st[q] = (ce != 0xFFFFu) ? T.dep_off[sp] : 0u;
                        const unsigned nq = (ce != 0xFFFFu) ? T.dep_off[sp + 1] - st[q] : 0u;
                        pre[q] = tot;
                        tot += nq;
                    }
                    for (unsigned b = (unsigned)lane; b < tot; b += 32u) {
                        const int q = (b >= pre[1]) + (b >= pre[2]) + (b >= pre[3]);
                        unsigned base = st[0], p0 = 0u;
#pragma unroll
                        for (int w = 1; w < 4; ++w)
                            if (q == w) { base = st[w]; p0 = pre[w]; }
                        int kk, slot;
                        smc_dep_entry(T.dep[base + (b - p0)], kk, slot);
                        at[slot] = smc_law_tab(kk, xs, T);
                        touched |= 1u << smc_owner(slot);
                    }
                } else
#endif
                if (TPW == 1 || !SMC_FLAT) {              // each tile walks its own dep(j) with its TW lanes
                    const smc_u32 tb = (TPW == 1) ? 0u : (smc_u32)(tile * TW);
                    for (unsigned b = (unsigned)tl; __any_sync(SMC_FULL, b < nd); b += (unsigned)TW) {
                        if (b < nd) {
#if SMC_FATDEP
                            const SmcDepFat D = ((const SmcDepFat*)T.dep)[d0 + b];
                            const int slot = (int)(D.ks >> 16);
                            at[slot] = smc_law_meta(D.meta, D.c, (int)(D.ks & 0xFFFFu), xs, T);
#else
                            int kk, slot;
                            smc_dep_entry(T.dep[d0 + b], kk, slot);
                            at[slot] = smc_law_tab(kk, xs, T);
#endif
                            touched |= 1u << (tb + (smc_u32)smc_owner(slot));
                        }
                    }
                } else {
                    // item b of the warp's concatenated dep lists belongs to tile u (prefix
                    // search) and reads entry b + (d0_u - pre_u), fetched from tile u by one shuffle
                    unsigned pre[TPW], tot = 0, mypre = 0;
#pragma unroll
                    for (int u = 0; u < TPW; ++u) {
                        pre[u] = tot;
                        if (u == tile) mypre = tot;
                        tot += __shfl_sync(SMC_FULL, nd, u * TW);
                    }
                    const unsigned mydelta = d0 - mypre;
                    for (unsigned b0 = 0; b0 < tot; b0 += 32u) {
                        const unsigned b = b0 + (unsigned)lane;
                        int u = 0;
#pragma unroll
                        for (int w = 1; w < TPW; ++w) u += (b >= pre[w]) ? 1 : 0;
                        const unsigned delta = __shfl_sync(SMC_FULL, mydelta, u * TW);
                        if (b < tot) {
                            double* at_u = (double*)(warp_base + (size_t)u * SMC_TILE_BYTES);
                            const int* xs_u = (const int*)(at_u + SMC_GSP * TW);
#if SMC_FATDEP
                            const SmcDepFat D = ((const SmcDepFat*)T.dep)[b + delta];
                            const int slot = (int)(D.ks >> 16);
                            at_u[slot] = smc_law_meta(D.meta, D.c, (int)(D.ks & 0xFFFFu), xs_u, T);
#else
                            int kk, slot;
                            smc_dep_entry(T.dep[b + delta], kk, slot);
                            at_u[slot] = smc_law_tab(kk, xs_u, T);
#endif
                            touched |= 1u << (u * TW + smc_owner(slot));
                        }
                    }
                }
            }
            touched = __reduce_or_sync(SMC_FULL, touched);
            __syncwarp();
            // ---- re-sum only the touched groups (fixed order)
            if ((touched >> lane) & 1u) S = smc_group_sum(at, tl);
            if (go) {
                if (tile_ovf) {
                    v = 2;                                // count overflow
                } else {
                    tp = t;
                    t = tn;
                    ++k;
                    mon.enter(k, t, tp, xs);
                    v = mon.verdict();
                    if (v < 0 && (smc_u64)k >= P.event_cap) v = mon.at_cap((long long)k);
                }
            }
            if (act && v >= 0) {
                const long long ke = mon.events((long long)k);   // the window monitor: the first
                if (tl == 0) {                                    // decision index
                    if (v == 1) ++c_true;
                    else if (v == 0) ++c_false;
                    else ++c_err;
                    c_ev += ke;
                    if (P.verdicts) { P.verdicts[rel] = (unsigned char)v; P.events_out[rel] = (int)ke; }
                }
                act = false;
            }
        }
    }
    smc_flush_counts(c_true, c_false, c_ev, c_err, P.counters);
}
