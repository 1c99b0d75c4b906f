// ssa_delta.cuh -- variant 5: persistent TILE-OWNED SSA + monitor kernel for large
// mass-action networks (C5: 200 x 1000) that keeps NO per-reaction propensities.
//
// Per trajectory the shared-memory slice holds only
//   * the counts x[N+1] (int32; x[N] = 1 is the operand of h = x * 1 and h = 1 * 1), and
//   * G exact fixed-point group sums  Sg = sum_{k in group g} Cq_k * h_k(x)  as unsigned
//     128-bit integers (two u64 words), where h_k is the EXACT integer count of the law in
//     the table's form (x0 * x1 with x[N] = 1; x (x - 1) for a homodimer, whose 1/2 is folded
//     into the table's rate exactly) and Cq_k = round(c_k * 2^L), L fixed per model so that
//     no sum can overflow (reading R26).
// Integer addition is exact and associative, so the group sums are maintained
// INCREMENTALLY and still never drift: after reaction j fires, every k in dep(j) adds
// Cq_k * (h_k(x_new) - h_k(x_old)) to its group with two 64-bit shared-memory atomics
// (carry propagated) -- at every step Sg equals sum Cq_k h_k(x) exactly, whatever the
// order of the updates.  This replaces the 8 B x M stored propensities of variant 2 (C5:
// 8 KiB per trajectory, 22 resident trajectories per SM) by G x 16 B (C5: 512 B).
//
// A tile of SMC_TW lanes owns a trajectory (TPW = 32 / TW tiles per warp, lock step).
// Lane l owns the GPL = G / TW consecutive groups [l GPL, (l+1) GPL); group g is stored at
// slot (g mod GPL) * TW + g / GPL so that the level-1 reads of a tile are conflict free.
// Per event:
//   * level 1: a0 = tile scan of the lane sums of the groups converted to binary64
//     (Sg * 2^-L; a fixed order, reading R12); tau = -log(u1) / a0 (Eq. 2a);
//   * the monitor advance (close windows t' passes; halt if decided);
//   * selection (Eq. 2b): the group g whose prefix first exceeds u2 a0 (ballot over the
//     lane prefixes, then the owner lane's groups in order), then the member inside g:
//     the TW lanes re-evaluate the S members' propensities a_k = c_k h_k in binary64 --
//     the oracle's own values bit for bit -- and scan them from the level-1 base;
//     rounding (no prefix exceeds the target) takes the last member with a_k > 0 (R11);
//   * x += v_j by <= 4 lanes, then the dependency deltas: dep(j) is packed in rounds of TW
//     entries, no group twice in a round, each entry carrying the changes R_j applies to
//     the law's operands, so h_k(x_new) - h_k(x_old) follows from the new counts alone and
//     every lane updates its group with a plain read-modify-write (no atomics);
//   * the monitor entry at the new state.
// Draws (Philox + log) of the next TW steps are computed by the TW lanes at once, as in
// variant 2.  Only mass action of order <= 2 (no Hill, explicit or order 3-4 law), and
// formulas inside the streaming templates, run here (Model::variant).
//
// Generated hooks (codegen.cpp): SMC_N, SMC_M, SMC_TW, SMC_DG, SMC_DS,
//   SMC_DSCALE (2^L), SMC_DINV (2^-L), SMC_DHI (2^(64-L)), SMC_OFF_X0/LAW/CQ/CHG/DOFF/DEP,
//   SMC_TAB_BYTES, SMC_TILE_BYTES, SMC_DBLOCK, SMC_TMAX, SmcMon.

struct __align__(16) SmcDLaw {       // the dependency pass's law entry
    unsigned ops;                     // s0 | s1 << 16 (x[N] = 1 for a missing operand)
    unsigned kind;                    // 0..3 (2: homodimer x (x - 1))
    smc_u64 cq;                       // Cq_k = round(c_k 2^L)
};

struct SmcDTabs {
    const int* x0;
    const SmcLaw* law;               // {s0 | kind << 16, s1, c} (kind 0..3, c folded for kind 2)
    const unsigned short* chg;       // [M][4]: species << 4 | (delta + 8), 0xFFFF = none
    const SmcDLaw* dlaw;             // [M]: operands, kind, Cq_k
#if SMC_DDESC64
    const smc_u64* dep_off;          // [M+1]: start | rounds << 24 | (entries of round r - 1) << (28 + 4 r)
#else
    const unsigned* dep_off;         // [M+1]: start | rounds << 24
#endif
    const unsigned char* rcnt;       // [M][DRMAX]: entries per round (without SMC_DDESC64)
#if SMC_DDEP16
    const unsigned short* dep;       // k | (d0 + 4) << 10 | (d1 + 4) << 13 (changes of operands s0, s1)
#else
    const unsigned* dep;             // k | (d0 + 8) << 16 | (d1 + 8) << 20
#endif
};

#ifndef SMC_DFAST
#define SMC_DFAST 1
#endif

// exact integer h_k in the table's form: x0 * x1 (kinds 0, 1, 3 with x[N] = 1), x0 (x0 - 1)
// (kind 2; 0 for x0 <= 1).  Counts < 2^31, so the product fits int64 exactly.
__device__ __forceinline__ smc_i64 smc_dh(const SmcDLaw& L, const int* xs) {
    const int v0 = xs[L.ops & 0xFFFFu];
    const int v1 = (L.kind == 2u) ? v0 - 1 : xs[L.ops >> 16];
    return (smc_i64)v0 * v1;
}
// a_k = c_k * h_k in binary64: h = fl(x0 * x1) (a single rounding of the exact integer
// product), the same operations as variants 1, 2 and 4 -- equal to the oracle's
// c_k * (double)h_k bit for bit (reading R20)
__device__ __forceinline__ double smc_dlaw(const SmcLaw& L, const int* xs) {
    // (double)(x0 * xb) of the exact int64 product: the same single rounding as fl(x0 * xb)
    // (the second operand is read only for x0 x1: kind 1 has x[N] = 1 -- fewer shared loads)
    const unsigned kind = (L.u0 >> 16) & 7u;
    const int v0 = xs[L.u0 & 0xFFFFu];
#if SMC_DFAST
    // branch-free: the second operand is x[N] = 1 for kinds 0 and 1, x0 - 1 for a homodimer
    // (x0 (x0 - 1) = 0 at x0 = 0 either way)
    const int xr = xs[L.u1 & 0xFFFFu];
    const int xb = (kind == 2u) ? v0 - 1 : xr;
#else
    int xb = 1;
    if (kind == 3u) xb = xs[L.u1 & 0xFFFFu];
    else if (kind == 2u) xb = max(v0 - 1, 0);
#endif
    return __dmul_rn(L.c, __ll2double_rn((smc_i64)v0 * xb));
}

#ifdef SMC_DBOUNDS
#define SMC_BC(i, lim, tag) do { if ((unsigned)(i) >= (unsigned)(lim)) { printf("DBOUNDS %s %d >= %d (lane %d warp %d)\n", tag, (int)(i), (int)(lim), (int)(threadIdx.x & 31), (int)(threadIdx.x >> 5)); asm volatile("trap;"); } } while (0)
#else
#define SMC_BC(i, lim, tag) do { } while (0)
#endif
// group g -> 16-byte slot in the tile's slice
constexpr int SMC_DGPL = SMC_DG / SMC_TW;
#ifndef SMC_DCHECK
#define SMC_DCHECK 0
#endif
__device__ __forceinline__ int smc_gslot(int g) { return (g % SMC_DGPL) * SMC_TW + g / SMC_DGPL; }

// Sg * 2^-L in binary64 (hi 2^(64-L) + lo 2^-L: two roundings, ulp-level -- reading R26)
__device__ __forceinline__ double smc_g2d(ulonglong2 w) {
    return __fma_rn(__ull2double_rn(w.y), SMC_DHI, __dmul_rn(__ull2double_rn(w.x), SMC_DINV));
}

// h_k(x_new) - h_k(x_old) from the new counts and the changes a, b that R_j applied to the
// operand species s0, s1 of law k:
//   x0 x1:       a x1 + b x0 - a b           (x_old = x_new - d; kind 1: x1 = x[N] = 1, b = 0)
//   x0 (x0 - 1): a (2 x0 - a - 1)            (homodimer, s0 = s1)
// exact in int64 (counts < 2^31, |d| <= 8)
__device__ __forceinline__ smc_i64 smc_ddh(const SmcDLaw& L, int a, int b, const int* xs) {
    const int x0 = xs[L.ops & 0xFFFFu];
    if (L.kind == 2u) return (smc_i64)a * (2 * (smc_i64)x0 - a - 1);
    if (L.kind != 3u) return (smc_i64)a;          // x0 * x[N]: b = 0, x1 = 1
    const int x1 = xs[L.ops >> 16];
    return (smc_i64)a * x1 + (smc_i64)b * x0 - (smc_i64)(a * b);
}

// Sg += Cq dh, two's complement 128-bit: low word = Cq dh mod 2^64, high word = the unsigned
// high product minus Cq when dh < 0 (signed correction), plus the carry of the low word.  A
// plain read-modify-write: the rounds of dep(j) are packed so that no two lanes of a round
// touch the same group.
__device__ __forceinline__ void smc_gadd(ulonglong2* w, smc_u64 cq, smc_i64 dh) {
    const smc_u64 d = (smc_u64)dh;
    const smc_u64 lo = cq * d;
    const smc_u64 hi = __umul64hi(cq, d) - (dh < 0 ? cq : 0ull);
    ulonglong2 v = *w;
    v.x += lo;
    v.y += hi + (v.x < lo ? 1ull : 0ull);
    *w = v;
}

// The same update without branches on the law's kind (a divergent warp ran every kind's path):
// h = x0 x1 with x1 = x0 - 1 for a homodimer (whose entry carries d1 = d0) and x1 = x[N] = 1
// for a first-order law (d1 = 0), so dh = d0 x1 + d1 x0 - d0 d1 for every kind; and, while
// |dh| < 2^32 (counts below ~2^28), Cq |dh| as two 32 x 32 -> 64-bit products added to the
// 128-bit sum in two's complement.  Bit-identical to smc_ddh + smc_gadd (SMC_DCHECK).
__device__ __forceinline__ void smc_gupd(ulonglong2* w, const SmcDLaw& L, int a, int b, const int* xs) {
    const int x0 = xs[L.ops & 0xFFFFu];
    const int xr = xs[L.ops >> 16];
    const int x1 = (L.kind == 2u) ? x0 - 1 : xr;
    const smc_i64 dh = (smc_i64)a * x1 + (smc_i64)b * x0 - (smc_i64)(a * b);
    const smc_u64 u = (smc_u64)(dh < 0 ? -dh : dh);
    if (u >> 32) { smc_gadd(w, L.cq, dh); return; }
    const smc_u32 u32 = (smc_u32)u;
    const smc_u64 p0 = (smc_u64)(smc_u32)L.cq * u32;
    const smc_u64 p1 = (smc_u64)(smc_u32)(L.cq >> 32) * u32;
    const smc_u64 lo = p0 + (p1 << 32);
    const smc_u64 hi = (p1 >> 32) + (lo < p0 ? 1ull : 0ull);
    const smc_u64 m = dh < 0 ? ~0ull : 0ull;                    // two's complement negation
    const smc_u64 l2 = (lo ^ m) - m;
    const smc_u64 h2 = (hi ^ m) + ((m & 1ull) & (lo == 0ull ? 1ull : 0ull));
    ulonglong2 v = *w;
    v.x += l2;
    v.y += h2 + (v.x < l2 ? 1ull : 0ull);
    *w = v;
}

extern "C" __global__ void __launch_bounds__(SMC_DBLOCK, 1) smc_ssa_delta(SmcParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ __align__(8) unsigned long long bar;
    const int lane = (int)(threadIdx.x & 31u), warp = (int)(threadIdx.x >> 5);
    constexpr int TW = SMC_TW, TPW = 32 / SMC_TW, GPL = SMC_DGPL, S = SMC_DS, CH = SMC_DS / SMC_TW;
    static_assert(SMC_DG % SMC_TW == 0 && SMC_DS % SMC_TW == 0, "G and S must be multiples of TW");
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
    SmcDTabs T;
    T.x0 = (const int*)(smem + SMC_OFF_X0);
    T.law = (const SmcLaw*)(smem + SMC_OFF_LAW);
    // per-event tables: global memory through the L1 (SMC_DGLOBAL) or the staged shared copy
#if SMC_DGLOBAL
    const unsigned char* const tb = (const unsigned char*)P.tables;
#else
    const unsigned char* const tb = smem;
#endif
    T.chg = (const unsigned short*)(tb + SMC_OFF_CHG);
#if SMC_DDESC64
    T.dep_off = (const smc_u64*)(tb + SMC_OFF_DOFF);
#else
    T.dep_off = (const unsigned*)(tb + SMC_OFF_DOFF);
#endif
    T.dlaw = (const SmcDLaw*)(smem + SMC_OFF_CQ);
    T.rcnt = (const unsigned char*)(tb + SMC_OFF_RCNT);
#if SMC_DDEP16
    T.dep = (const unsigned short*)(tb + SMC_OFF_DEP);
#else
    T.dep = (const unsigned*)(tb + SMC_OFF_DEP);
#endif
    unsigned char* const slice = smem + SMC_TAB_BYTES + ((size_t)warp * TPW + (size_t)tile) * SMC_TILE_BYTES;
    ulonglong2* const gs = (ulonglong2*)slice;                  // G exact group sums
    int* const xs = (int*)(slice + 16 * SMC_DG);

    // every tile's slice starts as the initial state (x0 and its exact group sums), so the
    // tiles that never get a trajectory (the tail of a launch: a warp with fewer trajectories
    // than tiles) run the warp's lock-step code on well-defined values
    for (int s = tl; s <= SMC_N; s += TW) xs[s] = T.x0[s];
    __syncwarp();
#pragma unroll 1
    for (int i = 0; i < GPL; ++i) {
        const int g = tl * GPL + i;
        smc_u64 lo = 0ull, hi = 0ull;
#pragma unroll 1
        for (int m = 0; m < S; ++m) {
            const int kk = g * S + m;
            if (kk < SMC_M) {
                const SmcDLaw L = T.dlaw[kk];
                const smc_u64 h = (smc_u64)smc_dh(L, xs), cq = L.cq;
                const smc_u64 plo = cq * h;
                lo += plo;
                hi += __umul64hi(cq, h) + (lo < plo ? 1ull : 0ull);
            }
        }
        gs[smc_gslot(g)] = make_ulonglong2(lo, hi);
    }
    __syncwarp();

    bool act = false, exhausted = false;
    smc_u64 rel = 0, traj = 0;
    double t = 0.0, tp = 0.0;
    smc_u32 k = 0, kb = 0;
    double Eb = 0.0, Ub = 0.0;          // draw of step kb + tl
    SmcMon mon;
    mon.bind(P, 0ull, tbits, tile * TW);
    smc_u32 c_true = 0, c_false = 0, c_err = 0;   // tile leader
    smc_i64 c_ev = 0;

#ifdef SMC_DTRACE
    long long guard = 0;
#endif
    for (;;) {
#ifdef SMC_DTRACE
        if (++guard > 20000) {
            if (tl == 0) printf("DTRACE guard: warp %d tile %d act %d exh %d rel %llu k %u x0 %d\n", warp, tile, (int)act,
                                (int)exhausted, rel, k, xs[0]);
            return;
        }
#endif
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
            if (init) {                                  // exact group sums from scratch
#pragma unroll 1
                for (int i = 0; i < GPL; ++i) {
                    const int g = tl * GPL + i;
                    smc_u64 lo = 0ull, hi = 0ull;
#pragma unroll 1
                    for (int m = 0; m < S; ++m) {
                        const int kk = g * S + m;
                        if (kk < SMC_M) {
                            const SmcDLaw L = T.dlaw[kk];
                            const smc_u64 h = (smc_u64)smc_dh(L, xs), cq = L.cq;
                            const smc_u64 plo = cq * h;
                            lo += plo;
                            hi += __umul64hi(cq, h) + (lo < plo ? 1ull : 0ull);
                        }
                    }
                    gs[smc_gslot(g)] = make_ulonglong2(lo, hi);
                }
            }
            __syncwarp();
            if (init) {
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
            // ---- level 1: this lane's groups in binary64, lane sum, tile scan -> a0
            double D[GPL];
            double Ls = 0.0;
#pragma unroll
            for (int i = 0; i < GPL; ++i) {
                D[i] = smc_g2d(gs[i * TW + tl]);
                Ls = (i == 0) ? D[0] : __dadd_rn(Ls, D[i]);
            }
            double Pl = Ls;
#pragma unroll
            for (int o = 1; o < TW; o <<= 1) {
                const double y = __shfl_up_sync(SMC_FULL, Pl, o, TW);
                if (tl >= o) Pl = __dadd_rn(y, Pl);
            }
            const double A = __shfl_sync(SMC_FULL, Pl, TW - 1, TW);
            const int q = (int)(k - kb) & (TW - 1);
            const double E = __shfl_sync(SMC_FULL, Eb, q, TW);
            const double U = __shfl_sync(SMC_FULL, Ub, q, TW);
            const double tau = smc_tau(E, A);
            const double tn = __dadd_rn(t, tau);
            int v = -1;
#ifdef SMC_DTRACE
            if (act && tl == 0 && !(A > 0.0)) printf("DTRACE absorb rel %llu k %u A %g x %d %d %d %d\n", rel, k, A, xs[0], xs[1], xs[2], xs[3]);
#endif
            if (act) {
                if (!(A >= SMC_A_MIN) || A > SMC_A_MAX) {            // A == 0: absorbed; else error (R19)
                    if (A == 0.0) { mon.absorb(); v = mon.verdict(); }     // absorbed (reading R7)
                    else v = 2;
                } else {
                    mon.advance(k, tn, tau);
                    v = mon.verdict();
                    if (v < 0 && SMC_TMAX > 0.0 && tn > SMC_TMAX) { mon.timeout(); v = mon.verdict(); }
                }
            }
            const bool go = act && v < 0;              // this tile applies a reaction
            __syncwarp();                              // reconverge after the tile-divergent monitor step
            // ---- selection (Eq. 2b), level 1: owner lane by ballot, then its groups in order
            const double target = __dmul_rn(U, A);
            const smc_u32 bo = (__ballot_sync(SMC_FULL, Pl > target) & tbits) >> (tile * TW);
            double acc = __shfl_up_sync(SMC_FULL, Pl, 1, TW);
            if (tl == 0) acc = 0.0;
            int gi = -1, lastpos = -1;
            double gbase = 0.0;
#pragma unroll
            for (int i = 0; i < GPL; ++i) {
                const double nx = __dadd_rn(acc, D[i]);
                if (gi < 0 && nx > target) { gi = i; gbase = acc; }
                if (D[i] > 0.0) lastpos = i;
                acc = nx;
            }
            // rounding (R11): the owner's running sum may not pass the target although its
            // prefix does, or no lane passes it at all -- then the last positive group of
            // the owner (resp. of the tile) and in it the last member with a_k > 0
            const smc_u32 bp = (__ballot_sync(SMC_FULL, lastpos >= 0) & tbits) >> (tile * TW);
            const int owner = bo ? __ffs(bo) - 1 : (bp ? 31 - __clz(bp) : 0);
            const bool found = gi >= 0;
            if (!found) gi = lastpos < 0 ? 0 : lastpos;
            const int og = __shfl_sync(SMC_FULL, gi, owner, TW);
            const bool fb = !bo || !__shfl_sync(SMC_FULL, (int)found, owner, TW);
            const double base = __shfl_sync(SMC_FULL, gbase, owner, TW);
            const int g = owner * GPL + og;
            // ---- level 2: the members of group g, CH per lane, re-evaluated in binary64
            double av[CH];
            double cs = 0.0;
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                SMC_BC(g * S + c * TW + tl, SMC_DG * SMC_DS, "law");
                av[c] = smc_dlaw(T.law[g * S + c * TW + tl], xs);   // member tl CH + c (permuted table)
                cs = (c == 0) ? av[0] : __dadd_rn(cs, av[c]);
            }
            double ps = cs;
#pragma unroll
            for (int o = 1; o < TW; o <<= 1) {
                const double y = __shfl_up_sync(SMC_FULL, ps, o, TW);
                if (tl >= o) ps = __dadd_rn(y, ps);
            }
            double a2 = __shfl_up_sync(SMC_FULL, ps, 1, TW);
            a2 = (tl == 0) ? base : __dadd_rn(base, a2);
            int hit = -1, lastm = -1;
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                a2 = __dadd_rn(a2, av[c]);
                if (hit < 0 && a2 > target) hit = c;
                if (av[c] > 0.0) lastm = c;
            }
            const smc_u32 bh = (__ballot_sync(SMC_FULL, hit >= 0) & tbits) >> (tile * TW);
            // the rounding fallback (R11: the last member with a_k > 0) and the regular hit, both
            // always computed: the shuffles run converged, outside any warp-level branch
            const smc_u32 bl = (__ballot_sync(SMC_FULL, lastm >= 0) & tbits) >> (tile * TW);
            const int src = bl ? 31 - __clz(bl) : 0;
            const int jl = __shfl_sync(SMC_FULL, src * CH + lastm, src, TW);
            const int hsrc = bh ? __ffs(bh) - 1 : 0;
            const int jh = __shfl_sync(SMC_FULL, hsrc * CH + hit, hsrc, TW);
            const int jm = (bh == 0u || fb) ? jl : jh;
            const int j = go ? g * S + jm : 0;
#ifdef SMC_DTRACE
            if (act && !(A > 0.0)) printf("DTRACE sel lane %d rel %llu g %d jm %d j %d go %d v %d owner %d og %d\n", lane, rel, g, jm, j, (int)go, v, owner, og);
#endif

            // ---- x += v_j (<= 4 distinct species, one lane each; wrapping add, sign = overflow);
            // a selection outside the reactions (never seen on C4/C5 networks; observed on small
            // absorbing models with several tiles per warp) ends the replica as an error
            bool ovf = go && (unsigned)j >= (unsigned)SMC_M;
            if (go && !ovf && tl < 4) {
                SMC_BC(j, SMC_M, "chg j");
                const unsigned e = T.chg[j * 4 + tl];
                if (e != 0xFFFFu) {
                    const int sp = (int)(e >> 4);
                    SMC_BC(sp, SMC_N, "chg sp");
                    const int nv = (int)((unsigned)xs[sp] + (unsigned)((int)(e & 15u) - 8));
                    ovf = nv < 0;
                    xs[sp] = nv;
                }
            }
            const bool tile_ovf = ((__ballot_sync(SMC_FULL, ovf) & tbits) != 0u);
#if SMC_DDESC64
            const smc_u64 desc = (go && !tile_ovf) ? T.dep_off[j] : 0ull;
#else
            const unsigned desc = (go && !tile_ovf) ? T.dep_off[j] : 0u;
#endif
            __syncwarp();
            // ---- Sg += Cq_k (h_k(x_new) - h_k(x_old)) for k in dep(j), exact, from the new
            // counts and the changes R_j applied to law k's operands; one round at a time (the
            // <= TW entries of a round touch distinct groups: plain read-modify-writes)
#if SMC_DDESC64
            const unsigned dlo = (unsigned)desc, dhi = (unsigned)(desc >> 32);
#else
            const unsigned dlo = desc;
#endif
            const int nr = (int)(dlo >> 24);
            unsigned at = dlo & 0xFFFFFFu;
#pragma unroll 1
            for (int r = 0; __any_sync(SMC_FULL, r < nr); ++r) {
#if SMC_DDESC64
                const int cnt = (r < nr) ? (int)((dhi >> (4 * r)) & 15u) + 1 : 0;
#else
                const int cnt = (r < nr) ? (int)T.rcnt[j * SMC_DRMAX + r] : 0;
#endif
                if (tl < cnt) {
#ifdef SMC_DBOUNDS
                    SMC_BC(SMC_OFF_DEP + (at + tl) * (SMC_DDEP16 ? 2 : 4), SMC_DTABEND, "dep");
#endif
                    const unsigned e = T.dep[at + (unsigned)tl];
#if SMC_DDEP16
                    const int kk = (int)(e & 1023u), a = (int)((e >> 10) & 7u) - 4, b = (int)(e >> 13) - 4;
#else
                    const int kk = (int)(e & 0xFFFFu), a = (int)((e >> 16) & 15u) - 8, b = (int)((e >> 20) & 15u) - 8;
#endif
                    SMC_BC(kk, SMC_M, "dlaw kk");
                    SMC_BC(smc_gslot(kk / S), SMC_DG, "gslot");
                    const SmcDLaw L = T.dlaw[kk];
#if SMC_DFAST
                    smc_gupd(gs + smc_gslot(kk / S), L, a, b, xs);
#else
                    smc_gadd(gs + smc_gslot(kk / S), L.cq, smc_ddh(L, a, b, xs));
#endif
                }
                at += (unsigned)cnt;
                __syncwarp();
            }
#if SMC_DCHECK
            // debug (SMC_DCHECK=1): the incrementally maintained group sums equal a fresh
            // exact recompute, and j is a valid reaction
            if (go && !tile_ovf) {
                bool bad = (j < 0 || j >= SMC_M);
                for (int i = 0; i < GPL; ++i) {
                    const int gg = tl * GPL + i;
                    smc_u64 lo = 0ull, hi = 0ull;
                    for (int m = 0; m < S; ++m) {
                        const int kk = gg * S + m;
                        if (kk < SMC_M) {
                            const SmcDLaw L = T.dlaw[kk];
                            const smc_u64 h = (smc_u64)smc_dh(L, xs), cq = L.cq;
                            const smc_u64 plo = cq * h;
                            lo += plo;
                            hi += __umul64hi(cq, h) + (lo < plo ? 1ull : 0ull);
                        }
                    }
                    const ulonglong2 w = gs[smc_gslot(gg)];
                    if (w.x != lo || w.y != hi) {
                        if (!bad) printf("SMC_DCHECK traj %llu k %u j %d group %d: have %llx:%llx want %llx:%llx\n", traj, k, j, gg,
                                         w.y, w.x, hi, lo);
                        bad = true;
                    }
                }
                if (bad) { printf("SMC_DCHECK traj %llu k %u j %d g %d jm %d\n", traj, k, j, g, jm); asm volatile("trap;"); }
            }
#endif
#ifdef SMC_DTRACE
            if (act && tl == 0 && (k < 4 || !(A > 0.0) || k % 500 == 0))
                printf("DTRACE rel %llu k %u A %.17g tn %.17g j %d x0 %d v %d go %d ovf %d nr %d\n", rel, k, A, tn, j, xs[0], v,
                       (int)go, (int)tile_ovf, nr);
#endif
            if (go) {
                if (tile_ovf) {
                    v = 2;                                // count overflow (R17)
                } else {
                    tp = t;
                    t = tn;
                    ++k;
                    mon.enter(k, t, tp, xs);
                    v = mon.verdict();
                    if (v < 0 && (smc_u64)k >= P.event_cap) v = 2;
                }
            }
            if (act && v >= 0) {
                if (tl == 0) {
                    if (v == 1) ++c_true;
                    else if (v == 0) ++c_false;
                    else ++c_err;
                    c_ev += k;
                    if (P.verdicts) { P.verdicts[rel] = (unsigned char)v; P.events_out[rel] = (int)k; }
                }
                act = false;
            }
        }
    }
    smc_flush_counts(c_true, c_false, c_ev, c_err, P.counters);
}
