// ssa_common.cuh -- device code shared by the SSA kernels (sm_100a).
// Embedded into the generated NVRTC source (jit.cpp) and into the AOT part of
// libsmc.so (aot_kernels.cu).  Independent of oracle/.
#pragma once

typedef unsigned long long smc_u64;
typedef long long smc_i64;
typedef unsigned int smc_u32;

#define SMC_FULL 0xffffffffu

// Launch parameters of one SSA kernel (one shard slice [first, first+count)).
struct SmcParams {
    smc_u64 seed;          // Philox key
    smc_u64 first;         // first trajectory index of the slice
    smc_u64 count;         // trajectories in the slice
    smc_u64* cursor;       // work cursor (relative index), zeroed before launch
    smc_i64* counters;     // {n_true, n_false, events, errors}, zeroed before launch
    unsigned char* verdicts;   // optional per-replica verdict (relative index)
    int* events_out;           // optional per-replica event count
    smc_u64 event_cap;     // per-replica event cap
    const void* tables;    // packed model tables (tile variant)
    double* lit_t;         // window monitor (ssa_window.cuh): every replica slot's rings
    double* lit_unused0;   //   (reserved)
    unsigned* lit_unused1;
    unsigned char* lit_unused2;
    smc_u64 lit_cap;       //   ring entries per replica slot (a power of two)
};

// Philox4x32-10 (Salmon et al. 2011), counter (c0..c3), key (k0, k1).
// Reading R10: c = (k_lo, k_hi, i_lo, i_hi) with k = events applied so far,
// i = trajectory index; key = (seed_lo, seed_hi).
__device__ __forceinline__ void smc_philox(smc_u32 c0, smc_u32 c1, smc_u32 c2, smc_u32 c3, smc_u32 k0, smc_u32 k1,
                                           smc_u32 r[4]) {
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const smc_u32 hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        const smc_u32 hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        const smc_u32 n0 = hi1 ^ c1 ^ k0;
        const smc_u32 n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    r[0] = c0; r[1] = c1; r[2] = c2; r[3] = c3;
}

// Quotient num / den for a positive normal den: reciprocal seed (MUFU), two Newton
// steps, then one residual correction q + r (num - q den).  The result is the
// correctly rounded quotient except in rare last-ulp cases; it is used where the
// parity bar tolerates ulp differences (tau = e / a0: the oracle's glibc log already
// differs from any device log by an ulp now and then).
__device__ __forceinline__ double smc_fdiv(double num, double den) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(den));
    double e = __fma_rn(-den, r, 1.0);
    r = __fma_rn(r, e, r);
    e = __fma_rn(-den, r, 1.0);
    r = __fma_rn(r, e, r);
    const double q = __dmul_rn(num, r);
    return __fma_rn(__fma_rn(-q, den, num), r, q);
}

// -log(x) for x in [2^-53, 1] (the u1 of smc_draw: positive, normal, <= 1).
// The classic argument reduction of fdlibm's __ieee754_log: x = 2^k m with
// m in [sqrt(2)/2, sqrt(2)), f = m - 1, s = f / (2 + f),
// log(1 + f) = f - (hfsq - s (hfsq + R(s^2))), R the minimax series of fdlibm's
// Lg1..Lg7, k ln2 split in ln2_hi + ln2_lo.  About 35 instructions instead of the
// ~80 of the general libdevice log (no special cases: x is never 0, negative,
// subnormal, inf or NaN here).  Accuracy: checked against glibc on the GPU
// (tests/test_gpu_parity.py::test_draws_vs_oracle).
// coefficients in the constant bank: DFMA reads them as c[bank][offset] operands, no
// per-event materialisation of 64-bit immediates in (uniform) registers
__constant__ double smc_lg_c[9] = {6.666666666666735130e-01, 3.999999999940941908e-01, 2.857142874366239149e-01,
                                   2.222219843214978396e-01, 1.818357216161805012e-01, 1.531383769920937332e-01,
                                   1.479819860511658591e-01, 6.93147180369123816490e-01, 1.90821492927058770002e-10};
__device__ __forceinline__ double smc_neglog(double x) {
    int hx = __double2hiint(x);
    const int lx = __double2loint(x);
    int k = (hx >> 20) - 1023;
    hx &= 0x000fffff;
    const int i = (hx + 0x95f64) & 0x100000;
    const double m = __hiloint2double(hx | (i ^ 0x3ff00000), lx);
    k += i >> 20;
    const double f = __dadd_rn(m, -1.0);
    const double s = smc_fdiv(f, __dadd_rn(2.0, f));
    const double dk = (double)k;
    const double z = __dmul_rn(s, s), w = __dmul_rn(z, z);
    const double* C = smc_lg_c;
    const double t1 = __dmul_rn(w, __fma_rn(w, __fma_rn(w, C[5], C[3]), C[1]));
    const double t2 = __dmul_rn(z, __fma_rn(w, __fma_rn(w, __fma_rn(w, C[6], C[4]), C[2]), C[0]));
    const double R = __dadd_rn(t2, t1);
    const double hfsq = __dmul_rn(__dmul_rn(0.5, f), f);
    const double inner = __fma_rn(s, __dadd_rn(hfsq, R), __dmul_rn(dk, C[8]));
    const double lg = __fma_rn(dk, C[7], -__dadd_rn(__dadd_rn(hfsq, -inner), -f));
    return -lg;
}

// The draw of SSA step `step` of trajectory `traj` ("standard Monte Carlo
// methods"):  e = -log(u1) (Eq. 2a numerator), u2 (Eq. 2b).
//   u1 = ((((r0<<32)|r1) >> 11) + 1) * 2^-53 in (0,1],  u2 = (((r2<<32)|r3) >> 11) * 2^-53 in [0,1)
// Split in its integer half (the Philox block) and its fp64 half (u53 + log) so the
// thread kernel can pipeline them one step apart.
__device__ __forceinline__ void smc_draw_words(smc_u64 seed, smc_u64 traj, smc_u64 step, smc_u32 r[4]) {
    smc_philox((smc_u32)step, (smc_u32)(step >> 32), (smc_u32)traj, (smc_u32)(traj >> 32), (smc_u32)seed,
               (smc_u32)(seed >> 32), r);
}
__device__ __forceinline__ void smc_draw_from(const smc_u32 r[4], double& e, double& u2) {
    const smc_u64 w1 = ((smc_u64)r[0] << 32) | r[1];
    const smc_u64 w2 = ((smc_u64)r[2] << 32) | r[3];
    const double u1 = __dmul_rn(__ull2double_rn((w1 >> 11) + 1ull), 0x1p-53);   // 2^-53, exact
    u2 = __dmul_rn(__ull2double_rn(w2 >> 11), 0x1p-53);
    e = smc_neglog(u1);
}
__device__ __forceinline__ void smc_draw(smc_u64 seed, smc_u64 traj, smc_u64 step, double& e, double& u2) {
    smc_u32 r[4];
    smc_draw_words(seed, traj, step, r);
    smc_draw_from(r, e, u2);
}

// tau = e / a0 (Eq. 2a).  The kernels call it only for a0 in [2^-1000, 2^1000], where
// the reciprocal seed is accurate; a0 outside that range (but > 0) ends the replica as
// an error (reading R19) instead of taking a slow IEEE path inside the event loop.
#define SMC_A_MIN 0x1p-1000
#define SMC_A_MAX 0x1p+1000
__device__ __forceinline__ double smc_tau(double e, double a0) { return smc_fdiv(e, a0); }

// functions of general val atoms, identical on both sides of the parity
// contract: min/max by comparison, pow(v, k) a left-to-right product (k = 0: 1)
__device__ __forceinline__ double smc_vmin(double a, double b) { return a < b ? a : b; }
__device__ __forceinline__ double smc_vmax(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ double smc_vpow(double b, int k) {
    double r = 1.0;
    for (int i = 0; i < k; ++i) r = (i == 0) ? b : __dmul_rn(r, b);
    return r;
}

// Kleene three-valued logic (reading R4): 0 false, 1 true, 2 unknown/pending.
__device__ __forceinline__ int smc_knot(int a) { return a == 2 ? 2 : 1 - a; }
__device__ __forceinline__ int smc_kand(int a, int b) { return (a == 0 || b == 0) ? 0 : ((a == 1 && b == 1) ? 1 : 2); }
__device__ __forceinline__ int smc_kor(int a, int b) { return (a == 1 || b == 1) ? 1 : ((a == 0 && b == 0) ? 0 : 2); }

// Leaf status: 0 pending, 1 true, 2 false, 3 unknown (t_max passed).
__device__ __forceinline__ int smc_tri(unsigned char s) { return s == 1 ? 1 : (s == 2 ? 0 : 2); }

// Block reduction of the per-thread verdict counters, then one 64-bit atomic
// per counter per block.  Every thread of the block calls it.
__device__ __forceinline__ void smc_flush_counts(smc_i64 ct, smc_i64 cf, smc_i64 ce, smc_i64 cr, smc_i64* g) {
    __shared__ unsigned long long s_cnt[4];
    if (threadIdx.x < 4) s_cnt[threadIdx.x] = 0ull;
    __syncthreads();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ct += __shfl_down_sync(SMC_FULL, ct, o);
        cf += __shfl_down_sync(SMC_FULL, cf, o);
        ce += __shfl_down_sync(SMC_FULL, ce, o);
        cr += __shfl_down_sync(SMC_FULL, cr, o);
    }
    if ((threadIdx.x & 31u) == 0) {
        atomicAdd(&s_cnt[0], (unsigned long long)ct);
        atomicAdd(&s_cnt[1], (unsigned long long)cf);
        atomicAdd(&s_cnt[2], (unsigned long long)ce);
        atomicAdd(&s_cnt[3], (unsigned long long)cr);
    }
    __syncthreads();
    if (threadIdx.x < 4) atomicAdd((unsigned long long*)&g[threadIdx.x], s_cnt[threadIdx.x]);
}

// ---- TMA bulk staging of the model tables (tile and sweep variants)
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

// Law table entry, one 16-byte load:
//   u0 = s0 | kind << 16 | hill << 31, u1 = s1 (both species indices are valid:
//   unused slots repeat s0), c = rate.  kind: 0 h = 1, 1 h = x0, 2 h = x0(x0-1)/2,
//   3 h = x0 x1, 4 general (order 3-4: C(x0,st0) C(x1,st1) in int64; st in u1 >> 16).
struct __align__(16) SmcLaw {
    unsigned u0;
    unsigned u1;
    double c;
};

#ifdef SMC_SWEEP
// (double)h for 0 <= h < 2^52, exact: the bit pattern 0x43300000:h is 2^52 + h
__device__ __forceinline__ double smc_u2d(smc_u64 h) {
    return __dadd_rn(__longlong_as_double((long long)(h | 0x4330000000000000ull)), -0x1p52);
}
// x[s] of this thread's trajectory in the sweep variant: a shared-memory column with
// stride SMC_BLOCK, so lane l always hits bank(s) l mod 32 (conflict-free for any s)
#if SMC_SW_XD
typedef double smc_xt;          // counts as binary64 (exact integers < 2^31)
#else
typedef int smc_xt;
#endif
struct SmcXCol {
    smc_xt* p;
    __device__ __forceinline__ smc_xt operator[](int s) const { return p[s * SMC_BLOCK]; }
};
#endif
