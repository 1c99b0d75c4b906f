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

// The draw of SSA step `step` of trajectory `traj` ("standard Monte Carlo
// methods"):  e = -log(u1) (Eq. 2a numerator), u2 (Eq. 2b).
//   u1 = ((((r0<<32)|r1) >> 11) + 1) * 2^-53 in (0,1],  u2 = (((r2<<32)|r3) >> 11) * 2^-53 in [0,1)
__device__ __forceinline__ void smc_draw(smc_u64 seed, smc_u64 traj, smc_u64 step, double& e, double& u2) {
    smc_u32 r[4];
    smc_philox((smc_u32)step, (smc_u32)(step >> 32), (smc_u32)traj, (smc_u32)(traj >> 32), (smc_u32)seed,
               (smc_u32)(seed >> 32), r);
    const smc_u64 w1 = ((smc_u64)r[0] << 32) | r[1];
    const smc_u64 w2 = ((smc_u64)r[2] << 32) | r[3];
    const double u1 = __dmul_rn(__ull2double_rn((w1 >> 11) + 1ull), 0x1p-53);   // 2^-53, exact
    u2 = __dmul_rn(__ull2double_rn(w2 >> 11), 0x1p-53);
    e = -log(u1);
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
