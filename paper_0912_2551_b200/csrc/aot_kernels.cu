// aot_kernels.cu -- kernels compiled ahead of time into libsmc.so for sm_100a
// (the SSA kernels themselves are specialised per model at run time by NVRTC,
// see jit.cpp).  smc_philox_debug exports the device Philox stream so tests
// can check it bit for bit against the oracle (SURVEY §8(c) pin table).
#include <cstdint>

#include "kernels/ssa_common.cuh"

__global__ void smc_philox_debug(smc_u64 seed, smc_u64 traj, smc_u64 step0, smc_u32 n, smc_u32* out) {
    const smc_u32 q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const smc_u64 step = step0 + q;
    smc_u32 r[4];
    smc_philox((smc_u32)step, (smc_u32)(step >> 32), (smc_u32)traj, (smc_u32)(traj >> 32), (smc_u32)seed,
               (smc_u32)(seed >> 32), r);
    out[4 * q + 0] = r[0];
    out[4 * q + 1] = r[1];
    out[4 * q + 2] = r[2];
    out[4 * q + 3] = r[3];
}

__global__ void smc_draw_debug(smc_u64 seed, smc_u64 traj, smc_u64 step0, smc_u32 n, double* out) {
    const smc_u32 q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    double e, u2;
    smc_draw(seed, traj, step0 + q, e, u2);
    out[2 * q] = e;
    out[2 * q + 1] = u2;
}

// Counts of the replicas [i0, i1) of a speculative batch whose per-replica
// verdicts / event counts sit at v[i - base], e[i - base] (prefix-exact Wilson
// rounds).  Adds into counters {n_true, n_false, events, errors}.
__global__ void smc_count_range(const unsigned char* __restrict__ v, const int* __restrict__ e, smc_u64 n,
                                smc_i64* counters) {
    smc_i64 ct = 0, cf = 0, ce = 0, cr = 0;
    for (smc_u64 i = (smc_u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (smc_u64)gridDim.x * blockDim.x) {
        const unsigned char vv = v[i];
        ct += vv == 1;
        cf += vv == 0;
        cr += vv == 2;
        ce += e[i];
    }
    smc_flush_counts(ct, cf, ce, cr, counters);
}

cudaError_t smc_launch_count_range(const unsigned char* v, const int* e, uint64_t n, long long* counters,
                                   cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    const uint64_t blocks = (n + 255) / 256;
    smc_count_range<<<(unsigned)(blocks < 592 ? blocks : 592), 256, 0, stream>>>(v, e, n, counters);
    return cudaGetLastError();
}

cudaError_t smc_launch_philox_debug(uint64_t seed, uint64_t traj, uint64_t step0, uint32_t n, uint32_t* dev_out,
                                    cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    smc_philox_debug<<<(n + 127) / 128, 128, 0, stream>>>(seed, traj, step0, n, dev_out);
    return cudaGetLastError();
}

cudaError_t smc_launch_draw_debug(uint64_t seed, uint64_t traj, uint64_t step0, uint32_t n, double* dev_out,
                                  cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    smc_draw_debug<<<(n + 127) / 128, 128, 0, stream>>>(seed, traj, step0, n, dev_out);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Device-resident Fig. 2 rounds: after a
// speculative batch, one CTA consumes as many Wilson rounds as the batch covers
// (prefix counts of the per-replica verdicts, then the Wilson step) and writes
// the loop state back once -- no host round trip per round.  The arithmetic is
// the host's (wilson.cpp, reading W8) operation for operation in IEEE binary64,
// so the rounds, N_tot and p_hat are bit-identical to the host loop.
struct SmcWState {
    unsigned long long cursor;   // next replica index
    long long n_tot, yes, events, errors, N;
    int rounds, status;          // status: 0 next round not covered, 1 done, 2 error rate, 3 round cap
    double p_hat;
};

__device__ long long smc_ws_device(double p, double eps, double z) {      // Eq. 4, ceil, N >= 1
    const double zz = __dmul_rn(z, z);
    const double A = __dmul_rn(p, __dadd_rn(1.0, -p));
    const double d = __dadd_rn(p, -0.5);
    const double e2 = __dmul_rn(eps, eps);
    const double s = __dadd_rn(__dadd_rn(A, -__dmul_rn(2.0, e2)),
                               __dsqrt_rn(__dadd_rn(__dmul_rn(A, A), __dmul_rn(__dmul_rn(4.0, e2), __dmul_rn(d, d)))));
    const double val = __ddiv_rn(__dmul_rn(zz, s), __dmul_rn(2.0, e2));
    const long long N = (long long)ceil(val);
    return N < 1 ? 1 : N;
}

__global__ void __launch_bounds__(1024, 1) smc_wilson_rounds(const unsigned char* __restrict__ v,
                                                             const int* __restrict__ e, smc_u64 begin, smc_u64 end,
                                                             SmcWState st, double z, double eps, SmcWState* out) {
    __shared__ unsigned long long s_cnt[4];
    __shared__ SmcWState s_st;
    if (threadIdx.x == 0) s_st = st;
    __syncthreads();
    for (;;) {
        st = s_st;
        if (st.status != 0) break;
        if (st.rounds >= 100000) { if (threadIdx.x == 0) s_st.status = 3; break; }
        const smc_u64 a = st.cursor, b = st.cursor + (smc_u64)st.N;
        if (a < begin || b > end) break;                       // next round not covered by the batch
        if (threadIdx.x < 4) s_cnt[threadIdx.x] = 0ull;
        __syncthreads();
        smc_i64 ct = 0, cf = 0, ce = 0, cr = 0;
        for (smc_u64 i = a + threadIdx.x; i < b; i += blockDim.x) {
            const unsigned char vv = v[i - begin];
            ct += vv == 1;
            cf += vv == 0;
            cr += vv == 2;
            ce += e[i - begin];
        }
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
        if (threadIdx.x == 0) {                                // the Wilson step of wilson_loop()
            SmcWState w = s_st;
            w.cursor += (smc_u64)w.N;
            w.n_tot += (long long)(s_cnt[0] + s_cnt[1]);
            w.yes += (long long)s_cnt[0];
            w.events += (long long)s_cnt[2];
            w.errors += (long long)s_cnt[3];
            w.rounds += 1;
            if (__ll2double_rn(w.errors) > __dmul_rn(0.01, __ull2double_rn(w.cursor))) {
                w.status = 2;
            } else if (w.n_tot == 0) {
                w.N = 1;
            } else {
                const double p_est = __ddiv_rn(__ll2double_rn(w.yes), __ll2double_rn(w.n_tot));
                w.p_hat = p_est;
                const double p_prime = p_est <= 0.5 ? __dadd_rn(p_est, eps) : __dadd_rn(p_est, -eps);
                const long long n_new = smc_ws_device(p_prime, eps, z) - w.n_tot;
                if (n_new > 0) w.N = n_new;
                else w.status = 1;
            }
            s_st = w;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = s_st;
}

cudaError_t smc_launch_wilson_rounds(const unsigned char* v, const int* e, uint64_t begin, uint64_t end,
                                     const SmcWState* st, double z, double eps, SmcWState* out,
                                     cudaStream_t stream) {
    smc_wilson_rounds<<<1, 1024, 0, stream>>>(v, e, begin, end, *st, z, eps, out);
    return cudaGetLastError();
}
