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
