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

cudaError_t smc_launch_philox_debug(uint64_t seed, uint64_t traj, uint64_t step0, uint32_t n, uint32_t* dev_out,
                                    cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    smc_philox_debug<<<(n + 127) / 128, 128, 0, stream>>>(seed, traj, step0, n, dev_out);
    return cudaGetLastError();
}
