// runtime.cpp -- the round driver: device buffers (through the allocator
// hook), launch configuration of the persistent kernels, shard slices,
// counters, the allreduce hook, and the iterative Wilson loop of Fig. 2.
#include <cuda_runtime.h>
#include <mutex>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>

#include "smc_internal.hpp"

// AOT kernel launcher (aot_kernels.cu)
cudaError_t smc_launch_philox_debug(uint64_t seed, uint64_t traj, uint64_t step0, uint32_t n, uint32_t* dev_out,
                                    cudaStream_t stream);
cudaError_t smc_launch_draw_debug(uint64_t seed, uint64_t traj, uint64_t step0, uint32_t n, double* dev_out,
                                  cudaStream_t stream);
struct SmcWState {               // aot_kernels.cu (device-resident Fig. 2 rounds)
    unsigned long long cursor;
    long long n_tot, yes, events, errors, N;
    int rounds, status;
    double p_hat;
};
cudaError_t smc_launch_wilson_rounds(const unsigned char* v, const int* e, uint64_t begin, uint64_t end,
                                     const SmcWState* st, double z, double eps, SmcWState* out,
                                     cudaStream_t stream);
cudaError_t smc_launch_count_range(const unsigned char* v, const int* e, uint64_t n, long long* counters,
                                   cudaStream_t stream);

namespace smc {

Hooks& hooks() {
    static Hooks h;
    return h;
}

namespace {

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(SMC_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
cudaStream_t stream() { return (cudaStream_t)hooks().stream; }

void* dalloc(size_t bytes) {
    Hooks& h = hooks();
    void* p = nullptr;
    if (h.alloc) {
        p = h.alloc(bytes, h.alloc_user);
        if (!p) fail(SMC_E_CUDA, "allocator hook returned NULL");
    } else {
        ck(cudaMalloc(&p, bytes), "cudaMalloc");
    }
    return p;
}
// Small pinned host blocks (the per-model count read-back and Wilson loop state) come
// from a process-wide pool: cudaMallocHost / cudaFreeHost cost ~1 ms each (and the free
// synchronises the device), which a user creating a model per query would pay every call.
constexpr size_t kPinnedBlock = 1024;
std::mutex g_pinned_mu;
std::vector<void*> g_pinned_free;
void* pinned_alloc(size_t bytes) {
    if (bytes > kPinnedBlock) fail(SMC_E_ARG, "internal: pinned block too large");
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    if (g_pinned_free.empty()) {
        constexpr size_t kSlab = 64;
        char* slab = nullptr;
        if (cudaMallocHost((void**)&slab, kSlab * kPinnedBlock) != cudaSuccess || !slab)
            fail(SMC_E_CUDA, "cudaMallocHost (pinned pool)");
        for (size_t i = 0; i < kSlab; ++i) g_pinned_free.push_back(slab + i * kPinnedBlock);
    }
    void* b = g_pinned_free.back();
    g_pinned_free.pop_back();
    std::memset(b, 0, kPinnedBlock);
    return b;
}
void pinned_free(void* b) {
    if (!b) return;
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    g_pinned_free.push_back(b);
}

void dfree(void* p) {
    if (!p) return;
    Hooks& h = hooks();
    if (h.free_) h.free_(p, h.alloc_user);
    else cudaFree(p);
}

}  // namespace

struct PropKernel {
    std::shared_ptr<Kernel> k;
    std::string source;
    int variant = 1;
    int block = 128;
    int grid_max = 0;
    int smem = 0;
    const void* tables = nullptr;
    bool timing_pending = false;
    int per_warp = 1;                      // trajectories per warp (variant 2)
    // window monitor (formulas outside the streaming templates, R27): per-slot rings
    double* lit_t = nullptr;               // all slots' rings
    unsigned long long lit_cap = 0;        // ring entries per replica slot of the current launch
    size_t lit_bytes = 0, lit_per_entry = 0, lit_small = 0;
    int lit_per_cta = 0;                   // replica slots per CTA (0: no window monitor)
    smc_launch_info info{};
    uint64_t cap_global = 0;               // sum of capacity() over the ranks (one allreduce)
    uint64_t capacity() const {            // trajectories resident at once on this GPU
        return (uint64_t)grid_max * (uint64_t)((variant != 2 && variant != 5) ? block : (block / 32) * per_warp);
    }
};

struct DeviceState {
    void* tables[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};   // per variant: [1] Hill, [2] tile, [4] sweep, [5] delta
    size_t table_bytes[6] = {0, 0, 0, 0, 0, 0};
    bool tables_ready[6] = {false, false, false, false, false, false};
    TileLayout layout;              // variant 2
    TileLayout sw_layout;           // variant 4
    TileLayout d_layout;            // variant 5
    void* ctl = nullptr;            // [0..8) cursor, [16..48) counters, [64..72) spec cursor, [80..112) spec scratch
    int64_t* host_counts = nullptr; // pinned
    // speculative batch of smc_estimate (prefix-exact rounds): this rank's slice [lo, hi)
    // of the batch [begin, end), per-replica verdicts/events at [i - lo]
    unsigned char* spec_v = nullptr;
    int* spec_e = nullptr;
    uint64_t spec_cap = 0, spec_begin = 0, spec_end = 0, spec_lo = 0, spec_hi = 0;
    bool spec_valid = false;
    bool spec_events_host = false;  // host_counts[10] holds the live batch's simulated events
    SmcWState* wst_dev = nullptr;   // device-resident Fig. 2 loop state
    SmcWState* wst_host = nullptr;  // pinned
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    int sm_count = 0, max_smem_optin = 0;
    uint64_t spec_max = 0;          // most replicas one rank's speculative batch may hold
    std::map<uint64_t, PropKernel> kernels;
    ~DeviceState() {
        for (auto& kv : kernels) {
            dfree(kv.second.lit_t);
        }
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        pinned_free(host_counts);
        pinned_free(wst_host);
        dfree(wst_dev);
        dfree(ctl);
        dfree(spec_v);
        dfree(spec_e);
        for (void* t : tables) dfree(t);
    }
    int64_t* counters() { return (int64_t*)((char*)ctl + 16); }
    unsigned long long* spec_cursor() { return (unsigned long long*)((char*)ctl + 64); }
    int64_t* spec_scratch() { return (int64_t*)((char*)ctl + 80); }
};

void DeviceStateDeleter::operator()(DeviceState* d) const { delete d; }

namespace {

DeviceState& device(Model& m) {
    if (!m.dev) {
        int n = 0;
        ck(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
        if (n < 1) fail(SMC_E_CUDA, "no CUDA device");
        auto d = std::make_unique<DeviceState>();
        int dev = 0;
        ck(cudaGetDevice(&dev), "cudaGetDevice");
        ck(cudaDeviceGetAttribute(&d->sm_count, cudaDevAttrMultiProcessorCount, dev), "attr");
        ck(cudaDeviceGetAttribute(&d->max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev), "attr");
        d->ctl = dalloc(128);
        d->host_counts = (int64_t*)pinned_alloc(128);
        ck(cudaEventCreate(&d->e0), "cudaEventCreate");
        ck(cudaEventCreate(&d->e1), "cudaEventCreate");
        // speculative per-replica buffers (1 byte verdict + 4 bytes events per replica) are
        // held to a quarter of the free memory and 8 GiB; a round needing more runs
        // non-speculatively into the counters (O(1) memory, identical counts)
        size_t free_b = 0, total_b = 0;
        ck(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
        d->spec_max = std::max<uint64_t>(1u << 20, std::min<uint64_t>(free_b / 4, (uint64_t)8 << 30) / 5);
        if (const char* e = std::getenv("SMC_SPEC_MAX")) d->spec_max = std::max<uint64_t>(1, std::strtoull(e, nullptr, 10));
        m.dev.reset(d.release());
    }
    return *m.dev;
}

// Rings of the window monitor (ssa_window.cuh, readings R23/R27), sized PER LAUNCH: every
// replica slot of the `grid` CTAs (`per_cta` slots each) gets W ring entries of
// `lit_per_entry` bytes (+ a small area for the single-position nodes), W the largest power of
// two up to SMC_WIN_W (default 32768) within the budget (60 % of the free device memory, at most
// 100 GiB: the B200's HBM holds C4's one-time-unit windows for every resident lane); a launch
// that cannot give every slot the full W runs down to half as many resident CTAs first, and one
// that cannot give every slot 1024 entries fewer still.  The rings hold the formula's windows
// (not the trace), so W bounds how many entries one window may span; a replica whose window
// would overflow its ring ends as an error.
void size_traces(Model& m, PropKernel& pk, int per_cta, int& grid) {
    (void)m;
    size_t free_b = 0, total_b = 0;
    ck(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
    const size_t held = pk.lit_bytes;                                  // ours, reusable
    const size_t budget = std::min<size_t>((size_t)((double)(free_b + held) * 0.6), (size_t)100 << 30);
    size_t want = 32768;
    if (const char* e = std::getenv("SMC_WIN_W")) want = std::max<size_t>(16, std::strtoull(e, nullptr, 10));
    int32_t g = grid;
    uint64_t cap = 0;
    if (smc_window_ring_plan(budget, pk.lit_per_entry, pk.lit_small, per_cta, grid, want, &g, &cap) != SMC_OK)
        fail(SMC_E_CUDA, "window monitor: not enough device memory for the rings");
    grid = g;
    const size_t need = (size_t)grid * (size_t)per_cta * ((size_t)cap * pk.lit_per_entry + pk.lit_small);
    if (need > pk.lit_bytes) {
        dfree(pk.lit_t);
        pk.lit_t = nullptr;
        pk.lit_bytes = 0;
        pk.lit_t = (double*)dalloc(need);
        pk.lit_bytes = need;
    }
    pk.lit_cap = cap;
}

PropKernel& prepare(Model& m, const Property& p) {
    DeviceState& d = device(m);
    auto it = d.kernels.find(p.id);
    if (it != d.kernels.end()) return it->second;
    m.build_deps();
    PropKernel pk;
    pk.variant = m.variant();
    // literal |= on the fly (reading R23): thread-owned models run variant 3, tile
    // models the tile kernel, both with the window monitor (R27)
    if (p.literal && pk.variant == 1) pk.variant = 3;
    // (the sweep is thread-owned and hosts the window monitor like variant 3; the delta kernel
    // does not, its formulas run the tile kernel)
    if (p.literal && pk.variant == 5) pk.variant = 2;
    const TileLayout* tl = nullptr;
    const int v = pk.variant == 3 ? 1 : pk.variant;      // table set (variant 3 uses variant 1's)
    if (!d.tables_ready[v]) {
        const void* src = nullptr;
        size_t bytes = 0;
        HillTables ht;
        if (v == 2) {
            d.layout = pack_tables(m);
            src = d.layout.blob.data();
            bytes = d.layout.bytes;
        } else if (v == 4) {
            d.sw_layout = pack_tables(m, true);
            src = d.sw_layout.blob.data();
            bytes = d.sw_layout.bytes;
        } else if (v == 5) {
            d.d_layout = pack_delta_tables(m);
            src = d.d_layout.blob.data();
            bytes = d.d_layout.bytes;
        } else {
            ht = pack_hill_tables(m);
            src = ht.values.data();
            bytes = ht.values.size() * sizeof(double);
        }
        if (bytes) {
            d.tables[v] = dalloc(bytes);
            ck(cudaMemcpyAsync(d.tables[v], src, bytes, cudaMemcpyHostToDevice, stream()), "upload tables");
            ck(cudaStreamSynchronize(stream()), "sync");
        }
        d.table_bytes[v] = bytes;
        d.tables_ready[v] = true;
    }
    if (v == 2) tl = &d.layout;
    if (v == 4) tl = &d.sw_layout;
    if (v == 5) tl = &d.d_layout;
    pk.tables = d.tables[v];
    pk.source = generate_source(m, p, pk.variant, tl);
    pk.k = get_kernel(pk.source, pk.variant == 1 ? "smc_ssa_thread"
                                 : (pk.variant == 2 ? "smc_ssa_tile"
                                                    : (pk.variant == 4 ? "smc_ssa_sweep"
                                                                       : (pk.variant == 5 ? "smc_ssa_delta" : "smc_ssa_literal"))));
    const void* fn = (const void*)pk.k->kernel;
    if (pk.variant == 3) {
        pk.block = 128;
        int nb = 0;
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, pk.block, 0), "occupancy");
        pk.grid_max = std::max(1, nb) * d.sm_count;
        pk.smem = 0;
        pk.lit_per_cta = pk.block;          // rings sized per launch (size_traces)
        pk.lit_per_entry = window_bytes_per_entry(p);
        pk.lit_small = window_small_bytes(p);
    } else if (pk.variant == 4) {
        pk.block = tl->sw_blk;
        if (p.literal) {                   // one window-monitor slot per thread (size_traces)
            pk.lit_per_cta = pk.block;
            pk.lit_per_entry = window_bytes_per_entry(p);
            pk.lit_small = window_small_bytes(p);
        }
        pk.smem = (int)(tl->bytes + (size_t)pk.block * (tl->sw_xd ? 8 : 4) * (size_t)(m.N + 1));
        cudaFuncAttributes fa;
        ck(cudaFuncGetAttributes(&fa, fn), "cudaFuncGetAttributes");
        if ((size_t)pk.smem + fa.sharedSizeBytes > (size_t)d.max_smem_optin)
            fail(SMC_E_CUDA, "sweep kernel: counts and tables do not fit in shared memory");
        ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, pk.smem), "smem attr");
        int nb = 0;
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, pk.block, (size_t)pk.smem), "occupancy");
        if (nb < 1) fail(SMC_E_CUDA, "sweep kernel: no resident CTA");
        pk.grid_max = nb * d.sm_count;
    } else if (pk.variant == 5) {
        // CTAs of SMC_DBLOCK threads (the compiled size); resident CTAs per SM from the
        // occupancy API under the shared-memory budget (tables + one slice per tile)
        // one CTA per SM: as many warps as the registers (the compiled bound) and the shared
        // memory (one copy of the tables + TPW slices per warp) allow
        cudaFuncAttributes fa;
        ck(cudaFuncGetAttributes(&fa, fn), "cudaFuncGetAttributes");
        pk.per_warp = 32 / tl->tw;
        const size_t wb = (size_t)pk.per_warp * tl->tile_bytes;
        const size_t avail = (size_t)d.max_smem_optin - fa.sharedSizeBytes;
        const size_t tb = tl->smem_bytes;              // the staged part of the tables
        if (tb + wb > avail) fail(SMC_E_CUDA, "delta kernel: tables and one warp's slices do not fit in shared memory");
        const int W = (int)std::min<size_t>((size_t)fa.maxThreadsPerBlock / 32, (avail - tb) / wb);
        pk.block = W * 32;
        pk.smem = (int)(tb + (size_t)W * wb);
        ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, pk.smem), "smem attr");
        int nb = 0;
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, pk.block, (size_t)pk.smem), "occupancy");
        if (nb < 1) fail(SMC_E_CUDA, "delta kernel: no resident CTA");
        pk.grid_max = nb * d.sm_count;
    } else if (pk.variant == 1) {
        pk.block = thread_block(m);
        int nb = 0;
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, pk.block, 0), "occupancy");
        pk.grid_max = std::max(1, nb) * d.sm_count;
        pk.smem = 0;
    } else {
        const size_t wb = tl->tile_bytes * (size_t)(32 / tl->tw);   // smem per warp
        cudaFuncAttributes fa;
        ck(cudaFuncGetAttributes(&fa, fn), "cudaFuncGetAttributes");
        const size_t max_dyn = (size_t)d.max_smem_optin - fa.sharedSizeBytes;
        ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_dyn), "smem attr");
        int best_total = 0, best_w = 0, best_nb = 0;
        int wmax = 24;                     // <= 768 threads (__launch_bounds__ of smc_ssa_tile)
        if (const char* e = std::getenv("SMC_TILE_WARPS")) wmax = std::max(1, std::min(24, std::atoi(e)));
        for (int W = wmax; W >= 1; --W) {
            size_t smem = tl->bytes + (size_t)W * wb;
            if (smem > max_dyn) continue;
            int nb = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, W * 32, smem) != cudaSuccess) continue;
            if (nb * W > best_total) { best_total = nb * W; best_w = W; best_nb = nb; }
        }
        if (!best_total) fail(SMC_E_CUDA, "tile kernel: model tables do not fit in shared memory");
        pk.block = best_w * 32;
        pk.smem = (int)(tl->bytes + (size_t)best_w * wb);
        pk.grid_max = best_nb * d.sm_count;
        pk.per_warp = 32 / tl->tw;
        if (p.literal) {                   // one ring slot per tile, sized per launch (size_traces)
            pk.lit_per_cta = best_w * pk.per_warp;
            pk.lit_per_entry = window_bytes_per_entry(p);
            pk.lit_small = window_small_bytes(p);
        }
    }
    pk.info.variant = pk.variant;
    pk.info.block_threads = pk.block;
    pk.info.smem_bytes = pk.smem;
    pk.info.regs_per_thread = pk.k->regs;
    pk.info.compile_ms = pk.k->compile_ms;
    pk.info.table_bytes = (double)d.table_bytes[v];
    return d.kernels.emplace(p.id, std::move(pk)).first->second;
}

// Launch one slice asynchronously on the stream; counters stay on the device.
// spec: cursor / counters of the speculative control block (the round counters are
// then filled by smc_count_range), else the main block (zeroed here).
void launch_slice(Model& m, PropKernel& pk, uint64_t seed, uint64_t lo, uint64_t hi, uint8_t* dev_verdict,
                  int32_t* dev_events, bool spec = false) {
    DeviceState& d = *m.dev;
    if (spec) ck(cudaMemsetAsync((char*)d.ctl + 64, 0, 64, stream()), "memset spec block");
    else ck(cudaMemsetAsync(d.ctl, 0, 64, stream()), "memset counters");
    if (hi <= lo) return;
    const uint64_t count = hi - lo;
    struct Params {
        unsigned long long seed, first, count;
        unsigned long long* cursor;
        long long* counters;
        unsigned char* verdicts;
        int* events_out;
        unsigned long long event_cap;
        const void* tables;
        double* lit_t;
        double* lit_tau;
        unsigned* lit_mask;
        unsigned char* lit_val;
        unsigned long long lit_cap;
    } P{seed, lo, count, spec ? d.spec_cursor() : (unsigned long long*)d.ctl,
        (long long*)(spec ? d.spec_scratch() : d.counters()), dev_verdict, dev_events, m.event_cap, pk.tables,
        pk.lit_t, nullptr, nullptr, nullptr, pk.lit_cap};
    // thread and sweep variants, slice smaller than the resident capacity: one CTA per SM with just
    // enough warps for the slice (the compiled CTA size is an upper bound), so a small
    // batch spreads over every SM instead of filling a few
    int block = pk.block;
    if ((pk.variant == 1 || pk.variant == 4) && count < pk.capacity()) {   // (sweep: the column stride stays)
        const uint64_t per_sm = (count + (uint64_t)d.sm_count - 1) / (uint64_t)d.sm_count;
        block = (int)std::min<uint64_t>((uint64_t)pk.block, std::max<uint64_t>(32, (per_sm + 31) / 32 * 32));
    }
    const uint64_t per_block = (pk.variant != 2 && pk.variant != 5) ? (uint64_t)block
                                                                    : (uint64_t)(pk.block / 32 * pk.per_warp);
    const uint64_t need = (count + per_block - 1) / per_block;
    int grid = (int)std::min<uint64_t>((uint64_t)pk.grid_max, need);
    if (pk.lit_per_cta) {                  // literal |=: this launch's trace buffers
        size_traces(m, pk, pk.lit_per_cta, grid);
        P.lit_t = pk.lit_t;
        P.lit_cap = pk.lit_cap;
    }
    void* args[] = {&P};
    ck(cudaEventRecord(d.e0, stream()), "event");
    ck(cudaLaunchKernel((const void*)pk.k->kernel, dim3((unsigned)grid), dim3((unsigned)block), args,
                        (size_t)pk.smem, stream()),
       "cudaLaunchKernel");
    ck(cudaEventRecord(d.e1, stream()), "event");
    pk.info.grid_blocks = grid;
    pk.info.block_threads = block;
    pk.info.launches += 1;
    pk.timing_pending = true;
}

void finish_timing(Model& m, PropKernel& pk, bool = true) {
    if (!pk.timing_pending) return;
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, m.dev->e0, m.dev->e1), "cudaEventElapsedTime");
    pk.info.kernel_ms += ms;
    pk.timing_pending = false;
}

void read_counts(Model& m, PropKernel& pk, smc_counts* out) {
    Hooks& h = hooks();
    if (h.allreduce) {
        if (h.allreduce(m.dev->counters(), 4, h.allreduce_user) != 0) fail(SMC_E_COMM, "allreduce hook failed");
    }
    // counters [16, 48) and, in the same copy, the speculative batch's own counters [80, 112)
    ck(cudaMemcpyAsync(m.dev->host_counts, m.dev->counters(), 96, cudaMemcpyDeviceToHost, stream()), "D2H counts");
    ck(cudaStreamSynchronize(stream()), "cudaStreamSynchronize");
    finish_timing(m, pk);
    m.dev->spec_events_host = m.dev->spec_valid;   // host_counts[10] = events of the live batch
    out->n_true = m.dev->host_counts[0];
    out->n_false = m.dev->host_counts[1];
    out->events = m.dev->host_counts[2];
    out->errors = m.dev->host_counts[3];
}

// Events simulated by the previous speculative batch (its own counters, which no
// round reads) -> launch info; called before the next batch reuses them and at the end.
void harvest_spec_events(Model& m, PropKernel& pk) {
    DeviceState& d = *m.dev;
    if (!d.spec_valid) return;
    int64_t ev = 0;
    if (d.spec_events_host) {                       // read with the last round's counts
        ev = d.host_counts[10];
    } else {
        ck(cudaMemcpyAsync(&ev, d.spec_scratch() + 2, 8, cudaMemcpyDeviceToHost, stream()), "D2H spec events");
        ck(cudaStreamSynchronize(stream()), "cudaStreamSynchronize");
    }
    pk.info.sim_events += (double)ev;
    d.spec_valid = false;
    d.spec_events_host = false;
}

// Sum of the ranks' resident capacities (world > 1): one allreduce of int64[4] through the
// hook, once per property.  Every rank must size speculative batches from the same number.
void global_capacity(Model& m, PropKernel& pk) {
    Hooks& h = hooks();
    if (h.world <= 1 || pk.cap_global) return;
    DeviceState& d = *m.dev;
    d.host_counts[0] = (int64_t)pk.capacity();
    d.host_counts[1] = d.host_counts[2] = d.host_counts[3] = 0;
    ck(cudaMemcpyAsync(d.counters(), d.host_counts, 32, cudaMemcpyHostToDevice, stream()), "H2D capacity");
    if (h.allreduce && h.allreduce(d.counters(), 4, h.allreduce_user) != 0) fail(SMC_E_COMM, "allreduce hook failed");
    ck(cudaMemcpyAsync(d.host_counts, d.counters(), 32, cudaMemcpyDeviceToHost, stream()), "D2H capacity");
    ck(cudaStreamSynchronize(stream()), "cudaStreamSynchronize");
    pk.cap_global = (uint64_t)std::max<int64_t>(1, d.host_counts[0]);
}

// Launch a speculative batch starting at replica `covered`: at least `need` replicas,
// else as many as all GPUs hold at once, never past the conservative size `limit`.
// S depends only on values every rank shares (need, limit, the allreduced capacity sum and
// the budget), so the ranks' slices tile [covered, covered + S) exactly.
void launch_batch(Model& m, PropKernel& pk, uint64_t seed, uint64_t covered, uint64_t need, uint64_t limit) {
    DeviceState& d = *m.dev;
    Hooks& h = hooks();
    const uint64_t cap_all = h.world > 1 ? pk.cap_global : pk.capacity();
    const uint64_t room = limit > covered ? limit - covered : 0;
    const uint64_t S = std::max(need, std::min(std::min(cap_all, room), d.spec_max * (uint64_t)h.world));
    uint64_t lo = covered, hi = covered + S;
    if (h.world > 1) smc_shard_range(covered, S, h.rank, h.world, &lo, &hi);
    if (hi - lo > d.spec_cap) {
        dfree(d.spec_v);
        dfree(d.spec_e);
        d.spec_v = nullptr;
        d.spec_e = nullptr;
        d.spec_cap = 0;
        const uint64_t c = hi - lo;
        d.spec_v = (unsigned char*)dalloc(c);
        d.spec_e = (int*)dalloc(4 * c);
        d.spec_cap = c;
    }
    harvest_spec_events(m, pk);
    launch_slice(m, pk, seed, lo, hi, d.spec_v, d.spec_e, true);
    ck(cudaGetLastError(), "kernel launch");
    d.spec_begin = covered;
    d.spec_end = covered + S;
    d.spec_lo = lo;
    d.spec_hi = hi;
    d.spec_valid = true;
}

// Prefix-exact speculative round.  The counts of the round
// range [base, base+n) are summed from per-replica results; when the range is not
// covered by the current batch, a new batch starting at the first uncovered index
// is launched with S = max(need, min(capacity of all GPUs, limit - start))
// replicas.  Fig. 2 only ever consumes prefixes of the index stream and every
// index is simulated exactly once by exactly one rank, so the counts -- and the
// estimate -- are identical to the non-speculative rounds; replicas past the
// final N_tot are simulated but never counted.
void spec_round(Model& m, PropKernel& pk, uint64_t seed, uint64_t base, uint64_t n, uint64_t limit, smc_counts* out) {
    DeviceState& d = *m.dev;
    const uint64_t end = base + n;
    ck(cudaMemsetAsync(d.ctl, 0, 64, stream()), "memset counters");
    auto count = [&](uint64_t a, uint64_t b) {       // [a, b) within this rank's slice of the batch
        a = std::max(a, d.spec_lo);
        b = std::min(b, d.spec_hi);
        if (b > a) {
            ck(smc_launch_count_range(d.spec_v + (a - d.spec_lo), d.spec_e + (a - d.spec_lo), b - a,
                                      (long long*)d.counters(), stream()),
               "count kernel");
            pk.info.aux_launches += 1;
        }
    };
    uint64_t covered = base;
    if (d.spec_valid && base >= d.spec_begin && base < d.spec_end) {
        count(base, std::min(end, d.spec_end));
        covered = std::min(end, d.spec_end);
    }
    if (covered < end) {
        launch_batch(m, pk, seed, covered, end - covered, limit);
        count(covered, end);
    }
    read_counts(m, pk, out);
}

}  // namespace

int run_round(Model& m, const Property& p, uint64_t seed, uint64_t base, uint64_t n, smc_counts* out) {
    PropKernel& pk = prepare(m, p);
    Hooks& h = hooks();
    uint64_t lo = base, hi = base + n;
    if (h.world > 1) smc_shard_range(base, n, h.rank, h.world, &lo, &hi);
    launch_slice(m, pk, seed, lo, hi, nullptr, nullptr);
    ck(cudaGetLastError(), "kernel launch");
    read_counts(m, pk, out);
    pk.info.sim_events += (double)out->events / (double)h.world;   // this GPU's share (equal slices)
    return SMC_OK;
}

// ------------------------------------------------------------ Fig. 2 ---
namespace {
// The Fig. 2 loop over any round runner (global counts).
// One Fig. 2 step after a round's counts; the device twin is
// smc_wilson_rounds() in aot_kernels.cu (same operations, same order).
void wilson_host_step(SmcWState& w, const smc_counts& c, double eps, double z) {
    // every replica of the round gives exactly one verdict or error on exactly one rank:
    // a mis-tiled shard (or a failed reduction) shows up here and fails loudly
    if (c.n_true < 0 || c.n_false < 0 || c.errors < 0 || c.n_true + c.n_false + c.errors != w.N) {
        w.status = 3;
        return;
    }
    w.cursor += (unsigned long long)w.N;
    w.n_tot += c.n_true + c.n_false;                     // errors excluded from trials
    w.yes += c.n_true;
    w.events += c.events;
    w.errors += c.errors;
    w.rounds += 1;
    if ((double)w.errors > 0.01 * (double)w.cursor) { w.status = 2; return; }
    if (w.n_tot == 0) { w.N = 1; return; }
    const double p_est = (double)w.yes / (double)w.n_tot;   // "pest = yess" (reading W2)
    w.p_hat = p_est;
    const double p_prime = round_estimate(p_est, eps);
    const int64_t n_new = wilson_sample_size(p_prime, eps, z) - w.n_tot;
    if (n_new > 0) w.N = n_new;
    else w.status = 1;
}

// loop state -> smc_estimate_t; the interval of a finished loop (Eq. 3 at p_hat, N_tot)
void wilson_state_out(const SmcWState& w, smc_estimate_t* out) {
    out->events = w.events;
    out->errors = w.errors;
    out->rounds = w.rounds;
    out->n_total = w.n_tot;
    out->n_true = w.yes;
    out->p_hat = w.p_hat;
}
int wilson_finish(const SmcWState& w, double z, smc_estimate_t* out) {
    wilson_state_out(w, out);
    if (w.status == 2) {
        set_error("more than 1% of replicas ended in error (overflow / event cap / bad propensity)");
        return SMC_E_ERRRATE;
    }
    if (w.status == 3) {
        set_error("a round's counts do not add up to its replica count (shards or reduction inconsistent)");
        return SMC_E_COMM;
    }
    if (w.status != 1) {
        set_error("Wilson loop did not terminate");
        return SMC_E_ARG;
    }
    wilson_interval(w.p_hat, (double)w.n_tot, z, &out->lower, &out->upper);
    return SMC_OK;
}

// The Fig. 2 loop over any round runner (global counts).
template <class Runner>
int wilson_loop(Runner&& run, double confidence, double eps, double start, smc_estimate_t* out) {
    std::memset(out, 0, sizeof *out);
    const double z = normal_quantile(confidence);
    out->z = z;
    SmcWState w{};
    w.N = wilson_sample_size(start, eps, z);             // "N = Wilson_Sample(1, epsilon, alpha)"
    while (w.status == 0 && w.rounds < 100000) {
        smc_counts c{};
        int rc = run(w.cursor, (uint64_t)w.N, &c);       // "Perform N experiments"
        if (rc != SMC_OK) {
            wilson_state_out(w, out);                    // partial state
            return rc;
        }
        wilson_host_step(w, c, eps, z);
    }
    return wilson_finish(w, z, out);
}

// Device-resident Fig. 2 loop (one GPU): after each speculative
// batch, smc_wilson_rounds consumes every round the batch covers and the host reads the
// loop state once.  A round only partly covered by the live batch is run on the host
// (spec_round: counts the covered part, launches the next batch).  Identical results to
// wilson_loop (test_speculative_rounds_identical).
int device_estimate(Model& m, const Property& p, PropKernel& pk, uint64_t seed, double confidence, double eps,
                    double start, uint64_t limit, smc_estimate_t* out) {
    std::memset(out, 0, sizeof *out);
    const double z = normal_quantile(confidence);
    out->z = z;
    DeviceState& d = *m.dev;
    if (!d.wst_dev) {
        d.wst_dev = (SmcWState*)dalloc(sizeof(SmcWState));
        d.wst_host = (SmcWState*)pinned_alloc(sizeof(SmcWState));
    }
    SmcWState w{};
    w.N = wilson_sample_size(start, eps, z);
    while (w.status == 0 && w.rounds < 100000) {
        const uint64_t end = w.cursor + (uint64_t)w.N;
        if ((uint64_t)w.N > d.spec_max && !(d.spec_valid && w.cursor >= d.spec_begin && end <= d.spec_end)) {
            harvest_spec_events(m, pk);                  // round too big to buffer: counters only
            smc_counts c{};
            run_round(m, p, seed, w.cursor, (uint64_t)w.N, &c);
            wilson_host_step(w, c, eps, z);
            continue;
        }
        if (!(d.spec_valid && w.cursor >= d.spec_begin && end <= d.spec_end)) {
            if (d.spec_valid && w.cursor >= d.spec_begin && w.cursor < d.spec_end) {
                smc_counts c{};
                spec_round(m, pk, seed, w.cursor, (uint64_t)w.N, limit, &c);
                wilson_host_step(w, c, eps, z);
                continue;
            }
            launch_batch(m, pk, seed, w.cursor, (uint64_t)w.N, limit);
        }
        ck(smc_launch_wilson_rounds(d.spec_v, d.spec_e, d.spec_begin, d.spec_end, &w, z, eps, d.wst_dev, stream()),
           "wilson rounds kernel");
        pk.info.aux_launches += 1;
        ck(cudaMemcpyAsync(d.wst_host, d.wst_dev, sizeof(SmcWState), cudaMemcpyDeviceToHost, stream()), "D2H state");
        ck(cudaMemcpyAsync(d.host_counts + 10, d.spec_scratch() + 2, 8, cudaMemcpyDeviceToHost, stream()),
           "D2H spec events");
        ck(cudaStreamSynchronize(stream()), "cudaStreamSynchronize");
        finish_timing(m, pk);
        d.spec_events_host = true;
        w = *d.wst_host;
    }
    return wilson_finish(w, z, out);
}

int guard(const std::function<int()>& f) {
    try {
        return f();
    } catch (const Error& e) {
        set_error(e.msg);
        return e.code;
    } catch (const std::exception& e) {
        set_error(e.what());
        return SMC_E_ARG;
    }
}
}  // namespace

}  // namespace smc

using namespace smc;

extern "C" {

int smc_set_allocator(void* (*alloc)(size_t, void*), void (*free_)(void*, void*), void* user) {
    if ((alloc == nullptr) != (free_ == nullptr)) { set_error("smc_set_allocator: set both or neither"); return SMC_E_ARG; }
    hooks().alloc = alloc;
    hooks().free_ = free_;
    hooks().alloc_user = user;
    return SMC_OK;
}
int smc_set_stream(void* s) { hooks().stream = s; return SMC_OK; }
int smc_set_shard(int32_t rank, int32_t world) {
    if (world < 1 || rank < 0 || rank >= world) { set_error("smc_set_shard: need 0 <= rank < world"); return SMC_E_ARG; }
    hooks().rank = rank;
    hooks().world = world;
    return SMC_OK;
}
int smc_set_allreduce(int (*fn)(int64_t*, int32_t, void*), void* user) {
    hooks().allreduce = fn;
    hooks().allreduce_user = user;
    return SMC_OK;
}

int smc_reset(smc_model* h) {
    if (!h) { set_error("smc_reset: NULL"); return SMC_E_ARG; }
    std::lock_guard<std::mutex> lk(h->m.mu);
    h->m.cursor = 0;
    return SMC_OK;
}

int smc_set_cursor(smc_model* h, uint64_t cursor, uint64_t seed) {
    if (!h) { set_error("smc_set_cursor: NULL"); return SMC_E_ARG; }
    std::lock_guard<std::mutex> lk(h->m.mu);
    h->m.cursor = cursor;
    h->m.last_seed = seed;
    h->m.has_seed = true;
    return SMC_OK;
}

int smc_run(smc_model* h, const smc_property* ph, uint64_t n, uint64_t seed, smc_counts* out) {
    if (!h || !ph || !out) { set_error("smc_run: NULL argument"); return SMC_E_ARG; }
    if (ph->p->N != h->m.N) { set_error("smc_run: property compiled for a model with another species count"); return SMC_E_ARG; }
    return guard([&] {
        Model& m = h->m;
        std::lock_guard<std::mutex> lk(m.mu);
        if (!m.has_seed || m.last_seed != seed) { m.cursor = 0; m.last_seed = seed; m.has_seed = true; }
        PropKernel& pk = prepare(m, *ph->p);
        pk.info.launches = 0;
        pk.info.aux_launches = 0;
        pk.info.sim_events = 0.0;
        pk.info.kernel_ms = 0.f;
        int rc = run_round(m, *ph->p, seed, m.cursor, n, out);
        if (rc == SMC_OK) m.cursor += n;
        return rc;
    });
}

int smc_estimate(smc_model* h, const smc_property* ph, double confidence, double half_width, uint64_t seed,
                 smc_estimate_t* out) {
    return smc_estimate_ex(h, ph, confidence, half_width, 1.0, seed, out);
}

int smc_estimate_ex(smc_model* h, const smc_property* ph, double confidence, double half_width, double start,
                    uint64_t seed, smc_estimate_t* out) {
    if (!h || !ph || !out || !(confidence > 0 && confidence < 1) || !(half_width > 0 && half_width < 0.5) ||
        !(start >= 0.0 && start <= 1.0)) {
        set_error("smc_estimate: need model, property, out, confidence in (0,1), half_width in (0,0.5), "
                  "start in [0,1]");
        return SMC_E_ARG;
    }
    if (ph->p->N != h->m.N) { set_error("smc_estimate: property compiled for a model with another species count"); return SMC_E_ARG; }
    return guard([&] {
        Model& m = h->m;
        std::lock_guard<std::mutex> lk(m.mu);
        PropKernel& pk = prepare(m, *ph->p);
        pk.info.launches = 0;
        pk.info.aux_launches = 0;
        pk.info.sim_events = 0.0;
        pk.info.kernel_ms = 0.f;
        m.dev->spec_valid = false;
        // no Fig. 2 round can reach past the conservative size Eq. 4(0.5) (N' <= Eq. 4(0.5))
        const uint64_t limit = (uint64_t)wilson_sample_size(0.5, half_width, normal_quantile(confidence));
        const bool speculate = m.speculate;
        if (speculate && hooks().world == 1) {
            const int rc = device_estimate(m, *ph->p, pk, seed, confidence, half_width, start, limit, out);
            harvest_spec_events(m, pk);
            return rc;
        }
        if (speculate) global_capacity(m, pk);
        const uint64_t world = (uint64_t)hooks().world;
        int rc = wilson_loop(
            [&](uint64_t base, uint64_t n, smc_counts* c) {
                const bool covered = m.dev->spec_valid && base >= m.dev->spec_begin && base + n <= m.dev->spec_end;
                if (speculate && (covered || n <= m.dev->spec_max * world)) {
                    spec_round(m, pk, seed, base, n, limit, c);
                    return (int)SMC_OK;
                }
                harvest_spec_events(m, pk);
                return run_round(m, *ph->p, seed, base, n, c);
            },
            confidence, half_width, start, out);
        harvest_spec_events(m, pk);
        return rc;
    });
}

int smc_estimate_with_runner(smc_run_fn run, void* user, double confidence, double half_width, double start,
                             smc_estimate_t* out) {
    if (!run || !out || !(confidence > 0 && confidence < 1) || !(half_width > 0 && half_width < 0.5) ||
        !(start >= 0 && start <= 1)) {
        set_error("smc_estimate_with_runner: bad arguments");
        return SMC_E_ARG;
    }
    return guard([&] {
        return wilson_loop(
            [&](uint64_t base, uint64_t n, smc_counts* c) -> int {
                Hooks& hk = hooks();
                uint64_t lo = base, hi = base + n;
                if (hk.world > 1) smc_shard_range(base, n, hk.rank, hk.world, &lo, &hi);
                smc_counts local{};
                if (hi > lo) {
                    int rc = run(lo, hi - lo, user, &local);
                    if (rc != 0) { set_error("runner callback failed"); return SMC_E_ARG; }
                }
                int64_t buf[4] = {local.n_true, local.n_false, local.events, local.errors};
                // with a runner the counts live in HOST memory; the hook sums them in place
                if (hk.allreduce && hk.allreduce(buf, 4, hk.allreduce_user) != 0) {
                    set_error("allreduce hook failed");
                    return SMC_E_COMM;
                }
                c->n_true = buf[0];
                c->n_false = buf[1];
                c->events = buf[2];
                c->errors = buf[3];
                return SMC_OK;
            },
            confidence, half_width, start, out);
    });
}

int smc_run_verdicts(smc_model* h, const smc_property* ph, uint64_t first, uint64_t n, uint64_t seed,
                     uint8_t* dev_verdict, int32_t* dev_events) {
    if (!h || !ph || !dev_verdict || !dev_events) { set_error("smc_run_verdicts: NULL argument"); return SMC_E_ARG; }
    if (ph->p->N != h->m.N) { set_error("smc_run_verdicts: property compiled for a model with another species count"); return SMC_E_ARG; }
    return guard([&] {
        Model& m = h->m;
        std::lock_guard<std::mutex> lk(m.mu);
        PropKernel& pk = prepare(m, *ph->p);
        pk.info.launches = 0;
        pk.info.aux_launches = 0;
        pk.info.sim_events = 0.0;
        pk.info.kernel_ms = 0.f;
        launch_slice(m, pk, seed, first, first + n, dev_verdict, dev_events);
        ck(cudaGetLastError(), "kernel launch");
        ck(cudaStreamSynchronize(stream()), "cudaStreamSynchronize");
        finish_timing(m, pk, n > 0);
        return SMC_OK;
    });
}

int smc_philox_blocks(uint64_t seed, uint64_t trajectory, uint64_t step0, uint32_t n, uint32_t* host_out) {
    if (!host_out) { set_error("smc_philox_blocks: NULL"); return SMC_E_ARG; }
    return guard([&] {
        void* d = dalloc((size_t)n * 16 + 16);
        try {
            ck(smc_launch_philox_debug(seed, trajectory, step0, n, (uint32_t*)d, stream()), "philox kernel");
            ck(cudaMemcpyAsync(host_out, d, (size_t)n * 16, cudaMemcpyDeviceToHost, stream()), "D2H");
            ck(cudaStreamSynchronize(stream()), "sync");
        } catch (...) {
            dfree(d);
            throw;
        }
        dfree(d);
        return SMC_OK;
    });
}

int smc_draw_blocks(uint64_t seed, uint64_t trajectory, uint64_t step0, uint32_t n, double* host_out) {
    if (!host_out) { set_error("smc_draw_blocks: NULL"); return SMC_E_ARG; }
    return guard([&] {
        void* d = dalloc((size_t)n * 16 + 16);
        try {
            ck(smc_launch_draw_debug(seed, trajectory, step0, n, (double*)d, stream()), "draw kernel");
            ck(cudaMemcpyAsync(host_out, d, (size_t)n * 16, cudaMemcpyDeviceToHost, stream()), "D2H");
            ck(cudaStreamSynchronize(stream()), "sync");
        } catch (...) {
            dfree(d);
            throw;
        }
        dfree(d);
        return SMC_OK;
    });
}

int smc_last_launch(const smc_model* h, const smc_property* ph, smc_launch_info* out) {
    if (!h || !ph || !out) { set_error("smc_last_launch: NULL"); return SMC_E_ARG; }
    const Model& m = h->m;
    if (!m.dev) { set_error("smc_last_launch: no run yet"); return SMC_E_ARG; }
    auto it = m.dev->kernels.find(ph->p->id);
    if (it == m.dev->kernels.end()) { set_error("smc_last_launch: no run of this property"); return SMC_E_ARG; }
    *out = it->second.info;
    return SMC_OK;
}

int smc_kernel_source(smc_model* h, const smc_property* ph, char* buf, size_t* len) {
    if (!h || !ph || !len) { set_error("smc_kernel_source: NULL"); return SMC_E_ARG; }
    if (ph->p->N != h->m.N) { set_error("smc_kernel_source: property compiled for a model with another species count"); return SMC_E_ARG; }
    return guard([&] {
        Model& m = h->m;
        std::lock_guard<std::mutex> lk(m.mu);
        m.build_deps();
        const int mv = m.variant();
        const int v = (ph->p->literal && mv == 1) ? 3 : mv;
        TileLayout tl;
        const int vv = (ph->p->literal && v == 5) ? 2 : v;
        if (vv == 2 || vv == 4) tl = pack_tables(m, vv == 4);
        if (vv == 5) tl = pack_delta_tables(m);
        std::string s = generate_source(m, *ph->p, vv, (vv == 2 || vv == 4 || vv == 5) ? &tl : nullptr);
        size_t need = s.size() + 1;
        if (buf) std::memcpy(buf, s.c_str(), std::min(*len, need));
        *len = need;
        return SMC_OK;
    });
}

}  // extern "C"

// The window monitor's ring plan (smc.h; DESIGN R27).  Capacity before residency: a window
// that overflows its ring ends the replica as an error, fewer resident CTAs only cost time.
extern "C" int smc_window_ring_plan(uint64_t budget, uint64_t per_entry, uint64_t small, int32_t per_cta, int32_t grid,
                                    uint64_t want, int32_t* grid_out, uint64_t* cap_out) {
    if (per_entry == 0 || per_cta < 1 || grid < 1 || want < 1 || !grid_out || !cap_out) {
        set_error("smc_window_ring_plan: sizes and counts must be positive");
        return SMC_E_ARG;
    }
    uint64_t g = (uint64_t)grid;
    const uint64_t pc = (uint64_t)per_cta;
    const uint64_t g_fit = budget / ((want * per_entry + small) * pc);          // CTAs that get the full W
    if (g_fit < g) g = std::max<uint64_t>(g_fit, std::max<uint64_t>(1, g / 2));
    const uint64_t min_cap = std::min<uint64_t>(want, 1024);
    if (budget / (g * pc) < min_cap * per_entry + small)
        g = std::max<uint64_t>(1, budget / ((min_cap * per_entry + small) * pc));
    const uint64_t per_slot = budget / (g * pc);
    const uint64_t lim = per_slot > small ? std::min<uint64_t>((per_slot - small) / per_entry, want) : 0;
    uint64_t cap = 1;
    while (cap * 2 <= lim) cap *= 2;
    *grid_out = (int32_t)g;
    *cap_out = cap;
    if (lim < 16) {
        set_error("window monitor: not enough device memory for the rings");
        return SMC_E_CUDA;
    }
    return SMC_OK;
}
