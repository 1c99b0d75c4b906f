/*
 * smc.h -- C ABI of libsmc.so, the B200-native hot path of the statistical
 * model checker of arXiv:0912.2551 (Ballarini, Forlin, Mazza, Prandi).
 *
 * Problem statement: given a CTMC model M of a
 * biochemical network, a BLTLc property phi and a desired confidence, estimate
 * P(phi) "with the estimated measure meeting the desired confidence".
 *
 * The path behind this ABI:
 *   batched Gillespie direct-method SSA trajectories on sm_100a,
 *   each checked on the fly against a time-bounded LTL formula and halted as
 *   soon as it is decided, true/false counts reduced per GPU and
 *   across GPUs, the Wilson interval and iterative stopping rule of
 *   Eq. 3 / Eq. 4 / Fig. 2 on the host.
 *
 * Conventions (all entry points):
 *   - Return status: SMC_OK (0) or a negative SMC_E_* code; never throws or
 *     aborts across the ABI.  smc_last_error() gives a thread-local message
 *     (parse position, all validation violations, CUDA/NVRTC log).
 *   - Ownership: input arrays are copied; the caller keeps them.  Handles are
 *     owned by the caller until *_destroy.  Outputs go to caller memory.
 *   - Device memory is obtained through the allocator hook (default
 *     cudaMalloc) and released in smc_model_destroy.  Kernels and copies run
 *     on the stream hook (default: the legacy default stream).
 *   - Units: times in model time units; counts are int32 on the device.
 *   - There is no CPU fallback: calls that need the GPU return SMC_E_CUDA
 *     when no sm_100 device is present.
 */
#ifndef SMC_H_
#define SMC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    SMC_OK = 0,
    SMC_E_ARG = -1,          /* bad argument (NULL, out of range)                         */
    SMC_E_MODEL = -2,        /* model validation failed (message lists every violation)   */
    SMC_E_PARSE = -3,        /* formula syntax / unknown species (message has position)   */
    SMC_E_UNSUPPORTED = -4,  /* formula outside the compiled fragment       */
    SMC_E_CUDA = -5,         /* CUDA runtime / NVRTC failure or no sm_100 device            */
    SMC_E_COMM = -6,         /* the allreduce hook returned non-zero                        */
    SMC_E_OVERFLOW = -7,     /* reserved: count overflow is a per-replica error (counted)  */
    SMC_E_EVENT_CAP = -8,    /* reserved: event cap is a per-replica error (counted)       */
    SMC_E_ERRRATE = -9       /* more than 1 % of replicas ended in error       */
};

/* Thread-local description of the last error on this thread. */
const char* smc_last_error(void);

/* ------------------------------------------------------------------------ */
/* Model: the CTMC M = (S, s0, Q, Var, Eval) of P:110-112, with Q implied by  */
/* reaction channels R_j: propensity a_j(x) and change v_j.       */
/* ------------------------------------------------------------------------ */
typedef struct smc_model smc_model;

/* n_species N >= 1, init_counts[N] >= 0 (the initial state s0),
 * n_reactions M >= 1.  Reaction j (row-major [M][2] arrays):
 *   reactant_idx[j][q] species index or -1 (none), reactant_st[j][q] in 1..2;
 *   product_idx[j][q]  species index or -1,        product_st[j][q]  in 1..2;
 *   rate[j] > 0: mass-action constant c_j, a_j = c_j * h_j(x) with
 *   h_j = prod over reactants of C(x_s, st_s) (x for st 1, x(x-1)/2 for st 2;
 *   P:141-143 and reading R8).  A species listed twice as reactant is merged
 *   (A + A == 2A); merged stoichiometry must be <= 2.
 * Null reactions (v_j = 0) are allowed and fire as events (reading G3).
 * The kernel variant (register-resident thread-owned, thread-owned sweep with
 * the counts in shared memory, or warp-owned tile) is chosen from (N, M); see
 * smc_model_set_variant.
 * Errors: SMC_E_ARG (NULL / sizes), SMC_E_MODEL (validation, all violations). */
int smc_model_create(int32_t n_species, const int32_t* init_counts,
                     int32_t n_reactions,
                     const int32_t* reactant_idx, const int32_t* reactant_st,
                     const int32_t* product_idx, const int32_t* product_st,
                     const double* rate, smc_model** out);

/* Hill repression on reaction j (reading R9):
 *   a_j = c_j h_j(x) / (1 + (x_r / K)^n),  q = x_r / K, q^n a left-to-right product.
 * K > 0, 1 <= n <= 8.  Must be called before the first run.  SMC_E_ARG otherwise. */
int smc_model_set_hill(smc_model* m, int32_t reaction, int32_t repressor, double K, int32_t n);

/* Explicit propensity for reaction j (Table 2),
 * replacing c_j h_j(x): an expression over species names (species_names[N],
 * NULL = S0..S{N-1}) and decimal constants with + - * /, unary minus and
 * parentheses, evaluated in IEEE binary64 in tree order (left-associative;
 * counts promoted to double).  The guard still applies: a_j = 0 while a
 * reactant count is below its stoichiometry.  A negative or NaN value is a
 * bad propensity (the replica ends as an error).  Not combinable with Hill.
 * Must be called before the first run.  SMC_E_PARSE (message with the
 * position) / SMC_E_ARG otherwise. */
int smc_model_set_rate_expr(smc_model* m, int32_t reaction, const char* expr, const char* const* species_names);

/* Force a kernel variant: 0 = automatic (1 for N, M <= 32; 4 for N <= 160,
 * M <= 1024; else 5 when eligible, else 2), 1 = thread-owned (registers;
 * requires N <= 32 and M <= 32), 2 = tile-owned (propensities and counts in
 * shared memory, dependency graph), 4 = thread-owned sweep (counts in a
 * shared-memory column, every law re-evaluated per event; requires the counts
 * of 128 trajectories to fit in shared memory), 5 = tile-owned delta kernel (no
 * stored propensities: exact 128-bit fixed-point group sums updated by the
 * dependency graph, reading R26; requires mass action of order <= 2 and rates
 * within ~2^20 of each other).  3 (buffered trace + literal |=) is not
 * selectable: it is chosen by the formula.  All variants compute the same
 * replicas up to the ulp-level summation orders of readings R12/R26 (DESIGN.md
 * §5).  Must be called before the first run (SMC_E_ARG afterwards, or if the
 * variant cannot hold the model). */
int smc_model_set_variant(smc_model* m, int32_t variant);

/* Per-replica event cap (default 2^31 - 1): a replica reaching it undecided is
 * counted as an error.  1 <= cap <= 2^31 - 1 (per-replica event
 * counts are int32 on the device).  Must be called before the first run. */
int smc_model_set_event_cap(smc_model* m, uint64_t cap);

/* smc_estimate runs each Fig. 2 round prefix-exactly from a speculative batch
 * (default on = 1): a round range not yet simulated starts a batch of
 * max(needed, min(resident capacity of all GPUs, Eq. 4(0.5) - start)) replicas
 * whose per-replica results later rounds consume by index.  Fig. 2 reads only
 * prefixes of the index stream, so the estimate is identical with 0 (off:
 * exactly the round's replicas per launch); only the time changes.  SMC_E_ARG on NULL. */
int smc_model_set_speculation(smc_model* m, int32_t on);

void smc_model_destroy(smc_model* m);

/* ------------------------------------------------------------------------ */
/* Property: a BLTLc formula compiled to a monitor program.       */
/* ------------------------------------------------------------------------ */
typedef struct smc_property smc_property;

/* formula: concrete syntax of reading R15:
 *   atoms      lin <|<=|>=|>|==|!= lin, lin integer-linear in species counts
 *   connectives ! & |   temporal X F G with interval, binary U with interval
 *   interval   [a,b] (a,b] [a,b) (a,b) [a,inf); omitted = [0,inf)
 *   precedence temporal unary > ! > & > U (right assoc.) > |
 * species_names: N names for the model's species, or NULL for S0..S{N-1}.
 * t_max: 0 = bounded formulas only; > 0 = cap for unbounded operators, an
 *   undecided replica at t_max counts as false (pessimistic).
 * Compiled fragment: a Kleene boolean combination of leaves
 *   beta, F^I beta, G^I beta, beta1 U^I beta2, X^I beta,
 *   F[0,a] G[0,b] beta, G[0,a] F[0,b] beta, (G[0,b] beta1) U[0,c] beta2,
 *   beta = boolean combination of atoms.
 * Errors: SMC_E_PARSE (message "col N: ..."), SMC_E_UNSUPPORTED, SMC_E_ARG. */
int smc_property_compile(const smc_model* m, const char* formula,
                         const char* const* species_names, double t_max,
                         smc_property** out);
void smc_property_destroy(smc_property* p);

/* ------------------------------------------------------------------------ */
/* Runs                                                                        */
/* ------------------------------------------------------------------------ */
typedef struct {
    int64_t n_true;    /* replicas whose verdict is true                        */
    int64_t n_false;   /* replicas whose verdict is false (incl. unknown at t_max) */
    int64_t events;    /* SSA reaction events applied, over all replicas          */
    int64_t errors;    /* replicas ended by overflow / event cap / bad propensity */
} smc_counts;

/* Replicas with trajectory indices [cursor, cursor + n) of the Philox stream
 * keyed by seed (reading R10); the model's cursor then advances by n.  The
 * cursor resets to 0 when seed differs from the previous call's.  With a
 * shard set (smc_set_shard) this rank runs its slice [lo, hi) of the range
 * and the counts are summed over ranks by the allreduce hook.
 * out: the (global) counts.  Errors: SMC_E_ARG (also: a property compiled for a
 * model with another species count), SMC_E_CUDA, SMC_E_COMM. */
int smc_run(smc_model* m, const smc_property* p, uint64_t n, uint64_t seed, smc_counts* out);

/* cursor <- 0 */
int smc_reset(smc_model* m);

/* Resume (SURVEY §5 checkpoint / resume): the next smc_run of this seed starts at
 * trajectory index `cursor`.  Because the Philox stream is keyed by (seed, trajectory,
 * step) (reading R10), a Fig. 2 loop interrupted after N_tot replicas continues exactly
 * where it stopped: its state {seed, N_tot, n_true, events, errors, rounds} is a complete
 * checkpoint.  SMC_E_ARG on NULL. */
int smc_set_cursor(smc_model* m, uint64_t cursor, uint64_t seed);

typedef struct {
    double p_hat, lower, upper;   /* estimate and Wilson interval (Eq. 3)       */
    int64_t n_total, n_true;      /* replicas used, successes                    */
    int64_t events;               /* SSA events over all rounds                  */
    int64_t errors;               /* replicas in error (excluded from n_total)   */
    int32_t rounds;               /* Fig. 2 iterations                           */
    double z;                     /* z_{1-alpha/2} used                          */
} smc_estimate_t;

/* Fig. 2: start estimate 1 (iterative), N = Eq. 4(1, eps),
 * run, p_hat = successes / N_tot, p' = p_hat +- eps toward 0.5, N' = Eq. 4(p'),
 * top up while N' > N_tot, return Eq. 3 at (p_hat, N_tot).  Always starts at
 * trajectory index 0, so the result is a pure function of (model, property,
 * confidence, half_width, seed) and of nothing else (not of the GPU count).
 * confidence = 1 - alpha in (0,1), half_width = eps in (0, 0.5).
 * On error after some rounds, out holds the partial state.
 * Every round's global counts must add up to its replica count (true + false +
 * errors == N), else SMC_E_COMM (mis-tiled shards or a failed reduction).
 * Speculative per-replica buffers are held to a quarter of the free device
 * memory and 8 GiB; a larger round runs non-speculatively (same result).
 * Errors: SMC_E_ARG, SMC_E_CUDA, SMC_E_COMM, SMC_E_ERRRATE. */
int smc_estimate(smc_model* m, const smc_property* p, double confidence, double half_width,
                 uint64_t seed, smc_estimate_t* out);

/* smc_estimate with the start estimate of the first round as an argument
 * (SURVEY §8(f) NEXT-4): start = 1.0 (or 0.0) is the iterative
 * method of Fig. 2 (smc_estimate), start = 0.5 the conservative sample size
 * Eq. 4(0.5) in one round (every later N' <= Eq. 4(0.5), so the loop stops
 * after it).  start in [0, 1]; other errors as smc_estimate. */
int smc_estimate_ex(smc_model* m, const smc_property* p, double confidence, double half_width,
                    double start, uint64_t seed, smc_estimate_t* out);

/* Same loop as smc_estimate with start estimate `start` (1.0 = iterative,
 * 0.5 = conservative) and the per-round replica runner supplied by the
 * caller (run(first, n, user, out) must return 0 and fill out with the counts
 * of replicas [first, first+n) of THIS rank's shard); the shard and allreduce
 * hooks apply exactly as in smc_estimate.  Host logic only: this is the seam
 * the multi-process CPU tests drive.  Errors as smc_estimate. */
typedef int (*smc_run_fn)(uint64_t first, uint64_t n, void* user, smc_counts* out);
int smc_estimate_with_runner(smc_run_fn run, void* user, double confidence, double half_width,
                             double start, smc_estimate_t* out);

/* ------------------------------------------------------------------------ */
/* Pure functions of §3.3 (bit-exact contract with the oracle, reading W8)    */
/* ------------------------------------------------------------------------ */
/* z_{1-alpha/2} = Phi^{-1}((1 + c)/2), the double nearest to the exact
 * quantile for the exact binary value of c (reading W1).  NaN if c not in (0,1). */
double smc_normal_quantile(double confidence);
/* Eq. 3 at p_hat = n_true / n, clamped to [0,1].  SMC_E_ARG if n < 1
 * or n_true not in [0, n]. */
int smc_wilson_interval(int64_t n_true, int64_t n, double confidence, double* lower, double* upper);
/* Eq. 4: smallest N >= the bound, N >= 1.  -1 on bad arguments. */
int64_t smc_wilson_sample_size(double p, double half_width, double confidence);
/* Rank r's slice [lo, hi) of the round range [base, base + n) over `world` ranks:
 * lo = base + floor(r n / world), hi = base + floor((r+1) n / world). */
int smc_shard_range(uint64_t base, uint64_t n, int32_t rank, int32_t world, uint64_t* lo, uint64_t* hi);
/* Ring plan of the window monitor (formulas outside the streaming templates, P:229-237;
 * DESIGN reading R27) for one launch; host arithmetic only, no device access.  `grid` CTAs
 * of `per_cta` replica slots each share `budget_bytes`; a slot needs W * per_entry + small
 * bytes for rings of W entries.  W is the largest power of two <= want that fits, after
 * giving up CTAs in this order: down to max(1, grid/2) CTAs to reach W = want, then as many
 * as needed to reach W = min(want, 1024).  *grid_out <= grid CTAs, *cap_out = W.
 * SMC_E_ARG on a zero size or count; SMC_E_CUDA ("not enough device memory") if W < 16. */
int smc_window_ring_plan(uint64_t budget_bytes, uint64_t per_entry, uint64_t small, int32_t per_cta, int32_t grid,
                         uint64_t want, int32_t* grid_out, uint64_t* cap_out);

/* ------------------------------------------------------------------------ */
/* Integration hooks (PyTorch owns device memory, streams, process groups)    */
/* ------------------------------------------------------------------------ */
/* alloc(bytes, user) -> device pointer or NULL; free_(ptr, user).  NULL/NULL
 * restores cudaMalloc/cudaFree.  Set before creating models. */
int smc_set_allocator(void* (*alloc)(size_t, void*), void (*free_)(void*, void*), void* user);
/* cudaStream_t on which every kernel, memset and copy is issued (NULL = default). */
int smc_set_stream(void* cuda_stream);
/* This process is rank `rank` of `world` (1 <= world, 0 <= rank < world). */
int smc_set_shard(int32_t rank, int32_t world);
/* fn(dev_counts, n, user) must sum the n int64 DEVICE values over all ranks in
 * place, ordered on the stream hook (e.g. torch.distributed.all_reduce on
 * NCCL); non-zero return -> SMC_E_COMM.  NULL = single process. */
int smc_set_allreduce(int (*fn)(int64_t* dev_counts, int32_t n, void* user), void* user);

/* ------------------------------------------------------------------------ */
/* Test / measurement exports                                                 */
/* ------------------------------------------------------------------------ */
/* Per-replica verdicts (0 false, 1 true, 2 error) and applied-event counts
 * for indices [first, first+n), written to DEVICE buffers dev_verdict[n],
 * dev_events[n].  No shard, no allreduce, cursor untouched. */
int smc_run_verdicts(smc_model* m, const smc_property* p, uint64_t first, uint64_t n,
                     uint64_t seed, uint8_t* dev_verdict, int32_t* dev_events);

/* n Philox4x32-10 blocks (seed, trajectory, step0 + q), q < n, computed by
 * the device code path, copied to host_out[4 n]. */
int smc_philox_blocks(uint64_t seed, uint64_t trajectory, uint64_t step0, uint32_t n, uint32_t* host_out);

/* n SSA draws of steps step0 + q, q < n, of (seed, trajectory) computed by the
 * device code path the kernels use (Eq. 2a numerator and the
 * Eq. 2b uniform): host_out[2q] = e = -log(u1), host_out[2q+1] = u2.
 * u2 is bit-exact with the oracle; e is within 1 ulp of glibc's -log(u1)
 * (reading R18).  Errors: SMC_E_ARG for NULL, SMC_E_CUDA. */
int smc_draw_blocks(uint64_t seed, uint64_t trajectory, uint64_t step0, uint32_t n, double* host_out);

typedef struct {
    int32_t variant;          /* 1 thread-owned, 2 tile, 3 literal, 4 sweep        */
    int32_t block_threads;    /* threads per CTA                                    */
    int32_t grid_blocks;      /* persistent CTAs                                    */
    int32_t smem_bytes;       /* dynamic shared memory per CTA                      */
    int32_t regs_per_thread;  /* from the compiled kernel                           */
    int32_t launches;         /* kernel launches by the last smc_run / smc_estimate */
    float kernel_ms;          /* CUDA-event time of the SSA kernels of that call    */
    float compile_ms;         /* NVRTC time of the kernel (first use)               */
    double table_bytes;       /* packed model + monitor tables read per CTA         */
    int32_t aux_launches;     /* other kernels of that call (per-round count kernels) */
    int32_t pad_;
    double sim_events;        /* SSA events this GPU's launches simulated in that call,
                                 incl. speculative replicas past the final N_tot */
} smc_launch_info;
/* Launch configuration and timing of the last run of (m, p). */
int smc_last_launch(const smc_model* m, const smc_property* p, smc_launch_info* out);

/* The generated CUDA source for (m, p) (for inspection); *len bytes incl. NUL
 * are needed; copies min(len, needed) bytes when buf != NULL. */
int smc_kernel_source(smc_model* m, const smc_property* p, char* buf, size_t* len);

#ifdef __cplusplus
}
#endif
#endif /* SMC_H_ */
