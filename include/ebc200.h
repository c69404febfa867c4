/*
 * ebc200.h -- C-ABI of the B200 (sm_100a) Exemplar-based Clustering hot path.
 *
 * Drop-in boundary for the reference package ebcsum 0.1.0 (arXiv 2105.12026).
 * The reference is pure Python, so "the FFI it would bind" is a ctypes binding
 * from its optimizer/objective layer; INTEGRATION.md shows that stub.  Every
 * entry point below names the reference function it replaces.
 *
 * Conventions
 *   - Plain pointers and sizes, no torch types.  The caller owns all host
 *     buffers; the library copies what it keeps.
 *   - Every call returns an ebc_status; on failure ebc_last_error(ctx) holds a
 *     message.  EBC_EINDEX carries the reference's exact IndexError text
 *     ("set {j}: index {i} out of range for ground size {n}", core.py:140-143).
 *   - A context is single-caller (not re-entrant); calls are synchronous.
 *   - There is no CPU fallback: without a usable CUDA device ebc_create fails
 *     with EBC_ECUDA.
 */
#ifndef EBC200_H
#define EBC200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ebc_ctx ebc_ctx;

typedef enum {
  EBC_OK = 0,
  EBC_EINVAL = 1, /* -> ValueError   (optimize.py:33-40,71-72; batched.py:190-191) */
  EBC_EINDEX = 2, /* -> IndexError   (core.py:136-143; ebc.py:119-120)             */
  EBC_ECUDA = 3,  /* -> RuntimeError (device / driver failure)                      */
  EBC_ECOMM = 4   /* -> RuntimeError (sharded exchange failure)                     */
} ebc_status;

/* Storage precision of the ground matrix (core.py:13-55 Precision). */
typedef enum {
  EBC_F32 = 0, /* Precision.FP32                                              */
  EBC_F16 = 1, /* Precision.FP16_STORAGE: IEEE half storage, fp32 arithmetic  */
  EBC_F64 = 2  /* Precision.FP64                                              */
} ebc_dtype;

/* Library version string, e.g. "ebc200 0.1.0 sm_100a". */
const char* ebc_version(void);

/* Number of CUDA devices visible to the library (0 when none). */
int ebc_device_count(void);

/* Upload the N x d row-major ground matrix V (element type `dtype`, already in
 * storage precision) and the fp64 auxiliary vector e0 (d entries; NULL = the
 * zero vector), pad V to 16-byte rows on `device`, and compute the baseline
 * loss L({e0}) once.
 * Replaces: GroundMatrix.__init__ (core.py:107-124) + EbcFunction.__init__
 *           (ebc.py:55-72, baseline at :72). */
int ebc_create(const void* V, int64_t n, int32_t d, int32_t dtype, const double* e0,
               int32_t device, ebc_ctx** out);

/* L({e0}) -- EbcFunction.baseline_loss (ebc.py:72). */
int ebc_baseline(const ebc_ctx* ctx, double* out);

/* f(S_j) for l sets given in CSR form (offsets has l+1 entries, idx holds the
 * members), fp64, in set order; empty sets give exactly 0.0.  On an index
 * outside [0, n) returns EBC_EINDEX and reports the first offending set/index
 * in set order.
 * Replaces: evaluate_with_backend (optimize.py:43-57) ->
 *           evaluate_multiset_batched (batched.py:180-240) / the naive oracle
 *           evaluate_multiset_naive (ebc.py:109-121). */
int ebc_eval_multiset(ebc_ctx* ctx, const int64_t* offsets, const int64_t* idx, int64_t l,
                      double* out_f, int64_t* out_bad_set, int64_t* out_bad_index);

/* ---- threshold sieves (sieve_stream_maximize, optimize.py:140-197) ----
 * Each live sieve occupies a slot holding its cached minima over S_r u {e0}
 * (N doubles), so one streamed element costs one distance pass shared by all
 * sieves.  Values equal ebc_eval_multiset's on the same sets bit for bit.
 *   ebc_sieve_reserve: storage for `slots` sieves (a new reservation starts
 *     from scratch: slot contents are not kept);
 *   ebc_sieve_step: (1) reset the reset slots to S = {}, (2) fold ground
 *     index commit_e into the commit slots (the previous element's admissions;
 *     commit_e < 0: none), (3) if e >= 0: *out_single = f({e}) and
 *     out_values[i] = f(S_r u {e}) for r = eval_slots[i].  One host round trip. */
int ebc_sieve_reserve(ebc_ctx* ctx, int32_t slots);
int ebc_sieve_step(ebc_ctx* ctx, int64_t commit_e, const int32_t* commit_slots, int32_t n_commit,
                   const int32_t* reset_slots, int32_t n_reset, int64_t e, const int32_t* eval_slots,
                   int32_t n_eval, double* out_single, double* out_values);

/* k-medoids loss of explicit representatives: mean over the ground rows of the
 * exact fp64 squared distance to the nearest of the r representatives
 * (reps: r x d row-major fp64, finite), the ground values widened exactly to
 * fp64.  EBC_EINVAL for r < 1 or a non-finite representative (the reference's
 * messages).  Replaces: k_medoids_loss (ebc.py:21-43). */
int ebc_kmedoids_loss(ebc_ctx* ctx, const double* reps, int64_t r, double* out);

/* Full Greedy(k) on this device: k steps of screen -> certified fp64 refine ->
 * argmax with the reference tie window -> cached-min update, no host sync
 * between steps.  out_sel/out_val/out_gain receive k entries (out_val[s] is
 * f after s+1 selections); *out_evals = sum over steps of the frontier size.
 * Replaces: greedy_maximize (optimize.py:60-91). */
int ebc_greedy(ebc_ctx* ctx, int32_t k, int64_t* out_sel, double* out_val, double* out_gain,
               int64_t* out_evals);

/* ---- candidate-sharded Greedy (one process per GPU) ----
 * V is replicated; this context screens only candidates [c0, c1).  A step is
 *   ebc_shard_step   -> local certified list (index, exact fp64 gain)
 *   (host exchange across ranks; global pick, see paper_2105_12026_b200/sharded.py)
 *   ebc_shard_commit -> fold the globally chosen index into the cached minima.
 */
/* c0 must be a multiple of 128 (the screens' candidate block) unless c0 == c1. */
int ebc_shard_set_range(ebc_ctx* ctx, int64_t c0, int64_t c1);

/* Screen + refine the local candidates for the current step.  Writes up to
 * `cap` (index, gain64) pairs; *out_count is the full list length (may exceed
 * cap: call again with a larger buffer, results are cached until commit).
 * *out_current = f(S) of the current selection. */
int ebc_shard_step(ebc_ctx* ctx, int64_t* out_idx, double* out_gain, int64_t cap,
                   int64_t* out_count, double* out_current);

/* Select ground index `s` (any rank's candidate): cm <- min(cm, d(., s)),
 * returns the new f(S) in *out_value. */
int ebc_shard_commit(ebc_ctx* ctx, int64_t s, double* out_value);

/* One host round trip per sharded Greedy step: commit `commit_idx` (if >= 0),
 * then (if run_step) screen + refine the local candidates; the first `cap`
 * window entries (index, gain64), the full window size and f(S) after the
 * commit come back with a single stream synchronisation.  If *out_count > cap,
 * fetch all of it with ebc_shard_fetch (the window stays on the device until
 * the next advance). */
int ebc_shard_advance(ebc_ctx* ctx, int64_t commit_idx, int32_t run_step, int64_t* out_idx,
                      double* out_gain, int64_t cap, int64_t* out_count, double* out_current);

/* Copy the first `count` entries of the current local window to the host. */
int ebc_shard_fetch(const ebc_ctx* ctx, int64_t* out_idx, double* out_gain, int64_t count);

/* ---- device-side sharded Greedy: the exchange runs on the GPU (NCCL over
 * NVLink/NVSwitch), no host round trip per step ----
 * Replaces the per-step host loop of greedy_maximize (optimize.py:75-88) across
 * ranks.  Per step every rank screens its candidate range, computes the exact
 * gains of its certified window, reduces its local tie set
 * {c : value_c >= top_r - 1e-12 max(1,|top_r|)} to its index-ordered Pareto
 * frontier (at most TIE_CAP = ebc_tie_cap() records of {index, gain} plus a
 * count: 128 B per rank), one ncclAllGather of the records, then every rank
 * applies the reference rule (optimize.py:83-85) to the identical union and
 * folds the winner into its cached minima.  After the last step the ranks
 * all-gather a 64-bit hash of (selection, values, gains) and fail on any
 * mismatch.  The k-step loop is graph-captured like ebc_greedy.  NCCL is
 * dlopen'ed (libnccl.so.2) on first use.
 *   ebc_comm_id_bytes / ebc_comm_unique_id -> rank 0 makes the id, the caller
 *     broadcasts it (e.g. torch.distributed), every rank calls ebc_comm_init;
 *   ebc_shard_set_range sets the rank's candidate range first (the start must
 *     be a multiple of 128, the candidate block of the screens, unless empty);
 *   ebc_greedy_sharded -> same outputs as ebc_greedy, identical on every rank;
 *     EBC_ECOMM if a frontier overflowed (ebc_comm_status bit 0: the caller
 *     falls back to ebc_shard_advance) or the ranks disagree (bit 1: a bug,
 *     never a fallback). */
int64_t ebc_comm_id_bytes(void);
int ebc_comm_unique_id(unsigned char* out_id, int64_t bytes);
int ebc_comm_init(ebc_ctx* ctx, const unsigned char* id, int64_t bytes, int32_t nranks, int32_t rank);
/* The communicator is per device and process; later contexts on the same device
 * attach to it without another ncclCommInitRank (EBC_ECOMM if none exists). */
int ebc_comm_attach(ebc_ctx* ctx);
int ebc_greedy_sharded(ebc_ctx* ctx, int32_t k, int64_t* out_sel, double* out_val, double* out_gain,
                       int64_t* out_evals);
/* Flags of the last ebc_greedy_sharded: 1 frontier overflow, 2 cross-rank mismatch. */
int ebc_comm_status(const ebc_ctx* ctx, int32_t* out_flags);
/* Host-fed form of the same step (tests / emulated ranks on one GPU): the local
 * frontier records ((TIE_CAP + 1) x {index, gain}, record 0 = {count, 0}) and
 * the global pick + commit from `world` gathered record blocks. */
int32_t ebc_tie_cap(void);
int ebc_shard_tie_step(ebc_ctx* ctx, double* out_rec, double* out_current);
int ebc_shard_pick_commit(ebc_ctx* ctx, const double* gathered, int32_t world, int32_t step, int64_t* out_best,
                          double* out_value);

/* Reset the selection state to S = {} (cached minima back to d(., e0)). */
int ebc_reset(ebc_ctx* ctx);

/* The cudaStream_t all work of this context is issued on (for callers that
 * record their own CUDA events around library calls). */
void* ebc_stream(const ebc_ctx* ctx);

/* Enable per-step CUDA-event timing of the kernel families (off by default). */
int ebc_set_timing(ebc_ctx* ctx, int on);

/* Device-time of the last ebc_greedy / ebc_eval_multiset call split by kernel
 * family, in milliseconds (CUDA events on the library stream): [0] screen,
 * [1] refine+pick, [2] cached-min update, [3] whole call.  For bench.py. */
int ebc_last_timings(const ebc_ctx* ctx, double* out_ms4);

/* Screen statistics since the last reset / Greedy run: [0] sum of certified
 * window sizes, [1] largest window, [2] screen rung in use at the end (0 fast
 * tensor Gram with one rounded FP16 product, 1 tensor Gram with the operand kind
 * of ebc_screen_info [2], 2 FFMA Gram, 3 direct, -1 n/a), [3] steps. */
int ebc_last_stats(const ebc_ctx* ctx, int64_t* out4);

/* Point-candidate pairs the tensor screen actually evaluated since the last
 * reset / Greedy run (tile pairs kept by the certified tile-pair pruning x
 * 128 x points per tile).  For bench.py's roofline. */
int ebc_last_screen_work(const ebc_ctx* ctx, int64_t* out_pairs);

/* Screen configuration: [0] mode (0 direct, 1 FFMA Gram, 2 ladder from FFMA
 * Gram, 3 ladder from the tensor screen), [1] points per tensor tile (0: no
 * tensor screen), [2] tensor operand kind (1 BF16 h+m split, 0 TF32 hi+lo split,
 * 2 FP16 values of fp16-stored grounds, -1 n/a; rung 0, when enabled, always
 * uses fp32 values rounded to FP16),
 * [3] padded K of the tensor operands. */
int ebc_screen_info(const ebc_ctx* ctx, int64_t* out4);

/* Lazy Greedy statistics of the last run: [0] lazy steps enabled (EBC200_LAZY),
 * [1] lazy steps (every step after the first), [2] of those decided by the
 * exact refine of the stale candidates alone (no screen launch did work),
 * [3] candidates re-examined by the lazy steps (first batches + stale lists).  A lazy step re-examines
 * only candidates whose last bound (screen upper bound or exact gain) can
 * still reach the reference tie window: gains only shrink as S grows
 * (submodularity), so the selection is unchanged. */
int ebc_last_lazy_stats(const ebc_ctx* ctx, int64_t* out4);

/* Page-lock a host buffer for direct DMA (cudaHostRegister, portable) /
 * release it.  No reference counterpart: the reference keeps its ground in
 * ordinary numpy memory.  A GroundMatrix's rows are registered once
 * (ebc.py), so every ebc_create from them uploads by one direct copy instead
 * of the staged pageable path.  ebc_host_register returns EBC_ECUDA (and
 * leaves the buffer pageable) when the driver refuses. */
int ebc_host_register(const void* ptr, int64_t bytes);
int ebc_host_unregister(const void* ptr);

/* Kernel launches issued by the last call (bench.py's gpu_launches). */
int64_t ebc_last_launches(const ebc_ctx* ctx);

/* Free all device state. */
void ebc_destroy(ebc_ctx* ctx);

/* Message for the last failing call on ctx (or a global message when ctx is
 * NULL, e.g. after a failed ebc_create). */
const char* ebc_last_error(const ebc_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* EBC200_H */
