/*
 * pfr.h -- C ABI of the B200 resampling library (libpfr.so).
 *
 * Drop-in boundary for the hot path of the reference package `pfresample`
 * (paths relative to /root/reference/pkg/src/pfresample).  Each entry point
 * names the reference function it replaces.  Conventions:
 *
 *   - all array arguments are DEVICE pointers (CUDA global memory, 16-byte
 *     aligned); scalars are passed by value;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream); every
 *     call only ENQUEUES work on that stream and returns without synchronising;
 *   - `ws`/`ws_bytes` is caller-owned scratch sized by pfr_workspace_bytes(),
 *     256-byte aligned and ZERO-FILLED when first allocated (the fused
 *     delivery keeps self-resetting counters in it); one stream at a time may
 *     use a given workspace; the library never allocates device memory;
 *   - inputs are never written (the reference never mutates inputs,
 *     SPEC.md:371); outputs are caller-allocated;
 *   - indices are int32 on output (N < 2^31); index inputs may be int32 or
 *     int64 (`idx_dtype`);
 *   - data-dependent validation (non-finite / negative / all-zero weights,
 *     out-of-range ancestries, ...) is OR-ed into the device word `*status`
 *     (PFR_ST_* bits; never cleared by the library).  The host reads it when
 *     it synchronises and raises the reference's ValueError / RuntimeError;
 *   - the return value is 0 (PFR_OK) or a PFR_E_* code for argument/launch
 *     errors detectable on the host; pfr_last_error() returns a thread-local
 *     message for the last failure.
 */
#ifndef PFR_H_
#define PFR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PFR_ABI_VERSION 1

/* element types */
enum pfr_dtype { PFR_F32 = 0, PFR_F64 = 1, PFR_I32 = 2, PFR_I64 = 3 };

/* accumulation precision for weight scans/positions */
enum pfr_accum {
  PFR_ACC_F64 = 0,    /* positions and carries in float64 (default; fp32 is storage only) */
  PFR_ACC_NATIVE = 1, /* accumulate in the weight dtype with the parallel (tree) association */
  PFR_ACC_SERIAL = 2  /* the reference's np.cumsum bit for bit: a left-to-right fold in the weight
                         dtype (parity mode; one serial thread, ~4.5 cycles per element) */
};
/* OR-ed into pfr_scan's `accum`: repair ulp-level non-monotonicity with an
 * exact running max (only meaningful for non-negative inputs such as weights) */
#define PFR_SCAN_MONOTONE 0x100
/* the input is a weight vector: the scan also reports check_weights' flags
 * (negative, any-positive; non-finite is always reported) */
#define PFR_SCAN_WEIGHTS 0x200

/* where the random draws come from */
enum pfr_rng_mode {
  PFR_RNG_PHILOX = 0, /* own Philox4x32-10 keyed by derive_seed(seed, *ids) */
  PFR_RNG_NUMPY = 1,  /* exact replay of numpy Philox4x64-10 as RngStream.generator() */
  PFR_RNG_ARRAYS = 2  /* draws supplied by the caller in device arrays */
};

/* status bits OR-ed into *status by the kernels */
enum pfr_status_bits {
  PFR_ST_NONFINITE = 1u << 0,      /* weight/log-weight NaN or +-inf (+inf only for log-weights) */
  PFR_ST_NEGATIVE = 1u << 1,       /* negative weight */
  PFR_ST_POSITIVE = 1u << 2,       /* SET when at least one weight > 0 */
  PFR_ST_RANGE = 1u << 3,          /* ancestry entry outside [0, N) */
  PFR_ST_REPAIRED = 1u << 4,       /* monotone repair of O was needed (informational) */
  PFR_ST_OVERFLOW = 1u << 5,       /* chain walk exceeded its bound: fallback kernel resolved it */
  PFR_ST_NOPROGRESS = 1u << 6,     /* rejection exceeded max_rounds proposals for a slot */
  PFR_ST_NOTMONOTONE = 1u << 7,    /* cumulative offspring input decreases */
  PFR_ST_BADEND = 1u << 8,         /* cumulative offspring input does not end at N */
  PFR_ST_NEGCOUNT = 1u << 9,       /* negative offspring count / cumulative start */
  PFR_ST_BADSUM = 1u << 10,        /* offspring counts do not sum to N */
  PFR_ST_RATIO = 1u << 11,         /* non-finite acceptance ratio w / bound */
  PFR_ST_NONTERMINATION = 1u << 12,/* permute chain did not terminate (cannot happen for valid a) */
  PFR_ST_NOTINT = 1u << 13,        /* non-integer value where an index was expected */
  PFR_ST_NEEDS_REPAIR = 1u << 14   /* internal: O must be max-scanned before use */
};

enum pfr_error {
  PFR_OK = 0,
  PFR_E_ARG = 1,       /* invalid argument (size, dtype, null pointer) */
  PFR_E_WORKSPACE = 2, /* workspace too small */
  PFR_E_CUDA = 3,      /* CUDA launch error */
  PFR_E_UNSUPPORTED = 4
};

/* operation ids for pfr_workspace_bytes */
enum pfr_op {
  PFR_OP_SCAN = 0,
  PFR_OP_OFFSPRING = 1, /* systematic / stratified cumulative offspring */
  PFR_OP_DELIVER = 2,   /* fused systematic/stratified -> in-place ancestry */
  PFR_OP_PERMUTE = 3,
  PFR_OP_MULTINOMIAL = 4,
  PFR_OP_METROPOLIS = 5,
  PFR_OP_REJECTION = 6,
  PFR_OP_EXPAND = 7,
  PFR_OP_LOGWEIGHTS = 8,
  PFR_OP_PREDICATE = 9,
  PFR_OP_ANY = 10 /* max over all ops */
};

/* the caller's RngStream(seed, ids) after key derivation (rng.py:39-74):
 * key0 = derive_seed(seed, 0, *ids), key1 = derive_seed(seed, 1, *ids) */
typedef struct pfr_rng {
  uint64_t key0;
  uint64_t key1;
  int32_t mode; /* enum pfr_rng_mode */
  int32_t reserved;
} pfr_rng;

/* ---- library --------------------------------------------------------- */
int pfr_abi_version(void);
const char* pfr_last_error(void);
size_t pfr_workspace_bytes(int op, int64_t n, int dtype);
/* number of kernels the library launched on this host thread since the last reset */
uint64_t pfr_launch_count(int reset);

/* one uniform in [0,1) of the stream, evaluated on the host with the same
 * generator code the kernels use: NUMPY mode = the index-th
 * Generator.random() draw (rng.py:69-74; resamplers.py:134 takes index 0);
 * PHILOX mode = 53-bit double from Philox4x32-10 counter (index, 0, tag, 0). */
double pfr_stream_uniform(const pfr_rng* rng, uint64_t index, uint32_t tag);

/* ---- primitives (primitives.py) ---------------------------------------- */

/* inclusive_prefix_sum (primitives.py:34-42), exclusive_prefix_sum (45-51),
 * vector_sum (60-66), offspring_to_cumulative (ancestry.py:85-88).
 * Single pass with a deterministic lookback tree.  `out_dtype` is the dtype of
 * `out` (float: same as input, or PFR_F64 for float32 input; integer input:
 * PFR_I64 or PFR_I32).  `total`
 * (nullable, device) receives the sum (double for floats, int64 for ints).
 * Validation bits: NONFINITE for floats, NEGCOUNT for negative ints. */
int pfr_scan(const void* in, void* out, int64_t n, int dtype, int out_dtype, int accum, int exclusive,
             void* total, uint32_t* status, void* ws, size_t ws_bytes, void* stream);

/* adjacent_difference (primitives.py:54-57) and cumulative_to_offspring
 * (ancestry.py:91-94; validates non-decreasing/ends at N when dtype is int). */
int pfr_adjacent_difference(const void* in, void* out, int64_t n, int dtype, int out_dtype, uint32_t* status,
                            void* stream);

/* lower_bound (primitives.py:91-106): out[i] = min(N-1, #{j : W[j] < u[i]}),
 * float32 W compared in float64 as numpy promotes. */
int pfr_lower_bound(const void* W, int64_t n, int dtype, const double* u, int64_t m, int32_t* out, void* stream);

/* check_weights (diagnostics.py:38-51): NONFINITE / NEGATIVE / POSITIVE bits */
int pfr_check_weights(const void* w, int64_t n, int dtype, uint32_t* status, void* stream);

/* logweights_to_weights (diagnostics.py:138-155): w = exp(lw - max lw) */
int pfr_logweights_to_weights(const void* lw, void* w, int64_t n, int dtype, uint32_t* status, void* ws,
                              size_t ws_bytes, void* stream);

/* ---- resamplers (resamplers.py) ------------------------------------------ */

/* systematic_cumulative_offspring (resamplers.py:127-136) when uniforms == NULL
 * (`offset` = the single u in [0,1)), stratified_cumulative_offspring
 * (resamplers.py:105-124) otherwise or when rng != NULL && stratified.
 * O[i] = min(N, floor(N*W[i]/W[N-1] + u[k-1])), k = min(N, floor(r)+1),
 * then the monotone repair and O[N-1] = N (resamplers.py:139-153).
 *   stratified == 0: systematic, u = offset cast to the weight dtype
 *   stratified == 1: per-stratum u from `uniforms` (float64, length N) if not
 *                    NULL, else from `rng` (PHILOX or NUMPY stream). */
int pfr_cumulative_offspring(const void* w, int64_t n, int dtype, int accum, int stratified, double offset,
                             const double* uniforms, const pfr_rng* rng, int32_t* O, uint32_t* status, void* ws,
                             size_t ws_bytes, void* stream);

/* Fused delivery: weights -> in-place-valid ancestry c, i.e.
 * permute_parallel(cumulative_offspring_to_ancestors(<systematic|stratified O>))
 * (bench.py:155-161 timed region for the offspring algorithms) without
 * materialising the sorted ancestry.  O_out (nullable) also returns O. */
int pfr_deliver_offspring(const void* w, int64_t n, int dtype, int accum, int stratified, double offset,
                          const double* uniforms, const pfr_rng* rng, int32_t* c, int32_t* O_out,
                          int32_t* max_steps, uint32_t* status, void* ws, size_t ws_bytes, void* stream);

/* The same delivery from LOG-weights: logweights_to_weights (diagnostics.py:
 * 138-155) fused into the delivery -- one max pass over lw (its validation:
 * NaN / +inf / all -inf), then the delivery computes w = exp(lw - max lw) as
 * it loads each tile (twice: K1 and K2), so w is never written.  Results are
 * identical to pfr_logweights_to_weights followed by pfr_deliver_offspring. */
int pfr_deliver_offspring_logw(const void* lw, int64_t n, int dtype, int accum, int stratified, double offset,
                               const double* uniforms, const pfr_rng* rng, int32_t* c, int32_t* O_out,
                               int32_t* max_steps, uint32_t* status, void* ws, size_t ws_bytes, void* stream);

/* Fused Metropolis delivery (own PHILOX stream): permute_parallel(
 * metropolis_ancestors(w, steps)) (resamplers.py:204-234, ancestry.py:
 * 125-174) with the permute's claims made by the chains as they finish, so
 * the ancestry is never re-read for claiming; c is the in-place-valid
 * ancestry.  Identical to pfr_metropolis followed by pfr_permute. */
int pfr_deliver_metropolis(const void* w, int64_t n, int dtype, int64_t steps, const pfr_rng* rng, int32_t* c,
                           int32_t* max_steps, uint32_t* status, void* ws, size_t ws_bytes, void* stream);

/* Fused rejection delivery (own PHILOX stream): permute_parallel(
 * rejection_ancestors(w, sup_w)) (resamplers.py:237-310, ancestry.py:
 * 125-174); a slot claims its ancestor when it accepts, so the ancestry is
 * never re-read for claiming.  Identical to pfr_rejection followed by
 * pfr_permute (max_rounds as there). */
int pfr_deliver_rejection(const void* w, int64_t n, int dtype, double bound, const pfr_rng* rng, int64_t max_rounds,
                          int32_t* c, int32_t* max_steps, uint32_t* status, void* ws, size_t ws_bytes, void* stream);

/* Fused multinomial delivery (own PHILOX stream): permute_parallel(
 * multinomial_ancestors(w)) (resamplers.py:56-74, ancestry.py:125-174); the
 * merge claims each slot's ancestor as it writes it.  Identical to
 * pfr_multinomial followed by pfr_permute. */
int pfr_deliver_multinomial(const void* w, int64_t n, int dtype, int accum, const pfr_rng* rng, int32_t* c,
                            int32_t* max_steps, uint32_t* status, void* ws, size_t ws_bytes, void* stream);

/* multinomial_ancestors (resamplers.py:56-74).
 *   rng mode ARRAYS: `uniforms` are the pre-scaled draws in [0, W[N-1]);
 *   rng mode NUMPY : u = random(N) * W[N-1] replayed from the stream; out a is unsorted;
 *   rng mode PHILOX: sorted order statistics (exponential spacings) merged
 *                    against W: a is sorted (the O(N) Code-4 formulation).
 * sorted_serial != 0 selects multinomial_ancestors_serial's log-spacing
 * construction (resamplers.py:77-102) with NUMPY draws. */
int pfr_multinomial(const void* w, int64_t n, int dtype, int accum, const pfr_rng* rng, const double* uniforms,
                    int sorted_serial, int32_t* a, uint32_t* status, void* ws, size_t ws_bytes, void* stream);

/* metropolis_ancestors (resamplers.py:204-234): N chains of B steps.
 * rng mode ARRAYS uses u_draws[B*N] (float64) and j_draws[B*N] (idx_dtype). */
int pfr_metropolis(const void* w, int64_t n, int dtype, int64_t steps, const pfr_rng* rng, const double* u_draws,
                   const void* j_draws, int idx_dtype, int32_t* a, uint32_t* status, void* ws, size_t ws_bytes,
                   void* stream);

/* rejection_ancestors / _rejection_loop (resamplers.py:237-255, 282-310) and,
 * with cap > 0, rejection_ancestors_capped (258-279): v = min(w, cap),
 * bound = cap, out_w[i] = w[a[i]] / v[a[i]] (1 where v[a[i]] == 0).
 * trips (nullable) gets per-slot proposal counts; max_rounds bounds them
 * (the reference raises after 100000 rounds: NOPROGRESS).  check_weights'
 * flags (diagnostics.py:38-51) go to status: from the certain-reject table
 * pass (4096 <= N <= 2^22, workspace with the O region) or a check pass. */
int pfr_rejection(const void* w, int64_t n, int dtype, double bound, double cap, const pfr_rng* rng,
                  int64_t max_rounds, int32_t* a, int32_t* trips, void* out_w, uint32_t* status, void* ws,
                  size_t ws_bytes, void* stream);

/* ---- ancestry (ancestry.py) ---------------------------------------------- */

/* cumulative_offspring_to_ancestors (ancestry.py:69-76): merge-path expand */
int pfr_cumulative_to_ancestors(const void* O, int64_t n, int idx_dtype, int32_t* a, uint32_t* status, void* ws,
                                size_t ws_bytes, void* stream);

/* ancestors_to_offspring (ancestry.py:79-82): histogram */
int pfr_ancestors_to_offspring(const void* a, int64_t n, int idx_dtype, int32_t* o, uint32_t* status, void* stream);

/* prepermute (ancestry.py:125-136): d[v] = min{i : a[i] = v}, sentinel N */
int pfr_prepermute(const void* a, int64_t n, int idx_dtype, int32_t* d, uint32_t* status, void* stream);

/* permute_parallel (ancestry.py:139-174): c with o[i] > 0 => c[i] = i; same
 * output as the reference for every input.  max_steps (nullable, device int32)
 * gets the longest chain walk (return_max_steps=True). */
int pfr_permute(const void* a, int64_t n, int idx_dtype, int32_t* c, int32_t* max_steps, uint32_t* status,
                void* ws, size_t ws_bytes, void* stream);

/* permute_parallel(cumulative_offspring_to_ancestors(O)) directly from O */
int pfr_permute_cumulative(const int32_t* O, int64_t n, int32_t* c, int32_t* max_steps, uint32_t* status,
                           void* ws, size_t ws_bytes, void* stream);

/* satisfies_inplace_predicate (ancestry.py:97-101): *result = 1/0 (device int32) */
int pfr_check_predicate(const void* c, int64_t n, int idx_dtype, int32_t* result, uint32_t* status, void* ws,
                        size_t ws_bytes, void* stream);

/* in-place copy step of the bootstrap filter (pf.py:86-97):
 * x[i] = x[c[i]] wherever c[i] != i, for `width` float64 values per particle */
int pfr_copy_particles(double* x, int64_t n, int64_t width, const int32_t* c, void* stream);

/* ---- one weight-sharded filter across GPUs --------------
 * Each rank holds a contiguous shard [index_base, index_base + n_loc) of the
 * N weights.  The host protocol (paper_1301_4019_b200/sharded.py) runs, per
 * rank: pfr_scan (float64 output) -> all-gather of shard totals -> the calls
 * below -> all-to-all of slot words / walkers.  The reference has no
 * distributed path; these calls reproduce resamplers.py:139-153 and
 * ancestry.py:139-174 over shards. */

/* metropolis_ancestors (resamplers.py:204-234) for chains [chain_begin,
 * chain_begin + chain_count) of the N-chain resampler, a[i - chain_begin];
 * draws are those of the global chain numbers (PHILOX or NUMPY stream), so
 * the union over ranks equals the single-GPU result. */
int pfr_metropolis_range(const void* w, int64_t n, int dtype, int64_t steps, const pfr_rng* rng, int64_t chain_begin,
                         int64_t chain_count, int32_t* a, uint32_t* status, void* stream);

/* rejection_ancestors / rejection_ancestors_capped (resamplers.py:237-310)
 * for slots [slot_begin, slot_begin + slot_count) of the N-slot resampler
 * over the full weight vector w[n]: a, trips, out_w indexed slot -
 * slot_begin; every slot draws from its global number's PHILOX stream, so
 * the union over ranks equals the single-GPU result (rejection
 * partitions the output slots over the all-gathered weights). */
int pfr_rejection_range(const void* w, int64_t n, int dtype, double bound, double cap, const pfr_rng* rng,
                        int64_t max_rounds, int64_t slot_begin, int64_t slot_count, int32_t* a, int32_t* trips,
                        void* out_w, uint32_t* status, void* ws, size_t ws_bytes, void* stream);

/* multinomial_ancestors (resamplers.py:56-74) for slots [slot_begin,
 * slot_begin + slot_count) of the N-slot resampler over the full weight
 * vector w[n]: a is indexed slot - slot_begin.  Own stream: the sorted
 * uniforms of those slots from the (replicated) spacing scan, merged with W
 * along their merge-path diagonals only; numpy stream / caller uniforms: the
 * slots' own draws.  The union over ranks equals pfr_multinomial (SURVEY
 * 8(e): the weight-sharded multinomial partitions the output slots). */
int pfr_multinomial_range(const void* w, int64_t n, int dtype, int accum, const pfr_rng* rng, const double* uniforms,
                          int64_t slot_begin, int64_t slot_count, int32_t* a, uint32_t* status, void* ws,
                          size_t ws_bytes, void* stream);

/* A rank's share of permute_parallel (ancestry.py:139-174): c[x - index_begin]
 * for x in [index_begin, index_begin + index_count), from the full ancestry
 * a[n] (claims over all of a, then backward loser walks for the range's
 * holes only).  The union over ranks equals pfr_permute; a chain longer than
 * 4096 hops sets PFR_ST_OVERFLOW (fall back to pfr_permute). */
int pfr_permute_range(const int32_t* a, int64_t n, int64_t index_begin, int64_t index_count, int32_t* c,
                      int32_t* max_steps, uint32_t* status, void* ws, size_t ws_bytes, void* stream);

/* Cumulative offspring of this shard's parents in global slot numbers
 * (_offspring_from_positions, resamplers.py:139-153): W = prefix + W_loc[i]
 * (W_loc = the shard's inclusive scan in float64), r = (W*N)/total,
 * O = min(N, floor(r + u[k-1])), O = N at the global last particle. */
int pfr_shard_offspring(const double* W_loc, int64_t n_loc, int dtype, double prefix, double total, int64_t n_global,
                        int last_global, int stratified, double offset, const double* uniforms, const pfr_rng* rng,
                        int32_t* O, void* stream);

/* Protocol v3 of the weight-sharded systematic / stratified delivery
 * (sharded.py): the shard's local work through the single-GPU kernels.
 * pfr_shard_local_end: the shard's float64 weight hierarchy (check_weights'
 * flags into status) and its END value -- W at its last element in the
 * delivery's association -- into *end (device), the value the next shard's
 * prefix adds.  pfr_shard_produce: O of the shard's parents in global slot
 * numbers with prefix_total = {weight before the shard (a left fold of the
 * END values in rank order), W_N} read on the device, and their slot words
 * (global parents) written to ext[slot - slot_lo] for slots in [slot_lo,
 * slot_hi) (ext is set to 0xFFFFFFFF first; a slot outside sets
 * PFR_ST_OVERFLOW).  pfr_shard_resolve_fast: the in-place ancestry of the
 * shard's indices from ext (after the neighbours' bands are merged in,
 * pfr_shard_merge_bands), c indexed locally, values global; a chain leaving
 * the window sets PFR_ST_OVERFLOW.  The three share one workspace. */
int pfr_shard_local_end(const void* w_loc, int64_t n_loc, int dtype, double* end, uint32_t* status, void* ws,
                        size_t ws_bytes, void* stream);
int pfr_shard_produce(const void* w_loc, int64_t n_loc, int dtype, int64_t index_base, int64_t n_global,
                      const double* prefix_total, int first, int last, int stratified, double offset,
                      const double* uniforms, const pfr_rng* rng, uint32_t* ext, int64_t slot_lo, int64_t slot_hi,
                      uint32_t* status, void* ws, size_t ws_bytes, void* stream);
int pfr_shard_resolve_fast(int64_t n_loc, int dtype, int64_t index_base, const uint32_t* ext, int64_t slot_lo,
                           int64_t slot_hi, int32_t* c, int32_t* max_steps, uint32_t* status, void* ws,
                           size_t ws_bytes, void* stream);

/* Fill ext's sentinels from the neighbours' boundary bands: from_left = the
 * left neighbour's ext[n, n + 2*halo), from_right = the right neighbour's
 * ext[0, 2*halo) (null at the ends of the rank order). */
int pfr_shard_merge_bands(uint32_t* ext, int64_t n_loc, int64_t halo, const uint32_t* from_left,
                          const uint32_t* from_right, void* stream);
/* Slot words of the shard's slot window [o_begin, O[n_loc-1]):
 * words[s - o_begin] = parent | 0x80000000 on a parent's first slot
 * (cumulative_offspring_to_ancestors, ancestry.py:69-76, + prepermute's
 * winner flag, ancestry.py:125-136); has[i] = o_i > 0. */
int pfr_shard_words(const int32_t* O_loc, int64_t n_loc, int64_t index_base, int32_t o_begin, uint32_t* words,
                    uint8_t* has, uint32_t* status, void* stream);

/* In-place ancestry of the shard's indices from the slot words of those
 * indices (received from their producers): c[x] for every x whose loser
 * chain stays in the shard; chains leaving it are appended to pend as
 * (hole, slot, steps) int32 triples, *pend_count (device, zeroed by caller). */
int pfr_shard_resolve(const uint32_t* words, const uint8_t* has, int64_t n_loc, int64_t index_base, int32_t* c,
                      int32_t* pend, int32_t* pend_count, int32_t* max_steps, uint32_t* status, void* stream);

/* Advance routed walkers (hole, slot, steps) whose slot lies in this shard:
 * resolved chains -> done (hole, value) pairs, chains leaving again -> fwd. */
int pfr_shard_advance(const int32_t* walkers, int64_t count, const uint32_t* words, int64_t n_loc, int64_t index_base,
                      int32_t* done, int32_t* done_count, int32_t* fwd, int32_t* fwd_count, int32_t* max_steps,
                      uint32_t* status, void* stream);

/* c[hole - index_base] = value for routed (hole, value) pairs */
int pfr_shard_scatter(const int32_t* done, int64_t count, int64_t index_base, int64_t n_loc, int32_t* c,
                      uint32_t* status, void* stream);

/* ---- remaining reference functions around the step ----------------------- */

/* permute_serial (ancestry.py:104-122, PAPER Code 11): the serial pairwise
 * swaps, run by one device thread (inherently sequential; API parity). */
int pfr_permute_serial(const void* a, int64_t n, int idx_dtype, int32_t* c, uint32_t* status, void* stream);

/* stable_sum (primitives.py:69-88): balanced pairwise tree over the
 * zero-padded power-of-two vector, bit-identical to the reference;
 * *result (device double). */
int pfr_stable_sum(const void* w, int64_t n, int dtype, double* result, void* ws, size_t ws_bytes, void* stream);

/* ess (diagnostics.py:54-63) and resampling_mse (diagnostics.py:66-80) in one
 * deterministic pass: out[4] (device) = {sum w, sum w^2, ESS, MSE}; MSE = 0
 * when o (offspring counts) is NULL. */
int pfr_weight_stats(const void* w, int64_t n, int dtype, const void* o, int idx_dtype, double* out, void* ws,
                     size_t ws_bytes, void* stream);

/* Measurement helper (not a reference interface): `gathers` random loads of
 * elem_bytes (4 or 8) words from buf[n] (n a power of two), indices from
 * per-thread LCGs -- the memory system's random-gather rate that bounds the
 * Metropolis and rejection kernels (bench.py times it with CUDA events).
 * *sink (device) only keeps the loads live. */
int pfr_probe_gather(const void* buf, int64_t n, int elem_bytes, int64_t gathers, unsigned long long* sink,
                     void* stream);

/* ---- batches of independent filters -----------
 * No communication between filters.  Arrays are [filters, n] row-major. */

size_t pfr_batched_workspace_bytes(int64_t filters, int64_t n);

/* systematic delivery of every filter: c[m] = permute_parallel(
 * cumulative_offspring_to_ancestors(systematic_cumulative_offspring(w[m])))
 * (resamplers.py:127-153, ancestry.py:69-76, 139-174) with local indices;
 * offsets[m] (nullable) are the filters' u in [0,1), else own Philox draws. */
int pfr_deliver_batched(const void* w, int64_t filters, int64_t n, int dtype, const double* offsets,
                        const pfr_rng* rng, int32_t* c, int32_t* max_steps, uint32_t* status, void* ws,
                        size_t ws_bytes, void* stream);

/* the scalar linear-Gaussian model of pf.py:41-64 */
typedef struct pfr_pf_model {
  double coeff;
  double trans_std;
  double obs_std;
  double initial_mean;
  double initial_std;
} pfr_pf_model;

size_t pfr_pf_workspace_bytes(int64_t filters, int64_t n);

/* pf_run (pf.py:111-204) for `filters` independent bootstrap filters of n
 * particles over `steps` observations y[filters, steps] (device): ESS-
 * triggered systematic resampling through the in-place ancestry, propagate,
 * weight, normalise.  Outputs (device): means[filters, steps],
 * loglik[filters], ess[filters, steps] (ESS at the start of each step),
 * resampled[filters, steps].  Weight collapse sets PFR_ST_NOPROGRESS. */
int pfr_pf_run(const pfr_pf_model* model, const double* y, int64_t filters, int64_t n, int64_t steps,
               double ess_threshold, const pfr_rng* rng, double* means, double* loglik, double* ess,
               uint8_t* resampled, uint32_t* status, void* ws, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PFR_H_ */
