// Internal declarations shared by the .cu translation units of libpfr.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/pfr.h"
#include "pfr_rng.cuh"

namespace pfr {

// ---------------------------------------------------------------------------
// workspace layout (one layout for every op; sized by n and the widest dtype)
struct WsHeader {
  unsigned int ticket[8];  // tile tickets (start at 0xFFFFFFFF: +1 wraps to 0)
  unsigned int done[8];    // last-block counters
  uint64_t cell[8];        // scalar cells (Cell<A> encoded): [0] total W[N-1]
  int32_t overflow;        // chain walk overflow marker (0xFFFFFFFF = none)
  int32_t pad[15];
};

// state of the fused delivery pipeline: zero at workspace allocation, kept
// consistent by the kernels themselves (never memset per call)
struct DvState {
  unsigned int done;   // K1 groups finished (the last one resets it)
  unsigned int flags;  // 1 = O needs the running-max repair, 2 = chain overflow
  unsigned int pad[62];
  unsigned int gcnt[8192];  // K1 tiles finished per group of 64 tiles (self-resetting)
};

struct Workspace {
  DvState* dv;
  WsHeader* hdr;
  uint64_t* sum_cells;  // lookback sum tree
  uint64_t* max_cells;  // lookback max tree
  uint64_t* sub_cells;  // [8 * tiles] subtile aggregates (fused delivery)
  int64_t tiles;
  int32_t* O;  // cumulative offspring scratch
  int32_t* d;  // claims
  int32_t* a;  // sorted ancestry scratch (fallback)
  int32_t* j0;
  int32_t* j1;
  int32_t* r0;
  int32_t* r1;
  double* f0;  // N+1 doubles (multinomial / logweights scratch)
  double* f1;  // N doubles
  size_t reset_bytes;  // header + trees: memset to 0xFF before each op
  size_t bytes;
};

size_t workspace_bytes(int64_t n);
bool workspace_carve(void* base, size_t bytes, int64_t n, Workspace& ws);
cudaError_t workspace_reset(const Workspace& ws, cudaStream_t s);

// launch accounting (pfr_launch_count)
void note_launch(int k = 1);

// ---------------------------------------------------------------------------
// launchers (pfr_scan.cu)
cudaError_t launch_scan(const void* in, void* out, int64_t n, int dtype, int out_dtype, int accum, int exclusive,
                        void* total, int64_t expect_total, uint32_t* status, const Workspace& ws, cudaStream_t s);
cudaError_t launch_offspring(const void* w, int64_t n, int dtype, int accum, int stratified, double offset,
                             const double* uniforms, const pfr_rng* rng, int32_t* O, uint32_t* status,
                             const Workspace& ws, cudaStream_t s);
cudaError_t launch_deliver(const void* w, int64_t n, int dtype, int accum, int stratified, double offset,
                           const double* uniforms, const pfr_rng* rng, int32_t* c, int32_t* O_out,
                           int32_t* max_steps, uint32_t* status, const Workspace& ws, cudaStream_t s, int logw = 0);
cudaError_t launch_check_weights(const void* w, int64_t n, int dtype, uint32_t* status, cudaStream_t s);
// serial (np.cumsum-exact) inclusive scan of a weight vector in its own dtype, with check_weights' flags;
// resets the delivery pipeline flags in `state` when given
cudaError_t launch_serial_weights_scan(const void* w, void* W, int64_t n, int dtype, uint32_t* status, DvState* state,
                                      cudaStream_t s);
cudaError_t launch_adjacent_difference(const void* in, void* out, int64_t n, int dtype, int out_dtype,
                                       uint32_t* status, cudaStream_t s);
cudaError_t launch_logw_max(const void* lw, int64_t n, int dtype, unsigned long long* cell, uint32_t* status,
                            cudaStream_t s);
cudaError_t launch_logweights(const void* lw, void* w, int64_t n, int dtype, uint32_t* status, const Workspace& ws,
                              cudaStream_t s);

// launchers (pfr_ancestry.cu)
cudaError_t launch_permute_cumulative(const int32_t* O, int64_t n, int32_t* c, int32_t* max_steps, uint32_t* status,
                                      const Workspace& ws, cudaStream_t s);
cudaError_t launch_claims_reset(int64_t n, int32_t* max_steps, const Workspace& ws, cudaStream_t s);
cudaError_t launch_walk(const int32_t* a, int64_t n, int32_t* c, int32_t* max_steps, uint32_t* status,
                        const Workspace& ws, cudaStream_t s);
cudaError_t launch_permute_range(const int32_t* a, int64_t n, int64_t c_begin, int64_t c_count, int32_t* c,
                                 int32_t* max_steps, uint32_t* status, const Workspace& ws, cudaStream_t s);
cudaError_t launch_permute(const void* a, int64_t n, int idx_dtype, int32_t* c, int32_t* max_steps,
                           uint32_t* status, const Workspace& ws, cudaStream_t s);
cudaError_t launch_prepermute(const void* a, int64_t n, int idx_dtype, int32_t* d, uint32_t* status,
                              cudaStream_t s);
cudaError_t launch_expand(const void* O, int64_t n, int idx_dtype, int32_t* a, uint32_t* status, bool validate,
                          cudaStream_t s);
cudaError_t launch_histogram(const void* a, int64_t n, int idx_dtype, int32_t* o, uint32_t* status, cudaStream_t s);
cudaError_t launch_predicate(const void* c, int64_t n, int idx_dtype, int32_t* result, uint32_t* status,
                             const Workspace& ws, cudaStream_t s);
cudaError_t launch_copy_particles(double* x, int64_t n, int64_t width, const int32_t* c, cudaStream_t s);

// launchers (pfr_resample.cu)
cudaError_t launch_lower_bound(const void* W, int64_t n, int dtype, const double* u, int64_t m, int32_t* out,
                               cudaStream_t s);
cudaError_t launch_multinomial(const void* w, int64_t n, int dtype, int accum, const pfr_rng* rng,
                               const double* uniforms, int sorted_serial, int32_t* a, uint32_t* status,
                               const Workspace& ws, cudaStream_t s, int64_t s_begin = 0, int64_t s_count = -1,
                               int32_t* claim = nullptr);
cudaError_t launch_metropolis(const void* w, int64_t n, int dtype, int64_t steps, const pfr_rng* rng,
                              const double* u_draws, const void* j_draws, int idx_dtype, int32_t* a,
                              uint32_t* status, cudaStream_t s, int64_t c_begin = 0, int64_t c_count = -1, int32_t* claim = nullptr);
cudaError_t launch_rejection(const void* w, int64_t n, int dtype, double bound, double cap, const pfr_rng* rng,
                             int64_t max_rounds, int32_t* a, int32_t* trips, void* out_w, uint32_t* status,
                             const Workspace& ws, cudaStream_t s, int64_t s_begin = 0,
                             int64_t s_count = -1, int32_t* claim = nullptr);

// launcher (pfr_rejreplay.cu): rejection on the reference's numpy stream (parity mode)
cudaError_t launch_rejection_replay(const void* w, int64_t n, int dtype, double bound, double cap,
                                    const pfr_rng* rng, int64_t max_rounds, int32_t* a, int32_t* trips, void* out_w,
                                    uint32_t* status, const Workspace& ws, cudaStream_t s);

// launchers (pfr_shard.cu): weight-sharded single filter
cudaError_t launch_shard_offspring(const double* W_loc, int64_t n_loc, int dtype, double prefix, double total,
                                   int64_t n_global, int last_global, int stratified, double offset,
                                   const double* uniforms, const pfr_rng* rng, int32_t* O, cudaStream_t s);
cudaError_t launch_shard_merge(uint32_t* ext, int64_t n_loc, int64_t H, const uint32_t* from_left,
                               const uint32_t* from_right, cudaStream_t s);
cudaError_t launch_shard_local_end(const void* w, int64_t n, int dtype, uint32_t* status, double* end,
                                   const Workspace& ws, cudaStream_t s);
cudaError_t launch_shard_produce(const void* w, int64_t n_loc, int dtype, int64_t base, int64_t n_global,
                                 const double* pt, int first, int last, int stratified, double offset,
                                 const double* uniforms, const pfr_rng* rng, uint32_t* ext, int64_t wlo, int64_t whi,
                                 uint32_t* status, const Workspace& ws, cudaStream_t s);
cudaError_t launch_shard_resolve_fast(int64_t n_loc, int dtype, int64_t base, const uint32_t* ext, int64_t wlo,
                                      int64_t whi, int32_t* c, int32_t* max_steps, uint32_t* status,
                                      const Workspace& ws, cudaStream_t s);
cudaError_t launch_shard_words(const int32_t* O, int64_t n_loc, int64_t index_base, int32_t o_begin, uint32_t* words,
                               uint8_t* has, uint32_t* status, cudaStream_t s);
cudaError_t launch_shard_resolve(const uint32_t* words, const uint8_t* has, int64_t n_loc, int64_t index_base,
                                 int32_t* c, int32_t* pend, int32_t* pend_count, int32_t* max_steps, uint32_t* status,
                                 cudaStream_t s);
cudaError_t launch_shard_advance(const int32_t* walkers, int64_t count, const uint32_t* words, int64_t n_loc,
                                 int64_t index_base, int32_t* done, int32_t* done_count, int32_t* fwd,
                                 int32_t* fwd_count, int32_t* max_steps, uint32_t* status, cudaStream_t s);
cudaError_t launch_shard_scatter(const int32_t* done, int64_t count, int64_t index_base, int64_t n_loc, int32_t* c,
                                 uint32_t* status, cudaStream_t s);

cudaError_t launch_dv_inplace(const uint32_t* words, const uint32_t* bitmap, int64_t n, int32_t* c, DvState* state,
                              uint32_t* status, cudaStream_t s, const uint32_t* seg_list = nullptr,
                              const uint32_t* seg_count = nullptr, int64_t seg_len = 0);

// launchers (pfr_batch.cu): batches of independent filters
size_t batched_workspace_bytes(int64_t M, int64_t N);
size_t pf_workspace_bytes(int64_t M, int64_t N);
cudaError_t launch_deliver_batched(const void* w, int64_t M, int64_t n, int dtype, const double* offsets,
                                   const pfr_rng* rng, int32_t* c, int32_t* max_steps, void* ws, cudaStream_t s);
cudaError_t launch_pf_run(const pfr_pf_model* model, const double* y, int64_t M, int64_t N, int64_t T,
                          double ess_threshold, const pfr_rng* rng, double* means, double* loglik, double* ess,
                          uint8_t* resampled, uint32_t* status, void* ws, cudaStream_t s);

// launchers (pfr_misc.cu)
cudaError_t launch_permute_serial(const void* a, int64_t n, int idx_dtype, int32_t* c, uint32_t* status,
                                  cudaStream_t s);
cudaError_t launch_stable_sum(const void* w, int64_t n, int dtype, void* result, void* scratch, cudaStream_t s);
cudaError_t launch_probe_gather(const void* buf, int64_t n, int elem_bytes, int64_t gathers, unsigned long long* sink,
                                cudaStream_t s);
cudaError_t launch_weight_stats(const void* w, int64_t n, int dtype, const void* o, int idx_dtype, double* out,
                                void* scratch, cudaStream_t s);

int num_sms();

}  // namespace pfr
