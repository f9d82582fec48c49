// extern "C" boundary of libpfr (declared in include/pfr.h).
//
// Host-side responsibilities only: argument checks, workspace carving, kernel
// launch sequencing on the caller's stream, error mapping.  No host compute on
// the data path and no device allocation.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "pfr_internal.h"
#include "pfr_tile.cuh"

namespace pfr {

namespace {
thread_local std::string g_last_error;
thread_local uint64_t g_launches = 0;

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Layout {
  size_t dv, hdr, sum, max, sub, O, d, a, scratch, end;
};

Layout layout(int64_t n) {
  Layout L;
  const int64_t tiles = num_tiles(n < 1 ? 1 : n);
  const size_t cells = (size_t)(Tree::cells_needed(tiles) + 2) * sizeof(uint64_t);
  size_t off = 0;
  L.dv = off;
  off = align_up(off + sizeof(DvState), 256);
  L.hdr = off;
  off = align_up(off + sizeof(WsHeader), 256);
  L.sum = off;
  off = align_up(off + cells, 256);
  L.max = off;
  off = align_up(off + cells, 256);
  L.sub = off;  // per-subtile (512 elements) aggregates of the fused delivery
  off = align_up(off + (size_t)(tiles * 8 + 16) * sizeof(uint64_t), 256);
  const size_t reset_end = off;
  (void)reset_end;
  L.O = off;
  off = align_up(off + (size_t)n * 4, 256);
  L.d = off;
  off = align_up(off + (size_t)n * 4, 256);
  L.a = off;
  off = align_up(off + (size_t)n * 4, 256);
  L.scratch = off;  // 4 x N int32 (fallback) or 2 x (N+1) float64 (multinomial)
  off = align_up(off + (size_t)(n + 1) * 16, 256);
  L.end = off;
  return L;
}

size_t op_bytes(int op, int64_t n) {
  const Layout L = layout(n);
  switch (op) {
    case PFR_OP_SCAN:
    case PFR_OP_METROPOLIS:
    case PFR_OP_EXPAND:
    case PFR_OP_LOGWEIGHTS:
      return L.O;
    case PFR_OP_REJECTION:  // + the O region: the certain-reject table
      return L.d;
    case PFR_OP_PREDICATE:
      return L.a;
    default:
      return L.end;
  }
}

int fail(int code, const char* msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return e == cudaErrorNotSupported ? PFR_E_UNSUPPORTED : PFR_E_CUDA;
}

bool valid_n(int64_t n) { return n >= 1 && n < 0x7F000000LL; }
bool is_float(int dt) { return dt == PFR_F32 || dt == PFR_F64; }
bool is_index(int dt) { return dt == PFR_I32 || dt == PFR_I64; }

#define PFR_REQUIRE(cond, msg) \
  do {                         \
    if (!(cond)) return fail(PFR_E_ARG, msg); \
  } while (0)

#define PFR_WS(op)                                                                   \
  Workspace ws;                                                                      \
  if (!workspace_carve(ws_ptr, ws_bytes, n, ws) || ws_bytes < op_bytes(op, n))       \
    return fail(PFR_E_WORKSPACE, "workspace too small (see pfr_workspace_bytes)");

#define PFR_CHECK_LAUNCH(expr, where)          \
  do {                                         \
    cudaError_t _e = (expr);                   \
    if (_e != cudaSuccess) return cuda_fail(_e, where); \
  } while (0)

}  // namespace

void note_launch(int k) { g_launches += (uint64_t)k; }

int num_sms() {
  static thread_local int dev_cached = -1, sms = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != dev_cached) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms < 1) sms = 1;
    dev_cached = dev;
  }
  return sms;
}

size_t workspace_bytes(int64_t n) { return layout(n).end; }

bool workspace_carve(void* base, size_t bytes, int64_t n, Workspace& ws) {
  std::memset(&ws, 0, sizeof(ws));
  if (!base) return false;
  const Layout L = layout(n);
  char* b = static_cast<char*>(base);
  if (reinterpret_cast<uintptr_t>(base) % 256) return false;
  if (bytes < L.O) return false;
  ws.dv = reinterpret_cast<DvState*>(b + L.dv);
  ws.hdr = reinterpret_cast<WsHeader*>(b + L.hdr);
  ws.tiles = num_tiles(n);
  ws.sum_cells = reinterpret_cast<uint64_t*>(b + L.sum);
  ws.max_cells = reinterpret_cast<uint64_t*>(b + L.max);
  ws.sub_cells = reinterpret_cast<uint64_t*>(b + L.sub);
  ws.reset_bytes = L.O - L.hdr;
  ws.bytes = bytes;
  if (bytes >= L.d) ws.O = reinterpret_cast<int32_t*>(b + L.O);
  if (bytes >= L.a) ws.d = reinterpret_cast<int32_t*>(b + L.d);
  if (bytes >= L.scratch) ws.a = reinterpret_cast<int32_t*>(b + L.a);
  if (bytes >= L.end) {
    int32_t* sc = reinterpret_cast<int32_t*>(b + L.scratch);
    const size_t q = align_up((size_t)(n + 1) * 4, 256) / 4;  // int32 elements per quarter
    ws.j0 = sc;
    ws.j1 = sc + q;
    ws.r0 = sc + 2 * q;
    ws.r1 = sc + 3 * q;
    ws.f0 = reinterpret_cast<double*>(sc);
    ws.f1 = reinterpret_cast<double*>(sc + 2 * q);
  }
  return true;
}

cudaError_t workspace_reset(const Workspace& ws, cudaStream_t s) {
  return cudaMemsetAsync(ws.hdr, 0xFF, ws.reset_bytes, s);
}

}  // namespace pfr

using namespace pfr;

extern "C" {

int pfr_abi_version(void) { return PFR_ABI_VERSION; }

const char* pfr_last_error(void) { return g_last_error.c_str(); }

size_t pfr_workspace_bytes(int op, int64_t n, int dtype) {
  (void)dtype;
  if (n < 1) n = 1;
  if (op == PFR_OP_ANY) return workspace_bytes(n);
  return op_bytes(op, n);
}

double pfr_stream_uniform(const pfr_rng* rng, uint64_t index, uint32_t tag) {
  if (!rng) return 0.0;
  if (rng->mode == PFR_RNG_NUMPY) return u64_to_unit(numpy_raw64(Key2x64{rng->key0, rng->key1}, index));
  uint32_t o[4];
  philox4x32_10((uint32_t)index, (uint32_t)(index >> 32), tag, 0, (uint32_t)rng->key0, (uint32_t)(rng->key0 >> 32), o);
  return u64_to_unit(((uint64_t)o[0] << 32) | o[1]);
}

uint64_t pfr_launch_count(int reset) {
  const uint64_t v = g_launches;
  if (reset) g_launches = 0;
  return v;
}

int pfr_scan(const void* in, void* out, int64_t n, int dtype, int out_dtype, int accum, int exclusive, void* total,
             uint32_t* status, void* ws_ptr, size_t ws_bytes, void* stream) {
  PFR_REQUIRE(valid_n(n), "n must be in [1, 2^31)");
  PFR_REQUIRE(in && out, "null array");
  PFR_REQUIRE(is_float(dtype) || is_index(dtype), "unsupported dtype");
  if (is_float(dtype))
    PFR_REQUIRE(out_dtype == dtype || (dtype == PFR_F32 && out_dtype == PFR_F64),
                "float scan keeps the input dtype (or widens float32 to float64)");
  if (is_index(dtype)) PFR_REQUIRE(is_index(out_dtype), "integer scan needs an integer output");
  PFR_REQUIRE((accum & 0xFF) <= PFR_ACC_SERIAL, "unknown accumulation mode");
  PFR_WS(PFR_OP_SCAN);
  const int64_t expect = (accum & 0x200) ? n : -1;  // internal: offspring_to_cumulative sum check
  PFR_CHECK_LAUNCH(launch_scan(in, out, n, dtype, out_dtype, accum & ~0x200, exclusive, total, expect, status, ws,
                               (cudaStream_t)stream),
                   "pfr_scan");
  return PFR_OK;
}

int pfr_adjacent_difference(const void* in, void* out, int64_t n, int dtype, int out_dtype, uint32_t* status,
                            void* stream) {
  PFR_REQUIRE(valid_n(n), "n must be in [1, 2^31)");
  PFR_REQUIRE(in && out, "null array");
  PFR_REQUIRE(is_float(dtype) ? out_dtype == dtype : (is_index(dtype) && is_index(out_dtype)), "bad dtypes");
  PFR_CHECK_LAUNCH(launch_adjacent_difference(in, out, n, dtype, out_dtype, status, (cudaStream_t)stream),
                   "pfr_adjacent_difference");
  return PFR_OK;
}

int pfr_lower_bound(const void* W, int64_t n, int dtype, const double* u, int64_t m, int32_t* out, void* stream) {
  PFR_REQUIRE(valid_n(n) && m >= 0, "bad sizes");
  PFR_REQUIRE(W && (m == 0 || (u && out)), "null array");
  PFR_REQUIRE(is_float(dtype), "W must be float32 or float64");
  if (m == 0) return PFR_OK;
  PFR_CHECK_LAUNCH(launch_lower_bound(W, n, dtype, u, m, out, (cudaStream_t)stream), "pfr_lower_bound");
  return PFR_OK;
}

int pfr_check_weights(const void* w, int64_t n, int dtype, uint32_t* status, void* stream) {
  PFR_REQUIRE(valid_n(n) && w && status, "bad arguments");
  PFR_REQUIRE(is_float(dtype), "weights must be float32 or float64");
  PFR_CHECK_LAUNCH(launch_check_weights(w, n, dtype, status, (cudaStream_t)stream), "pfr_check_weights");
  return PFR_OK;
}

int pfr_logweights_to_weights(const void* lw, void* w, int64_t n, int dtype, uint32_t* status, void* ws_ptr,
                              size_t ws_bytes, void* stream) {
  PFR_REQUIRE(valid_n(n) && lw && w, "bad arguments");
  PFR_REQUIRE(is_float(dtype), "log-weights must be float32 or float64");
  PFR_WS(PFR_OP_LOGWEIGHTS);
  PFR_CHECK_LAUNCH(launch_logweights(lw, w, n, dtype, status, ws, (cudaStream_t)stream), "pfr_logweights_to_weights");
  return PFR_OK;
}

int pfr_cumulative_offspring(const void* w, int64_t n, int dtype, int accum, int stratified, double offset,
                             const double* uniforms, const pfr_rng* rng, int32_t* O, uint32_t* status, void* ws_ptr,
                             size_t ws_bytes, void* stream) {
  PFR_REQUIRE(valid_n(n) && w && O, "bad arguments");
  PFR_REQUIRE(is_float(dtype), "weights must be float32 or float64");
  if (stratified) PFR_REQUIRE(uniforms || rng, "stratified needs uniforms or an rng");
  PFR_REQUIRE(accum >= 0 && accum <= PFR_ACC_SERIAL, "unknown accumulation mode");
  PFR_WS(PFR_OP_OFFSPRING);
  PFR_CHECK_LAUNCH(launch_offspring(w, n, dtype, accum, stratified, offset, uniforms, rng, O, status, ws,
                                    (cudaStream_t)stream),
                   "pfr_cumulative_offspring");
  return PFR_OK;
}

int pfr_deliver_offspring(const void* w, int64_t n, int dtype, int accum, int stratified, double offset,
                          const double* uniforms, const pfr_rng* rng, int32_t* c, int32_t* O_out, int32_t* max_steps,
                          uint32_t* status, void* ws_ptr, size_t ws_bytes, void* stream) {
  PFR_REQUIRE(valid_n(n) && w && c, "bad arguments");
  PFR_REQUIRE(is_float(dtype), "weights must be float32 or float64");
  if (stratified) PFR_REQUIRE(uniforms || rng, "stratified needs uniforms or an rng");
  PFR_REQUIRE(accum >= 0 && accum <= PFR_ACC_SERIAL, "unknown accumulation mode");
  PFR_WS(PFR_OP_DELIVER);
  cudaStream_t s = (cudaStream_t)stream;
  int32_t* O = O_out ? O_out : ws.O;
  (void)O;
  PFR_CHECK_LAUNCH(launch_deliver(w, n, dtype, accum, stratified, offset, uniforms, rng, c, O_out, max_steps, status,
                                  ws, s),
                   "pfr_deliver_offspring");
  return PFR_OK;
}

int pfr_deliver_offspring_logw(const void* lw, int64_t n, int dtype, int accum, int stratified, double offset,
                               const double* uniforms, const pfr_rng* rng, int32_t* c, int32_t* O_out,
                               int32_t* max_steps, uint32_t* status, void* ws_ptr, size_t ws_bytes, void* stream) {
  PFR_REQUIRE(valid_n(n) && lw && c && status, "bad arguments");
  PFR_REQUIRE(is_float(dtype), "log-weights must be float32 or float64");
  if (stratified) PFR_REQUIRE(uniforms || rng, "stratified needs uniforms or an rng");
  PFR_REQUIRE(accum >= 0 && accum <= PFR_ACC_SERIAL, "unknown accumulation mode");
  PFR_WS(PFR_OP_DELIVER);
  PFR_CHECK_LAUNCH(launch_deliver(lw, n, dtype, accum, stratified, offset, uniforms, rng, c, O_out, max_steps, status,
                                  ws, (cudaStream_t)stream, 1),
                   "pfr_deliver_offspring_logw");
  return PFR_OK;
}

int pfr_deliver_metropolis(const void* w, int64_t n, int dtype, int64_t steps, const pfr_rng* rng, int32_t* c,
                           int32_t* max_steps, uint32_t* status, void* ws_ptr, size_t ws_bytes, void* stream) {
  PFR_REQUIRE(valid_n(n) && w && c && status, "bad arguments");
  PFR_REQUIRE(is_float(dtype), "weights must be float32 or float64");
  PFR_REQUIRE(steps >= 0, "number of chain steps must be non-negative");
  PFR_REQUIRE(rng && rng->mode == PFR_RNG_PHILOX, "the fused Metropolis delivery uses the PHILOX stream");
  PFR_WS(PFR_OP_DELIVER);
  cudaStream_t s = (cudaStream_t)stream;
  // claims reset, chains + claims (a in the workspace's sorted-ancestry
  // scratch), then the permute's walk
  PFR_CHECK_LAUNCH(launch_claims_reset(n, max_steps, ws, s), "pfr_deliver_metropolis");
  PFR_CHECK_LAUNCH(launch_metropolis(w, n, dtype, steps, rng, nullptr, nullptr, PFR_I32, ws.a, status, s, 0, n, ws.d),
                   "pfr_deliver_metropolis");
  PFR_CHECK_LAUNCH(launch_walk(ws.a, n, c, max_steps, status, ws, s), "pfr_deliver_metropolis");
  return PFR_OK;
}

int pfr_deliver_rejection(const void* w, int64_t n, int dtype, double bound, const pfr_rng* rng, int64_t max_rounds,
                          int32_t* c, int32_t* max_steps, uint32_t* status, void* ws_ptr, size_t ws_bytes,
                          void* stream) {
  PFR_REQUIRE(valid_n(n) && w && c && status, "bad arguments");
  PFR_REQUIRE(is_float(dtype), "weights must be float32 or float64");
  PFR_REQUIRE(rng && rng->mode == PFR_RNG_PHILOX, "the fused rejection delivery uses the PHILOX stream");
  if (!(bound > 0) || !std::isfinite(bound)) return fail(PFR_E_ARG, "weight bound must be finite and positive");
  PFR_WS(PFR_OP_DELIVER);
  cudaStream_t s = (cudaStream_t)stream;
  // claims reset, slots + claims (a in the workspace's sorted-ancestry
  // scratch), then the permute's walk
  PFR_CHECK_LAUNCH(launch_claims_reset(n, max_steps, ws, s), "pfr_deliver_rejection");
  PFR_CHECK_LAUNCH(launch_rejection(w, n, dtype, bound, 0.0, rng, max_rounds, ws.a, nullptr, nullptr, status, ws, s, 0,
                                    n, ws.d),
                   "pfr_deliver_rejection");
  PFR_CHECK_LAUNCH(launch_walk(ws.a, n, c, max_steps, status, ws, s), "pfr_deliver_rejection");
  return PFR_OK;
}

int pfr_deliver_multinomial(const void* w, int64_t n, int dtype, int accum, const pfr_rng* rng, int32_t* c,
                            int32_t* max_steps, uint32_t* status, void* ws_ptr, size_t ws_bytes, void* stream) {
  PFR_REQUIRE(valid_n(n) && w && c && status, "bad arguments");
  PFR_REQUIRE(is_float(dtype), "weights must be float32 or float64");
  PFR_REQUIRE(rng && rng->mode == PFR_RNG_PHILOX, "the fused multinomial delivery uses the PHILOX stream");
  PFR_REQUIRE(accum >= 0 && accum <= PFR_ACC_SERIAL, "unknown accumulation mode");
  PFR_WS(PFR_OP_DELIVER);
  cudaStream_t s = (cudaStream_t)stream;
  PFR_CHECK_LAUNCH(launch_claims_reset(n, max_steps, ws, s), "pfr_deliver_multinomial");
  PFR_CHECK_LAUNCH(launch_multinomial(w, n, dtype, accum, rng, nullptr, 0, ws.a, status, ws, s, 0, n, ws.d),
                   "pfr_deliver_multinomial");
  PFR_CHECK_LAUNCH(launch_walk(ws.a, n, c, max_steps, status, ws, s), "pfr_deliver_multinomial");
  return PFR_OK;
}

int pfr_multinomial(const void* w, int64_t n, int dtype, int accum, const pfr_rng* rng, const double* uniforms,
                    int sorted_serial, int32_t* a, uint32_t* status, void* ws_ptr, size_t ws_bytes, void* stream) {
  PFR_REQUIRE(valid_n(n) && w && a, "bad arguments");
  PFR_REQUIRE(is_float(dtype), "weights must be float32 or float64");
  PFR_REQUIRE(uniforms || rng, "multinomial needs uniforms or an rng");
  PFR_REQUIRE(accum >= 0 && accum <= PFR_ACC_SERIAL, "unknown accumulation mode");
  PFR_WS(PFR_OP_MULTINOMIAL);
  PFR_CHECK_LAUNCH(launch_multinomial(w, n, dtype, accum, rng, uniforms, sorted_serial, a, status, ws,
                                      (cudaStream_t)stream),
                   "pfr_multinomial");
  return PFR_OK;
}

int pfr_metropolis(const void* w, int64_t n, int dtype, int64_t steps, const pfr_rng* rng, const double* u_draws,
                   const void* j_draws, int idx_dtype, int32_t* a, uint32_t* status, void* ws_ptr, size_t ws_bytes,
                   void* stream) {
  (void)ws_ptr;
  (void)ws_bytes;
  PFR_REQUIRE(valid_n(n) && w && a, "bad arguments");
  PFR_REQUIRE(is_float(dtype), "weights must be float32 or float64");
  PFR_REQUIRE(steps >= 0, "number of chain steps must be non-negative");
  const bool arrays = !rng || rng->mode == PFR_RNG_ARRAYS;
  if (arrays) PFR_REQUIRE((u_draws && j_draws && is_index(idx_dtype)) || steps == 0, "ARRAYS mode needs u and j draws");
  PFR_CHECK_LAUNCH(launch_metropolis(w, n, dtype, steps, rng, u_draws, j_draws, idx_dtype, a, status,
                                     (cudaStream_t)stream),
                   "pfr_metropolis");
  return PFR_OK;
}

int pfr_rejection(const void* w, int64_t n, int dtype, double bound, double cap, const pfr_rng* rng,
                  int64_t max_rounds, int32_t* a, int32_t* trips, void* out_w, uint32_t* status, void* ws_ptr,
                  size_t ws_bytes, void* stream) {
  PFR_REQUIRE(valid_n(n) && w && a && status, "bad arguments");
  PFR_REQUIRE(is_float(dtype), "weights must be float32 or float64");
  PFR_REQUIRE(rng, "rejection needs an rng");
  const double b = cap > 0 ? cap : bound;
  if (!(b > 0) || !std::isfinite(b)) return fail(PFR_E_ARG, "weight bound must be finite and positive");
  if (cap > 0) PFR_REQUIRE(out_w, "capped rejection needs out_w");
  PFR_WS(PFR_OP_REJECTION);
  PFR_CHECK_LAUNCH(launch_rejection(w, n, dtype, bound, cap, rng, max_rounds, a, trips, out_w, status, ws,
                                    (cudaStream_t)stream),
                   "pfr_rejection");
  return PFR_OK;
}

int pfr_rejection_range(const void* w, int64_t n, int dtype, double bound, double cap, const pfr_rng* rng,
                        int64_t max_rounds, int64_t slot_begin, int64_t slot_count, int32_t* a, int32_t* trips,
                        void* out_w, uint32_t* status, void* ws_ptr, size_t ws_bytes, void* stream) {
  PFR_REQUIRE(valid_n(n) && w && (a || slot_count == 0) && status, "bad arguments");
  PFR_REQUIRE(is_float(dtype), "weights must be float32 or float64");
  PFR_REQUIRE(rng && rng->mode == PFR_RNG_PHILOX, "slot ranges need the PHILOX stream");
  PFR_REQUIRE(slot_begin >= 0 && slot_count >= 0 && slot_begin + slot_count <= n, "slot range outside [0, N)");
  const double b = cap > 0 ? cap : bound;
  if (!(b > 0) || !std::isfinite(b)) return fail(PFR_E_ARG, "weight bound must be finite and positive");
  if (cap > 0) PFR_REQUIRE(out_w || slot_count == 0, "capped rejection needs out_w");
  if (slot_count == 0) return PFR_OK;
  PFR_WS(PFR_OP_REJECTION);
  PFR_CHECK_LAUNCH(launch_rejection(w, n, dtype, bound, cap, rng, max_rounds, a, trips, out_w, status, ws,
                                    (cudaStream_t)stream, slot_begin, slot_count),
                   "pfr_rejection_range");
  return PFR_OK;
}

int pfr_multinomial_range(const void* w, int64_t n, int dtype, int accum, const pfr_rng* rng, const double* uniforms,
                          int64_t slot_begin, int64_t slot_count, int32_t* a, uint32_t* status, void* ws_ptr,
                          size_t ws_bytes, void* stream) {
  PFR_REQUIRE(valid_n(n) && w && (a || slot_count == 0), "bad arguments");
  PFR_REQUIRE(is_float(dtype), "weights must be float32 or float64");
  PFR_REQUIRE(uniforms || rng, "multinomial needs uniforms or an rng");
  PFR_REQUIRE(accum >= 0 && accum < PFR_ACC_SERIAL, "unknown accumulation mode");
  PFR_REQUIRE(slot_begin >= 0 && slot_count >= 0 && slot_begin + slot_count <= n, "slot range outside [0, N)");
  if (slot_count == 0) return PFR_OK;
  PFR_WS(PFR_OP_MULTINOMIAL);
  PFR_CHECK_LAUNCH(launch_multinomial(w, n, dtype, accum, rng, uniforms, 0, a, status, ws, (cudaStream_t)stream,
                                      slot_begin, slot_count),
                   "pfr_multinomial_range");
  return PFR_OK;
}

int pfr_permute_range(const int32_t* a, int64_t n, int64_t index_begin, int64_t index_count, int32_t* c,
                      int32_t* max_steps, uint32_t* status, void* ws_ptr, size_t ws_bytes, void* stream) {
  PFR_REQUIRE(valid_n(n) && a && (c || index_count == 0) && status, "bad arguments");
  PFR_REQUIRE(index_begin >= 0 && index_count >= 0 && index_begin + index_count <= n, "index range outside [0, N)");
  PFR_WS(PFR_OP_PERMUTE);
  PFR_CHECK_LAUNCH(launch_permute_range(a, n, index_begin, index_count, c, max_steps, status, ws,
                                        (cudaStream_t)stream),
                   "pfr_permute_range");
  return PFR_OK;
}

int pfr_cumulative_to_ancestors(const void* O, int64_t n, int idx_dtype, int32_t* a, uint32_t* status, void* ws_ptr,
                                size_t ws_bytes, void* stream) {
  (void)ws_ptr;
  (void)ws_bytes;
  PFR_REQUIRE(valid_n(n) && O && a, "bad arguments");
  PFR_REQUIRE(is_index(idx_dtype), "O must be int32 or int64");
  PFR_CHECK_LAUNCH(launch_expand(O, n, idx_dtype, a, status, status != nullptr, (cudaStream_t)stream),
                   "pfr_cumulative_to_ancestors");
  return PFR_OK;
}

int pfr_ancestors_to_offspring(const void* a, int64_t n, int idx_dtype, int32_t* o, uint32_t* status, void* stream) {
  PFR_REQUIRE(valid_n(n) && a && o, "bad arguments");
  PFR_REQUIRE(is_index(idx_dtype), "a must be int32 or int64");
  PFR_CHECK_LAUNCH(launch_histogram(a, n, idx_dtype, o, status, (cudaStream_t)stream), "pfr_ancestors_to_offspring");
  return PFR_OK;
}

int pfr_prepermute(const void* a, int64_t n, int idx_dtype, int32_t* d, uint32_t* status, void* stream) {
  PFR_REQUIRE(valid_n(n) && a && d, "bad arguments");
  PFR_REQUIRE(is_index(idx_dtype), "a must be int32 or int64");
  PFR_CHECK_LAUNCH(launch_prepermute(a, n, idx_dtype, d, status, (cudaStream_t)stream), "pfr_prepermute");
  return PFR_OK;
}

int pfr_permute(const void* a, int64_t n, int idx_dtype, int32_t* c, int32_t* max_steps, uint32_t* status,
                void* ws_ptr, size_t ws_bytes, void* stream) {
  PFR_REQUIRE(valid_n(n) && a && c, "bad arguments");
  PFR_REQUIRE(is_index(idx_dtype), "a must be int32 or int64");
  PFR_WS(PFR_OP_PERMUTE);
  PFR_CHECK_LAUNCH(launch_permute(a, n, idx_dtype, c, max_steps, status, ws, (cudaStream_t)stream), "pfr_permute");
  return PFR_OK;
}

int pfr_permute_cumulative(const int32_t* O, int64_t n, int32_t* c, int32_t* max_steps, uint32_t* status,
                           void* ws_ptr, size_t ws_bytes, void* stream) {
  PFR_REQUIRE(valid_n(n) && O && c, "bad arguments");
  PFR_WS(PFR_OP_DELIVER);
  PFR_CHECK_LAUNCH(launch_permute_cumulative(O, n, c, max_steps, status, ws, (cudaStream_t)stream),
                   "pfr_permute_cumulative");
  return PFR_OK;
}

int pfr_check_predicate(const void* c, int64_t n, int idx_dtype, int32_t* result, uint32_t* status, void* ws_ptr,
                        size_t ws_bytes, void* stream) {
  PFR_REQUIRE(valid_n(n) && c && result, "bad arguments");
  PFR_REQUIRE(is_index(idx_dtype), "c must be int32 or int64");
  PFR_WS(PFR_OP_PREDICATE);
  PFR_CHECK_LAUNCH(launch_predicate(c, n, idx_dtype, result, status, ws, (cudaStream_t)stream),
                   "pfr_check_predicate");
  return PFR_OK;
}

int pfr_copy_particles(double* x, int64_t n, int64_t width, const int32_t* c, void* stream) {
  PFR_REQUIRE(valid_n(n) && width >= 1 && x && c, "bad arguments");
  PFR_CHECK_LAUNCH(launch_copy_particles(x, n, width, c, (cudaStream_t)stream), "pfr_copy_particles");
  return PFR_OK;
}


/* ---- weight-sharded single filter (pfr_shard.cu) ------------------------- */

int pfr_metropolis_range(const void* w, int64_t n, int dtype, int64_t steps, const pfr_rng* rng, int64_t chain_begin,
                         int64_t chain_count, int32_t* a, uint32_t* status, void* stream) {
  PFR_REQUIRE(valid_n(n) && w && (a || chain_count == 0), "bad arguments");
  PFR_REQUIRE(is_float(dtype), "weights must be float32 or float64");
  PFR_REQUIRE(steps >= 0, "number of chain steps must be non-negative");
  PFR_REQUIRE(rng && rng->mode != PFR_RNG_ARRAYS, "chain ranges need a PHILOX or NUMPY stream");
  PFR_REQUIRE(chain_begin >= 0 && chain_count >= 0 && chain_begin + chain_count <= n, "chain range outside [0, N)");
  PFR_CHECK_LAUNCH(launch_metropolis(w, n, dtype, steps, rng, nullptr, nullptr, PFR_I64, a, status,
                                     (cudaStream_t)stream, chain_begin, chain_count),
                   "pfr_metropolis_range");
  return PFR_OK;
}

int pfr_shard_offspring(const double* W_loc, int64_t n_loc, int dtype, double prefix, double total, int64_t n_global,
                        int last_global, int stratified, double offset, const double* uniforms, const pfr_rng* rng,
                        int32_t* O, void* stream) {
  PFR_REQUIRE(valid_n(n_loc) && valid_n(n_global) && n_loc <= n_global, "bad sizes");
  PFR_REQUIRE(W_loc && O, "null array");
  PFR_REQUIRE(is_float(dtype), "weights must be float32 or float64");
  PFR_REQUIRE(std::isfinite(total) && total > 0 && std::isfinite(prefix) && prefix >= 0, "bad prefix/total");
  if (stratified) PFR_REQUIRE(uniforms || (rng && rng->mode != PFR_RNG_ARRAYS), "stratified needs uniforms or an rng");
  PFR_CHECK_LAUNCH(launch_shard_offspring(W_loc, n_loc, dtype, prefix, total, n_global, last_global, stratified, offset,
                                          uniforms, rng, O, (cudaStream_t)stream),
                   "pfr_shard_offspring");
  return PFR_OK;
}

int pfr_shard_local_end(const void* w_loc, int64_t n_loc, int dtype, double* end, uint32_t* status, void* ws_ptr,
                        size_t ws_bytes, void* stream) {
  const int64_t n = n_loc;
  PFR_REQUIRE(valid_n(n) && w_loc && end && status, "bad arguments");
  PFR_REQUIRE(is_float(dtype), "weights must be float32 or float64");
  PFR_WS(PFR_OP_DELIVER);
  PFR_CHECK_LAUNCH(launch_shard_local_end(w_loc, n, dtype, status, end, ws, (cudaStream_t)stream),
                   "pfr_shard_local_end");
  return PFR_OK;
}

int pfr_shard_produce(const void* w_loc, int64_t n_loc, int dtype, int64_t index_base, int64_t n_global,
                      const double* prefix_total, int first, int last, int stratified, double offset,
                      const double* uniforms, const pfr_rng* rng, uint32_t* ext, int64_t slot_lo, int64_t slot_hi,
                      uint32_t* status, void* ws_ptr, size_t ws_bytes, void* stream) {
  const int64_t n = n_loc;
  PFR_REQUIRE(valid_n(n) && valid_n(n_global) && index_base >= 0 && index_base + n <= n_global, "bad sizes");
  PFR_REQUIRE(w_loc && prefix_total && ext && status, "null array");
  PFR_REQUIRE(is_float(dtype), "weights must be float32 or float64");
  PFR_REQUIRE(slot_hi > slot_lo && (slot_lo & 3) == 0 && slot_lo <= index_base && slot_hi >= index_base + n,
              "the slot window must cover the shard's indices and start at a multiple of 4");
  if (stratified) PFR_REQUIRE(uniforms || rng, "stratified needs uniforms or an rng");
  PFR_WS(PFR_OP_DELIVER);
  PFR_CHECK_LAUNCH(launch_shard_produce(w_loc, n, dtype, index_base, n_global, prefix_total, first, last, stratified,
                                        offset, uniforms, rng, ext, slot_lo, slot_hi, status, ws,
                                        (cudaStream_t)stream),
                   "pfr_shard_produce");
  return PFR_OK;
}

int pfr_shard_resolve_fast(int64_t n_loc, int dtype, int64_t index_base, const uint32_t* ext, int64_t slot_lo,
                           int64_t slot_hi, int32_t* c, int32_t* max_steps, uint32_t* status, void* ws_ptr,
                           size_t ws_bytes, void* stream) {
  const int64_t n = n_loc;
  PFR_REQUIRE(valid_n(n) && index_base >= 0 && ext && c && status, "bad arguments");
  PFR_REQUIRE(slot_lo <= index_base && slot_hi >= index_base + n, "the slot window must cover the shard's indices");
  PFR_WS(PFR_OP_DELIVER);
  PFR_CHECK_LAUNCH(launch_shard_resolve_fast(n, dtype, index_base, ext, slot_lo, slot_hi, c, max_steps, status, ws,
                                             (cudaStream_t)stream),
                   "pfr_shard_resolve_fast");
  return PFR_OK;
}

int pfr_shard_merge_bands(uint32_t* ext, int64_t n_loc, int64_t halo, const uint32_t* from_left,
                          const uint32_t* from_right, void* stream) {
  PFR_REQUIRE(valid_n(n_loc) && halo >= 0, "bad sizes");
  PFR_REQUIRE(ext, "null array");
  if (halo == 0 || (!from_left && !from_right)) return PFR_OK;
  PFR_CHECK_LAUNCH(launch_shard_merge(ext, n_loc, halo, from_left, from_right, (cudaStream_t)stream),
                   "pfr_shard_merge_bands");
  return PFR_OK;
}

int pfr_shard_words(const int32_t* O_loc, int64_t n_loc, int64_t index_base, int32_t o_begin, uint32_t* words,
                    uint8_t* has, uint32_t* status, void* stream) {
  PFR_REQUIRE(valid_n(n_loc) && index_base >= 0 && o_begin >= 0, "bad sizes");
  PFR_REQUIRE(O_loc && words, "null array");
  PFR_CHECK_LAUNCH(launch_shard_words(O_loc, n_loc, index_base, o_begin, words, has, status, (cudaStream_t)stream),
                   "pfr_shard_words");
  return PFR_OK;
}

int pfr_shard_resolve(const uint32_t* words, const uint8_t* has, int64_t n_loc, int64_t index_base, int32_t* c,
                      int32_t* pend, int32_t* pend_count, int32_t* max_steps, uint32_t* status, void* stream) {
  PFR_REQUIRE(valid_n(n_loc) && index_base >= 0, "bad sizes");
  PFR_REQUIRE(words && has && c && pend && pend_count, "null array");
  PFR_CHECK_LAUNCH(launch_shard_resolve(words, has, n_loc, index_base, c, pend, pend_count, max_steps, status,
                                        (cudaStream_t)stream),
                   "pfr_shard_resolve");
  return PFR_OK;
}

int pfr_shard_advance(const int32_t* walkers, int64_t count, const uint32_t* words, int64_t n_loc, int64_t index_base,
                      int32_t* done, int32_t* done_count, int32_t* fwd, int32_t* fwd_count, int32_t* max_steps,
                      uint32_t* status, void* stream) {
  PFR_REQUIRE(count >= 0 && valid_n(n_loc) && index_base >= 0, "bad sizes");
  PFR_REQUIRE(count == 0 || (walkers && words && done && done_count && fwd && fwd_count), "null array");
  PFR_CHECK_LAUNCH(launch_shard_advance(walkers, count, words, n_loc, index_base, done, done_count, fwd, fwd_count,
                                        max_steps, status, (cudaStream_t)stream),
                   "pfr_shard_advance");
  return PFR_OK;
}

int pfr_shard_scatter(const int32_t* done, int64_t count, int64_t index_base, int64_t n_loc, int32_t* c,
                      uint32_t* status, void* stream) {
  PFR_REQUIRE(count >= 0 && valid_n(n_loc), "bad sizes");
  PFR_REQUIRE(count == 0 || (done && c), "null array");
  PFR_CHECK_LAUNCH(launch_shard_scatter(done, count, index_base, n_loc, c, status, (cudaStream_t)stream),
                   "pfr_shard_scatter");
  return PFR_OK;
}

/* ---- batches of independent filters (pfr_batch.cu) ----------------------- */

size_t pfr_batched_workspace_bytes(int64_t filters, int64_t n) {
  return batched_workspace_bytes(filters < 1 ? 1 : filters, n < 1 ? 1 : n);
}

int pfr_deliver_batched(const void* w, int64_t filters, int64_t n, int dtype, const double* offsets,
                        const pfr_rng* rng, int32_t* c, int32_t* max_steps, uint32_t* status, void* ws,
                        size_t ws_bytes, void* stream) {
  (void)status;
  PFR_REQUIRE(filters >= 1 && valid_n(n) && filters * n < 0x7F000000LL * 64, "bad sizes");
  PFR_REQUIRE(w && c && ws, "null array");
  PFR_REQUIRE(is_float(dtype), "weights must be float32 or float64");
  PFR_REQUIRE(offsets || (rng && rng->mode == PFR_RNG_PHILOX), "need offsets or a PHILOX stream");
  PFR_REQUIRE(ws_bytes >= batched_workspace_bytes(filters, n), "workspace too small (see pfr_batched_workspace_bytes)");
  PFR_CHECK_LAUNCH(launch_deliver_batched(w, filters, n, dtype, offsets, rng, c, max_steps, ws, (cudaStream_t)stream),
                   "pfr_deliver_batched");
  return PFR_OK;
}

size_t pfr_pf_workspace_bytes(int64_t filters, int64_t n) {
  return pf_workspace_bytes(filters < 1 ? 1 : filters, n < 1 ? 1 : n);
}

int pfr_pf_run(const pfr_pf_model* model, const double* y, int64_t filters, int64_t n, int64_t steps,
               double ess_threshold, const pfr_rng* rng, double* means, double* loglik, double* ess,
               uint8_t* resampled, uint32_t* status, void* ws, size_t ws_bytes, void* stream) {
  PFR_REQUIRE(model && y && means && loglik && ess && resampled && status && ws && rng, "null argument");
  PFR_REQUIRE(filters >= 1 && n >= 2 && valid_n(n) && steps >= 1, "need filters >= 1, n >= 2, steps >= 1");
  PFR_REQUIRE(model->trans_std > 0 && model->obs_std > 0 && model->initial_std > 0,
              "trans_std, obs_std and initial_std must be strictly positive");
  PFR_REQUIRE(ess_threshold >= 0.0 && ess_threshold <= 1.0, "ess_threshold must lie in [0, 1]");
  PFR_REQUIRE(ws_bytes >= pf_workspace_bytes(filters, n), "workspace too small (see pfr_pf_workspace_bytes)");
  PFR_CHECK_LAUNCH(launch_pf_run(model, y, filters, n, steps, ess_threshold, rng, means, loglik, ess, resampled, status,
                                 ws, (cudaStream_t)stream),
                   "pfr_pf_run");
  return PFR_OK;
}

/* ---- remaining reference functions (pfr_misc.cu) ------------------------- */

int pfr_permute_serial(const void* a, int64_t n, int idx_dtype, int32_t* c, uint32_t* status, void* stream) {
  PFR_REQUIRE(valid_n(n) && a && c, "bad arguments");
  PFR_REQUIRE(is_index(idx_dtype), "ancestry must be int32 or int64");
  PFR_CHECK_LAUNCH(launch_permute_serial(a, n, idx_dtype, c, status, (cudaStream_t)stream), "pfr_permute_serial");
  return PFR_OK;
}

int pfr_stable_sum(const void* w, int64_t n, int dtype, double* result, void* ws_ptr, size_t ws_bytes, void* stream) {
  PFR_REQUIRE(valid_n(n) && w && result, "bad arguments");
  PFR_REQUIRE(is_float(dtype), "stable_sum needs float32 or float64");
  PFR_WS(PFR_OP_ANY);
  PFR_CHECK_LAUNCH(launch_stable_sum(w, n, dtype, result, ws.f0, (cudaStream_t)stream), "pfr_stable_sum");
  return PFR_OK;
}

int pfr_probe_gather(const void* buf, int64_t n, int elem_bytes, int64_t gathers, unsigned long long* sink,
                     void* stream) {
  PFR_REQUIRE(buf && sink && n >= 1 && n <= (int64_t(1) << 32) && (n & (n - 1)) == 0 && gathers > 0,
              "bad arguments (n must be a power of two <= 2^32)");
  PFR_REQUIRE(elem_bytes == 4 || elem_bytes == 8, "elem_bytes must be 4 or 8");
  PFR_CHECK_LAUNCH(launch_probe_gather(buf, n, elem_bytes, gathers, sink, (cudaStream_t)stream), "pfr_probe_gather");
  return PFR_OK;
}

int pfr_weight_stats(const void* w, int64_t n, int dtype, const void* o, int idx_dtype, double* out, void* ws_ptr,
                     size_t ws_bytes, void* stream) {
  PFR_REQUIRE(valid_n(n) && w && out, "bad arguments");
  PFR_REQUIRE(is_float(dtype), "weights must be float32 or float64");
  PFR_REQUIRE(!o || is_index(idx_dtype), "offspring must be int32 or int64");
  PFR_WS(PFR_OP_ANY);
  PFR_CHECK_LAUNCH(launch_weight_stats(w, n, dtype, o, idx_dtype, out, ws.f0, (cudaStream_t)stream),
                   "pfr_weight_stats");
  return PFR_OK;
}
}  // extern "C"
