// capi.cu -- the C ABI of libhack.so (include/hack.h): validation, status codes,
// dispatch to the sm_100a kernels.  No CPU fallback exists: without an sm_100
// device every compute entry point returns HACK_ERR_CUDA.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "capi_util.h"
#include "internal.h"

namespace hack {

thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};
void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

hack_status_t fail(hack_status_t st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

hack_status_t cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return HACK_OK;
  return fail(HACK_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

// The compute capability of the current device, queried once per device (every call checks it).
static std::atomic<int> g_dev_cc[64];  // 0 = not queried, else 10 * major + minor

hack_status_t check_device() {
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(HACK_ERR_CUDA, "no CUDA device: %s", cudaGetErrorString(e));
  int cc = dev >= 0 && dev < 64 ? g_dev_cc[dev].load(std::memory_order_relaxed) : 0;
  if (cc == 0) {
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    cc = 10 * major + minor;
    if (dev >= 0 && dev < 64 && major > 0) g_dev_cc[dev].store(cc, std::memory_order_relaxed);
  }
  if (cc != 100)
    return fail(HACK_ERR_CUDA, "libhack is built for sm_100a (B200); device %d is sm_%d", dev, cc);
  return HACK_OK;
}

hack_status_t make_kernel_cfg(const hack_config_t* c, KernelCfg* kc) {
  hack_status_t st = hack_config_validate(c);
  if (st != HACK_OK) return st;
  kc->Hq = c->num_q_heads;
  kc->Hkv = c->num_kv_heads;
  kc->G = c->num_q_heads / c->num_kv_heads;
  kc->d = c->head_dim;
  kc->Pi = c->partition;
  kc->bits = c->kv_bits;
  kc->kv_round = c->kv_round;
  kc->q_round = c->q_round;
  kc->p_round = c->p_round;
  kc->seed = c->seed;
  kc->layer = c->layer;
  kc->head_base = c->head_base;
  kc->out_fp32 = c->out_dtype == 1;
  kc->pl = page_layout(c->head_dim, c->partition, c->kv_bits);
  kc->hq_begin = 0;
  kc->hq_count = c->num_q_heads;
  kc->kvh_begin = 0;
  kc->kvh_count = c->num_kv_heads;
  kc->qt_begin = 0;
  kc->qt_count = INT32_MAX;
  return HACK_OK;
}

hack_status_t make_cache_view(const KernelCfg& kc, const hack_kv_cache_t* c, CacheView* cv) {
  if (!c) return fail(HACK_ERR_INVALID_ARG, "cache is NULL");
  if (!c->pages || !c->v_tail || !c->block_table || !c->seq_lens || !c->rng_ids)
    return fail(HACK_ERR_INVALID_ARG, "cache has a NULL device pointer");
  if (c->page_bytes != kc.pl.page_bytes)
    return fail(HACK_ERR_SHAPE, "cache page_bytes %d != layout %d", c->page_bytes, kc.pl.page_bytes);
  if (c->num_pages <= 0 || c->max_reqs <= 0 || c->max_pages_per_req <= 0)
    return fail(HACK_ERR_SHAPE, "cache dims must be positive");
  cv->pages = c->pages;
  cv->v_tail = c->v_tail;
  cv->block_table = c->block_table;
  cv->seq_lens = c->seq_lens;
  cv->rng_ids = c->rng_ids;
  cv->num_pages = c->num_pages;
  cv->max_reqs = c->max_reqs;
  cv->max_pages_per_req = c->max_pages_per_req;
  cv->page_bytes = c->page_bytes;
  cv->num_kv_heads = kc.Hkv;
  return HACK_OK;
}

}  // namespace hack

using namespace hack;

extern "C" {

void hack_config_default(hack_config_t* c) {
  if (!c) return;
  memset(c, 0, sizeof(*c));
  c->num_q_heads = 1;
  c->num_kv_heads = 1;
  c->head_dim = 128;
  c->partition = 64;
  c->kv_bits = 2;
  c->kv_round = HACK_ROUND_STOCHASTIC;
  c->q_round = HACK_ROUND_STOCHASTIC;
  c->p_round = HACK_ROUND_NEAREST_EVEN;
  c->seed = 0x48414BULL;
  c->layer = 0;
  c->head_base = 0;
  c->out_dtype = 0;
}

hack_status_t hack_config_validate(const hack_config_t* c) {
  if (!c) return fail(HACK_ERR_INVALID_ARG, "config is NULL");
  if (c->kv_bits != 2 && c->kv_bits != 4) return fail(HACK_ERR_INVALID_ARG, "kv_bits must be 2 or 4 (got %d)", c->kv_bits);
  if (c->num_q_heads <= 0 || c->num_kv_heads <= 0) return fail(HACK_ERR_INVALID_ARG, "head counts must be positive");
  if (c->num_q_heads % c->num_kv_heads) return fail(HACK_ERR_SHAPE, "H_q %% H_kv != 0");
  if (c->num_q_heads / c->num_kv_heads > 16) return fail(HACK_ERR_UNSUPPORTED, "GQA group > 16");
  if (c->head_dim != 128) return fail(HACK_ERR_UNSUPPORTED, "head_dim must be 128 (got %d)", c->head_dim);
  if (c->partition != 32 && c->partition != 64 && c->partition != 128)
    return fail(HACK_ERR_UNSUPPORTED, "partition must be 32, 64 or 128 (got %d)", c->partition);
  if (c->head_dim % c->partition) return fail(HACK_ERR_UNSUPPORTED, "head_dim %% partition != 0");
  if ((c->kv_round != 0 && c->kv_round != 1) || (c->q_round != 0 && c->q_round != 1))
    return fail(HACK_ERR_INVALID_ARG, "bad rounding mode");
  if (c->p_round != HACK_ROUND_NEAREST_EVEN && c->p_round != HACK_ROUND_STOCHASTIC)
    return fail(HACK_ERR_INVALID_ARG, "bad P rounding mode");
  if (c->out_dtype != 0 && c->out_dtype != 1) return fail(HACK_ERR_INVALID_ARG, "out_dtype must be 0 or 1");
  if (c->layer < 0 || c->layer > 0xFFFF || c->head_base < 0 || c->head_base > 0xFFF)
    return fail(HACK_ERR_INVALID_ARG, "layer/head_base out of counter range");
  return HACK_OK;
}

int64_t hack_page_bytes(const hack_config_t* c) {
  if (hack_config_validate(c) != HACK_OK) return -1;
  return page_layout(c->head_dim, c->partition, c->kv_bits).page_bytes;
}

hack_status_t hack_page_layout(const hack_config_t* c, int64_t off[12]) {
  hack_status_t st = hack_config_validate(c);
  if (st != HACK_OK) return st;
  if (!off) return fail(HACK_ERR_INVALID_ARG, "offsets_out is NULL");
  const PageLayout L = page_layout(c->head_dim, c->partition, c->kv_bits);
  const int d = c->head_dim, Pi = c->partition, b = c->kv_bits, nb = d / Pi;
  const int64_t v[12] = {L.k_codes, (int64_t)Pi * d * b / 8, L.k_meta, (int64_t)Pi * nb * 4,
                         L.k_sums, (int64_t)Pi * nb * L.sum_bytes, L.v_codes, (int64_t)d * Pi * b / 8,
                         L.v_meta, (int64_t)d * 4, L.v_sums, (int64_t)d * L.sum_bytes};
  memcpy(off, v, sizeof(v));
  return HACK_OK;
}

const char* hack_last_error(void) { return g_last_error.c_str(); }
const char* hack_version(void) { return "libhack 0.1 (sm_100a)"; }
int32_t hack_abi_version(void) { return HACK_ABI_VERSION; }
int64_t hack_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

hack_status_t hack_quantize_pack(const hack_config_t* cfg, int32_t mode, const void* x, int64_t rows,
                                 int32_t heads, int64_t pos0, int32_t head0, uint32_t rng_id, uint8_t* codes,
                                 void* meta, void* sums, void* stream) {
  KernelCfg kc;
  hack_status_t st = make_kernel_cfg(cfg, &kc);
  if (st != HACK_OK) return st;
  if (!x || !codes || !meta || !sums) return fail(HACK_ERR_INVALID_ARG, "quantize_pack: NULL pointer");
  if (mode != HACK_QMODE_K && mode != HACK_QMODE_V && mode != HACK_QMODE_Q)
    return fail(HACK_ERR_INVALID_ARG, "quantize_pack: bad mode %d", mode);
  if (rows <= 0 || heads <= 0) return fail(HACK_ERR_INVALID_ARG, "quantize_pack: empty input (S:45)");
  if (pos0 < 0 || head0 < 0) return fail(HACK_ERR_INVALID_ARG, "quantize_pack: negative position/head");
  if (mode == HACK_QMODE_V && (rows % kc.Pi || pos0 % 4))
    return fail(HACK_ERR_SHAPE, "quantize_pack V: rows must be a multiple of Pi and pos0 of 4");
  if ((st = check_device()) != HACK_OK) return st;
  return cuda_status(launch_quantize_pack(kc, mode, x, rows, heads, pos0, head0, rng_id, codes, meta, sums,
                                          (cudaStream_t)stream),
                     "quantize_pack");
}

}  // extern "C"

namespace hack {
namespace {

// Argument checks of each compute step, run in full before ANY launch of a combined call
// (hack.h: "argument errors are detected on the host before any launch"), so a rejected
// call never leaves the cache half-updated.
hack_status_t check_ingest(const KernelCfg& kc, const hack_kv_cache_t* cache, const void* k, const void* v,
                           const int32_t* cu, const int32_t* slots, int batch, int max_seqlen) {
  if (!k || !v || !cu || !slots) return fail(HACK_ERR_INVALID_ARG, "ingest: NULL pointer");
  if (batch <= 0 || max_seqlen <= 0) return fail(HACK_ERR_INVALID_ARG, "ingest: empty batch/prompt (S:303)");
  if ((max_seqlen + kc.Pi - 1) / kc.Pi > cache->max_pages_per_req)
    return fail(HACK_ERR_CAPACITY, "ingest: max_seqlen needs more pages than max_pages_per_req");
  if (batch > cache->max_reqs) return fail(HACK_ERR_CAPACITY, "ingest: batch > max_reqs");
  return HACK_OK;
}

hack_status_t check_debug(const KernelCfg& kc, const hack_debug_t* dbg, int max_seqlen, int op, const char* who) {
  if (!dbg) return HACK_OK;
  if (dbg->pcodes && dbg->pcodes_stride < max_seqlen)
    return fail(HACK_ERR_SHAPE, "%s: debug pcodes_stride < max_seqlen", who);
  if (dbg->qk_acc || dbg->pv_acc) {
    if (debug_acc_form(kc, op) == HACK_ACC_NONE)
      return fail(HACK_ERR_UNSUPPORTED, "%s: the kernel serving this config has no accumulator dump", who);
    if (dbg->acc_stride < max_seqlen || dbg->acc_stride % kc.Pi)
      return fail(HACK_ERR_SHAPE, "%s: debug acc_stride must be >= max_seqlen and a multiple of Pi", who);
    if (dbg->acc_head < -1 || dbg->acc_head >= kc.Hq)
      return fail(HACK_ERR_INVALID_ARG, "%s: debug acc_head out of range", who);
  }
  return HACK_OK;
}

hack_status_t check_prefill(const KernelCfg& kc, const hack_kv_cache_t* cache, const void* q, const int32_t* cu,
                            const int32_t* slots, int batch, int max_seqlen, const void* out, const void* ws,
                            size_t ws_bytes, const hack_debug_t* dbg) {
  if (!q || !cu || !slots || !out) return fail(HACK_ERR_INVALID_ARG, "prefill: NULL pointer");
  if (batch <= 0 || max_seqlen <= 0) return fail(HACK_ERR_INVALID_ARG, "prefill: empty batch/prompt (S:303)");
  if ((max_seqlen + kc.Pi - 1) / kc.Pi > cache->max_pages_per_req)
    return fail(HACK_ERR_CAPACITY, "prefill: max_seqlen needs more pages than max_pages_per_req");
  const size_t need = prefill_workspace_bytes(kc, batch, max_seqlen);
  if (ws_bytes < need || (need && !ws)) return fail(HACK_ERR_CAPACITY, "prefill: workspace %zu < %zu", ws_bytes, need);
  if (kc.p_round == HACK_ROUND_STOCHASTIC && !p_sr_supported(kc, 0))
    return fail(HACK_ERR_UNSUPPORTED, "prefill: P stochastic rounding needs the tcgen05 kernel (Pi = 64)");
  return check_debug(kc, dbg, max_seqlen, 0, "prefill");
}

hack_status_t check_append(const hack_kv_cache_t* cache, const void* k_new, const void* v_new, const int32_t* slots,
                           int batch) {
  if (!k_new || !v_new || !slots) return fail(HACK_ERR_INVALID_ARG, "decode_append: NULL pointer");
  if (batch <= 0) return fail(HACK_ERR_INVALID_ARG, "decode_append: empty batch");
  if (batch > cache->max_reqs) return fail(HACK_ERR_CAPACITY, "decode_append: batch > max_reqs");
  return HACK_OK;
}

hack_status_t check_decode(const KernelCfg& kc, const hack_kv_cache_t* cache, const void* q_new, const int32_t* slots,
                           int batch, int max_seqlen, const void* out, const void* ws, size_t ws_bytes,
                           const hack_debug_t* dbg) {
  if (!q_new || !slots || !out) return fail(HACK_ERR_INVALID_ARG, "decode: NULL pointer");
  if (batch <= 0 || max_seqlen <= 0) return fail(HACK_ERR_INVALID_ARG, "decode: empty batch");
  if ((max_seqlen + kc.Pi - 1) / kc.Pi > cache->max_pages_per_req)
    return fail(HACK_ERR_CAPACITY, "decode: max_seqlen needs more pages than max_pages_per_req");
  const size_t need = decode_workspace_bytes(kc, batch, max_seqlen);
  if (ws_bytes < need || (need && !ws)) return fail(HACK_ERR_CAPACITY, "decode: workspace %zu < %zu", ws_bytes, need);
  if (kc.p_round == HACK_ROUND_STOCHASTIC && !p_sr_supported(kc, 1))
    return fail(HACK_ERR_UNSUPPORTED, "decode: P stochastic rounding needs decode_mma_kernel (G <= 8)");
  return check_debug(kc, dbg, max_seqlen, 1, "decode");
}

// Library-owned copy streams and events of the host-buffer prefill (one set per device; the
// enqueue sequence of a call holds the mutex, so concurrent callers do not interleave).
constexpr int kMaxChunks = 16;
constexpr int kCompStreams = 4;  // attention chunks in flight at once
struct HostPipe {
  bool init = false;
  cudaStream_t up = nullptr, down = nullptr, comp[kCompStreams] = {};
  cudaEvent_t start = nullptr, kv = nullptr, ingested = nullptr, done = nullptr, q[kMaxChunks] = {},
              o[kMaxChunks] = {};
};
std::mutex g_pipe_mu;
HostPipe g_pipe[64];

cudaError_t host_pipe(int dev, HostPipe** out) {
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  HostPipe& p = g_pipe[dev];
  if (!p.init) {
    cudaError_t e;
    if ((e = cudaStreamCreateWithFlags(&p.up, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaStreamCreateWithFlags(&p.down, cudaStreamNonBlocking)) != cudaSuccess) return e;
    for (int i = 0; i < kCompStreams; ++i)
      if ((e = cudaStreamCreateWithFlags(&p.comp[i], cudaStreamNonBlocking)) != cudaSuccess) return e;
    cudaEvent_t* evs[4] = {&p.start, &p.kv, &p.ingested, &p.done};
    for (cudaEvent_t* ev : evs)
      if ((e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) != cudaSuccess) return e;
    for (int c = 0; c < kMaxChunks; ++c) {
      if ((e = cudaEventCreateWithFlags(&p.q[c], cudaEventDisableTiming)) != cudaSuccess) return e;
      if ((e = cudaEventCreateWithFlags(&p.o[c], cudaEventDisableTiming)) != cudaSuccess) return e;
    }
    p.init = true;
  }
  *out = &p;
  return cudaSuccess;
}

size_t up256(size_t x) { return (x + 255) / 256 * 256; }

// Device staging of the host-buffer prefill: q, k, v, out, cu_seqlens, slots, then the
// attention workspace.
struct HostLayout {
  size_t q, k, v, out, cu, slots, ws, total;
};
HostLayout host_layout(const KernelCfg& kc, int batch, int64_t T) {
  HostLayout l;
  const size_t qb = up256((size_t)T * kc.Hq * kc.d * 2), kb = up256((size_t)T * kc.Hkv * kc.d * 2);
  const size_t ob = up256((size_t)T * kc.Hq * kc.d * (kc.out_fp32 ? 4 : 2));
  l.q = 0;
  l.k = l.q + qb;
  l.v = l.k + kb;
  l.out = l.v + kb;
  l.cu = l.out + ob;
  l.slots = l.cu + up256((size_t)(batch + 1) * 4);
  l.ws = l.slots + up256((size_t)batch * 4);
  l.total = l.ws + up256(prefill_workspace_bytes(kc, batch, (int)std::min<int64_t>(T, INT32_MAX)));
  return l;
}

}  // namespace
}  // namespace hack

extern "C" {

int32_t hack_debug_acc_form(const hack_config_t* cfg, int32_t op) {
  KernelCfg kc;
  if (make_kernel_cfg(cfg, &kc) != HACK_OK || (op != 0 && op != 1)) return HACK_ACC_NONE;
  return debug_acc_form(kc, op);
}

hack_status_t hack_cache_ingest(const hack_config_t* cfg, const void* k, const void* v, const int32_t* cu,
                                const int32_t* slots, int32_t batch, int32_t max_seqlen,
                                const hack_kv_cache_t* cache, void* stream) {
  KernelCfg kc;
  CacheView cv;
  hack_status_t st = make_kernel_cfg(cfg, &kc);
  if (st != HACK_OK) return st;
  if ((st = make_cache_view(kc, cache, &cv)) != HACK_OK) return st;
  if ((st = check_ingest(kc, cache, k, v, cu, slots, batch, max_seqlen)) != HACK_OK) return st;
  if ((st = check_device()) != HACK_OK) return st;
  return cuda_status(launch_ingest(kc, k, v, cu, slots, batch, max_seqlen, cv, (cudaStream_t)stream), "ingest");
}

size_t hack_prefill_workspace_size(const hack_config_t* cfg, int32_t batch, int32_t max_seqlen) {
  KernelCfg kc;
  if (make_kernel_cfg(cfg, &kc) != HACK_OK) return 0;
  return prefill_workspace_bytes(kc, batch, max_seqlen);
}

hack_status_t hack_prefill_attention_cached(const hack_config_t* cfg, const void* q, const int32_t* cu,
                                            const int32_t* slots, int32_t batch, int32_t max_seqlen,
                                            const hack_kv_cache_t* cache, void* out, void* ws, size_t ws_bytes,
                                            const hack_debug_t* dbg, void* stream) {
  KernelCfg kc;
  CacheView cv;
  hack_status_t st = make_kernel_cfg(cfg, &kc);
  if (st != HACK_OK) return st;
  if ((st = make_cache_view(kc, cache, &cv)) != HACK_OK) return st;
  if ((st = check_prefill(kc, cache, q, cu, slots, batch, max_seqlen, out, ws, ws_bytes, dbg)) != HACK_OK) return st;
  if ((st = check_device()) != HACK_OK) return st;
  return cuda_status(launch_prefill_attention(kc, q, cu, slots, batch, max_seqlen, cv, out, ws, dbg,
                                              (cudaStream_t)stream),
                     "prefill_attention");
}

hack_status_t hack_prefill_attention(const hack_config_t* cfg, const void* q, const void* k, const void* v,
                                     const int32_t* cu, const int32_t* slots, int32_t batch, int32_t max_seqlen,
                                     const hack_kv_cache_t* cache, void* out, void* ws, size_t ws_bytes,
                                     const hack_debug_t* dbg, void* stream) {
  KernelCfg kc;
  CacheView cv;
  hack_status_t st = make_kernel_cfg(cfg, &kc);
  if (st != HACK_OK) return st;
  if ((st = make_cache_view(kc, cache, &cv)) != HACK_OK) return st;
  if ((st = check_ingest(kc, cache, k, v, cu, slots, batch, max_seqlen)) != HACK_OK) return st;
  if ((st = check_prefill(kc, cache, q, cu, slots, batch, max_seqlen, out, ws, ws_bytes, dbg)) != HACK_OK) return st;
  if ((st = check_device()) != HACK_OK) return st;
  if ((st = cuda_status(launch_ingest(kc, k, v, cu, slots, batch, max_seqlen, cv, (cudaStream_t)stream), "ingest")) !=
      HACK_OK)
    return st;
  return cuda_status(launch_prefill_attention(kc, q, cu, slots, batch, max_seqlen, cv, out, ws, dbg,
                                              (cudaStream_t)stream, /*pdl=*/true),
                     "prefill_attention");
}

// hack_prefill_attention_host for ONE prompt, by position: K and V up, one ingest, then per
// chunk c of query positions [a, b) (whole query tiles), LAST positions first: Q rows [a, b) up
// (contiguous), the attention of those rows' query tiles (kc.qt_begin / qt_count) on a library
// compute stream, the output rows [a, b) down.  The longest causal rows start first, so the
// last chunk's attention (the shortest rows) and download are a short tail after the last
// upload.  C2 (scripts/e2e_probe.py): 1.26 ms at 8 chunks against 1.35 ms for 8 query-head
// chunks; 4 / 12 / 16 chunks 1.36 / 1.29 / 1.35 ms.  (Streaming K/V/Q rows in ascending order
// with an ingest per chunk measured 1.47 ms: the longest rows then arrive last.)
static hack_status_t prefill_host_streamed(const KernelCfg& kc, const CacheView& cv, const void* q, const void* k,
                                           const void* v, const int32_t* cu, const int32_t* slots, int max_seqlen,
                                           void* out, void* ws, const HostLayout& lay, int tile_rows, int nch_req,
                                           void* stream) {
  const int L = cu[1];
  const int nqt = (L + tile_rows - 1) / tile_rows;  // query tiles of the prompt (rank 0 = the last)
  const int nch = std::max(1, std::min(std::min(nch_req > 0 ? nch_req : 8, nqt), kMaxChunks));
  uint8_t* base = reinterpret_cast<uint8_t*>(ws);
  uint8_t *qd = base + lay.q, *kd = base + lay.k, *vd = base + lay.v, *od = base + lay.out;
  int32_t* cud = reinterpret_cast<int32_t*>(base + lay.cu);
  int32_t* sld = reinterpret_cast<int32_t*>(base + lay.slots);
  const size_t row_q = (size_t)kc.Hq * kc.d * 2, row_o = (size_t)kc.Hq * kc.d * (kc.out_fp32 ? 4 : 2);
  const size_t kvb = (size_t)L * kc.Hkv * kc.d * 2;
  cudaStream_t s0 = (cudaStream_t)stream;
  int dev = 0;
  hack_status_t st;
  if ((st = cuda_status(cudaGetDevice(&dev), "prefill_host")) != HACK_OK) return st;
  std::lock_guard<std::mutex> lock(g_pipe_mu);
  HostPipe* p = nullptr;
  if ((st = cuda_status(host_pipe(dev, &p), "prefill_host: streams")) != HACK_OK) return st;
  auto chk = [](cudaError_t e) { return cuda_status(e, "prefill_host"); };
  if ((st = chk(cudaEventRecord(p->start, s0))) != HACK_OK) return st;
  if ((st = chk(cudaStreamWaitEvent(p->up, p->start, 0))) != HACK_OK) return st;
  if ((st = chk(cudaStreamWaitEvent(p->down, p->start, 0))) != HACK_OK) return st;
  if ((st = chk(cudaMemcpyAsync(cud, cu, 2 * 4, cudaMemcpyHostToDevice, p->up))) != HACK_OK) return st;
  if ((st = chk(cudaMemcpyAsync(sld, slots, 4, cudaMemcpyHostToDevice, p->up))) != HACK_OK) return st;
  if ((st = chk(cudaMemcpyAsync(kd, k, kvb, cudaMemcpyHostToDevice, p->up))) != HACK_OK) return st;
  if ((st = chk(cudaMemcpyAsync(vd, v, kvb, cudaMemcpyHostToDevice, p->up))) != HACK_OK) return st;
  if ((st = chk(cudaEventRecord(p->kv, p->up))) != HACK_OK) return st;
  if ((st = chk(cudaStreamWaitEvent(s0, p->kv, 0))) != HACK_OK) return st;
  if ((st = chk(launch_ingest(kc, kd, vd, cud, sld, 1, max_seqlen, cv, s0))) != HACK_OK) return st;
  if ((st = chk(cudaEventRecord(p->ingested, s0))) != HACK_OK) return st;
  for (int i = 0; i < std::min(nch, kCompStreams); ++i)
    if ((st = chk(cudaStreamWaitEvent(p->comp[i], p->ingested, 0))) != HACK_OK) return st;
  for (int c = 0; c < nch; ++c) {
    // ranks [r0, r1) = query tiles of positions [a, b), rank 0 = the last tile
    const int r0 = (int)((int64_t)c * nqt / nch), r1 = (int)((int64_t)(c + 1) * nqt / nch);
    const int a = (nqt - r1) * tile_rows, b = std::min(L, (nqt - r0) * tile_rows);
    if ((st = chk(cudaMemcpyAsync(qd + a * row_q, reinterpret_cast<const uint8_t*>(q) + a * row_q, (b - a) * row_q,
                                  cudaMemcpyHostToDevice, p->up))) != HACK_OK)
      return st;
    if ((st = chk(cudaEventRecord(p->q[c], p->up))) != HACK_OK) return st;
    cudaStream_t cs = p->comp[c % kCompStreams];
    if ((st = chk(cudaStreamWaitEvent(cs, p->q[c], 0))) != HACK_OK) return st;
    KernelCfg kca = kc;
    kca.qt_begin = r0;
    kca.qt_count = r1 - r0;
    if ((st = chk(launch_prefill_attention(kca, qd, cud, sld, 1, max_seqlen, cv, od, base + lay.ws, nullptr, cs))) !=
        HACK_OK)
      return st;
    if ((st = chk(cudaEventRecord(p->o[c], cs))) != HACK_OK) return st;
    if ((st = chk(cudaStreamWaitEvent(p->down, p->o[c], 0))) != HACK_OK) return st;
    if ((st = chk(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(out) + a * row_o, od + a * row_o, (b - a) * row_o,
                                  cudaMemcpyDeviceToHost, p->down))) != HACK_OK)
      return st;
  }
  // the caller's stream completes after the last download (which follows every chunk's
  // attention through the o[c] events)
  if ((st = chk(cudaEventRecord(p->done, p->down))) != HACK_OK) return st;
  return chk(cudaStreamWaitEvent(s0, p->done, 0));
}

size_t hack_prefill_host_workspace_size(const hack_config_t* cfg, int32_t batch, int32_t total_tokens) {
  KernelCfg kc;
  if (make_kernel_cfg(cfg, &kc) != HACK_OK || batch <= 0 || total_tokens <= 0) return 0;
  return host_layout(kc, batch, total_tokens).total;
}

hack_status_t hack_prefill_attention_host(const hack_config_t* cfg, const void* q, const void* k, const void* v,
                                          const int32_t* cu, const int32_t* slots, int32_t batch, int32_t max_seqlen,
                                          const hack_kv_cache_t* cache, void* out, void* ws, size_t ws_bytes,
                                          int32_t head_chunks, void* stream) {
  KernelCfg kc;
  CacheView cv;
  hack_status_t st = make_kernel_cfg(cfg, &kc);
  if (st != HACK_OK) return st;
  if ((st = make_cache_view(kc, cache, &cv)) != HACK_OK) return st;
  // every argument is checked before anything is enqueued (host pointers are only read here
  // for cu_seqlens, the token count)
  if ((st = check_ingest(kc, cache, k, v, cu, slots, batch, max_seqlen)) != HACK_OK) return st;
  if ((st = check_prefill(kc, cache, q, cu, slots, batch, max_seqlen, out, nullptr, 0, nullptr)) != HACK_OK) return st;
  const int64_t T = cu[batch];
  if (cu[0] != 0 || T <= 0) return fail(HACK_ERR_INVALID_ARG, "prefill_host: cu_seqlens must start at 0 and grow");
  for (int b = 0; b < batch; ++b)
    if (cu[b + 1] < cu[b] || cu[b + 1] - cu[b] > max_seqlen)
      return fail(HACK_ERR_INVALID_ARG, "prefill_host: cu_seqlens not increasing or a prompt > max_seqlen");
  const HostLayout lay = host_layout(kc, batch, T);
  if (!ws || ws_bytes < lay.total) return fail(HACK_ERR_CAPACITY, "prefill_host: workspace %zu < %zu", ws_bytes, lay.total);
  if ((st = check_device()) != HACK_OK) return st;
  int dev = 0;
  if ((st = cuda_status(cudaGetDevice(&dev), "prefill_host")) != HACK_OK) return st;
  // one prompt: stream it by position (below); else query-head chunks of whole GQA groups (the
  // CUDA-core baseline kernel has neither range)
  const int tile_rows = prefill_query_tile_rows(kc);
  if (batch == 1 && head_chunks <= 0 && tile_rows > 0)
    return prefill_host_streamed(kc, cv, q, k, v, cu, slots, max_seqlen, out, ws, lay, tile_rows,
                                 head_chunks < 0 ? -head_chunks : 0, stream);
  int nch = head_chunks <= 0 ? 8 : head_chunks;  // (C2: 1 / 2 / 4 / 8 chunks 1.97 / 1.52 / 1.42 / 1.37 ms)
  nch = std::max(1, std::min(std::min(nch, kc.Hkv), kMaxChunks));
  if (!prefill_head_range_supported(kc)) nch = 1;
  uint8_t* base = reinterpret_cast<uint8_t*>(ws);
  uint8_t *qd = base + lay.q, *kd = base + lay.k, *vd = base + lay.v, *od = base + lay.out;
  int32_t* cud = reinterpret_cast<int32_t*>(base + lay.cu);
  int32_t* sld = reinterpret_cast<int32_t*>(base + lay.slots);
  const size_t row_q = (size_t)kc.Hq * kc.d * 2, row_o = (size_t)kc.Hq * kc.d * (kc.out_fp32 ? 4 : 2);
  const size_t kvb = (size_t)T * kc.Hkv * kc.d * 2;
  cudaStream_t s0 = (cudaStream_t)stream;
  std::lock_guard<std::mutex> lock(g_pipe_mu);
  HostPipe* p = nullptr;
  if ((st = cuda_status(host_pipe(dev, &p), "prefill_host: streams")) != HACK_OK) return st;
  auto chk = [](cudaError_t e) { return cuda_status(e, "prefill_host"); };
  // K, V (and the small index arrays) up, then the ingest on the caller's stream
  if ((st = chk(cudaEventRecord(p->start, s0))) != HACK_OK) return st;
  if ((st = chk(cudaStreamWaitEvent(p->up, p->start, 0))) != HACK_OK) return st;
  if ((st = chk(cudaStreamWaitEvent(p->down, p->start, 0))) != HACK_OK) return st;
  if ((st = chk(cudaMemcpyAsync(cud, cu, (size_t)(batch + 1) * 4, cudaMemcpyHostToDevice, p->up))) != HACK_OK) return st;
  if ((st = chk(cudaMemcpyAsync(sld, slots, (size_t)batch * 4, cudaMemcpyHostToDevice, p->up))) != HACK_OK) return st;
  if ((st = chk(cudaMemcpyAsync(kd, k, kvb, cudaMemcpyHostToDevice, p->up))) != HACK_OK) return st;
  if ((st = chk(cudaMemcpyAsync(vd, v, kvb, cudaMemcpyHostToDevice, p->up))) != HACK_OK) return st;
  if ((st = chk(cudaEventRecord(p->kv, p->up))) != HACK_OK) return st;
  if ((st = chk(cudaStreamWaitEvent(s0, p->kv, 0))) != HACK_OK) return st;
  if ((st = chk(launch_ingest(kc, kd, vd, cud, sld, batch, max_seqlen, cv, s0))) != HACK_OK) return st;
  if ((st = chk(cudaEventRecord(p->ingested, s0))) != HACK_OK) return st;
  // the chunks' attention launches go to kCompStreams streams, so one chunk's CTAs fill the
  // SMs that the previous chunk's light items free (a head chunk alone cannot fill the GPU:
  // its longest causal rows set its duration).  (Uploading K/V per chunk of KV heads too, with
  // a per-chunk ingest (kc.kvh_begin / kvh_count), measured slower: 256-byte rows at 8 chunks
  // make the strided copies inefficient, 1.55 vs 1.37 ms.)
  for (int i = 0; i < std::min(nch, kCompStreams); ++i)
    if ((st = chk(cudaStreamWaitEvent(p->comp[i], p->ingested, 0))) != HACK_OK) return st;
  for (int c = 0; c < nch; ++c) {
    cudaStream_t cs = p->comp[c % kCompStreams];
    const int h0 = (int)((int64_t)c * kc.Hkv / nch) * kc.G, h1 = (int)((int64_t)(c + 1) * kc.Hkv / nch) * kc.G;
    const size_t qoff = (size_t)h0 * kc.d * 2, qw = (size_t)(h1 - h0) * kc.d * 2;
    const size_t ooff = (size_t)h0 * kc.d * (kc.out_fp32 ? 4 : 2), ow = (size_t)(h1 - h0) * kc.d * (kc.out_fp32 ? 4 : 2);
    // Q of heads [h0, h1) up (strided rows), attention of those heads, their output down
    if ((st = chk(cudaMemcpy2DAsync(qd + qoff, row_q, reinterpret_cast<const uint8_t*>(q) + qoff, row_q, qw, (size_t)T,
                                    cudaMemcpyHostToDevice, p->up))) != HACK_OK)
      return st;
    if ((st = chk(cudaEventRecord(p->q[c], p->up))) != HACK_OK) return st;
    if ((st = chk(cudaStreamWaitEvent(cs, p->q[c], 0))) != HACK_OK) return st;
    KernelCfg kcc = kc;
    kcc.hq_begin = nch > 1 ? h0 : 0;
    kcc.hq_count = nch > 1 ? h1 - h0 : kc.Hq;
    if ((st = chk(launch_prefill_attention(kcc, qd, cud, sld, batch, max_seqlen, cv, od, base + lay.ws, nullptr, cs))) !=
        HACK_OK)
      return st;
    if ((st = chk(cudaEventRecord(p->o[c], cs))) != HACK_OK) return st;
    if ((st = chk(cudaStreamWaitEvent(p->down, p->o[c], 0))) != HACK_OK) return st;
    if ((st = chk(cudaMemcpy2DAsync(reinterpret_cast<uint8_t*>(out) + ooff, row_o, od + ooff, row_o, ow, (size_t)T,
                                    cudaMemcpyDeviceToHost, p->down))) != HACK_OK)
      return st;
  }
  // the caller's stream completes after the last download (which follows every chunk's
  // attention through the o[c] events)
  if ((st = chk(cudaEventRecord(p->done, p->down))) != HACK_OK) return st;
  return chk(cudaStreamWaitEvent(s0, p->done, 0));
}

hack_status_t hack_decode_append(const hack_config_t* cfg, const void* k_new, const void* v_new,
                                 const int32_t* slots, int32_t batch, const hack_kv_cache_t* cache, void* stream) {
  KernelCfg kc;
  CacheView cv;
  hack_status_t st = make_kernel_cfg(cfg, &kc);
  if (st != HACK_OK) return st;
  if ((st = make_cache_view(kc, cache, &cv)) != HACK_OK) return st;
  if ((st = check_append(cache, k_new, v_new, slots, batch)) != HACK_OK) return st;
  if ((st = check_device()) != HACK_OK) return st;
  return cuda_status(launch_append(kc, k_new, v_new, slots, batch, cv, (cudaStream_t)stream), "decode_append");
}

size_t hack_decode_workspace_size(const hack_config_t* cfg, int32_t batch, int32_t max_seqlen) {
  KernelCfg kc;
  if (make_kernel_cfg(cfg, &kc) != HACK_OK) return 0;
  return decode_workspace_bytes(kc, batch, max_seqlen);
}

hack_status_t hack_decode_attention_cached(const hack_config_t* cfg, const void* q_new, const int32_t* slots,
                                           int32_t batch, int32_t max_seqlen, const hack_kv_cache_t* cache,
                                           void* out, void* ws, size_t ws_bytes, const hack_debug_t* dbg,
                                           void* stream) {
  KernelCfg kc;
  CacheView cv;
  hack_status_t st = make_kernel_cfg(cfg, &kc);
  if (st != HACK_OK) return st;
  if ((st = make_cache_view(kc, cache, &cv)) != HACK_OK) return st;
  if ((st = check_decode(kc, cache, q_new, slots, batch, max_seqlen, out, ws, ws_bytes, dbg)) != HACK_OK) return st;
  if ((st = check_device()) != HACK_OK) return st;
  return cuda_status(launch_decode_attention(kc, q_new, slots, batch, max_seqlen, cv, out, ws, dbg,
                                             (cudaStream_t)stream),
                     "decode_attention");
}

hack_status_t hack_decode_attention(const hack_config_t* cfg, const void* q_new, const void* k_new,
                                    const void* v_new, const int32_t* slots, int32_t batch, int32_t max_seqlen,
                                    const hack_kv_cache_t* cache, void* out, void* ws, size_t ws_bytes,
                                    const hack_debug_t* dbg, void* stream) {
  KernelCfg kc;
  CacheView cv;
  hack_status_t st = make_kernel_cfg(cfg, &kc);
  if (st != HACK_OK) return st;
  if ((st = make_cache_view(kc, cache, &cv)) != HACK_OK) return st;
  if ((st = check_append(cache, k_new, v_new, slots, batch)) != HACK_OK) return st;
  if ((st = check_decode(kc, cache, q_new, slots, batch, max_seqlen, out, ws, ws_bytes, dbg)) != HACK_OK) return st;
  if ((st = check_device()) != HACK_OK) return st;
  return cuda_status(launch_decode_step(kc, q_new, k_new, v_new, slots, batch, max_seqlen, cv, out, ws, dbg,
                                        (cudaStream_t)stream),
                     "decode_attention");
}

hack_status_t hack_dequantize_cache(const hack_config_t* cfg, const int32_t* slots, int32_t batch,
                                    int32_t max_seqlen, const hack_kv_cache_t* cache, void* k_out, void* v_out,
                                    void* stream) {
  KernelCfg kc;
  CacheView cv;
  hack_status_t st = make_kernel_cfg(cfg, &kc);
  if (st != HACK_OK) return st;
  if ((st = make_cache_view(kc, cache, &cv)) != HACK_OK) return st;
  if (!slots || !k_out || !v_out) return fail(HACK_ERR_INVALID_ARG, "dequantize_cache: NULL pointer");
  if (batch <= 0 || max_seqlen <= 0) return fail(HACK_ERR_INVALID_ARG, "dequantize_cache: empty batch");
  if ((max_seqlen + kc.Pi - 1) / kc.Pi > cache->max_pages_per_req)
    return fail(HACK_ERR_CAPACITY, "dequantize_cache: max_seqlen needs more pages than max_pages_per_req");
  if ((st = check_device()) != HACK_OK) return st;
  return cuda_status(launch_dequantize_cache(kc, slots, batch, max_seqlen, cv, k_out, v_out, (cudaStream_t)stream),
                     "dequantize_cache");
}

hack_status_t hack_homomorphic_matmul(const hack_config_t* cfg, const uint8_t* a_codes, const float* a_meta,
                                      const uint16_t* a_sums, const uint8_t* b_packed, const void* b_meta,
                                      const void* b_sums, int32_t M, int32_t N, int32_t Z, int32_t* d_blocks,
                                      float* c, void* stream) {
  KernelCfg kc;
  hack_status_t st = make_kernel_cfg(cfg, &kc);
  if (st != HACK_OK) return st;
  if (!a_codes || !a_meta || !a_sums || !b_packed || !b_meta || !b_sums || !c)
    return fail(HACK_ERR_INVALID_ARG, "homomorphic_matmul: NULL pointer");
  if (M <= 0 || N <= 0 || Z <= 0) return fail(HACK_ERR_INVALID_ARG, "homomorphic_matmul: empty shape");
  if (Z % kc.Pi) return fail(HACK_ERR_SHAPE, "homomorphic_matmul: Z %% Pi != 0 (S:143)");
  if ((st = check_device()) != HACK_OK) return st;
  return cuda_status(launch_homomorphic_matmul(kc, a_codes, a_meta, a_sums, b_packed, b_meta, b_sums, M, N, Z,
                                               d_blocks, c, (cudaStream_t)stream),
                     "homomorphic_matmul");
}

}  // extern "C"
