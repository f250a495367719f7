// comm.cu -- (a10) prefill -> decode KV transfer over NCCL p2p.
//
// The paper's prefill instance "transmits the first token, K', V', and the
// quantization metadata, the minimum value m and the scale value s, to the decode
// instance" with NCCL.  Here one request's pages (codes + fp16 meta +
// cached sums, reading R19) and its FP16 last-V block (RQE) for every layer
// are gathered behind a 64-byte header into one contiguous staging buffer and sent
// with a single ncclSend over NVLink/NVSwitch; the receiver validates the header on
// the device and scatters into its own pages.  Sizes are a closed form of
// (prompt_len, config), so both sides post matching sizes without a handshake.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>

#include "capi_util.h"
#include "internal.h"

namespace hack {

namespace {

constexpr uint32_t kMagic = 0x4B434148u;  // "HACK" little-endian
constexpr uint16_t kWireVersion = 1;
constexpr int kHeaderBytes = 64;
constexpr int kMaxLayers = 128;

struct WireHeader {  // 64 bytes, little-endian
  uint32_t magic;
  uint16_t version, num_layers;
  uint16_t num_kv_heads, head_dim;
  uint16_t partition;
  uint8_t kv_bits, sum_bytes;
  uint32_t prompt_len, tail_len;
  int32_t first_token;
  uint32_t rng_id;
  uint32_t page_bytes;
  uint32_t head_base;
  uint64_t payload_bytes;
  uint64_t seed;
  uint8_t pad[8];
};
static_assert(sizeof(WireHeader) == kHeaderBytes, "wire header is 64 bytes");

struct LayerPtrs {
  uint8_t* pages[kMaxLayers];
  __half* tail[kMaxLayers];
};

struct XferGeom {
  int npages, tail_len, Hkv, page_bytes, Pi, num_layers;
  int64_t layer_bytes;  // pages + tail bytes per layer
};

int64_t layer_bytes(const KernelCfg& kc, int prompt_len) {
  const int npages = (prompt_len + kc.Pi - 1) / kc.Pi;
  const int T = prompt_len % kc.Pi;
  return (int64_t)npages * kc.Hkv * kc.pl.page_bytes + (int64_t)kc.Hkv * T * 128 * 2;
}

// 16-byte copy by the whole CTA; four loads in flight per thread before their stores (the
// pointers may alias as far as the compiler knows, so a plain loop serialises load/store)
HACK_DEV void copy16(uint8_t* dst, const uint8_t* src, int64_t bytes) {
  const uint4* s = reinterpret_cast<const uint4*>(src);
  uint4* d = reinterpret_cast<uint4*>(dst);
  const int64_t n = bytes / 16, bd = blockDim.x;
  int64_t i = threadIdx.x;
  for (; i + 3 * bd < n; i += 4 * bd) {
    const uint4 a = s[i], b = s[i + bd], c = s[i + 2 * bd], e = s[i + 3 * bd];
    d[i] = a;
    d[i + bd] = b;
    d[i + 2 * bd] = c;
    d[i + 3 * bd] = e;
  }
  for (; i < n; i += bd) d[i] = s[i];
}

// grid (npages + 1, layers): block j < npages copies page j (all KV heads), block npages
// copies the FP16 tail rows; blockIdx.y = layer - layer0 (layer-pipelined send packs one).
// The header's rng_id is the cache's rng_ids[slot] (the stream the codes were drawn with, as
// hack_kv_pull copies it); a caller-supplied rng_id that disagrees poisons the header
// (magic 0), so the receiver's header check reports HACK_ERR_PROTOCOL.
__global__ void gather_kernel(LayerPtrs lp, const int32_t* __restrict__ block_table, int max_pages_per_req,
                              const uint32_t* __restrict__ rng_ids, int slot, XferGeom g, WireHeader hdr,
                              uint8_t* __restrict__ staging, int layer0) {
  const int j = blockIdx.x, l = layer0 + blockIdx.y;
  if (j == 0 && l == 0 && threadIdx.x == 0) {
    const uint32_t rid = rng_ids[slot];
    if (rid != hdr.rng_id) hdr.magic = 0u;
    hdr.rng_id = rid;
    *reinterpret_cast<WireHeader*>(staging) = hdr;
  }
  uint8_t* dst = staging + kHeaderBytes + (int64_t)l * g.layer_bytes;
  const int64_t pbytes = (int64_t)g.Hkv * g.page_bytes;
  if (j < g.npages) {
    const int pid = block_table[(int64_t)slot * max_pages_per_req + j];
    copy16(dst + j * pbytes, lp.pages[l] + pid * pbytes, pbytes);
  } else if (g.tail_len) {
    uint8_t* td = dst + g.npages * pbytes;
    const int64_t rowb = (int64_t)g.tail_len * 128 * 2;
    for (int h = 0; h < g.Hkv; ++h)
      copy16(td + h * rowb, reinterpret_cast<const uint8_t*>(lp.tail[l] + ((int64_t)slot * g.Hkv + h) * g.Pi * 128),
             rowb);
  }
}

HACK_DEV bool header_ok(const WireHeader& h, const WireHeader& e) {
  return h.magic == e.magic && h.version == e.version && h.num_layers == e.num_layers &&
         h.num_kv_heads == e.num_kv_heads && h.head_dim == e.head_dim && h.partition == e.partition &&
         h.kv_bits == e.kv_bits && h.sum_bytes == e.sum_bytes && h.prompt_len == e.prompt_len &&
         h.tail_len == e.tail_len && h.page_bytes == e.page_bytes && h.payload_bytes == e.payload_bytes &&
         h.seed == e.seed && h.head_base == e.head_base;  // same Philox streams as this rank's later appends
}

__global__ void scatter_kernel(LayerPtrs lp, const int32_t* __restrict__ block_table, int max_pages_per_req,
                               int32_t* __restrict__ seq_lens, uint32_t* __restrict__ rng_ids, int slot, XferGeom g,
                               WireHeader expect, const uint8_t* __restrict__ staging, int32_t* status) {
  const WireHeader h = *reinterpret_cast<const WireHeader*>(staging);
  const bool ok = header_ok(h, expect);
  const int j = blockIdx.x, l = blockIdx.y;
  if (j == 0 && l == 0 && threadIdx.x == 0) {
    if (status) {
      status[0] = ok ? HACK_OK : HACK_ERR_PROTOCOL;
      status[1] = ok ? h.first_token : -1;
    }
    if (ok) {
      seq_lens[slot] = (int32_t)h.prompt_len;
      rng_ids[slot] = h.rng_id;
    }
  }
  if (!ok) return;
  const uint8_t* src = staging + kHeaderBytes + (int64_t)l * g.layer_bytes;
  const int64_t pbytes = (int64_t)g.Hkv * g.page_bytes;
  if (j < g.npages) {
    const int pid = block_table[(int64_t)slot * max_pages_per_req + j];
    copy16(lp.pages[l] + pid * pbytes, src + j * pbytes, pbytes);
  } else if (g.tail_len) {
    const uint8_t* ts = src + g.npages * pbytes;
    const int64_t rowb = (int64_t)g.tail_len * 128 * 2;
    for (int h2 = 0; h2 < g.Hkv; ++h2)
      copy16(reinterpret_cast<uint8_t*>(lp.tail[l] + ((int64_t)slot * g.Hkv + h2) * g.Pi * 128), ts + h2 * rowb,
             rowb);
  }
}

hack_status_t prepare(const hack_config_t* cfg, const hack_kv_cache_t* caches, int num_layers, int slot,
                      int prompt_len, KernelCfg* kc, LayerPtrs* lp, XferGeom* g, WireHeader* hdr) {
  hack_status_t st = make_kernel_cfg(cfg, kc);
  if (st != HACK_OK) return st;
  if (!caches) return fail(HACK_ERR_INVALID_ARG, "kv transfer: caches is NULL");
  if (num_layers <= 0 || num_layers > kMaxLayers) return fail(HACK_ERR_INVALID_ARG, "kv transfer: 1..128 layers");
  if (prompt_len <= 0) return fail(HACK_ERR_INVALID_ARG, "kv transfer: empty prompt");
  for (int l = 0; l < num_layers; ++l) {
    CacheView cv;
    if ((st = make_cache_view(*kc, &caches[l], &cv)) != HACK_OK) return st;
    if (caches[l].block_table != caches[0].block_table || caches[l].seq_lens != caches[0].seq_lens ||
        caches[l].rng_ids != caches[0].rng_ids || caches[l].max_pages_per_req != caches[0].max_pages_per_req)
      return fail(HACK_ERR_INVALID_ARG, "kv transfer: layers must share block_table/seq_lens/rng_ids");
    lp->pages[l] = caches[l].pages;
    lp->tail[l] = reinterpret_cast<__half*>(caches[l].v_tail);
  }
  if (slot < 0 || slot >= caches[0].max_reqs) return fail(HACK_ERR_INVALID_ARG, "kv transfer: bad slot");
  if ((prompt_len + kc->Pi - 1) / kc->Pi > caches[0].max_pages_per_req)
    return fail(HACK_ERR_CAPACITY, "kv transfer: prompt needs more pages than max_pages_per_req");
  g->npages = (prompt_len + kc->Pi - 1) / kc->Pi;
  g->tail_len = prompt_len % kc->Pi;
  g->Hkv = kc->Hkv;
  g->page_bytes = kc->pl.page_bytes;
  g->Pi = kc->Pi;
  g->num_layers = num_layers;
  g->layer_bytes = layer_bytes(*kc, prompt_len);
  memset(hdr, 0, sizeof(*hdr));
  hdr->magic = kMagic;
  hdr->version = kWireVersion;
  hdr->num_layers = (uint16_t)num_layers;
  hdr->num_kv_heads = (uint16_t)kc->Hkv;
  hdr->head_dim = (uint16_t)kc->d;
  hdr->partition = (uint16_t)kc->Pi;
  hdr->kv_bits = (uint8_t)kc->bits;
  hdr->sum_bytes = (uint8_t)kc->pl.sum_bytes;
  hdr->prompt_len = (uint32_t)prompt_len;
  hdr->tail_len = (uint32_t)g->tail_len;
  hdr->page_bytes = (uint32_t)kc->pl.page_bytes;
  hdr->head_base = (uint32_t)kc->head_base;
  hdr->payload_bytes = (uint64_t)g->layer_bytes * num_layers;
  hdr->seed = kc->seed;
  return HACK_OK;
}

// Fused transfer (f1): grid (npages + 1, layers); block j < npages copies page j of every KV
// head from the source cache (any device-accessible memory: a peer GPU's cache mapped with
// CUDA IPC / peer access, so the loads cross NVLink) straight into the destination page,
// both resolved through their own block tables; block npages copies the FP16 tail rows.
// No staging buffer and no header: both sides' geometry comes from (cfg, prompt_len).
__global__ void pull_kernel(LayerPtrs src, LayerPtrs dst, const int32_t* __restrict__ src_bt, int src_mpr,
                            int src_slot, const uint32_t* __restrict__ src_rng, const int32_t* __restrict__ dst_bt,
                            int dst_mpr, int dst_slot, int32_t* __restrict__ dst_seq, uint32_t* __restrict__ dst_rng,
                            XferGeom g, int prompt_len) {
  const int j = blockIdx.x, l = blockIdx.y;
  if (j == 0 && l == 0 && threadIdx.x == 0) {
    dst_seq[dst_slot] = prompt_len;
    dst_rng[dst_slot] = src_rng[src_slot];
  }
  const int64_t pbytes = (int64_t)g.Hkv * g.page_bytes;
  if (j < g.npages) {
    const int sp = src_bt[(int64_t)src_slot * src_mpr + j], dp = dst_bt[(int64_t)dst_slot * dst_mpr + j];
    copy16(dst.pages[l] + dp * pbytes, src.pages[l] + sp * pbytes, pbytes);
  } else if (g.tail_len) {
    const int64_t rowb = (int64_t)g.tail_len * 128 * 2;
    for (int h = 0; h < g.Hkv; ++h)
      copy16(reinterpret_cast<uint8_t*>(dst.tail[l] + ((int64_t)dst_slot * g.Hkv + h) * g.Pi * 128),
             reinterpret_cast<const uint8_t*>(src.tail[l] + ((int64_t)src_slot * g.Hkv + h) * g.Pi * 128), rowb);
  }
}

hack_status_t nccl_status(ncclResult_t r, const char* where) {
  if (r == ncclSuccess) return HACK_OK;
  return fail(HACK_ERR_NCCL, "%s: %s", where, ncclGetErrorString(r));
}

}  // namespace
}  // namespace hack

using namespace hack;

extern "C" {

int64_t hack_kv_transfer_bytes(const hack_config_t* cfg, int32_t num_layers, int32_t prompt_len) {
  KernelCfg kc;
  if (make_kernel_cfg(cfg, &kc) != HACK_OK || num_layers <= 0 || prompt_len <= 0) return -1;
  return kHeaderBytes + layer_bytes(kc, prompt_len) * num_layers;
}

hack_status_t hack_comm_unique_id(uint8_t id_out[128]) {
  if (!id_out) return fail(HACK_ERR_INVALID_ARG, "comm_unique_id: NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  hack_status_t st = nccl_status(ncclGetUniqueId(&id), "ncclGetUniqueId");
  if (st != HACK_OK) return st;
  memcpy(id_out, &id, 128);
  return HACK_OK;
}

hack_status_t hack_comm_init(void** comm_out, int32_t nranks, int32_t rank, const uint8_t id[128]) {
  if (!comm_out || !id) return fail(HACK_ERR_INVALID_ARG, "comm_init: NULL");
  if (nranks <= 0 || rank < 0 || rank >= nranks) return fail(HACK_ERR_INVALID_ARG, "comm_init: bad rank");
  hack_status_t st = check_device();
  if (st != HACK_OK) return st;
  ncclUniqueId uid;
  memcpy(&uid, id, 128);
  ncclComm_t comm;
  st = nccl_status(ncclCommInitRank(&comm, nranks, uid, rank), "ncclCommInitRank");
  if (st != HACK_OK) return st;
  *comm_out = comm;
  return HACK_OK;
}

hack_status_t hack_comm_destroy(void* comm) {
  if (!comm) return fail(HACK_ERR_INVALID_ARG, "comm_destroy: NULL");
  return nccl_status(ncclCommDestroy((ncclComm_t)comm), "ncclCommDestroy");
}

hack_status_t hack_kv_pack(const hack_config_t* cfg, const hack_kv_cache_t* caches, int32_t num_layers,
                           int32_t slot, int32_t prompt_len, int32_t first_token, uint32_t rng_id, void* staging,
                           void* stream) {
  KernelCfg kc;
  LayerPtrs lp;
  XferGeom g;
  WireHeader hdr;
  if (!staging) return fail(HACK_ERR_INVALID_ARG, "kv_pack: NULL staging");
  hack_status_t st = prepare(cfg, caches, num_layers, slot, prompt_len, &kc, &lp, &g, &hdr);
  if (st != HACK_OK) return st;
  hdr.first_token = first_token;
  hdr.rng_id = rng_id;
  if ((st = check_device()) != HACK_OK) return st;
  gather_kernel<<<dim3(g.npages + 1, num_layers), 256, 0, (cudaStream_t)stream>>>(
      lp, caches[0].block_table, caches[0].max_pages_per_req, reinterpret_cast<const uint32_t*>(caches[0].rng_ids),
      slot, g, hdr, (uint8_t*)staging, 0);
  note_launch();
  return cuda_status(cudaGetLastError(), "kv_pack gather");
}

hack_status_t hack_kv_unpack(const hack_config_t* cfg, const hack_kv_cache_t* caches, int32_t num_layers,
                             int32_t slot, int32_t prompt_len, const void* staging, int32_t* status_dev,
                             void* stream) {
  KernelCfg kc;
  LayerPtrs lp;
  XferGeom g;
  WireHeader hdr;
  if (!staging) return fail(HACK_ERR_INVALID_ARG, "kv_unpack: NULL staging");
  hack_status_t st = prepare(cfg, caches, num_layers, slot, prompt_len, &kc, &lp, &g, &hdr);
  if (st != HACK_OK) return st;
  if ((st = check_device()) != HACK_OK) return st;
  scatter_kernel<<<dim3(g.npages + 1, num_layers), 256, 0, (cudaStream_t)stream>>>(
      lp, caches[0].block_table, caches[0].max_pages_per_req, caches[0].seq_lens, caches[0].rng_ids, slot, g, hdr,
      (const uint8_t*)staging, status_dev);
  note_launch();
  return cuda_status(cudaGetLastError(), "kv_unpack scatter");
}

hack_status_t hack_kv_send(void* comm, int32_t peer, const hack_config_t* cfg, const hack_kv_cache_t* caches,
                           int32_t num_layers, int32_t slot, int32_t prompt_len, int32_t first_token,
                           uint32_t rng_id, void* staging, void* stream) {
  if (!comm) return fail(HACK_ERR_INVALID_ARG, "kv_send: NULL comm");
  hack_status_t st = hack_kv_pack(cfg, caches, num_layers, slot, prompt_len, first_token, rng_id, staging, stream);
  if (st != HACK_OK) return st;
  const int64_t bytes = hack_kv_transfer_bytes(cfg, num_layers, prompt_len);
  return nccl_status(ncclSend(staging, (size_t)bytes, ncclUint8, peer, (ncclComm_t)comm, (cudaStream_t)stream),
                     "ncclSend");
}

hack_status_t hack_kv_recv(void* comm, int32_t peer, const hack_config_t* cfg, const hack_kv_cache_t* caches,
                           int32_t num_layers, int32_t slot, int32_t prompt_len, void* staging, int32_t* status_dev,
                           void* stream) {
  if (!comm || !staging) return fail(HACK_ERR_INVALID_ARG, "kv_recv: NULL comm/staging");
  const int64_t bytes = hack_kv_transfer_bytes(cfg, num_layers, prompt_len);
  if (bytes < 0) return fail(HACK_ERR_INVALID_ARG, "kv_recv: bad config/prompt");
  hack_status_t st = nccl_status(
      ncclRecv(staging, (size_t)bytes, ncclUint8, peer, (ncclComm_t)comm, (cudaStream_t)stream), "ncclRecv");
  if (st != HACK_OK) return st;
  return hack_kv_unpack(cfg, caches, num_layers, slot, prompt_len, staging, status_dev, stream);
}

int64_t hack_kv_layer_range(const hack_config_t* cfg, int32_t num_layers, int32_t layer, int32_t prompt_len,
                            int64_t* begin_out) {
  KernelCfg kc;
  if (make_kernel_cfg(cfg, &kc) != HACK_OK || num_layers <= 0 || prompt_len <= 0 || layer < 0 || layer >= num_layers)
    return -1;
  const int64_t lb = layer_bytes(kc, prompt_len);
  const int64_t b = layer == 0 ? 0 : kHeaderBytes + (int64_t)layer * lb;
  if (begin_out) *begin_out = b;
  return kHeaderBytes + (int64_t)(layer + 1) * lb - b;
}

hack_status_t hack_kv_send_layer(void* comm, int32_t peer, const hack_config_t* cfg, const hack_kv_cache_t* caches,
                                 int32_t num_layers, int32_t layer, int32_t slot, int32_t prompt_len,
                                 int32_t first_token, uint32_t rng_id, void* staging, void* stream) {
  KernelCfg kc;
  LayerPtrs lp;
  XferGeom g;
  WireHeader hdr;
  if (!comm || !staging) return fail(HACK_ERR_INVALID_ARG, "kv_send_layer: NULL comm/staging");
  if (layer < 0 || layer >= num_layers) return fail(HACK_ERR_INVALID_ARG, "kv_send_layer: layer out of range");
  hack_status_t st = prepare(cfg, caches, num_layers, slot, prompt_len, &kc, &lp, &g, &hdr);
  if (st != HACK_OK) return st;
  hdr.first_token = first_token;
  hdr.rng_id = rng_id;
  if ((st = check_device()) != HACK_OK) return st;
  gather_kernel<<<dim3(g.npages + 1, 1), 256, 0, (cudaStream_t)stream>>>(
      lp, caches[0].block_table, caches[0].max_pages_per_req, reinterpret_cast<const uint32_t*>(caches[0].rng_ids),
      slot, g, hdr, (uint8_t*)staging, layer);
  note_launch();
  if ((st = cuda_status(cudaGetLastError(), "kv_send_layer gather")) != HACK_OK) return st;
  int64_t b = 0;
  const int64_t n = hack_kv_layer_range(cfg, num_layers, layer, prompt_len, &b);
  return nccl_status(ncclSend((uint8_t*)staging + b, (size_t)n, ncclUint8, peer, (ncclComm_t)comm,
                              (cudaStream_t)stream),
                     "ncclSend (layer)");
}

hack_status_t hack_kv_recv_layer(void* comm, int32_t peer, const hack_config_t* cfg, int32_t num_layers,
                                 int32_t layer, int32_t prompt_len, void* staging, void* stream) {
  if (!comm || !staging) return fail(HACK_ERR_INVALID_ARG, "kv_recv_layer: NULL comm/staging");
  int64_t b = 0;
  const int64_t n = hack_kv_layer_range(cfg, num_layers, layer, prompt_len, &b);
  if (n < 0) return fail(HACK_ERR_INVALID_ARG, "kv_recv_layer: bad config/layer/prompt");
  return nccl_status(ncclRecv((uint8_t*)staging + b, (size_t)n, ncclUint8, peer, (ncclComm_t)comm,
                              (cudaStream_t)stream),
                     "ncclRecv (layer)");
}

hack_status_t hack_kv_pull(const hack_config_t* cfg, const hack_kv_cache_t* src, const hack_kv_cache_t* dst,
                           int32_t num_layers, int32_t src_slot, int32_t dst_slot, int32_t prompt_len, void* stream) {
  KernelCfg kc;
  LayerPtrs sp, dp;
  XferGeom g;
  WireHeader hdr;
  hack_status_t st = prepare(cfg, src, num_layers, src_slot, prompt_len, &kc, &sp, &g, &hdr);
  if (st != HACK_OK) return st;
  XferGeom g2;
  if ((st = prepare(cfg, dst, num_layers, dst_slot, prompt_len, &kc, &dp, &g2, &hdr)) != HACK_OK) return st;
  if ((st = check_device()) != HACK_OK) return st;
  pull_kernel<<<dim3(g.npages + 1, num_layers), 256, 0, (cudaStream_t)stream>>>(
      sp, dp, src[0].block_table, src[0].max_pages_per_req, src_slot, reinterpret_cast<const uint32_t*>(src[0].rng_ids),
      dst[0].block_table, dst[0].max_pages_per_req, dst_slot, dst[0].seq_lens,
      reinterpret_cast<uint32_t*>(dst[0].rng_ids), g, prompt_len);
  note_launch();
  return cuda_status(cudaGetLastError(), "kv_pull");
}

hack_status_t hack_comm_recv_bytes(void* comm, int32_t peer, void* buf, int64_t bytes, void* stream) {
  if (!comm || !buf || bytes <= 0) return fail(HACK_ERR_INVALID_ARG, "comm_recv_bytes: bad args");
  return nccl_status(ncclRecv(buf, (size_t)bytes, ncclUint8, peer, (ncclComm_t)comm, (cudaStream_t)stream),
                     "ncclRecv");
}

hack_status_t hack_comm_group_start(void) { return nccl_status(ncclGroupStart(), "ncclGroupStart"); }
hack_status_t hack_comm_group_end(void) { return nccl_status(ncclGroupEnd(), "ncclGroupEnd"); }

}  // extern "C"
