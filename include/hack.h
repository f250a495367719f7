/*
 * hack.h -- C ABI of libhack.so, the B200 (sm_100a) hot path of HACK
 * ("Homomorphic Acceleration via Compression of the Key-Value Cache for
 * Disaggregated LLM Inference", arXiv 2502.03589).
 *
 * Citations: P:<n> = line n of the paper's text,
 * S:<n> = line n of SPEC.md, R<k> = reading k in DESIGN.md ("Readings").
 *
 * What the library computes (fig:overview): attention directly on
 * per-partition asymmetric, stochastically rounded low-bit KV codes
 * with no dequantization.  Q.K^T and P.V are integer matmuls on codes; Eq. 4
 * rebuilds the real-valued result per Pi-block from the
 * per-partition min/scale and cached code sums (summation elimination,
 * P:679-691).  The partially filled last V block stays FP16 (requantization
 * elimination).
 *
 * Conventions (all entry points):
 *  - Pure C, POD arguments.  Pointers documented "device" must point to CUDA
 *    device memory of the current device; "host" pointers to host memory.
 *  - All device memory is CALLER-OWNED.  The library allocates nothing
 *    persistent except NCCL communicators (hack_comm_init/destroy).
 *  - `stream` is a cudaStream_t passed as void*; every call is asynchronous on
 *    it (no implicit device synchronisation).  NULL = legacy default stream.
 *  - fp16 tensors are IEEE binary16 (passed as void*).  Integers little-endian.
 *  - Every call returns hack_status_t and never aborts.  Argument errors are
 *    detected on the host before any launch; hack_last_error() (thread-local)
 *    gives a one-line message for the last non-OK status on this thread.
 *  - Thread-safety: stateless except for communicators.  Calls touching the
 *    same cache slot must be serialised by the caller.
 *  - There is no CPU fallback: a missing/unsupported GPU returns HACK_ERR_CUDA.
 */
#ifndef HACK_H_
#define HACK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define HACK_ABI_VERSION 2

typedef enum {
  HACK_OK = 0,
  HACK_ERR_INVALID_ARG = 1,   /* null pointer, bad enum, bits not in {2,4}, empty input */
  HACK_ERR_UNSUPPORTED = 2,   /* Pi not in {32,64,128}, head_dim != 128, G > 16 (R16) */
  HACK_ERR_SHAPE = 3,         /* inconsistent dimensions */
  HACK_ERR_CAPACITY = 4,      /* block table / page pool / workspace too small */
  HACK_ERR_PROTOCOL = 5,      /* kv_recv header mismatch */
  HACK_ERR_CUDA = 6,          /* CUDA launch / runtime failure, or no sm_100 device */
  HACK_ERR_NCCL = 7           /* NCCL failure */
} hack_status_t;

typedef enum {
  HACK_ROUND_STOCHASTIC = 0,   /* floor(y) + [u < frac(y)], u = 24-bit Philox uniform (R1) */
  HACK_ROUND_NEAREST_EVEN = 1  /* rint, ties to even (R17) */
} hack_round_t;

/* Quantizer modes for hack_quantize_pack (partition axes: fig:hoq_self_attn). */
typedef enum {
  HACK_QMODE_K = 0,  /* kv_bits codes, partitions of Pi along head_dim per token, fp16 meta, tag K */
  HACK_QMODE_V = 1,  /* kv_bits codes, partitions of Pi tokens per channel, fp16 meta, tag V */
  HACK_QMODE_Q = 2   /* 8-bit codes, partitions of Pi along head_dim, fp32 meta, tag Q */
} hack_qmode_t;

/* Configuration, validated by every call.  Start from hack_config_default(). */
typedef struct {
  int32_t num_q_heads;   /* H_q (local to this process) */
  int32_t num_kv_heads;  /* H_kv (local); H_q % H_kv == 0, G = H_q/H_kv <= 16 (GQA, R15) */
  int32_t head_dim;      /* d_h; must be 128 ("typically 128") */
  int32_t partition;     /* Pi in {32, 64, 128}; head_dim % Pi == 0 (R16) */
  int32_t kv_bits;       /* b for K/V codes: 2 or 4; Q and P are fixed at 8 */
  int32_t kv_round;      /* hack_round_t for K/V codes (default STOCHASTIC) */
  int32_t q_round;       /* hack_round_t for Q codes (default STOCHASTIC, R6) */
  int32_t p_round;       /* hack_round_t for P codes: NEAREST_EVEN (default, R6) or STOCHASTIC (the paper's
                            P:575-578 rounding; prefill at Pi = 64 and decode with G <= 8, else
                            HACK_ERR_UNSUPPORTED at the attention call) */
  uint64_t seed;         /* Philox4x32-10 key (R3) */
  int32_t layer;         /* layer index folded into the Philox counter (R3) */
  int32_t head_base;     /* global index of local KV head 0 (head sharding keeps codes identical, SURVEY e) */
  int32_t out_dtype;     /* 0 = fp16 output, 1 = fp32 output */
  int32_t reserved;
} hack_config_t;

/* Paged packed-KV cache of ONE layer.  All device,
 * caller-owned.  One page holds Pi tokens of every local KV head:
 *   pages[page][kv_head][page_bytes], sections K_CODES, K_META, K_SUMS,
 *   V_CODES, V_META, V_SUMS at hack_page_layout() offsets.
 * v_tail holds the FP16 last V block (RQE): [max_reqs][H_kv][Pi][d].
 * block_table[slot][j] = page id of the slot's j-th Pi-token block.
 * seq_lens[slot] = tokens cached (committed + tail); written by the library.
 * rng_ids[slot]  = the request's 32-bit Philox stream id (caller-set). */
typedef struct {
  uint8_t* pages;
  void* v_tail;
  int32_t* block_table;
  int32_t* seq_lens;
  uint32_t* rng_ids;
  int32_t num_pages;
  int32_t max_reqs;
  int32_t max_pages_per_req;
  int32_t page_bytes;
} hack_kv_cache_t;

/* Optional debug dumps (parity protocol); pass NULL in production.
 * Every pointer may be NULL independently; the dumps do not change any result.
 * pcodes: device u8 [total_q_rows][H_q][pcodes_stride]: the GPU's 8-bit P codes of
 *   committed V blocks, key t at column t (row-major per query row).
 * qk_acc: device int32 [total_q_rows][H_q][d/Pi][acc_stride]: for every key t the query
 *   row attends to, the QK integer MMA's own block accumulator of d-block beta, exactly as
 *   the kernel holds it (conversion bias removed).  It is an exact affine function of the
 *   paper's D_beta = sum_{z in beta} q'_z k'_z (Eq. 4) whose form is
 *   hack_debug_acc_form() (below).
 * pv_acc: device int32 [total_q_rows][H_q][acc_stride/Pi][d]: per committed V block j and
 *   channel c, the PV MMA's block accumulator, an exact affine function of
 *   D'_j = sum_{t in block j} p'_t v'_tc (the GPU's own P codes) of the same form.
 * acc_stride: keys per (row, head, beta) in qk_acc; >= max_seqlen, a multiple of Pi.
 * acc_head: -1 = every query head (the H_q dimension above); h >= 0 = only query head h
 *   (sampled dumps at full size), the arrays then being [total_q_rows][1][...]. */
typedef struct {
  uint8_t* pcodes;
  int64_t pcodes_stride;
  int32_t* qk_acc;
  int32_t* pv_acc;
  int64_t acc_stride;
  int32_t acc_head;
  int32_t reserved;
} hack_debug_t;

/* Affine form of the dumped accumulators, per hack_debug_acc_form(cfg, op):
 *   HACK_ACC_PLAIN     acc = D                                  (decode_mma: u8 x u8 on 2^23 bias)
 *   HACK_ACC_S8_2B     acc = 2 D - 256 S_B                      (prefill_tc: A' - 128 (s8) x 2 B' (u8))
 *   HACK_ACC_CENTERED4 acc = 4 D - 2(2^b-1) S_A + Pi 255 (2^b-1) (decode_pair / decode_g8: split planes)
 * with S_A the 8-bit operand's block code sum (SQ / SP) and S_B the b-bit operand's (SK / SV).
 * HACK_ACC_NONE: the kernel serving (cfg, op) has no accumulator dump (CUDA-core baselines);
 * a call with qk_acc / pv_acc set then returns HACK_ERR_UNSUPPORTED. */
typedef enum {
  HACK_ACC_NONE = 0,
  HACK_ACC_PLAIN = 1,
  HACK_ACC_S8_2B = 2,
  HACK_ACC_CENTERED4 = 3
} hack_acc_form_t;
/* op: 0 = prefill attention, 1 = decode attention (dispatch as the next call would). */
int32_t hack_debug_acc_form(const hack_config_t* cfg, int32_t op);

/* ---- configuration and layout ------------------------------------------ */
void hack_config_default(hack_config_t* cfg);          /* H=1/1, d=128, Pi=64, b=2, SR/SR/RN (K-V/Q/P), fp16 out */
hack_status_t hack_config_validate(const hack_config_t* cfg);
int64_t hack_page_bytes(const hack_config_t* cfg);     /* 5376 at (d=128, Pi=64, b=2); -1 if invalid */
/* offsets_out[12] = {off, size} x {K_CODES, K_META, K_SUMS, V_CODES, V_META, V_SUMS} (bytes) */
hack_status_t hack_page_layout(const hack_config_t* cfg, int64_t offsets_out[12]);
const char* hack_last_error(void);
const char* hack_version(void);
int32_t hack_abi_version(void);
/* Total kernels this library has launched in this process (bench launch accounting). */
int64_t hack_kernel_launches(void);

/* ---- (a1-a3) quantize_pack ---------------------------------------------- */
/* Quantize x (device fp16, dense [rows][heads][d]) per partition.
 * mode K : codes u8 [rows][heads][d*b/8] (LSB-first); meta fp16 (m,s) [rows][heads][d/Pi][2];
 *          sums [rows][heads][d/Pi] (u8 if b+ceil(log2 Pi) <= 8 else u16).
 * mode V : rows % Pi == 0; codes [rows/Pi][heads][d][Pi*b/8]; meta fp16 [rows/Pi][heads][d][2];
 *          sums [rows/Pi][heads][d].
 * mode Q : codes u8 [rows][heads][d]; meta fp32 (m,s) [rows][heads][d/Pi][2]; sums u16 [rows][heads][d/Pi].
 * Row r sits at sequence position pos0 + r; Philox head index = head0 + h (R3).
 * All outputs device, caller-allocated. */
hack_status_t hack_quantize_pack(const hack_config_t* cfg, int32_t mode, const void* x,
                                 int64_t rows, int32_t heads, int64_t pos0, int32_t head0,
                                 uint32_t rng_id, uint8_t* codes, void* meta, void* sums,
                                 void* stream);

/* ---- (a1-a2) prefill ingest: quantize a prompt's K/V into the paged cache ---- */
/* k, v: device fp16 [total_tokens][H_kv][d], requests packed by cu_seqlens (device
 * int32 [batch+1]); slots: device int32 [batch] cache slot of each request.  Writes
 * K rows of every token, V blocks of every full Pi block, FP16 tail rows of the
 * ragged remainder (R10), and seq_lens[slot].  max_seqlen: host upper bound. */
hack_status_t hack_cache_ingest(const hack_config_t* cfg, const void* k, const void* v,
                                const int32_t* cu_seqlens, const int32_t* slots, int32_t batch,
                                int32_t max_seqlen, const hack_kv_cache_t* cache, void* stream);

/* ---- (a1-a7) homomorphic prefill attention ------------------------------ */
/* Ingest K/V (as hack_cache_ingest) then causal HACK attention for every prompt token:
 * Q 8-bit (a3) -> Eq. 4 Q'K'^T per d-block (a4) -> online softmax (a5) -> P 8-bit per
 * (row, Pi-key block) (a6) -> Eq. 4 P'V' per block + FP tail, / l (a7).
 * q: device fp16 [total_tokens][H_q][d]; out: device [total_tokens][H_q][d] fp16/fp32
 * (cfg->out_dtype).  workspace: device, >= hack_prefill_workspace_size() bytes. */
size_t hack_prefill_workspace_size(const hack_config_t* cfg, int32_t batch, int32_t max_seqlen);
hack_status_t hack_prefill_attention(const hack_config_t* cfg, const void* q, const void* k,
                                     const void* v, const int32_t* cu_seqlens, const int32_t* slots,
                                     int32_t batch, int32_t max_seqlen, const hack_kv_cache_t* cache,
                                     void* out, void* workspace, size_t workspace_bytes,
                                     const hack_debug_t* debug, void* stream);
/* Attention only, on a cache already holding the prompts (what the roofline times). */
hack_status_t hack_prefill_attention_cached(const hack_config_t* cfg, const void* q,
                                            const int32_t* cu_seqlens, const int32_t* slots,
                                            int32_t batch, int32_t max_seqlen,
                                            const hack_kv_cache_t* cache, void* out, void* workspace,
                                            size_t workspace_bytes, const hack_debug_t* debug,
                                            void* stream);

/* The same call with HOST buffers (e2e path): q, k, v, out and cu_seqlens / slots are host
 * pointers (page-locked for copy/compute overlap; pageable works, serialised), total tokens
 * = cu_seqlens[batch].  The library stages them through `workspace` (device, >=
 * hack_prefill_host_workspace_size() bytes, any contents) and pipelines: K/V up -> ingest;
 * then per chunk, Q chunk up -> attention of that chunk -> out chunk down, the uploads, the
 * attention and the downloads of different chunks overlapping (copies on library-owned
 * streams, ordered after prior work on `stream`; `stream` completes after the last download).
 * head_chunks > 0: that many chunks of query heads (whole GQA groups).  head_chunks <= 0 and
 * batch == 1: chunks of query positions, the last positions (longest causal rows) first
 * (-n: n chunks, 0: 8); <= 0 with batch > 1: 8 query-head chunks.  Results identical to
 * hack_prefill_attention.  Same errors, plus HACK_ERR_CAPACITY for a small workspace. */
size_t hack_prefill_host_workspace_size(const hack_config_t* cfg, int32_t batch, int32_t total_tokens);
hack_status_t hack_prefill_attention_host(const hack_config_t* cfg, const void* q, const void* k,
                                          const void* v, const int32_t* cu_seqlens, const int32_t* slots,
                                          int32_t batch, int32_t max_seqlen, const hack_kv_cache_t* cache,
                                          void* out, void* workspace, size_t workspace_bytes,
                                          int32_t head_chunks, void* stream);

/* ---- (a8-a9) decode ------------------------------------------------------ */
/* Append one token per request (a8): quantize k_new into its own partitions,
 * put v_new in the FP16 tail, flush the tail into a V block when it reaches Pi
 * (R12), seq_lens[slot] += 1.  k_new, v_new: device fp16 [batch][H_kv][d].
 * Every append advances the cache's seq_lens, so the layers of a model must each decode on
 * their own seq_lens array (they may share pages' block_table and rng_ids; the KV
 * transfer calls, which need one seq_lens for all layers, only run before decode). */
hack_status_t hack_decode_append(const hack_config_t* cfg, const void* k_new, const void* v_new,
                                 const int32_t* slots, int32_t batch, const hack_kv_cache_t* cache,
                                 void* stream);
/* Append (a8) then attend (a9) with L_Q = 1: q_new device fp16 [batch][H_q][d];
 * out [batch][H_q][d].  max_seqlen: host upper bound of seq_lens after the append.
 * workspace: device, >= hack_decode_workspace_size() bytes (split partials and per-unit
 * merge counters): zero-filled before its first use; every launch leaves the counters zero
 * again, so it is reused without clearing.  One workspace per stream. */
size_t hack_decode_workspace_size(const hack_config_t* cfg, int32_t batch, int32_t max_seqlen);
hack_status_t hack_decode_attention(const hack_config_t* cfg, const void* q_new, const void* k_new,
                                    const void* v_new, const int32_t* slots, int32_t batch,
                                    int32_t max_seqlen, const hack_kv_cache_t* cache, void* out,
                                    void* workspace, size_t workspace_bytes,
                                    const hack_debug_t* debug, void* stream);
/* Attention only (the HBM-bound kernel the decode roofline times). */
hack_status_t hack_decode_attention_cached(const hack_config_t* cfg, const void* q_new,
                                           const int32_t* slots, int32_t batch, int32_t max_seqlen,
                                           const hack_kv_cache_t* cache, void* out, void* workspace,
                                           size_t workspace_bytes, const hack_debug_t* debug,
                                           void* stream);

/* ---- comparator export: dequantize-first baseline ------------- */
/* NOT part of the HACK path.  Expands the packed pages of every request into dense FP16
 * K-hat = m + s*code and V-hat = m + s*code per partition (P:575-578 meta, fp32 FMA, one
 * rounding to fp16), the FP16 last V block copied unchanged, as KV-quantization
 * systems that dequantize before attention do (KVQuant / CacheGen).
 * k_out, v_out: device fp16 [batch][num_kv_heads][max_seqlen][head_dim], caller-owned;
 * rows >= seq_len are not written.  Errors: INVALID_ARG (NULL, empty), CAPACITY
 * (max_seqlen beyond the block table), CUDA. */
hack_status_t hack_dequantize_cache(const hack_config_t* cfg, const int32_t* slots, int32_t batch,
                                    int32_t max_seqlen, const hack_kv_cache_t* cache, void* k_out,
                                    void* v_out, void* stream);

/* ---- test export: Eq. 4 homomorphic matmul on codes (N9) ---------------- */
/* A: 8-bit codes u8 [M][Z], meta fp32 (m,s) [M][Z/Pi][2], sums u16 [M][Z/Pi];
 * B: kv_bits codes packed per column u8 [N][Z*b/8] (column j's Z codes LSB-first),
 *    meta fp16 (m,s) [N][Z/Pi][2], sums [N][Z/Pi] (u8/u16 per sum width).
 * d_blocks (optional) int32 [Z/Pi][M][N] exact per-block partials; c fp32 [M][N]
 * = sum_beta Eq. 4.  All device. */
hack_status_t hack_homomorphic_matmul(const hack_config_t* cfg, const uint8_t* a_codes,
                                      const float* a_meta, const uint16_t* a_sums,
                                      const uint8_t* b_packed, const void* b_meta,
                                      const void* b_sums, int32_t M, int32_t N, int32_t Z,
                                      int32_t* d_blocks, float* c, void* stream);

/* ---- (a10) KV transfer over NCCL -------------------------- */
/* Bytes moved per request: header (64 B) + per layer ceil(L/Pi) pages x H_kv x page_bytes
 * + H_kv x (L mod Pi) x d x 2 tail bytes.  Sizes are a closed form of (prompt_len, cfg). */
int64_t hack_kv_transfer_bytes(const hack_config_t* cfg, int32_t num_layers, int32_t prompt_len);
hack_status_t hack_comm_unique_id(uint8_t id_out[128]);  /* broadcast it via torch.distributed */
hack_status_t hack_comm_init(void** comm_out, int32_t nranks, int32_t rank, const uint8_t id[128]);
hack_status_t hack_comm_destroy(void* comm);
/* hack_kv_pack: gather one request (slot) of num_layers caches (host array of structs,
 * <= 128 layers, sharing block_table/seq_lens/rng_ids) into `staging` (device, >=
 * hack_kv_transfer_bytes): 64-byte header (magic "HACK", version, dims, prompt_len,
 * tail_len, first_token, rng_id, page_bytes, head_base, payload_bytes, seed) + per
 * layer the request's pages (codes, fp16 meta, cached sums, R19) + its FP16 tail rows
 * (RQE).  first_token: the prefill output token.  rng_id must equal the
 * cache's rng_ids[slot] (the header carries rng_ids[slot]); a mismatch is detected on the
 * device and poisons the header (magic 0), so the receiver reports HACK_ERR_PROTOCOL. */
hack_status_t hack_kv_pack(const hack_config_t* cfg, const hack_kv_cache_t* caches, int32_t num_layers,
                           int32_t slot, int32_t prompt_len, int32_t first_token, uint32_t rng_id,
                           void* staging, void* stream);
/* hack_kv_unpack: validate the header in `staging` on the device against (cfg,
 * num_layers, prompt_len) -- dims, sizes, and the Philox seed and head_base, since this
 * rank's later appends continue the same streams (R3) -- and scatter into `slot` of the
 * local caches (block tables
 * already filled by the caller), setting seq_lens[slot] and rng_ids[slot].
 * status_dev (device int32[2], may be NULL) receives {hack_status_t, first_token}; a
 * header mismatch writes HACK_ERR_PROTOCOL and leaves the cache untouched. */
hack_status_t hack_kv_unpack(const hack_config_t* cfg, const hack_kv_cache_t* caches, int32_t num_layers,
                             int32_t slot, int32_t prompt_len, const void* staging, int32_t* status_dev,
                             void* stream);
/* kv_send = kv_pack + ncclSend(staging) to `peer`; kv_recv = ncclRecv(staging) from
 * `peer` + kv_unpack.  Stream-ordered; do not wrap kv_recv in a NCCL group (its unpack
 * kernel must follow the receive).  For a self-loop use group_start, kv_send,
 * comm_recv_bytes, group_end, then kv_unpack. */
hack_status_t hack_kv_send(void* comm, int32_t peer, const hack_config_t* cfg,
                           const hack_kv_cache_t* caches, int32_t num_layers, int32_t slot,
                           int32_t prompt_len, int32_t first_token, uint32_t rng_id,
                           void* staging, void* stream);
hack_status_t hack_kv_recv(void* comm, int32_t peer, const hack_config_t* cfg,
                           const hack_kv_cache_t* caches, int32_t num_layers, int32_t slot,
                           int32_t prompt_len, void* staging, int32_t* status_dev, void* stream);
/* Layer-pipelined transfer (P:313-321 overlap of transfer with compute): the
 * same wire bytes as hack_kv_send, sent as num_layers NCCL messages so that layer l leaves
 * as soon as its prefill finished (stream-ordered after it) while later layers compute.
 * hack_kv_layer_range: byte range [*begin_out, *begin_out + return) of layer `layer` in the
 * wire buffer (layer 0 includes the 64-byte header); -1 on bad arguments.
 * hack_kv_send_layer: pack layer `layer` of one request (and the header when layer == 0)
 * into `staging` at that range and ncclSend the range.  caches: all num_layers layers.
 * hack_kv_recv_layer: ncclRecv that range into `staging`.  After every layer arrived, one
 * hack_kv_unpack(staging) validates the header and scatters all layers. */
int64_t hack_kv_layer_range(const hack_config_t* cfg, int32_t num_layers, int32_t layer, int32_t prompt_len,
                            int64_t* begin_out);
hack_status_t hack_kv_send_layer(void* comm, int32_t peer, const hack_config_t* cfg,
                                 const hack_kv_cache_t* caches, int32_t num_layers, int32_t layer, int32_t slot,
                                 int32_t prompt_len, int32_t first_token, uint32_t rng_id, void* staging,
                                 void* stream);
hack_status_t hack_kv_recv_layer(void* comm, int32_t peer, const hack_config_t* cfg, int32_t num_layers,
                                 int32_t layer, int32_t prompt_len, void* staging, void* stream);
/* hack_kv_pull (fused transfer): copy one request of num_layers layers from
 * `src` caches straight into `dst` caches in ONE kernel, with no staging buffer, header or
 * NCCL: pages through both block tables (codes + fp16 meta + cached sums), the FP16 tail
 * rows, then dst seq_lens[dst_slot] = prompt_len and dst rng_ids[dst_slot] = src
 * rng_ids[src_slot].  src may be any device-accessible memory, e.g. a prefill rank's
 * cache on a peer GPU opened through CUDA IPC (the loads then cross NVLink) or a cache of
 * another process on the same GPU.  The caller guarantees src is complete (its prefill
 * finished) and stays valid until the pull's stream work completes; dst block tables
 * must already hold pages for the prompt.  Both sides: <= 128 layers sharing
 * block_table/seq_lens/rng_ids.  Errors: INVALID_ARG / SHAPE / CAPACITY as hack_kv_pack. */
hack_status_t hack_kv_pull(const hack_config_t* cfg, const hack_kv_cache_t* src, const hack_kv_cache_t* dst,
                           int32_t num_layers, int32_t src_slot, int32_t dst_slot, int32_t prompt_len,
                           void* stream);
hack_status_t hack_comm_recv_bytes(void* comm, int32_t peer, void* buf, int64_t bytes, void* stream);
hack_status_t hack_comm_group_start(void);
hack_status_t hack_comm_group_end(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* HACK_H_ */
