// internal.h -- host-side types shared by the libhack translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hack.h"
#include "common.cuh"

namespace hack {

// Counts every kernel this library launches (hack_kernel_launches()).
void note_launch(int n = 1);

// Validated, kernel-friendly copy of hack_config_t.
struct KernelCfg {
  int Hq, Hkv, G, d, Pi, bits;
  int kv_round, q_round, p_round;
  uint64_t seed;
  int layer, head_base;
  int out_fp32;
  PageLayout pl;
  int hq_begin, hq_count;    // prefill attention: the query heads this launch computes (all by default)
  int kvh_begin, kvh_count;  // ingest: the KV heads this launch quantizes (all by default)
  // prefill attention: the query tiles of rank [qt_begin, qt_begin + qt_count) of each request
  // (rank 0 = the last positions, the longest causal rows; all by default)
  int qt_begin, qt_count;
};

// Device view of one layer's paged cache (plain POD, passed by value to kernels).
struct CacheView {
  uint8_t* pages;
  void* v_tail;
  int32_t* block_table;
  int32_t* seq_lens;
  uint32_t* rng_ids;
  int num_pages, max_reqs, max_pages_per_req, page_bytes, num_kv_heads;
};

cudaError_t launch_quantize_pack(const KernelCfg& kc, int mode, const void* x, int64_t rows, int heads,
                                 int64_t pos0, int head0, uint32_t rng_id, uint8_t* codes, void* meta,
                                 void* sums, cudaStream_t st);
cudaError_t launch_ingest(const KernelCfg& kc, const void* k, const void* v, const int32_t* cu_seqlens,
                          const int32_t* slots, int batch, int max_seqlen, const CacheView& cv,
                          cudaStream_t st);
cudaError_t launch_append(const KernelCfg& kc, const void* k_new, const void* v_new, const int32_t* slots,
                          int batch, const CacheView& cv, cudaStream_t st);

size_t prefill_workspace_bytes(const KernelCfg& kc, int batch, int max_seqlen);
// pdl: launched right after this call's ingest on the same stream (programmatic dependent)
cudaError_t launch_prefill_attention(const KernelCfg& kc, const void* q, const int32_t* cu_seqlens,
                                     const int32_t* slots, int batch, int max_seqlen, const CacheView& cv,
                                     void* out, void* workspace, const hack_debug_t* dbg, cudaStream_t st,
                                     bool pdl = false);

// whether the prefill kernel serving kc computes a query-head range (kc.hq_begin / hq_count)
bool prefill_head_range_supported(const KernelCfg& kc);
// query positions per query tile of the prefill kernel serving kc (the unit of kc.qt_begin /
// qt_count); 0 if that kernel computes every tile in one launch
int prefill_query_tile_rows(const KernelCfg& kc);

size_t decode_workspace_bytes(const KernelCfg& kc, int batch, int max_seqlen);
// hack_acc_form_t of the kernel the next prefill (op 0) / decode (op 1) call dispatches to
int debug_acc_form(const KernelCfg& kc, int op);
// whether the kernel serving op (0 prefill, 1 decode) implements P stochastic rounding
bool p_sr_supported(const KernelCfg& kc, int op);
cudaError_t launch_decode_step(const KernelCfg& kc, const void* q_new, const void* k_new, const void* v_new,
                               const int32_t* slots, int batch, int max_seqlen, const CacheView& cv, void* out,
                               void* workspace, const hack_debug_t* dbg, cudaStream_t st);
cudaError_t launch_decode_attention(const KernelCfg& kc, const void* q_new, const int32_t* slots, int batch,
                                    int max_seqlen, const CacheView& cv, void* out, void* workspace,
                                    const hack_debug_t* dbg, cudaStream_t st);

cudaError_t launch_dequantize_cache(const KernelCfg& kc, const int32_t* slots, int batch, int max_seqlen,
                                    const CacheView& cv, void* k_out, void* v_out, cudaStream_t st);

cudaError_t launch_homomorphic_matmul(const KernelCfg& kc, const uint8_t* a_codes, const float* a_meta,
                                      const uint16_t* a_sums, const uint8_t* b_packed, const void* b_meta,
                                      const void* b_sums, int M, int N, int Z, int32_t* d_blocks, float* c,
                                      cudaStream_t st);

}  // namespace hack
