// dispatch.cu -- chooses the attention kernel for a launch.
//
// Prefill: the tcgen05 kernel (prefill_tc.cu) for Pi = 64, else the CUDA-core kernel
// (prefill_simt.cu).  Decode: the paired-page mma.sync kernel (decode_pair.cu) for b = 2,
// Pi = 64, G <= 4; the general split-KV mma.sync kernel (decode_mma.cu) for Pi = 64,
// G <= 8; else decode_simt.cu.  HACK_PREFILL_IMPL / HACK_DECODE_IMPL = "simt" force the
// baseline kernels (parity cross-checks); HACK_DECODE_IMPL = "mma" skips the paired kernel.
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace hack {

cudaError_t launch_prefill_simt(const KernelCfg& kc, const void* q, const int32_t* cu, const int32_t* slots,
                                int batch, int max_seqlen, const CacheView& cv, void* out,
                                const hack_debug_t* dbg, cudaStream_t st);
bool prefill_tc_supported(const KernelCfg& kc);
int prefill_tc_tile_rows(const KernelCfg& kc);

cudaError_t launch_prefill_tc(const KernelCfg& kc, const void* q, const int32_t* cu, const int32_t* slots, int batch,
                              int max_seqlen, const CacheView& cv, void* out, const hack_debug_t* dbg,
                              cudaStream_t st, bool pdl);
cudaError_t launch_decode_simt(const KernelCfg& kc, const void* q_new, const int32_t* slots, int batch,
                               const CacheView& cv, void* out, const hack_debug_t* dbg, cudaStream_t st);

bool decode_mma_supported(const KernelCfg& kc);
size_t decode_mma_workspace(const KernelCfg& kc, int batch, int max_seqlen);
cudaError_t launch_decode_mma(const KernelCfg& kc, const void* q_new, const int32_t* slots, int batch,
                              int max_seqlen, const CacheView& cv, void* out, void* workspace,
                              const hack_debug_t* dbg, cudaStream_t st);

bool decode_pair_supported(const KernelCfg& kc);
bool decode_pair_fuse_step(const KernelCfg& kc, int batch, int max_seqlen);
size_t decode_pair_workspace(const KernelCfg& kc, int batch, int max_seqlen);
cudaError_t launch_decode_pair(const KernelCfg& kc, const void* q_new, const int32_t* slots, int batch,
                               int max_seqlen, const CacheView& cv, void* out, void* workspace,
                               const hack_debug_t* dbg, cudaStream_t st, const void* k_new, const void* v_new);

static bool use_decode_mma(const KernelCfg& kc);
static bool use_decode_pair(const KernelCfg& kc);


static bool env_is(const char* name, const char* val) {
  const char* e = getenv(name);
  return e && strcmp(e, val) == 0;
}

size_t prefill_workspace_bytes(const KernelCfg& kc, int batch, int max_seqlen) {
  (void)kc; (void)batch; (void)max_seqlen;
  return 0;
}

cudaError_t launch_prefill_attention(const KernelCfg& kc, const void* q, const int32_t* cu_seqlens,
                                     const int32_t* slots, int batch, int max_seqlen, const CacheView& cv,
                                     void* out, void* workspace, const hack_debug_t* dbg, cudaStream_t st, bool pdl) {
  (void)workspace;
  if (prefill_tc_supported(kc) && !env_is("HACK_PREFILL_IMPL", "simt")) {
    return launch_prefill_tc(kc, q, cu_seqlens, slots, batch, max_seqlen, cv, out, dbg, st, pdl);
  }
  return launch_prefill_simt(kc, q, cu_seqlens, slots, batch, max_seqlen, cv, out, dbg, st);
}

bool prefill_head_range_supported(const KernelCfg& kc) {
  return prefill_tc_supported(kc) && !env_is("HACK_PREFILL_IMPL", "simt");  // (the CUDA-core kernel: all heads)
}

int prefill_query_tile_rows(const KernelCfg& kc) {
  return prefill_head_range_supported(kc) ? prefill_tc_tile_rows(kc) : 0;  // (the CUDA-core kernel: all tiles)
}

static bool use_decode_mma(const KernelCfg& kc) {
  return decode_mma_supported(kc) && !env_is("HACK_DECODE_IMPL", "simt");
}

static bool use_decode_pair(const KernelCfg& kc) {
  // P stochastic rounding (R6, selectable) runs on decode_mma_kernel
  return decode_pair_supported(kc) && kc.p_round == HACK_ROUND_NEAREST_EVEN && !env_is("HACK_DECODE_IMPL", "simt") &&
         !env_is("HACK_DECODE_IMPL", "mma");
}

bool p_sr_supported(const KernelCfg& kc, int op) {
  if (op == 0) return prefill_tc_supported(kc) && !env_is("HACK_PREFILL_IMPL", "simt");
  return use_decode_mma(kc);
}

int debug_acc_form(const KernelCfg& kc, int op) {
  if (op == 0) return prefill_tc_supported(kc) && !env_is("HACK_PREFILL_IMPL", "simt") ? HACK_ACC_S8_2B : HACK_ACC_NONE;
  if (use_decode_pair(kc)) return HACK_ACC_CENTERED4;
  return use_decode_mma(kc) ? HACK_ACC_PLAIN : HACK_ACC_NONE;
}

size_t decode_workspace_bytes(const KernelCfg& kc, int batch, int max_seqlen) {
  if (use_decode_pair(kc)) return decode_pair_workspace(kc, batch, max_seqlen);
  return use_decode_mma(kc) ? decode_mma_workspace(kc, batch, max_seqlen) : 0;
}

cudaError_t launch_decode_attention(const KernelCfg& kc, const void* q_new, const int32_t* slots, int batch,
                                    int max_seqlen, const CacheView& cv, void* out, void* workspace,
                                    const hack_debug_t* dbg, cudaStream_t st) {
  if (use_decode_pair(kc))
    return launch_decode_pair(kc, q_new, slots, batch, max_seqlen, cv, out, workspace, dbg, st, nullptr, nullptr);
  if (use_decode_mma(kc))
    return launch_decode_mma(kc, q_new, slots, batch, max_seqlen, cv, out, workspace, dbg, st);
  return launch_decode_simt(kc, q_new, slots, batch, cv, out, dbg, st);
}

// One decode step (hack_decode_attention): the append (a8) fused into the paired decode
// kernel when decode_pair_fuse_step says so (one launch per step; the SE / RQE ablations keep
// the separate append kernel), else the append kernel followed by the attention.
cudaError_t launch_decode_step(const KernelCfg& kc, const void* q_new, const void* k_new, const void* v_new,
                               const int32_t* slots, int batch, int max_seqlen, const CacheView& cv, void* out,
                               void* workspace, const hack_debug_t* dbg, cudaStream_t st) {
  if (use_decode_pair(kc) && !getenv("HACK_DECODE_NO_RQE") && !getenv("HACK_DECODE_NO_SE") &&
      decode_pair_fuse_step(kc, batch, max_seqlen))
    return launch_decode_pair(kc, q_new, slots, batch, max_seqlen, cv, out, workspace, dbg, st, k_new, v_new);
  const cudaError_t e = launch_append(kc, k_new, v_new, slots, batch, cv, st);
  if (e != cudaSuccess) return e;
  return launch_decode_attention(kc, q_new, slots, batch, max_seqlen, cv, out, workspace, dbg, st);
}

}  // namespace hack
