// dequant.cu -- the dequantize-first comparator.
//
// NOT on the HACK path: KV-quantization systems such as KVQuant / CacheGen decode the
// stored codes back to FP16 and then run ordinary attention.  This kernel expands the
// same packed pages into a dense FP16 cache, K̂ = m + s c and V̂ = m + s c per partition
// (fp32 FMA of the stored fp16 meta, rounded once to fp16), with the FP16 last V block
// copied as is, so that bench.py can time "dequantize + FP16 attention" on exactly the
// bytes HACK attends to homomorphically.  One CTA per (request, KV head, page); 128
// threads.  Output: k_out, v_out [batch][H_kv][max_seqlen][d] fp16, token-major; rows at
// and beyond the request's length are left untouched.
#include "common.cuh"
#include "internal.h"

namespace hack {

namespace {

template <int BITS>
__global__ void __launch_bounds__(128) dequant_pages_kernel(const int32_t* __restrict__ slots, CacheView cv,
                                                            KernelCfg kc, int max_seqlen, __half* __restrict__ k_out,
                                                            __half* __restrict__ v_out) {
  constexpr int qm = (1 << BITS) - 1;
  const int Pi = kc.Pi, H = kc.Hkv;
  const int b = blockIdx.z, hk = blockIdx.y, p = blockIdx.x;
  const int slot = slots[b];
  const int len = cv.seq_lens[slot];
  if (p * Pi >= len) return;
  const int nk = min(Pi, len - p * Pi);
  const bool committed = (p + 1) * Pi <= len;
  const PageLayout PL = kc.pl;
  const int pid = cv.block_table[(int64_t)slot * cv.max_pages_per_req + p];
  const uint8_t* pg = cv.pages + ((int64_t)pid * cv.num_kv_heads + hk) * cv.page_bytes;
  const int c = threadIdx.x;  // channel
  const int64_t base = (((int64_t)b * H + hk) * max_seqlen + (int64_t)p * Pi) * 128;
  const int nb = 128 / Pi;
  // K: token t, channel c, partition beta = c / Pi
  for (int t = 0; t < nk; ++t) {
    const int beta = c / Pi;
    const __half2 mh = reinterpret_cast<const __half2*>(pg + PL.k_meta)[t * nb + beta];
    const int code = (pg[PL.k_codes + t * (128 * BITS / 8) + c * BITS / 8] >> ((c * BITS) & 7)) & qm;
    k_out[base + (int64_t)t * 128 + c] = __float2half_rn(fmaf(__high2float(mh), (float)code, __low2float(mh)));
  }
  if (committed) {  // V: channel c's Pi tokens form one partition
    const __half2 mh = reinterpret_cast<const __half2*>(pg + PL.v_meta)[c];
    const float m = __low2float(mh), s = __high2float(mh);
    const uint8_t* row = pg + PL.v_codes + c * (Pi * BITS / 8);
    for (int t = 0; t < Pi; ++t) {
      const int code = (row[t * BITS / 8] >> ((t * BITS) & 7)) & qm;
      v_out[base + (int64_t)t * 128 + c] = __float2half_rn(fmaf(s, (float)code, m));
    }
  } else {  // the FP16 last V block (RQE)
    const __half* tail = reinterpret_cast<const __half*>(cv.v_tail) + ((int64_t)slot * H + hk) * Pi * 128;
    for (int t = 0; t < nk; ++t) v_out[base + (int64_t)t * 128 + c] = tail[t * 128 + c];
  }
}

}  // namespace

cudaError_t launch_dequantize_cache(const KernelCfg& kc, const int32_t* slots, int batch, int max_seqlen,
                                    const CacheView& cv, void* k_out, void* v_out, cudaStream_t st) {
  dim3 grid((max_seqlen + kc.Pi - 1) / kc.Pi, kc.Hkv, batch);
  if (kc.bits == 2)
    dequant_pages_kernel<2><<<grid, 128, 0, st>>>(slots, cv, kc, max_seqlen, reinterpret_cast<__half*>(k_out),
                                                   reinterpret_cast<__half*>(v_out));
  else
    dequant_pages_kernel<4><<<grid, 128, 0, st>>>(slots, cv, kc, max_seqlen, reinterpret_cast<__half*>(k_out),
                                                   reinterpret_cast<__half*>(v_out));
  note_launch();
  return cudaGetLastError();
}

}  // namespace hack
