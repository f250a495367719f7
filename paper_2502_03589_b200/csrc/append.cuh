// append.cuh -- the decode append (a8) of one (request, KV head), shared by the append
// kernel (quant_kernels.cu) and the fused decode step (decode_pair.cu).
#pragma once
#include "common.cuh"
#include "internal.h"

namespace hack {

HACK_DEV uint8_t* page_ptr(const CacheView& cv, int slot, int blk, int h) {
  const int pid = cv.block_table[(int64_t)slot * cv.max_pages_per_req + blk];
  return cv.pages + ((int64_t)pid * cv.num_kv_heads + h) * cv.page_bytes;
}

// One (request, KV head) of the append (a8) on NT threads (thread c = channels c, c + NT, ..):
// k_new's
// row quantized into its own partitions at row t % Pi of page t / Pi, v_new to the
// FP16 tail, the tail flushed into the page's V section when it reaches Pi.  t is the
// request's length before the append.  Used by append_kernel and by the fused decode step
// (decode_pair.cu); `sync` is a barrier over the NT threads (NT >= 32).
template <int BITS, bool RQE, int NT, class Sync>
HACK_DEV void append_unit(const __half* __restrict__ k_new, const __half* __restrict__ v_new, int b, int slot, int t,
                          int h, const CacheView& cv, const KernelCfg& kc, int tid, Sync sync) {
  static_assert(NT >= 32, "the K row takes a warp");
  const int H = kc.Hkv, Pi = kc.Pi;
  const int blk = t / Pi, row = t % Pi;
  const uint32_t rng_id = cv.rng_ids[slot];
  const PageLayout& PL = kc.pl;
  uint8_t* pg = page_ptr(cv, slot, blk, h);
  if (tid < 32) {  // K row: lanes 0-15 (16-31 duplicate, no store)
    const int lane16 = tid & 15;
    const uint4 raw = reinterpret_cast<const uint4*>(k_new + ((int64_t)b * H + h) * 128)[lane16];
    uint64_t packed;
    float m, s;
    int sum;
    quant_row16<BITS, true>(raw, lane16, Pi, t, kc.seed, rng_id,
                            stream_c3(kc.layer, kTagK, kc.head_base + h), kc.kv_round, packed, m, s,
                            sum);
    if (tid < 16) {
      store_lane_codes<BITS>(pg + PL.k_codes + row * (128 * BITS / 8), lane16, packed);
      const int nb = 128 / Pi;
      if ((lane16 & (Pi / 8 - 1)) == 0) {
        const int beta = lane16 / (Pi / 8);
        reinterpret_cast<__half2*>(pg + PL.k_meta)[row * nb + beta] = make_meta(m, s);
        store_sum(pg + PL.k_sums, row * nb + beta, PL.sum_bytes, sum);
      }
    }
  }
  __half* tail = reinterpret_cast<__half*>(cv.v_tail) + (((int64_t)slot * H + h) * Pi) * 128;
  for (int c = tid; c < 128; c += NT) tail[row * 128 + c] = v_new[((int64_t)b * H + h) * 128 + c];
  if (row == Pi - 1) {  // the tail reached Pi tokens: quantize and commit (RQE flush)
    sync();
    for (int c = tid; c < 128; c += NT) {
      float m, s;
      int sum;
      quant_vcol<BITS>(tail + c, 128, Pi, (int64_t)blk * Pi, c, kc.seed, rng_id,
                       stream_c3(kc.layer, kTagV, kc.head_base + h), kc.kv_round,
                       pg + PL.v_codes + c * (Pi * BITS / 8), m, s, sum);
      reinterpret_cast<__half2*>(pg + PL.v_meta)[c] = make_meta(m, s);
      store_sum(pg + PL.v_sums, c, PL.sum_bytes, sum);
    }
  } else if (!RQE) {
    static_assert(RQE || NT == 128, "the RQE ablation runs on 128 threads");
    const int c = tid;
    // "HACK/RQE" ablation: without requantization
    // elimination the partially filled last V block is requantized at every step, as one
    // partition of its row + 1 tokens per channel (same quantizer and position-keyed SR
    // counters as a flush), into the page's (otherwise unused) V section.  Attention still
    // reads the FP16 tail, so this variant measures the requantization cost only.
    sync();
    constexpr int qmax = (1 << BITS) - 1;
    const int nk = row + 1;
    const __half* xc = tail + c;
    float lo = __half2float(xc[0]), hi = lo;
    for (int tt = 1; tt < nk; ++tt) {
      const float v = __half2float(xc[tt * 128]);
      lo = fminf(lo, v);
      hi = fmaxf(hi, v);
    }
    const QMeta q = meta_fp16(lo, hi, qmax);
    uint32_t* dst = reinterpret_cast<uint32_t*>(pg + PL.v_codes + c * (Pi * BITS / 8));
    uint32_t word = 0;
    int sum = 0;
    const uint32_t c3 = stream_c3(kc.layer, kTagV, kc.head_base + h);
    for (int t0 = 0; t0 < nk; t0 += 4) {
      float u[4] = {0.f, 0.f, 0.f, 0.f};
      if (kc.kv_round == HACK_ROUND_STOCHASTIC) {
        const Philox4 r = philox_block(kc.seed, rng_id, c3, (uint64_t)((blk * Pi + t0) >> 2) * 128u + (uint64_t)c);
        u[0] = u24(r.x); u[1] = u24(r.y); u[2] = u24(r.z); u[3] = u24(r.w);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int tt = t0 + i;
        if (tt < nk) {
          const float x = __half2float(xc[tt * 128]);
          const int cc = kc.kv_round == HACK_ROUND_STOCHASTIC ? quant_sr(x, q, u[i], qmax) : quant_rn(x, q, qmax);
          word |= (uint32_t)cc << ((tt * BITS) & 31);
          sum += cc;
        }
        if (tt == nk - 1) dst[(tt * BITS) >> 5] = word;  // last (partial) word; codes past nk are 0
        if (((tt + 1) * BITS & 31) == 0) {
          if (tt < nk - 1) dst[(tt * BITS) >> 5] = word;
          word = 0;
        }
      }
    }
    reinterpret_cast<__half2*>(pg + PL.v_meta)[c] = make_meta(q.m, q.s);
    store_sum(pg + PL.v_sums, c, PL.sum_bytes, sum);
  }
}

}  // namespace hack
