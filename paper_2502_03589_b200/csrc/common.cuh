// common.cuh -- device helpers shared by the libhack kernels (sm_100a).
//
// Philox4x32-10 (R3), the exact fp32 quantizer op sequence (R1, R4,
// R17), packing, layout constants.
// The CPU oracle implements the same *specification* independently.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "../../include/hack.h"

#define HACK_DEV __device__ __forceinline__

namespace hack {

constexpr int kTagQ = 0, kTagK = 1, kTagV = 2, kTagP = 3;

#ifndef HACK_P_META_IEEE
#define HACK_P_META_IEEE 0  // 1: decode P' meta by IEEE division (meta_p_fast); measured slower
#endif

// ---------------------------------------------------------------- Philox4x32-10
struct Philox4 {
  uint32_t x, y, z, w;
};

HACK_DEV Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                               uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return {c0, c1, c2, c3};
}

// 24-bit uniform in [0,1) from a Philox word: exact in fp32.
HACK_DEV float u24(uint32_t w) { return __uint2float_rn(w >> 8) * 5.9604644775390625e-08f; }

// The counter word c3 of a (layer, tag, head) stream (R3).
HACK_DEV uint32_t stream_c3(int layer, int tag, int head) {
  return ((uint32_t)(layer & 0xFFFF) << 16) | ((uint32_t)(tag & 0xF) << 12) | (uint32_t)(head & 0xFFF);
}

// Four uniforms for Philox block n of a stream.
HACK_DEV Philox4 philox_block(uint64_t seed, uint32_t rng_id, uint32_t c3, uint64_t n) {
  return philox4x32_10((uint32_t)n, (uint32_t)(n >> 32), rng_id, c3, (uint32_t)seed,
                       (uint32_t)(seed >> 32));
}

HACK_DEV uint32_t pick(const Philox4& p, int w) {
  return w == 0 ? p.x : (w == 1 ? p.y : (w == 2 ? p.z : p.w));
}

// P stream (stochastic rounding of P, R6 selectable): the uniform of element (query
// position i, key position t) of global query head `ghead`; Philox block n = (i << 30) |
// (t >> 2), word t & 3 (oracle/philox.py uniforms_p).
HACK_DEV float p_uniform(uint64_t seed, uint32_t rng_id, int layer, int ghead, int64_t i, int t) {
  const Philox4 r = philox_block(seed, rng_id, stream_c3(layer, kTagP, ghead), ((uint64_t)i << 30) | (uint64_t)(t >> 2));
  return u24(pick(r, t & 3));
}
// SR of one P value y = (p - lo) / s (R1): floor(y) + [u < frac(y)], clamped to 255.
HACK_DEV uint32_t p_code_sr(float y, float u) {
  const float fl = floorf(y);
  return (uint32_t)min(255, max(0, (int)fl + (u < y - fl ? 1 : 0)));
}

// ---------------------------------------------------------------- quantizer
// Partition meta: K/V store fp16 (m, s) and compute codes against the stored
// values (R4); Q/P keep fp32 meta.  scale = fp32(fp32(hi - lo) / (2^b - 1)).
struct QMeta {
  float m, s, inv;
};

HACK_DEV QMeta meta_fp16(float lo, float hi, int qmax) {
  const float s32 = __fdiv_rn(__fsub_rn(hi, lo), (float)qmax);
  QMeta q;
  q.m = __half2float(__float2half_rn(lo));
  q.s = __half2float(__float2half_rn(s32));
  q.inv = q.s > 0.f ? __frcp_rn(q.s) : 0.f;  // scale 0: y = 0, every code 0 (R5)
  return q;
}

// Transient P' meta (never stored; decode kernels): a multiply and a fast reciprocal instead
// of the IEEE division and reciprocal.  The codes then agree with meta_fp32's up to near-ties
// (DESIGN "Parity protocol"); the caller zeroes a scale <= 1e-30 (R5).
HACK_DEV QMeta meta_p_fast(float lo, float hi) {
#if HACK_P_META_IEEE
  QMeta q;
  q.m = lo;
  q.s = __fdiv_rn(__fsub_rn(hi, lo), 255.f);
  q.inv = q.s > 0.f ? __frcp_rn(q.s) : 0.f;
  return q;
#else
  const float r = hi - lo;
  return {lo, r * (1.f / 255.f), __fdividef(255.f, r)};
#endif
}

HACK_DEV QMeta meta_fp32(float lo, float hi, int qmax) {
  QMeta q;
  q.m = lo;
  q.s = __fdiv_rn(__fsub_rn(hi, lo), (float)qmax);
  q.inv = q.s > 0.f ? __frcp_rn(q.s) : 0.f;  // scale 0: y = 0, every code 0 (R5)
  return q;
}

// One code: y = fp32(fp32(x - m) * inv); SR: floor(y) + [u < y - floor(y)] (R1);
// RN: rint half-even (R17); scale 0 -> 0 (R5, inv = 0 gives y = 0); clamp to [0, qmax].
// Branch-free: y is clamped to [0, qmax] first, which gives the same code as clamping the
// result (y < 0: floor(y) + [u < frac] <= 0; y > qmax: >= qmax; and u >= 0 so a clamped
// y adds nothing), and the integer part is read off the 1.5 * 2^23 magic sum (|y| < 2^22).
HACK_DEV int quant_sr(float x, const QMeta& q, float u, int qmax) {
  const float y = fminf(fmaxf(__fmul_rn(__fsub_rn(x, q.m), q.inv), 0.f), (float)qmax);
  const float fl = floorf(y);
  return (__float_as_int(__fadd_rn(fl, 12582912.f)) - 0x4B400000) + (u < __fsub_rn(y, fl) ? 1 : 0);
}

HACK_DEV int quant_rn(float x, const QMeta& q, int qmax) {
  const float y = fminf(fmaxf(__fmul_rn(__fsub_rn(x, q.m), q.inv), 0.f), (float)qmax);
  return __float_as_int(__fadd_rn(y, 12582912.f)) - 0x4B400000;  // round half to even
}

// -------------------------------------------------------------------------- K / Q rows
// Quantizes one row (d = 128) held by a 16-lane group; returns this lane's packed
// codes (8 codes, LSB-first: 16 bits at b=2, 32 at b=4, 64 at b=8) and, valid on the
// partition's first lane, the meta and sum.
template <int BITS, bool FP16META>
HACK_DEV void quant_row16(const uint4 raw, int lane16, int Pi, int64_t pos, uint64_t seed,
                          uint32_t rng_id, uint32_t c3, int round, uint64_t& packed, float& m,
                          float& s, int& sum) {
  constexpr int qmax = (1 << BITS) - 1;
  const __half* h = reinterpret_cast<const __half*>(&raw);
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = __half2float(h[i]);
  float lo = x[0], hi = x[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) {
    lo = fminf(lo, x[i]);
    hi = fmaxf(hi, x[i]);
  }
  const int lanes = Pi / 8;  // 4, 8 or 16 lanes per partition
  for (int o = 1; o < lanes; o <<= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  const QMeta q = FP16META ? meta_fp16(lo, hi, qmax) : meta_fp32(lo, hi, qmax);
  int c[8];
  if (round == HACK_ROUND_STOCHASTIC) {
    // element (pos, ch): Philox block n = (pos*d + ch) >> 2, word ch & 3 (R3)
    const uint64_t n0 = ((uint64_t)pos * 128u + (uint64_t)(lane16 * 8)) >> 2;
    const Philox4 r0 = philox_block(seed, rng_id, c3, n0);
    const Philox4 r1 = philox_block(seed, rng_id, c3, n0 + 1);
    c[0] = quant_sr(x[0], q, u24(r0.x), qmax);
    c[1] = quant_sr(x[1], q, u24(r0.y), qmax);
    c[2] = quant_sr(x[2], q, u24(r0.z), qmax);
    c[3] = quant_sr(x[3], q, u24(r0.w), qmax);
    c[4] = quant_sr(x[4], q, u24(r1.x), qmax);
    c[5] = quant_sr(x[5], q, u24(r1.y), qmax);
    c[6] = quant_sr(x[6], q, u24(r1.z), qmax);
    c[7] = quant_sr(x[7], q, u24(r1.w), qmax);
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = quant_rn(x[i], q, qmax);
  }
  uint64_t p = 0;
  int sm = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    p |= (uint64_t)c[i] << (i * BITS);
    sm += c[i];
  }
  for (int o = 1; o < lanes; o <<= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
  packed = p;
  m = q.m;
  s = q.s;
  sum = sm;
}

template <int BITS>
HACK_DEV void store_lane_codes(uint8_t* row_codes, int lane16, uint64_t packed) {
  if (BITS == 2)
    reinterpret_cast<uint16_t*>(row_codes)[lane16] = (uint16_t)packed;
  else if (BITS == 4)
    reinterpret_cast<uint32_t*>(row_codes)[lane16] = (uint32_t)packed;
  else
    reinterpret_cast<uint2*>(row_codes)[lane16] = make_uint2((uint32_t)packed, (uint32_t)(packed >> 32));
}

// -------------------------------------------------------------------------- V blocks
// Quantize one channel's Pi tokens (stride `ts` halves between tokens) starting at
// absolute position pos (a multiple of 4).  Writes Pi*b/8 packed bytes to out
// (16-byte aligned), returns meta + sum.
template <int BITS>
HACK_DEV void quant_vcol(const __half* __restrict__ xc, int64_t ts, int Pi, int64_t pos, int ch,
                         uint64_t seed, uint32_t rng_id, uint32_t c3, int round, uint8_t* out,
                         float& m_out, float& s_out, int& sum_out) {
  constexpr int qmax = (1 << BITS) - 1;
  float lo = __half2float(xc[0]), hi = lo;
  for (int t = 1; t < Pi; ++t) {
    const float v = __half2float(xc[(int64_t)t * ts]);
    lo = fminf(lo, v);
    hi = fmaxf(hi, v);
  }
  const QMeta q = meta_fp16(lo, hi, qmax);
  int sum = 0;
  uint32_t word = 0;
  for (int t0 = 0; t0 < Pi; t0 += 4) {
    int c[4];
    if (round == HACK_ROUND_STOCHASTIC) {
      // element (pos+t, ch): Philox block n = ((pos+t) >> 2)*d + ch, word (pos+t) & 3 (R3)
      const uint64_t n = ((uint64_t)(pos + t0) >> 2) * 128u + (uint64_t)ch;
      const Philox4 r = philox_block(seed, rng_id, c3, n);
      c[0] = quant_sr(__half2float(xc[(int64_t)(t0 + 0) * ts]), q, u24(r.x), qmax);
      c[1] = quant_sr(__half2float(xc[(int64_t)(t0 + 1) * ts]), q, u24(r.y), qmax);
      c[2] = quant_sr(__half2float(xc[(int64_t)(t0 + 2) * ts]), q, u24(r.z), qmax);
      c[3] = quant_sr(__half2float(xc[(int64_t)(t0 + 3) * ts]), q, u24(r.w), qmax);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) c[i] = quant_rn(__half2float(xc[(int64_t)(t0 + i) * ts]), q, qmax);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int t = t0 + i;
      word |= (uint32_t)c[i] << ((t * BITS) & 31);
      sum += c[i];
      if (((t + 1) * BITS & 31) == 0) {
        reinterpret_cast<uint32_t*>(out)[(t * BITS) >> 5] = word;
        word = 0;
      }
    }
  }
  m_out = q.m;
  s_out = q.s;
  sum_out = sum;
}

// ---------------------------------------------------------------- layout
// Page sections; every section 16-byte aligned.
struct PageLayout {
  int k_codes, k_meta, k_sums, v_codes, v_meta, v_sums, page_bytes;
  int sum_bytes;   // 1 (u8) or 2 (u16)
};

__host__ __device__ inline int up16(int x) { return (x + 15) / 16 * 16; }

__host__ __device__ inline int sum_bytes_for(int bits, int Pi) {
  int lg = 0;
  while ((1 << lg) < Pi) ++lg;
  return (bits + lg) <= 8 ? 1 : 2;
}

__host__ __device__ inline PageLayout page_layout(int d, int Pi, int bits) {
  PageLayout L;
  const int nb = d / Pi;
  L.sum_bytes = sum_bytes_for(bits, Pi);
  int o = 0;
  L.k_codes = o; o = up16(o + Pi * d * bits / 8);
  L.k_meta = o;  o = up16(o + Pi * nb * 4);
  L.k_sums = o;  o = up16(o + Pi * nb * L.sum_bytes);
  L.v_codes = o; o = up16(o + d * Pi * bits / 8);
  L.v_meta = o;  o = up16(o + d * 4);
  L.v_sums = o;  o = up16(o + d * L.sum_bytes);
  L.page_bytes = o;
  return L;
}

HACK_DEV void store_sum(uint8_t* base, int idx, int sum_bytes, int v) {
  if (sum_bytes == 1)
    base[idx] = (uint8_t)v;
  else
    reinterpret_cast<uint16_t*>(base)[idx] = (uint16_t)v;
}

HACK_DEV int load_sum(const uint8_t* base, int idx, int sum_bytes) {
  return sum_bytes == 1 ? (int)base[idx] : (int)reinterpret_cast<const uint16_t*>(base)[idx];
}

HACK_DEV __half2 make_meta(float m, float s) { return __halves2half2(__float2half_rn(m), __float2half_rn(s)); }

// ---------------------------------------------------------------- misc
HACK_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
HACK_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
HACK_DEV float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

}  // namespace hack
