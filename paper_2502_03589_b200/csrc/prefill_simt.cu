// prefill_simt.cu -- first correct homomorphic prefill attention (a3-a7), CUDA cores.
//
// FlashAttention-style tile loop over Pi-key tiles for a 64-row query tile of one
// query head, entirely on integer codes:
//   (a3) Q rows quantized in-kernel to 8-bit, partitions along d;
//   (a4) D_beta = Q'_beta K'_beta^T exact int32 (dp4a on unpacked codes), S by Eq. 4
//        per d-block in CENTERED form,
//        times log2(e)/sqrt(d) (Eq. 2, R9);
//   (a5) causal online softmax in fp32 (Eq. 3, R8);
//   (a6) P quantized per (row, Pi-key block) to 8 bits, RN (R6) on the
//        unnormalised p~ (codes are invariant to the row scale);
//   (a7) D' = P'V' exact int32, O += Eq. 4 (centered) per block; the FP16 tail block
//        (RQE) as fp32 FMAs; O /= l (R14).
// This is the correctness baseline the tcgen05 kernel (prefill_tc.cu) is checked
// against; it is not the tuned path.
#include "common.cuh"
#include "internal.h"

namespace hack {

namespace {

constexpr int BM = 64;        // query rows per CTA
constexpr int kThreads = 256;

template <int PI>
struct __align__(16) PrefillSmem {
  static constexpr int BN = PI;                 // key tile = one V block (Pi-aligned, a6)
  static constexpr int QS = 128 + 4;            // padded u8 row strides (bank spread)
  static constexpr int KS = 128 + 4;
  static constexpr int PS = BN + 4;
  static constexpr int VS = BN + 4;
  static constexpr int NB = 128 / PI;
  uint8_t q[BM * QS];
  uint8_t k[BN * KS];
  uint8_t p[BM * PS];
  union {
    uint8_t v[128 * VS];
    __half vt[BN * 128];
  } vv;
  float s[BM * (BN + 1)];
  // per query row, per d-block (centered Eq. 4 coefficients, scaled by log2e/sqrt(d))
  float aq[BM * NB], xq[BM * NB], muq[BM * NB];
  int rq[BM * NB];
  // per key, per d-block
  float sk[BN * NB], muk[BN * NB], yk[BN * NB];
  int rk[BN * NB];
  // per channel (V block)
  float sv[128], muv[128], yv[128];
  int rv[128];
  // per query row: softmax state and P-block coefficients
  float m_run[BM], l_run[BM], alpha[BM];
  float ap[BM], xp[BM], mup[BM];
  int rp[BM];
};

template <int BITS>
HACK_DEV uint32_t expand4(uint32_t byte_bits) {
  // BITS=2: 4 codes of one byte -> 4 bytes. BITS=4: 2 codes per byte (caller passes 2 bytes)
  if (BITS == 2)
    return (byte_bits & 3u) | ((byte_bits >> 2) & 3u) << 8 | ((byte_bits >> 4) & 3u) << 16 |
           ((byte_bits >> 6) & 3u) << 24;
  else
    return (byte_bits & 15u) | ((byte_bits >> 4) & 15u) << 8 | ((byte_bits >> 8) & 15u) << 16 |
           ((byte_bits >> 12) & 15u) << 24;
}

// Unpack `n` codes stored LSB-first at `src` into bytes at `dst` (n % 4 == 0).
template <int BITS>
HACK_DEV void unpack_codes(const uint8_t* src, uint8_t* dst, int n, int tid, int nthreads) {
  for (int w = tid; w < n / 4; w += nthreads) {
    uint32_t bits = BITS == 2 ? (uint32_t)src[w] : (uint32_t)reinterpret_cast<const uint16_t*>(src)[w];
    reinterpret_cast<uint32_t*>(dst)[w] = expand4<BITS>(bits);
  }
}

template <int PI, int BITS>
__global__ void __launch_bounds__(kThreads) prefill_simt_kernel(
    const __half* __restrict__ q, const int32_t* __restrict__ cu_seqlens, const int32_t* __restrict__ slots,
    CacheView cv, KernelCfg kc, void* __restrict__ out, uint8_t* __restrict__ dbg_pcodes,
    int64_t dbg_stride) {
  using SM = PrefillSmem<PI>;
  constexpr int BN = SM::BN, NB = SM::NB;
  constexpr int qkm = (1 << BITS) - 1;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);

  const int b = blockIdx.z, hq = blockIdx.y;
  const int start = cu_seqlens[b], L = cu_seqlens[b + 1] - start;
  const int nqt = (L + BM - 1) / BM;
  if ((int)blockIdx.x >= nqt) return;
  const int qt = nqt - 1 - blockIdx.x;  // longest (diagonal-heavy) tiles first
  const int i0 = qt * BM;
  const int slot = slots[b];
  const int hk = hq / kc.G;
  const int tid = threadIdx.x;
  const uint32_t rng_id = cv.rng_ids[slot];
  const float cscale = 1.4426950408889634f / sqrtf(128.f);  // log2(e)/sqrt(d) folded into S
  const PageLayout& PL = kc.pl;

  // ---- (a3) quantize the Q tile: 16 lanes per row, 16 rows per pass
  for (int r0 = 0; r0 < BM; r0 += 16) {
    const int r = r0 + (tid >> 4), lane16 = tid & 15;
    const int i = min(i0 + r, L - 1);
    const uint4 raw = reinterpret_cast<const uint4*>(q + ((int64_t)(start + i) * kc.Hq + hq) * 128)[lane16];
    uint64_t packed;
    float m, s;
    int sum;
    quant_row16<8, false>(raw, lane16, PI, i, kc.seed, rng_id,
                          stream_c3(kc.layer, kTagQ, kc.head_base * kc.G + hq), kc.q_round, packed, m, s, sum);
    uint32_t* qd = reinterpret_cast<uint32_t*>(&sm.q[r * SM::QS + lane16 * 8]);  // row stride is 4-aligned
    qd[0] = (uint32_t)packed;
    qd[1] = (uint32_t)(packed >> 32);
    if ((lane16 & (PI / 8 - 1)) == 0) {
      const int beta = lane16 / (PI / 8);
      // centered: q_hat = s (q' - 127.5) + mu,  mu = m + 127.5 s
      sm.aq[r * NB + beta] = cscale * s * 0.25f;
      sm.xq[r * NB + beta] = cscale * s * ((float)sum - 127.5f * PI);
      sm.muq[r * NB + beta] = cscale * (m + 127.5f * s);
      sm.rq[r * NB + beta] = 2 * qkm * sum - PI * 255 * qkm;
    }
  }
  if (tid < BM) {
    sm.m_run[tid] = -INFINITY;
    sm.l_run[tid] = 0.f;
  }

  float o[4][8];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 8; ++c) o[a][c] = 0.f;

  const int ty = tid >> 4, tx = tid & 15;
  const int nfull = L / PI;
  const int last_tile = min((i0 + BM - 1) / BN, (L - 1) / BN);
  const int T = L - nfull * PI;  // FP16 tail tokens

  for (int j = 0; j <= last_tile; ++j) {
    const int t0 = j * BN;
    const bool committed = j < nfull;
    const uint8_t* pg = cv.pages + ((int64_t)cv.block_table[(int64_t)slot * cv.max_pages_per_req + j] *
                                        cv.num_kv_heads + hk) * cv.page_bytes;
    __syncthreads();  // previous tile fully consumed
    // ---- load + unpack K tile (codes row-major [t][d]) and key coefficients
    {
      const int nk = min(BN, L - t0);
      for (int w = tid; w < BN * 32; w += kThreads) {  // 32 u32 words (128 codes) per key
        const int t = w >> 5, ww = w & 31;
        uint32_t val = 0;
        if (t < nk) {
          const uint8_t* row = pg + PL.k_codes + t * (128 * BITS / 8);
          val = BITS == 2 ? expand4<2>(row[ww]) : expand4<4>(reinterpret_cast<const uint16_t*>(row)[ww]);
        }
        *reinterpret_cast<uint32_t*>(&sm.k[t * SM::KS + ww * 4]) = val;
      }
      for (int e = tid; e < BN * NB; e += kThreads) {
        const int t = e / NB;
        float s = 0.f, m = 0.f;
        int sum = 0;
        if (t < nk) {
          const __half2 mh = reinterpret_cast<const __half2*>(pg + PL.k_meta)[e];
          m = __low2float(mh);
          s = __high2float(mh);
          sum = load_sum(pg + PL.k_sums, e, PL.sum_bytes);
        }
        const float mu = m + 0.5f * qkm * s;
        sm.sk[e] = s;
        sm.muk[e] = mu;
        sm.yk[e] = s * ((float)sum - 0.5f * qkm * PI) + PI * mu;
        sm.rk[e] = 510 * sum;
      }
    }
    // ---- load V: committed block codes (channel-major [c][t]) or the FP16 tail
    if (committed) {
      for (int w = tid; w < 128 * (BN / 4); w += kThreads) {
        const int c = w / (BN / 4), ww = w % (BN / 4);
        const uint8_t* row = pg + PL.v_codes + c * (BN * BITS / 8);
        const uint32_t val = BITS == 2 ? expand4<2>(row[ww]) : expand4<4>(reinterpret_cast<const uint16_t*>(row)[ww]);
        *reinterpret_cast<uint32_t*>(&sm.vv.v[c * SM::VS + ww * 4]) = val;
      }
      if (tid < 128) {
        const __half2 mh = reinterpret_cast<const __half2*>(pg + PL.v_meta)[tid];
        const float m = __low2float(mh), s = __high2float(mh);
        const int sum = load_sum(pg + PL.v_sums, tid, PL.sum_bytes);
        const float mu = m + 0.5f * qkm * s;
        sm.sv[tid] = s;
        sm.muv[tid] = mu;
        sm.yv[tid] = s * ((float)sum - 0.5f * qkm * PI) + PI * mu;
        sm.rv[tid] = 510 * sum;
      }
    } else {
      const __half* tail = reinterpret_cast<const __half*>(cv.v_tail) + ((int64_t)slot * kc.Hkv + hk) * PI * 128;
      for (int e = tid; e < BN * 128; e += kThreads) {
        const int t = e >> 7;
        sm.vv.vt[e] = t < T ? tail[e] : __float2half(0.f);
      }
    }
    __syncthreads();

    // ---- (a4) S tile: thread owns rows ty*4+a, keys tx + 16*n
    {
      constexpr int TN = BN / 16;
      float acc[4][TN];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int n = 0; n < TN; ++n) acc[a][n] = 0.f;
#pragma unroll
      for (int beta = 0; beta < NB; ++beta) {
        uint32_t dacc[4][TN];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int n = 0; n < TN; ++n) dacc[a][n] = 0u;
        for (int w = beta * (PI / 4); w < (beta + 1) * (PI / 4); ++w) {
          uint32_t qa[4], kb[TN];
#pragma unroll
          for (int a = 0; a < 4; ++a) qa[a] = *reinterpret_cast<const uint32_t*>(&sm.q[(ty * 4 + a) * SM::QS + w * 4]);
#pragma unroll
          for (int n = 0; n < TN; ++n) kb[n] = *reinterpret_cast<const uint32_t*>(&sm.k[(tx + 16 * n) * SM::KS + w * 4]);
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int n = 0; n < TN; ++n) dacc[a][n] = __dp4a(qa[a], kb[n], dacc[a][n]);
        }
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const int r = ty * 4 + a;
          const float aq = sm.aq[r * NB + beta], xq = sm.xq[r * NB + beta], muq = sm.muq[r * NB + beta];
          const int rq = sm.rq[r * NB + beta];
#pragma unroll
          for (int n = 0; n < TN; ++n) {
            const int t = tx + 16 * n;
            const int e = t * NB + beta;
            const int dc4 = 4 * (int)dacc[a][n] - rq - sm.rk[e];  // 4 * centered integer dot (exact)
            acc[a][n] += aq * sm.sk[e] * (float)dc4 + xq * sm.muk[e] + muq * sm.yk[e];
          }
        }
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int n = 0; n < TN; ++n) {
          const int r = ty * 4 + a, t = tx + 16 * n;
          const bool vis = (t0 + t) <= (i0 + r) && (t0 + t) < L;
          sm.s[r * (BN + 1) + t] = vis ? acc[a][n] : -INFINITY;
        }
    }
    __syncthreads();

    // ---- (a5) online softmax + (a6) P quantization: 4 threads per row
    {
      const int r = tid >> 2, part = tid & 3;
      constexpr int per = BN / 4;
      float* srow = &sm.s[r * (BN + 1) + part * per];
      float mx = -INFINITY;
      for (int n = 0; n < per; ++n) mx = fmaxf(mx, srow[n]);
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float m_old = sm.m_run[r];
      const float m_new = fmaxf(m_old, mx);   // finite: key 0 is visible to every row
      const float al = (m_old == -INFINITY) ? 0.f : ex2(m_old - m_new);
      float lsum = 0.f, lo = INFINITY, hi = -INFINITY;
      for (int n = 0; n < per; ++n) {
        const float sv = srow[n];
        const float p = (sv == -INFINITY) ? 0.f : ex2(sv - m_new);
        srow[n] = p;
        lsum += p;
        lo = fminf(lo, p);
        hi = fmaxf(hi, p);
      }
      lsum += __shfl_xor_sync(0xffffffffu, lsum, 1);
      lsum += __shfl_xor_sync(0xffffffffu, lsum, 2);
      __syncwarp();
      if (committed) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, 1));
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, 2));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, 1));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, 2));
        QMeta pm = meta_fp32(lo, hi, 255);
        if (!(pm.s > 1e-30f)) pm.s = 0.f;  // degenerate / underflowed block: constant (R5)
        int sum = 0;
        for (int n = 0; n < per; ++n) {
          const int code = quant_rn(srow[n], pm, 255);
          sm.p[r * SM::PS + part * per + n] = (uint8_t)code;
          sum += code;
          if (dbg_pcodes != nullptr && i0 + r < L)
            dbg_pcodes[((int64_t)(start + i0 + r) * kc.Hq + hq) * dbg_stride + t0 + part * per + n] = (uint8_t)code;
        }
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        sum += __shfl_xor_sync(0xffffffffu, sum, 2);
        if (part == 0) {
          sm.ap[r] = pm.s * 0.25f;
          sm.xp[r] = pm.s * ((float)sum - 127.5f * PI);
          sm.mup[r] = pm.m + 127.5f * pm.s;
          sm.rp[r] = 2 * qkm * sum - PI * 255 * qkm;
        }
      }
      if (part == 0) {
        sm.alpha[r] = al;
        sm.m_run[r] = m_new;
        sm.l_run[r] = sm.l_run[r] * al + lsum;
      }
    }
    __syncthreads();

    // ---- (a7) O update: thread owns rows ty*4+a, channels tx + 16*n
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const float al = sm.alpha[ty * 4 + a];
#pragma unroll
      for (int n = 0; n < 8; ++n) o[a][n] *= al;
    }
    if (committed) {
      uint32_t dacc[4][8];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int n = 0; n < 8; ++n) dacc[a][n] = 0u;
      for (int w = 0; w < BN / 4; ++w) {
        uint32_t pa[4], vb[8];
#pragma unroll
        for (int a = 0; a < 4; ++a) pa[a] = *reinterpret_cast<const uint32_t*>(&sm.p[(ty * 4 + a) * SM::PS + w * 4]);
#pragma unroll
        for (int n = 0; n < 8; ++n) vb[n] = *reinterpret_cast<const uint32_t*>(&sm.vv.v[(tx + 16 * n) * SM::VS + w * 4]);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int n = 0; n < 8; ++n) dacc[a][n] = __dp4a(pa[a], vb[n], dacc[a][n]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int r = ty * 4 + a;
        const float ap = sm.ap[r], xp = sm.xp[r], mup = sm.mup[r];
        const int rp = sm.rp[r];
#pragma unroll
        for (int n = 0; n < 8; ++n) {
          const int c = tx + 16 * n;
          const int dc4 = 4 * (int)dacc[a][n] - rp - sm.rv[c];
          o[a][n] += ap * sm.sv[c] * (float)dc4 + xp * sm.muv[c] + mup * sm.yv[c];
        }
      }
    } else {
      for (int t = 0; t < BN; ++t) {
        float vt[8];
#pragma unroll
        for (int n = 0; n < 8; ++n) vt[n] = __half2float(sm.vv.vt[t * 128 + tx + 16 * n]);
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const float p = sm.s[(ty * 4 + a) * (BN + 1) + t];
#pragma unroll
          for (int n = 0; n < 8; ++n) o[a][n] = fmaf(p, vt[n], o[a][n]);
        }
      }
    }
  }

  // ---- epilogue: O / l
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int r = ty * 4 + a;
    if (i0 + r >= L) continue;
    const float inv_l = 1.f / sm.l_run[r];
    const int64_t base = ((int64_t)(start + i0 + r) * kc.Hq + hq) * 128;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const int c = tx + 16 * n;
      const float v = o[a][n] * inv_l;
      if (kc.out_fp32)
        reinterpret_cast<float*>(out)[base + c] = v;
      else
        reinterpret_cast<__half*>(out)[base + c] = __float2half_rn(v);
    }
  }
}

template <int PI, int BITS>
cudaError_t launch_t(const KernelCfg& kc, const void* q, const int32_t* cu, const int32_t* slots, int batch,
                     int max_seqlen, const CacheView& cv, void* out, const hack_debug_t* dbg, cudaStream_t st) {
  const size_t smem = sizeof(PrefillSmem<PI>);
  auto kern = prefill_simt_kernel<PI, BITS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((max_seqlen + BM - 1) / BM, kc.Hq, batch);
  kern<<<grid, kThreads, smem, st>>>(reinterpret_cast<const __half*>(q), cu, slots, cv, kc, out,
                                     dbg ? dbg->pcodes : nullptr, dbg ? dbg->pcodes_stride : 0);
  note_launch();
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_prefill_simt(const KernelCfg& kc, const void* q, const int32_t* cu, const int32_t* slots,
                                int batch, int max_seqlen, const CacheView& cv, void* out,
                                const hack_debug_t* dbg, cudaStream_t st) {
#define HACK_PF(P, B) \
  if (kc.Pi == P && kc.bits == B) return launch_t<P, B>(kc, q, cu, slots, batch, max_seqlen, cv, out, dbg, st);
  HACK_PF(32, 2) HACK_PF(64, 2) HACK_PF(128, 2) HACK_PF(32, 4) HACK_PF(64, 4) HACK_PF(128, 4)
#undef HACK_PF
  return cudaErrorInvalidValue;
}

}  // namespace hack
