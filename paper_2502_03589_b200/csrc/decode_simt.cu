// decode_simt.cu -- first correct homomorphic decode attention (a9), CUDA cores.
//
// One CTA per (request, KV head): the G query rows of the KV head (GQA, R15) attend
// to every cached token, streaming the request's pages.  Per page:
//   S = Eq. 4 (centered) on K codes with the CACHED K sums (summation elimination,
//       P:687-690) -- no code is re-summed;
//   online softmax; P quantized to 8 bits per (row, page) when the page's V block is
//   committed, else the page is the FP16 tail (RQE) and P~.V
//   runs in fp32;  O += Eq. 4 (centered) with the CACHED V sums.
// Correctness baseline for the split-KV tensor-core kernel (decode_tc.cu).
#include "common.cuh"
#include "internal.h"

namespace hack {

namespace {

constexpr int kT = 128;
constexpr int kMaxG = 16;

template <int PI>
struct __align__(16) DecodeSmem {
  static constexpr int NB = 128 / PI;
  uint8_t q[kMaxG * 128];
  uint8_t p[kMaxG * PI];
  float s[kMaxG * PI];
  float aq[kMaxG * NB], xq[kMaxG * NB], muq[kMaxG * NB];
  int rq[kMaxG * NB];
  float m_run[kMaxG], l_run[kMaxG], alpha[kMaxG];
  float ap[kMaxG], xp[kMaxG], mup[kMaxG];
  int rp[kMaxG];
};

template <int BITS>
HACK_DEV uint32_t expand_word(const uint8_t* codes, int w) {
  if (BITS == 2) {
    const uint32_t b = codes[w];
    return (b & 3u) | ((b >> 2) & 3u) << 8 | ((b >> 4) & 3u) << 16 | ((b >> 6) & 3u) << 24;
  } else {
    const uint32_t b = reinterpret_cast<const uint16_t*>(codes)[w];
    return (b & 15u) | ((b >> 4) & 15u) << 8 | ((b >> 8) & 15u) << 16 | ((b >> 12) & 15u) << 24;
  }
}

template <int PI, int BITS>
__global__ void __launch_bounds__(kT) decode_simt_kernel(const __half* __restrict__ q_new,
                                                         const int32_t* __restrict__ slots, CacheView cv,
                                                         KernelCfg kc, void* __restrict__ out,
                                                         uint8_t* __restrict__ dbg_pcodes, int64_t dbg_stride) {
  using SM = DecodeSmem<PI>;
  constexpr int NB = SM::NB;
  constexpr int qkm = (1 << BITS) - 1;
  __shared__ SM sm;
  const int b = blockIdx.x, hk = blockIdx.y, G = kc.G;
  const int slot = slots[b];
  const int len = cv.seq_lens[slot];
  const int pos = len - 1;  // position of the new query token
  const uint32_t rng_id = cv.rng_ids[slot];
  const int tid = threadIdx.x;
  const float cscale = 1.4426950408889634f / sqrtf(128.f);
  const PageLayout& PL = kc.pl;

  // (a3) quantize the G query rows (8 rows per pass of 16-lane groups)
  for (int g0 = 0; g0 < G; g0 += 8) {
    const int g = g0 + (tid >> 4), lane16 = tid & 15;
    const int gg = min(g, G - 1);
    const int hq = hk * G + gg;
    const uint4 raw = reinterpret_cast<const uint4*>(q_new + ((int64_t)b * kc.Hq + hq) * 128)[lane16];
    uint64_t packed;
    float m, s;
    int sum;
    quant_row16<8, false>(raw, lane16, PI, pos, kc.seed, rng_id,
                          stream_c3(kc.layer, kTagQ, kc.head_base * G + hq), kc.q_round, packed, m, s, sum);
    if (g < G) {
      *reinterpret_cast<uint2*>(&sm.q[g * 128 + lane16 * 8]) = make_uint2((uint32_t)packed, (uint32_t)(packed >> 32));
      if ((lane16 & (PI / 8 - 1)) == 0) {
        const int beta = lane16 / (PI / 8);
        sm.aq[g * NB + beta] = cscale * s * 0.25f;
        sm.xq[g * NB + beta] = cscale * s * ((float)sum - 127.5f * PI);
        sm.muq[g * NB + beta] = cscale * (m + 127.5f * s);
        sm.rq[g * NB + beta] = 2 * qkm * sum - PI * 255 * qkm;
      }
    }
  }
  if (tid < G) {
    sm.m_run[tid] = -INFINITY;
    sm.l_run[tid] = 0.f;
  }
  float o[kMaxG];
#pragma unroll
  for (int g = 0; g < kMaxG; ++g) o[g] = 0.f;

  const int npages = (len + PI - 1) / PI;
  const int nfull = len / PI;
  for (int j = 0; j < npages; ++j) {
    const uint8_t* pg = cv.pages + ((int64_t)cv.block_table[(int64_t)slot * cv.max_pages_per_req + j] *
                                        cv.num_kv_heads + hk) * cv.page_bytes;
    const int nk = min(PI, len - j * PI);
    const bool committed = j < nfull;
    __syncthreads();
    // ---- S: thread t handles key t of the page
    if (tid < PI) {
      const int t = tid;
      float acc[kMaxG];
#pragma unroll
      for (int g = 0; g < kMaxG; ++g) acc[g] = 0.f;
      if (t < nk) {
        const uint8_t* row = pg + PL.k_codes + t * (128 * BITS / 8);
#pragma unroll
        for (int beta = 0; beta < NB; ++beta) {
          const __half2 mh = reinterpret_cast<const __half2*>(pg + PL.k_meta)[t * NB + beta];
          const float mk = __low2float(mh), sk = __high2float(mh);
          const int sumk = load_sum(pg + PL.k_sums, t * NB + beta, PL.sum_bytes);  // cached sum (SE)
          const float muk = mk + 0.5f * qkm * sk;
          const float yk = sk * ((float)sumk - 0.5f * qkm * PI) + PI * muk;
          const int rk = 510 * sumk;
          uint32_t kw[PI / 4];
#pragma unroll
          for (int w = 0; w < PI / 4; ++w) kw[w] = expand_word<BITS>(row, beta * (PI / 4) + w);
          for (int g = 0; g < G; ++g) {
            uint32_t dacc = 0;
#pragma unroll
            for (int w = 0; w < PI / 4; ++w)
              dacc = __dp4a(*reinterpret_cast<const uint32_t*>(&sm.q[g * 128 + (beta * (PI / 4) + w) * 4]), kw[w], dacc);
            const int dc4 = 4 * (int)dacc - sm.rq[g * NB + beta] - rk;
            acc[g] += sm.aq[g * NB + beta] * sk * (float)dc4 + sm.xq[g * NB + beta] * muk + sm.muq[g * NB + beta] * yk;
          }
        }
      }
      for (int g = 0; g < G; ++g) sm.s[g * PI + t] = t < nk ? acc[g] : -INFINITY;
    }
    __syncthreads();
    // ---- softmax + P quantization: warp w handles rows g = w, w+4, ...
    {
      const int warp = tid >> 5, lane = tid & 31;
      for (int g = warp; g < G; g += kT / 32) {
        float mx = -INFINITY;
        for (int t = lane; t < PI; t += 32) mx = fmaxf(mx, sm.s[g * PI + t]);
        mx = warp_max(mx);
        const float m_old = sm.m_run[g];
        const float m_new = fmaxf(m_old, mx);
        const float al = (m_old == -INFINITY) ? 0.f : ex2(m_old - m_new);
        float lsum = 0.f, lo = INFINITY, hi = -INFINITY;
        for (int t = lane; t < PI; t += 32) {
          const float sv = sm.s[g * PI + t];
          const float p = (sv == -INFINITY) ? 0.f : ex2(sv - m_new);
          sm.s[g * PI + t] = p;
          lsum += p;
          lo = fminf(lo, p);
          hi = fmaxf(hi, p);
        }
        lsum = warp_sum(lsum);
        if (committed) {
          lo = -warp_max(-lo);
          hi = warp_max(hi);
          QMeta pm = meta_fp32(lo, hi, 255);
          if (!(pm.s > 1e-30f)) pm.s = 0.f;
          int sum = 0;
          for (int t = lane; t < PI; t += 32) {
            const int code = quant_rn(sm.s[g * PI + t], pm, 255);
            sm.p[g * PI + t] = (uint8_t)code;
            sum += code;
            if (dbg_pcodes) dbg_pcodes[((int64_t)b * kc.Hq + hk * G + g) * dbg_stride + j * PI + t] = (uint8_t)code;
          }
#pragma unroll
          for (int o2 = 16; o2; o2 >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o2);
          if (lane == 0) {
            sm.ap[g] = pm.s * 0.25f;
            sm.xp[g] = pm.s * ((float)sum - 127.5f * PI);
            sm.mup[g] = pm.m + 127.5f * pm.s;
            sm.rp[g] = 2 * qkm * sum - PI * 255 * qkm;
          }
        }
        if (lane == 0) {
          sm.alpha[g] = al;
          sm.m_run[g] = m_new;
          sm.l_run[g] = sm.l_run[g] * al + lsum;
        }
      }
    }
    __syncthreads();
    // ---- O update: thread c owns channel c for every query row
    {
      const int c = tid;
      for (int g = 0; g < G; ++g) o[g] *= sm.alpha[g];
      if (committed) {
        const uint8_t* vrow = pg + PL.v_codes + c * (PI * BITS / 8);
        const __half2 mh = reinterpret_cast<const __half2*>(pg + PL.v_meta)[c];
        const float mv = __low2float(mh), sv = __high2float(mh);
        const int sumv = load_sum(pg + PL.v_sums, c, PL.sum_bytes);  // cached sum (SE)
        const float muv = mv + 0.5f * qkm * sv;
        const float yv = sv * ((float)sumv - 0.5f * qkm * PI) + PI * muv;
        const int rv = 510 * sumv;
        uint32_t vw[PI / 4];
#pragma unroll
        for (int w = 0; w < PI / 4; ++w) vw[w] = expand_word<BITS>(vrow, w);
        for (int g = 0; g < G; ++g) {
          uint32_t dacc = 0;
#pragma unroll
          for (int w = 0; w < PI / 4; ++w)
            dacc = __dp4a(*reinterpret_cast<const uint32_t*>(&sm.p[g * PI + w * 4]), vw[w], dacc);
          const int dc4 = 4 * (int)dacc - sm.rp[g] - rv;
          o[g] += sm.ap[g] * sv * (float)dc4 + sm.xp[g] * muv + sm.mup[g] * yv;
        }
      } else {
        const __half* tail = reinterpret_cast<const __half*>(cv.v_tail) + ((int64_t)slot * kc.Hkv + hk) * PI * 128;
        for (int t = 0; t < nk; ++t) {
          const float v = __half2float(tail[t * 128 + c]);
          for (int g = 0; g < G; ++g) o[g] = fmaf(sm.s[g * PI + t], v, o[g]);
        }
      }
    }
  }
  // ---- O / l
  for (int g = 0; g < G; ++g) {
    const float v = o[g] / sm.l_run[g];
    const int64_t idx = ((int64_t)b * kc.Hq + hk * G + g) * 128 + tid;
    if (kc.out_fp32)
      reinterpret_cast<float*>(out)[idx] = v;
    else
      reinterpret_cast<__half*>(out)[idx] = __float2half_rn(v);
  }
}

}  // namespace

cudaError_t launch_decode_simt(const KernelCfg& kc, const void* q_new, const int32_t* slots, int batch,
                               const CacheView& cv, void* out, const hack_debug_t* dbg, cudaStream_t st) {
  dim3 grid(batch, kc.Hkv);
  uint8_t* dp = dbg ? dbg->pcodes : nullptr;
  const int64_t ds = dbg ? dbg->pcodes_stride : 0;
  const __half* qh = reinterpret_cast<const __half*>(q_new);
#define HACK_DC(P, B) \
  if (kc.Pi == P && kc.bits == B) { decode_simt_kernel<P, B><<<grid, kT, 0, st>>>(qh, slots, cv, kc, out, dp, ds); note_launch(); return cudaGetLastError(); }
  HACK_DC(32, 2) HACK_DC(64, 2) HACK_DC(128, 2) HACK_DC(32, 4) HACK_DC(64, 4) HACK_DC(128, 4)
#undef HACK_DC
  return cudaErrorInvalidValue;
}

}  // namespace hack
