// decode_pair.cu -- HBM-bound homomorphic decode attention (a9) for GQA groups G <= 4,
// b = 2, Pi = 64 (the C3 Llama-3.1-8B / Mistral-7B shapes), split-KV.
//
// Same arithmetic as decode_mma.cu (Eq. 4 per block, in centered form; cached
// K/V code sums = summation elimination; P 8-bit RN per (row, V block), P:537;
// FP16 last V block, RQE), re-tiled so that every lane of every mma.sync does
// useful work when G = 4 and so that each unpacked plane costs ~1.25 ALU ops:
//   * S^T = K' Q'^T with tokens as M and N = 8 columns = (query row, d-block beta): both
//     d-blocks come out of ONE accumulator chain (B is zero outside the column's block),
//     so a lane holds (beta0, beta1) of one query row -> Eq. 4 on fp32x2 pairs, no
//     padding lanes.
//   * O^T = V' P'^T over a PAIR of pages with N = (query row, page): K = 128 tokens, B is
//     zero outside the column's page, so the PV epilogue runs on (page A, page B) pairs.
//   * each lane unpacks the codes of its OWN 32-bit words: plane q of a 2-bit word is
//     (w >> 4*(q>>1)) & (3 << 2*(q&1)), i.e. planes 1 and 3 come out multiplied by 4.
//     k-steps fed by scaled planes go to a second accumulator; 4*acc0 + acc1 = 4*D is
//     exactly the integer the centered Eq. 4 needs (one LEA).  The accumulator of the
//     scaled planes starts at 1.5*2^23 + (row constant) in integer form, so its float view
//     is 1.5*2^23 + 4D + RC and a single FADD2 with a per-token constant yields the
//     centered integer e exactly.
//   * K-side Eq. 4 coefficients are computed per lane from the page's fp16 meta and cached
//     sums; V-side coefficients are staged once per pair in shared memory (over the
//     consumed K codes of page A and a 2 KB per-warp area).
//   * one producer lane streams whole pages (cp.async.bulk, 12-slot ring, 3 CTAs/SM).
#include <cstdlib>

#include "common.cuh"
#include "internal.h"
#include "tc_ptx.cuh"

namespace hack {

namespace {

constexpr int PI = 64;
constexpr int NW = 4;       // compute warps per CTA
constexpr int NSTG = 12;    // page slots per CTA
constexpr int kThreads = (NW + 1) * 32;
constexpr int PB = 5376;    // page bytes at d = 128, Pi = 64, b = 2
constexpr uint32_t kMagic = 0x4B400000u;   // bits of 1.5 * 2^23
constexpr float kMagicF = 12582912.f;      // 1.5 * 2^23

struct PairSmem {
  union {
    uint8_t stage[NSTG][PB];
    float mrg_o[NW][4][128];  // after the page loop: per-warp partial O
  };
  float4 vc_hi[NW][64][2];    // V coefficients of channels 64..127 (channels 0..63: page A's K codes)
  uint8_t qcode[4][128];      // Q' rows, natural channel order
  float4 qc[4][2];            // per row: (QA0, QA1, QX0, QX1), (QM0, QM1, RC0, RC1)
  float mrg_m[NW][4], mrg_l[NW][4];
  uint64_t full[NSTG], empty[NSTG];
};

HACK_DEV void mma16832(uint32_t (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                       uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// d = a b + c with a separate accumulator input (no register moves for the initial value)
HACK_DEV void mma16832c(uint32_t (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                        uint32_t b1, uint32_t c0, uint32_t c1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%10,%11,%10,%11};"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "r"(c0), "r"(c1));
}

// The four planes of a 2-bit word: p[q] holds codes {q, q+4, q+8, q+12} in bytes 0..3;
// p[1], p[3] are scaled by 4 (no shift back).
struct Planes {
  uint32_t p0, p1, p2, p3;
};
HACK_DEV Planes planes2(uint32_t w) {
  const uint32_t x = w >> 4;
  return {w & 0x03030303u, w & 0x0C0C0C0Cu, x & 0x03030303u, x & 0x0C0C0C0Cu};
}

HACK_DEV float2 f2(float a, float b) { return make_float2(a, b); }
HACK_DEV float2 asf2(uint32_t a, uint32_t b) { return make_float2(__uint_as_float(a), __uint_as_float(b)); }

// Homomorphic S^T for one 64-token page: sc[mt][hh] = log2(e)/sqrt(d) * S(token 16mt+g+8hh, row tig).
// Tokens >= nk are -inf.  Returns the per-lane max/min over its 8 tokens.
HACK_DEV void qk_page(const uint8_t* pg, const PageLayout& PL, int g, int tig, int nk, const uint32_t (&qb)[4][2],
                      float2 QA, float2 QX, float2 QM, uint32_t rc0, uint32_t rc1, float (&sc)[4][2], float& mx,
                      float& mn) {
  mx = -INFINITY;
  mn = INFINITY;
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int t0 = 16 * mt + g, t1 = t0 + 8;
    const uint2 w0 = *reinterpret_cast<const uint2*>(pg + PL.k_codes + t0 * 32 + 8 * tig);
    const uint2 w1 = *reinterpret_cast<const uint2*>(pg + PL.k_codes + t1 * 32 + 8 * tig);
    const Planes a0 = planes2(w0.x), a1 = planes2(w1.x), a2 = planes2(w0.y), a3 = planes2(w1.y);
    uint32_t acc0[4], acc1[4];
    // k-steps: plane 0 -> acc0, plane 2 -> acc0, plane 1 (x4) -> acc1, plane 3 (x4) -> acc1;
    // acc1 starts at 1.5*2^23 + RC (integer view), acc0 at 0
    mma16832c(acc0, a0.p0, a1.p0, a2.p0, a3.p0, qb[0][0], qb[0][1], 0u, 0u);
    mma16832(acc0, a0.p2, a1.p2, a2.p2, a3.p2, qb[1][0], qb[1][1]);
    mma16832c(acc1, a0.p1, a1.p1, a2.p1, a3.p1, qb[2][0], qb[2][1], rc0, rc1);
    mma16832(acc1, a0.p3, a1.p3, a2.p3, a3.p3, qb[3][0], qb[3][1]);
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int t = hh ? t1 : t0;
      // per-token coefficients from fp16 meta + cached sums (SE): (beta0, beta1) pairs
      const uint2 mh = *reinterpret_cast<const uint2*>(pg + PL.k_meta + t * 8);
      const uint32_t sums = *reinterpret_cast<const uint16_t*>(pg + PL.k_sums + t * 2);
      const float2 m01 = __half22float2(__halves2half2(__ushort_as_half((unsigned short)(mh.x & 0xFFFF)),
                                                       __ushort_as_half((unsigned short)(mh.y & 0xFFFF))));
      const float2 s01 = __half22float2(__halves2half2(__ushort_as_half((unsigned short)(mh.x >> 16)),
                                                       __ushort_as_half((unsigned short)(mh.y >> 16))));
      // sum bytes -> floats exactly via 2^23 + byte
      const float2 sum2 = ptx::fadd2(asf2(0x4B000000u | (sums & 0xFF), 0x4B000000u | (sums >> 8)),
                                     f2(-8388608.f, -8388608.f));
      const float2 mu = ptx::ffma2(s01, f2(1.5f, 1.5f), m01);
      const float2 yk = ptx::ffma2(s01, ptx::fadd2(sum2, f2(-96.f, -96.f)), ptx::fmul2(f2(64.f, 64.f), mu));
      const float2 nr = ptx::ffma2(sum2, f2(-510.f, -510.f), f2(-kMagicF, -kMagicF));
      const uint32_t e0 = (acc0[2 * hh] << 2) + acc1[2 * hh], e1 = (acc0[2 * hh + 1] << 2) + acc1[2 * hh + 1];
      const float2 e = ptx::fadd2(asf2(e0, e1), nr);  // exact centered integer (beta0, beta1)
      const float2 s2 = ptx::ffma2(QA, ptx::fmul2(s01, e), ptx::ffma2(QX, mu, ptx::fmul2(QM, yk)));
      float s = s2.x + s2.y;
      if (t >= nk) s = -INFINITY;  // beyond the cache (tail page)
      sc[mt][hh] = s;
      mx = fmaxf(mx, s);
      if (t < nk) mn = fminf(mn, s);
    }
  }
}

__global__ void __launch_bounds__(kThreads, 3) decode_pair_kernel(const __half* __restrict__ q_new,
                                                                 const int32_t* __restrict__ slots, CacheView cv,
                                                                 KernelCfg kc, float* __restrict__ part, int nsplit,
                                                                 uint8_t* __restrict__ dbg_pcodes,
                                                                 int64_t dbg_stride) {
  constexpr int qkm = 3;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  PairSmem& sm = *reinterpret_cast<PairSmem*>(smem_raw);
  const int b = blockIdx.x, hk = blockIdx.y, split = blockIdx.z;
  const int G = kc.G;
  const int slot = slots[b];
  const int len = cv.seq_lens[slot];
  const int pos = len - 1;
  const int npages = (len + PI - 1) / PI;
  const int nfull = len / PI;
  int pps = (npages + nsplit - 1) / nsplit;
  pps = (pps + 1) & ~1;  // even: committed pages pair up inside a split
  const int p_beg = min(split * pps, npages), p_end = min(p_beg + pps, npages);
  const int np = p_end - p_beg;
  const int nc = max(0, min(p_end, nfull) - p_beg);  // committed pages of this split
  const bool has_tail = np > 0 && p_end > nfull;    // this split holds the partial last page
  const int nitems = (nc + 1) / 2 + (has_tail ? 1 : 0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tig = lane & 3;
  const PageLayout PL = kc.pl;
  const uint32_t rng_id = cv.rng_ids[slot];

  if (tid == 0) {
    for (int s = 0; s < NSTG; ++s) {
      ptx::mbar_init(&sm.full[s], 1);
      ptx::mbar_init(&sm.empty[s], 1);
    }
    ptx::fence_mbar_init();
  }
  // ---- (a3) quantize the query rows (8-bit SR, fp32 meta): warps 0-1, 16 lanes per row
  if (warp < 2) {
    const int row = warp * 2 + (lane >> 4), lane16 = lane & 15;
    const int rr = min(row, G - 1);
    const int hq = hk * G + rr;
    const uint4 raw = reinterpret_cast<const uint4*>(q_new + ((int64_t)b * kc.Hq + hq) * 128)[lane16];
    uint64_t packed;
    float m, s;
    int sum;
    quant_row16<8, false>(raw, lane16, PI, pos, kc.seed, rng_id,
                          stream_c3(kc.layer, kTagQ, kc.head_base * G + hq), kc.q_round, packed, m, s, sum);
    *reinterpret_cast<uint2*>(&sm.qcode[row][lane16 * 8]) =
        row < G ? make_uint2((uint32_t)packed, (uint32_t)(packed >> 32)) : make_uint2(0u, 0u);
    const int beta = lane16 >> 3;
    const float cscale = 1.4426950408889634f / sqrtf(128.f);
    // all lanes of a partition hold (m, s, sum): one writes each field
    float* qcf = reinterpret_cast<float*>(&sm.qc[row][0]);
    const bool ok = row < G;
    if ((lane16 & 7) == 0) {
      qcf[beta] = ok ? cscale * s * 0.25f : 0.f;                                  // QA
      qcf[2 + beta] = ok ? cscale * s * ((float)sum - 127.5f * PI) : 0.f;        // QX
      qcf[4 + beta] = ok ? cscale * (m + 127.5f * s) : 0.f;                      // QM
      qcf[6 + beta] = __int_as_float(ok ? -(2 * qkm * sum - PI * 255 * qkm) : 0);  // RC (int bits)
    }
  }
  __syncthreads();

  float m_run = -INFINITY, l_run = 0.f;
  float2 o[8][2];  // [m-tile][channel g / g+8] -> (page A, page B) partial sums, row tig
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) o[mt][0] = o[mt][1] = f2(0.f, 0.f);
  if (warp == NW) {
    // ------------------------------------------------------------------ producer
    if (lane == 0) {
      const int32_t* bt = cv.block_table + (int64_t)slot * cv.max_pages_per_req;
      for (int k = 0; k < np; ++k) {
        const int s = k % NSTG;
        // sleep-wait: a spinning producer lane steals issue slots from the compute warps
        while (!ptx::mbar_try_wait_sleep(&sm.empty[s], ((k / NSTG) & 1) ^ 1)) {
        }
        ptx::mbar_arrive_expect_tx(&sm.full[s], PB);
        const uint8_t* pg = cv.pages + ((int64_t)bt[p_beg + k] * cv.num_kv_heads + hk) * cv.page_bytes;
        ptx::bulk_g2s(sm.stage[s], pg, PB, &sm.full[s]);
      }
    }
  } else {
    // ------------------------------------------------------------------ compute warp
    // B fragments of Q' for column n = g = (row g>>1, block g&1); k-step ks covers channels
    // 32 tig' + 16 h + 4 i + q(ks), q = {0, 2, 1, 3}; the channel's block is tig' >> 1.
    uint32_t qb[4][2];
    {
      const int r = g >> 1;
      const bool live = r < G && (tig >> 1) == (g & 1);
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const int q = ks == 0 ? 0 : (ks == 1 ? 2 : (ks == 2 ? 1 : 3));
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t v = 0;
#pragma unroll
          for (int i = 0; i < 4; ++i) v |= (uint32_t)sm.qcode[r][32 * tig + 16 * h + 4 * i + q] << (8 * i);
          qb[ks][h] = live ? v : 0u;
        }
      }
    }
    const float4 qc0 = sm.qc[tig][0], qc1 = sm.qc[tig][1];
    const float2 QA = f2(qc0.x, qc0.y), QX = f2(qc0.z, qc0.w), QM = f2(qc1.x, qc1.y);
    const uint32_t rc0 = kMagic + __float_as_uint(qc1.z), rc1 = kMagic + __float_as_uint(qc1.w);


#pragma unroll 1
    for (int it = warp; it < nitems; it += NW) {
      const bool tail_item = has_tail && it == nitems - 1;
      const int kA = tail_item ? np - 1 : 2 * it;                  // split-relative page index
      const bool hasB = !tail_item && 2 * it + 1 < nc;
      const int kB = hasB ? kA + 1 : kA;
      const int sA = kA % NSTG, sB = kB % NSTG;
      ptx::mbar_wait(&sm.full[sA], (kA / NSTG) & 1);
      if (hasB) ptx::mbar_wait(&sm.full[sB], (kB / NSTG) & 1);
      uint8_t* pgA = sm.stage[sA];
      uint8_t* pgB = sm.stage[sB];
      const int jpA = p_beg + kA;
      const int nkA = tail_item ? len - jpA * PI : PI;

      // ---- (a4) homomorphic S^T for page A (and B)
      float sa[4][2], sbv[4][2];
      float mxA, mnA, mxB = -INFINITY, mnB = INFINITY;
      qk_page(pgA, PL, g, tig, nkA, qb, QA, QX, QM, rc0, rc1, sa, mxA, mnA);
      if (hasB) {
        qk_page(pgB, PL, g, tig, PI, qb, QA, QX, QM, rc0, rc1, sbv, mxB, mnB);
      } else {
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) sbv[mt][0] = sbv[mt][1] = -INFINITY;
      }
      __syncwarp();  // K codes/meta of the pair are dead from here on

      // ---- V coefficients of the pair (cached sums, SE): channel c -> (A, B) pairs
      float4* vc_lo = reinterpret_cast<float4*>(pgA + PL.k_codes);  // channels 0..63
      if (!tail_item) {
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const int c = lane + 32 * x;
          const __half2 mA = reinterpret_cast<const __half2*>(pgA + PL.v_meta)[c];
          const __half2 mB = reinterpret_cast<const __half2*>(pgB + PL.v_meta)[c];
          const float2 mv = f2(__low2float(mA), __low2float(mB));
          float2 sv = f2(__high2float(mA), __high2float(mB));
          float2 sum = f2((float)pgA[PL.v_sums + c], (float)pgB[PL.v_sums + c]);
          if (!hasB) {
            sv.y = 0.f;
            sum.y = 0.f;
          }
          const float2 mu = ptx::ffma2(sv, f2(1.5f, 1.5f), hasB ? mv : f2(mv.x, 0.f));
          const float2 yv = ptx::ffma2(sv, ptx::fadd2(sum, f2(-96.f, -96.f)), ptx::fmul2(f2(64.f, 64.f), mu));
          const float2 nr = ptx::ffma2(sum, f2(-510.f, -510.f), f2(-kMagicF, -kMagicF));
          float4* dst = x < 2 ? vc_lo + 2 * c : &sm.vc_hi[warp][c - 64][0];
          dst[0] = make_float4(sv.x, sv.y, mu.x, mu.y);
          dst[1] = make_float4(yv.x, yv.y, nr.x, nr.y);
        }
      }

      // ---- (a5) online softmax over the pair
      float mx = fmaxf(mxA, mxB);
#pragma unroll
      for (int o2 = 4; o2 < 32; o2 <<= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o2));
        mnA = fminf(mnA, __shfl_xor_sync(0xffffffffu, mnA, o2));
        mxA = fmaxf(mxA, __shfl_xor_sync(0xffffffffu, mxA, o2));
        mnB = fminf(mnB, __shfl_xor_sync(0xffffffffu, mnB, o2));
        mxB = fmaxf(mxB, __shfl_xor_sync(0xffffffffu, mxB, o2));
      }
      const float mnew = fmaxf(m_run, mx);
      const float al = m_run == -INFINITY ? 0.f : ex2(m_run - mnew);
      float ls = 0.f;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          sa[mt][hh] = ex2(sa[mt][hh] - mnew);  // p~; ex2(-inf) = 0
          sbv[mt][hh] = ex2(sbv[mt][hh] - mnew);
          ls += sa[mt][hh] + sbv[mt][hh];
        }
#pragma unroll
      for (int o2 = 4; o2 < 32; o2 <<= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o2);
      l_run = l_run * al + ls;
      m_run = mnew;
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        o[mt][0] = ptx::fmul2(o[mt][0], f2(al, al));
        o[mt][1] = ptx::fmul2(o[mt][1], f2(al, al));
      }

      if (!tail_item) {
        // ---- (a6) P' per (row, page): RN 8-bit against fp32 (lo, s) of the unnormalized p~
        uint8_t* pcode = pgA + PL.k_meta;  // [row 4][page 2][64] in B-fragment order
        float2 AP, XP, MP;
        uint32_t rcA, rcB;
        {
          const float loA = ex2(mnA - mnew), hiA = ex2(mxA - mnew);
          QMeta pA = meta_fp32(loA, hiA, 255);
          if (!(pA.s > 1e-30f)) { pA.s = 0.f; pA.inv = 0.f; }
          QMeta pB = {0.f, 0.f, 0.f};
          if (hasB) {
            pB = meta_fp32(ex2(mnB - mnew), ex2(mxB - mnew), 255);
            if (!(pB.s > 1e-30f)) { pB.s = 0.f; pB.inv = 0.f; }
          }
          const float2 inv = f2(pA.inv, pB.inv), nlo = f2(-pA.m * pA.inv, -pB.m * pB.inv);
          uint32_t spA = 0, spB = 0;
          const int base = 4 * (g & 3) + (g >> 2);
#pragma unroll
          for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const float2 y = ptx::fadd2(ptx::ffma2(f2(sa[mt][hh], sbv[mt][hh]), inv, nlo), f2(kMagicF, kMagicF));
              const uint32_t cA = __float_as_uint(y.x) & 0xFFu, cB = __float_as_uint(y.y) & 0xFFu;
              spA += cA;
              spB += cB;
              const int p = 16 * mt + base + 2 * hh;  // token 16mt + g + 8hh -> 16T + 4q + i
              pcode[(tig * 2 + 0) * 64 + p] = (uint8_t)cA;
              pcode[(tig * 2 + 1) * 64 + p] = (uint8_t)cB;
              if (dbg_pcodes != nullptr && tig < G) {
                const int t = 16 * mt + g + 8 * hh;
                uint8_t* dr = dbg_pcodes + ((int64_t)b * kc.Hq + hk * G + tig) * dbg_stride;
                dr[jpA * PI + t] = (uint8_t)cA;
                if (hasB) dr[(jpA + 1) * PI + t] = (uint8_t)cB;
              }
            }
#pragma unroll
          for (int o2 = 4; o2 < 32; o2 <<= 1) {
            spA += __shfl_xor_sync(0xffffffffu, spA, o2);
            spB += __shfl_xor_sync(0xffffffffu, spB, o2);
          }
          AP = f2(pA.s * 0.25f, pB.s * 0.25f);
          XP = f2(pA.s * ((float)spA - 127.5f * PI), pB.s * ((float)spB - 127.5f * PI));
          MP = f2(pA.m + 127.5f * pA.s, pB.m + 127.5f * pB.s);
          rcA = kMagic + (uint32_t)(-(2 * qkm * (int)spA - PI * 255 * qkm));
          rcB = kMagic + (uint32_t)(-(2 * qkm * (int)spB - PI * 255 * qkm));
        }
        __syncwarp();  // P' codes and V coefficients visible to the warp
        // B fragments of P'^T: column n = g = (row g>>1, page g&1); page P's k-steps 2P+u
        // hold tokens 16 tig + 4 i + q(u, h), q(0,0)=0, q(0,1)=2, q(1,0)=1, q(1,1)=3.
        uint32_t pb[4][2];
        {
          const uint4 R = *reinterpret_cast<const uint4*>(pcode + ((g >> 1) * 2 + (g & 1)) * 64 + 16 * tig);
          const bool onA = (g & 1) == 0, onB = (g & 1) == 1 && hasB;
          pb[0][0] = onA ? R.x : 0u; pb[0][1] = onA ? R.z : 0u;
          pb[1][0] = onA ? R.y : 0u; pb[1][1] = onA ? R.w : 0u;
          pb[2][0] = onB ? R.x : 0u; pb[2][1] = onB ? R.z : 0u;
          pb[3][0] = onB ? R.y : 0u; pb[3][1] = onB ? R.w : 0u;
        }
        // ---- (a7) O^T += V' P'^T over the pair; Eq. 4 (centered) with cached V sums
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          const int c0 = 16 * mt + g, c1 = c0 + 8;
          const Planes vaA = planes2(*reinterpret_cast<const uint32_t*>(pgA + PL.v_codes + c0 * 16 + 4 * tig));
          const Planes vbA = planes2(*reinterpret_cast<const uint32_t*>(pgA + PL.v_codes + c1 * 16 + 4 * tig));
          const Planes vaB = planes2(*reinterpret_cast<const uint32_t*>(pgB + PL.v_codes + c0 * 16 + 4 * tig));
          const Planes vbB = planes2(*reinterpret_cast<const uint32_t*>(pgB + PL.v_codes + c1 * 16 + 4 * tig));
          uint32_t acc0[4], acc1[4];
          mma16832c(acc0, vaA.p0, vbA.p0, vaA.p2, vbA.p2, pb[0][0], pb[0][1], 0u, 0u);
          mma16832c(acc1, vaA.p1, vbA.p1, vaA.p3, vbA.p3, pb[1][0], pb[1][1], rcA, rcB);
          mma16832(acc0, vaB.p0, vbB.p0, vaB.p2, vbB.p2, pb[2][0], pb[2][1]);
          mma16832(acc1, vaB.p1, vbB.p1, vaB.p3, vbB.p3, pb[3][0], pb[3][1]);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int c = hh ? c1 : c0;
            const float4* vsrc = c < 64 ? vc_lo + 2 * c : &sm.vc_hi[warp][c - 64][0];
            const float4 v0 = vsrc[0], v1 = vsrc[1];
            const uint32_t e0 = (acc0[2 * hh] << 2) + acc1[2 * hh], e1 = (acc0[2 * hh + 1] << 2) + acc1[2 * hh + 1];
            const float2 e = ptx::fadd2(asf2(e0, e1), f2(v1.z, v1.w));
            const float2 t2 = ptx::ffma2(AP, ptx::fmul2(f2(v0.x, v0.y), e),
                                         ptx::ffma2(XP, f2(v0.z, v0.w), ptx::fmul2(MP, f2(v1.x, v1.y))));
            o[mt][hh] = ptx::fadd2(o[mt][hh], t2);
          }
        }
      } else {
        // ---- FP16 last V block (RQE): O^T += V_tail^T p~ in fp32
        float* ptl = reinterpret_cast<float*>(pgA + PL.k_codes);  // [row 4][64]
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) ptl[tig * 64 + 16 * mt + g + 8 * hh] = sa[mt][hh];
        __syncwarp();
        const __half* tail = reinterpret_cast<const __half*>(cv.v_tail) + ((int64_t)slot * kc.Hkv + hk) * PI * 128;
        for (int t = 0; t < nkA; ++t) {
          const float p = ptl[tig * 64 + t];
#pragma unroll
          for (int mt = 0; mt < 8; ++mt)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const float v = __half2float(tail[t * 128 + 16 * mt + g + 8 * hh]);
              o[mt][hh].x = fmaf(p, v, o[mt][hh].x);
            }
        }
      }
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive(&sm.empty[sA]);
        if (hasB) ptx::mbar_arrive(&sm.empty[sB]);
      }
    }
  }
  __syncthreads();  // all pages consumed: the stage ring is reused for the merge
  if (warp < NW) {
    // -- publish this warp's partial (m, l, O) for the CTA merge (row tig)
    if (g == 0) {
      sm.mrg_m[warp][tig] = m_run;
      sm.mrg_l[warp][tig] = l_run;
    }
#pragma unroll
    for (int mt = 0; mt < 8; ++mt)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) sm.mrg_o[warp][tig][16 * mt + g + 8 * hh] = o[mt][hh].x + o[mt][hh].y;
  }
  __syncthreads();
  // ---- merge the NW warps; write this split's partial: part[b][hk][split][G][2 + 128]
  if (tid < 128) {
    const int c = tid;
    for (int n = 0; n < G; ++n) {
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < NW; ++w) M = fmaxf(M, sm.mrg_m[w][n]);
      float L = 0.f, O = 0.f;
      if (M != -INFINITY) {
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const float f = ex2(sm.mrg_m[w][n] - M);
          L += f * sm.mrg_l[w][n];
          O += f * sm.mrg_o[w][n][c];
        }
      }
      float* dst = part + ((((int64_t)b * kc.Hkv + hk) * nsplit + split) * G + n) * 130;
      if (c == 0) {
        dst[0] = M;
        dst[1] = L;
      }
      dst[2 + c] = O;
    }
  }
}

}  // namespace

cudaError_t launch_decode_combine(const float* part, int nsplit, const KernelCfg& kc, int batch, void* out,
                                  cudaStream_t st);

bool decode_pair_supported(const KernelCfg& kc) {
  return kc.Pi == 64 && kc.d == 128 && kc.bits == 2 && kc.G <= 4 && kc.pl.page_bytes == PB;
}

int decode_pair_nsplit(const KernelCfg& kc, int batch, int max_seqlen) {
  const int max_pages = (max_seqlen + PI - 1) / PI;
  const int units = batch * kc.Hkv;
  int ns = (148 * 3 * 4 + units - 1) / units;
  if (const char* e = getenv("HACK_DECODE_NSPLIT")) ns = atoi(e);
  ns = max(1, min(ns, (max_pages + 15) / 16));
  return min(ns, 64);
}

size_t decode_pair_workspace(const KernelCfg& kc, int batch, int max_seqlen) {
  return (size_t)batch * kc.Hkv * decode_pair_nsplit(kc, batch, max_seqlen) * kc.G * 130 * sizeof(float);
}

cudaError_t launch_decode_pair(const KernelCfg& kc, const void* q_new, const int32_t* slots, int batch,
                               int max_seqlen, const CacheView& cv, void* out, void* workspace,
                               const hack_debug_t* dbg, cudaStream_t st) {
  const int ns = decode_pair_nsplit(kc, batch, max_seqlen);
  float* part = reinterpret_cast<float*>(workspace);
  const size_t smem = sizeof(PairSmem);
  cudaError_t e = cudaFuncSetAttribute(decode_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  decode_pair_kernel<<<dim3(batch, kc.Hkv, ns), kThreads, smem, st>>>(
      reinterpret_cast<const __half*>(q_new), slots, cv, kc, part, ns, dbg ? dbg->pcodes : nullptr,
      dbg ? dbg->pcodes_stride : 0);
  note_launch();
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_decode_combine(part, ns, kc, batch, out, st);
}

}  // namespace hack
