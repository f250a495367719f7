// decode_pair.cu -- HBM-bound homomorphic decode attention (a9) for GQA groups G <= 4,
// b = 2, Pi = 64 (the C3 Llama-3.1-8B / Mistral-7B shapes).
//
// Same arithmetic as decode_mma.cu (Eq. 4 per block, in centered form; cached
// K/V code sums = summation elimination; P 8-bit RN per (row, V block), P:537;
// FP16 last V block, RQE), re-tiled for G <= 4:
//   * S^T = K' Q'^T with tokens as M and N = 8 columns = (query row, d-block beta): both
//     d-blocks come out of ONE accumulator chain (B is zero outside the column's block),
//     so a lane holds (beta0, beta1) of one query row -> Eq. 4 on fp32x2 pairs and no
//     padding lanes.
//   * O^T = V' P'^T over a PAIR of pages with N = (query row, page): K = 128 tokens, B is
//     zero outside the column's page, so the PV epilogue also runs on fp32x2 pairs.
//   * each lane unpacks the codes of its OWN 32-bit words: plane q of a 2-bit word is
//     (w >> 4*(q>>1)) & (3 << 2*(q&1)), i.e. planes 1 and 3 come out multiplied by 4.
//     k-steps fed by scaled planes go to a second accumulator; 4*acc0 + acc1 = 4*D is
//     exactly the integer the centered Eq. 4 needs (one LEA).  The scaled accumulator
//     starts at 1.5*2^23 + (row constant) in integer form, so its float view is
//     1.5*2^23 + 4D + RC and one FADD2 with a per-token constant gives the centered
//     integer e exactly.
//   * Eq. 4 coefficients of a page (per token for K, per channel for V) are computed once
//     per page from the fp16 meta and cached sums and staged in shared memory.
//   * persistent, stream-K style work split: the flattened sequence of all pages of all
//     (request, KV head) units is cut into equal page ranges, one per CTA (4 CTAs/SM);
//     a CTA walks the unit segments of its range, a producer warp streams the
//     pages in order (cp.async.bulk into a 9-slot ring), the 3 compute warps take page
//     pairs round-robin and flush one (m, l, O) partial per (segment, warp) to global
//     memory.  Partial slot of (unit u, CTA c) = u + c (injective: units and CTA ranges
//     are both monotone along the flattened order).  The CTA completing a unit merges its
//     partials (merge_units), no second kernel.
#include <cstdlib>
#include <type_traits>

#include "append.cuh"
#include "common.cuh"
#include "internal.h"
#include "tc_ptx.cuh"

namespace hack {

namespace {

constexpr int PI = 64;
#ifndef HACK_DEC_NW
#define HACK_DEC_NW 3
#endif
#ifndef HACK_DEC_NSTG
#define HACK_DEC_NSTG 9
#endif
#ifndef HACK_DEC_SPLIT
#define HACK_DEC_SPLIT 0
#endif
#ifndef HACK_DEC_PF
#define HACK_DEC_PF 0  // L2 prefetch distance in pages (measured: 0 best, 8 -> -1.6 %)
#endif
#ifndef HACK_DEC_CTAS
#define HACK_DEC_CTAS 4
#endif
#ifndef HACK_DEC_PIPES
#define HACK_DEC_PIPES 1
#endif
// decode_pair_kernel runs PIPES independent page pipelines (producer warp + NW compute
// warps + ring + stream-K range each).  PIPES = 1: one per CTA, HACK_DEC_CTAS CTAs per SM.
// PIPES = 4: one CTA per SM whose 4 producer warps form warpgroup 0, so setmaxnreg moves
// their unused registers to the compute warps.
constexpr int PIPES = HACK_DEC_PIPES;
constexpr int NW = HACK_DEC_NW;        // compute warps per pipeline
constexpr int NSTG = HACK_DEC_NSTG;    // page slots per pipeline
constexpr int kThreads = PIPES * (NW + 1) * 32;
constexpr int kThreads8 = (NW + 1) * 32;  // decode_g8_kernel: one pipeline per CTA
constexpr int kCtasPerSm = PIPES == 1 ? HACK_DEC_CTAS : 1;
static_assert(PIPES == 1 || (PIPES == 4 && NW * PIPES % 4 == 0), "warpgroup roles");
#ifndef HACK_DEC_REGPROD
#define HACK_DEC_REGPROD 72
#endif
// even split of the register file: what the launch allocates per thread (the launch-bound cap,
// a multiple of 8), also the share for the merge after the attention loop.  setmaxnreg only
// moves registers within this pool (an .inc beyond it never completes).
constexpr int kRegEven = 65536 / kThreads / 8 * 8 < 128 ? 65536 / kThreads / 8 * 8 : 128;
constexpr int kRegProd = HACK_DEC_REGPROD,
              kRegComp = PIPES == 1 ? 128 : (kRegEven * kThreads - 128 * kRegProd) / (32 * NW * PIPES) / 8 * 8;
static_assert(PIPES == 1 || kRegComp * 32 * NW * PIPES + 128 * kRegProd <= kRegEven * kThreads, "register pool");
constexpr int PB = 5376;    // page bytes at d = 128, Pi = 64, b = 2
constexpr int kPart = 130;  // floats per partial row: m, l, O[128]
constexpr uint32_t kMagic = 0x4B400000u;   // bits of 1.5 * 2^23
constexpr float kMagicF = 12582912.f;      // 1.5 * 2^23
constexpr int kMetaInts = 16;              // workspace header: R, P, grid, ...

struct alignas(128) PairSmem {
  uint8_t stage[NSTG][PB];
  struct Warp {
    float4 scr[64][2];      // K coefficients of the page in QK; V coefficients of channels 64..127 in PV
    uint8_t qcode[4][128];  // Q' rows of the current unit, natural channel order
    float4 qc[4][2];        // per row: (QA0, QA1, QX0, QX1), (QM0, QM1, RC0, RC1)
  } w[NW];
  int range_b0, range_base;  // request holding the CTA's first page, flattened offset of its first unit
  int R, P;
  uint64_t full[NSTG], fullv[NSTG], empty[NSTG];  // fullv: the V half of a split page copy
  int tag[NSTG];  // page index of the slot's latest issued fill (see wait_fill)
  int mflag;      // merge_units: this CTA completes the unit
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

// The request's length this step: seq_lens, + 1 in the fused decode step (its append runs in
// the kernel and seq_lens is bumped only when every CTA is done reading it), unless the
// capacity guard of the append (append_kernel) skips the request.
HACK_DEV int len_of(const CacheView& cv, int slot, int add) {
  const int t = cv.seq_lens[slot];
  return t + (add && t / PI < cv.max_pages_per_req ? 1 : 0);
}
HACK_DEV int npages_of(const CacheView& cv, const int32_t* slots, int b, int add) {
  return (len_of(cv, slots[b], add) + PI - 1) / PI;
}

// One unit segment of a CTA's page range.
struct Seg {
  int b, hk, p0, p1;  // request, KV head, page range [p0, p1) of the unit
  int uoff, npg;      // flattened offset of the unit's first page, its page count
};

// Walks the unit segments of the flattened page range [pos, end).
struct SegWalker {
  int b, base, pos, end;  // current request, flattened offset of its first unit, cursor, range end
  // add: fused append, lengths + 1 (len_of); from the kernel parameter at each call (no register
  // held across the attention loop)
  HACK_DEV bool next(const CacheView& cv, const int32_t* slots, int Hkv, Seg& s, int add) {
    if (pos >= end) return false;
    int npg = npages_of(cv, slots, b, add);
    while (pos >= base + npg * Hkv) {  // (only when the cursor sits exactly on a request boundary)
      base += npg * Hkv;
      ++b;
      npg = npages_of(cv, slots, b, add);
    }
    const int rel = pos - base;
    s.b = b;
    s.hk = rel / npg;
    s.p0 = rel - s.hk * npg;
    s.p1 = min(npg, s.p0 + (end - pos));
    s.uoff = base + s.hk * npg;
    s.npg = npg;
    pos += s.p1 - s.p0;
    return true;
  }
};

// Per-page K-side Eq. 4 coefficients (beta0, beta1 pairs) from fp16 meta + cached sums (SE):
// kcs[2t] = (s_k, mu_k), kcs[2t+1] = (y_k, -1.5*2^23 - 510 SK).  Two tokens per lane.
// Sum of the 16 2-bit codes of a word: popc(w & 0x55..) + 2 popc(w & 0xAA..).
HACK_DEV uint32_t codesum2(uint32_t w) { return __popc(w & 0x55555555u) + 2u * __popc(w & 0xAAAAAAAAu); }

// SE = false is the "HACK/SE" ablation: the code sums are
// recomputed from the codes on every decode step instead of read from the summation cache.
// The result is bit-identical; only the cost differs.
template <bool SE>
HACK_DEV void stage_kc(const uint8_t* pg, const PageLayout& PL, float4* kcs, int lane) {
  uint2 mh[2];
  uint32_t sums[2];
#pragma unroll
  for (int x = 0; x < 2; ++x) {  // issue all loads first
    const int t = lane + 32 * x;
    mh[x] = *reinterpret_cast<const uint2*>(pg + PL.k_meta + t * 8);
    if (SE) {
      sums[x] = *reinterpret_cast<const uint16_t*>(pg + PL.k_sums + t * 2);
    } else {  // beta0: words 0..3 of the token row, beta1: words 4..7
      const uint4 a = *reinterpret_cast<const uint4*>(pg + PL.k_codes + t * 32);
      const uint4 b = *reinterpret_cast<const uint4*>(pg + PL.k_codes + t * 32 + 16);
      const uint32_t s0 = codesum2(a.x) + codesum2(a.y) + codesum2(a.z) + codesum2(a.w);
      const uint32_t s1 = codesum2(b.x) + codesum2(b.y) + codesum2(b.z) + codesum2(b.w);
      sums[x] = s0 | (s1 << 8);
    }
  }
#pragma unroll
  for (int x = 0; x < 2; ++x) {
    const int t = lane + 32 * x;
    const float2 m01 = __half22float2(__halves2half2(__ushort_as_half((unsigned short)(mh[x].x & 0xFFFF)),
                                                     __ushort_as_half((unsigned short)(mh[x].y & 0xFFFF))));
    const float2 s01 = __half22float2(__halves2half2(__ushort_as_half((unsigned short)(mh[x].x >> 16)),
                                                     __ushort_as_half((unsigned short)(mh[x].y >> 16))));
    // sum bytes -> exact floats: bits 2^23 + byte, minus 2^23 (folded into the constants below)
    const float2 sm23 = asf2(ptx::prmt(sums[x], 0x4B00u, 0x5440u), ptx::prmt(sums[x], 0x4B00u, 0x5441u));
    const float2 sum2 = ptx::fadd2(sm23, f2(-8388608.f, -8388608.f));
    const float2 mu = ptx::ffma2(s01, f2(1.5f, 1.5f), m01);
    const float2 yk = ptx::ffma2(s01, ptx::fadd2(sum2, f2(-96.f, -96.f)), ptx::fmul2(f2(64.f, 64.f), mu));
    const float2 nr = ptx::ffma2(sum2, f2(-510.f, -510.f), f2(-kMagicF, -kMagicF));
    kcs[2 * t] = make_float4(s01.x, s01.y, mu.x, mu.y);
    kcs[2 * t + 1] = make_float4(yk.x, yk.y, nr.x, nr.y);
  }
}

// HACK_DEC_KDIRECT=1: each lane computes the K coefficients of its own 8 tokens from the page
// (same operations as stage_kc, 4 lanes per token) instead of one staging pass + __syncwarp +
// shared-memory loads per page (SE only).
// HACK_DEC_OSUM=1 (default): one O accumulator per (channel, row), pages A and B summed every
// pair (16 registers fewer, one FADD more per output per pair; C3 +0.3-0.4 %, two A/B runs);
// 0: separate (page A, page B) partials summed at the end
// HACK_DEC_LSUM=1 (default): the row max of a pair from the two pages' reduced maxima (no
// third reduction), and the row sum l kept per lane until the segment's flush (no per-pair
// reduction): 6 shuffles and 6 FP ops fewer per pair; C3 +0.7 % (4 A/B runs: 3096 vs
// 3068 GB/s).  (Moving the p~ arguments and row sums onto FADD2 pairs and the P-code sums
// onto the raw magic-number bits on top of it measured -0.4 %, not kept.)
#ifndef HACK_DEC_LSUM
#define HACK_DEC_LSUM 1
#endif
// HACK_G8_QSMEM=1: decode_g8 keeps the Q' fragments in shared memory and reloads them per
// MMA group (16 registers fewer in the page loop; spills 92 -> 56 bytes, C4 2-bit +1.0 %)
#ifndef HACK_G8_QSMEM
#define HACK_G8_QSMEM 1
#endif
#ifndef HACK_DEC_OSUM
#define HACK_DEC_OSUM 1
#endif
#ifndef HACK_DEC_KDIRECT
#define HACK_DEC_KDIRECT 0
#endif
HACK_DEV void kcoef(const uint8_t* pg, const PageLayout& PL, int t, float4& c0, float4& c1) {
  const uint2 mh = *reinterpret_cast<const uint2*>(pg + PL.k_meta + t * 8);
  const uint32_t sums = *reinterpret_cast<const uint16_t*>(pg + PL.k_sums + t * 2);
  const float2 m01 = __half22float2(__halves2half2(__ushort_as_half((unsigned short)(mh.x & 0xFFFF)),
                                                   __ushort_as_half((unsigned short)(mh.y & 0xFFFF))));
  const float2 s01 = __half22float2(__halves2half2(__ushort_as_half((unsigned short)(mh.x >> 16)),
                                                   __ushort_as_half((unsigned short)(mh.y >> 16))));
  const float2 sm23 = asf2(ptx::prmt(sums, 0x4B00u, 0x5440u), ptx::prmt(sums, 0x4B00u, 0x5441u));
  const float2 sum2 = ptx::fadd2(sm23, f2(-8388608.f, -8388608.f));
  const float2 mu = ptx::ffma2(s01, f2(1.5f, 1.5f), m01);
  const float2 yk = ptx::ffma2(s01, ptx::fadd2(sum2, f2(-96.f, -96.f)), ptx::fmul2(f2(64.f, 64.f), mu));
  const float2 nr = ptx::ffma2(sum2, f2(-510.f, -510.f), f2(-kMagicF, -kMagicF));
  c0 = make_float4(s01.x, s01.y, mu.x, mu.y);
  c1 = make_float4(yk.x, yk.y, nr.x, nr.y);
}

// Homomorphic S^T for one 64-token page: sc[mt][hh] = log2(e)/sqrt(d) * S(token 16mt+g+8hh, row tig).
// MASK: tokens >= nk (the partial last page) are -inf.  Also the per-lane max/min.
// dq (debug runs only, else nullptr): this lane's query row's qk_acc at the page's first token;
// receives the raw block accumulators 4 D_beta + RC (HACK_ACC_CENTERED4), beta 1 at + dstride.
template <bool MASK, bool KD = false>
HACK_DEV void qk_page(const uint8_t* pg, const PageLayout& PL, const float4* kcs, int g, int tig, int nk,
                      const uint32_t (&qb)[4][2], float2 QA, float2 QX, float2 QM, uint32_t rc0, uint32_t rc1,
                      float (&sc)[4][2], float& mx, float& mn, int32_t* dq = nullptr, int64_t dstride = 0) {
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
      float4 c0, c1;
      if (KD) {
        kcoef(pg, PL, t, c0, c1);
      } else {
        c0 = kcs[2 * t];
        c1 = kcs[2 * t + 1];
      }
      const uint32_t e0 = (acc0[2 * hh] << 2) + acc1[2 * hh], e1 = (acc0[2 * hh + 1] << 2) + acc1[2 * hh + 1];
      if (dq != nullptr && t < nk) {
        dq[t] = (int32_t)(e0 - kMagic);
        dq[dstride + t] = (int32_t)(e1 - kMagic);
      }
      const float2 e = ptx::fadd2(asf2(e0, e1), f2(c1.z, c1.w));  // exact centered integer (beta0, beta1)
      const float2 s2 = ptx::ffma2(QA, ptx::fmul2(f2(c0.x, c0.y), e),
                                   ptx::ffma2(QX, f2(c0.z, c0.w), ptx::fmul2(QM, f2(c1.x, c1.y))));
      float s = s2.x + s2.y;
      if (MASK && t >= nk) s = -INFINITY;  // beyond the cache (partial last page)
      sc[mt][hh] = s;
      mx = fmaxf(mx, s);
      if (!MASK || t < nk) mn = fminf(mn, s);
    }
  }
}

// This CTA's page range of the flattened (request, KV head, page) sequence: P = total
// pages, R = ceil(P / grid); the request holding the first page and its flattened offset.
// CTA 0 also publishes the per-request offsets and page counts for the merge kernel.
template <class SMT>
HACK_DEV void locate_range(SMT& sm, const CacheView& cv, const int32_t* __restrict__ slots, int batch, int Hkv,
                           int* __restrict__ ws_meta, bool leader, int lane, int add, int c, int nvirt) {
  if (leader) {
    int P = 0;
    for (int b0 = 0; b0 < batch; b0 += 32) {
      const int b = b0 + lane;
      const int n = b < batch ? npages_of(cv, slots, b, add) * Hkv : 0;
      int v = n;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {  // inclusive scan
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      if (c == 0 && b < batch) {
        ws_meta[kMetaInts + b] = P + v - n;            // flattened offset of request b
        ws_meta[kMetaInts + batch + b] = n / Hkv;      // its pages (per unit)
      }
      P += __shfl_sync(0xffffffffu, v, 31);
    }
    const int R = max(1, (P + nvirt - 1) / nvirt);
    const int start = c * R;
    // request holding page `start`
    int base = 0, bsel = batch, basesel = P;
    for (int b0 = 0; b0 < batch && bsel == batch; b0 += 32) {
      const int b = b0 + lane;
      const int n = b < batch ? npages_of(cv, slots, b, add) * Hkv : 0;
      int v = n;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      const int lo = base + v - n;  // exclusive prefix
      const unsigned hit = __ballot_sync(0xffffffffu, b < batch && start >= lo && start < lo + n);
      if (hit) {
        const int src = __ffs(hit) - 1;
        bsel = b0 + src;
        basesel = __shfl_sync(0xffffffffu, lo, src);
      }
      base += __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) {
      sm.R = R;
      sm.P = P;
      sm.range_b0 = bsel;
      sm.range_base = basesel;
      if (c == 0) {
        ws_meta[0] = R;
        ws_meta[1] = P;
        ws_meta[2] = nvirt;
      }
    }
  }
}

// Consumer wait for page k in slot k % N.  Pages are not consumed by a fixed warp per slot
// (items rotate over the warps per segment), so a warp may start waiting for fill k of a
// slot while fill k - N is still in flight; a bare phase-parity wait would then match the
// phase of fill k - 2N.  The producer tags each slot with the page index before issuing its
// fill, and fill k is only issued after fill k - N was consumed, so once the tag reads k
// the parity wait is exact.
// The slot tag is a flag, not data: relaxed (memory-model "strong") shared accesses, so
// they are neither reordered away nor counted as data races.
HACK_DEV int tag_load(const int* p) {
  int v;
  asm volatile("ld.relaxed.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(ptx::smem_u32(p)) : "memory");
  return v;
}
HACK_DEV void tag_store(int* p, int v) { atomicExch(p, v); }  // producer side, once per page

template <int N, class SMT>
HACK_DEV void wait_fill(SMT& sm, int k) {
  const int s = k % N;
  while (tag_load(&sm.tag[s]) != k) {
  }
  ptx::mbar_wait(&sm.full[s], (k / N) & 1);
}

// Fused decode step (hack_decode_attention): k_new / v_new of the step and the grid-wide
// completion counter (workspace, zero between launches).
struct StepIO {
  const __half* k_new;
  const __half* v_new;
  int* done;
};

// The append (a8) of every unit whose last page (at the new length) lies in this CTA's range,
// run by the producer warp (32 lanes) once the page ring is full or, before that, right
// before it issues such a page: the appended page (K row, and the V block of a flush) and the
// unit's FP16 tail are read by this CTA only, after that page's copy.  Generic-proxy stores,
// then a proxy fence, so the bulk copies (async proxy) see them; the compute warps see the tail
// through the page's full barrier (release by the producer's arrive, acquire by their wait).
// (Inlined: as a call, its ABI cost the attention loop registers and spills.)
HACK_DEV void producer_append(const StepIO& io, SegWalker walk, const CacheView& cv,
                                             const int32_t* __restrict__ slots, const KernelCfg& kc, int lane) {
  Seg s;
  while (walk.next(cv, slots, kc.Hkv, s, 1)) {
    if (s.p1 != s.npg) continue;  // the unit's last page is another CTA's
    const int slot = slots[s.b];
    const int t = cv.seq_lens[slot];
    if (t / PI >= cv.max_pages_per_req) continue;  // capacity guard (append_kernel)
    append_unit<2, true, 32>(io.k_new, io.v_new, s.b, slot, t, s.hk, cv, kc, lane, [] { __syncwarp(); });
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
  __threadfence_block();
  __syncwarp();
}

// Producer warp: streams the CTA's pages in order into an N-slot ring (cp.async.bulk).
template <int N, bool FUSED, class SMT>
HACK_DEV void produce_pages(SMT& sm, SegWalker walk, const CacheView& cv, const int32_t* __restrict__ slots,
                            int Hkv, const KernelCfg& kc, int lane, const StepIO& io) {
  const SegWalker walk0 = walk;
  bool appended = false;
    // ------------------------------------------------------------------ producer
  // The whole warp walks the segments; block-table entries are fetched 32 pages at a
  // time with one coalesced load, so the issuing lane never waits on a dependent global
  // load between two page copies (one such wait per page capped the issue rate).
  Seg s;
  int k = 0, kslot = 0;  // fill index, its slot k % N
  uint32_t kpar = 0;     // (k / N) & 1
  // page of block id p, KV head hk: (pages + hk * page_bytes) + p * (heads * page_bytes), the
  // product one 32 x 32 -> 64-bit multiply per page
  const uint32_t pg_stride = (uint32_t)cv.num_kv_heads * (uint32_t)cv.page_bytes;
  while (walk.next(cv, slots, Hkv, s, FUSED)) {
    const int32_t* bt = cv.block_table + (int64_t)slots[s.b] * cv.max_pages_per_req;
    const uint8_t* pg_hk = cv.pages + (int64_t)s.hk * cv.page_bytes;
    for (int p0 = s.p0; p0 < s.p1; p0 += 32) {
      const int n = min(32, s.p1 - p0);
      const int ent = lane < n ? bt[p0 + lane] : 0;
      // entries of the next 32 pages of the segment: L2 prefetch HACK_DEC_PF pages ahead
      // (the ring slots hold pages being computed on, so the pages in flight per SM are
      // few; the L2 prefetch keeps more bytes in flight without smem)
      const int ent2 = HACK_DEC_PF > 0 && lane < s.p1 - p0 - 32 ? bt[p0 + 32 + lane] : 0;
      for (int x = 0; x < n; ++x, ++k) {
        const int pid = __shfl_sync(0xffffffffu, ent, x);
        const int xf = x + HACK_DEC_PF;
        int pfa = 0, pfb = 0;
        if (HACK_DEC_PF > 0) {
          pfa = __shfl_sync(0xffffffffu, ent, xf & 31);
          pfb = __shfl_sync(0xffffffffu, ent2, xf & 31);
        }
        // fused step: the appends of the CTA's units run once the ring is full (the producer
        // would wait for a slot anyway) or before the first page that receives a new token
        if (FUSED && !appended && (k == N || (s.p1 == s.npg && p0 + x == s.p1 - 1))) {
          producer_append(io, walk0, cv, slots, kc, lane);
          appended = true;
        }
        if (lane == 0) {
          const int st = kslot;
#ifdef HACK_DEC_SPIN
          while (!ptx::mbar_try_wait(&sm.empty[st], kpar ^ 1)) {
          }
#else
          // sleep-wait: a spinning producer lane steals issue slots from the compute warps
          while (!ptx::mbar_try_wait_sleep(&sm.empty[st], kpar ^ 1)) {
          }
#endif
          tag_store(&sm.tag[st], k);  // fill k of slot st is being issued
#if HACK_DEC_SPLIT
          // two copies: the K half (codes + meta + sums) lands first and QK can start
          const uint32_t kb = (uint32_t)kc.pl.v_codes;
          ptx::mbar_arrive_expect_tx(&sm.full[st], kb);
#else
          ptx::mbar_arrive_expect_tx(&sm.full[st], PB);
#endif
          const uint8_t* pg = pg_hk + (uint64_t)(uint32_t)pid * pg_stride;
#if HACK_DEC_SPLIT
          ptx::bulk_g2s(sm.stage[st], pg, kb, &sm.full[st]);
          ptx::mbar_arrive_expect_tx(&sm.fullv[st], PB - kb);
          ptx::bulk_g2s(sm.stage[st] + kb, pg + kb, PB - kb, &sm.fullv[st]);
#else
          ptx::bulk_g2s(sm.stage[st], pg, PB, &sm.full[st]);
#endif
          if (HACK_DEC_PF > 0 && p0 + xf < s.p1) {
            const int pidf = xf < 32 ? pfa : pfb;
            ptx::bulk_prefetch_l2(cv.pages + ((int64_t)pidf * cv.num_kv_heads + s.hk) * cv.page_bytes, PB);
          }
        }
        // slot and phase of the next fill, kept incrementally (no division per page)
        if (++kslot == N) {
          kslot = 0;
          kpar ^= 1u;
        }
        __syncwarp();
      }
    }
  }
}

// In-kernel merge of the split partials (flash-decoding combine, no second kernel): after its
// last segment a CTA counts itself in on every unit it contributed to (one counter per unit
// in the workspace); the CTA that completes a unit's count merges the unit's partials (NW
// warps x contributing CTAs) into the output rows and resets the counter to zero for the
// next launch.  A partial covers slot (u + c, warp): CTA c of the unit's CTA span
// [uoff / R, (uoff + npg - 1) / R].  Writers fence their partial stores before the count;
// the merging CTA fences after it and reads the partials through L2 (ld.cg).
// All warps of the CTA (compute + producer) run it.
template <int NWp, class Sync>
HACK_DEV void merge_units(SegWalker walk, int R, const CacheView& cv, const int32_t* __restrict__ slots,
                          const KernelCfg& kc, int* __restrict__ cnt, const float* __restrict__ part,
                          void* __restrict__ out, int* flag_smem, int tid, int add, Sync sync) {
  __threadfence();  // this thread's partial stores precede the CTA's count below
  sync();
  const int G = kc.G;
  Seg s;
  while (walk.next(cv, slots, kc.Hkv, s, add)) {
    const int u = s.b * kc.Hkv + s.hk;
    const int cf = s.uoff / R, cl = (s.uoff + s.npg - 1) / R;
    if (tid == 0) {
      const int n = atomicAdd(cnt + u, 1) + 1;
      const bool last = n == cl - cf + 1;
      if (last) cnt[u] = 0;  // no other CTA touches it again in this launch
      *flag_smem = last;
    }
    sync();
    const bool last = *flag_smem != 0;
    sync();  // (flag reused by the next segment)
    if (!last) continue;
    __threadfence();
    const int np = (cl - cf + 1) * NWp;
    const int64_t stride = (int64_t)G * kPart;  // partial k at base + k * stride
    const float* base = part + ((int64_t)(u + cf) * NWp) * stride;
    // warp w merges row n0 + w, lane = 4 channels: every partial load of the row in flight
    // at once (one L2 round trip per 8 partials)
    const int w = tid >> 5, lane = tid & 31;
    for (int n = w; n < G; n += NWp + 1) {
      float M = -INFINITY, L = 0.f;
      float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int k0 = 0; k0 < np; k0 += 8) {
        float ms[8], ls[8];
        float4 os[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const bool ok = k0 + k < np;
          const float* src = base + (k0 + k) * stride + n * kPart;
          ms[k] = ok ? __ldcg(src) : -INFINITY;
          ls[k] = ok ? __ldcg(src + 1) : 0.f;
          os[k] = ok ? make_float4(__ldcg(src + 2 + 4 * lane), __ldcg(src + 3 + 4 * lane), __ldcg(src + 4 + 4 * lane),
                                   __ldcg(src + 5 + 4 * lane))
                     : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        float Mn = M;
#pragma unroll
        for (int k = 0; k < 8; ++k) Mn = fmaxf(Mn, ms[k]);
        if (Mn == -INFINITY) continue;
        const float r = ex2(M - Mn);  // 0 when M = -inf
        L *= r;
        O.x *= r; O.y *= r; O.z *= r; O.w *= r;
        M = Mn;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float f = ex2(ms[k] - M);  // ex2(-inf) = 0 for empty partials
          L = fmaf(f, ls[k], L);
          O.x = fmaf(f, os[k].x, O.x);
          O.y = fmaf(f, os[k].y, O.y);
          O.z = fmaf(f, os[k].z, O.z);
          O.w = fmaf(f, os[k].w, O.w);
        }
      }
      const float il = 1.f / L;
      const int64_t idx = ((int64_t)s.b * kc.Hq + s.hk * G + n) * 128 + 4 * lane;
      if (kc.out_fp32) {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + idx) = make_float4(O.x * il, O.y * il, O.z * il, O.w * il);
      } else {
        __half2 hv[2] = {__floats2half2_rn(O.x * il, O.y * il), __floats2half2_rn(O.z * il, O.w * il)};
        *reinterpret_cast<uint2*>(reinterpret_cast<__half*>(out) + idx) = *reinterpret_cast<uint2*>(hv);
      }
    }
  }
}

// seq_lens += 1 for the step's requests, by the last CTA to finish: every CTA has read the old
// lengths (range geometry, walks, merge) before it counts itself done.
template <class Sync>
HACK_DEV void bump_lengths(const StepIO& io, const CacheView& cv, const int32_t* __restrict__ slots, int batch,
                           int* flag_smem, int tid, int nthreads, int nvirt, Sync sync) {
  sync();
  if (tid == 0) {
    __threadfence();
    *flag_smem = atomicAdd(io.done, 1) == nvirt - 1;
  }
  sync();
  if (*flag_smem == 0) return;
  __threadfence();
  for (int b = tid; b < batch; b += nthreads) {
    const int slot = slots[b];
    const int t = __ldcg(cv.seq_lens + slot);
    if (t / PI < cv.max_pages_per_req) cv.seq_lens[slot] = t + 1;  // capacity guard (append_kernel)
  }
  if (tid == 0) *io.done = 0;
}

// DBG: parity runs only (hack_debug_t): P-code and raw QK / PV accumulator dumps.
struct DecDbg {
  uint8_t* pcodes;
  int64_t pstride;
  int32_t* qk;
  int32_t* pv;
  int64_t astride;
  int head;  // hack_debug_t.acc_head
  // dump row of query head hq: index in the dumped head dimension, -1 = not dumped
  HACK_DEV int hsel(int hq) const { return head < 0 ? hq : (hq == head ? 0 : -1); }
  HACK_DEV int hdim(int Hq) const { return head < 0 ? Hq : 1; }
};

template <bool DBG, bool SE, bool FUSED>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
    decode_pair_kernel(const __half* __restrict__ q_new, const int32_t* __restrict__ slots, int batch, CacheView cv,
                       KernelCfg kc, int* __restrict__ ws_meta, int* __restrict__ cnt, float* __restrict__ part,
                       void* __restrict__ out, int merge, StepIO io, DecDbg dbg) {
  uint8_t* const dbg_pcodes = dbg.pcodes;
  const int64_t dbg_stride = dbg.pstride;
  constexpr int qkm = 3;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int G = kc.G, Hkv = kc.Hkv;
  const int tid = threadIdx.x, lane = tid & 31;
  const int g = lane >> 2, tig = lane & 3;
  // roles: PIPES = 1: warps 0..NW-1 compute, warp NW produces.  PIPES = 4: warps 0-3 are the
  // 4 pipelines' producers (warpgroup 0), then NW compute warps per pipeline.
  const int w_ = tid >> 5;
  const bool producer = PIPES == 1 ? w_ == NW : w_ < PIPES;
  const int pipe = PIPES == 1 ? 0 : (producer ? w_ : (w_ - PIPES) / NW);
  const int warp = PIPES == 1 ? w_ : (producer ? NW : (w_ - PIPES) % NW);  // compute warp of the pipeline
  const int ltid = 32 * warp + lane;  // thread of the pipeline (0 .. 32 (NW + 1) - 1)
  const int c = blockIdx.x * PIPES + pipe, nvirt = gridDim.x * PIPES;  // page range (virtual CTA)
  PairSmem& sm = reinterpret_cast<PairSmem*>(smem_raw)[pipe];
  auto psync = [pipe] { asm volatile("bar.sync %0, %1;" ::"r"(1 + pipe), "n"(32 * (NW + 1)) : "memory"); };
  const PageLayout PL = kc.pl;

  if (tid < PIPES) {
    PairSmem& sp = reinterpret_cast<PairSmem*>(smem_raw)[tid];
    for (int s = 0; s < NSTG; ++s) {
      ptx::mbar_init(&sp.full[s], 1);
      ptx::mbar_init(&sp.fullv[s], 1);
      sp.tag[s] = -1;
      ptx::mbar_init(&sp.empty[s], 1);
    }
    ptx::fence_mbar_init();
  }
#ifndef HACK_DEC_NOPDL
  // launched as a programmatic dependent of the append kernel: everything above touched
  // only shared memory; seq_lens, pages and the FP16 tail are read after this wait
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
  locate_range(sm, cv, slots, batch, Hkv, ws_meta, PIPES == 1 ? w_ == 0 : producer, lane, FUSED, c, nvirt);
  __syncthreads();
  const int R = sm.R, P = sm.P;
  SegWalker walk{sm.range_b0, sm.range_base, min(c * R, P), min(c * R + R, P)};

  // PIPES = 4: the producers' registers go to the compute warps (warpgroup-wide setmaxnreg)
  if (producer) {
    if (PIPES > 1) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegProd));
    produce_pages<NSTG, FUSED>(sm, walk, cv, slots, Hkv, kc, lane, io);
    if (PIPES > 1) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegEven));  // even split for the merge below
  } else {
  if (PIPES > 1) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegComp));

  // -------------------------------------------------------------------- compute warps
  typename PairSmem::Warp& ws = sm.w[warp];
  const float cscale = 1.4426950408889634f / sqrtf(128.f);
  Seg s;
  int it_base = 0, k_base = 0;
  while (walk.next(cv, slots, Hkv, s, FUSED)) {
    const int slot = slots[s.b];
    const int len = len_of(cv, slot, FUSED);
    const int nfull = len / PI;
    const int nc = max(0, min(s.p1, nfull) - s.p0);  // committed pages of the segment
    const bool has_tail = s.p1 > nfull;              // the segment ends with the partial last page
    const int nitems = (nc + 1) / 2 + (has_tail ? 1 : 0);
    const int my0 = ((warp - it_base) % NW + NW) % NW;  // first item of this warp in the segment
    const int u = s.b * Hkv + s.hk;
    float m_run = -INFINITY, l_run = 0.f;
#if HACK_DEC_OSUM
    float2 o[8];  // [m-tile] -> (channel g, channel g + 8), row tig (pages A + B summed every pair)
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) o[mt] = f2(0.f, 0.f);
#else
    float2 o[8][2];  // [m-tile][channel g / g+8] -> (page A, page B) partial sums, row tig
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) o[mt][0] = o[mt][1] = f2(0.f, 0.f);
#endif

    if (my0 < nitems) {
      const uint32_t rng_id = cv.rng_ids[slot];
      // ---- (a3) quantize the unit's query rows (8-bit SR, fp32 meta), 16 lanes per row
#pragma unroll 1
      for (int r2 = 0; r2 < 2; ++r2) {
        const int row = 2 * r2 + (lane >> 4), lane16 = lane & 15;
        const int hq = s.hk * G + min(row, G - 1);
        const uint4 raw = reinterpret_cast<const uint4*>(q_new + ((int64_t)s.b * kc.Hq + hq) * 128)[lane16];
        uint64_t packed;
        float m, sc;
        int sum;
        quant_row16<8, false>(raw, lane16, PI, len - 1, kc.seed, rng_id,
                              stream_c3(kc.layer, kTagQ, kc.head_base * G + hq), kc.q_round, packed, m, sc, sum);
        const bool ok = row < G;
        *reinterpret_cast<uint2*>(&ws.qcode[row][lane16 * 8]) =
            ok ? make_uint2((uint32_t)packed, (uint32_t)(packed >> 32)) : make_uint2(0u, 0u);
        const int beta = lane16 >> 3;
        float* qcf = reinterpret_cast<float*>(&ws.qc[row][0]);
        if ((lane16 & 7) == 0) {  // every lane of a partition holds (m, s, sum)
          qcf[beta] = ok ? cscale * sc * 0.25f : 0.f;                                  // QA
          qcf[2 + beta] = ok ? cscale * sc * ((float)sum - 127.5f * PI) : 0.f;        // QX
          qcf[4 + beta] = ok ? cscale * __fmaf_rn(127.5f, sc, m) : 0.f;                  // QM
          qcf[6 + beta] = __int_as_float(ok ? -(2 * qkm * sum - PI * 255 * qkm) : 0);  // RC (int bits)
        }
      }
      __syncwarp();
      // B fragments of Q' for column n = g = (row g>>1, block g&1); k-step ks covers channels
      // 32 tig + 16 h + 4 i + q(ks), q = {0, 2, 1, 3}; the channel's block is tig >> 1.
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
            for (int i = 0; i < 4; ++i) v |= (uint32_t)ws.qcode[r][32 * tig + 16 * h + 4 * i + q] << (8 * i);
            qb[ks][h] = live ? v : 0u;
          }
        }
      }
      const float4 qc0 = ws.qc[tig][0], qc1 = ws.qc[tig][1];
      const float2 QA = f2(qc0.x, qc0.y), QX = f2(qc0.z, qc0.w), QM = f2(qc1.x, qc1.y);
      const uint32_t rc0 = kMagic + __float_as_uint(qc1.z), rc1 = kMagic + __float_as_uint(qc1.w);

#pragma unroll 1
      for (int j = my0; j < nitems; j += NW) {
        const bool tail_item = has_tail && j == nitems - 1;
        const int kA = k_base + (tail_item ? s.p1 - s.p0 - 1 : 2 * j);  // CTA-relative page index
        const bool hasB = !tail_item && 2 * j + 1 < nc;
        const int kB = hasB ? kA + 1 : kA;
        const int sA = kA % NSTG, sB = kB % NSTG;
        const int jpA = s.p0 + (kA - k_base);  // page index in the unit
        const int nkA = tail_item ? len - jpA * PI : PI;
        uint8_t* pgA = sm.stage[sA];
        uint8_t* pgB = sm.stage[sB];

        // ---- (a4) homomorphic S^T for page A (and B)
        float sa[4][2], sbv[4][2];
        float mxA, mnA, mxB = -INFINITY, mnB = INFINITY;
        wait_fill<NSTG>(sm, kA);
#ifdef HACK_DEC_STREAM
        // timing experiment only (wrong outputs): the page pipeline without any compute
        if (hasB) wait_fill<NSTG>(sm, kB);
        __syncwarp();
        if (lane == 0) {
          ptx::mbar_arrive(&sm.empty[sA]);
          if (hasB) ptx::mbar_arrive(&sm.empty[sB]);
        }
        continue;
#endif
        constexpr bool KD = HACK_DEC_KDIRECT && SE;
        int32_t* dqA = nullptr;
        if (DBG && dbg.qk != nullptr && tig < G && dbg.hsel(s.hk * G + tig) >= 0)
          dqA = dbg.qk + ((int64_t)s.b * dbg.hdim(kc.Hq) + dbg.hsel(s.hk * G + tig)) * 2 * dbg.astride + jpA * PI;
        if (KD && !tail_item) {
          // both pages first, then both QKs with no barrier between them (page B = page A
          // when the pair has one page: computed, then discarded)
          if (hasB) wait_fill<NSTG>(sm, kB);
          __syncwarp();
          qk_page<false, true>(pgA, PL, &ws.scr[0][0], g, tig, PI, qb, QA, QX, QM, rc0, rc1, sa, mxA, mnA, dqA,
                               dbg.astride);
          qk_page<false, true>(pgB, PL, &ws.scr[0][0], g, tig, PI, qb, QA, QX, QM, rc0, rc1, sbv, mxB, mnB,
                               hasB && dqA != nullptr ? dqA + PI : nullptr, dbg.astride);
          if (!hasB) {
            mxB = -INFINITY;
            mnB = INFINITY;
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) sbv[mt][0] = sbv[mt][1] = -INFINITY;
          }
        } else {
        if (!KD) {
          stage_kc<SE>(pgA, PL, &ws.scr[0][0], lane);
          __syncwarp();
        }
        if (tail_item)
          qk_page<true, KD>(pgA, PL, &ws.scr[0][0], g, tig, nkA, qb, QA, QX, QM, rc0, rc1, sa, mxA, mnA, dqA, dbg.astride);
        else
          qk_page<false, KD>(pgA, PL, &ws.scr[0][0], g, tig, PI, qb, QA, QX, QM, rc0, rc1, sa, mxA, mnA, dqA,
                         dbg.astride);
        if (hasB) {
          wait_fill<NSTG>(sm, kB);
          __syncwarp();
          if (!KD) {
            stage_kc<SE>(pgB, PL, &ws.scr[0][0], lane);
            __syncwarp();
          }
          qk_page<false, KD>(pgB, PL, &ws.scr[0][0], g, tig, PI, qb, QA, QX, QM, rc0, rc1, sbv, mxB, mnB,
                         dqA != nullptr ? dqA + PI : nullptr, dbg.astride);
        } else {
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) sbv[mt][0] = sbv[mt][1] = -INFINITY;
        }
        }
        __syncwarp();  // K codes/meta of the pair and the K coefficients are dead from here on
#if HACK_DEC_SPLIT
        ptx::mbar_wait(&sm.fullv[sA], (kA / NSTG) & 1);
        if (hasB) ptx::mbar_wait(&sm.fullv[sB], (kB / NSTG) & 1);
#endif

        // ---- V coefficients of the pair (cached sums, SE): channel c -> (A, B) pairs
        float4* vc_lo = reinterpret_cast<float4*>(pgA + PL.k_codes);  // channels 0..63
        if (!tail_item) {
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const int ch = lane + 32 * x;
            const __half2 hA = reinterpret_cast<const __half2*>(pgA + PL.v_meta)[ch];
            const __half2 hB = reinterpret_cast<const __half2*>(pgB + PL.v_meta)[ch];
            // (a single-page pair has pgB = pgA: finite page-B values, multiplied by its zero P meta)
            const float2 mv = f2(__low2float(hA), __low2float(hB));
            const float2 sv = f2(__high2float(hA), __high2float(hB));
            uint32_t sumA, sumB;
            if (SE) {  // cached sums (summation elimination)
              sumA = pgA[PL.v_sums + ch];
              sumB = pgB[PL.v_sums + ch];
            } else {   // HACK/SE ablation: the channel's 64 codes are 4 words of its V row
              const uint4 a = *reinterpret_cast<const uint4*>(pgA + PL.v_codes + ch * 16);
              sumA = codesum2(a.x) + codesum2(a.y) + codesum2(a.z) + codesum2(a.w);
              sumB = 0u;
              if (hasB) {
                const uint4 b2 = *reinterpret_cast<const uint4*>(pgB + PL.v_codes + ch * 16);
                sumB = codesum2(b2.x) + codesum2(b2.y) + codesum2(b2.z) + codesum2(b2.w);
              }
            }
            const float2 sum = ptx::fadd2(asf2(0x4B000000u | sumA, 0x4B000000u | sumB), f2(-8388608.f, -8388608.f));
            const float2 mu = ptx::ffma2(sv, f2(1.5f, 1.5f), mv);
            const float2 yv = ptx::ffma2(sv, ptx::fadd2(sum, f2(-96.f, -96.f)), ptx::fmul2(f2(64.f, 64.f), mu));
            const float2 nr = ptx::ffma2(sum, f2(-510.f, -510.f), f2(-kMagicF, -kMagicF));
            float4* dst = x < 2 ? vc_lo + 2 * ch : &ws.scr[ch - 64][0];
            dst[0] = make_float4(sv.x, sv.y, mu.x, mu.y);
            dst[1] = make_float4(yv.x, yv.y, nr.x, nr.y);
          }
        }

        // ---- (a5) online softmax over the pair
#if HACK_DEC_LSUM
        // row max of the pair = max of the two pages' row maxima (reduced anyway for P')
#pragma unroll
        for (int o2 = 4; o2 < 32; o2 <<= 1) {
          mnA = fminf(mnA, __shfl_xor_sync(0xffffffffu, mnA, o2));
          mxA = fmaxf(mxA, __shfl_xor_sync(0xffffffffu, mxA, o2));
          mnB = fminf(mnB, __shfl_xor_sync(0xffffffffu, mnB, o2));
          mxB = fmaxf(mxB, __shfl_xor_sync(0xffffffffu, mxB, o2));
        }
        const float mx = fmaxf(mxA, mxB);
#else
        float mx = fmaxf(mxA, mxB);
#pragma unroll
        for (int o2 = 4; o2 < 32; o2 <<= 1) {
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o2));
          mnA = fminf(mnA, __shfl_xor_sync(0xffffffffu, mnA, o2));
          mxA = fmaxf(mxA, __shfl_xor_sync(0xffffffffu, mxA, o2));
          mnB = fminf(mnB, __shfl_xor_sync(0xffffffffu, mnB, o2));
          mxB = fmaxf(mxB, __shfl_xor_sync(0xffffffffu, mxB, o2));
        }
#endif
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
#if !HACK_DEC_LSUM  // (LSUM: l_run stays this lane's partial sum until the flush)
#pragma unroll
        for (int o2 = 4; o2 < 32; o2 <<= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o2);
#endif
        l_run = __fmaf_rn(l_run, al, ls);
        m_run = mnew;
        // O *= al is fused into the PV update below (o = o al + t, one explicit FFMA2): a
        // separate FMUL2 + FADD2 pair may or may not be contracted by ptxas depending on the
        // surrounding code, which made the debug and production instantiations differ in ulps
        const float2 al2 = f2(al, al);

        if (!tail_item) {
          // ---- (a6) P' per (row, page): RN 8-bit against fp32 (lo, s) of the unnormalized p~
          uint8_t* pcode = pgA + PL.k_meta;  // [row 4][page 2][64] in B-fragment order
          float2 AP, XP, MP;
          uint32_t rcA, rcB;
          {
            QMeta pA = meta_p_fast(ex2(mnA - mnew), ex2(mxA - mnew));
            if (!(pA.s > 1e-30f)) { pA.s = 0.f; pA.inv = 0.f; }
            QMeta pB = {0.f, 0.f, 0.f};
            if (hasB) {
              pB = meta_p_fast(ex2(mnB - mnew), ex2(mxB - mnew));
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
                if (DBG && tig < G) {
                  const int t = 16 * mt + g + 8 * hh;
                  uint8_t* dr = dbg_pcodes + ((int64_t)s.b * kc.Hq + s.hk * G + tig) * dbg_stride;
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
            MP = f2(__fmaf_rn(127.5f, pA.s, pA.m), __fmaf_rn(127.5f, pB.s, pB.m));
            rcA = kMagic + (uint32_t)(-(2 * qkm * (int)spA - PI * 255 * qkm));
            rcB = kMagic + (uint32_t)(-(2 * qkm * (int)spB - PI * 255 * qkm));
          }
          __syncwarp();  // P' codes and V coefficients visible to the warp
          // B fragments of P'^T: column n = g = (row g>>1, page g&1); page P's k-steps 2P+u
          // hold tokens 16 tig + 4 i + q(u, h), q(0,0)=0, q(0,1)=2, q(1,0)=1, q(1,1)=3.
          uint32_t pb[4][2];
          {
            const uint4 Rw = *reinterpret_cast<const uint4*>(pcode + ((g >> 1) * 2 + (g & 1)) * 64 + 16 * tig);
            // (a single-page pair's page-B P' row holds zero codes: p~ = 0 and zero meta)
            const bool onA = (g & 1) == 0, onB = (g & 1) == 1;
            pb[0][0] = onA ? Rw.x : 0u; pb[0][1] = onA ? Rw.z : 0u;
            pb[1][0] = onA ? Rw.y : 0u; pb[1][1] = onA ? Rw.w : 0u;
            pb[2][0] = onB ? Rw.x : 0u; pb[2][1] = onB ? Rw.z : 0u;
            pb[3][0] = onB ? Rw.y : 0u; pb[3][1] = onB ? Rw.w : 0u;
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
#if HACK_DEC_OSUM
            float2 tq[2];  // t2 of channels g, g + 8: (page A, page B)
#endif
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const int ch = hh ? c1 : c0;
              const float4* vsrc = ch < 64 ? vc_lo + 2 * ch : &ws.scr[ch - 64][0];
              const float4 v0 = vsrc[0], v1 = vsrc[1];
              const uint32_t e0 = (acc0[2 * hh] << 2) + acc1[2 * hh], e1 = (acc0[2 * hh + 1] << 2) + acc1[2 * hh + 1];
              if (DBG && dbg.pv != nullptr && tig < G && dbg.hsel(s.hk * G + tig) >= 0) {  // 4 D' + RC, pages A, B
                int32_t* dp = dbg.pv + (((int64_t)s.b * dbg.hdim(kc.Hq) + dbg.hsel(s.hk * G + tig)) * (dbg.astride / PI) +
                                        jpA) * 128 + ch;
                dp[0] = (int32_t)(e0 - kMagic);
                if (hasB) dp[128] = (int32_t)(e1 - kMagic);
              }
              const float2 e = ptx::fadd2(asf2(e0, e1), f2(v1.z, v1.w));
              const float2 t2 = ptx::ffma2(AP, ptx::fmul2(f2(v0.x, v0.y), e),
                                           ptx::ffma2(XP, f2(v0.z, v0.w), ptx::fmul2(MP, f2(v1.x, v1.y))));
#if HACK_DEC_OSUM
              tq[hh] = t2;
#else
              o[mt][hh] = ptx::ffma2(o[mt][hh], al2, t2);
#endif
            }
#if HACK_DEC_OSUM
            // o = o al + (page A + page B) for both channels on paired ops (same values as the
            // scalar fma(o, al, a + b) per channel)
            o[mt] = ptx::ffma2(o[mt], al2, ptx::fadd2(f2(tq[0].x, tq[1].x), f2(tq[0].y, tq[1].y)));
#endif
          }
        } else {
          // ---- FP16 last V block (RQE): O^T += V_tail^T p~ in fp32
#pragma unroll
          for (int mt = 0; mt < 8; ++mt) {
#if HACK_DEC_OSUM
            o[mt] = ptx::fmul2(o[mt], al2);
#else
            o[mt][0] = ptx::fmul2(o[mt][0], al2);
            o[mt][1] = ptx::fmul2(o[mt][1], al2);
#endif
          }
          float* ptl = reinterpret_cast<float*>(pgA + PL.k_codes);  // [row 4][64]
#pragma unroll
          for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) ptl[tig * 64 + 16 * mt + g + 8 * hh] = sa[mt][hh];
          __syncwarp();
          const __half* tail = reinterpret_cast<const __half*>(cv.v_tail) + ((int64_t)slot * Hkv + s.hk) * PI * 128;
          for (int t = 0; t < nkA; ++t) {
            const float p = ptl[tig * 64 + t];
#pragma unroll
            for (int mt = 0; mt < 8; ++mt)
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const float v = __half2float(tail[t * 128 + 16 * mt + g + 8 * hh]);
#if HACK_DEC_OSUM
                if (hh)
                  o[mt].y = fmaf(p, v, o[mt].y);
                else
                  o[mt].x = fmaf(p, v, o[mt].x);
#else
                o[mt][hh].x = fmaf(p, v, o[mt][hh].x);
#endif
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
    // -- flush this warp's (m, l, O) partial of the segment: slot (u + c, warp), row tig
#if HACK_DEC_LSUM
#pragma unroll
    for (int o2 = 4; o2 < 32; o2 <<= 1) l_run += __shfl_xor_sync(0xffffffffu, l_run, o2);
#endif
    if (tig < G) {
      float* dst = part + ((((int64_t)(u + c)) * NW + warp) * G + tig) * kPart;
      if (g == 0) {
        dst[0] = m_run;
        dst[1] = l_run;
      }
#pragma unroll
      for (int mt = 0; mt < 8; ++mt)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
#if HACK_DEC_OSUM
          dst[2 + 16 * mt + g + 8 * hh] = hh ? o[mt].y : o[mt].x;
#else
          dst[2 + 16 * mt + g + 8 * hh] = o[mt][hh].x + o[mt][hh].y;
#endif
    }
    it_base += nitems;
    k_base += s.p1 - s.p0;
  }
  if (PIPES > 1) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegEven));
  }  // compute warps
  if (merge)
    merge_units<NW>(SegWalker{sm.range_b0, sm.range_base, min(c * sm.R, sm.P), min(c * sm.R + sm.R, sm.P)}, sm.R, cv,
                    slots, kc, cnt, part, out, &sm.mflag, ltid, FUSED, psync);
  if (FUSED && merge)  // (else decode_pair_combine)
    bump_lengths(io, cv, slots, batch, &sm.mflag, ltid, 32 * (NW + 1), nvirt, psync);
}

// ============================================================================ G in (4, 8]
// The same pipeline for GQA groups of up to 8 query rows (C4, Llama-3.1-70B: G = 8).
// S^T = K' Q'^T runs on TWO n-tiles of (row, d-block) columns (rows 0-3 and 4-7), so a lane
// holds rows tig and 4 + tig.  P'V' runs per page with the 8 N-columns = query rows (the
// 8 rows fill them without page pairing): a lane holds rows 2 tig, 2 tig + 1 and the
// per-row P meta / rescale factors move between the two row ownerships through a small
// per-warp table.  Items are single pages.
#ifndef HACK_DEC8_NSTG
#define HACK_DEC8_NSTG 6
#endif
#ifndef HACK_DEC8_CTAS
#define HACK_DEC8_CTAS 4
#endif
constexpr int NSTG8 = HACK_DEC8_NSTG;
constexpr int kCtas8 = HACK_DEC8_CTAS;

struct G8Smem {
  uint8_t stage[NSTG8][PB];
  struct Warp {
    float4 scr[64][2];      // K coefficients of the page in QK; V coefficients (float4 per channel) in PV
    uint8_t qcode[8][128];  // Q' rows of the current unit
    float4 qc[8][2];        // per row: (QA0, QA1, QX0, QX1), (QM0, QM1, RC0, RC1)
    float4 rowinfo[8];      // per row, this page: alpha, s_p, m_p, SP (as float)
#if HACK_G8_QSMEM
    uint4 qf[2][2][32];     // B fragments of Q' per (n-tile, k-step pair, lane), reloaded per use
#endif
  } w[NW];
  int range_b0, range_base;
  int R, P;
  uint64_t full[NSTG8], fullv[NSTG8], empty[NSTG8];
  int tag[NSTG8];
  int mflag;
};

template <bool DBG, bool FUSED>
__global__ void __launch_bounds__(kThreads8, kCtas8)
    decode_g8_kernel(const __half* __restrict__ q_new, const int32_t* __restrict__ slots, int batch, CacheView cv,
                     KernelCfg kc, int* __restrict__ ws_meta, int* __restrict__ cnt, float* __restrict__ part,
                     void* __restrict__ out, int merge, StepIO io, DecDbg dbg) {
  uint8_t* const dbg_pcodes = dbg.pcodes;
  const int64_t dbg_stride = dbg.pstride;
  constexpr int qkm = 3;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  G8Smem& sm = *reinterpret_cast<G8Smem*>(smem_raw);
  const int G = kc.G, Hkv = kc.Hkv;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int c = blockIdx.x;
  const PageLayout PL = kc.pl;
  if (tid == 0) {
    for (int s = 0; s < NSTG8; ++s) {
      ptx::mbar_init(&sm.full[s], 1);
      ptx::mbar_init(&sm.fullv[s], 1);
      sm.tag[s] = -1;
      ptx::mbar_init(&sm.empty[s], 1);
    }
    ptx::fence_mbar_init();
  }
#ifndef HACK_DEC_NOPDL
  // launched as a programmatic dependent of the append kernel: everything above touched
  // only shared memory; seq_lens, pages and the FP16 tail are read after this wait
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
  locate_range(sm, cv, slots, batch, Hkv, ws_meta, warp == 0, lane, FUSED, c, (int)gridDim.x);
  __syncthreads();
  const int R = sm.R, P = sm.P;
  SegWalker walk{sm.range_b0, sm.range_base, min(c * R, P), min(c * R + R, P)};
  if (warp == NW) {
    produce_pages<NSTG8, FUSED>(sm, walk, cv, slots, Hkv, kc, lane, io);
  } else {

  typename G8Smem::Warp& ws = sm.w[warp];
  const float cscale = 1.4426950408889634f / sqrtf(128.f);
  const int n0 = 2 * tig, n1 = 2 * tig + 1;  // rows of this lane in the PV fragments
  Seg s;
  int it_base = 0, k_base = 0;
  while (walk.next(cv, slots, Hkv, s, FUSED)) {
    const int slot = slots[s.b];
    const int len = len_of(cv, slot, FUSED);
    const int nfull = len / PI;
    const int nitems = s.p1 - s.p0;  // single pages
    const int my0 = ((warp - it_base) % NW + NW) % NW;
    const int u = s.b * Hkv + s.hk;
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};  // rows tig, 4 + tig
    float2 o[8][2];  // [m-tile][channel g / g+8] -> rows (n0, n1)
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) o[mt][0] = o[mt][1] = f2(0.f, 0.f);

    if (my0 < nitems) {
      const uint32_t rng_id = cv.rng_ids[slot];
      // ---- (a3) quantize the unit's 8 query rows (8-bit SR, fp32 meta), 16 lanes per row
#pragma unroll 1
      for (int r2 = 0; r2 < 4; ++r2) {
        const int row = 2 * r2 + (lane >> 4), lane16 = lane & 15;
        const int hq = s.hk * G + min(row, G - 1);
        const uint4 raw = reinterpret_cast<const uint4*>(q_new + ((int64_t)s.b * kc.Hq + hq) * 128)[lane16];
        uint64_t packed;
        float m, sc;
        int sum;
        quant_row16<8, false>(raw, lane16, PI, len - 1, kc.seed, rng_id,
                              stream_c3(kc.layer, kTagQ, kc.head_base * G + hq), kc.q_round, packed, m, sc, sum);
        const bool ok = row < G;
        *reinterpret_cast<uint2*>(&ws.qcode[row][lane16 * 8]) =
            ok ? make_uint2((uint32_t)packed, (uint32_t)(packed >> 32)) : make_uint2(0u, 0u);
        const int beta = lane16 >> 3;
        float* qcf = reinterpret_cast<float*>(&ws.qc[row][0]);
        if ((lane16 & 7) == 0) {
          qcf[beta] = ok ? cscale * sc * 0.25f : 0.f;
          qcf[2 + beta] = ok ? cscale * sc * ((float)sum - 127.5f * PI) : 0.f;
          qcf[4 + beta] = ok ? cscale * __fmaf_rn(127.5f, sc, m) : 0.f;
          qcf[6 + beta] = __int_as_float(ok ? -(2 * qkm * sum - PI * 255 * qkm) : 0);
        }
      }
      __syncwarp();
      // B fragments of Q' for n-tile nt, column n = g = (row 4 nt + (g>>1), block g&1)
      uint32_t qb[2][4][2];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int r = 4 * nt + (g >> 1);
        const bool live = r < G && (tig >> 1) == (g & 1);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const int q = ks == 0 ? 0 : (ks == 1 ? 2 : (ks == 2 ? 1 : 3));
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t v = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) v |= (uint32_t)ws.qcode[r][32 * tig + 16 * h + 4 * i + q] << (8 * i);
            qb[nt][ks][h] = live ? v : 0u;
          }
        }
      }
#if HACK_G8_QSMEM
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        ws.qf[nt][0][lane] = make_uint4(qb[nt][0][0], qb[nt][0][1], qb[nt][1][0], qb[nt][1][1]);
        ws.qf[nt][1][lane] = make_uint4(qb[nt][2][0], qb[nt][2][1], qb[nt][3][0], qb[nt][3][1]);
      }
      __syncwarp();
#endif
      float2 QA[2], QX[2], QM[2];
      uint32_t rc[2][2];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const float4 q0 = ws.qc[4 * nt + tig][0], q1 = ws.qc[4 * nt + tig][1];
        QA[nt] = f2(q0.x, q0.y);
        QX[nt] = f2(q0.z, q0.w);
        QM[nt] = f2(q1.x, q1.y);
        rc[nt][0] = kMagic + __float_as_uint(q1.z);
        rc[nt][1] = kMagic + __float_as_uint(q1.w);
      }

#pragma unroll 1
      for (int j = my0; j < nitems; j += NW) {
        const int k = k_base + j;
        const int st = k % NSTG8;
        const int jp = s.p0 + j;
        const bool committed = jp < nfull;
        const int nk = committed ? PI : len - jp * PI;
        uint8_t* pg = sm.stage[st];
        wait_fill<NSTG8>(sm, k);
        stage_kc<true>(pg, PL, &ws.scr[0][0], lane);
        __syncwarp();
        // ---- (a4) S^T for the 8 rows: sc[nt][mt][hh] = row 4 nt + tig, token 16 mt + g + 8 hh
        float sc[2][4][2];
        float mx[2] = {-INFINITY, -INFINITY}, mn[2] = {INFINITY, INFINITY};
        const float4* kcs = &ws.scr[0][0];
        // the partial last page's mask only where it applies (MASK: a compile-time flag)
        auto qk8 = [&](auto maskc) {
          constexpr bool MASK = decltype(maskc)::value;
  #pragma unroll
          for (int mt = 0; mt < 4; ++mt) {
            const int t0 = 16 * mt + g, t1 = t0 + 8;
            const uint2 w0 = *reinterpret_cast<const uint2*>(pg + PL.k_codes + t0 * 32 + 8 * tig);
            const uint2 w1 = *reinterpret_cast<const uint2*>(pg + PL.k_codes + t1 * 32 + 8 * tig);
            const Planes a0 = planes2(w0.x), a1 = planes2(w1.x), a2 = planes2(w0.y), a3 = planes2(w1.y);
  #pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              uint32_t acc0[4], acc1[4];
#if HACK_G8_QSMEM
              // (volatile shared loads: reloaded per use, not kept live across the page)
              uint4 f0, f1;
              asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(f0.x), "=r"(f0.y), "=r"(f0.z), "=r"(f0.w)
                           : "r"(ptx::smem_u32(&ws.qf[nt][0][lane])));
              asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(f1.x), "=r"(f1.y), "=r"(f1.z), "=r"(f1.w)
                           : "r"(ptx::smem_u32(&ws.qf[nt][1][lane])));
              mma16832c(acc0, a0.p0, a1.p0, a2.p0, a3.p0, f0.x, f0.y, 0u, 0u);
              mma16832(acc0, a0.p2, a1.p2, a2.p2, a3.p2, f0.z, f0.w);
              mma16832c(acc1, a0.p1, a1.p1, a2.p1, a3.p1, f1.x, f1.y, rc[nt][0], rc[nt][1]);
              mma16832(acc1, a0.p3, a1.p3, a2.p3, a3.p3, f1.z, f1.w);
#else
              mma16832c(acc0, a0.p0, a1.p0, a2.p0, a3.p0, qb[nt][0][0], qb[nt][0][1], 0u, 0u);
              mma16832(acc0, a0.p2, a1.p2, a2.p2, a3.p2, qb[nt][1][0], qb[nt][1][1]);
              mma16832c(acc1, a0.p1, a1.p1, a2.p1, a3.p1, qb[nt][2][0], qb[nt][2][1], rc[nt][0], rc[nt][1]);
              mma16832(acc1, a0.p3, a1.p3, a2.p3, a3.p3, qb[nt][3][0], qb[nt][3][1]);
#endif
  #pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const int t = hh ? t1 : t0;
                const float4 c0 = kcs[2 * t], c1 = kcs[2 * t + 1];
                const uint32_t e0 = (acc0[2 * hh] << 2) + acc1[2 * hh], e1 = (acc0[2 * hh + 1] << 2) + acc1[2 * hh + 1];
                if (DBG && dbg.qk != nullptr && 4 * nt + tig < G && t < nk && dbg.hsel(s.hk * G + 4 * nt + tig) >= 0) {
                  int32_t* dq = dbg.qk + ((int64_t)s.b * dbg.hdim(kc.Hq) + dbg.hsel(s.hk * G + 4 * nt + tig)) * 2 * dbg.astride +
                                jp * PI + t;  // raw 4 D_beta + RC
                  dq[0] = (int32_t)(e0 - kMagic);
                  dq[dbg.astride] = (int32_t)(e1 - kMagic);
                }
                const float2 e = ptx::fadd2(asf2(e0, e1), f2(c1.z, c1.w));
                const float2 s2 = ptx::ffma2(QA[nt], ptx::fmul2(f2(c0.x, c0.y), e),
                                             ptx::ffma2(QX[nt], f2(c0.z, c0.w), ptx::fmul2(QM[nt], f2(c1.x, c1.y))));
                float sv = s2.x + s2.y;
                if (MASK && t >= nk) sv = -INFINITY;
                sc[nt][mt][hh] = sv;
                mx[nt] = fmaxf(mx[nt], sv);
                if (!MASK || t < nk) mn[nt] = fminf(mn[nt], sv);
              }
            }
          }
        };
        if (nk == PI)
          qk8(std::false_type{});
        else
          qk8(std::true_type{});
        __syncwarp();  // K codes/meta and K coefficients are dead
        // ---- (a5) online softmax, rows tig and 4 + tig
        float al[2], ls[2] = {0.f, 0.f};
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
          for (int o2 = 4; o2 < 32; o2 <<= 1) {
            mx[nt] = fmaxf(mx[nt], __shfl_xor_sync(0xffffffffu, mx[nt], o2));
            mn[nt] = fminf(mn[nt], __shfl_xor_sync(0xffffffffu, mn[nt], o2));
          }
          const float mnew = fmaxf(m_run[nt], mx[nt]);
          al[nt] = m_run[nt] == -INFINITY ? 0.f : ex2(m_run[nt] - mnew);
          m_run[nt] = mnew;
#pragma unroll
          for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              sc[nt][mt][hh] = ex2(sc[nt][mt][hh] - mnew);
              ls[nt] += sc[nt][mt][hh];
            }
#if !HACK_DEC_LSUM  // (LSUM: l_run stays this lane's partial sum until the flush)
#pragma unroll
          for (int o2 = 4; o2 < 32; o2 <<= 1) ls[nt] += __shfl_xor_sync(0xffffffffu, ls[nt], o2);
#endif
          l_run[nt] = __fmaf_rn(l_run[nt], al[nt], ls[nt]);
        }
        uint8_t* pcode = pg + PL.k_meta;                          // [row 8][64] in B-fragment order
        float* ptl = reinterpret_cast<float*>(pg + PL.k_codes);    // [row 8][64] p~ of a partial page
        if (committed) {
          // ---- (a6) P' per row (RN 8-bit on p~) + the row table for the PV lanes
          const int base = 4 * (g & 3) + (g >> 2);
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            const int row = 4 * nt + tig;
            QMeta pm = meta_p_fast(ex2(mn[nt] - m_run[nt]), ex2(mx[nt] - m_run[nt]));
            if (!(pm.s > 1e-30f)) { pm.s = 0.f; pm.inv = 0.f; }
            const float nlo = -pm.m * pm.inv;
            uint32_t sp = 0;
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const float y = fmaf(sc[nt][mt][hh], pm.inv, nlo) + kMagicF;
                const uint32_t cc = __float_as_uint(y) & 0xFFu;
                sp += cc;
                pcode[row * 64 + 16 * mt + base + 2 * hh] = (uint8_t)cc;
                if (DBG && row < G)
                  dbg_pcodes[((int64_t)s.b * kc.Hq + s.hk * G + row) * dbg_stride + jp * PI + 16 * mt + g + 8 * hh] =
                      (uint8_t)cc;
              }
#pragma unroll
            for (int o2 = 4; o2 < 32; o2 <<= 1) sp += __shfl_xor_sync(0xffffffffu, sp, o2);
            if (g == 0) ws.rowinfo[row] = make_float4(al[nt], pm.s, pm.m, (float)sp);
          }
          __syncwarp();  // K region free: V coefficients overwrite the K coefficient scratch
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const int ch = lane + 32 * x;
            const __half2 hm = reinterpret_cast<const __half2*>(pg + PL.v_meta)[ch];
            const float mv = __low2float(hm), sv = __high2float(hm);
            const float sum = (float)pg[PL.v_sums + ch];
            const float mu = fmaf(sv, 1.5f, mv);
            reinterpret_cast<float4*>(&ws.scr[0][0])[ch] =
                make_float4(sv, mu, fmaf(sv, sum - 96.f, 64.f * mu), fmaf(sum, -510.f, -kMagicF));
          }
          __syncwarp();
          // PV lanes: rows n0, n1
          const float4 r0 = ws.rowinfo[n0], r1 = ws.rowinfo[n1];
          const float2 alp = f2(r0.x, r1.x);  // O *= alp fused into the PV update (explicit FFMA2)
          const float2 AP = f2(r0.y * 0.25f, r1.y * 0.25f);
          const float2 XP = f2(r0.y * (r0.w - 127.5f * PI), r1.y * (r1.w - 127.5f * PI));
          const float2 MP = f2(__fmaf_rn(127.5f, r0.y, r0.z), __fmaf_rn(127.5f, r1.y, r1.z));
          const uint32_t rp0 = kMagic + (uint32_t)(-(2 * qkm * (int)r0.w - PI * 255 * qkm));
          const uint32_t rp1 = kMagic + (uint32_t)(-(2 * qkm * (int)r1.w - PI * 255 * qkm));
          // B fragments of P'^T: column n = g = row g; k-steps u: tokens 16 tig + 4 i + q(u, h)
          const uint4 Rw = *reinterpret_cast<const uint4*>(pcode + g * 64 + 16 * tig);
          const float4* vcs = reinterpret_cast<const float4*>(&ws.scr[0][0]);
#pragma unroll
          for (int mt = 0; mt < 8; ++mt) {
            const int c0 = 16 * mt + g, c1 = c0 + 8;
            const Planes va = planes2(*reinterpret_cast<const uint32_t*>(pg + PL.v_codes + c0 * 16 + 4 * tig));
            const Planes vb = planes2(*reinterpret_cast<const uint32_t*>(pg + PL.v_codes + c1 * 16 + 4 * tig));
            uint32_t acc0[4], acc1[4];
            mma16832c(acc0, va.p0, vb.p0, va.p2, vb.p2, Rw.x, Rw.z, 0u, 0u);
            mma16832c(acc1, va.p1, vb.p1, va.p3, vb.p3, Rw.y, Rw.w, rp0, rp1);
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const float4 v4 = vcs[hh ? c1 : c0];
              const uint32_t e0 = (acc0[2 * hh] << 2) + acc1[2 * hh], e1 = (acc0[2 * hh + 1] << 2) + acc1[2 * hh + 1];
              if (DBG && dbg.pv != nullptr) {  // raw 4 D'_page + RC_page, rows n0, n1
                const int ch = hh ? c1 : c0;
                const int64_t nbk = dbg.astride / PI;
                const int hs0 = dbg.hsel(s.hk * G + n0), hs1 = dbg.hsel(s.hk * G + n1);
                int32_t* dp = dbg.pv + (int64_t)s.b * dbg.hdim(kc.Hq) * nbk * 128 + (int64_t)jp * 128 + ch;
                if (n0 < G && hs0 >= 0) dp[(int64_t)hs0 * nbk * 128] = (int32_t)(e0 - kMagic);
                if (n1 < G && hs1 >= 0) dp[(int64_t)hs1 * nbk * 128] = (int32_t)(e1 - kMagic);
              }
              const float2 e = ptx::fadd2(asf2(e0, e1), f2(v4.w, v4.w));
              const float2 t2 = ptx::ffma2(AP, ptx::fmul2(f2(v4.x, v4.x), e),
                                           ptx::ffma2(XP, f2(v4.y, v4.y), ptx::fmul2(MP, f2(v4.z, v4.z))));
              o[mt][hh] = ptx::ffma2(o[mt][hh], alp, t2);
            }
          }
        } else {
          // ---- FP16 last V block (RQE)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            const int row = 4 * nt + tig;
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) ptl[row * 64 + 16 * mt + g + 8 * hh] = sc[nt][mt][hh];
            if (g == 0) ws.rowinfo[row] = make_float4(al[nt], 0.f, 0.f, 0.f);
          }
          __syncwarp();
          const float2 alp = f2(ws.rowinfo[n0].x, ws.rowinfo[n1].x);
#pragma unroll
          for (int mt = 0; mt < 8; ++mt) {
            o[mt][0] = ptx::fmul2(o[mt][0], alp);
            o[mt][1] = ptx::fmul2(o[mt][1], alp);
          }
          const __half* tail = reinterpret_cast<const __half*>(cv.v_tail) + ((int64_t)slot * Hkv + s.hk) * PI * 128;
          for (int t = 0; t < nk; ++t) {
            const float2 p2 = f2(ptl[n0 * 64 + t], ptl[n1 * 64 + t]);
#pragma unroll
            for (int mt = 0; mt < 8; ++mt)
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const float v = __half2float(tail[t * 128 + 16 * mt + g + 8 * hh]);
                o[mt][hh] = ptx::ffma2(p2, f2(v, v), o[mt][hh]);
              }
          }
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&sm.empty[st]);
      }
    }
    // -- flush: (m, l) from the QK-side rows (tig, 4 + tig), O from the PV-side rows (n0, n1)
#if HACK_DEC_LSUM
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int o2 = 4; o2 < 32; o2 <<= 1) l_run[nt] += __shfl_xor_sync(0xffffffffu, l_run[nt], o2);
#endif
    float* dst = part + (((int64_t)(u + c)) * NW + warp) * G * kPart;
    if (g == 0) {
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int row = 4 * nt + tig;
        if (row < G) {
          dst[row * kPart] = m_run[nt];
          dst[row * kPart + 1] = l_run[nt];
        }
      }
    }
#pragma unroll
    for (int mt = 0; mt < 8; ++mt)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int ch = 16 * mt + g + 8 * hh;
        if (n0 < G) dst[n0 * kPart + 2 + ch] = o[mt][hh].x;
        if (n1 < G) dst[n1 * kPart + 2 + ch] = o[mt][hh].y;
      }
    it_base += nitems;
    k_base += s.p1 - s.p0;
  }
  }  // compute warps
  if (merge)
    merge_units<NW>(SegWalker{sm.range_b0, sm.range_base, min(c * sm.R, sm.P), min(c * sm.R + sm.R, sm.P)}, sm.R, cv,
                    slots, kc, cnt, part, out, &sm.mflag, tid, FUSED, [] { __syncthreads(); });
  if (FUSED && merge)  // (else decode_pair_combine)
    bump_lengths(io, cv, slots, batch, &sm.mflag, tid, (int)blockDim.x, (int)gridDim.x, [] { __syncthreads(); });
}

// out[b][hk*G + n][c] = sum_parts e^(m - M) O / sum_parts e^(m - M) l over the partials of
// unit u = b*Hkv + hk: CTAs c_first..c_last of its flattened page range, NW warps each.
// Fused step (bump != 0): seq_lens += 1 here, after the main grid (every read of the old
// lengths) completed.
__global__ void __launch_bounds__(128) decode_pair_combine(const int* __restrict__ ws_meta,
                                                           const float* __restrict__ part, KernelCfg kc,
                                                           void* __restrict__ out, CacheView cv,
                                                           const int32_t* __restrict__ slots, int bump) {
  const int b = blockIdx.x, hq = blockIdx.y, c = threadIdx.x, batch = gridDim.x;
  const int hk = hq / kc.G, n = hq % kc.G;
  // launched with programmatic stream serialization: wait for the main kernel's results
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (bump && hq == 0 && c == 0) {
    const int slot = slots[b];
    const int t = cv.seq_lens[slot];
    if (t / PI < cv.max_pages_per_req) cv.seq_lens[slot] = t + 1;  // capacity guard (append_kernel)
  }
  const int R = ws_meta[0];
  const int npg = ws_meta[kMetaInts + batch + b];
  const int off = ws_meta[kMetaInts + b] + hk * npg;
  const int u = b * kc.Hkv + hk;
  const int c0 = off / R, c1 = (off + npg - 1) / R;
  // all partial loads are issued before any is consumed (two dependent round trips in
  // total instead of one per partial); units spanning more than 4 CTAs loop
  const int np = (c1 - c0 + 1) * NW;
  const float* base = part + ((((int64_t)(u + c0)) * NW) * kc.G + n) * kPart;  // partial k at + k G kPart
  const int64_t stride = (int64_t)kc.G * kPart;
  float M = -INFINITY, L = 0.f, O = 0.f;
  for (int k0 = 0; k0 < np; k0 += 16) {
    float ms[16], ls[16], os[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const bool ok = k0 + k < np;
      const float* src = base + (k0 + k) * stride;
      ms[k] = ok ? src[0] : -INFINITY;
      ls[k] = ok ? src[1] : 0.f;
      os[k] = ok ? src[2 + c] : 0.f;
    }
    float Mn = M;
#pragma unroll
    for (int k = 0; k < 16; ++k) Mn = fmaxf(Mn, ms[k]);
    if (Mn == -INFINITY) continue;
    const float r = ex2(M - Mn);  // 0 when M = -inf
    L *= r;
    O *= r;
    M = Mn;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float f = ex2(ms[k] - M);  // ex2(-inf) = 0 for empty partials
      L = fmaf(f, ls[k], L);
      O = fmaf(f, os[k], O);
    }
  }
  const float v = O / L;
  const int64_t idx = ((int64_t)b * kc.Hq + hq) * 128 + c;
  if (kc.out_fp32)
    reinterpret_cast<float*>(out)[idx] = v;
  else
    reinterpret_cast<__half*>(out)[idx] = __float2half_rn(v);
}

int grid_size(bool g8 = false) {
  // per call and per current device (a process may drive several GPUs)
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (const char* e = getenv("HACK_DECODE_GRID")) return atoi(e);
  return sms * (g8 ? kCtas8 : kCtasPerSm * PIPES);  // page ranges (virtual CTAs)
}

// Where the split partials are merged: in the main kernel by the CTA completing a unit
// (merge_units) when units span few CTAs -- the merging CTA's few L2 round trips beat a
// second launch -- else by decode_pair_combine, whose B x H_q CTAs merge in parallel (long
// units over many CTAs, e.g. head-sharded decode).  Estimated from the host bound
// max_seqlen: CTAs per unit ~ pages per unit / pages per CTA.  (C3: 1.2 -> in the kernel;
// head-sharded N = 2: 2.3, measured 5 % slower in the kernel.)
bool merge_in_kernel(const KernelCfg& kc, int batch, int max_seqlen) {
  if (const char* e = getenv("HACK_DECODE_MERGE")) return e[0] == '1';  // A/B timing knob
  const double npg = (double)((max_seqlen + PI - 1) / PI);
  const double per_cta = npg * batch * kc.Hkv / grid_size(kc.G > 4);
  return npg <= 1.5 * per_cta;
}

size_t meta_bytes(int batch) { return ((size_t)(kMetaInts + 2 * batch) * sizeof(int) + 255) / 256 * 256; }
// merge counters, one per (request, KV head) unit: zero before the first launch, and every
// launch leaves them zero (merge_units)
size_t cnt_bytes(const KernelCfg& kc, int batch) { return ((size_t)batch * kc.Hkv * sizeof(int) + 255) / 256 * 256; }
// workspace: meta | merge counters | fused-step completion counter (256 B) | partials

}  // namespace

// The decode step (hack_decode_attention) fuses the append into this kernel when the merge
// runs in decode_pair_combine, which then bumps seq_lens.  With the merge in the kernel the
// bump needs a grid-wide completion count, and the fused step measured 1.5 % slower than the
// append kernel + attention (C3: 122.0 vs 120.2 us); HACK_DECODE_FUSED=1 / 0 forces a path.
bool decode_pair_fuse_step(const KernelCfg& kc, int batch, int max_seqlen) {
  if (const char* e = getenv("HACK_DECODE_FUSED")) return e[0] == '1';
  return !merge_in_kernel(kc, batch, max_seqlen);
}

bool decode_pair_supported(const KernelCfg& kc) {
  return kc.Pi == 64 && kc.d == 128 && kc.bits == 2 && kc.G <= 8 && kc.pl.page_bytes == PB &&
         !(kc.G > 4 && getenv("HACK_DECODE_NO_G8"));
}

size_t decode_pair_workspace(const KernelCfg& kc, int batch, int max_seqlen) {
  (void)max_seqlen;
  const size_t slots = (size_t)batch * kc.Hkv + grid_size(kc.G > 4);
  return meta_bytes(batch) + cnt_bytes(kc, batch) + 256 + slots * NW * kc.G * kPart * sizeof(float);
}

cudaError_t launch_decode_pair(const KernelCfg& kc, const void* q_new, const int32_t* slots, int batch,
                               int max_seqlen, const CacheView& cv, void* out, void* workspace,
                               const hack_debug_t* dbg, cudaStream_t st, const void* k_new, const void* v_new) {
  int* meta = reinterpret_cast<int*>(workspace);
  int* cnt = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(workspace) + meta_bytes(batch));
  int* done = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(workspace) + meta_bytes(batch) + cnt_bytes(kc, batch));
  float* part = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(workspace) + meta_bytes(batch) + cnt_bytes(kc, batch) + 256);
  // fused decode step (k_new given): the append runs inside the attention kernel
  const StepIO io = {reinterpret_cast<const __half*>(k_new), reinterpret_cast<const __half*>(v_new), done};
  const bool g8 = kc.G > 4;
  const size_t smem = g8 ? sizeof(G8Smem) : PIPES * sizeof(PairSmem);
  const bool with_dbg = dbg != nullptr && (dbg->pcodes != nullptr || dbg->qk_acc != nullptr ||
                                           dbg->pv_acc != nullptr);  // dumps: parity runs only
  const bool no_se = !g8 && getenv("HACK_DECODE_NO_SE") != nullptr;  // f2 ablation only
  const int grid = grid_size(g8);
  const bool merge = merge_in_kernel(kc, batch, max_seqlen);
  const bool fused = k_new != nullptr;  // (the SE ablation never runs fused: launch_decode_step)
  auto kern = g8 ? (with_dbg ? (fused ? decode_g8_kernel<true, true> : decode_g8_kernel<true, false>)
                             : (fused ? decode_g8_kernel<false, true> : decode_g8_kernel<false, false>))
          : with_dbg ? (no_se ? decode_pair_kernel<true, false, false>
                              : (fused ? decode_pair_kernel<true, true, true> : decode_pair_kernel<true, true, false>))
                     : (no_se ? decode_pair_kernel<false, false, false>
                              : (fused ? decode_pair_kernel<false, true, true> : decode_pair_kernel<false, true, false>));
  // the attribute is per device / context: set it on every launch (cheap), no process-wide cache
  {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  {
    // programmatic dependent launch: the grid launches (and its prologue runs) while the
    // preceding kernel on the stream (the append) drains; griddepcontrol.wait in the
    // kernel orders its global reads after that kernel's writes
    cudaLaunchConfig_t mc = {};
    mc.gridDim = dim3(g8 ? grid : grid / PIPES);
    mc.blockDim = dim3(g8 ? kThreads8 : kThreads);
    mc.dynamicSmemBytes = smem;
    mc.stream = st;
    cudaLaunchAttribute ma[1];
    ma[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    ma[0].val.programmaticStreamSerializationAllowed = 1;
    mc.attrs = ma;
#ifdef HACK_DEC_NOPDL
    mc.numAttrs = 0;
#else
    mc.numAttrs = 1;
#endif
    DecDbg dd = {nullptr, 0, nullptr, nullptr, 0, -1};
    if (with_dbg) dd = {dbg->pcodes, dbg->pcodes_stride, dbg->qk_acc, dbg->pv_acc, dbg->acc_stride, dbg->acc_head};
    const cudaError_t e1 = cudaLaunchKernelEx(&mc, kern, reinterpret_cast<const __half*>(q_new), slots, batch, cv, kc,
                                              meta, cnt, part, out, merge ? 1 : 0, io, dd);
    if (e1 != cudaSuccess) return e1;
  }
  note_launch();
  if (merge) return cudaGetLastError();
  // the merge kernel is launched as a programmatic dependent of the main kernel (PDL): its CTAs
  // can be resident before the main grid drains and wait in griddepcontrol.wait.  (Computing
  // the page geometry from seq_lens before the wait, with an early launch_dependents trigger
  // in the main grid, measured 2 us slower.)
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(batch, kc.Hq);
  lc.blockDim = dim3(128);
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  const cudaError_t e2 = cudaLaunchKernelEx(&lc, decode_pair_combine, (const int*)meta, (const float*)part, kc, out, cv,
                                            slots, k_new != nullptr ? 1 : 0);
  if (e2 != cudaSuccess) return e2;
  note_launch();
  return cudaGetLastError();
}

}  // namespace hack
