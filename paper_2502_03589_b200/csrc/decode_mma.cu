// decode_mma.cu -- HBM-bound homomorphic decode attention (a9), split-KV.
//
// Decode reads every cached token once per step (L_Q = 1), so the kernel is
// bound by streaming packed pages (84 B per token per KV head at b=2, Pi=64) and
// is designed around HBM, not the tensor cores:
//   * grid (request, KV head, split); each CTA owns a contiguous page range of one
//     (request, KV head) and its G query rows (GQA, R15);
//   * one producer lane streams whole pages (codes + fp16 meta + CACHED sums,
//     summation elimination P:687-690) into an 8-deep smem ring with cp.async.bulk
//     (TMA) + mbarrier; 4 compute warps each consume whole pages;
//   * codes are unpacked straight into mma.sync m16n8k32 u8 fragments in registers
//     (no smem round trip; (w >> 2 tig) & 0x03030303 plane extraction, Q' and P'
//     stored in the matching permutation);
//       S^T[token][row]  = K'[token][ch] . Q'[row][ch]   (tokens = M, rows = N <= 8)
//       O^T[ch][row]    += V'[ch][token] . P'[row][token] (channels = M)
//   * Eq. 4 in centered form on packed fp32x2 (FFMA2) pairs of query rows;
//   * online softmax per warp, P 8-bit RN per (row, committed V block); the
//     FP16 last V block (RQE) in fp32; warps merged in smem, splits merged by
//     decode_combine_kernel.
#include <type_traits>

#include "common.cuh"
#include "internal.h"
#include "tc_ptx.cuh"

// HACK_DMMA_LSUM=1 (default): the row sums stay per lane until the CTA merge (no per-page
// cross-lane reduction)
#ifndef HACK_DMMA_LSUM
#define HACK_DMMA_LSUM 1
#endif

namespace hack {

namespace {

#ifndef HACK_DMMA_NW
#define HACK_DMMA_NW 4
#endif
#ifndef HACK_DMMA_NSTG
#define HACK_DMMA_NSTG 8
#endif
#ifndef HACK_DMMA_CTAS
#define HACK_DMMA_CTAS 3
#endif
constexpr int NW = HACK_DMMA_NW;      // compute warps per CTA
constexpr int NSTG = HACK_DMMA_NSTG;  // page stages per CTA
constexpr int kCtas = HACK_DMMA_CTAS;  // resident CTAs per SM (launch bounds)
constexpr int kThreads = (NW + 1) * 32;
constexpr uint32_t kMagicI = 0x4B000000u;  // bits of 2^23

constexpr int up16(int x) { return (x + 15) / 16 * 16; }
// Page bytes at d = 128 (the closed form of hack_page_bytes).
constexpr int page_bytes_of(int bits, int pi) {
  const int nb = 128 / pi, sw = (bits == 2 ? pi * 3 : pi * 15) > 255 ? 2 : 1;
  return up16(pi * 128 * bits / 8) + up16(pi * nb * 4) + up16(pi * nb * sw) + up16(128 * pi * bits / 8) +
         up16(128 * 4) + up16(128 * sw);
}

// PI_ = partition size Pi in {32, 64, 128}: a page holds PI_ tokens (one V partition per
// channel), a K row holds NB = 128 / PI_ partitions (beta), the QK m-tiles per page are
// PI_ / 16 and the PV k-steps per page PI_ / 32.
template <int BITS, int PI_>
struct DecSmem {
  static constexpr int PI = PI_;
  static constexpr int NB = 128 / PI_;
  static constexpr int PB = page_bytes_of(BITS, PI_);
  // ring depth: NSTG pages at Pi = 64 (as tuned); other Pi keep the ring within ~48 KB.
  // NS must be a multiple of NW: warp w takes pages w, w + NW, ..., so slot k % NS is then
  // only ever refilled for the same warp and a phase-parity wait can never alias a fill
  // two phases behind.
  static constexpr int NS_FIT = 48 * 1024 / PB / NW * NW;
  static constexpr int NS = (PI_ == 64 || PB * NSTG <= 48 * 1024) ? NSTG : (NS_FIT < NW ? NW : NS_FIT);
  static_assert(NS % NW == 0, "ring depth must be a multiple of the compute warps");
  static constexpr int RING = PB * NS > NW * 8 * 128 * 4 ? PB * NS : NW * 8 * 128 * 4;
  union {
    uint8_t stage[RING];      // NS page slots of PB bytes
    float mrg_o[NW][8][128];  // after the page loop: per-warp partial O for the CTA merge
  };
  struct Warp {
    float4 kc[NB][PI];                // [beta][token]: sk, mu_k, y_k, -r_k
    float4 vc[128];                   // [channel]: sv, mu_v, y_v, -r_v
    alignas(16) uint8_t pcode[8][PI]; // P' in B-fragment order
    float ptl[8][PI];                 // p~ of the FP16 tail page
  } w[NW];
  uint8_t qcode[8][128];              // Q' rows (natural channel order)
  float4 qconst[NB][8];               // per (beta, row): aq, xq, mu_q, -r_q
  float mrg_m[NW][8], mrg_l[NW][8];
  uint64_t full[NS], empty[NS];
};

HACK_DEV float u2f(uint32_t x) { return __int2float_rn((int)x); }

HACK_DEV void mma16832(uint32_t (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Plane `p` of a packed word: codes {p, p+4, p+8, p+12} (2-bit) / {p, p+2, p+4, p+6} (4-bit) as bytes.
template <int BITS>
HACK_DEV uint32_t plane(uint32_t w, int sh) {
  return BITS == 2 ? (w >> sh) & 0x03030303u : (w >> sh) & 0x0F0F0F0Fu;
}

// Token / channel index held by byte i of plane `tig` of packed word W (16-code words at
// b=2: index 16W + 4i + tig; at b=4 words hold 8 codes: index 8W + 2i + tig, tig in {0,1}).
// resident CTAs per SM the shared memory allows (up to kCtas): the register budget of the
// launch bounds follows it (a 104 KB b = 4 ring fits twice, so 204 registers, no spills)
template <int BITS, int PI_>
constexpr int dmma_ctas() {
  constexpr size_t sm = sizeof(DecSmem<BITS, PI_>) + 1024;
  return sm * kCtas <= 227 * 1024 ? kCtas : (sm * 2 <= 227 * 1024 ? 2 : 1);
}

// DBG: parity runs only (hack_debug_t): P-code and raw QK / PV accumulator dumps (the
// accumulators hold 2^23 + D exactly: HACK_ACC_PLAIN).
template <int BITS, int PI_, bool DBG>
__global__ void __launch_bounds__(kThreads, dmma_ctas<BITS, PI_>()) decode_mma_kernel(const __half* __restrict__ q_new,
                                                              const int32_t* __restrict__ slots, CacheView cv,
                                                              KernelCfg kc, float* __restrict__ part, int nsplit,
                                                              uint8_t* __restrict__ dbg_pcodes, int64_t dbg_stride,
                                                              int32_t* __restrict__ dbg_qk, int32_t* __restrict__ dbg_pv,
                                                              int64_t acc_stride, int acc_head) {
  // dumped head dimension and index of query row n (-1 = not dumped), hack_debug_t.acc_head
  const int hdim = acc_head < 0 ? kc.Hq : 1;
  auto hsel = [&](int n) { return acc_head < 0 ? blockIdx.y * kc.G + n : (blockIdx.y * kc.G + n == acc_head ? 0 : -1); };
  using SM = DecSmem<BITS, PI_>;
  constexpr int PI = PI_, NB = SM::NB, NS = SM::NS;
  constexpr int MT = PI / 16, KSV = PI / 32;  // QK m-tiles, PV k-steps per page
  constexpr int qkm = (1 << BITS) - 1;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  const int b = blockIdx.x, hk = blockIdx.y, split = blockIdx.z;
  const int G = kc.G;
  const int slot = slots[b];
  const int len = cv.seq_lens[slot];
  const int pos = len - 1;
  const int npages = (len + PI - 1) / PI;
  const int nfull = len / PI;
  const int pps = (npages + nsplit - 1) / nsplit;
  const int p_beg = min(split * pps, npages), p_end = min(p_beg + pps, npages);
  const int np = p_end - p_beg;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tig = lane & 3;
  const PageLayout PL = kc.pl;
  const uint32_t rng_id = cv.rng_ids[slot];

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      ptx::mbar_init(&sm.full[s], 1);
      ptx::mbar_init(&sm.empty[s], 1);
    }
    ptx::fence_mbar_init();
  }
  // ---- (a3) quantize the G query rows (8-bit SR, fp32 meta): warps 0-3, 16 lanes per row
  for (int row0 = 2 * warp; warp < NW && row0 < 8; row0 += 2 * NW) {
    const int row = row0 + (lane >> 4), lane16 = lane & 15;  // rows 0..7
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
    if ((lane16 & (PI / 8 - 1)) == 0) {  // first lane of the row's partition beta
      const int beta = lane16 / (PI / 8);
      const float cscale = 1.4426950408889634f / sqrtf(128.f);
      sm.qconst[beta][row] = row < G ? make_float4(cscale * s * 0.25f, cscale * s * ((float)sum - 127.5f * PI),
                                                   cscale * __fmaf_rn(127.5f, s, m), -(float)(2 * qkm * sum - PI * 255 * qkm))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  __syncthreads();

  const int n0 = 2 * tig, n1 = 2 * tig + 1;  // this thread's query rows in C fragments
  float2 m_run = make_float2(-INFINITY, -INFINITY), l_run = make_float2(0.f, 0.f);
  float2 o[8][2];  // [m-tile][channel g / g+8] -> rows (n0, n1)
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) o[mt][0] = o[mt][1] = make_float2(0.f, 0.f);

  if (warp == NW) {
    // ------------------------------------------------------------------ producer
    if (lane == 0) {
      const int32_t* bt = cv.block_table + (int64_t)slot * cv.max_pages_per_req;
      for (int k = 0; k < np; ++k) {
        const int s = k % NS;
        ptx::mbar_wait(&sm.empty[s], ((k / NS) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&sm.full[s], SM::PB);
        const uint8_t* pg = cv.pages + ((int64_t)bt[p_beg + k] * cv.num_kv_heads + hk) * cv.page_bytes;
        ptx::bulk_g2s(sm.stage + s * SM::PB, pg, SM::PB, &sm.full[s]);
      }
    }
  } else {
    // ------------------------------------------------------------------ compute warp
    typename SM::Warp& ws = sm.w[warp];
    // B fragments of Q' (query row n = g) in the K-unpack permutation, and row constants
    uint32_t qb[4][2];
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t v = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int ch = BITS == 2 ? 32 * ks + 16 * h + 4 * i + tig : 32 * ks + 16 * h + 8 * (tig >> 1) + 2 * i + (tig & 1);
          v |= (uint32_t)sm.qcode[g][ch] << (8 * i);
        }
        qb[ks][h] = v;
      }
    float2 QA[NB], QX[NB], QM[NB], QN[NB];
#pragma unroll
    for (int beta = 0; beta < NB; ++beta) {
      const float4 c0 = sm.qconst[beta][n0], c1 = sm.qconst[beta][n1];
      QA[beta] = make_float2(c0.x, c1.x);
      QX[beta] = make_float2(c0.y, c1.y);
      QM[beta] = make_float2(c0.z, c1.z);
      QN[beta] = make_float2(c0.w, c1.w);
    }
    const int sh = BITS == 2 ? 2 * tig : 4 * (tig & 1);

#pragma unroll 1
    for (int k = warp; k < np; k += NW) {
      const int s = k % NS;
      const int jp = p_beg + k;              // page index in the request
      const bool committed = jp < nfull;
      const int nk = min(PI, len - jp * PI);
      ptx::mbar_wait(&sm.full[s], (k / NS) & 1);
      const uint8_t* pg = sm.stage + s * SM::PB;
      // -- per-token (beta) and per-channel Eq. 4 coefficients from fp16 meta + cached sums
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const int e = lane + 32 * x;        // (token, beta) = (e / NB, e % NB): PI x NB = 128 entries
        const int t = e / NB, beta = e % NB;
        float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
        if (t < nk) {
          const __half2 mh = reinterpret_cast<const __half2*>(pg + PL.k_meta)[e];
          const float mk = __low2float(mh), sk = __high2float(mh);
          const int sum = load_sum(pg + PL.k_sums, e, PL.sum_bytes);  // cached (SE)
          const float mu = __fmaf_rn(0.5f * qkm, sk, mk);
          c0 = sk;
          c1 = mu;
          c2 = __fmaf_rn(sk, (float)sum - 0.5f * qkm * PI, __fmul_rn((float)PI, mu));
          c3 = -(float)(510 * sum);
        }
        ws.kc[beta][t] = make_float4(c0, c1, c2, c3);
      }
      if (committed) {
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const int c = lane + 32 * x;
          const __half2 mh = reinterpret_cast<const __half2*>(pg + PL.v_meta)[c];
          const float mv = __low2float(mh), sv = __high2float(mh);
          const int sum = load_sum(pg + PL.v_sums, c, PL.sum_bytes);  // cached (SE)
          const float mu = __fmaf_rn(0.5f * qkm, sv, mv);
          ws.vc[c] = make_float4(sv, mu, __fmaf_rn(sv, (float)sum - 0.5f * qkm * PI, __fmul_rn((float)PI, mu)),
                                 -(float)(510 * sum));
        }
      }
      __syncwarp();
      // -- S^T = K' Q'^T per m-tile of 16 tokens; Eq. 4 on (row n0, n1) pairs
      float2 sv2[MT][2];  // [m-tile][token g / g+8]
      float2 mx2 = make_float2(-INFINITY, -INFINITY), mn2 = make_float2(INFINITY, INFINITY);
      // the tail page's mask only where it applies (TAIL: a compile-time flag)
      auto qk = [&](auto tailc) {
        constexpr bool TAIL = decltype(tailc)::value;
  #pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int t0 = 16 * mt + g, t1 = t0 + 8;
          const uint4* r0 = reinterpret_cast<const uint4*>(pg + PL.k_codes + t0 * (128 * BITS / 8));
          const uint4* r1 = reinterpret_cast<const uint4*>(pg + PL.k_codes + t1 * (128 * BITS / 8));
          uint32_t w0[8 * BITS / 2], w1[8 * BITS / 2];
  #pragma unroll
          for (int x = 0; x < 2 * BITS / 2; ++x) {
            const uint4 a = r0[x], c = r1[x];
            w0[4 * x] = a.x; w0[4 * x + 1] = a.y; w0[4 * x + 2] = a.z; w0[4 * x + 3] = a.w;
            w1[4 * x] = c.x; w1[4 * x + 1] = c.y; w1[4 * x + 2] = c.z; w1[4 * x + 3] = c.w;
          }
          // accumulate on top of 0x4B000000: asfloat(acc) = 2^23 + D exactly (D < 2^22)
          uint32_t acc[NB][4];
  #pragma unroll
          for (int beta = 0; beta < NB; ++beta) acc[beta][0] = acc[beta][1] = acc[beta][2] = acc[beta][3] = kMagicI;
  #pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            uint32_t a[4];
            if (BITS == 2) {
              a[0] = plane<2>(w0[2 * ks], sh);
              a[1] = plane<2>(w1[2 * ks], sh);
              a[2] = plane<2>(w0[2 * ks + 1], sh);
              a[3] = plane<2>(w1[2 * ks + 1], sh);
            } else {
              // 4-bit: 8 codes per word; K-cols 4tig+i of half h <- word 4ks + 2h + (tig >> 1)
              const bool odd = tig >> 1;  // select, not a dynamic register-array index
              a[0] = plane<4>(odd ? w0[4 * ks + 1] : w0[4 * ks], sh);
              a[1] = plane<4>(odd ? w1[4 * ks + 1] : w1[4 * ks], sh);
              a[2] = plane<4>(odd ? w0[4 * ks + 3] : w0[4 * ks + 2], sh);
              a[3] = plane<4>(odd ? w1[4 * ks + 3] : w1[4 * ks + 2], sh);
            }
            mma16832(acc[ks * 32 / PI], a, qb[ks][0], qb[ks][1]);  // k-step ks: channels 32ks.. of block beta
          }
          if (DBG && dbg_qk != nullptr) {  // rows n0, n1; tokens t0 / t1; every beta
  #pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const int t = hh ? t1 : t0;
              if (t < nk) {
  #pragma unroll
                for (int beta = 0; beta < NB; ++beta) {
                  int32_t* dq = dbg_qk + (int64_t)b * hdim * NB * acc_stride + beta * acc_stride + jp * PI + t;
                  if (n0 < G && hsel(n0) >= 0) dq[(int64_t)hsel(n0) * NB * acc_stride] = (int32_t)(acc[beta][2 * hh] - kMagicI);
                  if (n1 < G && hsel(n1) >= 0)
                    dq[(int64_t)hsel(n1) * NB * acc_stride] = (int32_t)(acc[beta][2 * hh + 1] - kMagicI);
                }
              }
            }
          }
          float2 st[2];
  #pragma unroll
          for (int hh = 0; hh < 2; ++hh) {  // token t0 (c0, c1) / t1 (c2, c3)
            const int t = hh ? t1 : t0;
            float2 accf = make_float2(0.f, 0.f);
  #pragma unroll
            for (int beta = 0; beta < NB; ++beta) {
              const float4 k4 = ws.kc[beta][t];
              const float sk = k4.x, mu = k4.y, yk = k4.z, nr = k4.w;
              const float2 df = ptx::fadd2(make_float2(__uint_as_float(acc[beta][2 * hh]), __uint_as_float(acc[beta][2 * hh + 1])),
                                           make_float2(-8388608.f, -8388608.f));
              const float2 e = ptx::ffma2(make_float2(4.f, 4.f), df, ptx::fadd2(QN[beta], make_float2(nr, nr)));
              const float2 base = ptx::ffma2(QM[beta], make_float2(yk, yk), accf);
              accf = ptx::ffma2(QA[beta], ptx::fmul2(make_float2(sk, sk), e), ptx::ffma2(QX[beta], make_float2(mu, mu), base));
            }
            if (TAIL && t >= nk) accf = make_float2(-INFINITY, -INFINITY);  // beyond the cache (tail page)
            st[hh] = accf;
            mx2 = make_float2(fmaxf(mx2.x, accf.x), fmaxf(mx2.y, accf.y));
            if (!TAIL || t < nk) mn2 = make_float2(fminf(mn2.x, accf.x), fminf(mn2.y, accf.y));
          }
          sv2[mt][0] = st[0];
          sv2[mt][1] = st[1];
        }
      };
      if (committed)
        qk(std::false_type{});
      else
        qk(std::true_type{});
      // row reductions over the 8 lanes sharing tig
#pragma unroll
      for (int o2 = 4; o2 < 32; o2 <<= 1) {
        mx2.x = fmaxf(mx2.x, __shfl_xor_sync(0xffffffffu, mx2.x, o2));
        mx2.y = fmaxf(mx2.y, __shfl_xor_sync(0xffffffffu, mx2.y, o2));
        mn2.x = fminf(mn2.x, __shfl_xor_sync(0xffffffffu, mn2.x, o2));
        mn2.y = fminf(mn2.y, __shfl_xor_sync(0xffffffffu, mn2.y, o2));
      }
      const float2 mnew = make_float2(fmaxf(m_run.x, mx2.x), fmaxf(m_run.y, mx2.y));
      const float2 al = make_float2(m_run.x == -INFINITY ? 0.f : ex2(m_run.x - mnew.x),
                                    m_run.y == -INFINITY ? 0.f : ex2(m_run.y - mnew.y));
      float2 ls = make_float2(0.f, 0.f);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const float2 a2 = ptx::fadd2(sv2[mt][hh], make_float2(-mnew.x, -mnew.y));
          sv2[mt][hh] = make_float2(ex2(a2.x), ex2(a2.y));  // p~; ex2(-inf) = 0
          ls = ptx::fadd2(ls, sv2[mt][hh]);
        }
#if !HACK_DMMA_LSUM  // (LSUM: l_run stays this lane's partial sum until the merge)
#pragma unroll
      for (int o2 = 4; o2 < 32; o2 <<= 1) {
        ls.x += __shfl_xor_sync(0xffffffffu, ls.x, o2);
        ls.y += __shfl_xor_sync(0xffffffffu, ls.y, o2);
      }
#endif
      l_run = ptx::ffma2(l_run, al, ls);
      m_run = mnew;
      // O *= al is fused into the PV update (o = o al + t, one explicit FFMA2): a separate
      // FMUL2 + FADD2 pair may be contracted by ptxas or not depending on the surrounding code
      if (committed) {
        // -- (a6) P' per (row, V block): lo/hi from the score min/max (ex2 is monotone)
        const float2 lo = make_float2(ex2(mn2.x - mnew.x), ex2(mn2.y - mnew.y));
        const float2 hi = make_float2(ex2(mx2.x - mnew.x), ex2(mx2.y - mnew.y));
        QMeta pm0 = meta_p_fast(lo.x, hi.x), pm1 = meta_p_fast(lo.y, hi.y);
        if (!(pm0.s > 1e-30f)) { pm0.s = 0.f; pm0.inv = 0.f; }
        if (!(pm1.s > 1e-30f)) { pm1.s = 0.f; pm1.inv = 0.f; }
        const float2 inv2 = make_float2(pm0.inv, pm1.inv), nlo2 = make_float2(-lo.x * pm0.inv, -lo.y * pm1.inv);
        uint32_t sp0 = 0, sp1 = 0;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int t = 16 * mt + g + 8 * hh;
            uint32_t c0, c1;
            if (kc.p_round == HACK_ROUND_NEAREST_EVEN) {
              const float2 y = ptx::fadd2(ptx::ffma2(sv2[mt][hh], inv2, nlo2), make_float2(12582912.f, 12582912.f));
              c0 = __float_as_uint(y.x) & 0xFFu;
              c1 = __float_as_uint(y.y) & 0xFFu;
            } else {  // the paper's stochastic rounding of P (R6, selectable)
              const float2 y = ptx::ffma2(sv2[mt][hh], inv2, nlo2);
              const int ta = jp * PI + t, gh = (kc.head_base * G + hk * G);
              c0 = n0 < G ? p_code_sr(y.x, p_uniform(kc.seed, rng_id, kc.layer, gh + n0, pos, ta)) : 0u;
              c1 = n1 < G ? p_code_sr(y.y, p_uniform(kc.seed, rng_id, kc.layer, gh + n1, pos, ta)) : 0u;
            }
            sp0 += c0;
            sp1 += c1;
            // B-fragment position of token t: t' = t mod 16 = 4i + tig' -> 4 tig' + i (b=2)
            const int tp = t & 15;
            const int posn = BITS == 2 ? (t & ~15) + 4 * (tp & 3) + (tp >> 2)
                                       : (t & ~15) + 4 * (((tp >> 3) << 1) | (tp & 1)) + ((tp >> 1) & 3);
            ws.pcode[n0][posn] = (uint8_t)c0;
            ws.pcode[n1][posn] = (uint8_t)c1;
          }
#pragma unroll
        for (int o2 = 4; o2 < 32; o2 <<= 1) {
          sp0 += __shfl_xor_sync(0xffffffffu, sp0, o2);
          sp1 += __shfl_xor_sync(0xffffffffu, sp1, o2);
        }
        __syncwarp();
        if (DBG && dbg_pcodes != nullptr && g < G) {  // debug dump (natural token order) of row g
          for (int t = tig; t < PI; t += 4) {
            const int tp = t & 15;
            const int posn = BITS == 2 ? (t & ~15) + 4 * (tp & 3) + (tp >> 2)
                                       : (t & ~15) + 4 * (((tp >> 3) << 1) | (tp & 1)) + ((tp >> 1) & 3);
            dbg_pcodes[((int64_t)b * kc.Hq + hk * G + g) * dbg_stride + jp * PI + t] = ws.pcode[g][posn];
          }
        }
        // P' B fragments (row n = g): positions 32ks + 4tig (b0) and 32ks + 16 + 4tig (b1)
        uint32_t pb[KSV][2];
#pragma unroll
        for (int ks = 0; ks < KSV; ++ks) {
          pb[ks][0] = *reinterpret_cast<const uint32_t*>(&ws.pcode[g][32 * ks + 4 * tig]);
          pb[ks][1] = *reinterpret_cast<const uint32_t*>(&ws.pcode[g][32 * ks + 16 + 4 * tig]);
        }
        const float2 AP = make_float2(pm0.s * 0.25f, pm1.s * 0.25f);
        const float2 XP = make_float2(pm0.s * ((float)sp0 - 127.5f * PI), pm1.s * ((float)sp1 - 127.5f * PI));
        const float2 MP = make_float2(__fmaf_rn(127.5f, pm0.s, pm0.m), __fmaf_rn(127.5f, pm1.s, pm1.m));
        const float2 NRP = make_float2(-(float)(2 * qkm * (int)sp0 - PI * 255 * qkm),
                                       -(float)(2 * qkm * (int)sp1 - PI * 255 * qkm));
        // -- O^T += V' P'^T per m-tile of 16 channels; Eq. 4 (centered) with cached V sums
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          const int c0 = 16 * mt + g, c1 = c0 + 8;
          // the channel's PI codes: PI * BITS / 32 words (2 per 32-token k-step at b = 2, 4 at b = 4)
          constexpr int NWD = PI * BITS / 32;
          uint32_t wa[NWD], wb[NWD];
          if constexpr (NWD % 4 == 0) {  // 16-byte loads (all but Pi = 32, b = 2)
#pragma unroll
            for (int x = 0; x < NWD; x += 4) {
              const uint4 a4 = *reinterpret_cast<const uint4*>(pg + PL.v_codes + c0 * (PI * BITS / 8) + 4 * x);
              const uint4 b4 = *reinterpret_cast<const uint4*>(pg + PL.v_codes + c1 * (PI * BITS / 8) + 4 * x);
              wa[x] = a4.x; wa[x + 1] = a4.y; wa[x + 2] = a4.z; wa[x + 3] = a4.w;
              wb[x] = b4.x; wb[x + 1] = b4.y; wb[x + 2] = b4.z; wb[x + 3] = b4.w;
            }
          } else {
#pragma unroll
            for (int x = 0; x < NWD; x += 2) {
              const uint2 a2 = *reinterpret_cast<const uint2*>(pg + PL.v_codes + c0 * (PI * BITS / 8) + 4 * x);
              const uint2 b2 = *reinterpret_cast<const uint2*>(pg + PL.v_codes + c1 * (PI * BITS / 8) + 4 * x);
              wa[x] = a2.x; wa[x + 1] = a2.y;
              wb[x] = b2.x; wb[x + 1] = b2.y;
            }
          }
          uint32_t dacc[4] = {kMagicI, kMagicI, kMagicI, kMagicI};
          if (BITS == 2) {
#pragma unroll
            for (int ks = 0; ks < KSV; ++ks) {
              const uint32_t a[4] = {plane<2>(wa[2 * ks], sh), plane<2>(wb[2 * ks], sh), plane<2>(wa[2 * ks + 1], sh),
                                     plane<2>(wb[2 * ks + 1], sh)};
              mma16832(dacc, a, pb[ks][0], pb[ks][1]);
            }
          } else {
#pragma unroll
            for (int ks = 0; ks < KSV; ++ks) {
              const bool odd = tig >> 1;
              const uint32_t a[4] = {plane<4>(odd ? wa[4 * ks + 1] : wa[4 * ks], sh),
                                     plane<4>(odd ? wb[4 * ks + 1] : wb[4 * ks], sh),
                                     plane<4>(odd ? wa[4 * ks + 3] : wa[4 * ks + 2], sh),
                                     plane<4>(odd ? wb[4 * ks + 3] : wb[4 * ks + 2], sh)};
              mma16832(dacc, a, pb[ks][0], pb[ks][1]);
            }
          }
          if (DBG && dbg_pv != nullptr) {  // rows n0, n1; channels c0 / c1 of block jp
            const int64_t nbk = acc_stride / PI;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              int32_t* dp = dbg_pv + (int64_t)b * hdim * nbk * 128 + (int64_t)jp * 128 + (hh ? c1 : c0);
              if (n0 < G && hsel(n0) >= 0) dp[(int64_t)hsel(n0) * nbk * 128] = (int32_t)(dacc[2 * hh] - kMagicI);
              if (n1 < G && hsel(n1) >= 0) dp[(int64_t)hsel(n1) * nbk * 128] = (int32_t)(dacc[2 * hh + 1] - kMagicI);
            }
          }
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int c = hh ? c1 : c0;
            const float4 v4 = ws.vc[c];
            const float svv = v4.x, mu = v4.y, yv = v4.z, nr = v4.w;
            const float2 df = ptx::fadd2(make_float2(__uint_as_float(dacc[2 * hh]), __uint_as_float(dacc[2 * hh + 1])),
                                         make_float2(-8388608.f, -8388608.f));
            const float2 e = ptx::ffma2(make_float2(4.f, 4.f), df, ptx::fadd2(NRP, make_float2(nr, nr)));
            const float2 t2 = ptx::ffma2(AP, ptx::fmul2(make_float2(svv, svv), e),
                                         ptx::ffma2(XP, make_float2(mu, mu), ptx::fmul2(MP, make_float2(yv, yv))));
            o[mt][hh] = ptx::ffma2(o[mt][hh], al, t2);
          }
        }
      } else {
        // -- FP16 last V block (RQE): O^T += V_tail^T p~ in fp32
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          o[mt][0] = ptx::fmul2(o[mt][0], al);
          o[mt][1] = ptx::fmul2(o[mt][1], al);
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int t = 16 * mt + g + 8 * hh;
            ws.ptl[n0][t] = sv2[mt][hh].x;
            ws.ptl[n1][t] = sv2[mt][hh].y;
          }
        __syncwarp();
        const __half* tail = reinterpret_cast<const __half*>(cv.v_tail) + ((int64_t)slot * kc.Hkv + hk) * PI * 128;
        for (int t = 0; t < nk; ++t) {
          const float2 p2 = make_float2(ws.ptl[n0][t], ws.ptl[n1][t]);
#pragma unroll
          for (int mt = 0; mt < 8; ++mt)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const float v = __half2float(tail[t * 128 + 16 * mt + g + 8 * hh]);
              o[mt][hh] = ptx::ffma2(p2, make_float2(v, v), o[mt][hh]);
            }
        }
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&sm.empty[s]);
    }
  }
  __syncthreads();  // all pages consumed: the stage ring is reused for the merge
  if (warp < NW) {
    // -- publish this warp's partial (m, l, O) for the CTA merge
#if HACK_DMMA_LSUM
#pragma unroll
    for (int o2 = 4; o2 < 32; o2 <<= 1) {
      l_run.x += __shfl_xor_sync(0xffffffffu, l_run.x, o2);
      l_run.y += __shfl_xor_sync(0xffffffffu, l_run.y, o2);
    }
#endif
    if (g == 0) {
      sm.mrg_m[warp][n0] = m_run.x;
      sm.mrg_m[warp][n1] = m_run.y;
      sm.mrg_l[warp][n0] = l_run.x;
      sm.mrg_l[warp][n1] = l_run.y;
    }
#pragma unroll
    for (int mt = 0; mt < 8; ++mt)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int c = 16 * mt + g + 8 * hh;
        sm.mrg_o[warp][n0][c] = o[mt][hh].x;
        sm.mrg_o[warp][n1][c] = o[mt][hh].y;
      }
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
          L = __fmaf_rn(f, sm.mrg_l[w][n], L);
          O = __fmaf_rn(f, sm.mrg_o[w][n][c], O);
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

// out[b][hk*G + n][c] = sum_s e^(m_s - M) O_s / sum_s e^(m_s - M) l_s
__global__ void decode_combine_kernel(const float* __restrict__ part, int nsplit, KernelCfg kc,
                                      void* __restrict__ out) {
  const int b = blockIdx.x, hq = blockIdx.y, c = threadIdx.x;
  const int hk = hq / kc.G, n = hq % kc.G;
  const float* base = part + (((int64_t)b * kc.Hkv + hk) * nsplit * kc.G + n) * 130;
  const int64_t stride = (int64_t)kc.G * 130;
  float M = -INFINITY;
  for (int s = 0; s < nsplit; ++s) M = fmaxf(M, base[s * stride]);
  float L = 0.f, O = 0.f;
  for (int s = 0; s < nsplit; ++s) {
    const float ms = base[s * stride];
    if (ms == -INFINITY) continue;
    const float f = ex2(ms - M);
    L = __fmaf_rn(f, base[s * stride + 1], L);
    O = __fmaf_rn(f, base[s * stride + 2 + c], O);
  }
  const float v = O / L;
  const int64_t idx = ((int64_t)b * kc.Hq + hq) * 128 + c;
  if (kc.out_fp32)
    reinterpret_cast<float*>(out)[idx] = v;
  else
    reinterpret_cast<__half*>(out)[idx] = __float2half_rn(v);
}

template <int BITS, int PI_>
cudaError_t launch_t(const KernelCfg& kc, const void* q_new, const int32_t* slots, int batch, int nsplit,
                     const CacheView& cv, void* out, float* part, const hack_debug_t* dbg, cudaStream_t st) {
  if (kc.pl.page_bytes != DecSmem<BITS, PI_>::PB) return cudaErrorInvalidValue;  // layout drift guard
  const size_t smem = sizeof(DecSmem<BITS, PI_>);
  const bool with_dbg = dbg != nullptr && (dbg->pcodes != nullptr || dbg->qk_acc != nullptr || dbg->pv_acc != nullptr);
  auto kern = with_dbg ? decode_mma_kernel<BITS, PI_, true> : decode_mma_kernel<BITS, PI_, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<dim3(batch, kc.Hkv, nsplit), kThreads, smem, st>>>(
      reinterpret_cast<const __half*>(q_new), slots, cv, kc, part, nsplit, dbg ? dbg->pcodes : nullptr,
      dbg ? dbg->pcodes_stride : 0, dbg ? dbg->qk_acc : nullptr, dbg ? dbg->pv_acc : nullptr,
      dbg ? dbg->acc_stride : 0, dbg ? dbg->acc_head : -1);
  decode_combine_kernel<<<dim3(batch, kc.Hq), 128, 0, st>>>(part, nsplit, kc, out);
  note_launch(2);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_decode_combine(const float* part, int nsplit, const KernelCfg& kc, int batch, void* out,
                                  cudaStream_t st) {
  decode_combine_kernel<<<dim3(batch, kc.Hq), 128, 0, st>>>(part, nsplit, kc, out);
  note_launch();
  return cudaGetLastError();
}

bool decode_mma_supported(const KernelCfg& kc) {
  return (kc.Pi == 32 || kc.Pi == 64 || kc.Pi == 128) && kc.d == 128 && kc.G <= 8;
}

// resident CTAs per SM of the kernel instantiation serving kc
static int dmma_resident(const KernelCfg& kc) {
  switch (kc.Pi * 8 + kc.bits) {
    case 32 * 8 + 2: return dmma_ctas<2, 32>();
    case 32 * 8 + 4: return dmma_ctas<4, 32>();
    case 64 * 8 + 2: return dmma_ctas<2, 64>();
    case 64 * 8 + 4: return dmma_ctas<4, 64>();
    case 128 * 8 + 2: return dmma_ctas<2, 128>();
    default: return dmma_ctas<4, 128>();
  }
}

int decode_nsplit(const KernelCfg& kc, int batch, int max_seqlen) {
  const int max_pages = (max_seqlen + kc.Pi - 1) / kc.Pi;
  const int units = batch * kc.Hkv;
  // aim for ~4 waves of the CTAs that are actually resident (148 SMs x 2 or 3), at least
  // ~8 pages per split (C4 b = 4: 2 resident -> 10 splits, 3.09 vs 2.87 TB/s with 14)
  int ns = (148 * dmma_resident(kc) * 4 + units - 1) / units;
  ns = max(1, min(ns, (max_pages + 7) / 8));
  return min(ns, 64);
}

size_t decode_mma_workspace(const KernelCfg& kc, int batch, int max_seqlen) {
  return (size_t)batch * kc.Hkv * decode_nsplit(kc, batch, max_seqlen) * kc.G * 130 * sizeof(float);
}

cudaError_t launch_decode_mma(const KernelCfg& kc, const void* q_new, const int32_t* slots, int batch,
                              int max_seqlen, const CacheView& cv, void* out, void* workspace,
                              const hack_debug_t* dbg, cudaStream_t st) {
  const int ns = decode_nsplit(kc, batch, max_seqlen);
  float* part = reinterpret_cast<float*>(workspace);
  switch (kc.Pi * 8 + kc.bits) {
    case 32 * 8 + 2: return launch_t<2, 32>(kc, q_new, slots, batch, ns, cv, out, part, dbg, st);
    case 32 * 8 + 4: return launch_t<4, 32>(kc, q_new, slots, batch, ns, cv, out, part, dbg, st);
    case 64 * 8 + 2: return launch_t<2, 64>(kc, q_new, slots, batch, ns, cv, out, part, dbg, st);
    case 64 * 8 + 4: return launch_t<4, 64>(kc, q_new, slots, batch, ns, cv, out, part, dbg, st);
    case 128 * 8 + 2: return launch_t<2, 128>(kc, q_new, slots, batch, ns, cv, out, part, dbg, st);
    case 128 * 8 + 4: return launch_t<4, 128>(kc, q_new, slots, batch, ns, cv, out, part, dbg, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hack
