// decode_tc.cu -- homomorphic decode attention (a9) on tcgen05 with operands in TMEM.
//
// Decode reads every cached token once per step (L_Q = 1): it must stream packed
// pages (84 B per token per KV head at b=2, Pi=64) at HBM speed.  The cost that decides
// it is CUDA-core work per page, so the kernel is organised to make that minimal:
//   grid (request, KV head, split), pages processed in PAIRS (128 tokens = MMA M):
//   warp 0      producer: both pages of a pair -> smem ring (cp.async.bulk / TMA)
//   warp 1      MMA issuer, tcgen05.mma kind::i8 with the A operand in TMEM:
//                 S^T[token][row]  = K'[token][d] . (Q' - 128)[row][d]   (M=128 tokens, N=8)
//                 O'^T[ch][row]   = V'[ch][token] . (P' - 128)[row][token] per page (M=128 ch)
//   warps 4-7   K/S warpgroup, thread = token (TMEM lane): unpacks its K row straight
//               into TMEM (tcgen05.st; no smem round trip), Eq. 4 (centered) with its own
//               per-token coefficients from fp16 meta + CACHED sums (summation
//               elimination) in registers, online softmax with warp CREDUX
//               reductions, P 8-bit RN per (row, V block) -> smem B operand
//   warps 8-11  V/O warpgroup, thread = channel (TMEM lane): unpacks its V row into TMEM,
//               O = alpha O + Eq. 4 (centered) on D' with per-channel coefficients in
//               registers; the FP16 last V block (RQE) in fp32.
// Partial (m, l, O) per split -> decode_combine_kernel (decode_mma.cu).
#include "common.cuh"
#include "internal.h"
#include "tc_common.cuh"

namespace hack {

namespace {

constexpr int PI = 64;
constexpr int NST = 3;  // page-pair stages
constexpr int kThreads = 384;

template <int BITS>
struct DtSmem {
  static constexpr int PB = BITS == 2 ? 5376 : 9728;
  uint8_t stage[NST][2][PB];
  alignas(128) uint8_t qb[8 * 128];       // (q' - 128) s8, N=8 x K=128, K-major [kc][row][16]
  alignas(128) uint8_t pb[2][2][8 * 64];  // (p' - 128) s8 per (buf, page), N=8 x K=64
  uint8_t qtmp[8][128];                   // Q' codes, natural order (staging)
  float ptl[8][PI];                       // p~ of the FP16 tail page
  float4 qconst[2][8];                    // (beta, row): aq, xq, mu_q, nrq
  float2 xw[2][4][8];                     // (parity, K/S warp, row): max S, min S (valid tokens)
  uint32_t xs[2][4][8];                   // (buf, K/S warp, row): P-code sums
  float4 rmeta[2][2][8];                  // (buf, page, row): ap, xp, mup, nrp
  float alpha[2][8];
  float lred[4][8];
  uint64_t full[NST], empty[NST], ka_ready[2], ka_free[2], s_full[2], s_free[2], va_ready[2], va_free[2],
      p_ready[2], p_free[2], d_full[2], d_free[2], m_free[2];
  uint32_t tmem_base;
};

HACK_DEV float u2f(uint32_t x) { return __int2float_rn((int)x); }

template <int BITS>
__global__ void __launch_bounds__(kThreads, 2) decode_tc_kernel(const __half* __restrict__ q_new,
                                                                const int32_t* __restrict__ slots, CacheView cv,
                                                                KernelCfg kc, float* __restrict__ part, int nsplit,
                                                                uint8_t* __restrict__ dbg_pcodes,
                                                                int64_t dbg_stride) {
  using SM = DtSmem<BITS>;
  constexpr int qkm = (1 << BITS) - 1;
  constexpr float ck = 0.5f * qkm;
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
  const int npair = (np + 1) / 2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const PageLayout PL = kc.pl;

  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      ptx::mbar_init(&sm.full[s], 1);
      ptx::mbar_init(&sm.empty[s], 256);
    }
    for (int x = 0; x < 2; ++x) {
      ptx::mbar_init(&sm.ka_ready[x], 128);
      ptx::mbar_init(&sm.ka_free[x], 1);
      ptx::mbar_init(&sm.s_full[x], 1);
      ptx::mbar_init(&sm.s_free[x], 128);
      ptx::mbar_init(&sm.va_ready[x], 128);
      ptx::mbar_init(&sm.va_free[x], 1);
      ptx::mbar_init(&sm.p_ready[x], 128);
      ptx::mbar_init(&sm.p_free[x], 1);
      ptx::mbar_init(&sm.d_full[x], 1);
      ptx::mbar_init(&sm.d_free[x], 128);
      ptx::mbar_init(&sm.m_free[x], 128);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(&sm.tmem_base, 256);
  // ---- (a3) quantize the G query rows (8-bit SR, fp32 meta): K/S warpgroup, 16 lanes/row
  if (warp >= 4 && warp < 8) {
    const int t = tid - 128;
    const int row = t >> 4, lane16 = t & 15;  // rows 0..7
    const int rr = min(row, G - 1);
    const int hq = hk * G + rr;
    const uint4 raw = reinterpret_cast<const uint4*>(q_new + ((int64_t)b * kc.Hq + hq) * 128)[lane16];
    uint64_t packed;
    float m, s;
    int sum;
    quant_row16<8, false>(raw, lane16, PI, pos, kc.seed, cv.rng_ids[slot],
                          stream_c3(kc.layer, kTagQ, kc.head_base * G + hq), kc.q_round, packed, m, s, sum);
    *reinterpret_cast<uint2*>(&sm.qtmp[row][lane16 * 8]) =
        row < G ? make_uint2((uint32_t)packed, (uint32_t)(packed >> 32)) : make_uint2(0x80808080u, 0x80808080u);
    if ((lane16 & 7) == 0) {
      const int beta = lane16 >> 3;
      const float cscale = 1.4426950408889634f / sqrtf(128.f);
      const int sqs = sum - 128 * PI;  // sum (q' - 128)
      sm.qconst[beta][row] = row < G ? make_float4(cscale * s * 0.5f, cscale * s * (float)sqs,
                                                   cscale * (m + 128.f * s), -(float)(qkm * sqs))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    ptx::named_bar_sync(1, 128);
    if (t < 64) {  // permuted s8 B operand: chunk (row n, 16-group g)
      const int n = t >> 3, g = t & 7;
      uint32_t wv[4];
#pragma unroll
      for (int x4 = 0; x4 < 4; ++x4) {
        uint32_t wd = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) wd |= (uint32_t)sm.qtmp[n][16 * g + perm_src<BITS>(4 * x4 + e)] << (8 * e);
        wv[x4] = wd ^ 0x80808080u;
      }
      *reinterpret_cast<uint4*>(sm.qb + g * 128 + n * 16) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    }
    ptx::fence_proxy_async_smem();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const uint32_t tAK = tmem, tS = tmem + 64, tAV = tmem + 96, tD = tmem + 160;

  if (warp == 0) {
    // ------------------------------------------------------------------ producer
    if (lane == 0) {
      const int32_t* bt = cv.block_table + (int64_t)slot * cv.max_pages_per_req;
      for (int u = 0; u < npair; ++u) {
        const int s = u % NST;
        const int npg = min(2, np - 2 * u);
        ptx::mbar_wait(&sm.empty[s], ((u / NST) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&sm.full[s], SM::PB * npg);
        for (int x = 0; x < npg; ++x) {
          const uint8_t* pg = cv.pages + ((int64_t)bt[p_beg + 2 * u + x] * cv.num_kv_heads + hk) * cv.page_bytes;
          ptx::bulk_g2s(sm.stage[s][x], pg, SM::PB, &sm.full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    const uint32_t idesc = ptx::idesc_u8s8(128, 8);
    const uint32_t qa = ptx::smem_u32(sm.qb);
    auto issue_pv = [&](int v) {
      const int bb = v & 1;
      ptx::mbar_wait(&sm.p_ready[bb], (v >> 1) & 1);
      ptx::mbar_wait(&sm.va_ready[bb], (v >> 1) & 1);
      ptx::mbar_wait(&sm.d_free[bb], ((v >> 1) & 1) ^ 1);
      ptx::tc_fence_after();
      if (lane == 0) {
        for (int x = 0; x < 2; ++x) {
          const int jp = p_beg + 2 * v + x;
          if (2 * v + x >= np || jp >= nfull) continue;  // absent or FP16 tail page
          const uint32_t pa = ptx::smem_u32(sm.pb[bb][x]);
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
            ptx::mma_u8_ts(tD + 16 * bb + 8 * x, tAV + 32 * bb + 16 * x + 8 * ks,
                           ptx::smem_desc_kmajor(pa + 256 * ks, 128, 512), idesc, ks > 0);
        }
        ptx::mma_commit(&sm.d_full[bb]);
        ptx::mma_commit(&sm.p_free[bb]);
        ptx::mma_commit(&sm.va_free[bb]);
      }
      __syncwarp();
    };
    for (int u = 0; u < npair; ++u) {
      const int bu = u & 1;
      ptx::mbar_wait(&sm.ka_ready[bu], (u >> 1) & 1);
      ptx::mbar_wait(&sm.s_free[bu], ((u >> 1) & 1) ^ 1);
      ptx::tc_fence_after();
      if (lane == 0) {
#pragma unroll
        for (int beta = 0; beta < 2; ++beta)
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const int kg = 2 * beta + ks;  // 32-channel K step
            ptx::mma_u8_ts(tS + 16 * bu + 8 * beta, tAK + 32 * bu + 8 * kg,
                           ptx::smem_desc_kmajor(qa + 256 * kg, 128, 1024), idesc, ks > 0);
          }
        ptx::mma_commit(&sm.s_full[bu]);
        ptx::mma_commit(&sm.ka_free[bu]);
      }
      __syncwarp();
      if (u >= 1) issue_pv(u - 1);
    }
    if (npair >= 1) issue_pv(npair - 1);
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------------ K/S warpgroup
    const int t = tid - 128;                 // token slot in the pair = TMEM lane
    const int wq = warp - 4;                 // 0,1: page 0; 2,3: page 1
    const int x = t >> 6, row = t & 63;      // page of the pair, token row in the page
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    float m_run[8], l_run[8];
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      m_run[n] = -INFINITY;
      l_run[n] = 0.f;
    }
    // stage pair u: unpack this token's K row straight into TMEM (A operand, 4 codes per
    // column) and compute its Eq. 4 coefficients (cached sums, SE).
    auto stage_k = [&](int u, float (&sk)[2], float (&mu)[2], float (&yk)[2]) {
      const int s = u % NST, bu = u & 1;
      const int jp = p_beg + 2 * u + x;
      const bool present = (2 * u + x) < np;
      const bool valid = present && jp * PI + row < len;
      ptx::mbar_wait(&sm.full[s], (u / NST) & 1);
      ptx::mbar_wait(&sm.ka_free[bu], ((u >> 1) & 1) ^ 1);
      const uint8_t* pg = sm.stage[s][x];
      {
        uint32_t wk[4 * BITS];
        const uint4* src = reinterpret_cast<const uint4*>(pg + PL.k_codes + row * (128 * BITS / 8));
#pragma unroll
        for (int h = 0; h < BITS; ++h) {
          const uint4 pw = present ? src[h] : make_uint4(0u, 0u, 0u, 0u);
          wk[4 * h] = pw.x; wk[4 * h + 1] = pw.y; wk[4 * h + 2] = pw.z; wk[4 * h + 3] = pw.w;
        }
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t a[16];
#pragma unroll
          for (int wi = 0; wi < 2 * BITS; ++wi) {
            const uint32_t wd = wk[2 * BITS * half + wi];
            if (BITS == 2) {
              const uint4 q4 = unpack16_2b(wd);
              a[4 * wi] = q4.x; a[4 * wi + 1] = q4.y; a[4 * wi + 2] = q4.z; a[4 * wi + 3] = q4.w;
            } else {
              const uint2 q2 = unpack8_4b(wd);
              a[2 * wi] = q2.x; a[2 * wi + 1] = q2.y;
            }
          }
          ptx::tmem_st16(tAK + 32 * bu + 16 * half + lane_base, a);
        }
      }
#pragma unroll
      for (int beta = 0; beta < 2; ++beta) {
        sk[beta] = mu[beta] = yk[beta] = 0.f;
        if (valid) {
          const __half2 mh = reinterpret_cast<const __half2*>(pg + PL.k_meta)[2 * row + beta];
          const float m = __low2float(mh), s2 = __high2float(mh);
          const int sum = load_sum(pg + PL.k_sums, 2 * row + beta, PL.sum_bytes);
          sk[beta] = s2;
          mu[beta] = m + ck * s2;
          yk[beta] = s2 * ((float)sum - ck * PI) + PI * mu[beta];
        }
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&sm.ka_ready[bu]);
      ptx::mbar_arrive(&sm.empty[s]);  // this warpgroup is done with the stage
    };
    float sk[2], mu[2], yk[2];
#pragma unroll 1
    for (int u = 0; u < npair; ++u) {
      const int bu = u & 1;
      const int jp = p_beg + 2 * u + x;                 // page index in the request
      const bool present = (2 * u + x) < np;
      const int tok = jp * PI + row;
      const bool valid = present && tok < len;
      const bool committed = present && jp < nfull;
      stage_k(u, sk, mu, yk);
      // -- S for this token, all rows
      ptx::mbar_wait(&sm.s_full[bu], (u >> 1) & 1);
      ptx::tc_fence_after();
      uint32_t d0[8], d1[8];
      ptx::tmem_ld8(tS + 16 * bu + lane_base, d0);
      ptx::tmem_ld8(tS + 16 * bu + 8 + lane_base, d1);
      ptx::tmem_wait_ld();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&sm.s_free[bu]);
      float sv[8];
#pragma unroll
      for (int n = 0; n < 8; n += 2) {
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int beta = 0; beta < 2; ++beta) {
          const float4 c0 = sm.qconst[beta][n], c1 = sm.qconst[beta][n + 1];
          const uint32_t* d = beta ? d1 : d0;
          const float2 e = ptx::ffma2(make_float2(2.f, 2.f), make_float2(u2f(d[n]), u2f(d[n + 1])),
                                      make_float2(c0.w, c1.w));  // 2 x centered int dot (exact)
          const float2 g = ptx::fmul2(make_float2(sk[beta], sk[beta]), e);
          acc = ptx::ffma2(make_float2(c0.x, c1.x), g,
                           ptx::ffma2(make_float2(c0.y, c1.y), make_float2(mu[beta], mu[beta]),
                                      ptx::ffma2(make_float2(c0.z, c1.z), make_float2(yk[beta], yk[beta]), acc)));
        }
        sv[n] = valid ? acc.x : -INFINITY;
        sv[n + 1] = valid ? acc.y : -INFINITY;
      }
      // -- row max over the pair; per-page min/max (warps 0,1 -> page 0; 2,3 -> page 1)
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        if (n < G) {
          const float mxw = ptx::redux_max(sv[n]);
          const float mnw = ptx::redux_min(valid ? sv[n] : INFINITY);
          if (lane == 0) sm.xw[u & 1][wq][n] = make_float2(mxw, mnw);
        }
      }
      ptx::named_bar_sync(1, 128);
      ptx::mbar_wait(&sm.m_free[bu], ((u >> 1) & 1) ^ 1);  // V/O done with pair u-2's row meta
      float p[8];
      uint32_t code[8];
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        p[n] = 0.f;
        code[n] = 0;
        if (n >= G) continue;
        const float2 a0 = sm.xw[u & 1][0][n], a1 = sm.xw[u & 1][1][n], a2 = sm.xw[u & 1][2][n],
                     a3 = sm.xw[u & 1][3][n];
        const float mx = fmaxf(fmaxf(a0.x, a1.x), fmaxf(a2.x, a3.x));
        const float m_new = fmaxf(m_run[n], mx);
        const float al = (m_run[n] == -INFINITY) ? 0.f : ex2(m_run[n] - m_new);
        p[n] = valid ? ex2(sv[n] - m_new) : 0.f;
        l_run[n] = fmaf(l_run[n], al, p[n]);
        m_run[n] = m_new;
        if (t == 0) sm.alpha[bu][n] = al;
        if (committed) {
          // (a6) P' per (row, V block) -- this page's min/max of p~ from its score min/max
          const float pmx = x ? fmaxf(a2.x, a3.x) : fmaxf(a0.x, a1.x);
          const float pmn = x ? fminf(a2.y, a3.y) : fminf(a0.y, a1.y);
          const float lo = ex2(pmn - m_new), hi = ex2(pmx - m_new);
          QMeta pm = meta_fp32(lo, hi, 255);
          if (!(pm.s > 1e-30f)) {
            pm.s = 0.f;
            pm.inv = 0.f;
          }
          const float y = fmaf(p[n], pm.inv, -lo * pm.inv) + 12582912.f;
          code[n] = __float_as_uint(y) & 0xFFu;
          if (row == 0) sm.rmeta[bu][x][n] = make_float4(0.5f * pm.s, pm.s, pm.m + 128.f * pm.s, 0.f);
        }
      }
      if (committed) {
        ptx::mbar_wait(&sm.p_free[bu], ((u >> 1) & 1) ^ 1);
        // K position of this token inside its 16-group (V is unpacked in the pi order)
        const int tp = row & 15;
        const int posn = BITS == 2 ? (row & ~15) + 4 * (tp & 3) + (tp >> 2)
                                   : (row & ~15) + 8 * (tp >> 3) + 4 * (tp & 1) + ((tp >> 1) & 3);
        const int off = (posn >> 4) * 128 + (posn & 15);  // [kc][n][16]
#pragma unroll
        for (int n = 0; n < 8; ++n) sm.pb[bu][x][off + 16 * n] = (uint8_t)(code[n] ^ 0x80u);
        if (dbg_pcodes != nullptr)
          for (int n = 0; n < G; ++n) dbg_pcodes[((int64_t)b * kc.Hq + hk * G + n) * dbg_stride + tok] = (uint8_t)code[n];
#pragma unroll
        for (int n = 0; n < 8; ++n)
          if (n < G) {
            const uint32_t sw = ptx::redux_add(code[n]);
            if (lane == 0) sm.xs[bu][wq][n] = sw;
          }
        ptx::fence_proxy_async_smem();
      } else if (present) {
#pragma unroll
        for (int n = 0; n < 8; ++n) sm.ptl[n][row] = p[n];  // FP16 tail page (RQE)
      }
      ptx::mbar_arrive(&sm.p_ready[bu]);
    }
    // -- final l per row: sum over the 128 token slots
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      float v = l_run[n];
#pragma unroll
      for (int o2 = 16; o2; o2 >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o2);
      if (lane == 0) sm.lred[wq][n] = v;
    }
    ptx::named_bar_sync(1, 128);
    if (t < G) {
      float* dst = part + ((((int64_t)b * kc.Hkv + hk) * nsplit + split) * G + t) * 130;
      dst[0] = np > 0 ? m_run[t] : -INFINITY;
      dst[1] = sm.lred[0][t] + sm.lred[1][t] + sm.lred[2][t] + sm.lred[3][t];
    }
  } else if (warp >= 8) {
    // ------------------------------------------------------------------ V/O warpgroup
    const int c = tid - 256;  // output channel = TMEM lane
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    float o[8];
#pragma unroll
    for (int n = 0; n < 8; ++n) o[n] = 0.f;
    // stage pair u: unpack this channel's V rows (both pages) into TMEM and compute the
    // per-channel Eq. 4 coefficients.
    auto stage_v = [&](int u, bool (&comm)[2], float (&svv)[2], float (&mu)[2], float (&yv)[2]) {
      const int s = u % NST, bu = u & 1;
      ptx::mbar_wait(&sm.full[s], (u / NST) & 1);
      ptx::mbar_wait(&sm.va_free[bu], ((u >> 1) & 1) ^ 1);
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const int jp = p_beg + 2 * u + x;
        comm[x] = (2 * u + x) < np && jp < nfull;
        svv[x] = mu[x] = yv[x] = 0.f;
        uint32_t a[16];
        const uint8_t* pg = sm.stage[s][x];
        if (comm[x]) {
          const uint4* src = reinterpret_cast<const uint4*>(pg + PL.v_codes + c * (PI * BITS / 8));
#pragma unroll
          for (int h = 0; h < BITS / 2; ++h) {
            const uint4 pw = src[h];
            const uint32_t w4[4] = {pw.x, pw.y, pw.z, pw.w};
#pragma unroll
            for (int wi = 0; wi < 4; ++wi) {
              if (BITS == 2) {
                const uint4 q4 = unpack16_2b(w4[wi]);
                a[4 * wi] = q4.x; a[4 * wi + 1] = q4.y; a[4 * wi + 2] = q4.z; a[4 * wi + 3] = q4.w;
              } else {
                const uint2 q2 = unpack8_4b(w4[wi]);
                a[8 * h + 2 * wi] = q2.x; a[8 * h + 2 * wi + 1] = q2.y;
              }
            }
          }
          const __half2 mh = reinterpret_cast<const __half2*>(pg + PL.v_meta)[c];
          const float m = __low2float(mh), s2 = __high2float(mh);
          const int sum = load_sum(pg + PL.v_sums, c, PL.sum_bytes);  // cached sum (SE)
          svv[x] = s2;
          mu[x] = m + ck * s2;
          yv[x] = s2 * ((float)sum - ck * PI) + PI * mu[x];
        } else {
#pragma unroll
          for (int wi = 0; wi < 16; ++wi) a[wi] = 0u;
        }
        ptx::tmem_st16(tAV + 32 * bu + 16 * x + lane_base, a);
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&sm.va_ready[bu]);
      ptx::mbar_arrive(&sm.empty[s]);
    };
    bool comm[2];
    float svv[2], mu[2], yv[2];
#pragma unroll 1
    for (int u = 0; u < npair; ++u) {
      const int bu = u & 1;
      stage_v(u, comm, svv, mu, yv);
      // -- O update for this pair
      ptx::mbar_wait(&sm.p_ready[bu], (u >> 1) & 1);
      const bool anyc = comm[0] || comm[1];
      uint32_t dd[2][8];
      if (anyc) {
        ptx::mbar_wait(&sm.d_full[bu], (u >> 1) & 1);
        ptx::tc_fence_after();
        ptx::tmem_ld8(tD + 16 * bu + lane_base, dd[0]);
        ptx::tmem_ld8(tD + 16 * bu + 8 + lane_base, dd[1]);
        ptx::tmem_wait_ld();
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&sm.d_free[bu]);
#pragma unroll
      for (int n = 0; n < 8; ++n) o[n] *= sm.alpha[bu][n];
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        if (comm[x]) {
#pragma unroll
          for (int n = 0; n < 8; ++n) {
            if (n >= G) continue;
            const float4 rm = sm.rmeta[bu][x][n];
            const int sps = (int)(sm.xs[bu][2 * x][n] + sm.xs[bu][2 * x + 1][n]) - 128 * PI;  // sum (p' - 128)
            const float e = fmaf(2.f, u2f(dd[x][n]), -(float)(qkm * sps));  // 2 x centered int dot
            o[n] += rm.x * (svv[x] * e) + rm.y * (float)sps * mu[x] + rm.z * yv[x];
          }
        } else if ((2 * u + x) < np) {
          // FP16 last V block (RQE): O += sum_t p~_t v_t (last pair of the request)
          const int jp = p_beg + 2 * u + x;
          const int nk = len - jp * PI;
          const __half* tail = reinterpret_cast<const __half*>(cv.v_tail) + ((int64_t)slot * kc.Hkv + hk) * PI * 128;
          for (int tt = 0; tt < nk; ++tt) {
            const float v = __half2float(tail[tt * 128 + c]);
#pragma unroll
            for (int n = 0; n < 8; ++n) o[n] = fmaf(sm.ptl[n][tt], v, o[n]);
          }
        }
      }
      ptx::mbar_arrive(&sm.m_free[bu]);  // alpha / rmeta / xs of this pair consumed
    }
    for (int n = 0; n < G; ++n)
      part[((((int64_t)b * kc.Hkv + hk) * nsplit + split) * G + n) * 130 + 2 + c] = o[n];
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem, 256);
}

template <int BITS>
cudaError_t launch_t(const KernelCfg& kc, const void* q_new, const int32_t* slots, int batch, int nsplit,
                     const CacheView& cv, void* out, float* part, const hack_debug_t* dbg, cudaStream_t st) {
  const size_t smem = sizeof(DtSmem<BITS>);
  auto kern = decode_tc_kernel<BITS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<dim3(batch, kc.Hkv, nsplit), kThreads, smem, st>>>(reinterpret_cast<const __half*>(q_new), slots, cv, kc,
                                                            part, nsplit, dbg ? dbg->pcodes : nullptr,
                                                            dbg ? dbg->pcodes_stride : 0);
  note_launch();
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_decode_combine(const float* part, int nsplit, const KernelCfg& kc, int batch, void* out,
                                  cudaStream_t st);
int decode_nsplit(const KernelCfg& kc, int batch, int max_seqlen);

cudaError_t launch_decode_tc(const KernelCfg& kc, const void* q_new, const int32_t* slots, int batch,
                             int max_seqlen, const CacheView& cv, void* out, void* workspace,
                             const hack_debug_t* dbg, cudaStream_t st) {
  const int ns = decode_nsplit(kc, batch, max_seqlen);
  float* part = reinterpret_cast<float*>(workspace);
  cudaError_t e = kc.bits == 2 ? launch_t<2>(kc, q_new, slots, batch, ns, cv, out, part, dbg, st)
                               : launch_t<4>(kc, q_new, slots, batch, ns, cv, out, part, dbg, st);
  if (e != cudaSuccess) return e;
  return launch_decode_combine(part, ns, kc, batch, out, st);
}

}  // namespace hack
