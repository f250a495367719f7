// prefill_tc.cu -- homomorphic prefill attention on the 5th-gen tensor cores (a3-a7).
//
// One CTA = 128 query rows of one query head, warp-specialised (12 warps):
//   warp 0     producer: whole packed pages (K' + V' codes, fp16 meta, cached sums;
//              DESIGN.md "HBM layout") -> smem ring via cp.async.bulk (TMA) + mbarrier
//   warp 1     MMA issuer: tcgen05.mma kind::i8 (u8 x u8 -> s32, accumulators in TMEM)
//                QK: per d-block beta D_beta[128 x 64] = Q'_beta K'_beta^T
//                PV: D'[128 x 128] = P'_j V'_j^T per 64-token V block
//   warps 2-3  unpack: 2/4-bit codes -> u8 K-major UMMA tiles (tc_common.cuh) + per-key /
//              per-channel Eq. 4 coefficients from the page meta and CACHED sums
//   warps 4-7  softmax WG (thread = query row, TMEM lanes): in-kernel Q quantization
//              (a3, 8-bit SR); S = centered Eq. 4 (a4) x log2e/sqrt(d);
//              causal online softmax (a5); P 8-bit RN per (row, V block) (a6)
//   warps 8-11 correction WG (thread = row): O = alpha O + centered Eq. 4 on D' (a7);
//              the FP16 last V block (RQE) as fp32 FMAs; O / l; store.
// TMEM (512 columns): S (2 x 64) | D'[2] (2 x 128) | spare.  The softmax WG pulls the
// whole S tile into registers and frees TMEM immediately, so QK(j+1) overlaps
// softmax(j); D' is double-buffered so PV(j+1) overlaps correction(j).
// Pi = 64 (C2); other partitions use prefill_simt.cu.
#include "common.cuh"
#include "internal.h"
#include "tc_common.cuh"

namespace hack {

namespace {

constexpr int PI = 64;
constexpr int BM = 128;
constexpr int BN = 64;
constexpr int NS = 4;  // page stages
constexpr int kThreads = 384;

template <int BITS>
struct TcSmem {
  static constexpr int PB = BITS == 2 ? 5376 : 9728;  // page bytes (d=128, Pi=64)
  uint8_t stage[NS][PB];
  alignas(128) uint8_t q[BM * 128];       // Q' K-major, SBO 1024
  alignas(128) uint8_t k[2][BN * 128];    // K' K-major, SBO 1024
  alignas(128) uint8_t v[2][128 * BN];    // V' K-major (keys = K), SBO 512
  alignas(128) uint8_t p[2][BM * BN];     // P' K-major, SBO 512
  float4 kconst[2][BN * 2];               // per (key, beta): sk, mu_k, y_k, r_k
  float4 vconst[2][128];                  // per channel: sv, mu_v, y_v, r_v
  float4 rowmeta[2][BM];                  // per row: alpha, ap, xp, mup
  float rowrp[2][BM];                     // per row: rp
  float ptail[BM][BN + 1];                // p~ of the FP16 tail tile
  float lfinal[BM];
  uint64_t full[NS], empty[NS], kv_ready[2], kv_free[2], s_full, s_free, p_ready[2], p_free[2], d_full[2],
      d_free[2], q_ready;
  uint32_t tmem_base;
};

HACK_DEV float u2f(uint32_t x) { return __int2float_rn((int)x); }

template <int BITS>
__global__ void __launch_bounds__(kThreads, 1) prefill_tc_kernel(
    const __half* __restrict__ q, const int32_t* __restrict__ cu_seqlens, const int32_t* __restrict__ slots,
    CacheView cv, KernelCfg kc, void* __restrict__ out, uint8_t* __restrict__ dbg_pcodes, int64_t dbg_stride) {
  using SM = TcSmem<BITS>;
  constexpr int qkm = (1 << BITS) - 1;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);

  const int b = blockIdx.z, hq = blockIdx.y;
  const int start = cu_seqlens[b], L = cu_seqlens[b + 1] - start;
  const int nqt = (L + BM - 1) / BM;
  if ((int)blockIdx.x >= nqt) return;
  const int qt = nqt - 1 - blockIdx.x;  // heavy (long causal rows) tiles first
  const int i0 = qt * BM;
  const int slot = slots[b];
  const int hk = hq / kc.G;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nkt = min((i0 + BM - 1) / BN, (L - 1) / BN) + 1;  // key tiles (causal)
  const int nfull = L / PI;                                    // committed V blocks
  const PageLayout PL = kc.pl;

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      ptx::mbar_init(&sm.full[s], 1);
      ptx::mbar_init(&sm.empty[s], 64);
    }
    for (int x = 0; x < 2; ++x) {
      ptx::mbar_init(&sm.kv_ready[x], 64);
      ptx::mbar_init(&sm.kv_free[x], 128);
      ptx::mbar_init(&sm.p_ready[x], 128);
      ptx::mbar_init(&sm.p_free[x], 1);
      ptx::mbar_init(&sm.d_full[x], 1);
      ptx::mbar_init(&sm.d_free[x], 128);
    }
    ptx::mbar_init(&sm.s_full, 1);
    ptx::mbar_init(&sm.s_free, 128);
    ptx::mbar_init(&sm.q_ready, 128);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(&sm.tmem_base, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const uint32_t tS = tmem;            // columns 0..127: D_0 | D_1
  const uint32_t tD0 = tmem + 128;     // D'[0] columns 128..255, D'[1] 256..383

  if (warp == 0) {
    // ------------------------------------------------------------------ producer
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    if (lane == 0) {
      const int32_t* bt = cv.block_table + (int64_t)slot * cv.max_pages_per_req;
      for (int j = 0; j < nkt; ++j) {
        const int s = j % NS;
        ptx::mbar_wait(&sm.empty[s], ((j / NS) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&sm.full[s], SM::PB);
        const uint8_t* pg = cv.pages + ((int64_t)bt[j] * cv.num_kv_heads + hk) * cv.page_bytes;
        ptx::bulk_g2s(sm.stage[s], pg, SM::PB, &sm.full[s]);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    const uint32_t idesc_qk = ptx::idesc_u8(BM, BN), idesc_pv = ptx::idesc_u8(BM, 128);
    const uint32_t qa = ptx::smem_u32(sm.q);
    auto issue_pv = [&](int jj) {
      if (jj >= nfull) return;  // FP16 tail block: no integer PV (RQE)
      const int bb = jj & 1;
      ptx::mbar_wait(&sm.p_ready[bb], (jj >> 1) & 1);
      ptx::mbar_wait(&sm.d_free[bb], ((jj >> 1) & 1) ^ 1);
      ptx::tc_fence_after();
      if (lane == 0) {
        const uint32_t pa = ptx::smem_u32(sm.p[bb]), va = ptx::smem_u32(sm.v[bb]);
        for (int ks = 0; ks < BN / 32; ++ks)
          ptx::mma_u8(tD0 + 128 * bb, ptx::smem_desc_kmajor(pa + ks * 256, 128, 512),
                      ptx::smem_desc_kmajor(va + ks * 256, 128, 512), idesc_pv, ks > 0);
        ptx::mma_commit(&sm.d_full[bb]);
        ptx::mma_commit(&sm.p_free[bb]);
      }
      __syncwarp();
    };
    ptx::mbar_wait(&sm.q_ready, 0);
    for (int j = 0; j < nkt; ++j) {
      const int bj = j & 1;
      ptx::mbar_wait(&sm.kv_ready[bj], (j >> 1) & 1);
      ptx::mbar_wait(&sm.s_free, (j & 1) ^ 1);
      ptx::tc_fence_after();
      if (lane == 0) {
        const uint32_t ka = ptx::smem_u32(sm.k[bj]);
        for (int beta = 0; beta < 2; ++beta)
          for (int ks = 0; ks < PI / 32; ++ks) {
            const uint32_t koff = (uint32_t)(beta * 4 + ks * 2) * 128;  // 16-byte K chunks
            ptx::mma_u8(tS + 64 * beta, ptx::smem_desc_kmajor(qa + koff, 128, 1024),
                        ptx::smem_desc_kmajor(ka + koff, 128, 1024), idesc_qk, ks > 0);
          }
        ptx::mma_commit(&sm.s_full);
      }
      __syncwarp();
      if (j >= 1) issue_pv(j - 1);
    }
    issue_pv(nkt - 1);
  } else if (warp < 4) {
    // ------------------------------------------------------------------ unpack
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    const int ut = tid - 64;  // 0..63
    for (int j = 0; j < nkt; ++j) {
      const int s = j % NS, bj = j & 1;
      ptx::mbar_wait(&sm.full[s], (j / NS) & 1);
      ptx::mbar_wait(&sm.kv_free[bj], ((j >> 1) & 1) ^ 1);
      const uint8_t* pg = sm.stage[s];
      const int nk = min(BN, L - j * BN);
      // K' codes [64 keys][128 ch] -> K-major tile (pi permutation inside 16-groups)
      constexpr int kwords = BN * 128 * BITS / 32;
      const uint32_t* kw = reinterpret_cast<const uint32_t*>(pg + PL.k_codes);
      for (int w = ut; w < kwords; w += 64) {
        if (BITS == 2) {
          const int key = w >> 3, wi = w & 7;
          *reinterpret_cast<uint4*>(sm.k[bj] + kmaj_off(key, 16 * wi, 1024)) = unpack16_2b(kw[w]);
        } else {
          const int key = w >> 4, wi = w & 15;
          *reinterpret_cast<uint2*>(sm.k[bj] + kmaj_off(key, 8 * wi, 1024)) = unpack8_4b(kw[w]);
        }
      }
      for (int e = ut; e < BN * 2; e += 64) {  // (key, beta)
        const int key = e >> 1;
        float4 c4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (key < nk) {
          const __half2 mh = reinterpret_cast<const __half2*>(pg + PL.k_meta)[e];
          const float m = __low2float(mh), s2 = __high2float(mh);
          const int sum = load_sum(pg + PL.k_sums, e, PL.sum_bytes);  // cached sum (SE)
          const float mu = m + 0.5f * qkm * s2;
          c4 = make_float4(s2, mu, s2 * ((float)sum - 0.5f * qkm * PI) + PI * mu, (float)(510 * sum));
        }
        sm.kconst[bj][e] = c4;
      }
      if (j < nfull) {
        constexpr int vwords = 128 * BN * BITS / 32;
        const uint32_t* vw = reinterpret_cast<const uint32_t*>(pg + PL.v_codes);
        for (int w = ut; w < vwords; w += 64) {
          if (BITS == 2) {
            const int ch = w >> 2, wi = w & 3;
            *reinterpret_cast<uint4*>(sm.v[bj] + kmaj_off(ch, 16 * wi, 512)) = unpack16_2b(vw[w]);
          } else {
            const int ch = w >> 3, wi = w & 7;
            *reinterpret_cast<uint2*>(sm.v[bj] + kmaj_off(ch, 8 * wi, 512)) = unpack8_4b(vw[w]);
          }
        }
        for (int c = ut; c < 128; c += 64) {
          const __half2 mh = reinterpret_cast<const __half2*>(pg + PL.v_meta)[c];
          const float m = __low2float(mh), s2 = __high2float(mh);
          const int sum = load_sum(pg + PL.v_sums, c, PL.sum_bytes);  // cached sum (SE)
          const float mu = m + 0.5f * qkm * s2;
          sm.vconst[bj][c] = make_float4(s2, mu, s2 * ((float)sum - 0.5f * qkm * PI) + PI * mu, (float)(510 * sum));
        }
      }
      ptx::fence_proxy_async_smem();
      ptx::mbar_arrive(&sm.kv_ready[bj]);
      ptx::mbar_arrive(&sm.empty[s]);
    }
  } else if (warp < 8) {
    // ------------------------------------------------------------------ softmax WG
    const int r = tid - 128;
    const int i = min(i0 + r, L - 1);  // this thread's query position (padding rows clamp)
    const float cscale = 1.4426950408889634f / sqrtf(128.f);
    const uint32_t rng_id = cv.rng_ids[slot];
    const uint32_t c3 = stream_c3(kc.layer, kTagQ, kc.head_base * kc.G + hq);
    float aq[2], xq[2], muq[2], rqf[2];
    // (a3) quantize this row of Q: 8-bit, fp32 meta, SR (same op sequence as quant_row16)
    {
      const uint4* qrow = reinterpret_cast<const uint4*>(q + ((int64_t)(start + i) * kc.Hq + hq) * 128);
      for (int beta = 0; beta < 2; ++beta) {
        float x[64];
#pragma unroll
        for (int v8 = 0; v8 < 8; ++v8) {
          const uint4 raw = qrow[beta * 8 + v8];
          const __half* hh = reinterpret_cast<const __half*>(&raw);
#pragma unroll
          for (int e = 0; e < 8; ++e) x[v8 * 8 + e] = __half2float(hh[e]);
        }
        float lo = x[0], hi = x[0];
#pragma unroll
        for (int e = 1; e < 64; ++e) {
          lo = fminf(lo, x[e]);
          hi = fmaxf(hi, x[e]);
        }
        const QMeta qm = meta_fp32(lo, hi, 255);
        uint8_t cds[64];
        int sum = 0;
#pragma unroll
        for (int e4 = 0; e4 < 16; ++e4) {
          int cc[4];
          if (kc.q_round == HACK_ROUND_STOCHASTIC) {
            const uint64_t n = ((uint64_t)i * 128u + (uint64_t)(beta * 64 + e4 * 4)) >> 2;
            const Philox4 rr = philox_block(kc.seed, rng_id, c3, n);
            cc[0] = quant_sr(x[e4 * 4 + 0], qm, u24(rr.x), 255);
            cc[1] = quant_sr(x[e4 * 4 + 1], qm, u24(rr.y), 255);
            cc[2] = quant_sr(x[e4 * 4 + 2], qm, u24(rr.z), 255);
            cc[3] = quant_sr(x[e4 * 4 + 3], qm, u24(rr.w), 255);
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) cc[e] = quant_rn(x[e4 * 4 + e], qm, 255);
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            cds[e4 * 4 + e] = (uint8_t)cc[e];
            sum += cc[e];
          }
        }
        // store in the K-unpack permutation: chunk g byte p <- channel 16g + perm_src(p)
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          uint32_t wv[4];
#pragma unroll
          for (int x4 = 0; x4 < 4; ++x4) {
            uint32_t w = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) w |= (uint32_t)cds[16 * g + perm_src<BITS>(4 * x4 + e)] << (8 * e);
            wv[x4] = w;
          }
          *reinterpret_cast<uint4*>(sm.q + kmaj_off(r, beta * 64 + 16 * g, 1024)) =
              make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
        aq[beta] = cscale * qm.s * 0.25f;
        xq[beta] = cscale * qm.s * ((float)sum - 127.5f * PI);
        muq[beta] = cscale * (qm.m + 127.5f * qm.s);
        rqf[beta] = (float)(2 * qkm * sum - PI * 255 * qkm);
      }
      ptx::fence_proxy_async_smem();
      ptx::mbar_arrive(&sm.q_ready);
    }
    float m_run = -INFINITY, l_run = 0.f;
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    for (int j = 0; j < nkt; ++j) {
      const int bj = j & 1, t0 = j * BN;
      ptx::mbar_wait(&sm.s_full, j & 1);
      ptx::tc_fence_after();
      float s[BN];
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t d0[32], d1[32];
        ptx::tmem_ld32(tS + lane_base + 32 * half, d0);
        ptx::tmem_ld32(tS + lane_base + 64 + 32 * half, d1);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          const int kk = 32 * half + t;
          const float4 k0 = sm.kconst[bj][2 * kk], k1 = sm.kconst[bj][2 * kk + 1];
          const float e0 = fmaf(4.f, u2f(d0[t]), -(rqf[0] + k0.w));  // 4 x centered int dot, exact
          const float e1 = fmaf(4.f, u2f(d1[t]), -(rqf[1] + k1.w));
          float acc = aq[0] * (k0.x * e0) + xq[0] * k0.y + muq[0] * k0.z;
          acc += aq[1] * (k1.x * e1) + xq[1] * k1.y + muq[1] * k1.z;
          s[kk] = (t0 + kk <= i) ? acc : -INFINITY;  // causal mask (R8)
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&sm.s_free);  // S columns may be overwritten by QK(j+1)
      float mx = -INFINITY, mn = INFINITY;
      bool masked = false;
#pragma unroll
      for (int kk = 0; kk < BN; ++kk) {
        mx = fmaxf(mx, s[kk]);
        if (s[kk] == -INFINITY)
          masked = true;
        else
          mn = fminf(mn, s[kk]);
      }
      const float m_new = fmaxf(m_run, mx);
      const float al = (m_run == -INFINITY) ? 0.f : ex2(m_run - m_new);
      float lsum = 0.f;
#pragma unroll
      for (int kk = 0; kk < BN; ++kk) {
        s[kk] = (s[kk] == -INFINITY) ? 0.f : ex2(s[kk] - m_new);  // p~ (unnormalised)
        lsum += s[kk];
      }
      l_run = l_run * al + lsum;
      m_run = m_new;
      if (j < nfull) {
        // (a6) P' per (row, V block): 8-bit RN on p~ (codes invariant to the row scale)
        const float lo = masked ? 0.f : ex2(mn - m_new);
        const float hi = ex2(mx - m_new);
        QMeta pm = meta_fp32(lo, hi, 255);
        if (!(pm.s > 1e-30f)) pm.s = 0.f;
        ptx::mbar_wait(&sm.p_free[bj], ((j >> 1) & 1) ^ 1);
        int sum = 0;
        uint32_t cw[BN / 4];
#pragma unroll
        for (int x4 = 0; x4 < BN / 4; ++x4) {
          uint32_t w = 0;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int pos = 4 * x4 + e;                              // byte position in P' row
            const int key = 16 * (pos >> 4) + perm_src<BITS>(pos & 15);  // key it holds
            const int code = quant_rn(s[key], pm, 255);
            sum += code;
            w |= (uint32_t)code << (8 * e);
          }
          cw[x4] = w;
        }
#pragma unroll
        for (int g = 0; g < BN / 16; ++g)
          *reinterpret_cast<uint4*>(sm.p[bj] + kmaj_off(r, 16 * g, 512)) =
              make_uint4(cw[4 * g], cw[4 * g + 1], cw[4 * g + 2], cw[4 * g + 3]);
        if (dbg_pcodes != nullptr && i0 + r < L) {
          uint8_t* dp = dbg_pcodes + ((int64_t)(start + i0 + r) * kc.Hq + hq) * dbg_stride + t0;
#pragma unroll
          for (int pos = 0; pos < BN; ++pos)
            dp[16 * (pos >> 4) + perm_src<BITS>(pos & 15)] = (uint8_t)((cw[pos >> 2] >> (8 * (pos & 3))) & 0xFF);
        }
        sm.rowmeta[bj][r] = make_float4(al, pm.s * 0.25f, pm.s * ((float)sum - 127.5f * PI), pm.m + 127.5f * pm.s);
        sm.rowrp[bj][r] = (float)(2 * qkm * sum - PI * 255 * qkm);
        ptx::fence_proxy_async_smem();
      } else {
#pragma unroll
        for (int kk = 0; kk < BN; ++kk) sm.ptail[r][kk] = s[kk];
        sm.rowmeta[bj][r] = make_float4(al, 0.f, 0.f, 0.f);
      }
      ptx::mbar_arrive(&sm.p_ready[bj]);
    }
    sm.lfinal[r] = l_run;
    ptx::named_bar_sync(1, 256);
  } else {
    // ------------------------------------------------------------------ correction WG
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
    const int r = tid - 256;
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    float o[128];
#pragma unroll
    for (int c = 0; c < 128; ++c) o[c] = 0.f;
    const int T = L - nfull * PI;
    for (int j = 0; j < nkt; ++j) {
      const int bj = j & 1;
      ptx::mbar_wait(&sm.p_ready[bj], (j >> 1) & 1);
      const float4 rm = sm.rowmeta[bj][r];
      if (j < nfull) {
        ptx::mbar_wait(&sm.d_full[bj], (j >> 1) & 1);
        ptx::mbar_wait(&sm.kv_ready[bj], (j >> 1) & 1);
        ptx::tc_fence_after();
        const float rp = sm.rowrp[bj][r];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t d[32];
          ptx::tmem_ld32(tD0 + 128 * bj + lane_base + 32 * cc, d);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const float4 v4 = sm.vconst[bj][32 * cc + c];
            const float e = fmaf(4.f, u2f(d[c]), -(rp + v4.w));  // 4 x centered int dot, exact
            o[32 * cc + c] = fmaf(rm.x, o[32 * cc + c], rm.y * (v4.x * e) + rm.z * v4.y + rm.w * v4.z);
          }
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&sm.d_free[bj]);
      } else {
        // FP16 last V block (RQE): O = alpha O + sum_t p~_t v_t in fp32
        const __half* tail = reinterpret_cast<const __half*>(cv.v_tail) + ((int64_t)slot * kc.Hkv + hk) * PI * 128;
#pragma unroll
        for (int c = 0; c < 128; ++c) o[c] *= rm.x;
        for (int t = 0; t < T; ++t) {
          const float pt = sm.ptail[r][t];
          const uint4* vr = reinterpret_cast<const uint4*>(tail + t * 128);
#pragma unroll
          for (int c8 = 0; c8 < 16; ++c8) {
            const uint4 raw = vr[c8];
            const __half2* h2 = reinterpret_cast<const __half2*>(&raw);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __half22float2(h2[e]);
              o[c8 * 8 + 2 * e] = fmaf(pt, f.x, o[c8 * 8 + 2 * e]);
              o[c8 * 8 + 2 * e + 1] = fmaf(pt, f.y, o[c8 * 8 + 2 * e + 1]);
            }
          }
        }
      }
      ptx::mbar_arrive(&sm.kv_free[bj]);
    }
    ptx::named_bar_sync(1, 256);
    if (i0 + r < L) {
      const float inv_l = 1.f / sm.lfinal[r];
      const int64_t base = ((int64_t)(start + i0 + r) * kc.Hq + hq) * 128;
      if (kc.out_fp32) {
        float4* op = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + base);
#pragma unroll
        for (int c4 = 0; c4 < 32; ++c4)
          op[c4] = make_float4(o[4 * c4] * inv_l, o[4 * c4 + 1] * inv_l, o[4 * c4 + 2] * inv_l, o[4 * c4 + 3] * inv_l);
      } else {
        uint4* op = reinterpret_cast<uint4*>(reinterpret_cast<__half*>(out) + base);
#pragma unroll
        for (int c8 = 0; c8 < 16; ++c8) {
          __half2 h[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) h[e] = __floats2half2_rn(o[8 * c8 + 2 * e] * inv_l, o[8 * c8 + 2 * e + 1] * inv_l);
          op[c8] = *reinterpret_cast<uint4*>(h);
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}

template <int BITS>
cudaError_t launch_t(const KernelCfg& kc, const void* q, const int32_t* cu, const int32_t* slots, int batch,
                     int max_seqlen, const CacheView& cv, void* out, const hack_debug_t* dbg, cudaStream_t st) {
  const size_t smem = sizeof(TcSmem<BITS>) + 1024;
  auto kern = prefill_tc_kernel<BITS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((max_seqlen + BM - 1) / BM, kc.Hq, batch);
  kern<<<grid, kThreads, smem, st>>>(reinterpret_cast<const __half*>(q), cu, slots, cv, kc, out,
                                     dbg ? dbg->pcodes : nullptr, dbg ? dbg->pcodes_stride : 0);
  note_launch();
  return cudaGetLastError();
}

}  // namespace

bool prefill_tc_supported(const KernelCfg& kc) { return kc.Pi == 64 && kc.d == 128; }

cudaError_t launch_prefill_tc(const KernelCfg& kc, const void* q, const int32_t* cu, const int32_t* slots, int batch,
                              int max_seqlen, const CacheView& cv, void* out, const hack_debug_t* dbg,
                              cudaStream_t st) {
  if (kc.bits == 2) return launch_t<2>(kc, q, cu, slots, batch, max_seqlen, cv, out, dbg, st);
  return launch_t<4>(kc, q, cu, slots, batch, max_seqlen, cv, out, dbg, st);
}

}  // namespace hack
