// prefill_tc.cu -- homomorphic prefill attention on the 5th-gen tensor cores (a3-a7),
// for every partition size Pi in {32, 64, 128}.
//
// One CTA = 128 query rows (GQA row packing: gp query heads of one KV head x 128/gp
// positions), warp-specialised (20 warps).  A key tile is one V block: BN = Pi keys.
//   warp 0      producer: whole packed pages (K' + V' codes, fp16 meta, cached sums;
//               DESIGN.md "HBM layout") -> NS-stage smem ring via cp.async.bulk (TMA)
//   warp 1      MMA issuer: tcgen05.mma kind::i8, accumulators in TMEM
//                 QK: per d-block beta D_beta[128 x BN] = (Q'-128)_beta (2K')_beta^T
//                 R : rank terms of Eq. 4 (3-way split TF32 MMA, fp32-level accuracy)
//                 PV: D'[128 x 128] = (P'-128) (2V')^T per BN-token V block
//   warps 2-3   unpack: 2/4-bit codes c -> doubled codes 2c (u8) in K-major UMMA tiles
//               (tc_common.cuh) + per-key / per-channel Eq. 4 coefficients from the page
//               meta and CACHED sums (SE)
//   warps 4-11  two S warpgroups; thread = query row = TMEM lane; SW s owns keys
//               KPT s .. KPT s + KPT - 1 of every tile (KPT = BN / 2):
//                 (a3) Q quantization, 8-bit SR, partitions of Pi channels
//                 (a4) S = centered Eq. 4 x log2e/sqrt(d), d/Pi blocks
//                 (a5) causal online softmax, row max/min combined through smem (2 warps)
//                 (a6) P' 8-bit RN (or SR, R6) per (row, V block) -> smem A tile
//               at Pi = 128 (KPT = 64 scores per thread) pass 1 writes the scores back over
//               the accumulator in TMEM 16 at a time and pass 2 reads them back
//   warps 12-19 two O warpgroups; thread = row; OW o owns output channels 64o..64o+63:
//                 (a7) O = alpha O + centered Eq. 4 on D' (TMEM, double-buffered, so the
//                      S warps run up to NB tiles ahead); FP16 last V block (RQE)
//                      with the S warps' p~ handed over in TMEM; O / l.
// Centering: with s8 A codes a' - 128 and B = 2c the MMA gives
// E = 2 D_s = 2 sum (a'-128) c exactly (|E| < 2^18, so its fp32 conversion is exact).  The
// remaining Eq. 4 terms are a rank-2 update per block:
//   S  = cs sum_beta [ (s_q/2) s_k 2D_s + s_q SQ_s m_k + mu_q y_k ],  y_k = s_k SK + Pi m_k
//   O += (s_p/2) s_v 2D_s + s_p SP_s m_v + mu_p y_v,                  y_v = s_v SV + Pi m_v
// (mu = m + 128 s for the 8-bit side; m_k, m_v the stored fp16 minima).
// Online softmax with lazy rescaling: the running max only moves when a row's tile max
// exceeds it by more than 8 (log2 units; p~ <= 256), warp-uniformly, so most tiles skip the
// O *= alpha pass.  P' codes are invariant to the row scale (R13).
// TMEM (512 columns): S buffers [NSB] (d/Pi x BN = 128 | R (BN)) | D'[NDB] (128 each); NSB = 1,
// NDB = 2 (HACK_PRE_NSB=2 double-buffers S with one D' at Pi <= 64, measured slower).
#include <cstdlib>
#include "common.cuh"
#include "internal.h"
#include "tc_common.cuh"

namespace hack {

namespace {

constexpr int BM = 128;
#ifndef HACK_PRE_GP
#define HACK_PRE_GP 2  // query heads of one KV head packed into a CTA's 128 rows (1: one head x 128 positions)
#endif
constexpr int NOW = 256;       // O-warpgroup threads
constexpr float kMagic = 12582912.f;  // 1.5 * 2^23 (P' rounding)
constexpr float kRescaleTh = 8.f;     // lazy-rescale threshold (log2 units)
// Named barriers: 0 = __syncthreads, 3..6 = the row exchange of the NSG S warps sharing 32
// rows, 7..9 = S -> O.
// Generations of barrier kPBar0 + b alternate strictly: the S warps arrive for tile j only
// after the O warps finished tile j - NB (o_done), which they synced on for tile j - NB.
constexpr uint32_t kPBar0 = 7;

// Integer accumulators are preset to the fp32 bits of 1.5*2^23 by one bf16 MMA (A = e_0,
// B = 1.5*2^23 e_0) before the kind::i8 MMAs accumulate onto them, so the float view of an
// accumulated integer E (|E| < 2^22) is 1.5*2^23 + E and one FADD2 converts two exactly.
#ifndef HACK_ABL
#define HACK_ABL 0  // timing ablations only, bit flags (1 O math, 2 P-quant math, 4 Eq. 4, 8 exp2, 16 unpack)
#endif

#ifndef HACK_PRE_TMEMP
#define HACK_PRE_TMEMP 0  // P' tiles in TMEM where they fit (Geo::TP); measured 3.5 % slower on C2
#endif
#ifndef HACK_PRE_NSB
#define HACK_PRE_NSB 1  // S accumulator buffers in TMEM (Geo::NSB)
#endif
#ifndef HACK_PRE_NSG
#define HACK_PRE_NSG 2  // S warpgroups at Pi >= 64 (4: 16 keys per thread at Pi = 64, measured 6 % slower)
#endif
// service / S / O registers per thread with 4 S warpgroups (setmaxnreg shares of 64K)
#ifndef HACK_PRE_RSVC
#define HACK_PRE_RSVC 40
#endif
#ifndef HACK_PRE_RS
#define HACK_PRE_RS 56
#endif
#ifndef HACK_PRE_RO
#define HACK_PRE_RO 112
#endif
#ifndef HACK_PRE_RS1
#define HACK_PRE_RS1 200  // S registers with one S warpgroup (HACK_PRE_NSG=1)
#endif

// Shapes per partition size: one key tile = one V block (BN = Pi keys); d/Pi d-blocks.
template <int PI_, int BITS>
struct Geo {
  static constexpr int PI = PI_, BN = PI_, NBETA = 128 / PI_;
  // S warpgroups: each owns BN / NSG keys of every tile (more, shorter S warps hide the
  // latency of the per-key epilogue chain; the S side is the kernel's critical path)
  static constexpr int NSG = PI_ == 32 ? 2 : HACK_PRE_NSG;
  static constexpr int THREADS = 128 + 128 * NSG + 256;  // service WG + S WGs + 2 O WGs
  // NSG = 1 (one S warpgroup, 64 keys per thread at Pi = 64): 512 threads, so the S and O
  // shares can exceed 128 (40 + S + 2 O <= 512)
  static constexpr int REG_SVC = NSG == 2 ? 40 : NSG == 1 ? 40 : HACK_PRE_RSVC;
  static constexpr int REG_S = NSG == 2 ? 88 : NSG == 1 ? HACK_PRE_RS1 : HACK_PRE_RS;
  static constexpr int REG_O = NSG == 2 ? 128 : NSG == 1 ? (512 - 40 - HACK_PRE_RS1) / 2 / 8 * 8 : HACK_PRE_RO;
  static_assert(REG_SVC * 128 + REG_S * 128 * NSG + REG_O * 256 <= 65536, "register file");
  static constexpr int KPT = BN / NSG;                  // keys per S thread per tile
  static constexpr bool WB = KPT > (NSG == 2 ? 32 : NSG == 1 ? 64 : 16);  // scores written back to TMEM between passes
  static constexpr int SB = (BITS + (PI_ == 32 ? 5 : PI_ == 64 ? 6 : 7)) <= 8 ? 1 : 2;  // sum bytes (R13)
  static constexpr int up16(int x) { return (x + 15) / 16 * 16; }
  static constexpr int PB = up16(PI_ * 128 * BITS / 8) + up16(PI_ * NBETA * 4) + up16(PI_ * NBETA * SB) +
                            up16(128 * PI_ * BITS / 8) + up16(128 * 4) + up16(128 * SB);  // page bytes
  static constexpr int NS = PI_ == 128 ? 2 : 4;         // page stages
  static constexpr int NB = PI_ == 128 ? 2 : 3;         // K/V/P tile buffer sets
  // S accumulator buffers in TMEM (d/Pi x BN accumulator columns + BN rank-term columns
  // each).  HACK_PRE_NSB=2 (where two fit beside one D' buffer): the MMA warp issues
  // QK(j + 1) while the S warps still read tile j, at the price of a single D' buffer --
  // measured 1.4 % slower on C2 (401 vs 395 us), so one S buffer and two D' buffers.
  static constexpr int SBC = (128 + BN + 31) / 32 * 32;  // columns of one S buffer
  static constexpr int NSB = HACK_PRE_NSB == 2 && 2 * SBC + 128 <= 512 ? 2 : 1;
  static constexpr int NDB = NSB == 2 ? 1 : 2;          // D' (PV accumulator) TMEM buffers
  static constexpr int KR = NBETA * 12 < 16 ? 16 : NBETA * 12;  // rank-term K (tf32), 12 per block
  static constexpr int SBO_R = KR * 32;                 // K-major SBO of the rank operands
  static constexpr int SBO_T = BN * 8;                  // K-major SBO of the P and V tiles (K = BN)
  static constexpr int TR = 128;                        // TMEM: rank-term columns (in an S buffer)
  static constexpr int TD = NSB * SBC;                  // TMEM: first D' column
  // HACK_PRE_TMEMP=1: P' tiles in TMEM (the PV MMA's A operand from tensor memory, 4 codes
  // per column) where NB of them fit after the D' buffers, written by the S warps with
  // tcgen05.st instead of STS + a generic->async proxy fence per tile.  Parity-clean, but the
  // C2 kernel measured 411 vs 397 us (the proxy fence is cheaper than it looked in the stall
  // samples), so P' stays in smem.
  static constexpr int TPC = TD + NDB * 128;            // TMEM: first P' column
  static constexpr bool TP = HACK_PRE_TMEMP && TPC + NB * (BN / 4) <= 512;
  static_assert(TD + NDB * 128 <= 512, "TMEM budget");
};

template <int PI_, int BITS>
struct TcSmem {
  using Gm = Geo<PI_, BITS>;
  static constexpr int NS = Gm::NS, NB = Gm::NB, BN = Gm::BN;
  uint8_t stage[NS][Gm::PB];
  alignas(128) uint8_t q[BM * 128];          // Q' - 128 (s8), K-major, SBO 1024
  alignas(128) uint8_t k[NB][BN * 128];      // K' (u8, doubled), K-major, SBO 1024
  alignas(128) uint8_t v[NB][128 * BN];      // V' (u8, doubled), K-major (keys = K), SBO 8 BN
  alignas(128) uint8_t p[NB][Gm::TP ? 128 : BM * BN];  // P' - 128 (s8), K-major, SBO 8 BN (unless in TMEM)
  alignas(128) float ar[BM * Gm::KR];        // rank-term A operand (tf32): per row, per beta X, M split 3 ways
  alignas(128) float br[NB][BN * Gm::KR];    // rank-term B operand per key: m_k, y_k split 3 ways
  alignas(128) uint16_t pre_a[128 * 16];     // bf16 preset operands: A[:, 0] = 1, B[:, 0] = 1.5 * 2^23 (K-major,
  alignas(128) uint16_t pre_b[128 * 16];     //   SBO 256): one kind::f16 MMA writes the magic into D
  alignas(16) float kcf[NB][Gm::NBETA][BN];  // [buf][beta][key]: s_k
  alignas(16) float vcf[NB][3][128];         // [buf][field][channel]: s_v, m_v, y_v
  float qa[Gm::NBETA][BM];                   // per (beta, row): cs s_q / 2
  int sp_part[NB][Gm::NSG][BM];              // partial P-code sums (per S warpgroup)
  float4 pinfo[NB][BM];                      // per (tile, row): alpha, rescaled?, s_p, m_p
  float2 xch[2][Gm::NSG][BM];                // partial (max, min | -inf if masked) per tile
  float2 xq[Gm::NSG][BM];                    // Q prologue: partial (min, max) of a partition
  int xs[Gm::NSG][BM];                       // Q prologue: partial code sums of a partition
  float lpart[Gm::NSG][BM];
  uint64_t full[NS], empty[NS], k_ready[NB], k_free[NB], v_ready[NB], o_done[NB], p_ready[NB], d_full[2],
      d_free[2], s_full[2], s_free[2], q_ready, l_ready, l_free;
  uint32_t tmem_base;
};

HACK_DEV float2 acc2f(uint32_t a, uint32_t b) {
  return ptx::fadd2(make_float2(__uint_as_float(a), __uint_as_float(b)), make_float2(-kMagic, -kMagic));
}

// Exact 3-way tf32 split x = h + m + l (11 + 11 + <= 2 significant bits); a product x y is
// then hh' + hm' + mh' + hl' + lh' + mm' up to ~2^-33 relative (the dropped ml', lm', ll').
// A-side (row constant) and B-side (key coefficient) orders pair up those six terms.
HACK_DEV void split3(float x, float& h, float& m, float& l) {
  h = ptx::tf32_hi(x);
  const float r = x - h;
  m = ptx::tf32_hi(r);
  l = r - m;
}
HACK_DEV void rank_a(float x, float* v) {
  float h, m, l;
  split3(x, h, m, l);
  v[0] = h; v[1] = h; v[2] = m; v[3] = h; v[4] = l; v[5] = m;
}
HACK_DEV void rank_b(float y, float* v) {
  float h, m, l;
  split3(y, h, m, l);
  v[0] = h; v[1] = m; v[2] = h; v[3] = l; v[4] = h; v[5] = m;
}

// Query heads packed per CTA (they share the KV head): HACK_PRE_GP if it divides the GQA group.
__host__ __device__ __forceinline__ int pack_heads(const KernelCfg& kc) {
  return (HACK_PRE_GP >= 4 && kc.G % 4 == 0) ? 4 : ((HACK_PRE_GP >= 2 && kc.G % 2 == 0) ? 2 : 1);
}

// Causal mask (R8) of n scores at keys t0.. for the row at position i, and the running max /
// min over the visible keys.
template <int N>
HACK_DEV void mask_minmax_t(float* s, int t0, int i, bool full, bool& masked, float& mx, float& mn) {
  if (!full) {
#pragma unroll
    for (int x = 0; x < N; ++x) {
      const bool vis = (t0 + x) <= i;
      masked |= !vis;
      mn = fminf(mn, vis ? s[x] : INFINITY);  // min over the visible keys only
      s[x] = vis ? s[x] : -INFINITY;
    }
  } else {
#pragma unroll
    for (int x = 0; x < N; ++x) mn = fminf(mn, s[x]);
  }
#pragma unroll
  for (int x = 0; x < N; ++x) mx = fmaxf(mx, s[x]);
}

// 16 P values -> 16 code bytes (RN by the 1.5*2^23 magic number, or SR) packed in the
// permuted order of the V unpacking; returns the four words and adds their code sum.
template <int BITS, bool PSR>
HACK_DEV uint4 p_codes16(const float* s, float inv, float nlo, uint64_t seed, uint32_t rid, uint32_t c3, int64_t i,
                         int t, uint32_t& sum) {
  uint32_t bits[16];
  if (!PSR) {
    const float2 inv2 = make_float2(inv, inv), nlo2 = make_float2(nlo, nlo), magic = make_float2(kMagic, kMagic);
#pragma unroll
    for (int kk = 0; kk < 16; kk += 2) {
      const float2 y = ptx::fadd2(ptx::ffma2(make_float2(s[kk], s[kk + 1]), inv2, nlo2), magic);
      bits[kk] = __float_as_uint(y.x);
      bits[kk + 1] = __float_as_uint(y.y);
    }
  } else {
    // the paper's stochastic rounding for P (R6, selectable): floor(y) + [u < frac(y)], u from
    // the position-keyed P stream (query position i, key t, global query head)
#pragma unroll
    for (int k4 = 0; k4 < 16; k4 += 4) {
      const Philox4 rr = philox_block(seed, rid, c3, ((uint64_t)i << 30) | (uint64_t)((t + k4) >> 2));
      const float u4[4] = {u24(rr.x), u24(rr.y), u24(rr.z), u24(rr.w)};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float y = fmaf(s[k4 + e], inv, nlo);
        const float fl = floorf(y);
        bits[k4 + e] = (uint32_t)min(255, (int)fl + (u4[e] < y - fl ? 1 : 0));
      }
    }
  }
  uint32_t cw[4];
#pragma unroll
  for (int x4 = 0; x4 < 4; ++x4) {
    // byte position p of this 16-key chunk holds local key perm_src(p)
    const uint32_t lo2 = ptx::prmt(bits[perm_src<BITS>(4 * x4 + 0)], bits[perm_src<BITS>(4 * x4 + 1)], 0x0040u);
    const uint32_t hi2 = ptx::prmt(bits[perm_src<BITS>(4 * x4 + 2)], bits[perm_src<BITS>(4 * x4 + 3)], 0x0040u);
    cw[x4] = ptx::prmt(lo2, hi2, 0x5410u);
    sum = __dp4a(cw[x4], 0x01010101u, sum);
  }
  return make_uint4(cw[0], cw[1], cw[2], cw[3]);
}

// DBG: parity runs only (hack_debug_t): dumps the P codes and the raw QK / PV block
// accumulators E = 2 D - 256 S_B (HACK_ACC_S8_2B); the production instantiation has none of it.
// PSR: P codes by the paper's stochastic rounding (R6, selectable) instead of RN.
template <int PI_, int BITS, bool DBG, bool PSR>
__global__ void __launch_bounds__(Geo<PI_, BITS>::THREADS, 1) prefill_tc_kernel(
    const __half* __restrict__ q, const int32_t* __restrict__ cu_seqlens, const int32_t* __restrict__ slots,
    CacheView cv, KernelCfg kc, void* __restrict__ out, uint8_t* __restrict__ dbg_pcodes, int64_t dbg_stride,
    int32_t* __restrict__ dbg_qk, int32_t* __restrict__ dbg_pv, int64_t acc_stride, int acc_head, int nitems) {
  using Gm = Geo<PI_, BITS>;
  using SM = TcSmem<PI_, BITS>;
  constexpr int PI = Gm::PI, BN = Gm::BN, NBETA = Gm::NBETA, KPT = Gm::KPT, NS = Gm::NS, NB = Gm::NB;
  constexpr int NDB = Gm::NDB, KR = Gm::KR, SBO_R = Gm::SBO_R, SBO_T = Gm::SBO_T;
  constexpr bool WB = Gm::WB;
  constexpr int NSG = Gm::NSG, NSW = 128 * NSG;  // S warpgroups, S threads
  constexpr int OBASE = 128 + NSW;              // first O thread
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);

  // Work items: (request, query-tile rank, head pair); rank 0 = the heaviest (longest causal
  // rows).  GQA row packing: the 128 MMA rows are gp query heads (of one KV head) x pbp
  // positions, so the K'/V' tiles a CTA unpacks serve gp heads and the causal diagonal is pbp
  // wide.  Persistent launch (nitems > 0, one request): CTA c runs items c, 2G-1-c, 2G+c, ...
  // of the heaviest-first order (a snake over the G CTAs balances the causal triangle), the
  // next item's pages, Q quantization and first tiles overlapping the previous item's drain
  // (no per-CTA launch, TMEM allocation and pipeline fill per item).  Otherwise one item per
  // CTA from the grid (head pair fastest, heaviest first).
  const int gp = pack_heads(kc), pbp = BM / gp;
  const int npk = kc.hq_count / gp;  // head groups of this launch (from kc.hq_begin)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const PageLayout PL = kc.pl;
  struct Item {
    int start, L, i0, hq0, hk, slot, nkt, nfull;
  };
  auto get_item = [&](int it, Item& w) -> bool {
    int b, lin;
    if (nitems > 0) {
      const int G = gridDim.x, c = blockIdx.x;
      lin = it * G + ((it & 1) ? G - 1 - c : c);
      if (lin >= nitems) return false;
      b = 0;
    } else {
      if (it > 0) return false;
      b = blockIdx.z;
      lin = blockIdx.x + gridDim.x * blockIdx.y;
    }
    const int rank = kc.qt_begin + lin / npk;
    w.hq0 = kc.hq_begin + (lin % npk) * gp;  // heads hq0 .. hq0 + gp - 1
    w.start = cu_seqlens[b];
    w.L = cu_seqlens[b + 1] - w.start;
    const int nqt = (w.L + pbp - 1) / pbp;
    if (rank >= nqt) return false;
    w.i0 = (nqt - 1 - rank) * pbp;  // first position of the item
    w.slot = slots[b];
    w.hk = w.hq0 / kc.G;
    w.nkt = min((w.i0 + pbp - 1) / BN, (w.L - 1) / BN) + 1;  // key tiles (causal)
    w.nfull = w.L / PI;                                      // committed V blocks
    return true;
  };
  {
    Item w0;
    if (!get_item(0, w0)) return;
  }

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      ptx::mbar_init(&sm.full[s], 1);
      ptx::mbar_init(&sm.empty[s], 64);
    }
    for (int x = 0; x < NB; ++x) {
      ptx::mbar_init(&sm.k_ready[x], 64);
      ptx::mbar_init(&sm.k_free[x], NSW);
      ptx::mbar_init(&sm.v_ready[x], 64);
      ptx::mbar_init(&sm.o_done[x], NOW);
      ptx::mbar_init(&sm.p_ready[x], NSW);
    }
    for (int x = 0; x < 2; ++x) {
      ptx::mbar_init(&sm.d_full[x], 1);
      ptx::mbar_init(&sm.d_free[x], NOW);
    }
    for (int x = 0; x < 2; ++x) {
      ptx::mbar_init(&sm.s_full[x], 1);
      ptx::mbar_init(&sm.s_free[x], NSW);
    }
    ptx::mbar_init(&sm.q_ready, NSW);
    ptx::mbar_init(&sm.l_ready, NSW);
    ptx::mbar_init(&sm.l_free, NOW);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(&sm.tmem_base, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  // S buffer b at columns b SBC: D_beta (BN each; scores / tail p~ in WB), then at + TR the
  // rank terms of S (BN columns): sum_beta X m_k + M y_k (3xTF32).  Tile g uses buffer g % NSB.
  const uint32_t tS = tmem;
  const uint32_t tR = tmem + Gm::TR;
  const uint32_t tD0 = tmem + Gm::TD;    // D'[0 .. NDB) (128 columns each)
  constexpr int NSB = Gm::NSB, SBC = Gm::SBC;

  if (warp < 4) {
    // register budget (launch: THREADS x the launch-bound cap): service, S and O shares (Geo)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(Gm::REG_SVC));
    if (warp == 0) {
      // ---------------------------------------------------------------- producer
      // launched as a programmatic dependent of the ingest (hack_prefill_attention): the
      // pages are read only after that grid completed
      asm volatile("griddepcontrol.wait;" ::: "memory");
      if (lane == 0) {
        int jg = 0;  // tiles of all items so far (ring phases)
        Item w;
        for (int it = 0; get_item(it, w); ++it) {
          const int32_t* bt = cv.block_table + (int64_t)w.slot * cv.max_pages_per_req;
          for (int j = 0; j < w.nkt; ++j, ++jg) {
            const int s = jg % NS;
            ptx::mbar_wait(&sm.empty[s], ((jg / NS) & 1) ^ 1);
            ptx::mbar_arrive_expect_tx(&sm.full[s], Gm::PB);
            const uint8_t* pg = cv.pages + ((int64_t)bt[j] * cv.num_kv_heads + w.hk) * cv.page_bytes;
            ptx::bulk_g2s(sm.stage[s], pg, Gm::PB, &sm.full[s]);
          }
        }
      }
    } else if (warp == 1) {
      // ---------------------------------------------------------------- MMA issuer
      const uint32_t idesc_qk = ptx::idesc_s8u8(BM, BN), idesc_pv = ptx::idesc_s8u8(BM, 128);
      const uint32_t qa = ptx::smem_u32(sm.q);
      const uint64_t pre_a = ptx::smem_desc_kmajor(ptx::smem_u32(sm.pre_a), 128, 256);
      const uint64_t pre_b = ptx::smem_desc_kmajor(ptx::smem_u32(sm.pre_b), 128, 256);
      const uint32_t idesc_pre = ptx::idesc_bf16(BM, 128);
      int jg = 0, jpv = 0;  // tiles / PV tiles of all items so far (ring phases)
      int last_tail = -1 - NSB;  // global index of the latest FP16-tail tile (its p~ sits in its S buffer)
      Item w;
#pragma unroll 1
      for (int it = 0; get_item(it, w); ++it) {
      ptx::mbar_wait(&sm.q_ready, it & 1);  // this item's Q' and rank-term rows in smem
#pragma unroll 1
      for (int j = 0; j <= w.nkt; ++j) {
        if (j < w.nkt) {
          const int g = jg + j, bq = g % NB;
          ptx::mbar_wait(&sm.k_ready[bq], (g / NB) & 1);
          const uint32_t sbo = (uint32_t)(SBC * (g % NSB));
          ptx::mbar_wait(&sm.s_free[g % NSB], ((g / NSB) & 1) ^ 1);
          // an earlier item's FP16 tail p~ sits in this S buffer: the O warps must be done
          if (last_tail == g - NSB) ptx::mbar_wait(&sm.o_done[(g - NSB) % NB], ((g - NSB) / NB) & 1);
          ptx::tc_fence_after();
          if (lane == 0) {
            const uint32_t ka = ptx::smem_u32(sm.k[bq]);
            ptx::mma_bf16(tS + sbo, pre_a, pre_b, idesc_pre, 0u);  // D_beta := 1.5 * 2^23 (all 128 columns)
#pragma unroll
            for (int beta = 0; beta < NBETA; ++beta)
#pragma unroll
              for (int ks = 0; ks < PI / 32; ++ks) {
                const uint32_t koff = (uint32_t)(beta * PI / 16 + ks * 2) * 128;  // 16-byte K chunks
                ptx::mma_u8(tS + sbo + BN * beta, ptx::smem_desc_kmajor(qa + koff, 128, 1024),
                            ptx::smem_desc_kmajor(ka + koff, 128, 1024), idesc_qk, 1u);
              }
            // rank-2-per-block terms of Eq. 4 on the tensor pipe: R = [X | M] [m_k ; y_k]
            // with both sides split 3 ways (exact tf32 parts, fp32-level product), so the S
            // epilogue keeps one FMUL2 + FFMA2 per key pair and block
            const uint32_t ra = ptx::smem_u32(sm.ar), rb = ptx::smem_u32(sm.br[bq]);
#pragma unroll
            for (int ks = 0; ks < KR / 8; ++ks)
              ptx::mma_tf32(tR + sbo, ptx::smem_desc_kmajor(ra + ks * 256, 128, SBO_R),
                            ptx::smem_desc_kmajor(rb + ks * 256, 128, SBO_R), ptx::idesc_tf32(BM, BN), ks > 0);
            ptx::mma_commit(&sm.s_full[g % NSB]);
          }
          __syncwarp();
        }
        const int jj = j - 1;  // PV of the previous tile, after QK of this one (overlap)
        if (jj >= 0 && jj < w.nfull) {
          const int g = jg + jj, bd = jpv % NDB, bq = g % NB;
          const uint32_t ph = (g / NB) & 1;
          ptx::mbar_wait(&sm.p_ready[bq], ph);
          ptx::mbar_wait(&sm.v_ready[bq], ph);
          ptx::mbar_wait(&sm.d_free[bd], ((jpv / NDB) & 1) ^ 1);
          ++jpv;
          ptx::tc_fence_after();
          if (lane == 0) {
            const uint32_t pa = ptx::smem_u32(sm.p[bq]), va = ptx::smem_u32(sm.v[bq]);
            ptx::mma_bf16(tD0 + 128 * bd, pre_a, pre_b, idesc_pre, 0u);  // D' := 1.5 * 2^23
#pragma unroll
            for (int ks = 0; ks < BN / 32; ++ks) {
              if (Gm::TP)  // A = P' from TMEM: lane = row, 8 columns per 32-key step
                ptx::mma_u8_ts(tD0 + 128 * bd, tmem + Gm::TPC + bq * (BN / 4) + 8 * ks,
                               ptx::smem_desc_kmajor(va + ks * 256, 128, SBO_T), idesc_pv, 1u);
              else
                ptx::mma_u8(tD0 + 128 * bd, ptx::smem_desc_kmajor(pa + ks * 256, 128, SBO_T),
                            ptx::smem_desc_kmajor(va + ks * 256, 128, SBO_T), idesc_pv, 1u);
            }
            ptx::mma_commit(&sm.d_full[bd]);
          }
          __syncwarp();
        }
      }
      if (w.nfull < w.nkt) last_tail = jg + w.nkt - 1;  // the item's last tile is the FP16 tail
      jg += w.nkt;
      }
    } else {
      // ---------------------------------------------------------------- unpack (64 threads)
      const int ut = tid - 64;
      // bf16 preset operands (visible to the MMA through the proxy fence before k_ready)
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const int row = ut + 64 * rr;
        *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(sm.pre_a) + kmaj_off(row, 0, 256)) =
            make_uint4(0x3F80u, 0u, 0u, 0u);  // bf16 1.0 at k = 0
        *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(sm.pre_a) + kmaj_off(row, 16, 256)) = make_uint4(0u, 0u, 0u, 0u);
        *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(sm.pre_b) + kmaj_off(row, 0, 256)) =
            make_uint4(0x4B40u, 0u, 0u, 0u);  // bf16 1.5 * 2^23 at k = 0
        *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(sm.pre_b) + kmaj_off(row, 16, 256)) = make_uint4(0u, 0u, 0u, 0u);
      }
      int jg = 0;
      Item w;
#pragma unroll 1
      for (int it = 0; get_item(it, w); ++it) {
#pragma unroll 1
      for (int j = 0; j < w.nkt; ++j, ++jg) {
        const int s = jg % NS, bj = jg % NB;
        const uint32_t ph = (jg / NB) & 1;
        ptx::mbar_wait(&sm.full[s], (jg / NS) & 1);
        ptx::mbar_wait(&sm.k_free[bj], ph ^ 1);
        const uint8_t* pg = sm.stage[s];
        const int nk = min(BN, w.L - j * BN);
        if (!(HACK_ABL & 16)) {
          // K' codes: thread = key; 8 consecutive keys fill one 128-byte core matrix per store
#pragma unroll
          for (int key = ut; key < BN; key += 64) {
            const uint4* src = reinterpret_cast<const uint4*>(pg + PL.k_codes + key * (128 * BITS / 8));
#pragma unroll
            for (int h = 0; h < BITS; ++h) {  // 16-byte pieces of the packed row
              const uint4 pw = src[h];
              const uint32_t w4[4] = {pw.x, pw.y, pw.z, pw.w};
#pragma unroll
              for (int x = 0; x < 4; ++x) {
                const int wi = 4 * h + x;
                if (BITS == 2)
                  *reinterpret_cast<uint4*>(sm.k[bj] + kmaj_off(key, 16 * wi, 1024)) = unpack16_2b_x2(w4[x]);
                else
                  *reinterpret_cast<uint2*>(sm.k[bj] + kmaj_off(key, 8 * wi, 1024)) = unpack8_4b_x2(w4[x]);
              }
            }
          }
          // per-(key, beta) Eq. 4 coefficients: BN x d/Pi = 128 entries, 2 per thread
#pragma unroll
          for (int e0 = 0; e0 < BN * NBETA; e0 += 64) {
            // entry e = (key, beta); a thread takes consecutive betas of one key when it can
            const int e = (NBETA == 2 ? 2 * ut + (e0 >> 6) : e0 + ut);
            const int key = e / NBETA, beta = e % NBETA;
            float c0 = 0.f, c1 = 0.f, c2 = 0.f;
            if (key < nk) {
              const __half2 mh = reinterpret_cast<const __half2*>(pg + PL.k_meta)[e];
              const float m = __low2float(mh), s2 = __high2float(mh);
              const int sum = load_sum(pg + PL.k_sums, e, PL.sum_bytes);  // cached sum (SE)
              c0 = s2;
              c1 = m;
              c2 = fmaf(s2, (float)sum, PI * m);  // y_k = s_k SK + Pi m_k
            }
            sm.kcf[bj][beta][key] = c0;
            float rv[12];
            rank_b(c1, rv);
            rank_b(c2, rv + 6);
            uint8_t* brk = reinterpret_cast<uint8_t*>(sm.br[bj]);
#pragma unroll
            for (int x = 0; x < 12; x += 4)
              *reinterpret_cast<float4*>(brk + kmaj_off(key, 4 * (12 * beta + x), SBO_R)) =
                  make_float4(rv[x], rv[x + 1], rv[x + 2], rv[x + 3]);
            if (KR > 12 * NBETA)  // K padding of the rank MMA (Pi = 128: 12 -> 16)
              *reinterpret_cast<float4*>(brk + kmaj_off(key, 4 * 12 * NBETA, SBO_R)) = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
        ptx::fence_proxy_async_smem();
        ptx::mbar_arrive(&sm.k_ready[bj]);
        ptx::mbar_wait(&sm.o_done[bj], ph ^ 1);  // O warps done with tile j - NB
        if (j < w.nfull && !(HACK_ABL & 16)) {
          constexpr int WPC = BN * BITS / 32;  // packed 32-bit words per V channel row
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2) {
            const int ch = ut + 64 * c2;
            uint32_t wv[WPC];  // the channel's packed row, 16-byte loads where it allows
            if constexpr (WPC % 4 == 0) {
#pragma unroll
              for (int x = 0; x < WPC; x += 4) {
                const uint4 w4 = *reinterpret_cast<const uint4*>(pg + PL.v_codes + ch * (BN * BITS / 8) + 4 * x);
                wv[x] = w4.x; wv[x + 1] = w4.y; wv[x + 2] = w4.z; wv[x + 3] = w4.w;
              }
            } else {
#pragma unroll
              for (int x = 0; x < WPC; x += 2) {
                const uint2 w2 = *reinterpret_cast<const uint2*>(pg + PL.v_codes + ch * (BN * BITS / 8) + 4 * x);
                wv[x] = w2.x; wv[x + 1] = w2.y;
              }
            }
#pragma unroll
            for (int wi = 0; wi < WPC; ++wi) {
              if (BITS == 2)
                *reinterpret_cast<uint4*>(sm.v[bj] + kmaj_off(ch, 16 * wi, SBO_T)) = unpack16_2b_x2(wv[wi]);
              else
                *reinterpret_cast<uint2*>(sm.v[bj] + kmaj_off(ch, 8 * wi, SBO_T)) = unpack8_4b_x2(wv[wi]);
            }
            const __half2 mh = reinterpret_cast<const __half2*>(pg + PL.v_meta)[ch];
            const float m = __low2float(mh), s2 = __high2float(mh);
            const int sum = load_sum(pg + PL.v_sums, ch, PL.sum_bytes);  // cached sum (SE)
            sm.vcf[bj][0][ch] = s2;
            sm.vcf[bj][1][ch] = m;
            sm.vcf[bj][2][ch] = fmaf(s2, (float)sum, PI * m);  // y_v = s_v SV + Pi m_v
          }
        }
        ptx::fence_proxy_async_smem();
        ptx::mbar_arrive(&sm.v_ready[bj]);
        ptx::mbar_arrive(&sm.empty[s]);
      }
      }
    }
  } else if (warp < 4 + 4 * NSG) {
    // ------------------------------------------------------------------ S warpgroups (NSG)
    // thread = query row r = TMEM lane; SW s owns keys KPT s .. KPT s + KPT - 1 of every tile
    if (Gm::REG_S <= 65536 / Gm::THREADS)
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(Gm::REG_S));
    else  // NSG = 1: the S warpgroup takes part of the service warps' share
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(Gm::REG_S));
    const int sw = (warp - 4) >> 2;
    const int r = (tid - 128) & (BM - 1);
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    const uint32_t qbar = 3 + (warp & 3);  // the NSG S warps sharing these 32 rows
    constexpr uint32_t QBN = 32 * NSG;      // ... their thread count
    const float cscale = 1.4426950408889634f / sqrtf(128.f);
    const int kb = KPT * sw;
    // Q prologue geometry: this thread quantizes CW channels of its row; a partition of Pi
    // channels is NPL partitions of one thread or spans PW warpgroups (min/max and code
    // sums exchanged through xq / xs)
    constexpr int CW = 128 / NSG, NQV = CW / 8;
    constexpr int NPL = PI >= CW ? 1 : CW / PI;
    constexpr int PW = PI > CW ? PI / CW : 1;
    constexpr int VPP = NQV / NPL;  // 16-byte pieces per (local) partition
    const int g0 = sw - sw % PW;    // first warpgroup of this thread's partition
    int jg = 0;  // tiles of all items so far
    Item w;
#pragma unroll 1
    for (int it = 0; get_item(it, w); ++it) {
    const int pos = w.i0 + (r & (pbp - 1)), hq = w.hq0 + r / pbp;  // this row's position and head
    const int L = w.L, start = w.start;
    const int i = min(pos, L - 1);  // this thread's query position (padding rows clamp)
    {
      // (QK of the previous item complete: this thread waited its last s_full)
      // (a3) quantize Q[i, CW sw .. CW sw + CW - 1]: 8-bit, fp32 meta, SR, partitions of Pi
      // channels.  xq / xs reuse across items: a warpgroup writes them again only after the
      // tile barriers of this item, which its partners pass after their reads.
      const uint4* qrow = reinterpret_cast<const uint4*>(q + ((int64_t)(start + i) * kc.Hq + hq) * 128 + CW * sw);
      // all loads of the slice in flight at once (one memory latency per CTA), kept in
      // registers for the quantization pass; min/max on packed halves
      uint4 qr[NQV];
#pragma unroll
      for (int v8 = 0; v8 < NQV; ++v8) qr[v8] = __ldg(qrow + v8);
      QMeta qm[NPL];
#pragma unroll
      for (int pp = 0; pp < NPL; ++pp) {
        __half2 lo2 = *reinterpret_cast<const __half2*>(&qr[pp * VPP].x), hi2 = lo2;
#pragma unroll
        for (int v8 = pp * VPP; v8 < (pp + 1) * VPP; ++v8) {
          const __half2* h2 = reinterpret_cast<const __half2*>(&qr[v8]);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            lo2 = __hmin2(lo2, h2[e]);
            hi2 = __hmax2(hi2, h2[e]);
          }
        }
        float lo = fminf(__low2float(lo2), __high2float(lo2)), hi = fmaxf(__low2float(hi2), __high2float(hi2));
        if (PW > 1) {  // the rest of the partition lives in the partner warpgroups
          sm.xq[sw][r] = make_float2(lo, hi);
          ptx::named_bar_sync(qbar, QBN);
#pragma unroll
          for (int w2 = 0; w2 < PW; ++w2) {
            const float2 o = sm.xq[g0 + w2][r];
            lo = fminf(lo, o.x);
            hi = fmaxf(hi, o.y);
          }
        }
        qm[pp] = meta_fp32(lo, hi, 255);
      }
      const uint32_t c3 = stream_c3(kc.layer, kTagQ, kc.head_base * kc.G + hq);
      const uint32_t rng_id = cv.rng_ids[w.slot];
      int sum[NPL];
#pragma unroll
      for (int pp = 0; pp < NPL; ++pp) sum[pp] = 0;
#pragma unroll
      for (int g = 0; g < CW / 16; ++g) {  // 16-channel groups
        const int pp = PI >= CW ? 0 : (16 * g) / PI;
        float x[16];
        const __half* ha = reinterpret_cast<const __half*>(&qr[2 * g]);
        const __half* hb = reinterpret_cast<const __half*>(&qr[2 * g + 1]);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          x[e] = __half2float(ha[e]);
          x[8 + e] = __half2float(hb[e]);
        }
        int cc[16];
        if (kc.q_round == HACK_ROUND_STOCHASTIC) {
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            const uint64_t n = ((uint64_t)i * 128u + (uint64_t)(CW * sw + 16 * g + 4 * k4)) >> 2;
            const Philox4 rr = philox_block(kc.seed, rng_id, c3, n);
            cc[4 * k4 + 0] = quant_sr(x[4 * k4 + 0], qm[pp], u24(rr.x), 255);
            cc[4 * k4 + 1] = quant_sr(x[4 * k4 + 1], qm[pp], u24(rr.y), 255);
            cc[4 * k4 + 2] = quant_sr(x[4 * k4 + 2], qm[pp], u24(rr.z), 255);
            cc[4 * k4 + 3] = quant_sr(x[4 * k4 + 3], qm[pp], u24(rr.w), 255);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) cc[e] = quant_rn(x[e], qm[pp], 255);
        }
        uint32_t wv[4];
#pragma unroll
        for (int x4 = 0; x4 < 4; ++x4) {
          uint32_t wd = 0;
#pragma unroll
          for (int e = 0; e < 4; ++e) wd |= (uint32_t)cc[perm_src<BITS>(4 * x4 + e)] << (8 * e);
          wv[x4] = wd ^ 0x80808080u;  // s8 operand: code - 128
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) sum[pp] += cc[e];
        *reinterpret_cast<uint4*>(sm.q + kmaj_off(r, CW * sw + 16 * g, 1024)) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      }
      if (PW > 1) {  // code sum over the whole partition
        sm.xs[sw][r] = sum[0];
        ptx::named_bar_sync(qbar, QBN);
        sum[0] = 0;
#pragma unroll
        for (int w2 = 0; w2 < PW; ++w2) sum[0] += sm.xs[g0 + w2][r];
      }
      if (sw == g0) {  // the partition's constants: written once
#pragma unroll
        for (int pp = 0; pp < NPL; ++pp) {
          const int beta = (CW * sw) / PI + pp;
          const int sqs = sum[pp] - 128 * PI;  // sum (q' - 128)
          sm.qa[beta][r] = cscale * qm[pp].s * 0.5f;
          const float X = cscale * qm[pp].s * (float)sqs, M = cscale * __fmaf_rn(128.f, qm[pp].s, qm[pp].m);
          float av[12];
          rank_a(X, av);
          rank_a(M, av + 6);
          uint8_t* arr = reinterpret_cast<uint8_t*>(sm.ar);
#pragma unroll
          for (int x = 0; x < 12; x += 4)
            *reinterpret_cast<float4*>(arr + kmaj_off(r, 4 * (12 * beta + x), SBO_R)) =
                make_float4(av[x], av[x + 1], av[x + 2], av[x + 3]);
          if (KR > 12 * NBETA && beta == 0)
            *reinterpret_cast<float4*>(arr + kmaj_off(r, 4 * 12 * NBETA, SBO_R)) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      ptx::fence_proxy_async_smem();
      ptx::mbar_arrive(&sm.q_ready);
    }
    ptx::named_bar_sync(qbar, QBN);  // the row's Q constants (all partitions) visible
    float qa[NBETA];
#pragma unroll
    for (int beta = 0; beta < NBETA; ++beta) qa[beta] = sm.qa[beta][r];
    float m_run = -INFINITY, l_run = 0.f;
    const uint32_t p_c3 = PSR ? stream_c3(kc.layer, kTagP, kc.head_base * kc.G + hq) : 0u;
    const uint32_t p_rid = PSR ? cv.rng_ids[w.slot] : 0u;

#pragma unroll 1
    for (int j = 0; j < w.nkt; ++j, ++jg) {
      const int bj = jg % NB, t0 = j * BN;
      const uint32_t ph = (jg / NB) & 1;
      const bool full = (t0 + BN - 1) <= w.i0;  // every key visible to every row of the item
      const uint32_t sbo = (uint32_t)(SBC * (jg % NSB));  // this tile's S buffer
      ptx::mbar_wait(&sm.s_full[jg % NSB], (jg / NSB) & 1);
      ptx::tc_fence_after();
      // ---- pass 1: S = R + sum_beta (s_q/2) s_k E_beta (centered Eq. 4) x log2(e)/sqrt(d),
      // causal mask, row max / min; 16 keys per TMEM load (register pressure)
      float s[WB ? 16 : KPT];
      float mx = -INFINITY, mn = INFINITY;
      bool masked = false;
#pragma unroll
      for (int c = 0; c < KPT / 16; ++c) {
        const int so = WB ? 0 : 16 * c;  // this chunk's scores: s[so .. so + 15]
        {
          uint32_t d[16];
          ptx::tmem_ld16(tR + sbo + lane_base + kb + 16 * c, d);  // rank terms (tensor pipe) seed S
          ptx::tmem_wait_ld();
#pragma unroll
          for (int x = 0; x < 16; ++x) s[so + x] = __uint_as_float(d[x]);
        }
#pragma unroll
        for (int beta = 0; beta < NBETA && !(HACK_ABL & 4); ++beta) {
          const float2 A = make_float2(qa[beta], qa[beta]);
          uint32_t d[16];
          ptx::tmem_ld16(tS + sbo + lane_base + BN * beta + kb + 16 * c, d);
          ptx::tmem_wait_ld();
          if (DBG && dbg_qk != nullptr && pos < L && (acc_head < 0 || hq == acc_head)) {  // E = 2 D - 256 SK
            const int hs = acc_head < 0 ? hq : 0, hn = acc_head < 0 ? kc.Hq : 1;
            int32_t* dq = dbg_qk + (((int64_t)(start + pos) * hn + hs) * NBETA + beta) * acc_stride;
#pragma unroll
            for (int x = 0; x < 16; ++x) {
              const int t = t0 + kb + 16 * c + x;
              if (t < L) dq[t] = (int32_t)(d[x] - 0x4B400000u);
            }
          }
#pragma unroll
          for (int g4 = 0; g4 < 4; ++g4) {
            const float4 sk4 = *reinterpret_cast<const float4*>(&sm.kcf[bj][beta][kb + 16 * c + 4 * g4]);
#pragma unroll
            for (int pr = 0; pr < 2; ++pr) {
              const int k2 = 4 * g4 + 2 * pr;
              const float2 E = acc2f(d[k2], d[k2 + 1]);
              const float2 skp = pr ? make_float2(sk4.z, sk4.w) : make_float2(sk4.x, sk4.y);
              const float2 t = ptx::fmul2(skp, E);  // s_k 2D_s
              const float2 a = ptx::ffma2(A, t, make_float2(s[so + k2], s[so + k2 + 1]));
              s[so + k2] = a.x;
              s[so + k2 + 1] = a.y;
            }
          }
        }
        if (WB) {  // mask, max / min of this chunk, then keep it in TMEM (over its consumed D_0)
          mask_minmax_t<16>(s + so, t0 + kb + 16 * c, i, full, masked, mx, mn);
          uint32_t su[16];
#pragma unroll
          for (int x = 0; x < 16; ++x) su[x] = __float_as_uint(s[so + x]);
          ptx::tmem_st16(tS + sbo + lane_base + kb + 16 * c, su);
        }
      }
      if (WB) {
        ptx::tmem_wait_st();
      } else {
        ptx::tc_fence_before();
        ptx::mbar_arrive(&sm.s_free[jg % NSB]);  // S columns may now be overwritten by QK(j+1)
        mask_minmax_t<KPT>(s, t0 + kb, i, full, masked, mx, mn);
      }
      ptx::mbar_arrive(&sm.k_free[bj]);  // K' tile + key coefficients may be refilled
      sm.xch[jg & 1][sw][r] = make_float2(mx, masked ? -INFINITY : mn);
      ptx::named_bar_sync(qbar, QBN);
      bool any_masked = masked;
      if (masked) mn = INFINITY;
#pragma unroll
      for (int w2 = 1; w2 < NSG; ++w2) {  // the other warpgroups' keys of these rows
        const float2 o = sm.xch[jg & 1][(sw + w2) % NSG][r];
        mx = fmaxf(mx, o.x);
        any_masked |= o.y == -INFINITY;
        mn = fminf(mn, o.y == -INFINITY ? INFINITY : o.y);
      }
      // lazy rescaling: move the running max only when some row of this warp outgrew it by
      // more than kRescaleTh (identical decision in both S warps sharing these rows)
      float al = 1.f;
      const bool resc = __any_sync(0xffffffffu, mx > m_run + kRescaleTh);
      if (resc) {
        const float m_new = fmaxf(m_run, mx);
        al = (m_run == -INFINITY) ? 0.f : ex2(m_run - m_new);
        m_run = m_new;
      }
      // tile j-NB must be fully consumed by the O warps before its P / info slots are reused
      ptx::mbar_wait(&sm.o_done[bj], ph ^ 1);
      const bool committed = j < w.nfull;
      float pinv = 0.f, pnlo = 0.f, ps = 0.f, plo = 0.f;
      if (committed) {
        // (a6) P' per (row, V block): 8-bit on p~ (codes invariant to the row scale);
        // transient meta (never stored; the codes only need to agree up to near-ties, DESIGN
        // "Parity protocol"): multiply and a fast reciprocal instead of IEEE division
        plo = any_masked ? 0.f : ex2(mn - m_run);
        const float phi = ex2(mx - m_run);
        ps = (phi - plo) * (1.f / 255.f);
        pinv = __fdividef(255.f, phi - plo);
        if (!(ps > 1e-30f)) ps = pinv = 0.f;
        pnlo = -plo * pinv;
      }
      // ---- pass 2: p~ = 2^(S - m), row sum, P' codes (or the FP16 tail tile's p~ -> TMEM),
      // 16 keys at a time (issuing all exp2 first measured 2 % slower at Pi = 64)
      float2 ls2 = make_float2(0.f, 0.f);
      const float2 mneg = make_float2(-m_run, -m_run);
      uint32_t psum = 0;
      auto exp_chunk = [&](int so) {
#pragma unroll
        for (int kk = 0; kk < 16; kk += 2) {
          const float2 a2 = ptx::fadd2(make_float2(s[so + kk], s[so + kk + 1]), mneg);
#if (HACK_ABL & 8)
          s[so + kk] = a2.x;
          s[so + kk + 1] = a2.y;
#else
          s[so + kk] = ex2(a2.x);  // ex2(-inf) = +0 for masked keys
          s[so + kk + 1] = ex2(a2.y);
#endif
          ls2 = ptx::fadd2(ls2, make_float2(s[so + kk], s[so + kk + 1]));
        }
      };
      auto out_chunk = [&](int so, int c) {
        if (committed) {
          const uint4 cw = p_codes16<BITS, PSR>(s + so, pinv, pnlo, kc.seed, p_rid, p_c3, i, t0 + kb + 16 * c, psum);
          if (Gm::TP)
            ptx::tmem_st4(tmem + lane_base + Gm::TPC + bj * (BN / 4) + (kb + 16 * c) / 4, cw.x ^ 0x80808080u,
                          cw.y ^ 0x80808080u, cw.z ^ 0x80808080u, cw.w ^ 0x80808080u);
          else
            *reinterpret_cast<uint4*>(sm.p[bj] + kmaj_off(r, kb + 16 * c, SBO_T)) =
                make_uint4(cw.x ^ 0x80808080u, cw.y ^ 0x80808080u, cw.z ^ 0x80808080u, cw.w ^ 0x80808080u);
          if (DBG && dbg_pcodes != nullptr && pos < L) {
            uint8_t* dp = dbg_pcodes + ((int64_t)(start + pos) * kc.Hq + hq) * dbg_stride + t0 + kb + 16 * c;
            const uint32_t cwa[4] = {cw.x, cw.y, cw.z, cw.w};
#pragma unroll
            for (int p = 0; p < 16; ++p) dp[perm_src<BITS>(p)] = (uint8_t)((cwa[p >> 2] >> (8 * (p & 3))) & 0xFF);
          }
        } else {  // FP16 tail tile (the last one): p~ to the O warps through TMEM (no later QK)
          uint32_t su[16];
#pragma unroll
          for (int x = 0; x < 16; ++x) su[x] = __float_as_uint(s[so + x]);
          ptx::tmem_st16(tS + sbo + lane_base + kb + 16 * c, su);
        }
      };
      if (WB) {
#pragma unroll
        for (int c = 0; c < KPT / 16; ++c) {
          uint32_t su[16];
          ptx::tmem_ld16(tS + sbo + lane_base + kb + 16 * c, su);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int x = 0; x < 16; ++x) s[x] = __uint_as_float(su[x]);
          exp_chunk(0);
          out_chunk(0, c);
        }
      } else {
#pragma unroll
        for (int c = 0; c < KPT / 16; ++c) {
          exp_chunk(16 * c);
          out_chunk(16 * c, c);
        }
      }
      l_run = __fmaf_rn(l_run, al, ls2.x + ls2.y);
      if (Gm::TP || !committed) ptx::tmem_wait_st();
      if (Gm::TP || WB || !committed) ptx::tc_fence_before();
      if (WB) ptx::mbar_arrive(&sm.s_free[jg % NSB]);  // scores consumed: S may be overwritten by QK(j+1)
      sm.sp_part[bj][sw][r] = (int)psum;
      if (sw == 0) sm.pinfo[bj][r] = make_float4(al, resc ? 1.f : 0.f, ps, plo);
      if (committed && !Gm::TP) ptx::fence_proxy_async_smem();
      ptx::mbar_arrive(&sm.p_ready[bj]);              // for the MMA warp (PV)
      ptx::named_bar_arrive(kPBar0 + bj, NSW + NOW);  // for the O warps (hardware barrier: no polling)
    }
    ptx::mbar_wait(&sm.l_free, (it & 1) ^ 1);  // the O warps read the previous item's sums
    sm.lpart[sw][r] = l_run;
    ptx::mbar_arrive(&sm.l_ready);
    }
  } else {
    // ------------------------------------------------------------------ O warpgroups (2)
    // thread = query row r = TMEM lane; OW o owns output channels 64o..64o+63
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(Gm::REG_O));
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the FP16 tail is the ingest's output too
    const int ow = (warp - 4 - 4 * NSG) >> 2;
    const int r = (tid - OBASE) & (BM - 1);
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    const int cb = 64 * ow;
    int jg = 0, jpv = 0;  // tiles / PV tiles of all items so far
    Item w;
#pragma unroll 1
    for (int it = 0; get_item(it, w); ++it) {
    const int pos = w.i0 + (r & (pbp - 1)), hq = w.hq0 + r / pbp;
    const int L = w.L, start = w.start;
    float2 o2[32];  // channels cb + 2x, cb + 2x + 1
#pragma unroll
    for (int x = 0; x < 32; ++x) o2[x] = make_float2(0.f, 0.f);
#pragma unroll 1
    for (int j = 0; j < w.nkt; ++j, ++jg) {
      const int bj = jg % NB;
      const uint32_t ph = (jg / NB) & 1;
      ptx::named_bar_sync(kPBar0 + bj, NSW + NOW);  // S warps' P' and row info of tile j
      const float4 pi4 = sm.pinfo[bj][r];
      if (pi4.y != 0.f) {  // warp-uniform (lazy rescaling decided per S warp = same 32 rows)
        const float2 al2 = make_float2(pi4.x, pi4.x);
#pragma unroll
        for (int x = 0; x < 32; ++x) o2[x] = ptx::fmul2(o2[x], al2);
      }
      if (j < w.nfull) {
        const int bd = jpv % NDB;
        const uint32_t dph = (jpv / NDB) & 1;
        ++jpv;
        // (a7) O += (s_p/2) s_v E + s_p SP_s m_v + mu_p y_v on D' of this tile
        int sps = -128 * PI;  // sum (p' - 128)
#pragma unroll
        for (int w2 = 0; w2 < NSG; ++w2) sps += sm.sp_part[bj][w2][r];
        const float2 ap2 = make_float2(0.5f * pi4.z, 0.5f * pi4.z);
        const float2 xp2 = make_float2(pi4.z * (float)sps, pi4.z * (float)sps);
        const float mp = __fmaf_rn(128.f, pi4.z, pi4.w);
        const float2 mp2 = make_float2(mp, mp);
        ptx::mbar_wait(&sm.v_ready[bj], ph);
        ptx::mbar_wait(&sm.d_full[bd], dph);
        ptx::tc_fence_after();
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          uint32_t d[16];
          ptx::tmem_ld16(tD0 + 128 * bd + lane_base + cb + 16 * h, d);
          ptx::tmem_wait_ld();
          if (DBG && dbg_pv != nullptr && pos < L && (acc_head < 0 || hq == acc_head)) {  // E' = 2 D' - 256 SV
            const int hs = acc_head < 0 ? hq : 0, hn = acc_head < 0 ? kc.Hq : 1;
            int32_t* dp = dbg_pv + (((int64_t)(start + pos) * hn + hs) * (acc_stride / PI) + j) * 128 + cb + 16 * h;
#pragma unroll
            for (int x = 0; x < 16; ++x) dp[x] = (int32_t)(d[x] - 0x4B400000u);
          }
#if (HACK_ABL & 1)
          if (d[0] == 0x12345u) o2[h].x += 1.f;  // (ablation: no PV Eq. 4 math)
#else
#pragma unroll
          for (int x4 = 0; x4 < 4; ++x4) {
            const int c0 = cb + 16 * h + 4 * x4;
            const float4 sv4 = *reinterpret_cast<const float4*>(&sm.vcf[bj][0][c0]);
            const float4 mv4 = *reinterpret_cast<const float4*>(&sm.vcf[bj][1][c0]);
            const float4 y4 = *reinterpret_cast<const float4*>(&sm.vcf[bj][2][c0]);
#pragma unroll
            for (int pr = 0; pr < 2; ++pr) {
              const int xo = 4 * x4 + 2 * pr;
              const int oi = 8 * h + 2 * x4 + pr;
              const float2 E = acc2f(d[xo], d[xo + 1]);
              const float2 svp = pr ? make_float2(sv4.z, sv4.w) : make_float2(sv4.x, sv4.y);
              const float2 t = ptx::fmul2(svp, E);  // s_v 2D_s
              const float2 mvp = pr ? make_float2(mv4.z, mv4.w) : make_float2(mv4.x, mv4.y);
              const float2 yp = pr ? make_float2(y4.z, y4.w) : make_float2(y4.x, y4.y);
              float2 a = ptx::ffma2(ap2, t, o2[oi]);
              a = ptx::ffma2(xp2, mvp, a);
              o2[oi] = ptx::ffma2(mp2, yp, a);
            }
          }
#endif
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(&sm.d_free[bd]);
      } else {
        // FP16 last V block (RQE): O += sum_t p~_t v_t in fp32, p~ from the S warps
        // through TMEM (columns = the tile's local keys)
        ptx::tc_fence_after();
        const int T = L - w.nfull * PI;
        const __half* tail =
            reinterpret_cast<const __half*>(cv.v_tail) + ((int64_t)w.slot * kc.Hkv + w.hk) * PI * 128 + cb;
#pragma unroll 1
        for (int c = 0; 16 * c < T; ++c) {
          uint32_t pt16[16];
          ptx::tmem_ld16(tS + (uint32_t)(SBC * (jg % NSB)) + lane_base + 16 * c, pt16);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int x = 0; x < 16; ++x) {
            if (16 * c + x >= T) break;
            const float pt = __uint_as_float(pt16[x]);
            const uint4* vr = reinterpret_cast<const uint4*>(tail + (16 * c + x) * 128);
#pragma unroll
            for (int c8 = 0; c8 < 8; ++c8) {
              const uint4 raw = vr[c8];
              const __half2* h2 = reinterpret_cast<const __half2*>(&raw);
#pragma unroll
              for (int e = 0; e < 4; ++e)
                o2[c8 * 4 + e] = ptx::ffma2(make_float2(pt, pt), __half22float2(h2[e]), o2[c8 * 4 + e]);
            }
          }
        }
      }
      ptx::mbar_arrive(&sm.o_done[bj]);
    }
    ptx::mbar_wait(&sm.l_ready, it & 1);
    float lsum = sm.lpart[0][r];
#pragma unroll
    for (int w2 = 1; w2 < NSG; ++w2) lsum += sm.lpart[w2][r];
    const float inv_l = 1.f / lsum;
    ptx::mbar_arrive(&sm.l_free);
    if (pos < L) {
      const int64_t base = ((int64_t)(start + pos) * kc.Hq + hq) * 128 + cb;
      if (kc.out_fp32) {
        float4* op = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + base);
#pragma unroll
        for (int c4 = 0; c4 < 16; ++c4)
          op[c4] = make_float4(o2[2 * c4].x * inv_l, o2[2 * c4].y * inv_l, o2[2 * c4 + 1].x * inv_l,
                               o2[2 * c4 + 1].y * inv_l);
      } else {
        uint4* op = reinterpret_cast<uint4*>(reinterpret_cast<__half*>(out) + base);
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) {
          __half2 hh[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) hh[e] = __floats2half2_rn(o2[4 * c8 + e].x * inv_l, o2[4 * c8 + e].y * inv_l);
          op[c8] = *reinterpret_cast<uint4*>(hh);
        }
      }
    }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}

// HACK_PREFILL_PERSIST=0 forces one CTA per item (A/B runs); default persistent for batch 1.
bool persistent_enabled() {
  static const bool on = [] {
    const char* v = getenv("HACK_PREFILL_PERSIST");
    return v == nullptr || v[0] != '0';
  }();
  return on;
}

template <int PI_, int BITS>
cudaError_t launch_t(const KernelCfg& kc, const void* q, const int32_t* cu, const int32_t* slots, int batch,
                     int max_seqlen, const CacheView& cv, void* out, const hack_debug_t* dbg, cudaStream_t st,
                     bool pdl) {
  if (kc.pl.page_bytes != Geo<PI_, BITS>::PB) return cudaErrorInvalidValue;  // layout drift guard
  const size_t smem = sizeof(TcSmem<PI_, BITS>) + 1024;
  const bool with_dbg = dbg != nullptr && (dbg->pcodes != nullptr || dbg->qk_acc != nullptr || dbg->pv_acc != nullptr);
  const bool psr = kc.p_round == HACK_ROUND_STOCHASTIC;
  auto kern = with_dbg ? (psr ? prefill_tc_kernel<PI_, BITS, true, true> : prefill_tc_kernel<PI_, BITS, true, false>)
                       : (psr ? prefill_tc_kernel<PI_, BITS, false, true> : prefill_tc_kernel<PI_, BITS, false, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int gp = pack_heads(kc);
  cudaLaunchConfig_t lc = {};
  const int nqt = (max_seqlen + BM / gp - 1) / (BM / gp);
  int nitems = 0;  // persistent launch: one request, at most one CTA per SM looping over items
  if (batch == 1 && persistent_enabled()) {
    int dev = 0, nsm = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    nitems = min(nqt - kc.qt_begin, kc.qt_count) * (kc.hq_count / gp);
    if (nitems <= 0) return cudaSuccess;
    lc.gridDim = dim3(min(nitems, nsm), 1, 1);
  } else {
    if (min(nqt - kc.qt_begin, kc.qt_count) <= 0) return cudaSuccess;
    lc.gridDim = dim3(min(nqt - kc.qt_begin, kc.qt_count), kc.hq_count / gp, batch);
  }
  lc.blockDim = dim3(Geo<PI_, BITS>::THREADS);
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  // pdl: a programmatic dependent of the ingest just launched on `st` (hack_prefill_attention):
  // the Q quantization prologue (which reads only q and rng_ids) overlaps the ingest; the
  // producer and O warps wait in griddepcontrol.wait before they read pages or the FP16 tail.
  // Without pdl griddepcontrol.wait returns at once (the stream order already holds).
  // Not for the persistent launch: its one CTA per SM would share the SMs with the ingest
  // blocks and slow the ingest it waits for (C2 step measured 446 us with, 434 us without).
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = pdl && nitems == 0 ? 1 : 0;
  e = cudaLaunchKernelEx(&lc, kern, reinterpret_cast<const __half*>(q), cu, slots, cv, kc, out,
                         dbg ? dbg->pcodes : (uint8_t*)nullptr, dbg ? dbg->pcodes_stride : (int64_t)0,
                         dbg ? dbg->qk_acc : (int32_t*)nullptr, dbg ? dbg->pv_acc : (int32_t*)nullptr,
                         dbg ? dbg->acc_stride : (int64_t)0, dbg ? dbg->acc_head : -1, nitems);
  if (e != cudaSuccess) return e;
  note_launch();
  return cudaGetLastError();
}

}  // namespace

// query positions per work item of one request (the granularity of kc.qt_begin / qt_count)
int prefill_tc_tile_rows(const KernelCfg& kc) { return BM / pack_heads(kc); }

bool prefill_tc_supported(const KernelCfg& kc) {
  return (kc.Pi == 32 || kc.Pi == 64 || kc.Pi == 128) && kc.d == 128;
}

cudaError_t launch_prefill_tc(const KernelCfg& kc, const void* q, const int32_t* cu, const int32_t* slots, int batch,
                              int max_seqlen, const CacheView& cv, void* out, const hack_debug_t* dbg,
                              cudaStream_t st, bool pdl) {
  switch (kc.Pi * 8 + kc.bits) {
    case 32 * 8 + 2: return launch_t<32, 2>(kc, q, cu, slots, batch, max_seqlen, cv, out, dbg, st, pdl);
    case 32 * 8 + 4: return launch_t<32, 4>(kc, q, cu, slots, batch, max_seqlen, cv, out, dbg, st, pdl);
    case 64 * 8 + 2: return launch_t<64, 2>(kc, q, cu, slots, batch, max_seqlen, cv, out, dbg, st, pdl);
    case 64 * 8 + 4: return launch_t<64, 4>(kc, q, cu, slots, batch, max_seqlen, cv, out, dbg, st, pdl);
    case 128 * 8 + 2: return launch_t<128, 2>(kc, q, cu, slots, batch, max_seqlen, cv, out, dbg, st, pdl);
    case 128 * 8 + 4: return launch_t<128, 4>(kc, q, cu, slots, batch, max_seqlen, cv, out, dbg, st, pdl);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hack
