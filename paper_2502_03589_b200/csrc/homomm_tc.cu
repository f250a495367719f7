// homomm_tc.cu -- test export N9 on the tensor cores: the Eq. 4 homomorphic matmul
// block by block with the prefill kernel's MMA configuration
// (prefill_tc.cu): per d-block beta, A' - 128 as s8 and the doubled b-bit codes 2 B' as
// u8 go through tcgen05.mma kind::i8 (s8 x u8 -> s32) into TMEM, so the accumulator is
// E = 2 D_beta - 256 SB_beta (HACK_ACC_S8_2B) and the epilogue is the prefill's centered
// Eq. 4:  C += (s_a / 2) s_b E + s_a (SA - 128 Pi) m_b + mu_a y_b,
//         mu_a = m_a + 128 s_a,  y_b = s_b SB + Pi m_b.
// d_blocks exports D_beta = (E + 256 SB) / 2, inverted from the MMA's own accumulator.
// One CTA = one 128 x 64 output tile; each block beta is staged on its own (any Z).
// There is no CUDA-core fallback.
#include "common.cuh"
#include "internal.h"
#include "tc_common.cuh"

namespace hack {

namespace {

constexpr int TM = 128, TN = 64;

template <int BITS>
__global__ void __launch_bounds__(128, 1) homomm_tc_kernel(
    const uint8_t* __restrict__ a, const float2* __restrict__ am, const uint16_t* __restrict__ as,
    const uint8_t* __restrict__ bp, const __half2* __restrict__ bm, const uint8_t* __restrict__ bs, int sum_bytes,
    int M, int N, int Z, int Pi, int32_t* __restrict__ dblk, float* __restrict__ c) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  const int sbo = (Pi / 16) * 128;              // one block's K extent per 8-row group
  uint8_t* As = smem;                           // [128 rows][Pi] K-major, s8 (a' - 128)
  uint8_t* Bs = smem + TM * Pi;                 // [64 cols][Pi] K-major, u8 (2 b')
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (TM + TN) * Pi);
  uint32_t* tbase = reinterpret_cast<uint32_t*>(bar + 1);
  const int nb = Z / Pi;

  if (tid == 0) {
    ptx::mbar_init(bar, 1);
    ptx::fence_mbar_init();
  }
  if (tid < 32) ptx::tmem_alloc(tbase, TN);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tbase;
  const uint32_t idesc = ptx::idesc_s8u8(TM, TN);
  const uint32_t a_base = ptx::smem_u32(As), b_base = ptx::smem_u32(Bs);
  const int row = m0 + tid;
  float acc[TN];
#pragma unroll
  for (int j = 0; j < TN; ++j) acc[j] = 0.f;
  const int wpb = Pi * BITS / 32;  // packed 32-bit words per column and block
  for (int beta = 0; beta < nb; ++beta) {
    // stage block beta: A' - 128 in the permuted order of B's unpacking (tc_common.cuh)
    for (int e = tid; e < TM * (Pi / 16); e += blockDim.x) {
      const int r = e / (Pi / 16), g = e % (Pi / 16);
      uint8_t v[16];
#pragma unroll
      for (int p = 0; p < 16; ++p)
        v[p] = (m0 + r < M) ? (uint8_t)(a[(int64_t)(m0 + r) * Z + beta * Pi + 16 * g + perm_src<BITS>(p)] ^ 0x80u)
                            : (uint8_t)0x80u;  // padding rows: code 128 -> 0
      *reinterpret_cast<uint4*>(As + kmaj_off(r, 16 * g, sbo)) = *reinterpret_cast<uint4*>(v);
    }
    for (int e = tid; e < TN * wpb; e += blockDim.x) {
      const int col = e / wpb, w = e % wpb;
      const uint32_t word =
          (n0 + col < N) ? reinterpret_cast<const uint32_t*>(bp + (int64_t)(n0 + col) * (Z * BITS / 8))[beta * wpb + w]
                         : 0u;
      if (BITS == 2)
        *reinterpret_cast<uint4*>(Bs + kmaj_off(col, 16 * w, sbo)) = unpack16_2b_x2(word);
      else
        *reinterpret_cast<uint2*>(Bs + kmaj_off(col, 8 * w, sbo)) = unpack8_4b_x2(word);
    }
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      ptx::tc_fence_after();
      for (int ks = 0; ks < Pi / 32; ++ks)
        ptx::mma_u8(tmem, ptx::smem_desc_kmajor(a_base + ks * 256, 128, sbo),
                    ptx::smem_desc_kmajor(b_base + ks * 256, 128, sbo), idesc, ks > 0);
      ptx::mma_commit(bar);
    }
    __syncwarp();
    ptx::mbar_wait(bar, beta & 1);
    ptx::tc_fence_after();
    uint32_t d[TN];
    // warp w reads TMEM lanes 32w..32w+31 (= its rows)
    const uint32_t taddr = tmem + ((uint32_t)(32 * (tid / 32)) << 16);
    ptx::tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(&d[0]));
    ptx::tmem_ld32(taddr + 32, *reinterpret_cast<uint32_t(*)[32]>(&d[32]));
    ptx::tmem_wait_ld();
    if (row < M) {
      const float2 ma = am[(int64_t)row * nb + beta];
      const int sa = as[(int64_t)row * nb + beta];
      const float ah = 0.5f * ma.y, xa = ma.y * (float)(sa - 128 * Pi), mua = fmaf(128.f, ma.y, ma.x);
#pragma unroll 8
      for (int j = 0; j < TN; ++j) {
        const int col = n0 + j;
        if (col >= N) continue;
        const int E = (int)d[j];
        const int sbs = sum_bytes == 1 ? (int)bs[(int64_t)col * nb + beta]
                                       : (int)reinterpret_cast<const uint16_t*>(bs)[(int64_t)col * nb + beta];
        if (dblk) dblk[((int64_t)beta * M + row) * N + col] = (E + 256 * sbs) / 2;
        const __half2 mbh = bm[(int64_t)col * nb + beta];
        const float mb = __low2float(mbh), sb = __high2float(mbh);
        const float yb = fmaf(sb, (float)sbs, Pi * mb);
        acc[j] += fmaf(ah * sb, (float)E, fmaf(xa, mb, mua * yb));
      }
    }
    ptx::tc_fence_before();
    __syncthreads();  // smem tiles and TMEM free for the next block
    ptx::tc_fence_after();
  }
  if (row < M)
    for (int j = 0; j < TN; ++j)
      if (n0 + j < N) c[(int64_t)row * N + n0 + j] = acc[j];
  __syncthreads();
  if (tid < 32) ptx::tmem_dealloc(tmem, TN);
}

template <int BITS>
cudaError_t launch_t(const KernelCfg& kc, const uint8_t* a_codes, const float* a_meta, const uint16_t* a_sums,
                     const uint8_t* b_packed, const void* b_meta, const void* b_sums, int M, int N, int Z,
                     int32_t* d_blocks, float* c, cudaStream_t st) {
  const size_t smem = (size_t)(TM + TN) * kc.Pi + 16;
  dim3 grid((N + TN - 1) / TN, (M + TM - 1) / TM);
  cudaError_t e = cudaFuncSetAttribute(homomm_tc_kernel<BITS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  homomm_tc_kernel<BITS><<<grid, 128, smem, st>>>(a_codes, (const float2*)a_meta, a_sums, b_packed,
                                                  (const __half2*)b_meta, (const uint8_t*)b_sums,
                                                  sum_bytes_for(kc.bits, kc.Pi), M, N, Z, kc.Pi, d_blocks, c);
  note_launch();
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_homomorphic_matmul(const KernelCfg& kc, const uint8_t* a_codes, const float* a_meta,
                                      const uint16_t* a_sums, const uint8_t* b_packed, const void* b_meta,
                                      const void* b_sums, int M, int N, int Z, int32_t* d_blocks, float* c,
                                      cudaStream_t st) {
  if (kc.bits == 2)
    return launch_t<2>(kc, a_codes, a_meta, a_sums, b_packed, b_meta, b_sums, M, N, Z, d_blocks, c, st);
  return launch_t<4>(kc, a_codes, a_meta, a_sums, b_packed, b_meta, b_sums, M, N, Z, d_blocks, c, st);
}

}  // namespace hack
