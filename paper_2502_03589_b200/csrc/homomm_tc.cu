// homomm_tc.cu -- test export N9 on the tensor cores: Eq. 4 homomorphic matmul whose
// integer part D_beta = A'_beta B'_beta^T runs as tcgen05.mma kind::i8 (u8 x u8 -> s32)
// with the accumulator in TMEM, on codes unpacked into K-major smem tiles -- the same
// unpack / descriptor / MMA / tcgen05.ld path as the prefill kernel (prefill_tc.cu).
// One CTA = one 128 x 64 output tile; one d-block (Pi) of MMAs at a time.
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
  const int sbo = (Z / 16) * 128;
  uint8_t* As = smem;                         // [128 rows][Z] K-major
  uint8_t* Bs = smem + TM * Z;                // [64 cols][Z] K-major
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (TM + TN) * Z);
  uint32_t* tbase = reinterpret_cast<uint32_t*>(bar + 1);
  constexpr int qkm = (1 << BITS) - 1;

  // A (8-bit codes) in the permuted order of B's unpacking
  for (int e = tid; e < TM * (Z / 16); e += blockDim.x) {
    const int r = e / (Z / 16), g = e % (Z / 16);
    uint8_t v[16];
#pragma unroll
    for (int p = 0; p < 16; ++p) v[p] = (m0 + r < M) ? a[(int64_t)(m0 + r) * Z + 16 * g + perm_src<BITS>(p)] : 0;
    *reinterpret_cast<uint4*>(As + kmaj_off(r, 16 * g, sbo)) = *reinterpret_cast<uint4*>(v);
  }
  // B (packed columns) unpacked
  const int wpc = Z * BITS / 32;  // 32-bit packed words per column
  for (int e = tid; e < TN * wpc; e += blockDim.x) {
    const int col = e / wpc, w = e % wpc;
    const uint32_t word = (n0 + col < N) ? reinterpret_cast<const uint32_t*>(bp + (int64_t)(n0 + col) * (Z * BITS / 8))[w] : 0u;
    if (BITS == 2) {
      *reinterpret_cast<uint4*>(Bs + kmaj_off(col, 16 * w, sbo)) = unpack16_2b(word);
    } else {
      *reinterpret_cast<uint2*>(Bs + kmaj_off(col, 8 * w, sbo)) = unpack8_4b(word);
    }
  }
  if (tid == 0) {
    ptx::mbar_init(bar, 1);
    ptx::fence_mbar_init();
  }
  if (tid < 32) ptx::tmem_alloc(tbase, TN);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tbase;
  const uint32_t idesc = ptx::idesc_u8(TM, TN);
  const uint32_t a_base = ptx::smem_u32(As), b_base = ptx::smem_u32(Bs);
  const int nb = Z / Pi;
  const int row = m0 + tid;
  float acc[TN];
#pragma unroll
  for (int j = 0; j < TN; ++j) acc[j] = 0.f;
  for (int beta = 0; beta < nb; ++beta) {
    if (tid == 0) {
      ptx::tc_fence_after();
      for (int ks = 0; ks < Pi / 32; ++ks) {
        const uint32_t koff = (uint32_t)((beta * Pi + ks * 32) / 16) * 128;
        ptx::mma_u8(tmem, ptx::smem_desc_kmajor(a_base + koff, 128, sbo),
                    ptx::smem_desc_kmajor(b_base + koff, 128, sbo), idesc, ks > 0);
      }
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
      const float mua = ma.x + 127.5f * ma.y;
      const int rq = 2 * qkm * sa - Pi * 255 * qkm;
      const float xq = ma.y * ((float)sa - 127.5f * Pi);
#pragma unroll 8
      for (int j = 0; j < TN; ++j) {
        const int col = n0 + j;
        if (col >= N) continue;
        if (dblk) dblk[((int64_t)beta * M + row) * N + col] = (int32_t)d[j];
        const __half2 mbh = bm[(int64_t)col * nb + beta];
        const float mb = __low2float(mbh), sb = __high2float(mbh);
        const int sbs = sum_bytes == 1 ? (int)bs[(int64_t)col * nb + beta]
                                       : (int)reinterpret_cast<const uint16_t*>(bs)[(int64_t)col * nb + beta];
        const float mub = mb + 0.5f * qkm * sb;
        const int dc4 = 4 * (int)d[j] - rq - 510 * sbs;
        acc[j] += ma.y * 0.25f * sb * (float)dc4 + xq * mub + mua * (sb * ((float)sbs - 0.5f * qkm * Pi) + Pi * mub);
      }
    }
    ptx::tc_fence_before();
    __syncthreads();
  }
  if (row < M)
    for (int j = 0; j < TN; ++j)
      if (n0 + j < N) c[(int64_t)row * N + n0 + j] = acc[j];
  __syncthreads();
  if (tid < 32) ptx::tmem_dealloc(tmem, TN);
}

}  // namespace

cudaError_t launch_homomm_tc(const KernelCfg& kc, const uint8_t* a_codes, const float* a_meta, const uint16_t* a_sums,
                             const uint8_t* b_packed, const void* b_meta, const void* b_sums, int M, int N, int Z,
                             int32_t* d_blocks, float* c, cudaStream_t st) {
  const size_t smem = (size_t)(TM + TN) * Z + 16;
  dim3 grid((N + TN - 1) / TN, (M + TM - 1) / TM);
  const int sb = sum_bytes_for(kc.bits, kc.Pi);
  cudaError_t e;
  if (kc.bits == 2) {
    e = cudaFuncSetAttribute(homomm_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    homomm_tc_kernel<2><<<grid, 128, smem, st>>>(a_codes, (const float2*)a_meta, a_sums, b_packed,
                                                 (const __half2*)b_meta, (const uint8_t*)b_sums, sb, M, N, Z, kc.Pi,
                                                 d_blocks, c);
  } else {
    e = cudaFuncSetAttribute(homomm_tc_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    homomm_tc_kernel<4><<<grid, 128, smem, st>>>(a_codes, (const float2*)a_meta, a_sums, b_packed,
                                                 (const __half2*)b_meta, (const uint8_t*)b_sums, sb, M, N, Z, kc.Pi,
                                                 d_blocks, c);
  }
  note_launch();
  return cudaGetLastError();
}

}  // namespace hack
