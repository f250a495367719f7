// homomm.cu -- test export N9: Eq. 4 homomorphic matmul on arbitrary codes.
//
// C[i][j] = sum_beta Eq. 4 over Pi-blocks of the inner dim, with
// the exact int32 per-block partials D_beta = sum_{z in beta} a'_iz b'_zj exported for
// bit-exact comparison.  A: 8-bit codes (Q-like, fp32 meta); B: kv_bits codes packed
// per column (K-like, fp16 meta).  Uses the same centered evaluation as the attention
// kernels.
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace hack {

namespace {

template <int BITS>
__global__ void homomm_kernel(const uint8_t* __restrict__ a, const float2* __restrict__ am,
                              const uint16_t* __restrict__ as, const uint8_t* __restrict__ bp,
                              const __half2* __restrict__ bm, const uint8_t* __restrict__ bs, int sum_bytes,
                              int M, int N, int Z, int Pi, int32_t* __restrict__ dblk, float* __restrict__ c) {
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M || j >= N) return;
  constexpr int qkm = (1 << BITS) - 1;
  const int nb = Z / Pi;
  const uint8_t* arow = a + (int64_t)i * Z;
  const uint8_t* bcol = bp + (int64_t)j * (Z * BITS / 8);
  float acc = 0.f;
  for (int beta = 0; beta < nb; ++beta) {
    uint32_t d = 0;
    for (int w = beta * (Pi / 4); w < (beta + 1) * (Pi / 4); ++w) {
      uint32_t bw;
      if (BITS == 2) {
        const uint32_t x = bcol[w];
        bw = (x & 3u) | ((x >> 2) & 3u) << 8 | ((x >> 4) & 3u) << 16 | ((x >> 6) & 3u) << 24;
      } else {
        const uint32_t x = reinterpret_cast<const uint16_t*>(bcol)[w];
        bw = (x & 15u) | ((x >> 4) & 15u) << 8 | ((x >> 8) & 15u) << 16 | ((x >> 12) & 15u) << 24;
      }
      d = __dp4a(reinterpret_cast<const uint32_t*>(arow)[w], bw, d);
    }
    if (dblk) dblk[((int64_t)beta * M + i) * N + j] = (int32_t)d;
    const float2 ma = am[(int64_t)i * nb + beta];
    const int sa = as[(int64_t)i * nb + beta];
    const __half2 mbh = bm[(int64_t)j * nb + beta];
    const float mb = __low2float(mbh), sb = __high2float(mbh);
    const int sbs = sum_bytes == 1 ? (int)bs[(int64_t)j * nb + beta]
                                   : (int)reinterpret_cast<const uint16_t*>(bs)[(int64_t)j * nb + beta];
    const float mua = ma.x + 127.5f * ma.y, mub = mb + 0.5f * qkm * sb;
    const int dc4 = 4 * (int)d - (2 * qkm * sa - Pi * 255 * qkm) - 510 * sbs;
    acc += ma.y * 0.25f * sb * (float)dc4 + ma.y * ((float)sa - 127.5f * Pi) * mub +
           mua * (sb * ((float)sbs - 0.5f * qkm * Pi) + Pi * mub);
  }
  c[(int64_t)i * N + j] = acc;
}

}  // namespace

cudaError_t launch_homomm_tc(const KernelCfg& kc, const uint8_t* a_codes, const float* a_meta, const uint16_t* a_sums,
                             const uint8_t* b_packed, const void* b_meta, const void* b_sums, int M, int N, int Z,
                             int32_t* d_blocks, float* c, cudaStream_t st);

cudaError_t launch_homomorphic_matmul(const KernelCfg& kc, const uint8_t* a_codes, const float* a_meta,
                                      const uint16_t* a_sums, const uint8_t* b_packed, const void* b_meta,
                                      const void* b_sums, int M, int N, int Z, int32_t* d_blocks, float* c,
                                      cudaStream_t st) {
  // tcgen05 path (the prefill kernel's MMA core) unless HACK_HOMOMM_IMPL=simt
  const char* impl = getenv("HACK_HOMOMM_IMPL");
  if (Z <= 512 && !(impl && impl[0] == 's'))
    return launch_homomm_tc(kc, a_codes, a_meta, a_sums, b_packed, b_meta, b_sums, M, N, Z, d_blocks, c, st);
  dim3 blk(32, 8), grid((N + 31) / 32, (M + 7) / 8);
  const int sb = sum_bytes_for(kc.bits, kc.Pi);
  if (kc.bits == 2)
    homomm_kernel<2><<<grid, blk, 0, st>>>(a_codes, (const float2*)a_meta, a_sums, b_packed, (const __half2*)b_meta,
                                           (const uint8_t*)b_sums, sb, M, N, Z, kc.Pi, d_blocks, c);
  else
    homomm_kernel<4><<<grid, blk, 0, st>>>(a_codes, (const float2*)a_meta, a_sums, b_packed, (const __half2*)b_meta,
                                           (const uint8_t*)b_sums, sb, M, N, Z, kc.Pi, d_blocks, c);
  note_launch();
  return cudaGetLastError();
}

}  // namespace hack
