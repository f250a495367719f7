// Microbenchmark: tcgen05.ld (32x32b.x16) throughput per SM vs number of warps.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) k(int iters, unsigned long long* out, uint32_t* sink) {
  __shared__ uint32_t tbase;
  int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t t = tbase + (((uint32_t)(32 * (warp & 3))) << 16) + 16 * (warp >> 2) % 512;
  uint32_t acc = 0;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(t + (it & 7) * 16 * 4));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
    for (int x = 0; x < 16; ++x) acc += r[x];
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
}
template <int NW>
void run() {
  int iters = 4096, blocks = 148;
  unsigned long long* d; uint32_t* s;
  cudaMalloc(&d, blocks * 8); cudaMalloc(&s, blocks * NW * 32 * 4);
  k<NW><<<blocks, NW * 32>>>(iters, d, s);
  k<NW><<<blocks, NW * 32>>>(iters, d, s);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double bytes = (double)iters * NW * 32 * 16 * 4;
  printf("warps %2d: %.1f cycles/iter/warp-ld, %.1f B/cycle/SM  (%s)\n", NW, (double)h[0] / iters, bytes / h[0],
         cudaGetErrorString(cudaGetLastError()));
}
int main() { run<1>(); run<4>(); run<8>(); run<16>(); run<32>(); }
