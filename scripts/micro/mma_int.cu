// Microbenchmark: legacy mma.sync integer throughput on sm_100a (u8 m16n8k32 vs u4 m16n8k64),
// and a few ALU ops used by the decode unpack.  Prints clocks per warp-instruction per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int KIND>
__global__ void __launch_bounds__(512, 1) k(int iters, uint32_t* sink) {
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
  uint32_t b0 = threadIdx.x ^ 0x55u, b1 = threadIdx.x ^ 0x33u;
  uint32_t d[8][4] = {};
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (KIND == 0)
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+r"(d[c][0]), "+r"(d[c][1]), "+r"(d[c][2]), "+r"(d[c][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
      else
        asm volatile("mma.sync.aligned.m16n8k64.row.col.s32.u4.u4.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+r"(d[c][0]), "+r"(d[c][1]), "+r"(d[c][2]), "+r"(d[c][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    }
  }
  long long t1 = clock64();
  uint32_t s = 0;
  for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 0x12345) sink[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[1] = (uint32_t)(t1 - t0);
}

int main() {
  uint32_t* sink;
  cudaMalloc(&sink, 64);
  const int iters = 4096;
  for (int kind = 0; kind < 2; ++kind)
    for (int warps = 4; warps <= 16; warps *= 2) {
      uint32_t clk;
      for (int rep = 0; rep < 2; ++rep) {
        if (kind == 0) k<0><<<148, warps * 32>>>(iters, sink);
        else k<1><<<148, warps * 32>>>(iters, sink);
        cudaDeviceSynchronize();
      }
      cudaMemcpy(&clk, sink + 1, 4, cudaMemcpyDeviceToHost);
      const double insts = (double)iters * 8 * warps;
      const double macs = insts * 16 * 8 * (kind == 0 ? 32 : 64);
      printf("%s warps/SM=%2d: %.3f clk per mma per SM, %.0f MAC/clk/SM\n", kind == 0 ? "u8 m16n8k32" : "u4 m16n8k64",
             warps, clk / insts, macs / clk);
    }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
