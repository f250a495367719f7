// Which hardware warp slot (%warpid; SMSP = %warpid % 4) does each warp of co-resident CTAs
// get?  Launch like decode_pair: 592 CTAs x 128 threads, 56 KB smem (4 CTAs per SM).
#include <cstdio>
#include <cstdint>
__global__ void k(int* out, long long spin) {
  extern __shared__ char sm[];
  unsigned smid, wid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  long long t0 = clock64();
  while (clock64() - t0 < spin) {}
  if ((threadIdx.x & 31) == 0) {
    int* o = out + (blockIdx.x * 4 + threadIdx.x / 32) * 3;
    o[0] = smid; o[1] = wid; o[2] = sm[0];
  }
}
int main() {
  int* d; cudaMalloc(&d, 592 * 4 * 3 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 56 * 1024);
  k<<<592, 128, 56 * 1024>>>(d, 2000000);
  int h[592 * 12]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  int cnt[4][4] = {};  // [warp of CTA][smsp]
  for (int b = 0; b < 592; ++b) for (int w = 0; w < 4; ++w) cnt[w][h[(b * 4 + w) * 3 + 1] % 4]++;
  for (int w = 0; w < 4; ++w) printf("warp %d of CTA -> SMSP counts %d %d %d %d\n", w, cnt[w][0], cnt[w][1], cnt[w][2], cnt[w][3]);
  for (int b = 0; b < 8; ++b) printf("cta %d sm %d warpids %d %d %d %d\n", b, h[b*12], h[b*12+1], h[b*12+4], h[b*12+7], h[b*12+10]);
  return 0;
}
