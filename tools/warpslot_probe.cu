// Which SM sub-partition does each warp of a 4-warp CTA land on, with four CTAs
// resident per SM?  Records (smid, %warpid) per warp; sub-partition = %warpid % 4.
#include <cstdio>
#include <vector>
__global__ void probe(int* out) {
  extern __shared__ char sm[];
  unsigned wid, smid;
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  sm[threadIdx.x] = 0;
  long long t = clock64();
  while (clock64() - t < 2000000) {}
  if ((threadIdx.x & 31) == 0) {
    int w = threadIdx.x >> 5;
    out[(blockIdx.x * 4 + w) * 2] = smid;
    out[(blockIdx.x * 4 + w) * 2 + 1] = wid;
  }
}
int main() {
  int nb = 148 * 4;
  int* d; cudaMalloc(&d, nb * 8 * sizeof(int));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 56 * 1024);
  probe<<<nb, 128, 56 * 1024>>>(d);
  std::vector<int> h(nb * 8);
  cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
  int hist[4][4] = {};  // [warp in CTA][warpid % 4]
  for (int b = 0; b < nb; ++b)
    for (int w = 0; w < 4; ++w) hist[w][h[(b * 4 + w) * 2 + 1] % 4]++;
  for (int w = 0; w < 4; ++w) printf("cta warp %d -> smsp histogram %d %d %d %d\n", w, hist[w][0], hist[w][1], hist[w][2], hist[w][3]);
  for (int b = 0; b < 8; ++b) printf("block %d sm %d warpids %d %d %d %d\n", b, h[b * 8], h[b * 8 + 1], h[b * 8 + 3], h[b * 8 + 5], h[b * 8 + 7]);
  return 0;
}
