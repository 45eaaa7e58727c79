// DMMA (mma.sync m8n8k4 f64) dependent-chain latency and issue interval on sm_100a:
// one warp (and 4 / 16 warps per CTA = 1 / 4 per scheduler) issuing R rounds of C
// independent accumulator chains.  cycles / (R * C) per DMMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_chain_probe tools/dmma_chain_probe.cu
#include <cstdio>
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <int C>
__global__ void probe(long long* out, double seed, int R) {
  double acc[C][2];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c][0] = acc[c][1] = seed * c;
  const double a = seed + threadIdx.x * 1e-3, b = 1.0 - seed;
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < R; ++r) {
#pragma unroll
    for (int c = 0; c < C; ++c) dmma(acc[c], a, b);
  }
  const long long t1 = clock64();
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[1] = 1;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}
template <int C>
void run(int warps, long long* d) {
  const int R = 512;
  probe<C><<<1, 32 * warps>>>(d, 0.5, R);
  probe<C><<<1, 32 * warps>>>(d, 0.5, R);
  long long h = 0;
  cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("warps/CTA %2d  chains/warp %d: %7.1f cycles per round, %6.1f cycles per DMMA (per warp)\n", warps, C,
         (double)h / R, (double)h / R / C);
}
int main() {
  long long* d;
  cudaMalloc(&d, 16);
  for (int w : {1, 4, 8, 16}) {
    run<1>(w, d); run<2>(w, d); run<4>(w, d); run<8>(w, d);
  }
  return 0;
}
