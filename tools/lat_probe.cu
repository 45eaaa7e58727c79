// Dependent-chain latencies on sm_100a (cycles per op), single warp:
// DFMA, DADD, rsqrt(double), 1.0/x, shared load->use, generic load of shared,
// __syncwarp, __shfl_sync of a double, FFMA for reference.
#include <cstdio>
__device__ double sink;
__global__ void probe(long long* out, double seed) {
  __shared__ double sh[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sh[i] = 1.0 + i * 1e-3;
  __syncthreads();
  const int R = 256;
  double x = seed, y = 1.0000001;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < R; ++i) x = fma(x, y, 1e-9);
  t1 = clock64(); out[0] = t1 - t0;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < R; ++i) x = x + 1e-9;
  t1 = clock64(); out[1] = t1 - t0;
  // rsqrt chain
  t0 = clock64();
  for (int i = 0; i < R; ++i) x = rsqrt(x) + 0.5;
  t1 = clock64(); out[2] = t1 - t0;
  // division chain
  t0 = clock64();
  for (int i = 0; i < R; ++i) x = 1.0 / x + 0.5;
  t1 = clock64(); out[3] = t1 - t0;
  // shared pointer chase (index from value)
  int idx = threadIdx.x & 7;
  t0 = clock64();
  for (int i = 0; i < R; ++i) { double v = sh[idx]; idx = ((int)v) & 7; x += v; }
  t1 = clock64(); out[4] = t1 - t0;
  // generic pointer chase into shared
  volatile double* gp = (double*)(void*)sh;
  double* gpp = (double*)gp;
  idx = threadIdx.x & 7;
  t0 = clock64();
  for (int i = 0; i < R; ++i) { double v = gpp[idx]; idx = ((int)v) & 7; x += v; asm volatile("" ::: "memory"); }
  t1 = clock64(); out[5] = t1 - t0;
  // syncwarp
  t0 = clock64();
  for (int i = 0; i < R; ++i) __syncwarp();
  t1 = clock64(); out[6] = t1 - t0;
  // shfl double chain
  t0 = clock64();
  for (int i = 0; i < R; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1e-9;
  t1 = clock64(); out[7] = t1 - t0;
  float f = (float)seed, g = 1.0001f;
  t0 = clock64();
  for (int i = 0; i < R; ++i) f = fmaf(f, g, 1e-6f);
  t1 = clock64(); out[8] = t1 - t0;
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < R; ++i) x = x * y;
  t1 = clock64(); out[9] = t1 - t0;
  // store + syncwarp + load (shared RAW through memory)
  t0 = clock64();
  for (int i = 0; i < R; ++i) { if ((threadIdx.x & 31) == (i & 31)) sh[i & 63] = x; __syncwarp(); x += sh[(i & 63)]; }
  t1 = clock64(); out[10] = t1 - t0;
  // __syncthreads with one warp
  t0 = clock64();
  for (int i = 0; i < R; ++i) __syncthreads();
  t1 = clock64(); out[11] = t1 - t0;
  sink = x + f;
}
int main() {
  long long* d; cudaMalloc(&d, 16 * sizeof(long long));
  const char* nm[] = {"dfma", "dadd", "rsqrt+add", "rcp+add", "lds-chase", "ld-generic-shared-chase", "syncwarp", "shfl.f64+add", "ffma", "dmul", "sts-syncwarp-lds", "syncthreads(1 warp)"};
  for (int threads : {32, 128}) {
    probe<<<1, threads>>>(d, 1.5);
    probe<<<1, threads>>>(d, 1.5);
    long long h[16];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("block of %d threads (thread 0's chains):\n", threads);
    for (int i = 0; i < 12; ++i) printf("  %-26s %7.1f cycles/op\n", nm[i], h[i] / 256.0);
  }
  return 0;
}
