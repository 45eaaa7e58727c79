// FP64 peak microbenchmark for B200 (sm_100a): DFMA (CUDA cores) and DMMA
// (mma.sync f64 tensor path, m8n8k4 and m16n8k16).  Writes one JSON line.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int ILP>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int ILP>
__global__ void dmma884_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[ILP][2];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int ILP>
__global__ void dmma16816_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-4 * i;
  double c[ILP][4];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                   "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// dependent-chain latency (one warp): cycles per DMMA / DFMA / SHFL
__global__ void latency_kernel(long long* out, int iters, double a, double b) {
  double c0 = threadIdx.x, c1 = 1.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  long long t1 = clock64();
  double f = c0;
  for (int i = 0; i < iters; ++i) f = fma(f, a, b);
  long long t2 = clock64();
  double g = c1;
  for (int i = 0; i < iters; ++i) g = __shfl_xor_sync(0xffffffffu, g, 1) + 1.0;
  long long t3 = clock64();
  double h = c0 + 1.0;
  for (int i = 0; i < iters; ++i) h = sqrt(h) + 1.0;
  long long t4 = clock64();
  double q = c1 + 2.0;
  for (int i = 0; i < iters; ++i) q = 1.0 / q + 1.5;
  long long t5 = clock64();
  if (threadIdx.x == 0) {
    out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4;
    out[5] = (long long)(c0 + c1 + f + g + h + q);
  }
}


// warps alternate: even warps DMMA m8n8k4, odd warps DFMA — do the two FP64 paths share issue bandwidth?
__global__ void mixed_kernel(double* out, int iters, double a, double b) {
  int w = threadIdx.x >> 5;
  double s = 0;
  if (w & 1) {
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters * 2; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
  } else {
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = -i; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  }
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <typename K>
float time_kernel(K launch, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch();  // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 1024 * sizeof(double)));
  const int iters = 20000;
  printf("{\"gpu\": \"%s\", \"sms\": %d", prop.name, sms);
  for (int tpb : {256, 512, 1024}) {
    int blocks = sms * (2048 / tpb);
    float ms = time_kernel([&] { dfma_kernel<8><<<blocks, tpb>>>(out, iters, 0.999, 1e-3); }, 5);
    double flops = 2.0 * 8 * iters * (double)blocks * tpb;
    printf(", \"dfma_tflops_tpb%d\": %.2f", tpb, flops / ms / 1e9);
  }
  CK(cudaGetLastError());
  for (int tpb : {128, 256, 512}) {
    int blocks = sms * (1024 / tpb);
    float ms = time_kernel([&] { dmma884_kernel<8><<<blocks, tpb>>>(out, iters); }, 5);
    double flops = 2.0 * 8 * 8 * 4 * 8 * iters * (double)blocks * (tpb / 32);
    printf(", \"dmma884_tflops_tpb%d\": %.2f", tpb, flops / ms / 1e9);
  }
  CK(cudaGetLastError());
  for (int tpb : {128, 256, 512}) {
    int blocks = sms * (1024 / tpb);
    float ms = time_kernel([&] { dmma16816_kernel<4><<<blocks, tpb>>>(out, iters / 4); }, 5);
    double flops = 2.0 * 16 * 8 * 16 * 4 * (iters / 4) * (double)blocks * (tpb / 32);
    printf(", \"dmma16816_tflops_tpb%d\": %.2f", tpb, flops / ms / 1e9);
  }
  CK(cudaGetLastError());
  // sustained: DMMA for ~4 s
  {
    int blocks = sms * 4, tpb = 256;
    int it2 = 400000;
    float ms = time_kernel([&] { dmma884_kernel<8><<<blocks, tpb>>>(out, it2); }, 2);
    double flops = 2.0 * 8 * 8 * 4 * 8 * it2 * (double)blocks * (tpb / 32);
    printf(", \"dmma884_sustained_tflops\": %.2f, \"sustained_ms\": %.1f", flops / ms / 1e9, ms);
    ms = time_kernel([&] { dfma_kernel<8><<<blocks * 2, 512>>>(out, it2, 0.999, 1e-3); }, 2);
    flops = 2.0 * 8 * it2 * (double)blocks * 2 * 512;
    printf(", \"dfma_sustained_tflops\": %.2f", flops / ms / 1e9);
  }
  CK(cudaGetLastError());
  {
    long long* lat;
    CK(cudaMalloc(&lat, 8 * sizeof(long long)));
    const int it = 4096;
    latency_kernel<<<1, 32>>>(lat, it, 0.999, 1e-3);
    latency_kernel<<<1, 32>>>(lat, it, 0.999, 1e-3);
    long long h[8];
    CK(cudaMemcpy(h, lat, sizeof(h), cudaMemcpyDeviceToHost));
    printf(", \"lat_dmma_cyc\": %.1f, \"lat_dfma_cyc\": %.1f, \"lat_shfl_add_cyc\": %.1f, \"lat_dsqrt_add_cyc\": %.1f, \"lat_drcp_add_cyc\": %.1f",
           (double)h[0] / it, (double)h[1] / it, (double)h[2] / it, (double)h[3] / it, (double)h[4] / it);
  }
  {
    // mixed: 512 threads/CTA, 2 CTAs/SM; 8 DMMA warps (each 8*iters mma = 2048*8*iters FLOP... per warp 512 FLOP/mma)
    int blocks = sms * 2, tpb = 512;
    float ms_m = time_kernel([&] { mixed_kernel<<<blocks, tpb>>>(out, iters, 0.999, 1e-3); }, 5);
    double dmma_flops = 2.0 * 8 * 8 * 4 * 8 * iters * (double)blocks * (tpb / 64);
    double dfma_flops = 2.0 * 8 * 2 * iters * (double)blocks * (tpb / 2);
    float ms_d = time_kernel([&] { dmma884_kernel<8><<<blocks, tpb / 2>>>(out, iters); }, 5);
    printf(", \"mixed_ms\": %.3f, \"mixed_dmma_only_ms\": %.3f, \"mixed_total_tflops\": %.2f",
           ms_m, ms_d, (dmma_flops + dfma_flops) / ms_m / 1e9);
  }
  CK(cudaGetLastError());
  printf("}\n");
  return 0;
}
