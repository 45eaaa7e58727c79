// Probe for the warp-per-pixel greedy plan: one warp forms the
// lower 8 x 8 tiles of the Gram B^T B of B = basis[mask, S] (M rows, K columns)
// by DMMA with its A/B fragments loaded straight from the L2-resident basis
// (no shared-memory copy of B), with 2, 4 or 8 k-steps of fragments in flight.  Reports cycles per
// Gram per warp and Grams per second for several warps-per-SM counts, and
// checks the tiles against a CPU Gram.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/gram_l2_probe tools/gram_l2_probe.cu
//   tools/gram_l2_probe [M=90] [K=28] [N=224]
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

constexpr int kMaxNB = 6;          // column blocks (K <= 48)
constexpr int kTiles = kMaxNB * (kMaxNB + 1) / 2;

// mask: P x M row indices; cols: P x K column indices; G out: P x kTiles x 64
template <int D>
__global__ void gram_l2_kernel(const double* __restrict__ basis, int N, int M, int K, int P,
                               const uint8_t* __restrict__ mask, const uint8_t* __restrict__ cols,
                               double* __restrict__ gout, long long* __restrict__ cyc, int reps) {
  extern __shared__ double sG[];   // warps x kTiles x 64
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gw = blockIdx.x * (blockDim.x >> 5) + w;
  if (gw >= P) return;
  double* G = sG + (size_t)w * kTiles * 64;
  const uint8_t* mk = mask + (size_t)gw * M;
  const uint8_t* cl = cols + (size_t)gw * K;
  const int nb = (K + 7) >> 3, M4 = (M + 3) & ~3;
  // this lane's column in each block and its k-row within each k-step
  int col[kMaxNB];
#pragma unroll
  for (int b = 0; b < kMaxNB; ++b) {
    const int c = 8 * b + (lane >> 2);
    col[b] = (b < nb && c < K) ? cl[c] : -1;
  }
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    double acc[kTiles][2];
#pragma unroll
    for (int t = 0; t < kTiles; ++t) acc[t][0] = acc[t][1] = 0.0;
    // fragments of k-step ks for every block: f[b] = B[4 ks + (lane & 3)][8 b + (lane >> 2)],
    // D k-steps in flight
    double f[D][kMaxNB];
    auto load = [&](int ks, double (&fr)[kMaxNB]) {
      const int r = 4 * ks + (lane & 3);
      const int row = r < M ? mk[r] : -1;
#pragma unroll
      for (int b = 0; b < kMaxNB; ++b)
        fr[b] = (b < nb && row >= 0 && col[b] >= 0) ? __ldg(basis + (size_t)row * N + col[b]) : 0.0;
    };
    auto mma = [&](const double (&fr)[kMaxNB]) {
      int t = 0;
#pragma unroll
      for (int bi = 0; bi < kMaxNB; ++bi)
#pragma unroll
        for (int bj = 0; bj <= bi; ++bj, ++t)
          if (bi < nb) dmma(acc[t], fr[bi], fr[bj]);
    };
    const int KS = M4 >> 2;
#pragma unroll
    for (int d = 0; d < D; ++d) load(d, f[d]);
    for (int ks = 0; ks < KS; ks += D) {
#pragma unroll
      for (int d = 0; d < D; ++d) {
        if (ks + d < KS) mma(f[d]);
        load(ks + d + D, f[d]);
      }
    }
    int t = 0;
#pragma unroll
    for (int bi = 0; bi < kMaxNB; ++bi)
#pragma unroll
      for (int bj = 0; bj <= bi; ++bj, ++t)
        if (bi < nb) {
          G[t * 64 + (2 * (lane & 3)) * 8 + (lane >> 2)] = acc[t][0];
          G[t * 64 + (2 * (lane & 3) + 1) * 8 + (lane >> 2)] = acc[t][1];
        }
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) cyc[gw] = (t1 - t0) / reps;
  for (int i = lane; i < kTiles * 64; i += 32) gout[(size_t)gw * kTiles * 64 + i] = G[i];
}

int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 90, K = argc > 2 ? atoi(argv[2]) : 28, N = argc > 3 ? atoi(argv[3]) : 224;
  if (K > 8 * kMaxNB || M > N) { fprintf(stderr, "K <= %d, M <= N\n", 8 * kMaxNB); return 1; }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  std::mt19937_64 rng(7);
  std::vector<double> basis((size_t)N * N);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  for (auto& v : basis) v = U(rng);
  const int reps = 20;
  double *d_basis, *d_g;
  uint8_t *d_mask, *d_cols;
  long long* d_cyc;
  cudaMalloc(&d_basis, basis.size() * 8);
  cudaMemcpy(d_basis, basis.data(), basis.size() * 8, cudaMemcpyHostToDevice);
  for (int depth : {2, 4, 8})
  for (int wps : {8, 12, 16}) {
    const int cta_warps = 4, ctas = sms * (wps / cta_warps), P = ctas * cta_warps;
    std::vector<uint8_t> mask((size_t)P * M), cols((size_t)P * K);
    std::vector<int> idx(N);
    for (int p = 0; p < P; ++p) {
      for (int i = 0; i < N; ++i) idx[i] = i;
      std::shuffle(idx.begin(), idx.end(), rng);
      std::sort(idx.begin(), idx.begin() + M);
      for (int i = 0; i < M; ++i) mask[(size_t)p * M + i] = (uint8_t)idx[i];
      std::shuffle(idx.begin(), idx.end(), rng);
      std::sort(idx.begin(), idx.begin() + K);
      for (int i = 0; i < K; ++i) cols[(size_t)p * K + i] = (uint8_t)idx[i];
    }
    cudaMalloc(&d_mask, mask.size());
    cudaMalloc(&d_cols, cols.size());
    cudaMalloc(&d_g, (size_t)P * kTiles * 64 * 8);
    cudaMalloc(&d_cyc, (size_t)P * 8);
    cudaMemcpy(d_mask, mask.data(), mask.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(d_cols, cols.data(), cols.size(), cudaMemcpyHostToDevice);
    const size_t smem = (size_t)cta_warps * kTiles * 64 * 8;
    auto launch = [&]() {
      if (depth == 2) gram_l2_kernel<2><<<ctas, 32 * cta_warps, smem>>>(d_basis, N, M, K, P, d_mask, d_cols, d_g, d_cyc, reps);
      else if (depth == 4) gram_l2_kernel<4><<<ctas, 32 * cta_warps, smem>>>(d_basis, N, M, K, P, d_mask, d_cols, d_g, d_cyc, reps);
      else gram_l2_kernel<8><<<ctas, 32 * cta_warps, smem>>>(d_basis, N, M, K, P, d_mask, d_cols, d_g, d_cyc, reps);
    };
    cudaFuncSetAttribute(gram_l2_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(gram_l2_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(gram_l2_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) { fprintf(stderr, "%s\n", cudaGetErrorString(err)); return 1; }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> cyc(P);
    std::vector<double> g((size_t)P * kTiles * 64);
    cudaMemcpy(cyc.data(), d_cyc, (size_t)P * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(g.data(), d_g, g.size() * 8, cudaMemcpyDeviceToHost);
    // check two pixels against a CPU Gram
    double maxerr = 0.0;
    for (int p : {0, P - 1}) {
      int t = 0;
      for (int bi = 0; bi < (K + 7) / 8; ++bi)
        for (int bj = 0; bj <= bi; ++bj, ++t)
          for (int i = 0; i < 8; ++i)
            for (int j = 0; j < 8; ++j) {
              const int ci = 8 * bi + i, cj = 8 * bj + j;
              double ref = 0.0;
              if (ci < K && cj < K)
                for (int r = 0; r < M; ++r)
                  ref += basis[(size_t)mask[(size_t)p * M + r] * N + cols[(size_t)p * K + ci]] *
                         basis[(size_t)mask[(size_t)p * M + r] * N + cols[(size_t)p * K + cj]];
              const double got = g[((size_t)p * kTiles + t) * 64 + j * 8 + i];
              maxerr = std::max(maxerr, std::abs(got - ref));
            }
    }
    double mean = 0.0;
    for (auto c : cyc) mean += (double)c;
    mean /= P;
    printf("depth %d warps/SM %2d: %6.0f cycles per Gram per warp (M=%d K=%d), %.3g Grams/s, max |err| %.1e\n", depth, wps, mean, M, K,
           (double)P * reps / (ms * 1e-3), maxerr);
    cudaFree(d_mask);
    cudaFree(d_cols);
    cudaFree(d_g);
    cudaFree(d_cyc);
  }
  return 0;
}
