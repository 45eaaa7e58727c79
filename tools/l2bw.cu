// L2-resident read bandwidth: every CTA streams the same `kb` KB buffer
// (16-byte __ldg per lane, like the convex engine's A fragments).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2bw tools/l2bw.cu && ./l2bw
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const double2* __restrict__ buf, int n2, int reps, double* out) {
  double2 acc = make_double2(0, 0);
  for (int r = 0; r < reps; ++r)
    for (int i = threadIdx.x + (blockIdx.x * 37 % 64) * 32; i < n2 + (blockIdx.x * 37 % 64) * 32; i += blockDim.x) {
      double2 v = __ldg(buf + (i % n2));
      acc.x += v.x; acc.y += v.y;
    }
  if (acc.x == 12345.0) out[0] = acc.y;
}
int main() {
  for (int kb : {64, 401, 4096}) {
    int n2 = kb * 1024 / 16;
    double2* buf; double* out;
    cudaMalloc(&buf, n2 * 16); cudaMemset(buf, 0, n2 * 16); cudaMalloc(&out, 8);
    for (int threads : {256, 512}) for (int per : {1, 2, 4}) {
      int grid = 148 * per, reps = 20;
      rd<<<grid, threads>>>(buf, n2, 2, out);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      rd<<<grid, threads>>>(buf, n2, reps, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double bytes = (double)grid * reps * n2 * 16;
      printf("buf %5d KB  grid %4d x %3d  %.2f TB/s\n", kb, grid, threads, bytes / ms / 1e9);
    }
    cudaFree(buf); cudaFree(out);
  }
}
