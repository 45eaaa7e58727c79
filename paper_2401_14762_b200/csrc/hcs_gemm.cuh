// hcs_gemm.cuh -- FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) tile GEMM used
// by the batched shared-basis solvers.
//
// One CTA owns a tile of kSlots = 32 pixel columns.  A GEMM computes
//     Out[n, s] = sum_k Mat[n, k] * In[k, s],   n, k < Np (N padded to 16)
// where Mat is Psi or Psi^T (N x N, shared by every pixel, L2-resident) and
// In is the CTA's 32 pixel vectors held in shared memory.  Warp w owns output
// rows [16 w, 16 w + 16) for all 32 columns: 2 x 4 DMMA 8x8 accumulators.
//
// Mat is pre-arranged once per call ("fragment order") so that each warp's A
// fragments for one k-step are one coalesced 512-byte double2 load:
//     frag[(w * KS + ks) * 32 + lane] = (Mat[16w + lane/4][4ks + lane%4],
//                                        Mat[16w + 8 + lane/4][4ks + lane%4])
// In is stored in B-fragment order so the 4 B fragments of a k-step are
// conflict-free 256-byte shared loads:  in_idx(k, s) below.
#pragma once
#include "hcs_common.cuh"

namespace hcs {

constexpr int kSlots = 32;

__device__ __forceinline__ int in_idx(int k, int s) {
  return (((k >> 2) * 4 + (s >> 3)) << 5) + ((s & 7) << 2) + (k & 3);
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// Element coordinates of accumulator acc[rb][cb][i] held by `lane` of warp w.
__device__ __forceinline__ int acc_row(int w, int rb, int lane) { return 16 * w + 8 * rb + (lane >> 2); }
__device__ __forceinline__ int acc_col(int cb, int i, int lane) { return 8 * cb + 2 * (lane & 3) + i; }

// acc = Mat(rows of warp w) * In.  KS = Np / 4 (a multiple of 4).
__device__ __forceinline__ void tile_gemm(const double2* __restrict__ frag, const double* In, int KS,
                                          double (&acc)[2][4][2]) {
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const double2* fa = frag + (size_t)w * KS * 32 + lane;
#pragma unroll
  for (int rb = 0; rb < 2; ++rb)
#pragma unroll
    for (int cb = 0; cb < 4; ++cb) acc[rb][cb][0] = acc[rb][cb][1] = 0.0;
  double2 a[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = __ldg(fa + i * 32);
  for (int ks0 = 0; ks0 < KS; ks0 += 4) {
    double2 nxt[4];
    const bool more = ks0 + 4 < KS;
#pragma unroll
    for (int i = 0; i < 4; ++i) nxt[i] = more ? __ldg(fa + (ks0 + 4 + i) * 32) : a[i];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double* b = In + ((ks0 + i) << 7) + lane;
      double b0 = b[0], b1 = b[32], b2 = b[64], b3 = b[96];
      dmma(acc[0][0], a[i].x, b0);
      dmma(acc[1][0], a[i].y, b0);
      dmma(acc[0][1], a[i].x, b1);
      dmma(acc[1][1], a[i].y, b1);
      dmma(acc[0][2], a[i].x, b2);
      dmma(acc[1][2], a[i].y, b2);
      dmma(acc[0][3], a[i].x, b3);
      dmma(acc[1][3], a[i].y, b3);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = nxt[i];
  }
}

}  // namespace hcs
