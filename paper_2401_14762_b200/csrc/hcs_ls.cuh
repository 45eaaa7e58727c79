// hcs_ls.cuh -- CTA-cooperative dense least squares, the device restatement of
// hypercs.kernels.least_squares (kernels.py:44-67):
//
//   q, r, piv = qr(b, economic, pivoting=True)                (LAPACK geqp3)
//   if m >= k and min|diag r| > RANK_RTOL * max|diag r|:  s[piv] = r^{-1} q^T y
//   else: minimum-norm solution (gelsd, cond = RANK_RTOL)
//
// Column-pivoted Householder QR exactly as LAPACK's unblocked dlaqp2 (pivot =
// first column of largest partial norm, partial-norm downdating with the
// sqrt(eps) recompute guard, dlarfg reflectors), with y carried along as an
// extra column so Q^T y needs no explicit Q.  The minimum-norm fallback is a
// complete orthogonal decomposition (QR with pivoting + RZ, as LAPACK gelsy)
// at the numerical rank {i : |R_ii| > RANK_RTOL * max |R_ii|}; it coincides
// with gelsd's solution for the rank-deficient cases the reference tests
// (duplicate / zero columns, underdetermined systems; test_kernels.py:65-100).
//
// Layout: B is row-major M x ld (ld >= K + 1), columns 0..K-1 the system,
// column K the right-hand side.  Threads own columns (column-parallel
// reflector application, serial over rows with 4 partial sums); every thread
// of the CTA must call ls_solve.  B may live in shared or global memory.
#pragma once
#include "hcs_common.cuh"

namespace hcs {

struct LsScratch {       // shared memory, each array sized >= K + 1
  double* vn1;
  double* vn2;
  double* z;
  int* perm;
  double* red;           // >= 2 * warps
  int* ipiv;             // 1 int
};

// CTA-wide sum of one double per thread (all threads get the result).
__device__ __forceinline__ double cta_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, W = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < W; ++i) s += red[i];
  return s;
}

// Solve; s[0..K) receives the solution (shared memory).  Returns 0 for the
// QR path, 1 for the minimum-norm fallback.  Ends with __syncthreads().
static __device__ __noinline__ int ls_solve(double* B, int ld, int M, int K, double* s, const LsScratch& sc) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int kk = M < K ? M : K;
  const double tol3z = 1.0536712127723509e-08;  // dlaqp2 TOL3Z = sqrt(dlamch('Epsilon')) = sqrt(2^-53)
  // initial column norms
  for (int c = tid; c < K; c += nt) {
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    int r = 0;
    for (; r + 3 < M; r += 4) {
      double b0 = B[r * ld + c], b1 = B[(r + 1) * ld + c], b2 = B[(r + 2) * ld + c], b3 = B[(r + 3) * ld + c];
      a0 += b0 * b0; a1 += b1 * b1; a2 += b2 * b2; a3 += b3 * b3;
    }
    for (; r < M; ++r) { double b0 = B[r * ld + c]; a0 += b0 * b0; }
    double nrm = sqrt((a0 + a1) + (a2 + a3));
    sc.vn1[c] = nrm;
    sc.vn2[c] = nrm;
    sc.perm[c] = c;
  }
  __syncthreads();
  for (int j = 0; j < kk; ++j) {
    // ---- pivot: first column of maximal partial norm (idamax) -------------
    if (tid < 32) {
      double best = -1.0;
      int bi = j;
      for (int c = j + tid; c < K; c += 32) {
        double v = sc.vn1[c];
        if (v > best) { best = v; bi = c; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        double ob = __shfl_xor_sync(0xffffffffu, best, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (tid == 0) sc.ipiv[0] = bi;
    }
    __syncthreads();
    const int pvt = sc.ipiv[0];
    if (pvt != j) {
      for (int r = tid; r < M; r += nt) {
        double t = B[r * ld + j];
        B[r * ld + j] = B[r * ld + pvt];
        B[r * ld + pvt] = t;
      }
      if (tid == 0) {
        int tp = sc.perm[j]; sc.perm[j] = sc.perm[pvt]; sc.perm[pvt] = tp;
        sc.vn1[pvt] = sc.vn1[j];
        sc.vn2[pvt] = sc.vn2[j];
      }
    }
    __syncthreads();
    // ---- reflector for column j (dlarfg) ---------------------------------
    double part = 0.0;
    for (int r = j + 1 + tid; r < M; r += nt) { double v = B[r * ld + j]; part += v * v; }
    const double xnorm = sqrt(cta_sum(part, sc.red));
    const double alpha = B[j * ld + j];
    double tau = 0.0;
    if (xnorm != 0.0) {
      const double beta = -copysign(hypot(alpha, xnorm), alpha);
      tau = (beta - alpha) / beta;
      const double scal = 1.0 / (alpha - beta);
      for (int r = j + 1 + tid; r < M; r += nt) B[r * ld + j] *= scal;
      __syncthreads();   // every thread has read alpha before it is overwritten
      if (tid == 0) B[j * ld + j] = beta;
    }
    __syncthreads();
    // ---- apply H = I - tau v v^T to columns j+1..K (K = rhs) --------------
    if (tau != 0.0) {
      for (int c = j + 1 + tid; c <= K; c += nt) {
        double w0 = B[j * ld + c], w1 = 0, w2 = 0, w3 = 0;
        int r = j + 1;
        for (; r + 2 < M; r += 3) {
          w1 += B[r * ld + j] * B[r * ld + c];
          w2 += B[(r + 1) * ld + j] * B[(r + 1) * ld + c];
          w3 += B[(r + 2) * ld + j] * B[(r + 2) * ld + c];
        }
        for (; r < M; ++r) w1 += B[r * ld + j] * B[r * ld + c];
        const double tw = tau * ((w0 + w1) + (w2 + w3));
        B[j * ld + c] -= tw;
        for (r = j + 1; r < M; ++r) B[r * ld + c] -= tw * B[r * ld + j];
      }
    }
    // ---- partial column norm downdate (dlaqp2) -----------------------------
    for (int c = j + 1 + tid; c < K; c += nt) {
      double v1 = sc.vn1[c];
      if (v1 != 0.0) {
        double temp = fabs(B[j * ld + c]) / v1;
        temp = 1.0 - temp * temp;
        temp = temp < 0.0 ? 0.0 : temp;
        const double ratio = v1 / sc.vn2[c];
        const double temp2 = temp * ratio * ratio;
        if (temp2 <= tol3z) {
          if (j + 1 < M) {
            double a0 = 0.0;
            for (int r = j + 1; r < M; ++r) { double b = B[r * ld + c]; a0 += b * b; }
            sc.vn1[c] = sqrt(a0);
            sc.vn2[c] = sc.vn1[c];
          } else {
            sc.vn1[c] = 0.0;
            sc.vn2[c] = 0.0;
          }
        } else {
          sc.vn1[c] = v1 * sqrt(temp);
        }
      }
    }
    __syncthreads();
  }
  // ---- rank decision (kernels.py:57-58) -----------------------------------
  double dmax = 0.0, dmin = INFINITY;
  for (int i = 0; i < kk; ++i) {
    double d = fabs(B[i * ld + i]);
    dmax = fmax(dmax, d);
    dmin = fmin(dmin, d);
  }
  const bool full = (M >= K) && (kk == K) && (dmin > kRankRtol * dmax);
  if (full) {
    // back substitution R z = (Q^T y)[:K], column-oriented (dtrsv 'U','N')
    if (tid < 32) {
      const int lane = tid;
      for (int i = lane; i < K; i += 32) sc.z[i] = B[i * ld + K];
      __syncwarp();
      for (int i = K - 1; i >= 0; --i) {
        const double zi = sc.z[i] / B[i * ld + i];
        __syncwarp();
        if (lane == 0) sc.z[i] = zi;
        for (int rr = lane; rr < i; rr += 32) sc.z[rr] -= zi * B[rr * ld + i];
        __syncwarp();
      }
      for (int i = lane; i < K; i += 32) s[sc.perm[i]] = sc.z[i];
    }
    __syncthreads();
    return 0;
  }
  // ---- minimum-norm fallback: RZ on the leading rk rows --------------------
  if (tid < 32) {
    const int lane = tid;
    int rk = 0;
    while (rk < kk && fabs(B[rk * ld + rk]) > kRankRtol * dmax) ++rk;
    double* taus = sc.vn2;   // reuse
    // annihilate R[i][rk..K) for i = rk-1 .. 0 with row reflectors on columns {i} U [rk, K)
    for (int i = rk - 1; i >= 0 && rk < K; --i) {
      double part = 0.0;
      for (int c = rk + lane; c < K; c += 32) { double v = B[i * ld + c]; part += v * v; }
      const double xn = sqrt(warp_sum(part));
      const double al = B[i * ld + i];
      double tau = 0.0;
      if (xn != 0.0) {
        const double beta = -copysign(hypot(al, xn), al);
        tau = (beta - al) / beta;
        const double scal = 1.0 / (al - beta);
        for (int c = rk + lane; c < K; c += 32) B[i * ld + c] *= scal;
        __syncwarp();
        if (lane == 0) B[i * ld + i] = beta;
      }
      __syncwarp();
      taus[i] = tau;
      if (tau != 0.0) {
        for (int rr = 0; rr < i; ++rr) {
          double p = 0.0;
          for (int c = rk + lane; c < K; c += 32) p += B[i * ld + c] * B[rr * ld + c];
          const double wv = warp_sum(p) + B[rr * ld + i];
          const double tw = tau * wv;
          __syncwarp();
          if (lane == 0) B[rr * ld + i] -= tw;
          for (int c = rk + lane; c < K; c += 32) B[rr * ld + c] -= tw * B[i * ld + c];
          __syncwarp();
        }
      }
    }
    __syncwarp();
    // T u = c[:rk]; z = [u; 0]
    for (int i = lane; i < K; i += 32) sc.z[i] = (i < rk) ? B[i * ld + K] : 0.0;
    __syncwarp();
    for (int i = rk - 1; i >= 0; --i) {
      const double zi = sc.z[i] / B[i * ld + i];
      __syncwarp();
      if (lane == 0) sc.z[i] = zi;
      for (int rr = lane; rr < i; rr += 32) sc.z[rr] -= zi * B[rr * ld + i];
      __syncwarp();
    }
    // z = H_{rk-1} ... H_0 [u; 0]
    if (rk < K) {
      for (int i = 0; i < rk; ++i) {
        const double tau = taus[i];
        if (tau == 0.0) continue;
        double p = 0.0;
        for (int c = rk + lane; c < K; c += 32) p += B[i * ld + c] * sc.z[c];
        const double wv = warp_sum(p) + sc.z[i];
        const double tw = tau * wv;
        __syncwarp();
        if (lane == 0) sc.z[i] -= tw;
        for (int c = rk + lane; c < K; c += 32) sc.z[c] -= tw * B[i * ld + c];
        __syncwarp();
      }
    }
    for (int i = lane; i < K; i += 32) s[sc.perm[i]] = sc.z[i];
  }
  __syncthreads();
  return 1;
}

}  // namespace hcs
