// hcs_batched.cu -- batched forms of the reference's numeric kernels
// (hypercs/kernels.py:14-76), the Lipschitz constant (transform.py:176-217)
// and the PSNR partial sums (metrics.py:30-55).  These back the kernel-level
// parity tests and the output-side PSNR; the solvers use the same device
// routines inline.
#include "hcs_gemm.cuh"
#include "hcs_internal.cuh"
#include "hcs_ls.cuh"
#include "hcs_ls_csne.cuh"

namespace hcs {

#ifdef HCS_PHASES
__device__ unsigned long long g_phase_ls[16];
#endif

__global__ void soft_kernel(long long n, const double* __restrict__ v, double t, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = soft(v[i], t);
}

cudaError_t launch_soft(long long n, const double* v, double t, double* out, cudaStream_t stream) {
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  soft_kernel<<<(int)blocks, 256, 0, stream>>>(n, v, t, out);
  return cudaGetLastError();
}

// one warp per row
__global__ void argmax_k_kernel(long long P, int n, const double* __restrict__ v, int k, int32_t* __restrict__ idx) {
  __shared__ double row[4][kMaxN];
  __shared__ uint32_t bm[4][8];
  __shared__ int list[4][kMaxN];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (long long p = blockIdx.x * 4LL + w; p < P; p += (long long)gridDim.x * 4) {
    for (int i = lane; i < n; i += 32) row[w][i] = v[p * n + i];
    __syncwarp();
    warp_topk(row[w], n, k, bm[w]);
    const int cnt = [&] {
      int base = 0;
      for (int e = 0; e < 8; ++e) {
        const uint32_t word = bm[w][e];
        if ((word >> lane) & 1u) list[w][base + __popc(word & ((1u << lane) - 1u))] = 32 * e + lane;
        base += __popc(word);
      }
      return base;
    }();
    __syncwarp();
    for (int i = lane; i < cnt; i += 32) idx[p * k + i] = list[w][i];
    __syncwarp();
  }
}

cudaError_t launch_argmax_k(long long P, int n, const double* v, int k, int32_t* idx, cudaStream_t stream) {
  long long blocks = (P + 3) / 4;
  if (blocks > 148 * 8) blocks = 148 * 8;
  argmax_k_kernel<<<(int)blocks, 128, 0, stream>>>(P, n, v, k, idx);
  return cudaGetLastError();
}

// one CTA per system; b_p row-major M x K, y_p length M.  CSNE first (path 0),
// the exact pivoted restatement when a guard trips (path 0 if that is full
// rank, 1 for the minimum-norm fallback).
struct LsShared {
  double red[16];
  int ipiv, flag, ctr;   // ctr must follow flag: ls_csne's Gram tile counter (flag[1])
};

__host__ __device__ inline size_t ls_batched_doubles(int M, int K) {
  const size_t blk = (size_t)csne_ld(M) * csne_cols(K), piv = (size_t)M * ((K + 1) | 1);
  return blk > piv ? blk : piv;
}

// gscr: per-CTA global scratch for B and its Gram when the system does not
// fit in shared memory (nullptr: both in shared memory)
__global__ void __launch_bounds__(128) ls_kernel(long long P, int M, int K, const double* __restrict__ b,
                                                 const double* __restrict__ y, double* __restrict__ s,
                                                 int32_t* __restrict__ path, double* gscr) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const size_t sys = ls_batched_doubles(M, K) + csne_gram_doubles(K);
  double* B = gscr ? gscr + (size_t)blockIdx.x * sys : reinterpret_cast<double*>(smraw);
  double* G = B + ls_batched_doubles(M, K);
  double* rv = gscr ? reinterpret_cast<double*>(smraw) : G + csne_gram_doubles(K);
  double* sv = rv + M + 1;
  double* vn1 = sv + K + 9;
  double* vn2 = vn1 + K + 9;
  double* zt = vn2 + K + 9;
  LsShared* sh = reinterpret_cast<LsShared*>(zt + K + 9);
  int* perm = reinterpret_cast<int*>(sh + 1);
  const LsScratch sc{vn1, vn2, zt, perm, sh->red, &sh->ipiv};
  const CsneScratch cs{G, vn1, vn2, rv, sh->red, &sh->flag};
  const int ldb = csne_ld(M), nc = csne_cols(K), ldp = (K + 1) | 1;
#ifdef HCS_PHASES
  long long hcs_ph[16] = {0};
  hcs_ph[15] = clock64();
  long long* php = hcs_ph;
#else
  long long* php = nullptr;
#endif
  for (long long p = blockIdx.x; p < P; p += gridDim.x) {
    int pth = 0;
    bool done = false;
    if (M >= K) {
      if (threadIdx.x == 0) sh->ctr = 1;
      for (int idx = threadIdx.x; idx < ldb * nc; idx += blockDim.x) {
        const int c = idx / ldb, rr = idx - c * ldb;
        double v = 0.0;
        if (rr < M) v = c < K ? b[(p * M + rr) * K + c] : (c == K ? y[p * M + rr] : 0.0);
        B[idx] = v;
      }
      __syncthreads();
      HCS_MARKP(php, 3);
      done = ls_csne(B, ldb, M, K, sv, cs, php);
    }
    if (!done) {
      for (int idx = threadIdx.x; idx < M * (K + 1); idx += blockDim.x) {
        const int rr = idx / (K + 1), c = idx - rr * (K + 1);
        B[rr * ldp + c] = (c < K) ? b[(p * M + rr) * K + c] : y[p * M + rr];
      }
      __syncthreads();
      pth = ls_solve(B, ldp, M, K, sv, sc);
    }
    for (int c = threadIdx.x; c < K; c += blockDim.x) s[p * K + c] = sv[c];
    if (path && threadIdx.x == 0) path[p] = pth;
    __syncthreads();
    HCS_MARKP(php, 10);
  }
#ifdef HCS_PHASES
  if (threadIdx.x == 0)
    for (int k = 0; k < 15; ++k) atomicAdd(&g_phase_ls[k], (unsigned long long)hcs_ph[k]);
#endif
}

cudaError_t launch_batched_ls(long long P, int M, int K, const double* b, const double* y, double* s, int32_t* path,
                              cudaStream_t stream) {
  const size_t sys = ls_batched_doubles(M, K) + csne_gram_doubles(K);
  const size_t vecs = sizeof(double) * (M + 1 + 4 * (K + 9)) + sizeof(LsShared) + sizeof(int) * (K + 2);
  size_t smem = sizeof(double) * sys + vecs;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long blocks = P < 4LL * sms ? P : 4LL * sms;
  // systems whose matrix and Gram exceed shared memory keep both in a
  // stream-ordered global scratch (one per CTA); only the vectors stay shared
  double* gscr = nullptr;
  if (smem > 220 * 1024) {
    smem = vecs;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&gscr), sizeof(double) * sys * blocks, stream);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = cudaFuncSetAttribute(ls_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) {
    ls_kernel<<<(int)blocks, 128, smem, stream>>>(P, M, K, b, y, s, path, gscr);
    e = cudaGetLastError();
  }
  if (gscr) {
    cudaError_t f = cudaFreeAsync(gscr, stream);
    if (e == cudaSuccess) e = f;
  }
  return e;
}

// masks must be strictly increasing band indices < N (the reference's
// Dictionary rows, transform.py:106-113): one thread per pixel row; any
// violation sets kErrMask in the workspace error word, and every solver
// kernel of the call then exits before reading a mask
__global__ void validate_masks_kernel(long long P, int M, int N, const uint8_t* __restrict__ mask, int* err) {
  int bad = 0;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < P; p += (long long)gridDim.x * blockDim.x) {
    const uint8_t* row = mask + p * M;
    int prev = -1;
    for (int j = 0; j < M; ++j) {
      const int v = row[j];
      bad |= (v <= prev) | (v >= N);
      prev = v;
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, kErrMask);
}

cudaError_t launch_validate_masks(long long P, int M, int N, const uint8_t* mask, int* err, int sms,
                                  cudaStream_t stream) {
  long long blocks = (P + 255) / 256;
  if (blocks > 8LL * sms) blocks = 8LL * sms;
  if (blocks < 1) blocks = 1;
  validate_masks_kernel<<<(int)blocks, 256, 0, stream>>>(P, M, N, mask, err);
  return cudaGetLastError();
}

// max_ij |(Psi^T Psi - I)_ij| of an N x N basis: one thread per entry, the
// maximum by an atomic on the (non-negative) double's bits
__global__ void basis_gram_dev_kernel(int N, const double* __restrict__ basis, unsigned long long* out) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < N * N; idx += gridDim.x * blockDim.x) {
    const int i = idx / N, j = idx - i * N;
    double s = 0.0;
    for (int k = 0; k < N; ++k) s = fma(basis[(size_t)k * N + i], basis[(size_t)k * N + j], s);
    double dev = fabs(s - (i == j ? 1.0 : 0.0));
    if (dev != dev) dev = INFINITY;
    atomicMax(out, (unsigned long long)__double_as_longlong(dev));
  }
}

cudaError_t launch_basis_gram_dev(int N, const double* basis, unsigned long long* out, cudaStream_t stream) {
  basis_gram_dev_kernel<<<(N * N + 255) / 256, 256, 0, stream>>>(N, basis, out);
  return cudaGetLastError();
}

__global__ void rdelta_kernel(long long P, int n, const double* __restrict__ r, const double* __restrict__ rp,
                              double* __restrict__ out) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (long long p = blockIdx.x * 4LL + w; p < P; p += (long long)gridDim.x * 4) {
    double s = 0.0;
    for (int i = lane; i < n; i += 32) {
      const double d = r[p * n + i] - rp[p * n + i];
      s += d * d;
    }
    s = warp_sum(s);
    if (lane == 0) out[p] = sqrt(s);
  }
}

cudaError_t launch_rdelta(long long P, int n, const double* r, const double* rp, double* out, cudaStream_t stream) {
  long long blocks = (P + 3) / 4;
  if (blocks > 148 * 8) blocks = 148 * 8;
  rdelta_kernel<<<(int)blocks, 128, 0, stream>>>(P, n, r, rp, out);
  return cudaGetLastError();
}

__global__ void lipschitz_kernel(long long P, int N, int M, const double* __restrict__ basis,
                                 const uint8_t* __restrict__ mask, double* __restrict__ out) {
  __shared__ double u0[kMaxN];
  __shared__ uint8_t msk[4][kMaxN];
  const double inv = 1.0 / sqrt((double)N);
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < N; ++k) s += basis[(size_t)j * N + k] * inv;
    u0[j] = s;
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (long long p = blockIdx.x * 4LL + w; p < P; p += (long long)gridDim.x * 4) {
    for (int j = lane; j < M; j += 32) msk[w][j] = mask[p * M + j];
    __syncwarp();
    const double L = warp_lipschitz(u0, msk[w], M);
    if (lane == 0) out[p] = L;
    __syncwarp();
  }
}

cudaError_t launch_lipschitz(long long P, int N, int M, const double* basis, const uint8_t* mask, double* out,
                             cudaStream_t stream) {
  long long blocks = (P + 3) / 4;
  if (blocks > 148 * 2) blocks = 148 * 2;
  lipschitz_kernel<<<(int)blocks, 128, 0, stream>>>(P, N, M, basis, mask, out);
  return cudaGetLastError();
}

// PSNR partials: tiles of 32 pixels, rec = Psi x by the DMMA tile GEMM with A
// fragments read straight from the row-major basis (L1/L2 resident).
__global__ void __launch_bounds__(512) psnr_kernel(long long P, int N, int Np, const double* __restrict__ ref,
                                                   const double* __restrict__ x, const double* __restrict__ basis,
                                                   double* sse, double* amax) {
  extern __shared__ __align__(16) unsigned char smraw[];
  double* In = reinterpret_cast<double*>(smraw);
  __shared__ double red[32];
  __shared__ double redm[32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
  const int KS = Np >> 2;
  double local = 0.0, lmax = 0.0;
  for (long long t0 = blockIdx.x * (long long)kSlots; t0 < P; t0 += (long long)gridDim.x * kSlots) {
    for (int idx = threadIdx.x; idx < Np * kSlots; idx += blockDim.x) {
      const int s = idx / Np, n = idx - s * Np;
      const long long p = t0 + s;
      In[in_idx(n, s)] = (p < P && n < N) ? x[p * N + n] : 0.0;
    }
    __syncthreads();
    double acc[2][4][2];
#pragma unroll
    for (int rb = 0; rb < 2; ++rb)
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) acc[rb][cb][0] = acc[rb][cb][1] = 0.0;
    for (int ks = 0; ks < KS; ++ks) {
      const int c = 4 * ks + (lane & 3);
      const int r0 = 16 * w + (lane >> 2), r1 = r0 + 8;
      const double a0 = (r0 < N && c < N) ? __ldg(basis + (size_t)r0 * N + c) : 0.0;
      const double a1 = (r1 < N && c < N) ? __ldg(basis + (size_t)r1 * N + c) : 0.0;
      const double* b = In + (ks << 7) + lane;
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) {
        dmma(acc[0][cb], a0, b[32 * cb]);
        dmma(acc[1][cb], a1, b[32 * cb]);
      }
    }
#pragma unroll
    for (int rb = 0; rb < 2; ++rb)
#pragma unroll
      for (int cb = 0; cb < 4; ++cb)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int n = acc_row(w, rb, lane), s = acc_col(cb, i, lane);
          const long long p = t0 + s;
          if (p < P && n < N) {
            const double f = ref[p * N + n];
            const double d = f - acc[rb][cb][i];
            local += d * d;
            lmax = fmax(lmax, fabs(f));
          }
        }
    __syncthreads();
  }
  local = warp_sum(local);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lmax = fmax(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
  if (lane == 0) { red[w] = local; redm[w] = lmax; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0, m = 0.0;
    for (int i = 0; i < W; ++i) { s += red[i]; m = fmax(m, redm[i]); }
    atomicAdd(sse, s);
    // non-negative doubles order like their bit patterns
    atomicMax(reinterpret_cast<unsigned long long*>(amax), (unsigned long long)__double_as_longlong(m));
  }
}

cudaError_t launch_psnr(long long P, int N, const double* ref, const double* x, const double* basis, double* sse,
                        double* amax, cudaStream_t stream) {
  const int Np = (N + 15) & ~15;
  const size_t smem = sizeof(double) * (size_t)Np * kSlots;
  cudaError_t e = cudaFuncSetAttribute(psnr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  long long tiles = (P + kSlots - 1) / kSlots;
  int blocks = (int)(tiles < 148 * 2 ? tiles : 148 * 2);
  psnr_kernel<<<blocks, 2 * Np, smem, stream>>>(P, N, Np, ref, x, basis, sse, amax);
  return cudaGetLastError();
}


// Coefficient-domain PSNR partials: for an orthonormal basis
// ||f_ref - Psi x||^2 = ||c_ref - x||^2 (Parseval), so the squared error of the
// recovered spectra needs only the reference coefficients and the recovered
// coefficients: a pure HBM stream of 16 bytes per voxel, no GEMM and no
// spectra cube.  Grid-stride double2 loads, four pairs in flight per thread,
// evict-first (each byte is read once); one atomic per CTA.
__global__ void __launch_bounds__(256) sse_coeff_kernel(long long n, const double* __restrict__ a,
                                                        const double* __restrict__ b, double* sse) {
  __shared__ double red[8];
  const long long n2 = n >> 1;
  const double2* a2 = reinterpret_cast<const double2*>(a);
  const double2* b2 = reinterpret_cast<const double2*>(b);
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double s0 = 0.0, s1 = 0.0;
  for (; i + 3 * stride < n2; i += 4 * stride) {
    double2 va[4], vb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      va[u] = __ldcs(a2 + i + u * stride);
      vb[u] = __ldcs(b2 + i + u * stride);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double dx = va[u].x - vb[u].x, dy = va[u].y - vb[u].y;
      s0 += dx * dx;
      s1 += dy * dy;
    }
  }
  for (; i < n2; i += stride) {
    const double2 va = __ldcs(a2 + i), vb = __ldcs(b2 + i);
    const double dx = va.x - vb.x, dy = va.y - vb.y;
    s0 += dx * dx;
    s1 += dy * dy;
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const double d = a[n - 1] - b[n - 1];
    s0 += d * d;
  }
  double s = warp_sum(s0 + s1);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[w] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += red[k];
    atomicAdd(sse, t);
  }
}

// scalar fallback for operands that are not 16-byte aligned
__global__ void __launch_bounds__(256) sse_coeff_scalar_kernel(long long n, const double* __restrict__ a,
                                                               const double* __restrict__ b, double* sse) {
  __shared__ double red[8];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double d = a[i] - b[i];
    s += d * d;
  }
  s = warp_sum(s);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[w] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += red[k];
    atomicAdd(sse, t);
  }
}

cudaError_t launch_sse_coeff(long long n, const double* a, const double* b, double* sse, int sms,
                             cudaStream_t stream) {
  const bool aligned = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0;
  const long long work = aligned ? (n >> 1) : n;
  long long blocks = (work + 255) / 256;
  const long long cap = (long long)sms * 8;   // 8 x 256 threads per SM, grid-stride beyond
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (aligned) sse_coeff_kernel<<<(int)blocks, 256, 0, stream>>>(n, a, b, sse);
  else sse_coeff_scalar_kernel<<<(int)blocks, 256, 0, stream>>>(n, a, b, sse);
  return cudaGetLastError();
}

}  // namespace hcs

// ---------------------------------------------------------------------------
// FP64 DMMA peak microbenchmark (the roofline denominator; MEASURED_PEAKS.json
// carries no FP64 figure).  Independent m8n8k4 chains, 8 per warp.
namespace hcs {
__global__ void dmma_peak_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}
}  // namespace hcs

extern "C" int hcs_dmma_peak_tflops(double* tflops_out, int iters) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* buf = nullptr;
  if (cudaMalloc(&buf, 1024 * sizeof(double)) != cudaSuccess) return 2;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 4, threads = 256;
  hcs::dmma_peak_kernel<<<blocks, threads>>>(buf, 1000);   // warm-up
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    hcs::dmma_peak_kernel<<<blocks, threads>>>(buf, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * (threads / 32);
  *tflops_out = flops / (best * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

// debug builds: per-phase cycle totals of the batched least-squares kernel
extern "C" int hcs_debug_phases_ls(unsigned long long* out16, int reset) {
#ifdef HCS_PHASES
  cudaMemcpyFromSymbol(out16, hcs::g_phase_ls, 16 * sizeof(unsigned long long));
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(hcs::g_phase_ls, z, sizeof(z));
  }
  return 0;
#else
  (void)out16;
  (void)reset;
  return 1;
#endif
}

// Self-check of ddiv_fast / soft_fast (hcs_common.cuh) against __ddiv_rn / soft
// on n pseudo-random operand pairs per mode: mode 0 moderate exponents
// (2^-12 .. 2^12), 1 the full exponent range incl. subnormals, infinities and
// NaN, 2 soft-threshold operands (|v| near and above t).
// out[0] = accepted (ok) quotients, out[1] = accepted quotients that differ
// from __ddiv_rn (must be 0), out[2] = rejected (redone by the caller).
namespace hcs {
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__global__ void divcheck_kernel(unsigned long long n, unsigned long long seed, int mode, unsigned long long* out) {
  unsigned long long acc = 0, bad = 0, rej = 0;
  for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < n;
       k += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long u = mix64(seed + 2 * k), v = mix64(seed + 2 * k + 1);
    double a, b;
    if (mode == 0) {
      a = __longlong_as_double((long long)((u & 0x800fffffffffffffull) | ((1011ull + (u >> 52) % 25) << 52)));
      b = __longlong_as_double((long long)((v & 0x800fffffffffffffull) | ((1011ull + (v >> 52) % 25) << 52)));
    } else if (mode == 1) {
      a = __longlong_as_double((long long)u);
      b = __longlong_as_double((long long)v);
    } else {
      const double t = ldexp(1.0 + (double)(u & 0xffff) / 65536.0, (int)((u >> 16) % 21) - 10);
      const double rel = ldexp((double)(v >> 12), -52 - (int)((v & 0xfff) % 40));   // |v| = t (1 + rel)
      const double mag = t * (1.0 + rel);
      bool ok = true;
      const double f = soft_fast((v >> 11) & 1 ? -mag : mag, t, ok), g = soft((v >> 11) & 1 ? -mag : mag, t);
      if (ok) { ++acc; bad += __double_as_longlong(f) != __double_as_longlong(g); } else ++rej;
      continue;
    }
    bool ok = true;
    const double q = ddiv_fast(a, b, ok), ref = __ddiv_rn(a, b);
    if (ok) { ++acc; bad += __double_as_longlong(q) != __double_as_longlong(ref); } else ++rej;
  }
  atomicAdd(out + 0, acc);
  atomicAdd(out + 1, bad);
  atomicAdd(out + 2, rej);
}
}  // namespace hcs

extern "C" int hcs_debug_divcheck(unsigned long long n, unsigned long long seed, int mode, unsigned long long* out3) {
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, 3 * sizeof(unsigned long long)) != cudaSuccess) return 1;
  cudaMemset(d, 0, 3 * sizeof(unsigned long long));
  hcs::divcheck_kernel<<<148 * 8, 256>>>(n, seed, mode, d);
  cudaError_t e = cudaMemcpy(out3, d, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e == cudaSuccess ? 0 : 1;
}
