// hcs_input.cu -- the input side of the recovery pipeline on the GPU
// (SURVEY.md §8(f)1): synthetic spectra, sparsification in the DCT domain and
// per-pixel measurement.
//
// Reference analogues: cli.run_sparsify (cli.py:97-126: per pixel
// to_sparse_domain -> sparsify -> from_sparse_domain), cli.run_compress
// (cli.py:129-139: seeded band selection, y = f[mask]), transform.sparsify
// (transform.py:73-97: keep (|x| - mean|x|) >= factor * std|x|) and
// transform.measure (transform.py:168-173).  The BASELINE.json model replaces
// the reference's shared mask and DFT by per-pixel masks and the orthonormal
// DCT-II, with its own threshold rule |c| < T max|c| (synth.py); both rules
// are supported.
//
//   synth_spectra_kernel     f = clip(sum_i a_i exp(-z_i^2 / 2) + noise, 0, 1),
//                            z_i = (b - c_i) / w_i: the synth.py v1 recipe on
//                            host-drawn parameters (elementwise, HBM-bound).
//   sparsify_measure_kernel  32-pixel tiles: c = Psi^T f (DMMA), per-pixel
//                            threshold, f_s = Psi c_s (DMMA), mask = the M
//                            smallest keys (warp bisection select), y = f_s[mask].
#include "hcs_gemm.cuh"
#include "hcs_internal.cuh"

namespace hcs {

// ---------------------------------------------------------------- spectra

// Evaluated in the order numpy evaluates synth._tile: z = (b - c) / w,
// e = exp((-0.5 * z) * z), t = a * e, ((t0 + t1) + t2) + t3 + noise, clip.
// Explicit _rn intrinsics keep nvcc from contracting into FMAs numpy never
// does; exp() itself may differ from numpy's by an ulp.
__global__ void synth_spectra_kernel(long long P, int N, const double* __restrict__ centres,
                                     const double* __restrict__ widths, const double* __restrict__ amps,
                                     const double* __restrict__ noise, double* __restrict__ f) {
  const long long total = P * N;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long p = idx / N;
    const double b = (double)(int)(idx - p * N);
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double z = __ddiv_rn(__dsub_rn(b, __ldg(centres + 4 * p + i)), __ldg(widths + 4 * p + i));
      const double e = exp(__dmul_rn(__dmul_rn(-0.5, z), z));
      const double t = __dmul_rn(__ldg(amps + 4 * p + i), e);
      s = (i == 0) ? t : __dadd_rn(s, t);
    }
    s = __dadd_rn(s, __ldg(noise + idx));
    f[idx] = fmin(fmax(s, 0.0), 1.0);
  }
}

// ---------------------------------------------------------------- sparsify + measure

// Order-preserving 64-bit key of a double (larger key = larger value); the
// complement selects the smallest.
__device__ __forceinline__ unsigned long long order_key(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Warp: bitmap of the k largest keys among key[e] (lane + 32 e < n), ties to
// the lowest index (MSB-first bisection of the k-th key, as warp_topk).
__device__ __forceinline__ void warp_select_keys(const unsigned long long (&key)[8], int n, int k, uint32_t* bitmap) {
  const int lane = threadIdx.x & 31;
  unsigned long long T = 0ull;
  for (int bit = 63; bit >= 0; --bit) {
    const unsigned long long cand = T | (1ull << bit);
    int c = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) c += (lane + 32 * e < n && key[e] >= cand) ? 1 : 0;
    if (warp_sum_i(c) >= k) T = cand;
  }
  int gt = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) gt += (lane + 32 * e < n && key[e] > T) ? 1 : 0;
  const int need = k - warp_sum_i(gt);
  int seen = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const bool valid = lane + 32 * e < n;
    const bool eq = valid && key[e] == T;
    const unsigned int eqm = __ballot_sync(0xffffffffu, eq);
    const int rank = seen + __popc(eqm & ((1u << lane) - 1u));
    const unsigned int selm = __ballot_sync(0xffffffffu, valid && (key[e] > T || (eq && rank < need)));
    if (lane == 0) bitmap[e] = selm;
    seen += __popc(eqm);
  }
  __syncwarp();
}

// Column max over the 8 lanes sharing a column (lane bits 2..4) of an
// accumulator-layout quantity; lane l ends with column col_of_reduced(l).
__device__ __forceinline__ double col_max8(const double (&v)[8], int lane) {
  const bool b = (lane >> 2) & 1, c = (lane >> 3) & 1, e = (lane >> 4) & 1;
  double u[4], q[2];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double send = b ? v[k] : v[k + 4], keep = b ? v[k + 4] : v[k];
    u[k] = fmax(keep, __shfl_xor_sync(0xffffffffu, send, 4));
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double send = c ? u[k] : u[k + 2], keep = c ? u[k + 2] : u[k];
    q[k] = fmax(keep, __shfl_xor_sync(0xffffffffu, send, 8));
  }
  const double send = e ? q[0] : q[1], keep = e ? q[1] : q[0];
  return fmax(keep, __shfl_xor_sync(0xffffffffu, send, 16));
}
__device__ __forceinline__ double col_sum8(const double (&v)[8], int lane) {
  const bool b = (lane >> 2) & 1, c = (lane >> 3) & 1, e = (lane >> 4) & 1;
  double u[4], q[2];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double send = b ? v[k] : v[k + 4], keep = b ? v[k + 4] : v[k];
    u[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double send = c ? u[k] : u[k + 2], keep = c ? u[k + 2] : u[k];
    q[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  const double send = e ? q[0] : q[1], keep = e ? q[1] : q[0];
  return keep + __shfl_xor_sync(0xffffffffu, send, 16);
}
__device__ __forceinline__ int col_of_reduced8(int lane) {
  return 8 * (2 * ((lane >> 2) & 1) + ((lane >> 3) & 1)) + 2 * (lane & 3) + ((lane >> 4) & 1);
}

struct InputArgs {
  long long P;
  int N, M, rule;
  double factor;
  const double* basis;
  const double* f;
  const double* keys;       // P x N or null (then mask is an input)
  uint8_t* mask;            // P x M
  double* coeffs;           // P x N or null
  double* spectra;          // P x N or null
  double* y;                // P x M
  unsigned long long* nzero;   // zeroed coefficients (device counter) or null
};

// blockDim = 2 Np (Np / 16 warps of 16 rows); dynamic smem: In (Np x 32), red (2 x W x 32).
__global__ void __launch_bounds__(512, 1) sparsify_measure_kernel(InputArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int N = a.N, M = a.M, Np = (N + 15) & ~15, KS = Np >> 2;
  const int W = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* In = reinterpret_cast<double*>(smraw);        // Np x 32, B-fragment order (GEMM input / spectra rows)
  double* red = In + Np * kSlots;                        // 2 x W x 32 column partials
  double* colv = red + 2 * W * kSlots;                   // 2 x 32: per-pixel threshold statistics
  uint32_t* bm = reinterpret_cast<uint32_t*>(colv + 2 * kSlots);   // W x 8 selection bitmaps
  uint8_t* mrow = reinterpret_cast<uint8_t*>(bm + 8 * W);          // 32 x 256 mask rows
  const int cred = col_of_reduced8(lane);
  unsigned long long zeros = 0;
  for (long long t0 = blockIdx.x * (long long)kSlots; t0 < a.P; t0 += (long long)gridDim.x * kSlots) {
    // ---- load the spectra tile ------------------------------------------------
    for (int idx = threadIdx.x; idx < Np * kSlots; idx += blockDim.x) {
      const int s = idx / Np, n = idx - s * Np;
      const long long p = t0 + s;
      In[in_idx(n, s)] = (p < a.P && n < N) ? __ldg(a.f + p * N + n) : 0.0;
    }
    __syncthreads();
    // ---- c = Psi^T f ----------------------------------------------------------
    double acc[2][4][2];
    basis_tile_gemm(a.basis, N, KS, true, In, acc);
    // ---- per-pixel threshold statistics over the N rows -------------------------
    double v[8];
#pragma unroll
    for (int cb = 0; cb < 4; ++cb)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        double m = 0.0;
#pragma unroll
        for (int rb = 0; rb < 2; ++rb) {
          const double mag = acc_row(w, rb, lane) < N ? fabs(acc[rb][cb][i]) : 0.0;
          m = a.rule == 0 ? fmax(m, mag) : m + mag;
        }
        v[2 * cb + i] = m;
      }
    const double part = a.rule == 0 ? col_max8(v, lane) : col_sum8(v, lane);
    red[w * kSlots + cred] = part;
    __syncthreads();
    if (threadIdx.x < kSlots) {
      double s = 0.0;
      for (int q = 0; q < W; ++q) s = a.rule == 0 ? fmax(s, red[q * kSlots + threadIdx.x]) : s + red[q * kSlots + threadIdx.x];
      colv[threadIdx.x] = a.rule == 0 ? a.factor * s : s / N;   // maxrel: T max|c|; meanstd: mean |c|
    }
    __syncthreads();
    if (a.rule == 1) {   // population std of |c| (numpy: sqrt(mean(|x - mean|^2)))
#pragma unroll
      for (int cb = 0; cb < 4; ++cb)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const double mu = colv[acc_col(cb, i, lane)];
          double m = 0.0;
#pragma unroll
          for (int rb = 0; rb < 2; ++rb) {
            if (acc_row(w, rb, lane) < N) {
              const double d = fabs(acc[rb][cb][i]) - mu;
              m += d * d;
            }
          }
          v[2 * cb + i] = m;
        }
      const double p2 = col_sum8(v, lane);
      red[(W + w) * kSlots + cred] = p2;
      __syncthreads();
      if (threadIdx.x < kSlots) {
        double s = 0.0;
        for (int q = 0; q < W; ++q) s += red[(W + q) * kSlots + threadIdx.x];
        colv[kSlots + threadIdx.x] = a.factor * sqrt(s / N);
      }
    }
    __syncthreads();   // In free: GEMM 1 is done everywhere
    // ---- threshold, coefficient output, GEMM 2 input ------------------------------
#pragma unroll
    for (int cb = 0; cb < 4; ++cb)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int s = acc_col(cb, i, lane);
        const long long p = t0 + s;
        const double s0 = colv[s], s1 = colv[kSlots + s];
#pragma unroll
        for (int rb = 0; rb < 2; ++rb) {
          const int n = acc_row(w, rb, lane);
          double c = acc[rb][cb][i];
          if (n < N) {
            const double mag = fabs(c);
            const bool keep = a.rule == 0 ? !(mag < s0) : (mag - s0 >= s1);
            if (!keep) {
              c = 0.0;
              if (p < a.P) ++zeros;
            }
            if (a.coeffs && p < a.P) a.coeffs[p * N + n] = c;
          } else {
            c = 0.0;
          }
          In[in_idx(n, s)] = c;
        }
      }
    __syncthreads();
    // ---- f_s = Psi c_s ----------------------------------------------------------
    basis_tile_gemm(a.basis, N, KS, false, In, acc);
    __syncthreads();   // In free again: spectra rows go there (row-major 32 x Np)
#pragma unroll
    for (int cb = 0; cb < 4; ++cb)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int s = acc_col(cb, i, lane);
        const long long p = t0 + s;
#pragma unroll
        for (int rb = 0; rb < 2; ++rb) {
          const int n = acc_row(w, rb, lane);
          In[s * Np + n] = acc[rb][cb][i];
          if (a.spectra && p < a.P && n < N) a.spectra[p * N + n] = acc[rb][cb][i];
        }
      }
    // ---- masks: the M smallest keys of each pixel (sorted band list) -----------------
    for (int s = w; s < kSlots; s += W) {
      const long long p = t0 + s;
      if (p >= a.P) break;
      uint8_t* mr = mrow + s * kMaxN;
      if (a.keys) {
        unsigned long long key[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int j = lane + 32 * e;
          key[e] = j < N ? ~order_key(__ldg(a.keys + p * N + j)) : 0ull;
        }
        uint32_t* b = bm + 8 * w;
        warp_select_keys(key, N, M, b);
        int base = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint32_t word = b[e];
          if ((word >> lane) & 1u) {
            const int o = base + __popc(word & ((1u << lane) - 1u));
            mr[o] = (uint8_t)(32 * e + lane);
            a.mask[p * M + o] = (uint8_t)(32 * e + lane);
          }
          base += __popc(word);
        }
      } else {
        for (int j = lane; j < M; j += 32) mr[j] = a.mask[p * M + j];
      }
      __syncwarp();
    }
    __syncthreads();
    // ---- y = f_s[mask] ------------------------------------------------------------
    for (int idx = threadIdx.x; idx < kSlots * M; idx += blockDim.x) {
      const int s = idx / M, j = idx - s * M;
      const long long p = t0 + s;
      if (p < a.P) a.y[p * M + j] = In[s * Np + mrow[s * kMaxN + j]];
    }
    __syncthreads();
  }
  if (a.nzero) {
    for (int o = 16; o > 0; o >>= 1) zeros += __shfl_xor_sync(0xffffffffu, zeros, o);
    if (lane == 0 && zeros) atomicAdd(a.nzero, zeros);
  }
}

cudaError_t launch_synth_spectra(long long P, int N, const double* centres, const double* widths, const double* amps,
                                 const double* noise, double* f, int sms, cudaStream_t stream) {
  long long blocks = (P * N + 255) / 256;
  if (blocks > (long long)sms * 16) blocks = (long long)sms * 16;
  synth_spectra_kernel<<<(int)blocks, 256, 0, stream>>>(P, N, centres, widths, amps, noise, f);
  return cudaGetLastError();
}

cudaError_t launch_sparsify_measure(long long P, int N, int M, int rule, double factor, const double* basis,
                                    const double* f, const double* keys, uint8_t* mask, double* coeffs,
                                    double* spectra, double* y, unsigned long long* nzero, int sms,
                                    cudaStream_t stream) {
  const int Np = (N + 15) & ~15, W = Np >> 4;
  const size_t smem = sizeof(double) * ((size_t)Np * kSlots + 2 * W * kSlots + 2 * kSlots) +
                      sizeof(uint32_t) * 8 * W + (size_t)kSlots * kMaxN;
  cudaError_t e = cudaFuncSetAttribute(sparsify_measure_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sparsify_measure_kernel, 2 * Np, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const long long tiles = (P + kSlots - 1) / kSlots;
  const int blocks = (int)(tiles < (long long)per_sm * sms ? tiles : (long long)per_sm * sms);
  InputArgs args{P, N, M, rule, factor, basis, f, keys, mask, coeffs, spectra, y, nzero};
  sparsify_measure_kernel<<<blocks, 2 * Np, smem, stream>>>(args);
  return cudaGetLastError();
}

}  // namespace hcs
