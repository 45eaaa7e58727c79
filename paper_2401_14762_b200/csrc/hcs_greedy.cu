// hcs_greedy.cu -- persistent CTA-per-pixel greedy solvers: gOMP, BIHT, CoSaMP.
//
// Reference: hypercs/solvers.py:248-297 (gomp), :300-342 (biht), :345-394
// (cosamp), stop rule :115-127, y = 0 shortcut :145-152, non-finite failure
// :155-157; selection = kernels.argmax_k (kernels.py:31-41), least squares =
// kernels.least_squares (kernels.py:44-67) -> hcs_ls.cuh.
//
// Each CTA (128 threads) pulls pixels from a global atomic work queue and runs
// the whole solver for that pixel out of shared memory:
//   * correlation p = A^T r = sum_j r_j Psi[mask_j, :]  (threads over bands,
//     Psi rows streamed from L2; 2NM flops);
//   * warp top-k by MSB-first key bisection (exact tie rule of argmax_k);
//   * support sets as 256-bit bitmaps; union = OR, sorted list = ballot/popc;
//   * the support-outgrew-m break happens before the solve and without
//     counting the iteration (solvers.py:274-276, 320-321, 372-373);
//   * column-pivoted Householder least squares on the gathered M x k
//     dictionary columns (+ rhs) in shared memory;
//   * residual y - A x recomputed from Psi rows, delta and the stop rule.
// Optional trace: the 256-bit bitmap of every argmax_k call, for the parity
// harness's tie classification.
#include "hcs_ls.cuh"
#include "hcs_internal.cuh"

namespace hcs {

constexpr int kGreedyThreads = 128;

struct GreedyShared {
  uint32_t supp[8], sel[8], keep[8];
  double red[16];
  long long pid;
  long long start;
  int dec;
  int ipiv;
  int count;
  int brk;
  int bad;
};

// Sorted index list of a 256-bit bitmap (warp 0); returns the count.
__device__ __forceinline__ int bitmap_to_list(const uint32_t* bm, int* list) {
  const int lane = threadIdx.x & 31;
  int base = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const uint32_t word = bm[e];
    const bool on = (word >> lane) & 1u;
    if (on) list[base + __popc(word & ((1u << lane) - 1u))] = 32 * e + lane;
    base += __popc(word);
  }
  __syncwarp();
  return base;
}

template <int ALGO>
__global__ void __launch_bounds__(kGreedyThreads) greedy_kernel(GreedyArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int N = a.N, M = a.M, ld = a.ld;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int KMAX = M + 1;  // support <= m (break before solve) ... +1 guard
  // ---- shared memory carve-up -------------------------------------------
  double* Bs = reinterpret_cast<double*>(smraw);
  double* B = a.gscratch ? a.gscratch + (size_t)blockIdx.x * M * ld : Bs;
  double* vec = Bs + (a.gscratch ? 0 : (size_t)M * ld);   // N: p / u / x_full
  double* x = vec + kMaxN;                                 // N: current iterate
  double* ys = x + kMaxN;                                  // M
  double* r = ys + M;                                      // M
  double* sv = r + M;                                      // KMAX: LS solution
  double* vn1 = sv + KMAX + 1;
  double* vn2 = vn1 + KMAX + 1;
  double* zt = vn2 + KMAX + 1;
  int* perm = reinterpret_cast<int*>(zt + KMAX + 1);       // KMAX + 1
  int* list = perm + KMAX + 1;                             // 256: sorted support
  int* tlist = list + kMaxN;                               // 256: refit support (gomp top)
  uint8_t* msk = reinterpret_cast<uint8_t*>(tlist + kMaxN);  // M
  GreedyShared& g = *reinterpret_cast<GreedyShared*>(reinterpret_cast<uintptr_t>(msk + M + 15) & ~uintptr_t(15));
  LsScratch sc{vn1, vn2, zt, perm, g.red, &g.ipiv};
  const double NaN = __longlong_as_double(0x7ff8000000000000ll);

  for (;;) {
    if (tid == 0) g.pid = (long long)atomicAdd(a.counter, 1ull);
    __syncthreads();
    const long long pid = g.pid;
    if (pid >= a.P) break;
    // ---- load the pixel -----------------------------------------------------
    int nz = 0, bad = 0;
    for (int j = tid; j < M; j += nt) {
      const double v = a.y[pid * M + j];
      ys[j] = v;
      r[j] = v;
      msk[j] = a.mask[pid * M + j];
      nz |= (v != 0.0);
      bad |= !isfinite(v);
    }
    for (int n = tid; n < kMaxN; n += nt) x[n] = 0.0;
    if (tid < 8) { g.supp[tid] = 0u; }
    nz = __syncthreads_or(nz);
    bad = __syncthreads_or(bad);
    if (!nz) {   // y == 0 shortcut
      for (int n = tid; n < N; n += nt) a.x_out[pid * N + n] = 0.0;
      if (tid == 0) {
        a.st.iterations[pid] = 0;
        a.st.converged[pid] = 1;
        a.st.final_delta[pid] = 0.0;
        a.st.failed_at[pid] = -1;
        if (a.st.trace_len) a.st.trace_len[pid] = 0;
        if (a.st.elapsed) a.st.elapsed[pid] = 0.0;
      }
      __syncthreads();
      continue;
    }
    if (bad) {   // scipy's finiteness check raises ValueError (kernels.py:61)
      if (tid == 0) atomicOr(a.err, 1);
      for (int n = tid; n < N; n += nt) a.x_out[pid * N + n] = 0.0;
      if (tid == 0) {
        a.st.iterations[pid] = 0;
        a.st.converged[pid] = 0;
        a.st.final_delta[pid] = NaN;
        a.st.failed_at[pid] = -1;
        if (a.st.trace_len) a.st.trace_len[pid] = 0;
        if (a.st.elapsed) a.st.elapsed[pid] = 0.0;
      }
      __syncthreads();
      continue;
    }
    double delta = 1.0;
    int iters = 0, ncall = 0, ksupp = 0;
    bool converged = false, failed = false;
    if (tid == 0) g.start = now_ns();
    __syncthreads();
    const long long t0 = g.start;
    for (;;) {
      // ---- stop rule before the pass (solvers.py:115-127) -------------------
      if (tid == 0) g.dec = stop_decision(delta, iters, t0, a.prm);
      __syncthreads();
      const int dec = g.dec;
      __syncthreads();
      if (dec != kContinue) { converged = dec == kConverged; break; }
      // ---- correlation / gradient proxy over all bands ----------------------
      for (int n = tid; n < N; n += nt) {
        double p = 0.0;
        for (int j = 0; j < M; ++j) p += r[j] * __ldg(a.basis + (size_t)msk[j] * N + n);
        if (ALGO == kBiht) p = __dadd_rn(x[n], __dmul_rn(a.prm.mu, p));   // solvers.py:318
        vec[n] = p;
      }
      __syncthreads();
      // ---- selection + union ------------------------------------------------
      if (warp == 0) {
        const int k = (ALGO == kGomp) ? a.prm.G : (ALGO == kBiht ? a.prm.kappa : 2 * a.prm.kappa);
        warp_topk(vec, N, k, g.sel);
        trace_store(a.st, pid, ncall, g.sel);
        if (lane < 8) {
          uint32_t u = g.sel[lane];
          if (ALGO == kBiht) {   // union with flatnonzero(x)
            uint32_t nzw = 0;
            for (int b = 0; b < 32; ++b) nzw |= (x[32 * lane + b] != 0.0 ? 1u : 0u) << b;
            u |= nzw;
          } else {
            u |= g.supp[lane];
          }
          g.supp[lane] = u;
        }
        __syncwarp();
        const int cnt = bitmap_to_list(g.supp, list);
        if (lane == 0) { g.count = cnt; g.brk = cnt > M; }
      }
      __syncthreads();
      if (g.brk) break;                          // keep the last iterate, no count
      ksupp = g.count;
      // ---- gather A[:, support] and y, least squares --------------------------
      for (int idx = tid; idx < M * (ksupp + 1); idx += nt) {
        const int rr = idx / (ksupp + 1), c = idx - rr * (ksupp + 1);
        B[rr * ld + c] = (c < ksupp) ? __ldg(a.basis + (size_t)msk[rr] * N + list[c]) : ys[rr];
      }
      __syncthreads();
      ls_solve(B, ld, M, ksupp, sv, sc);
      int kx;          // support size of the new iterate, indices in tlist
      if (ALGO == kGomp) {
        // x = scatter(s); top = argmax_k(x, kappa) over all N; refit on top
        for (int n = tid; n < N; n += nt) vec[n] = 0.0;
        __syncthreads();
        for (int c = tid; c < ksupp; c += nt) vec[list[c]] = sv[c];
        __syncthreads();
        if (warp == 0) {
          warp_topk(vec, N, a.prm.kappa, g.sel);
          trace_store(a.st, pid, ncall, g.sel);
          bitmap_to_list(g.sel, tlist);
        }
        __syncthreads();
        kx = a.prm.kappa;
        for (int idx = tid; idx < M * (kx + 1); idx += nt) {
          const int rr = idx / (kx + 1), c = idx - rr * (kx + 1);
          B[rr * ld + c] = (c < kx) ? __ldg(a.basis + (size_t)msk[rr] * N + tlist[c]) : ys[rr];
        }
        __syncthreads();
        ls_solve(B, ld, M, kx, sv, sc);
      } else {
        // keep = argmax_k(s, min(kappa, k)); zero (biht) or drop (cosamp) the rest
        const int kk = a.prm.kappa < ksupp ? a.prm.kappa : ksupp;
        if (warp == 0) {
          warp_topk(sv, ksupp, kk, g.keep);
          trace_store(a.st, pid, ncall, g.keep);
          if (ALGO == kCosamp) {
            // support = support[keep]  (stays sorted)
            if (lane == 0) {
              int o = 0;
              for (int c = 0; c < ksupp; ++c)
                if (bm_test(g.keep, c)) { tlist[o] = list[c]; zt[o] = sv[c]; ++o; }
              for (int e = 0; e < 8; ++e) g.supp[e] = 0u;
              for (int c = 0; c < o; ++c) g.supp[tlist[c] >> 5] |= 1u << (tlist[c] & 31);
            }
          } else {
            if (lane == 0) {
              for (int c = 0; c < ksupp; ++c) {
                tlist[c] = list[c];
                zt[c] = bm_test(g.keep, c) ? sv[c] : 0.0;
              }
            }
          }
        }
        __syncthreads();
        kx = (ALGO == kCosamp) ? kk : ksupp;
        for (int c = tid; c < kx; c += nt) sv[c] = zt[c];
        __syncthreads();
      }
      // ---- new iterate, residual, delta (solvers.py:285-290) -----------------
      for (int n = tid; n < N; n += nt) x[n] = 0.0;
      __syncthreads();
      for (int c = tid; c < kx; c += nt) x[tlist[c]] = sv[c];
      double part = 0.0;
      int nf = 0;
      for (int j = tid; j < M; j += nt) {
        const double* row = a.basis + (size_t)msk[j] * N;
        double ax = 0.0;
        for (int c = 0; c < kx; ++c) ax += __ldg(row + tlist[c]) * sv[c];
        const double rn = ys[j] - ax;
        const double d = rn - r[j];
        part += d * d;
        r[j] = rn;
      }
      for (int c = tid; c < kx; c += nt) nf |= !isfinite(sv[c]);
      delta = sqrt(cta_sum(part, g.red));
      nf = __syncthreads_or(nf);
      ++iters;
      if (nf || !isfinite(delta)) { failed = true; break; }
    }
    // ---- results ----------------------------------------------------------------
    for (int n = tid; n < N; n += nt) a.x_out[pid * N + n] = failed ? 0.0 : x[n];
    if (tid == 0) {
      a.st.iterations[pid] = failed ? 0 : iters;
      a.st.converged[pid] = converged ? 1 : 0;
      a.st.final_delta[pid] = failed ? NaN : delta;
      a.st.failed_at[pid] = failed ? iters : -1;
      if (a.st.trace_len) a.st.trace_len[pid] = ncall;
      if (a.st.elapsed) a.st.elapsed[pid] = 1e-9 * (double)(now_ns() - t0);
    }
    __syncthreads();
  }
}

size_t greedy_smem_bytes(int N, int M, int ld, bool global_ls) {
  const int KMAX = M + 1;
  size_t b = global_ls ? 0 : sizeof(double) * (size_t)M * ld;
  b += sizeof(double) * (2 * kMaxN + 2 * M + 4 * (KMAX + 1));
  b += sizeof(int) * (KMAX + 1 + 2 * kMaxN);
  b += M + 16 + sizeof(GreedyShared);
  (void)N;
  return (b + 15) & ~(size_t)15;
}

cudaError_t launch_greedy(int algo, const GreedyArgs& args, int grid, size_t smem, cudaStream_t stream) {
  cudaError_t e = cudaSuccess;
#define HCS_LAUNCH_GREEDY(A)                                                                        \
  e = cudaFuncSetAttribute(greedy_kernel<A>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
  if (e != cudaSuccess) return e;                                                                   \
  greedy_kernel<A><<<grid, kGreedyThreads, smem, stream>>>(args);
  if (algo == kGomp) {
    HCS_LAUNCH_GREEDY(kGomp)
  } else if (algo == kBiht) {
    HCS_LAUNCH_GREEDY(kBiht)
  } else {
    HCS_LAUNCH_GREEDY(kCosamp)
  }
#undef HCS_LAUNCH_GREEDY
  return cudaGetLastError();
}

int greedy_blocks_per_sm(int algo, size_t smem) {
  int nb = 0;
  if (algo == kGomp) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, greedy_kernel<kGomp>, kGreedyThreads, smem);
  else if (algo == kBiht) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, greedy_kernel<kBiht>, kGreedyThreads, smem);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, greedy_kernel<kCosamp>, kGreedyThreads, smem);
  return nb;
}

}  // namespace hcs
