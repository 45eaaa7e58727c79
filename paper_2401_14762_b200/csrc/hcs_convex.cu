// hcs_convex.cu -- persistent slot engine for the convex solvers (FISTA, ADMM).
//
// Reference: hypercs/solvers.py:164-203 (fista), :206-245 (admm), stop rule
// :115-127, y = 0 shortcut :145-152, non-finite failure :155-157; the
// Lipschitz constant of transform.py:176-217.
//
// Design (B200-first):
//  * one persistent CTA per SM owns 32 "slots"; every slot holds one pixel;
//  * each tick runs one solver iteration for all 32 slots as two FP64 DMMA
//    GEMMs against the shared basis (Psi^T g, then Psi x), with the per-pixel
//    mask, soft threshold, momentum / dual update, residual and
//    residual-delta stop test fused into the GEMM epilogues;
//  * a slot whose pixel stops (converged / cap / non-finite) writes its result
//    and is refilled from a global atomic work queue in the same tick
//    (active-pixel compaction at slot granularity: no tick is spent on a
//    finished pixel, no host round trip, one launch per cube);
//  * per-pixel iterates live in registers in the accumulator layout (x, z or
//    z, w), residuals and measurements in shared memory.
//
// FISTA uses linearity to keep two GEMMs per iteration: with r_k = y - A x_k,
//     A z_k - y = -(1 + b_k) r_k + b_k r_{k-1},  b_k = (t_{k-1} - 1) / t_k,
// so the gradient input needs no extra forward product.
// ADMM uses the eigendecomposition of A^T A + alpha I = Psi^T diag(d + alpha) Psi
// (d = mask indicator; Psi orthonormal): the "cached factorisation" of
// transform.py:253-264 is the mask itself, and
//     x = Psi^T diag(1/(d + alpha)) (yhat + alpha Psi (z - w)),   A x = u'[mask],
// two GEMMs per iteration and the residual for free.
#include "hcs_gemm.cuh"
#include "hcs_internal.cuh"

namespace hcs {

enum { kEmpty = 0, kActive = 1, kRetire = 2 };

#ifdef HCS_PHASES
__device__ unsigned long long g_phase_cx[16];
#endif

struct SlotState {
  long long pid[kSlots];
  long long rpid[kSlots];
  long long start[kSlots];
  double delta[kSlots], t[kSlots], tn[kSlots], beta[kSlots], betan[kSlots];
  double inv_l[kSlots], thr[kSlots], gap2[kSlots];
  int status[kSlots], iter[kSlots], flag[kSlots], rfail[kSlots];
  int n_active;
  int exhausted;
};

// Pull pixels from the work queue into slot s until one needs iterating
// (zero pixels retire on the spot, solvers.py:169-170 / 212-213).
template <int ALGO>
__device__ void refill_slot(const ConvexArgs& a, SlotState& ss, double* ys, double* r, double* rp,
                            uint8_t* msk, uint8_t* pos, int s) {
  const int lane = threadIdx.x & 31;
  const int M = a.M, N = a.N;
  for (;;) {
    long long pid = 0;
    if (lane == 0) {
      pid = ss.exhausted ? a.P : (long long)atomicAdd(a.counter, 1ull);
      if (pid >= a.P) ss.exhausted = 1;
    }
    pid = __shfl_sync(0xffffffffu, pid, 0);
    if (pid >= a.P) {
      if (lane == 0) ss.status[s] = kEmpty;
      if (ALGO == kAdmm)
        for (int b = lane; b < kMaxN; b += 32) pos[s * kMaxN + b] = 0xFF;
      __syncwarp();
      return;
    }
    bool nz = false, bad = false;
    for (int j = lane; j < M; j += 32) {
      double v = a.y[pid * M + j];
      uint8_t mj = a.mask[pid * M + j];
      ys[s * M + j] = v;
      r[s * M + j] = v;
      if (ALGO == kFista) rp[s * M + j] = v;
      msk[s * M + j] = mj;
      nz |= (v != 0.0);
      bad |= !isfinite(v);
    }
    nz = __any_sync(0xffffffffu, nz);
    bad = __any_sync(0xffffffffu, bad);
    __syncwarp();
    double lip = 0.0;
    if (ALGO == kFista) lip = warp_lipschitz(a.u0, msk + s * M, M);
    if (lane == 0 && a.st.lipschitz) a.st.lipschitz[pid] = (ALGO == kFista) ? lip : __longlong_as_double(0x7ff8000000000000ll);
    if (!nz) {  // y == 0: x = 0, 0 iterations, converged, delta 0, no admm_gap
      for (int n = lane; n < N; n += 32) a.x_out[pid * N + n] = 0.0;
      if (lane == 0) {
        a.st.iterations[pid] = 0;
        a.st.converged[pid] = 1;
        a.st.final_delta[pid] = 0.0;
        a.st.failed_at[pid] = -1;
        if (a.st.admm_gap) a.st.admm_gap[pid] = __longlong_as_double(0x7ff8000000000000ll);
        if (a.st.elapsed) a.st.elapsed[pid] = 0.0;
        if (a.st.work) a.st.work[pid] = 0.0;
      }
      continue;
    }
    if (ALGO == kAdmm && bad && lane == 0) atomicOr(a.err, 1);   // cho_solve would raise
    // stop rule before the first pass (delta0 = 1): epsilon > 1 or an expired budget
    const long long t0 = now_ns();
    const int dec = stop_decision(1.0, 0, t0, a.prm);
    if (dec != kContinue) {
      for (int n = lane; n < N; n += 32) a.x_out[pid * N + n] = 0.0;
      if (lane == 0) {
        a.st.iterations[pid] = 0;
        a.st.converged[pid] = dec == kConverged;
        a.st.final_delta[pid] = 1.0;
        a.st.failed_at[pid] = -1;
        if (a.st.admm_gap) a.st.admm_gap[pid] = 0.0;
        if (a.st.elapsed) a.st.elapsed[pid] = 1e-9 * (double)(now_ns() - t0);
        if (a.st.work) a.st.work[pid] = 0.0;
      }
      continue;
    }
    if (ALGO == kAdmm) {
      for (int b = lane; b < kMaxN; b += 32) pos[s * kMaxN + b] = 0xFF;
      __syncwarp();
      for (int j = lane; j < M; j += 32) pos[s * kMaxN + msk[s * M + j]] = (uint8_t)j;
    }
    if (lane == 0) {
      ss.pid[s] = pid;
      ss.start[s] = t0;
      ss.status[s] = kActive;
      ss.iter[s] = 0;
      ss.delta[s] = 1.0;
      ss.t[s] = 1.0;
      ss.beta[s] = 0.0;
      if (ALGO == kFista) {
        ss.inv_l[s] = 1.0 / lip;
        ss.thr[s] = __dmul_rn(a.prm.lam, ss.inv_l[s]);
      } else {
        ss.thr[s] = a.prm.lam / a.prm.alpha;
      }
    }
    __syncwarp();
    return;
  }
}

// Stop rule after an iteration (solvers.py:115-127 evaluated before the next
// pass) plus the non-finite check (solvers.py:155-157).
__device__ __forceinline__ void finish_iteration(const ConvexArgs& a, SlotState& ss, int s, double delta,
                                                 bool admm) {
  // lane 0 only
  int it = ss.iter[s] + 1;
  ss.iter[s] = it;
  ss.delta[s] = delta;
  const bool failed = ss.flag[s] || !isfinite(delta);
  const int dec = failed ? kContinue : stop_decision(delta, it, ss.start[s], a.prm);
  const bool conv = dec == kConverged;
  if (failed || dec != kContinue) {
    long long pid = ss.pid[s];
    ss.status[s] = kRetire;
    ss.rpid[s] = pid;
    ss.rfail[s] = failed;
    a.st.iterations[pid] = failed ? 0 : it;
    a.st.converged[pid] = conv ? 1 : 0;
    a.st.final_delta[pid] = failed ? __longlong_as_double(0x7ff8000000000000ll) : delta;
    a.st.failed_at[pid] = failed ? it : -1;
    if (admm && a.st.admm_gap)
      a.st.admm_gap[pid] = failed ? __longlong_as_double(0x7ff8000000000000ll) : sqrt(ss.gap2[s]);
    if (a.st.elapsed) a.st.elapsed[pid] = 1e-9 * (double)(now_ns() - ss.start[s]);
    if (a.st.work) a.st.work[pid] = 4.0 * (double)a.N * (double)a.N * (double)it;
  }
}

// 13..16 warps put 4 warps on one SM sub-partition (16K registers): <= 128 regs
template <int ALGO, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) convex_kernel(ConvexArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int Np = a.Np, M = a.M, N = a.N, KS = Np >> 2;
  const int W = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* In = reinterpret_cast<double*>(smraw);        // Np * 32, B-fragment order
  double* zs = In + Np * kSlots;                        // Np * 32 (fista: extrapolated point z)
  double* ys = zs + (ALGO == kFista ? Np * kSlots : 0); // 32 * M
  double* r = ys + kSlots * M;                          // 32 * M
  double* rp = r + kSlots * M;                          // 32 * M (fista)
  SlotState& ss = *reinterpret_cast<SlotState*>(rp + (ALGO == kFista ? kSlots * M : 0));
  uint8_t* msk = reinterpret_cast<uint8_t*>(&ss + 1);   // 32 * M
  uint8_t* pos = msk + kSlots * M;                      // 32 * 256 (admm)

  // per-element iterates in the accumulator layout: fista x (z in shared
  // memory, register budget is 128 at 13+ warps); admm z, w
  double p0[2][4][2], p1[2][4][2];
#pragma unroll
  for (int rb = 0; rb < 2; ++rb)
#pragma unroll
    for (int cb = 0; cb < 4; ++cb)
#pragma unroll
      for (int i = 0; i < 2; ++i) p0[rb][cb][i] = p1[rb][cb][i] = 0.0;
  if (ALGO == kFista)
    for (int idx = threadIdx.x; idx < Np * kSlots; idx += blockDim.x) zs[idx] = 0.0;
  if (threadIdx.x < kSlots) ss.status[threadIdx.x] = kEmpty;
  if (threadIdx.x == 0) ss.exhausted = 0;
  __syncthreads();

  double acc[2][4][2];
#ifdef HCS_PHASES
  long long cph[16] = {0};
  cph[15] = clock64();
#define CMARK(k) HCS_MARKP(cph, k)
#else
#define CMARK(k) do {} while (0)
#endif
  for (;;) {
    // ---- writeback of retiring slots (element layout) ---------------------
#pragma unroll
    for (int cb = 0; cb < 4; ++cb)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int s = acc_col(cb, i, lane);
        if (ss.status[s] == kRetire) {
          const long long pid = ss.rpid[s];
          const bool fail = ss.rfail[s];
#pragma unroll
          for (int rb = 0; rb < 2; ++rb) {
            const int n = acc_row(w, rb, lane);
            const double v = (ALGO == kFista) ? p0[rb][cb][i] : p0[rb][cb][i];
            if (n < N) a.x_out[pid * N + n] = fail ? 0.0 : v;
            p0[rb][cb][i] = 0.0;
            p1[rb][cb][i] = 0.0;
            if (ALGO == kFista) zs[in_idx(n, s)] = 0.0;
          }
        }
      }
    if (ALGO == kFista) {
      for (int idx = threadIdx.x; idx < Np * kSlots; idx += blockDim.x) In[idx] = 0.0;
    } else {
      // q = z - w is the GEMM input of the next ADMM pass
#pragma unroll
      for (int rb = 0; rb < 2; ++rb)
#pragma unroll
        for (int cb = 0; cb < 4; ++cb)
#pragma unroll
          for (int i = 0; i < 2; ++i)
            In[in_idx(acc_row(w, rb, lane), acc_col(cb, i, lane))] = p0[rb][cb][i] - p1[rb][cb][i];
    }
    if (threadIdx.x == 0) ss.n_active = 0;
    __syncthreads();
    CMARK(0);

    // ---- per-slot phase R: refill, momentum weights, GEMM input (fista) ----
    for (int s = w; s < kSlots; s += W) {
      if (ss.status[s] != kActive) refill_slot<ALGO>(a, ss, ys, r, rp, msk, pos, s);
      if (ss.status[s] == kActive) {
        if (lane == 0) {
          atomicAdd(&ss.n_active, 1);
          ss.flag[s] = 0;
          ss.gap2[s] = 0.0;
          if (ALGO == kFista) {
            const double t = ss.t[s];
            const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));   // solvers.py:160-161
            ss.tn[s] = tn;
            ss.betan[s] = (t - 1.0) / tn;
          }
        }
        if (ALGO == kFista) {
          // g = A z - y = -(1 + b) r + b r_prev at the measured rows
          const double b = ss.beta[s];
          for (int j = lane; j < M; j += 32) {
            const double g = -(1.0 + b) * r[s * M + j] + b * rp[s * M + j];
            In[in_idx(msk[s * M + j], s)] = (b == 0.0) ? -r[s * M + j] : g;
          }
        }
      } else if (lane == 0) {
        ss.inv_l[s] = 0.0;
        ss.thr[s] = 0.0;
        ss.betan[s] = 0.0;
      }
    }
    __syncthreads();
    CMARK(1);
    if (ss.n_active == 0) break;

    if (ALGO == kFista) {
      // ---- GEMM A: grad = Psi^T g; epilogue: prox-gradient + momentum -----
      tile_gemm(a.fragT, In, KS, acc);
      __syncthreads();
      CMARK(2);
#pragma unroll
      for (int cb = 0; cb < 4; ++cb)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int s = acc_col(cb, i, lane);
          const double il = ss.inv_l[s], th = ss.thr[s], bn = ss.betan[s];
          bool bad = false;
#pragma unroll
          for (int rb = 0; rb < 2; ++rb) {
            const int zi = in_idx(acc_row(w, rb, lane), s);
            const double x = p0[rb][cb][i], z = zs[zi];
            const double aux = __dsub_rn(z, __dmul_rn(il, acc[rb][cb][i]));   // solvers.py:183
            const double xn = soft(aux, th);                                    // solvers.py:185
            zs[zi] = __dadd_rn(xn, __dmul_rn(bn, __dsub_rn(xn, x)));           // solvers.py:189
            p0[rb][cb][i] = xn;
            bad |= !isfinite(xn);
            In[in_idx(acc_row(w, rb, lane), s)] = xn;
          }
          if (bad) ss.flag[s] = 1;
        }
      __syncthreads();
      CMARK(3);
      // ---- GEMM B: F = Psi x_new; epilogue: stage F for the residual -----
      tile_gemm(a.fragS, In, KS, acc);
      __syncthreads();
      CMARK(4);
#pragma unroll
      for (int rb = 0; rb < 2; ++rb)
#pragma unroll
        for (int cb = 0; cb < 4; ++cb)
#pragma unroll
          for (int i = 0; i < 2; ++i) In[in_idx(acc_row(w, rb, lane), acc_col(cb, i, lane))] = acc[rb][cb][i];
      __syncthreads();
      CMARK(5);
      // ---- per-slot phase S: residual, delta, stop rule (solvers.py:192-196)
      for (int s = w; s < kSlots; s += W) {
        if (ss.status[s] != kActive) continue;
        double d2 = 0.0;
        for (int j = lane; j < M; j += 32) {
          const double rn = ys[s * M + j] - In[in_idx(msk[s * M + j], s)];
          const double d = rn - r[s * M + j];
          d2 += d * d;
          rp[s * M + j] = r[s * M + j];
          r[s * M + j] = rn;
        }
        d2 = warp_sum(d2);
        if (lane == 0) {
          ss.t[s] = ss.tn[s];
          ss.beta[s] = ss.betan[s];
          finish_iteration(a, ss, s, sqrt(d2), false);
        }
      }
      __syncthreads();
      CMARK(6);
    } else {
      // ---- GEMM S: v = Psi (z - w); epilogue: u' = (yhat + alpha v) / (d + alpha)
      tile_gemm(a.fragS, In, KS, acc);
      __syncthreads();
      CMARK(2);
      const double alpha = a.prm.alpha;
#pragma unroll
      for (int cb = 0; cb < 4; ++cb)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int s = acc_col(cb, i, lane);
#pragma unroll
          for (int rb = 0; rb < 2; ++rb) {
            const int n = acc_row(w, rb, lane);
            const int pj = pos[s * kMaxN + n];
            const bool in_mask = pj != 0xFF && n < N;
            const double yh = in_mask ? ys[s * M + pj] : 0.0;
            const double u = yh + alpha * acc[rb][cb][i];
            In[in_idx(n, s)] = u / ((in_mask ? 1.0 : 0.0) + alpha);
          }
        }
      __syncthreads();
      CMARK(3);
      // ---- GEMM C: x = Psi^T u'; epilogue: shrink, dual update, gap --------
      tile_gemm(a.fragT, In, KS, acc);
      CMARK(4);
#pragma unroll
      for (int cb = 0; cb < 4; ++cb)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int s = acc_col(cb, i, lane);
          const double th = ss.thr[s];
          bool bad = false;
          double g2 = 0.0;
#pragma unroll
          for (int rb = 0; rb < 2; ++rb) {
            const double x = acc[rb][cb][i], z = p0[rb][cb][i], wv = p1[rb][cb][i];
            (void)z;
            const double zn = soft(__dadd_rn(x, wv), th);                 // solvers.py:229
            p1[rb][cb][i] = __dsub_rn(__dadd_rn(wv, x), zn);              // solvers.py:231
            p0[rb][cb][i] = zn;
            const double dg = x - zn;
            g2 += dg * dg;
            bad |= !isfinite(zn);
          }
          // sum the 8 row-lanes sharing this column, then one shared atomic
          g2 += __shfl_xor_sync(0xffffffffu, g2, 4);
          g2 += __shfl_xor_sync(0xffffffffu, g2, 8);
          g2 += __shfl_xor_sync(0xffffffffu, g2, 16);
          if (lane < 4) atomicAdd(&ss.gap2[s], g2);
          if (bad) ss.flag[s] = 1;
        }
      __syncthreads();
    CMARK(5);
      // ---- per-slot phase S: residual from u' (A x = u'[mask]), stop rule ----
      for (int s = w; s < kSlots; s += W) {
        if (ss.status[s] != kActive) continue;
        double d2 = 0.0;
        for (int j = lane; j < M; j += 32) {
          const double rn = ys[s * M + j] - In[in_idx(msk[s * M + j], s)];
          const double d = rn - r[s * M + j];
          d2 += d * d;
          r[s * M + j] = rn;
        }
        d2 = warp_sum(d2);
        if (lane == 0) finish_iteration(a, ss, s, sqrt(d2), true);
      }
      __syncthreads();
    CMARK(6);
    }
  }
#ifdef HCS_PHASES
  if (threadIdx.x == 0)
    for (int k = 0; k < 15; ++k) atomicAdd(&g_phase_cx[k], (unsigned long long)cph[k]);
#endif
}

// Fragment-order copies of Psi and Psi^T, and u0 = Psi * (1/sqrt(N)) 1.
__global__ void prep_basis_kernel(const double* __restrict__ basis, int N, int Np, double2* fragS,
                                  double2* fragT, double* u0) {
  const int KS = Np >> 2;
  const long long total = (long long)(Np / 16) * KS * 32;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int lane = (int)(idx & 31);
    const long long t = idx >> 5;
    const int ks = (int)(t % KS);
    const int w = (int)(t / KS);
    const int r0 = 16 * w + (lane >> 2), r1 = r0 + 8, c = 4 * ks + (lane & 3);
    auto at = [&](int rr, int cc) { return (rr < N && cc < N) ? basis[(size_t)rr * N + cc] : 0.0; };
    fragS[idx] = make_double2(at(r0, c), at(r1, c));
    fragT[idx] = make_double2(at(c, r0), at(c, r1));
  }
  if (blockIdx.x == 0) {
    const double inv = 1.0 / sqrt((double)N);
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
      double s = 0.0;
      for (int k = 0; k < N; ++k) s += basis[(size_t)j * N + k] * inv;
      u0[j] = s;
    }
  }
}

cudaError_t launch_prep_basis(const double* basis, int N, int Np, double2* fragS, double2* fragT, double* u0,
                              cudaStream_t stream) {
  prep_basis_kernel<<<64, 256, 0, stream>>>(basis, N, Np, fragS, fragT, u0);
  return cudaGetLastError();
}

size_t convex_smem_bytes(int algo, int Np, int M) {
  size_t b = sizeof(double) * (size_t)Np * kSlots * (algo == kFista ? 2 : 1);   // In (+ z)
  b += sizeof(double) * (size_t)kSlots * M * (algo == kFista ? 3 : 2);
  b += sizeof(SlotState);
  b += (size_t)kSlots * M;                                           // msk
  if (algo == kAdmm) b += (size_t)kSlots * kMaxN;                    // pos
  return (b + 15) & ~(size_t)15;
}

template <int ALGO, int MAXT>
static cudaError_t launch_convex_t(const ConvexArgs& args, int grid, size_t smem, cudaStream_t stream) {
  cudaError_t e = cudaFuncSetAttribute(convex_kernel<ALGO, MAXT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  convex_kernel<ALGO, MAXT><<<grid, 2 * args.Np, smem, stream>>>(args);   // Np / 16 warps
  return cudaGetLastError();
}

cudaError_t launch_convex(int algo, const ConvexArgs& args, int grid, cudaStream_t stream) {
  const size_t smem = convex_smem_bytes(algo, args.Np, args.M);
  if (algo == kFista) return launch_convex_t<kFista, 512>(args, grid, smem, stream);
  return launch_convex_t<kAdmm, 512>(args, grid, smem, stream);
}

}  // namespace hcs

// debug builds: per-phase cycle totals of the convex kernel (summed over CTAs)
extern "C" int hcs_debug_phases_cx(unsigned long long* out16, int reset) {
#ifdef HCS_PHASES
  cudaMemcpyFromSymbol(out16, hcs::g_phase_cx, 16 * sizeof(unsigned long long));
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(hcs::g_phase_cx, z, sizeof(z));
  }
  return 0;
#else
  (void)out16;
  (void)reset;
  return 1;
#endif
}
