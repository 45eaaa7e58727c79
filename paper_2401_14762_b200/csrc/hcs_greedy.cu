// hcs_greedy.cu -- persistent CTA-per-pixel greedy solvers: gOMP, BIHT, CoSaMP.
//
// Reference: hypercs/solvers.py:248-297 (gomp), :300-342 (biht), :345-394
// (cosamp), stop rule :115-127, y = 0 shortcut :145-152, non-finite failure
// :155-157; selection = kernels.argmax_k (kernels.py:31-41), least squares =
// kernels.least_squares (kernels.py:44-67).
//
// Each CTA (4 warps) pulls pixels from a global atomic work queue and runs the
// whole solver for that pixel out of shared memory:
//   * correlation p = A^T r = sum_j r_j Psi[mask_j, :]  (threads over bands,
//     Psi rows streamed from L2; 2NM flops);
//   * warp top-k by MSB-first key bisection (exact tie rule of argmax_k);
//   * support sets as 256-bit bitmaps; union = OR, sorted list = ballot/popc;
//   * the support-outgrew-m break happens before the solve and without
//     counting the iteration (solvers.py:274-276, 320-321, 372-373);
//   * least squares on the gathered M x k dictionary columns: corrected
//     semi-normal equations with a DMMA Gram and blocked Cholesky
//     (hcs_ls_csne.cuh), falling back to the exact column-pivoted restatement
//     (hcs_ls.cuh) when a guard trips;
//   * residual y - A x recomputed from Psi rows, delta and the stop rule.
// Optional trace: the 256-bit bitmap of every argmax_k call, for the parity
// harness's tie classification.
#include "hcs_internal.cuh"
#include "hcs_ls.cuh"
#include "hcs_ls_csne.cuh"
#include <cstdlib>

namespace hcs {

#ifdef HCS_PHASES
__device__ unsigned long long g_phase[16];
#endif

constexpr int kGreedyThreads = 128;
#ifndef HCS_SMEM_ARGS_ALL
#define HCS_SMEM_ARGS_ALL 0   // experiments: BIHT / gOMP also pass ls_csne's argument block through shared memory
#endif
constexpr int kRing = 64;  // state hashes kept for cycle detection (periods 2..63)

struct GreedyShared {
  uint32_t supp[8], sel[8], keep[8];
  double red[16];
  unsigned long long ringh[kRing];   // hash of (residual bits, support bitmap) per pass
  uint32_t snapbm[8];
  unsigned long long hpart[4];
  long long pid;
  long long start;
  int mis;
  int period;
  int dec;
  int ipiv;
  int count;
  int brk;
  int flag;
  int ctr;   // must follow flag: ls_csne's Gram tile counter (flag[1])
  // CoSaMP: argument blocks of ls_csne in shared memory (hcs_greedy.cu: solve)
  CsneScratch cs;
  DctGram dg;
};

// Shared-memory layout (doubles unless noted), identical on host and device.
// The LS region holds systems of up to `kalloc` columns (B and its Gram);
// larger systems (rare: gOMP supports beyond kalloc) use the CTA's global
// scratch.
struct GreedyLayout {
  int Mp, bmax, gmax;        // padded rows; doubles for B and for the Gram tiles
  int vec, x, ys, r, yv, sv, vn1, vn2, zt, keys, ring, dinv, cv, F, q;   // double offsets
  int ints;                  // pivoted-fallback perm (ints) offset, in doubles
  int lists;                 // uint8 support lists + mask bytes offset, in doubles
  size_t bytes;
};

// doubles for B: the CSNE layout (column-major, y appended) or the pivoted
// fallback's row-major M x (K+1)|1, whichever is larger
__host__ __device__ inline int ls_doubles(int M, int K) {
  const int piv = M * ((K + 1) | 1);
  const int blk = csne_ld(M) * csne_cols(K);
  return piv > blk ? piv : blk;
}

// per-CTA global scratch: the widest system's columns and Gram tiles, F and A^T y
__host__ __device__ inline int cta_scratch_doubles(int M) {
  return ls_doubles(M, M) + csne_gram_doubles(M) + 2 * kMaxN;
}

__host__ __device__ inline GreedyLayout greedy_layout(int M, int kalloc) {
  GreedyLayout L;
  L.Mp = (M + 7) & ~7;
  L.bmax = ls_doubles(M, kalloc);
  if (L.bmax < 4 * kMaxN) L.bmax = 4 * kMaxN;     // also the correlation / residual / top-k key scratch
  L.gmax = csne_gram_doubles(kalloc);
  if (L.gmax < 4 * (M + 2)) L.gmax = 4 * (M + 2);  // also the pivoted fallback's vn1, vn2, z, perm
  if (L.gmax < 136) L.gmax = 136;                   // and the post-solve top-k scratch (1 KB + 48 B)
  L.keys = 0;                   // aliases the LS region (free outside solve())
  L.vn1 = L.bmax;               // vn1 / vn2 / zt / perm alias the Gram region (free outside the
  L.vn2 = L.vn1 + M + 2;        // CSNE solve; zt is also the CoSaMP prune buffer after it)
  L.zt = L.vn2 + M + 2;
  const int perm = L.zt + M + 2;
  int o = L.bmax + L.gmax;
  L.vec = o; o += kMaxN;
  L.x = o; o += kMaxN;
  L.ys = o; o += M;
  L.r = o; o += M;
  L.yv = o; o += L.Mp;
  L.sv = o; o += M + 2;
  L.dinv = o; o += M + 9;
  L.cv = o; o += M + 9;
  L.ring = o; o += M;           // residual snapshot for exact cycle confirmation
  // the closed-form Gram's generator F(d) and A^T y (hcs_ls_csne.cuh: DctGram)
  // are kept in the CTA's global scratch and staged over vec / x, which are
  // dead while a least-squares system is being solved: 4 KB more shared
  // memory per CTA cost CoSaMP 5% through the smaller L1
  L.F = L.vec;
  L.q = L.x;
  L.ints = perm;
  // lists (2 x 256 uint8), msk (M bytes), then GreedyShared
  L.lists = o;
  size_t b = sizeof(double) * (size_t)o + 2 * kMaxN + (size_t)M;
  b = (b + 15) & ~(size_t)15;
  b += sizeof(GreedyShared);
  L.bytes = (b + 15) & ~(size_t)15;
  return L;
}

// Columns the shared-memory LS region is sized for: the largest system each
// solver builds on its fast path (support bounds of solvers.py:273, 319, 371).
__host__ __device__ inline int greedy_kalloc(int algo, int M, int kappa) {
  int k = M;
  if (algo == kCosamp) k = 3 * kappa;           // kept kappa + 2 kappa new
  else if (algo == kBiht) k = 2 * kappa;        // supp(x) <= kappa + kappa new
  else if (algo == kGomp) k = kappa > 40 ? kappa : 40;   // refit kappa; supports beyond 40 spill
  return k < M ? k : M;
}

// Sorted index list of a 256-bit bitmap (one warp); returns the count.
__device__ __forceinline__ int bitmap_to_list(const uint32_t* bm, uint8_t* list) {
  const int lane = threadIdx.x & 31;
  int base = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const uint32_t word = bm[e];
    const bool on = (word >> lane) & 1u;
    if (on) list[base + __popc(word & ((1u << lane) - 1u))] = (uint8_t)(32 * e + lane);
    base += __popc(word);
  }
  __syncwarp();
  return base;
}

template <int ALGO>
__global__ void __launch_bounds__(kGreedyThreads, 4) greedy_kernel(GreedyArgs a) {
  if (*(volatile const int*)a.err & kErrMask) return;   // invalid masks (validate_masks_kernel)
  extern __shared__ __align__(16) unsigned char smraw[];
  hcs_smem_poison(smraw, a.smem_bytes);
  HCS_CHECK(a.err, blockIdx.x < a.slots);   // one global LS scratch slot per CTA
  const int N = a.N, M = a.M;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int kalloc = a.kalloc;
  const GreedyLayout L = greedy_layout(M, kalloc);
  double* S = reinterpret_cast<double*>(smraw);
  double* Bglob = a.gscratch + (size_t)blockIdx.x * cta_scratch_doubles(M);
  double* Gglob = Bglob + ls_doubles(M, M);
  double* Fq = Gglob + csne_gram_doubles(M);   // 2 kMaxN: the pixel's F and A^T y between solves
  double* vec = S + L.vec;      // N: p / u / x_full
  double* x = S + L.x;          // N: current iterate
  double* ys = S + L.ys;        // M
  double* r = S + L.r;          // M
  double* yv = S + L.yv;        // Mp: blocked rhs
  double* sv = S + L.sv;        // LS solution
  int* perm = reinterpret_cast<int*>(S + L.ints);
  uint8_t* list = reinterpret_cast<uint8_t*>(S + L.lists);   // sorted support
  uint8_t* tlist = list + kMaxN;                             // support of the new iterate
  uint8_t* msk = tlist + kMaxN;
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(S + L.keys);
  double* snap = S + L.ring;    // residual snapshot (cycle confirmation)
  GreedyShared& g = *reinterpret_cast<GreedyShared*>(reinterpret_cast<uintptr_t>(msk + M + 15) & ~uintptr_t(15));
  const LsScratch sc{S + L.vn1, S + L.vn2, S + L.zt, perm, g.red, &g.ipiv};
  int* lsflag = &g.flag;
  const double NaN = __longlong_as_double(0x7ff8000000000000ll);
  const int Mp = L.Mp;
#ifdef HCS_PHASES
  long long hcs_ph[16] = {0};
  hcs_ph[15] = clock64();
  long long* php = hcs_ph;
#define GMARK(k) HCS_MARKP(php, k)
#else
  long long* php = nullptr;
#define GMARK(k) do {} while (0)
#endif

  // least squares on the dictionary columns `cols[0..K)` (+ y): blocked DMMA
  // Householder, exact pivoted restatement when the rank guard trips
  // ls_b: the gathered columns (column-major, ld csne_ld(M), y as column K)
  // stay intact after a successful CSNE solve, so the residual reads them
  // there instead of re-gathering dictionary rows from L2
  bool ls_ok = false, ls_shared = true;
  const double* ls_b = S;
  // DCT-II basis (verified by transpose_basis_kernel): closed-form Gram entries
  const bool use_dct = ALGO == kCosamp && a.ls_mode == 0 && a.notdct != nullptr && *(volatile const int*)a.notdct == 0;
  const double s0n = sqrt(1.0 / (double)N), s1n = sqrt(2.0 / (double)N);
  bool f_ready = false;   // this pixel's F and y^T y are computed (at its first wide system)
  double yty = 0.0;
  auto solve = [&](const uint8_t* cols, int K) {
    const bool shared_b = K <= kalloc;
    // wide systems (columns in the L2 scratch) of a DCT-II basis: closed-form Gram
    const bool dct_far = use_dct && !shared_b;
    if (dct_far && !f_ready) {
      // F(d) = sum_j cos(theta_{mask_j} d) = (A^T 1)[d] / s_d: the column sums of
      // the measured rows, accumulated like the correlation; once per pixel
      double* part = S;          // the LS region is free until the gather
      double acc[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = 0.0;
#pragma unroll 4
      for (int j = warp; j < M; j += 4) {
        const double* row = a.basis + (size_t)msk[j] * N + lane;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (lane + 32 * c < N) acc[c] += __ldg(row + 32 * c);
      }
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (lane + 32 * c < N) part[warp * kMaxN + lane + 32 * c] = acc[c];
      double py = 0.0;
      for (int j = tid; j < M; j += nt) py += ys[j] * ys[j];
      __syncthreads();
      for (int n = tid; n < N; n += nt) {
        const double u = (part[n] + part[kMaxN + n]) + (part[2 * kMaxN + n] + part[3 * kMaxN + n]);
        Fq[n] = u / (n ? s1n : s0n);
      }
      yty = cta_sum(py, g.red);
      f_ready = true;
      __syncthreads();
    }
    if (dct_far) {   // stage F and A^T y over vec / x (dead until the new iterate is built)
      for (int n = tid; n < N; n += nt) {
        S[L.F + n] = Fq[n];
        S[L.q + n] = Fq[kMaxN + n];
      }
    }
    HCS_CHECK(a.err, K >= 1 && K <= M + 1 && K <= kMaxN);
    double* B = shared_b ? S : Bglob;
    ls_shared = shared_b;
    ls_b = B;
    ls_ok = false;
    if (a.ls_mode == 1) {
      // pivoted Householder QR (the reference's algorithm), row-major B with y as column K
      const int ldp = (K + 1) | 1;
      for (int idx = tid; idx < M * (K + 1); idx += nt) {
        const int rr = idx / (K + 1), c = idx - rr * (K + 1);
        B[rr * ldp + c] = (c < K) ? __ldg(a.basis + (size_t)msk[rr] * N + cols[c]) : ys[rr];
      }
      __syncthreads();
      ls_solve(B, ldp, M, K, sv, sc);
      GMARK(9);
      return;
    }
    const int ldb = csne_ld(M);                  // column-major; y is column K
    const int nc = csne_cols(K);
    // asynchronous gather (cp.async, L2 -> shared, no register staging): warp w
    // copies columns w, w+4, ...; lanes over rows (consecutive shared words)
    if (shared_b) {
      for (int c = warp; c < nc; c += 4) {
        const int col = c < K ? cols[c] : 0;
        for (int rr = lane; rr < ldb; rr += 32) {
          double* dst = B + c * ldb + rr;
          if (rr < M && c < K) cp_async8(dst, a.basis_t + (size_t)col * N + msk[rr]);   // one column: ascending rows
          else *dst = (rr < M && c == K) ? ys[rr] : 0.0;
        }
      }
      cp_async_wait_all();
    } else {
      // global scratch: warp w copies columns w, w + 4, ... two at a time,
      // lanes over rows, six independent loads in flight per thread
      for (int c0 = warp; c0 < nc; c0 += 8) {
#pragma unroll 1
        for (int r0 = lane; r0 < ldb; r0 += 96) {
          double v[2][3];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int c = c0 + 4 * u;
            const int col = c < K ? cols[c] : 0;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              const int rr = r0 + 32 * q;
              v[u][q] = 0.0;
              if (c < nc && rr < M) v[u][q] = c < K ? __ldg(a.basis_t + (size_t)col * N + msk[rr]) : (c == K ? ys[rr] : 0.0);
            }
          }
#pragma unroll
          for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int q = 0; q < 3; ++q)
              if (c0 + 4 * u < nc && r0 + 32 * q < ldb) B[(c0 + 4 * u) * ldb + r0 + 32 * q] = v[u][q];
        }
      }
    }
    // Gram tiles in shared memory whenever they fit the whole LS region (B then
    // lives in the global scratch), else in the global scratch too
    double* G = shared_b ? S + L.bmax : (csne_gram_doubles(K) <= L.bmax + L.gmax ? S : Gglob);
    bool solved;
    if constexpr (ALGO == kCosamp) {
      // argument blocks in shared memory: as locals they live on the stack, and
      // with four 48 KB CTAs per SM the L1 left over does not hold the stacks
      if (tid == 0) {
        g.cs = CsneScratch{G, S + L.dinv, S + L.cv, yv, g.red, lsflag};
        g.dg = DctGram{S + L.F, S + L.q, cols, N, s0n, s1n, yty};
      }
      __syncthreads();
      GMARK(3);
      solved = ls_csne<true>(B, ldb, M, K, sv, g.cs, php, dct_far ? &g.dg : nullptr);
    } else if constexpr (HCS_SMEM_ARGS_ALL) {
      if (tid == 0) g.cs = CsneScratch{G, S + L.dinv, S + L.cv, yv, g.red, lsflag};
      __syncthreads();
      GMARK(3);
      solved = ls_csne<false>(B, ldb, M, K, sv, g.cs, php);
    } else {
      __syncthreads();
      GMARK(3);
      const CsneScratch cs{G, S + L.dinv, S + L.cv, yv, g.red, lsflag};
      solved = ls_csne<false>(B, ldb, M, K, sv, cs, php);
    }
    if (solved) {
      ls_ok = true;
      return;
    }
    const int ldp = (K + 1) | 1;
    for (int idx = tid; idx < M * (K + 1); idx += nt) {
      const int rr = idx / (K + 1), c = idx - rr * (K + 1);
      B[rr * ldp + c] = (c < K) ? __ldg(a.basis + (size_t)msk[rr] * N + cols[c]) : ys[rr];
    }
    __syncthreads();
    ls_solve(B, ldp, M, K, sv, sc);
    GMARK(9);
  };

  for (;;) {
    if (tid == 0) { g.pid = (long long)atomicAdd(a.counter, 1ull); g.ctr = 1; }
    __syncthreads();
    long long pid = g.pid;
    if (a.plist) {
      if ((unsigned long long)pid >= *a.plist_n) break;
      pid = a.plist[pid];
    } else if (pid >= a.P) {
      break;
    }
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
    if (tid < 8) g.supp[tid] = 0u;
    if (tid == 0) g.start = now_ns();
    nz = __syncthreads_or(nz);
    bad = __syncthreads_or(bad);
    if (!nz || bad) {   // y == 0 shortcut; non-finite y: scipy raises ValueError (kernels.py:61)
      if (bad && tid == 0) atomicOr(a.err, 1);
      for (int n = tid; n < N; n += nt) a.x_out[pid * N + n] = 0.0;
      if (tid == 0) {
        a.st.iterations[pid] = 0;
        a.st.converged[pid] = bad ? 0 : 1;
        a.st.final_delta[pid] = bad ? NaN : 0.0;
        a.st.failed_at[pid] = -1;
        if (a.st.trace_len) a.st.trace_len[pid] = 0;
        if (a.st.elapsed) a.st.elapsed[pid] = 0.0;
        if (a.st.work) a.st.work[pid] = 0.0;
      }
      __syncthreads();
      continue;
    }
    f_ready = false;
    const long long t0 = g.start;
    double delta = 1.0;
    int iters = 0, ncall = 0, ksupp = 0;
    bool converged = false, failed = false;
    // Cycle skip (CoSaMP / gOMP): the next pass is a deterministic function of
    // (support, residual) and y, so once that state recurs bit for bit after p
    // passes the trajectory is exactly p-periodic; whole periods up to the cap
    // are skipped, giving the same x, delta and iteration count as iterating.
    // Disabled under a wall-clock budget (timeouts depend on elapsed time).
    bool skipped = !(ALGO != kBiht && a.prm.limit_ns < 0 && a.prm.max_iter > 0);
    int pend_p = 0, pend_t = 0;   // candidate period (hash match) awaiting exact confirmation
    double work = 0.0;            // algorithmic FLOPs executed (thread 0's tally)
    for (;;) {
      // ---- stop rule before the pass (solvers.py:115-127) -------------------
      if (tid == 0) g.dec = stop_decision(delta, iters, t0, a.prm);
      __syncthreads();
      const int dec = g.dec;
      GMARK(0);
      if (dec != kContinue) { converged = dec == kConverged; break; }
      // ---- correlation / gradient proxy over all bands ----------------------
      // p = A^T r = sum_j r_j Psi[mask_j, :]: warp w takes rows j = w, w+4, ...,
      // lanes take bands (coalesced Psi row segments, 7 independent loads per
      // row in flight); the four warp partials are summed through shared memory
      {
        double* part = S;          // the LS region is free outside solve()
        double acc[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = 0.0;
#pragma unroll 4
        for (int j = warp; j < M; j += 4) {
          const double rj = r[j];
          const double* row = a.basis + (size_t)msk[j] * N + lane;
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (lane + 32 * c < N) acc[c] += rj * __ldg(row + 32 * c);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (lane + 32 * c < N) part[warp * kMaxN + lane + 32 * c] = acc[c];
        __syncthreads();
        for (int n = tid; n < N; n += nt) {
          double p = (part[n] + part[kMaxN + n]) + (part[2 * kMaxN + n] + part[3 * kMaxN + n]);
          if (ALGO == kCosamp && iters == 0 && use_dct) Fq[kMaxN + n] = p;   // r = y on the first pass: A^T y (DctGram's y row)
          if (ALGO == kBiht) p = __dadd_rn(x[n], __dmul_rn(a.prm.mu, p));   // solvers.py:318
          vec[n] = p;
        }
      }
      __syncthreads();
      GMARK(1);
      // ---- selection + union ------------------------------------------------
      {
        const int k = (ALGO == kGomp) ? a.prm.G : (ALGO == kBiht ? a.prm.kappa : 2 * a.prm.kappa);
        cta_topk(vec, N, k, g.sel, keys);
        trace_store(a.st, pid, ncall, g.sel);
      }
      if (warp == 0) {
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
      GMARK(2);
      work += 2.0 * N * M;                       // correlation
      if (g.brk) break;                          // keep the last iterate, no count
      ksupp = g.count;
      solve(list, ksupp);
      work += ls_flops(M, ksupp);
      int kx;          // support size of the new iterate, indices in tlist, values in sv
      if (ALGO == kGomp) {
        // x = scatter(s); top = argmax_k(x, kappa) over all N; refit on top
        for (int n = tid; n < N; n += nt) vec[n] = 0.0;
        __syncthreads();
        for (int c = tid; c < ksupp; c += nt) vec[list[c]] = sv[c];
        __syncthreads();
        cta_topk_sparse(vec, N, a.prm.kappa, g.sel, keys);
        trace_store(a.st, pid, ncall, g.sel);
        if (warp == 0) bitmap_to_list(g.sel, tlist);
        __syncthreads();
        kx = a.prm.kappa;
        solve(tlist, kx);
        work += ls_flops(M, kx);
      } else {
        // keep = argmax_k(s, min(kappa, k)); zero (biht) or drop (cosamp) the rest
        const int kk = a.prm.kappa < ksupp ? a.prm.kappa : ksupp;
        double* zt = S + L.zt;
        // scratch outside the gathered columns (kept for the residual)
        unsigned long long* keys2 = reinterpret_cast<unsigned long long*>(ls_shared ? S + L.bmax : S);
        cta_topk(sv, ksupp, kk, g.keep, keys2);
        trace_store(a.st, pid, ncall, g.keep);
        // the pass's coefficients over the solve's columns, zero where not kept
        for (int c = tid; c < ksupp; c += nt) S[L.cv + c] = bm_test(g.keep, c) ? sv[c] : 0.0;
        if (ALGO == kCosamp) {   // support = support[keep]  (stays sorted)
          if (tid < 8) g.supp[tid] = 0u;
          __syncthreads();
          for (int c = tid; c < ksupp; c += nt) {
            if (bm_test(g.keep, c)) {
              int o = __popc(g.keep[c >> 5] & ((1u << (c & 31)) - 1u));
              for (int e = 0; e < (c >> 5); ++e) o += __popc(g.keep[e]);
              tlist[o] = list[c];
              zt[o] = sv[c];
              atomicOr(&g.supp[list[c] >> 5], 1u << (list[c] & 31));
            }
          }
        } else {
          for (int c = tid; c < ksupp; c += nt) {
            tlist[c] = list[c];
            zt[c] = bm_test(g.keep, c) ? sv[c] : 0.0;
          }
        }
        __syncthreads();
        kx = (ALGO == kCosamp) ? kk : ksupp;
        for (int c = tid; c < kx; c += nt) sv[c] = zt[c];
        __syncthreads();
      }
      GMARK(7);
      // ---- new iterate, residual, delta (solvers.py:285-290) -----------------
      for (int n = tid; n < N; n += nt) x[n] = 0.0;
      __syncthreads();
      for (int c = tid; c < kx; c += nt) x[tlist[c]] = sv[c];
      double part = 0.0;
      int nf = 0;
      if (ls_ok) {
        // r = y - A x from the solve's gathered columns (y is column ks): x's
        // support is those columns (gOMP) or the kept subset (zeros elsewhere)
        const int ks = (ALGO == kGomp) ? kx : ksupp;
        const double* cs_ = (ALGO == kGomp) ? sv : S + L.cv;
        const int ld = csne_ld(M);
        __syncthreads();
        for (int j = tid; j < M; j += nt) {
          double a0 = 0.0, a1 = 0.0;
          int c = 0;
          for (; c + 1 < ks; c += 2) {
            a0 += ls_b[c * ld + j] * cs_[c];
            a1 += ls_b[(c + 1) * ld + j] * cs_[c + 1];
          }
          if (c < ks) a0 += ls_b[c * ld + j] * cs_[c];
          const double rn = ls_b[ks * ld + j] - (a0 + a1);
          const double d = rn - r[j];
          part += d * d;
          r[j] = rn;
        }
      } else {
        // A x over the kx support columns from the transposed dictionary in L2:
        // lanes own rows, warps split the columns
        double* pbuf = S;          // free again after solve()
        double ax[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) ax[q] = 0.0;
        for (int c = warp; c < kx; c += 4) {
          const int col = tlist[c];
          const double sc_ = sv[c];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int j = lane + 32 * q;
            if (j < M) ax[q] += __ldg(a.basis_t + (size_t)col * N + msk[j]) * sc_;
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (lane + 32 * q < M) pbuf[warp * kMaxN + lane + 32 * q] = ax[q];
        __syncthreads();
        for (int j = tid; j < M; j += nt) {
          const double* pp = S + j;
          const double axj = (pp[0] + pp[kMaxN]) + (pp[2 * kMaxN] + pp[3 * kMaxN]);
          const double rn = ys[j] - axj;
          const double d = rn - r[j];
          part += d * d;
          r[j] = rn;
        }
      }
      for (int c = tid; c < kx; c += nt) nf |= !isfinite(sv[c]);
      delta = sqrt(cta_sum(part, g.red));
      work += 2.0 * M * kx;                      // residual
      nf = __syncthreads_or(nf);
      GMARK(8);
      ++iters;
      if (nf || !isfinite(delta)) { failed = true; break; }
      if (!skipped) {
        // 64-bit hash of the residual bits (order-aware mix, summed over rows)
        unsigned long long h = 0ull;
        int mis = 0;
        for (int j = tid; j < M; j += nt) {
          unsigned long long z = (unsigned long long)__double_as_longlong(r[j]) + 0x9E3779B97F4A7C15ull * (j + 1);
          z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
          z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
          h += z ^ (z >> 31);
          if (pend_p) mis |= __double_as_longlong(snap[j]) != __double_as_longlong(r[j]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
        if (lane == 0) g.hpart[warp] = h;
        mis = __syncthreads_or(mis);
        h = g.hpart[0] + g.hpart[1] + g.hpart[2] + g.hpart[3];
#pragma unroll
        for (int e = 0; e < 8; ++e) h = (h ^ g.supp[e]) * 0x100000001B3ull;   // support bitmap (FNV-style)
        int per = 0;
        if (pend_p && iters == pend_t + pend_p) {
          // exact confirmation: the state recurred bit for bit after pend_p passes
          bool same = !mis;
          for (int e = 0; e < 8; ++e) same &= g.snapbm[e] == g.supp[e];
          if (same) per = pend_p;
          pend_p = 0;
        }
        if (!per && !pend_p) {
          const int hist = iters - 1 < kRing - 1 ? iters - 1 : kRing - 1;
          for (int pp = 2; pp <= hist && !pend_p; ++pp) {
            const int slot = (iters - pp) % kRing;
            if (g.ringh[slot] == h) { pend_p = pp; pend_t = iters; }
          }
          if (pend_p) {
            for (int j = tid; j < M; j += nt) snap[j] = r[j];
            if (tid < 8) g.snapbm[tid] = g.supp[tid];
          }
        }
        __syncthreads();
        if (tid == 0) {
          g.ringh[iters % kRing] = h;
        }
        if (per) {
          iters += ((a.prm.max_iter - iters) / per) * per;
          skipped = true;
        }
      }
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
      if (a.st.work) a.st.work[pid] = work;
    }
    __syncthreads();
    GMARK(10);
  }
#ifdef HCS_PHASES
  if (tid == 0)
    for (int k = 0; k < 15; ++k) atomicAdd(&g_phase[k], (unsigned long long)hcs_ph[k]);
#endif
  hcs_smem_canary(smraw, a.smem_bytes, a.err);
}

size_t greedy_smem_bytes(int algo, int M, int kalloc) { (void)algo; return greedy_layout(M, kalloc).bytes; }

int greedy_kalloc_host(int algo, int M, int kappa, size_t smem_cap) {
  // Shared-memory LS capacity: the solver's bound (greedy_kalloc), trimmed so
  // that four CTAs fit on an SM (228 KB, 1 KB reserved per CTA; the register
  // budget, launch bounds (128, 4), allows four too); systems wider than that
  // spill to the CTA's global scratch.  The kernel is latency-bound (serial
  // pivot chains, L2 gathers): four resident pixels per SM beat wider
  // shared-memory systems at two or three (measured: BIHT k=33 1.7x, CoSaMP
  // k=27 1.15x).
  const size_t four_per_sm = 55 * 1024;
  size_t cap = smem_cap < four_per_sm ? smem_cap : four_per_sm;
  if (const char* ov = getenv("HCS_GREEDY_CAP_KB")) {   // experiments: tighter capacity, more CTAs per SM
    const size_t v = (size_t)atoi(ov) * 1024;
    if (v >= 16 * 1024 && v < cap) cap = v;
  }
  int k = greedy_kalloc(algo, M, kappa);
  while (k > 8 && greedy_layout(M, k).bytes > cap) --k;
  return k;
}

size_t greedy_ls_doubles(int M) { return (size_t)cta_scratch_doubles(M); }

template <int ALGO>
static cudaError_t launch_t(const GreedyArgs& args, int grid, size_t smem, cudaStream_t stream) {
  cudaError_t e = cudaFuncSetAttribute(greedy_kernel<ALGO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(smem + kSmemExtra));
  if (e != cudaSuccess) return e;
  GreedyArgs ga = args;
  ga.smem_bytes = (unsigned)smem;
  greedy_kernel<ALGO><<<grid, kGreedyThreads, smem + kSmemExtra, stream>>>(ga);
  return cudaGetLastError();
}

cudaError_t launch_greedy(int algo, const GreedyArgs& args, int grid, size_t smem, cudaStream_t stream) {
  if (algo == kGomp) return launch_t<kGomp>(args, grid, smem, stream);
  if (algo == kBiht) return launch_t<kBiht>(args, grid, smem, stream);
  return launch_t<kCosamp>(args, grid, smem, stream);
}

template <int ALGO>
static int blocks_t(size_t smem) {
  // the dynamic shared-memory limit must be raised before the occupancy query
  cudaFuncSetAttribute(greedy_kernel<ALGO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem + kSmemExtra));
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, greedy_kernel<ALGO>, kGreedyThreads, smem + kSmemExtra);
  return nb;
}

int greedy_blocks_per_sm(int algo, int M, size_t smem) {
  (void)M;
  if (algo == kGomp) return blocks_t<kGomp>(smem);
  if (algo == kBiht) return blocks_t<kBiht>(smem);
  return blocks_t<kCosamp>(smem);
}

// basis_t[c N + r] = basis[r N + c]: a dictionary column gathered at the mask
// rows then reads ascending addresses of one column (~20 sectors per 32 rows
// instead of 32)
// Also checks, entry by entry, whether the basis is the orthonormal DCT-II
// synthesis matrix Psi[r][c] = s_c cos(pi c (2 r + 1) / (2 N)) (exact integer
// range reduction of c (2 r + 1) mod 4 N, cospi): *notdct stays 0 iff every
// entry agrees to 1e-15 (entries are <= sqrt(2/N); a closed-form host basis
// differs by ~1e-16).  Only then may the CSNE Gram use the DCT closed form.
__global__ void transpose_basis_kernel(const double* __restrict__ basis, int N, double* __restrict__ bt,
                                       int* notdct) {
  const double s0 = sqrt(1.0 / (double)N), s1 = sqrt(2.0 / (double)N);
  bool bad = false;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < N * N; idx += gridDim.x * blockDim.x) {
    const int c = idx / N, r = idx - c * N;
    const double v = basis[(size_t)r * N + c];
    bt[idx] = v;
    const int q = (c * (2 * r + 1)) % (4 * N);
    const double ref = (c ? s1 : s0) * cospi((double)q / (double)(2 * N));
    bad |= !(fabs(v - ref) <= 1e-15);
  }
  if (bad && notdct) atomicOr(notdct, 1);
}

cudaError_t launch_transpose_basis(const double* basis, int N, double* bt, int* notdct, cudaStream_t stream) {
  transpose_basis_kernel<<<64, 256, 0, stream>>>(basis, N, bt, notdct);
  return cudaGetLastError();
}

}  // namespace hcs

// debug builds: per-phase cycle totals of the greedy kernel (summed over CTAs)
extern "C" int hcs_debug_phases(unsigned long long* out16, int reset) {
#ifdef HCS_PHASES
  cudaMemcpyFromSymbol(out16, hcs::g_phase, 16 * sizeof(unsigned long long));
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(hcs::g_phase, z, sizeof(z));
  }
  return 0;
#else
  (void)out16;
  (void)reset;
  return 1;
#endif
}

// diagnostics: shared-memory LS capacity, dynamic shared bytes and CTAs per SM
// the greedy kernel would use for (algo, M, kappa)
extern "C" int hcs_debug_greedy_config(int algo, int M, int kappa, long long* out3) {
  const int k = hcs::greedy_kalloc_host(algo, M, kappa, 200 * 1024);
  const size_t smem = hcs::greedy_smem_bytes(algo, M, k);
  out3[0] = k;
  out3[1] = (long long)smem;
  out3[2] = hcs::greedy_blocks_per_sm(algo, M, smem);
  return 0;
}

// selection tests: cta_topk (variant 1) or the ranking reference (variant 0)
// on `batch` vectors of length n (device pointers), one CTA each
namespace hcs {
__global__ void topk_test_kernel(const double* v, int n, int k, uint32_t* bm, int variant) {
  __shared__ unsigned long long keys[256 + 16];
  __shared__ uint32_t bmap[8];
  const double* vv = v + (size_t)blockIdx.x * n;
  if (variant) cta_topk(vv, n, k, bmap, keys);
  else cta_topk_rank(vv, n, k, bmap, keys);
  if (threadIdx.x < 8) bm[(size_t)blockIdx.x * 8 + threadIdx.x] = bmap[threadIdx.x];
}
}  // namespace hcs

extern "C" int hcs_debug_cta_topk(const double* v, int batch, int n, int k, uint32_t* bm, int variant) {
  if (n < 1 || n > 256 || k < 1 || k > n || batch < 1) return 1;
  hcs::topk_test_kernel<<<batch, hcs::kGreedyThreads>>>(v, n, k, bm, variant);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 2;
}
