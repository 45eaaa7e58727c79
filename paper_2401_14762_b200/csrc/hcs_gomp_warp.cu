// hcs_gomp_warp.cu -- warp-per-pixel gOMP with register-resident Householder QR.
//
// Reference: hypercs/solvers.py:248-297 (gomp), stop rule :115-127, y = 0
// shortcut :145-152, non-finite failure :155-157; selection = argmax_k
// (kernels.py:31-41); least squares = kernels.least_squares (kernels.py:44-67,
// Householder QR + triangular solve).
//
// Why Householder and not normal equations: gOMP's second pass selects its G
// atoms from A^T r where r is the residual of an (often exact) fit, i.e. from
// roundoff.  Which noise columns win depends on the rounding statistics of the
// least-squares solve: a QR solve leaves a component of size ~eps ||y|| in
// range(A) that a refined normal-equations solve removes, and with it the
// selection drifts towards columns outside the fitted set.  Measured on the
// oracle (tools/gomp_rounding_study.py) and on the GPU (profiles/
// gomp_ls_statistics_r02.txt): CSNE gives 2.5x the oracle's 1-ulp tie rate
// and cube PSNR outside the oracle's 1-ulp band; Householder QR sits inside.
//
// Organisation: one warp per pixel, 8 independent warps per CTA (no CTA
// barriers), pixels from a global atomic queue.  Per pass:
//   * correlation p = A^T r: lanes over bands, Psi rows streamed from L2;
//   * top-G by G warp argmax rounds (key = |p| bits, ties to the lowest index);
//   * the columns of the least-squares systems are ordered [S | fills]: when
//     |S| <= kappa the reference's second system top = argmax_k(scatter(s),
//     kappa) is S plus the kappa - |S| lowest-index zero fills (checked after
//     the fact), so ONE Householder QR of [S | fills] gives both solutions:
//     LS(S) from its leading |S| x |S| block and LS(top) from the whole;
//   * the QR: lanes own columns (column c in lane c's registers, up to 96
//     rows), the reflector vector is broadcast through shared memory, each
//     lane applies it to its own column (no cross-lane reductions); y is
//     carried in lanes-over-rows form (Q^T y with a warp sum per reflector);
//     columns beyond the 32 lanes (kappa = 33's top system; |S| up to M
//     once the support outgrows kappa) are "pre-columns": the first
//     K - 32 columns, factored lanes over rows in the warp's global scratch
//     and applied to the lane columns like any other reflector;
//   * residual y - A x from the gathered columns (kept in shared memory),
//     delta, stop rule.
// Pixels outside the fast path (a rank guard min|R_ii| <= 1e-6 max|R_ii|
// where the reference's pivoted rank decision could differ) are handed to
// the CTA kernel (hcs_greedy.cu, pivoted QR mode) through a spill list and
// solved there from scratch.
#include "hcs_internal.cuh"

namespace hcs {

constexpr int kWarpCols = 33;   // columns kept in shared memory (orig): the top system, kappa <= 33
constexpr int kWarpMaxK = 96;   // LS columns of the fast path: 32 lane columns + up to 64 pre-columns
constexpr int kGwWarps = 8;     // warps (pixels) per CTA

struct GwBytes {
  uint8_t msk[128];
  uint8_t cols[128];
  uint32_t supp[8];
  uint32_t sel[8];
};

struct GwLayout {
  int ldc;                // leading dimension of the gathered columns (odd: conflict-free lane-column reads)
  int orig, vb, r, y, xv;     // double offsets (vb: reflector vector / back-substitution buffers / x row)
  int bytes_off;          // byte region offset (in doubles)
  size_t bytes;           // per warp, 16-byte aligned
};

__host__ __device__ inline GwLayout gw_layout(int M) {
  GwLayout L;
  L.ldc = M | 1;
  int o = 0;
  L.orig = o; o += kWarpCols * L.ldc;
  o = (o + 1) & ~1;
  L.vb = o; o += kMaxN;       // reflector vector (MR) / dense x row / scatter scratch (N)
  L.r = o; o += M;
  L.y = o; o += M;
  L.xv = o; o += kWarpMaxK;    // x values (and the pre-columns' during the solve)
  L.bytes_off = o;
  size_t b = sizeof(double) * (size_t)o;
  b += sizeof(GwBytes);       // mask, column list, bitmaps
  L.bytes = (b + 15) & ~(size_t)15;
  return L;
}


__device__ __forceinline__ unsigned long long gw_key(double v) {
  // argmax_k order (stable argsort of -|v|): larger |v| first, NaN last; 0 = taken
  const double a = fabs(v);
  if (a != a) return 1ull;
  return (unsigned long long)__double_as_longlong(a) + 2ull;
}

__device__ __forceinline__ void gw_trace(const Stats& st, long long pid, int& ncall, const uint32_t* bm, int lane) {
  if (st.trace != nullptr && ncall < st.trace_calls && lane < 4) {
    uint64_t* dst = st.trace + ((size_t)pid * st.trace_calls + ncall) * 4;
    dst[lane] = (uint64_t)bm[2 * lane] | ((uint64_t)bm[2 * lane + 1] << 32);
  }
  ++ncall;
}

// sorted index list of a 256-bit bitmap (one warp); returns the count
__device__ __forceinline__ int bitmap_to_list_warp(const uint32_t* bm, uint8_t* list, int lane) {
  int base = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const uint32_t word = bm[e];
    if ((word >> lane) & 1u) list[base + __popc(word & ((1u << lane) - 1u))] = (uint8_t)(32 * e + lane);
    base += __popc(word);
  }
  __syncwarp();
  return base;
}

// ---------------------------------------------------------------- QR passes
// a[MR]: this lane's column (rows 0..MR, MR a multiple of 4).  Loops over the
// rows >= some runtime bound must index a[] statically: a switch on the first
// 4-row chunk falls through an unrolled sequence of per-chunk bodies (Duff's
// device; nvcc emits one indexed branch).  Chunks past MR compile to nothing.
#define GW_CASES(X) X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) \
  X(12) X(13) X(14) X(15) X(16) X(17) X(18) X(19) X(20) X(21) X(22) X(23)

template <int MR>
__host__ __device__ constexpr int gw_slots() { return (MR + 31) / 32; }   // lanes-over-rows slots (y, z)

template <int MR, int CB>
__device__ __forceinline__ void gw_dot_chunk(const double (&a)[MR], const double2* v2, double (&d)[8]) {
  if constexpr (4 * CB + 3 < MR) {
    constexpr int o = 4 * (CB & 1);   // even / odd chunks: two sets of four partial sums (FP64 latency)
    const double2 va = v2[2 * CB], vc = v2[2 * CB + 1];
    d[o] = fma(va.x, a[4 * CB], d[o]);
    d[o + 1] = fma(va.y, a[4 * CB + 1], d[o + 1]);
    d[o + 2] = fma(vc.x, a[4 * CB + 2], d[o + 2]);
    d[o + 3] = fma(vc.y, a[4 * CB + 3], d[o + 3]);
  }
}

template <int MR, int CB>
__device__ __forceinline__ void gw_upd_chunk(double (&a)[MR], const double2* v2, double f) {
  if constexpr (4 * CB + 3 < MR) {
    const double2 va = v2[2 * CB], vc = v2[2 * CB + 1];
    a[4 * CB] = fma(-f, va.x, a[4 * CB]);
    a[4 * CB + 1] = fma(-f, va.y, a[4 * CB + 1]);
    a[4 * CB + 2] = fma(-f, vc.x, a[4 * CB + 2]);
    a[4 * CB + 3] = fma(-f, vc.y, a[4 * CB + 3]);
  }
}

template <int MR, int CB>
__device__ __forceinline__ void gw_nrm_chunk(const double (&a)[MR], double (&n)[4]) {
  if constexpr (4 * CB + 3 < MR) {
#pragma unroll
    for (int t = 0; t < 4; ++t) n[t] = fma(a[4 * CB + t], a[4 * CB + t], n[t]);
  }
}

// rows >= lo of chunk CB only (the partial chunk of a norm)
template <int MR, int CB>
__device__ __forceinline__ void gw_nrm_part(const double (&a)[MR], int lo, double (&n)[4]) {
  if constexpr (4 * CB + 3 < MR) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (4 * CB + t >= lo) n[t] = fma(a[4 * CB + t], a[4 * CB + t], n[t]);
  }
}

template <int MR, int CB>
__device__ __forceinline__ void gw_copy_chunk(const double (&a)[MR], double2* v2) {
  if constexpr (4 * CB + 3 < MR) {
    v2[2 * CB] = make_double2(a[4 * CB], a[4 * CB + 1]);
    v2[2 * CB + 1] = make_double2(a[4 * CB + 2], a[4 * CB + 3]);
  }
}

// d = sum_i v_i a_i and a_i -= f v_i over the rows >= 16 (j / 16): v is zero
// on every row below j (gw_qr keeps the finished rows of vb cleared), so the
// extra terms add exact zeros and leave the finished rows of a (R) unchanged,
// bit for bit what a loop from row j would give.  Entering the row loop at a
// 4-row chunk made every chunk its own basic block with the latency of its
// two shared loads exposed (45% of the kernel's stall samples,
// ncu_gomp_warp27_r02_v16); 16-row groups issue eight loads ahead of their
// FMAs (all rows straight-line spills: the column fills the register file).
#define GW_GROUPS(X) X(0) X(1) X(2) X(3) X(4) X(5)
template <int MR>
__device__ __forceinline__ double gw_dot(const double (&a)[MR], const double* vb, int j) {
  double d[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const double2* v2 = reinterpret_cast<const double2*>(vb);
  switch (j >> 4) {
#define GW_DOT_CASE(g) case g: gw_dot_chunk<MR, 4 * g>(a, v2, d); gw_dot_chunk<MR, 4 * g + 1>(a, v2, d); \
                               gw_dot_chunk<MR, 4 * g + 2>(a, v2, d); gw_dot_chunk<MR, 4 * g + 3>(a, v2, d);
    GW_GROUPS(GW_DOT_CASE)
#undef GW_DOT_CASE
    default: break;
  }
  return ((d[0] + d[4]) + (d[1] + d[5])) + ((d[2] + d[6]) + (d[3] + d[7]));
}

template <int MR>
__device__ __forceinline__ void gw_update(double (&a)[MR], const double* vb, int j, double f) {
  const double2* v2 = reinterpret_cast<const double2*>(vb);
  switch (j >> 4) {
#define GW_UPD_CASE(g) case g: gw_upd_chunk<MR, 4 * g>(a, v2, f); gw_upd_chunk<MR, 4 * g + 1>(a, v2, f); \
                               gw_upd_chunk<MR, 4 * g + 2>(a, v2, f); gw_upd_chunk<MR, 4 * g + 3>(a, v2, f);
    GW_GROUPS(GW_UPD_CASE)
#undef GW_UPD_CASE
    default: break;
  }
}

// sum_{rows >= lo} a_i^2 (per lane): the partial chunk, then whole chunks
template <int MR>
__device__ __forceinline__ double gw_norm(const double (&a)[MR], int lo) {
  double n[4] = {0.0, 0.0, 0.0, 0.0};
  if (lo & 3) {
    switch (lo >> 2) {
#define GW_NP_CASE(k) case k: gw_nrm_part<MR, k>(a, lo, n); break;
      GW_CASES(GW_NP_CASE)
#undef GW_NP_CASE
      default: break;
    }
  }
  switch ((lo + 3) >> 2) {
#define GW_NRM_CASE(k) case k: gw_nrm_chunk<MR, k>(a, n);
    GW_CASES(GW_NRM_CASE)
#undef GW_NRM_CASE
    default: break;
  }
  return (n[0] + n[1]) + (n[2] + n[3]);
}

// the owner's column, rows >= 16 (j / 16), into vb (gw_qr clears the rows below j)
template <int MR>
__device__ __forceinline__ void gw_copy(const double (&a)[MR], double* vb, int j) {
  double2* v2 = reinterpret_cast<double2*>(vb);
  switch (j >> 4) {
#define GW_CPY_CASE(g) case g: gw_copy_chunk<MR, 4 * g>(a, v2); gw_copy_chunk<MR, 4 * g + 1>(a, v2); \
                               gw_copy_chunk<MR, 4 * g + 2>(a, v2); gw_copy_chunk<MR, 4 * g + 3>(a, v2);
    GW_GROUPS(GW_CPY_CASE)
#undef GW_CPY_CASE
    default: break;
  }
}

// the owner's rows 0 .. 16 ceil(c / 16) - 1 into cb (R's column c above the
// diagonal, plus rows >= c that the reader ignores): reverse Duff over 16-row groups
template <int MR, int CB>
__device__ __forceinline__ void gw_rcol_chunk(const double (&a)[MR], double2* c2) {
  if constexpr (4 * CB + 3 < MR) {
    c2[2 * CB] = make_double2(a[4 * CB], a[4 * CB + 1]);
    c2[2 * CB + 1] = make_double2(a[4 * CB + 2], a[4 * CB + 3]);
  }
}
template <int MR>
__device__ __forceinline__ void gw_rcol(const double (&a)[MR], double* cb, int c) {
  double2* c2 = reinterpret_cast<double2*>(cb);
  switch ((c + 15) >> 4) {   // 16-row groups (c+15)/16 - 1 .. 0
#define GW_RC_CASE(g) case g + 1: gw_rcol_chunk<MR, 4 * g + 3>(a, c2); gw_rcol_chunk<MR, 4 * g + 2>(a, c2); \
                                  gw_rcol_chunk<MR, 4 * g + 1>(a, c2); gw_rcol_chunk<MR, 4 * g>(a, c2);
    GW_RC_CASE(5) GW_RC_CASE(4) GW_RC_CASE(3) GW_RC_CASE(2) GW_RC_CASE(1) GW_RC_CASE(0)
#undef GW_RC_CASE
    default: break;
  }
}

// Householder QR of the K gathered columns and Q^T y.  Columns e .. K-1
// (e = max(0, K - 32)) are in the lanes' registers (lane L owns column e + L,
// loaded from orig slot e + L - e0); the e "pre-columns" 0 .. e-1 live in
// the warp's global scratch P (column c at P + c M) and are factored lanes
// over rows, in place.  Returns: each lane's R column part in a[0..] and its
// diagonal in rdiag; P's columns hold R above and on their diagonal; yw
// (lanes over rows) = Q^T y.
// Reflector j (LAPACK dlarfg, unscaled: H c = c - g (v^T c) v with
// v = [alpha - beta; x], beta = -sign(alpha) ||[alpha; x]||,
// g = 1 / (beta (beta - alpha))): its column goes to vb (the owner lane's
// registers, or the pre-column), every lane reads xnorm^2 = sum_{i>j} v_i^2
// (lanes over rows + warp sum) and alpha = v_j, then applies H to its own
// column; the warp applies it to y and to the later pre-columns.
template <int MR>
__device__ __forceinline__ void gw_qr(double (&a)[MR], double& rdiag, double (&yw)[gw_slots<MR>()],
                                      const double* orig, int ldc, int e0, double* P, double* vb, int K, int M,
                                      int lane) {
  constexpr int Q = gw_slots<MR>();
  const int e = K > 32 ? K - 32 : 0;
  const int myc = e + lane;
#pragma unroll
  for (int i = 0; i < MR; ++i) a[i] = (myc < K && i < M) ? orig[(myc - e0) * ldc + i] : 0.0;
  rdiag = 0.0;
  for (int j = 0; j < K; ++j) {
    const int owner = j - e;   // < 0: pre-column j (lanes over rows, in P)
    if (owner < 0) {
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int row = lane + 32 * q;
        if (row < MR) vb[row] = row < M ? P[j * M + row] : 0.0;
      }
    } else if (lane == owner) {
      gw_copy<MR>(a, vb, j);
    }
    __syncwarp();
    double part = 0.0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int row = lane + 32 * q;
      if (row > j && row < M) part = fma(vb[row], vb[row], part);
    }
    const double xn2 = warp_sum(part);
    const double al = vb[j];
    double g = 0.0, amb = 0.0, beta = al;
    if (xn2 != 0.0) {
      beta = -copysign(sqrt(fma(al, al, xn2)), al);
      amb = al - beta;
      g = __drcp_rn(beta * (beta - al));   // correctly rounded, as 1.0 / x, off the DDIV path
    }
    if (owner < 0) {
      if (lane == (j & 31)) P[j * M + j] = beta;   // R_jj of the pre-column
    } else if (lane == owner) {
      rdiag = beta;
    }
    __syncwarp();   // every lane has read v_j
    if (owner < 0) {   // pre-columns: v over all rows (lanes over rows read them)
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int row = lane + 32 * q;
        if (row < j) vb[row] = 0.0;
      }
      if (lane == 0) vb[j] = amb;
    } else {
      // v: row j -> alpha - beta; the rows below j of its 16-row group (just
      // copied: R entries of the owner) -> 0, and row j - 1 (the last
      // reflector's alpha - beta, possibly in the group before) -> 0, so
      // that vb is zero on every row below j for the group-wise dot / update
      const int g0 = j & ~15;
      if (lane <= j - g0) vb[g0 + lane] = (g0 + lane == j) ? amb : 0.0;
      if (j > 0 && lane == 31) vb[j - 1] = 0.0;
    }
    __syncwarp();
    double py = 0.0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int row = lane + 32 * q;
      if (row >= j && row < M) py = fma(vb[row], yw[q], py);
    }
    const double f = gw_dot<MR>(a, vb, j) * g;
    gw_update<MR>(a, vb, j, f);
    // the later pre-columns (rare: supports beyond 32 columns), two at a time
    for (int k = j + 1; k < e; k += 2) {
      const bool two = k + 1 < e;
      double p0 = 0.0, p1 = 0.0;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int row = lane + 32 * q;
        if (row >= j && row < M) {
          p0 = fma(vb[row], P[k * M + row], p0);
          if (two) p1 = fma(vb[row], P[(k + 1) * M + row], p1);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        p0 += __shfl_xor_sync(0xffffffffu, p0, o);
        p1 += __shfl_xor_sync(0xffffffffu, p1, o);
      }
      p0 *= g;
      p1 *= g;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int row = lane + 32 * q;
        if (row >= j && row < M) {
          P[k * M + row] = fma(-p0, vb[row], P[k * M + row]);
          if (two) P[(k + 1) * M + row] = fma(-p1, vb[row], P[(k + 1) * M + row]);
        }
      }
    }
    const double fy = warp_sum(py) * g;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int row = lane + 32 * q;
      if (row >= j && row < M) yw[q] = fma(-fy, vb[row], yw[q]);
    }
    __syncwarp();   // vb (and P) are rewritten by the next reflector
  }
}

// z / r given ri ~ 1/r: q = z ri, corrected by the exact residual z - q r
// (one FMA-based correction: the quotient within an ulp of z / r)
__device__ __forceinline__ double gw_div(double z, double r, double ri) {
  const double q = z * ri;
  return fma(fma(-q, r, z), ri, q);
}

// Back substitution R x = z, column-oriented as LAPACK's dtrsv ('U', 'N'):
// for c = K-1 .. 0: x_c = z_c / R_cc, then z_i -= R_ic x_c for i < c.
// Column c of R is staged through shared memory (cbuf, two 96-double
// buffers) from its owner lane's registers, or read from P for a
// pre-column.  Solves the full system (xt) and the leading s x s block
// (xs, the LS(S) prefix; s <= 33) together.  Lane L receives x of column
// e + L; pre-column x values go to xpre[c] (and x0s for c = 0).
template <int MR>
__device__ __forceinline__ void gw_solve(const double (&a)[MR], double rdiag, const double (&yw)[gw_slots<MR>()],
                                         const double* P, int M, int K, int s, int lane, double* cbuf, double& xt,
                                         double& xs, double* xpre, double& x0s) {
  const int e = K > 32 ? K - 32 : 0;
  constexpr int Q = gw_slots<MR>();
  double zt0 = yw[0];                                   // rows lane, lane + 32, lane + 64
  double zt1 = Q > 1 ? yw[Q > 1 ? 1 : 0] : 0.0;
  double zt2 = Q > 2 ? yw[Q > 2 ? 2 : 0] : 0.0;
  double zs0 = zt0, zs1 = zt1;
  xt = 0.0;
  xs = 0.0;
  x0s = 0.0;
  for (int c = K - 1; c >= 0; --c) {
    const int owner = c - e;   // < 0: a pre-column
    const double* cb;
    double rcc;
    if (owner >= 0) {
      double* w = cbuf + (c & 1) * 96;
      if (lane == owner) gw_rcol<MR>(a, w, c);
      rcc = __shfl_sync(0xffffffffu, rdiag, owner & 31);
      cb = w;
    } else {
      cb = P + c * M;
      rcc = P[c * M + c];
    }
    const double zct = __shfl_sync(0xffffffffu, (c >> 5) == 2 ? zt2 : ((c >> 5) ? zt1 : zt0), c & 31);
    const double zcs = __shfl_sync(0xffffffffu, (c >> 5) ? zs1 : zs0, c & 31);
    // x = z / R_cc: the reciprocal's Newton step and one residual correction
    // (the division's own refinement, off the 100-cycle DDIV path)
    double ri = __drcp_rn(rcc);
    const double vt = gw_div(zct, rcc, ri);
    const double vs = c < s ? gw_div(zcs, rcc, ri) : 0.0;
    if (owner < 0) {
      if (lane == 0) xpre[c] = vt;
      if (c == 0) x0s = vs;
    } else if (lane == owner) {
      xt = vt;
      xs = vs;
    }
    __syncwarp();
    // z_i -= R_ic x_c for rows i < c (slot 0: i < 32; slot 1: 32 <= i < c)
    if (lane < c) {
      const double r = cb[lane];
      zt0 = fma(-r, vt, zt0);
      if (c < s) zs0 = fma(-r, vs, zs0);
    }
    if (lane + 32 < c) zt1 = fma(-cb[lane + 32], vt, zt1);
    if (lane + 64 < c) zt2 = fma(-cb[lane + 64], vt, zt2);
  }
}

// ---------------------------------------------------------------- kernel

template <int MR>
__global__ void __launch_bounds__(32 * kGwWarps, 1) gomp_warp_kernel(GreedyArgs a, GwSpill sp) {
  if (*(volatile const int*)a.err & kErrMask) return;   // invalid masks (validate_masks_kernel)
  extern __shared__ __align__(16) unsigned char smraw[];
  hcs_smem_poison(smraw, a.smem_bytes);
  const int N = a.N, M = a.M;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const GwLayout L = gw_layout(M);
  double* S = reinterpret_cast<double*>(smraw + (size_t)warp * L.bytes);
  double* orig = S + L.orig;
  double* vb = S + L.vb;
  double* rs = S + L.r;
  double* ys = S + L.y;
  double* xv = S + L.xv;
  GwBytes& gb = *reinterpret_cast<GwBytes*>(S + L.bytes_off);
  // this warp's global scratch for pre-columns (least-squares systems beyond 32 columns)
  double* P = sp.pre + (size_t)(blockIdx.x * (blockDim.x >> 5) + warp) * (size_t)sp.pre_stride;
  const int kappa = a.prm.kappa, G = a.prm.G;
  const double NaN = __longlong_as_double(0x7ff8000000000000ll);
  constexpr int Q = gw_slots<MR>();

  for (;;) {
    long long pid = 0;
    if (lane == 0) pid = (long long)atomicAdd(a.counter, 1ull);
    pid = __shfl_sync(0xffffffffu, pid, 0);
    if (pid >= a.P) break;
    // ---- load the pixel ---------------------------------------------------
    int nz = 0, bad = 0;
    for (int j = lane; j < M; j += 32) {
      const double v = a.y[pid * M + j];
      ys[j] = v;
      rs[j] = v;
      gb.msk[j] = a.mask[pid * M + j];
      nz |= (v != 0.0);
      bad |= !isfinite(v);
    }
    if (lane < 8) gb.supp[lane] = 0u;
    const long long t0 = now_ns();
    nz = __any_sync(0xffffffffu, nz);
    bad = __any_sync(0xffffffffu, bad);
    __syncwarp();
    if (!nz || bad) {   // y == 0 shortcut; non-finite y: scipy raises ValueError (kernels.py:61)
      if (bad && lane == 0) atomicOr(a.err, 1);
      for (int n = lane; n < N; n += 32) a.x_out[pid * N + n] = 0.0;
      if (lane == 0) {
        a.st.iterations[pid] = 0;
        a.st.converged[pid] = bad ? 0 : 1;
        a.st.final_delta[pid] = bad ? NaN : 0.0;
        a.st.failed_at[pid] = -1;
        if (a.st.trace_len) a.st.trace_len[pid] = 0;
        if (a.st.elapsed) a.st.elapsed[pid] = 0.0;
        if (a.st.work) a.st.work[pid] = 0.0;
      }
      continue;
    }
    double delta = 1.0;
    int iters = 0, ncall = 0, kx = 0;
    bool converged = false, failed = false, spill = false;
    double work = 0.0;
    for (;;) {
      // ---- stop rule before the pass (solvers.py:115-127) -------------------
      int dec = 0;
      if (lane == 0) dec = stop_decision(delta, iters, t0, a.prm);
      dec = __shfl_sync(0xffffffffu, dec, 0);
      if (dec != kContinue) { converged = dec == kConverged; break; }
      // ---- correlation p = A^T r: lanes over bands, Psi rows from L2 --------
      double p[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) p[c] = 0.0;
      {
        // four measured rows per step: 32 independent L2 loads in flight per
        // lane (the same FMA order as one row at a time)
        int j = 0;
        for (; j + 3 < M; j += 4) {
          double b[4][8], rr[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            rr[u] = rs[j + u];
            const double* row = a.basis + (size_t)gb.msk[j + u] * N + lane;
#pragma unroll
            for (int c = 0; c < 8; ++c) b[u][c] = lane + 32 * c < N ? __ldg(row + 32 * c) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int c = 0; c < 8; ++c) p[c] = fma(b[u][c], rr[u], p[c]);
        }
        for (; j < M; ++j) {
          const double r0 = rs[j];
          const double* row0 = a.basis + (size_t)gb.msk[j] * N + lane;
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (lane + 32 * c < N) p[c] = fma(__ldg(row0 + 32 * c), r0, p[c]);
        }
      }
      // ---- top-G (argmax_k, kernels.py:31-41) by G warp argmax rounds ---------
      {
        unsigned long long key[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) key[c] = lane + 32 * c < N ? gw_key(p[c]) : 0ull;
        uint32_t selw = 0u;   // lane's word: bit c <-> index lane + 32 c
        for (int g = 0; g < G; ++g) {
          unsigned long long bk = 0ull;
          int bi = 1 << 30;
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (key[c] > bk) { bk = key[c]; bi = lane + 32 * c; }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long ok = __shfl_xor_sync(0xffffffffu, bk, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ok > bk || (ok == bk && oi < bi)) { bk = ok; bi = oi; }
          }
          if ((bi & 31) == lane) {
            const int c = bi >> 5;
#pragma unroll
            for (int cc = 0; cc < 8; ++cc)
              if (cc == c) key[cc] = 0ull;
            selw |= 1u << c;
          }
        }
        // transpose to index bitmaps: word w bit b <-> index 32 w + b
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint32_t m = __ballot_sync(0xffffffffu, (selw >> c) & 1u);
          if (lane == c) gb.sel[c] = m;
        }
        __syncwarp();
        gw_trace(a.st, pid, ncall, gb.sel, lane);
      }
      // ---- support union, outgrowth break ------------------------------------
      uint32_t sw = lane < 8 ? (gb.supp[lane] | gb.sel[lane]) : 0u;
      const int ks = __reduce_add_sync(0xffffffffu, __popc(sw));
      work += 2.0 * N * M;   // correlation
      if (ks > M) break;     // keep the last iterate, no count (solvers.py:274-276)
      __syncwarp();
      if (lane < 8) gb.supp[lane] = sw;
      __syncwarp();
      if (ks > kWarpMaxK) { spill = true; break; }
      // ---- column order [S | fills] ------------------------------------------
      // S sorted, then (ks <= kappa) the kappa - ks lowest indices outside S
      int K;
      {
        int base = 0, fbase = ks, fill_need = ks <= kappa ? kappa - ks : 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          const uint32_t word = gb.supp[w];
          const bool on = (word >> lane) & 1u;
          const int idx = 32 * w + lane;
          if (on) gb.cols[base + __popc(word & ((1u << lane) - 1u))] = (uint8_t)idx;
          base += __popc(word);
          const bool fz = !on && idx < N;
          const uint32_t fm = __ballot_sync(0xffffffffu, fz);
          const int rk = __popc(fm & ((1u << lane) - 1u));
          if (fz && rk < fill_need) gb.cols[fbase + rk] = (uint8_t)idx;
          const int take = __popc(fm) < fill_need ? __popc(fm) : fill_need;
          fbase += take;
          fill_need -= take;
        }
        K = ks <= kappa ? kappa : ks;
      }
      __syncwarp();
      double xt = 0.0;
      bool second = false;
      for (int round = 0; round < 2; ++round) {
        // ---- gather the columns at the measured rows (L2 -> shared / scratch) --
        // K <= 33: all columns to orig slots 0..K-1 (kept for the residual);
        // K > 33 (round 0 of |S| > 33 only): the 32 lane columns to orig slots
        // 0..31; pre-columns (e = K - 32) to the warp's scratch P, factored in place
        const int e = K > 32 ? K - 32 : 0;
        const int e0 = K > kWarpCols ? e : 0;
        HCS_CHECK(a.err, K >= 1 && K <= kWarpMaxK && K - e0 <= kWarpCols && (long long)e * M <= sp.pre_stride);
        for (int c = e0; c < K; ++c) {
          const double* col = a.basis_t + (size_t)gb.cols[c] * N;
          for (int i = lane; i < M; i += 32) cp_async8(orig + (c - e0) * L.ldc + i, col + gb.msk[i]);
        }
        for (int c = 0; c < e; ++c) {
          const double* col = a.basis_t + (size_t)gb.cols[c] * N;
          for (int i = lane; i < M; i += 32) P[c * M + i] = __ldg(col + gb.msk[i]);
        }
        cp_async_wait_all();
        __syncwarp();
        double acol[MR];
        double rdiag;
        double yw[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) yw[q] = lane + 32 * q < M ? ys[lane + 32 * q] : 0.0;
        gw_qr<MR>(acol, rdiag, yw, orig, L.ldc, e0, P, vb, K, M, lane);
        // rank guard on the diagonal of R (see header)
        {
          const double dl = (e + lane < K) ? fabs(rdiag) : 0.0;
          double dmax = dl, dmin = (e + lane < K) ? dl : INFINITY;
          for (int c = lane; c < e; c += 32) {
            const double dp = fabs(P[c * M + c]);
            dmax = fmax(dmax, dp);
            dmin = fmin(dmin, dp);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
            dmin = fmin(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
          }
          if (!(dmin > 1e-6 * dmax) || K > M) { spill = true; break; }
        }
        const int s = (!second && ks <= kappa) ? ks : 0;
        double xs, x0s;
        gw_solve<MR>(acol, rdiag, yw, P, M, K, s, lane, vb, xt, xs, xv, x0s);
        if (second) break;   // second round done: xt is LS(top)
        // the top call: argmax_k(scatter(LS(S)), kappa) over all N bands.
        // |S| <= kappa: the predicted top [S | fills] is the real one iff every
        // LS(S) coefficient is nonzero (zeros tie with the fills, NaN ranks
        // last); otherwise (or |S| > kappa) the exact warp top-k selects it and
        // a second QR solves on those columns
        const int myc = e + lane;
        bool general = ks > kappa;
        double sv = xs;
        if (general) {
          sv = xt;      // |S| > kappa: the first round solved S itself (pre-columns in xv)
        } else {
          bool zero = (myc < s) && !(xs != 0.0 && xs == xs);
          if (e && lane == 0) zero |= !(x0s != 0.0 && x0s == x0s);
          general = __any_sync(0xffffffffu, zero);
          if (general && e && lane == 0) xv[0] = x0s;   // the pre-column's LS(S) value for the scatter
        }
        if (general) {
          for (int n = lane; n < N; n += 32) vb[n] = 0.0;
          __syncwarp();
          for (int c = lane; c < e; c += 32) vb[gb.cols[c]] = xv[c];
          if (myc < ks) vb[gb.cols[myc]] = sv;
          __syncwarp();
          warp_topk(vb, N, kappa, gb.sel);
          __syncwarp();
          gw_trace(a.st, pid, ncall, gb.sel, lane);
          bitmap_to_list_warp(gb.sel, gb.cols, lane);
          K = kappa;
          second = true;
          __syncwarp();
          continue;
        }
        {
          // trace record of the top call: the bitmap of [S | fills]
          uint32_t tw = 0u;
          for (int c = 0; c < K; ++c) {
            const int idx = gb.cols[c];
            if ((idx >> 5) == lane) tw |= 1u << (idx & 31);
          }
          if (lane < 8) gb.sel[lane] = tw;
          __syncwarp();
          gw_trace(a.st, pid, ncall, gb.sel, lane);
        }
        break;
      }
      if (spill) break;
      work += ls_flops(M, ks) + ls_flops(M, kappa);
      // ---- new iterate, residual, delta (solvers.py:285-290) ------------------
      // x over cols[0..K): pre-column values are in xv already (gw_solve)
      kx = K;
      {
        const int e = K > 32 ? K - 32 : 0;
        __syncwarp();
        if (e + lane < K) xv[e + lane] = xt;
      }
      __syncwarp();
      double part = 0.0;
      int nf = 0;
      for (int i = lane; i < M; i += 32) {
        double acc0 = 0.0, acc1 = 0.0;
        int c = 0;
        for (; c + 1 < K; c += 2) {
          acc0 = fma(orig[c * L.ldc + i], xv[c], acc0);
          acc1 = fma(orig[(c + 1) * L.ldc + i], xv[c + 1], acc1);
        }
        if (c < K) acc0 = fma(orig[c * L.ldc + i], xv[c], acc0);
        const double rn = ys[i] - (acc0 + acc1);
        const double d = rn - rs[i];
        part = fma(d, d, part);
        rs[i] = rn;
      }
      for (int c = lane; c < K; c += 32) nf |= !isfinite(xv[c]);
      delta = sqrt(warp_sum(part));
      work += 2.0 * M * K;
      nf = __any_sync(0xffffffffu, nf);
      __syncwarp();
      ++iters;
      if (nf || !isfinite(delta)) { failed = true; break; }
    }
    if (spill) {
      if (lane == 0) {
        const unsigned long long k = atomicAdd(sp.count, 1ull);
        sp.list[k] = pid;
      }
      __syncwarp();
      continue;
    }
    // ---- results: dense x row through shared memory -------------------------------
    for (int n = lane; n < N; n += 32) vb[n] = 0.0;
    __syncwarp();
    if (!failed)
      for (int c = lane; c < kx; c += 32) vb[gb.cols[c]] = xv[c];
    __syncwarp();
    for (int n = lane; n < N; n += 32) a.x_out[pid * N + n] = vb[n];
    if (lane == 0) {
      a.st.iterations[pid] = failed ? 0 : iters;
      a.st.converged[pid] = converged ? 1 : 0;
      a.st.final_delta[pid] = failed ? NaN : delta;
      a.st.failed_at[pid] = failed ? iters : -1;
      if (a.st.trace_len) a.st.trace_len[pid] = ncall;
      if (a.st.elapsed) a.st.elapsed[pid] = 1e-9 * (double)(now_ns() - t0);
      if (a.st.work) a.st.work[pid] = work;
    }
    __syncwarp();
  }
#ifdef HCS_CHECKS
  if (a.selftest && blockIdx.x == 0 && threadIdx.x == 0) smraw[a.smem_bytes + 8] ^= 1;   // positive control
#endif
  hcs_smem_canary(smraw, a.smem_bytes, a.err);
}

bool gomp_warp_supported(int N, int M, int kappa) {
  // pre-column scratch: the columns beyond the 32 lanes (K <= M, so at most
  // M - 32 of them) of M rows each per warp, in a CTA scratch slot
  const size_t pre = M > 32 ? (size_t)(M - 32) : 0;
  return M >= 1 && M <= 96 && kappa <= kWarpCols && N <= kMaxN && pre * (size_t)M <= greedy_ls_doubles(M);
}

size_t gomp_warp_smem(int M, int* warps) {
  const GwLayout L = gw_layout(M);
  int w = kGwWarps;
  while (w > 1 && L.bytes * w + kSmemExtra > 227 * 1024) --w;
  *warps = w;
  return L.bytes * w;
}

template <int MR>
static cudaError_t launch_gw_t(const GreedyArgs& args, const GwSpill& sp, int grid, int warps, size_t smem,
                               cudaStream_t stream) {
  cudaError_t e = cudaFuncSetAttribute(gomp_warp_kernel<MR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(smem + kSmemExtra));
  if (e != cudaSuccess) return e;
  GreedyArgs ga = args;
  ga.smem_bytes = (unsigned)smem;
  gomp_warp_kernel<MR><<<grid, 32 * warps, smem + kSmemExtra, stream>>>(ga, sp);
  return cudaGetLastError();
}

cudaError_t launch_gomp_warp(const GreedyArgs& args, const GwSpill& sp, int sms, long long slots,
                             cudaStream_t stream) {
  int warps = 0;
  const size_t smem = gomp_warp_smem(args.M, &warps);
  long long grid = sms;
  if (grid * warps > slots) grid = slots / warps;   // one pre-column scratch slot per warp
  const long long need = (args.P + warps - 1) / warps;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  // register column of MR rows, the smallest instantiation >= M
  if (args.M <= 32) return launch_gw_t<32>(args, sp, (int)grid, warps, smem, stream);
  if (args.M <= 48) return launch_gw_t<48>(args, sp, (int)grid, warps, smem, stream);
  if (args.M <= 64) return launch_gw_t<64>(args, sp, (int)grid, warps, smem, stream);
  if (args.M <= 80) return launch_gw_t<80>(args, sp, (int)grid, warps, smem, stream);
  if (args.M <= 92) return launch_gw_t<92>(args, sp, (int)grid, warps, smem, stream);
  return launch_gw_t<96>(args, sp, (int)grid, warps, smem, stream);
}

}  // namespace hcs
