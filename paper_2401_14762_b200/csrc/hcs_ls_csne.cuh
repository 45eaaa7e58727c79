// hcs_ls_csne.cuh -- least squares by corrected semi-normal equations on FP64
// tensor cores: the fast path of hypercs.kernels.least_squares
// (kernels.py:44-67) for the greedy solvers.
//
//   [B y]^T [B y] by DMMA (lower 8 x 8 tiles)      -> G = B^T B, g = B^T y
//   blocked Cholesky of the augmented Gram          -> L (= R^T), z = L^-1 g (its last row)
//   back substitution L^T s = z                     -> s
//   one refinement step (CSNE): r = y - B s, s += (L L^T)^-1 B^T r
//
// For full-rank B the Cholesky factor equals the R of an (unpivoted) QR up to
// signs, and one step of refinement with the exact residual brings the
// semi-normal-equations solution to the accuracy of a backward-stable QR solve
// when cond(B)^2 eps << 1 (Bjorck 1987); the greedy systems here have
// cond(B) <= 1.1e3.  The reference's rank decision
// (pivoted QR, min|R_ii| > 1e-10 max|R_ii|) is guarded: a non-positive pivot,
// min|L_ii| <= kCsneGuard max|L_ii|, or a refinement step larger than
// kCsneStep relative to s sends the caller to the exact column-pivoted
// restatement (hcs_ls.cuh).  The serial work is one 8 x 8 Cholesky and one
// 8 x 8 inverse per 8 columns; everything else is DMMA tiles or
// column-parallel.
//
// Layout: B COLUMN-major (element (r, c) at B[c * ld + r]), rows >= M zero, the
// measurements y as column K, columns K+1 .. round8(K+1)-1 zero.  G holds the
// lower 8 x 8 tiles of the augmented Gram, tile (bi, bj) (bi >= bj) at
// ((bi (bi + 1) / 2 + bj) * kTileSlot, column-major inside the tile (element
// (i, k) at (k & 7) * 8 + (i & 7)); the padded slot keeps lanes that walk the
// rows of one column conflict-free.  Diagonal tiles keep L in their lower part
// and the inverse Linv (transposed) in their strictly upper part.
#pragma once
#include "hcs_common.cuh"

namespace hcs {

constexpr double kCsneGuard = 1e-6;
constexpr double kCsneStep = 1e-6;
constexpr int kTileSlot = 68;

__device__ __forceinline__ void dmma8x(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// Column-major leading dimension for M rows: a multiple of 4 that is 4 or 12
// mod 16 (DMMA fragments: 8 columns x 4 consecutive rows conflict-free).
__host__ __device__ __forceinline__ int csne_ld(int M) {
  const int m4 = (M + 3) & ~3;
  return (m4 & 7) ? m4 : m4 + 4;
}
__host__ __device__ __forceinline__ int csne_cols(int K) { return (K + 1 + 7) & ~7; }
__host__ __device__ __forceinline__ int csne_gram_doubles(int K) {
  const int nb = csne_cols(K) >> 3;
  return nb * (nb + 1) / 2 * kTileSlot;
}
__host__ __device__ __forceinline__ int gtile(int bi, int bj) { return (bi * (bi + 1) / 2 + bj) * kTileSlot; }
// element (i, k), i >= k block-wise
__device__ __forceinline__ int gel(int i, int k) { return gtile(i >> 3, k >> 3) + (k & 7) * 8 + (i & 7); }

// Row a of linear index t in a lower-triangular enumeration (t = a (a + 1) / 2 + b,
// b <= a): closed form with a one-step correction (exact for t < 2^20).
__device__ __forceinline__ int tri_row(int t) {
  int a = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
  if ((a + 1) * (a + 2) / 2 <= t) ++a;
  if (a * (a + 1) / 2 > t) --a;
  return a;
}

// Gram entries of a DCT-II dictionary without touching its rows.  With
// Psi[m][c] = s_c cos(theta_m c), theta_m = pi (2 m + 1) / (2 N), s_0 = sqrt(1/N),
// s_c = sqrt(2/N), the product-to-sum identity gives, for A = Psi[mask, :],
//     (A^T A)[i][j] = s_i s_j / 2 (F(|i - j|) + F(i + j)),
//     F(d) = sum_{m in mask} cos(theta_m d),  F(N) = 0,  F(d) = -F(2 N - d) for d > N:
// every Gram entry of every support is two lookups in the pixel's F (N
// doubles, computed once per pixel as (A^T 1)[d] / s_d) instead of an M-term
// dot product.  Used only when the basis was verified to be the DCT-II
// (transpose_basis_kernel); any other orthonormal basis takes the DMMA Gram.
struct DctGram {
  const double* F;       // F(d), d < N (shared memory)
  const double* q;       // A^T y over all N atoms (shared memory): the Gram's y row is q[cols[.]]
  const uint8_t* cols;   // the system's dictionary column indices
  int N;
  double s0, s1;         // sqrt(1/N), sqrt(2/N)
  double yty;            // y^T y
};
__device__ __forceinline__ double dct_gram_entry(const DctGram& dg, int ci, int cj) {
  const int dm = ci > cj ? ci - cj : cj - ci, dp = ci + cj;
  const double fm = dg.F[dm];
  const double fp = dp < dg.N ? dg.F[dp] : (dp == dg.N ? 0.0 : -dg.F[2 * dg.N - dp]);
  return (0.5 * (ci ? dg.s1 : dg.s0) * (cj ? dg.s1 : dg.s0)) * (fm + fp);
}

struct CsneScratch {   // shared memory
  double* G;      // csne_gram_doubles(K)
  double* dinv;   // >= round8(K + 1): 1 / L_ii
  double* c;      // >= round8(K + 1): right-hand side / solution workspace
  double* r;      // >= M: residual
  double* red;    // >= 2 * warps
  int* flag;      // 2: [0] guard flag, [1] Gram tile counter (1 between calls)
};

// Back substitution L^T x = c on the first K entries (c in/out, x overwrites c).  Warp 0.
static __device__ __noinline__ void csne_backward(const double* G, const double* dinv, double* c, int K) {
  const int lane = threadIdx.x & 31;
  const int nb = (K + 7) >> 3;
  for (int bb = nb - 1; bb >= 0; --bb) {
    const int o = 8 * bb;
    const int base = gtile(bb, bb);
    double xj = 0.0;
    if (lane < 8 && o + lane < K) {
      // x_j = sum_{m >= j} Linv[m][j] c_m ; Linv[m][j] (m > j) sits at (row j, col m) of the tile
      const int j = lane;
      xj = dinv[o + j] * c[o + j];
#pragma unroll
      for (int m = 1; m < 8; ++m)
        if (m > j && o + m < K) xj += G[base + m * 8 + j] * c[o + m];
    }
    __syncwarp();
    if (lane < 8 && o + lane < K) c[o + lane] = xj;
    __syncwarp();
    // c_t -= sum_kk L[o + kk][t] x_kk for t < o
    for (int t = lane; t < o; t += 32) {
      const int tb = gtile(bb, t >> 3) + (t & 7) * 8;
      double acc = c[t];
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        if (o + kk < K) acc -= G[tb + kk] * c[o + kk];
      c[t] = acc;
    }
    __syncwarp();
  }
}

// Forward substitution L x = c on the first K entries (in place).  Warp 0.
static __device__ __noinline__ void csne_forward(const double* G, const double* dinv, double* c, int K) {
  const int lane = threadIdx.x & 31;
  const int nb = (K + 7) >> 3;
  for (int bb = 0; bb < nb; ++bb) {
    const int o = 8 * bb;
    const int base = gtile(bb, bb);
    double xj = 0.0;
    if (lane < 8 && o + lane < K) {
      // x_j = sum_{m <= j} Linv[j][m] c_m ; Linv[j][m] (m < j) sits at (row m, col j)
      const int j = lane;
      xj = dinv[o + j] * c[o + j];
#pragma unroll
      for (int m = 0; m < 7; ++m)
        if (m < j) xj += G[base + j * 8 + m] * c[o + m];
    }
    __syncwarp();
    if (lane < 8 && o + lane < K) c[o + lane] = xj;
    __syncwarp();
    // c_t -= sum_kk L[t][o + kk] x_kk for t >= o + 8
    for (int t = o + 8 + lane; t < K; t += 32) {
      const int tb = gtile(t >> 3, bb) + (t & 7);
      double acc = c[t];
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        if (o + kk < K) acc -= G[tb + kk * 8] * c[o + kk];
      c[t] = acc;
    }
    __syncwarp();
  }
}

// One trailing tile: G_ij -= L_ik L_jk^T (one warp, 2 DMMAs).
__device__ __forceinline__ void csne_tile_update(double* G, int bi, int bj, int kb) {
  const int lane = threadIdx.x & 31;
  const int tij = gtile(bi, bj), tik = gtile(bi, kb), tjk = gtile(bj, kb);
  const int ii = lane >> 2, jj0 = 2 * (lane & 3);
  double d[2] = {G[tij + jj0 * 8 + ii], G[tij + (jj0 + 1) * 8 + ii]};
  const int m0 = lane & 3, m1 = 4 + (lane & 3);
  const double a0 = -G[tik + m0 * 8 + ii], a1 = -G[tik + m1 * 8 + ii];
  const double b0 = G[tjk + m0 * 8 + ii], b1 = G[tjk + m1 * 8 + ii];    // B[m][n] = L_jk[n][m], n = lane >> 2
  dmma8x(d, a0, b0);
  dmma8x(d, a1, b1);
  G[tij + jj0 * 8 + ii] = d[0];
  G[tij + (jj0 + 1) * 8 + ii] = d[1];
}

// Warp 0: Cholesky of the 8 x 8 diagonal tile kb (lane ii < 8 holds row ii),
// reciprocal pivots into dinv, and the inverse L_kk^-1 (column jj per lane)
// stored transposed in the tile's strictly upper part.  A non-positive pivot
// clears sc.flag.  Branch-free: lane-dependent conditions are selects and
// predicated stores, and the inverse reads the tile with lane-uniform
// (broadcast) loads issued ahead of its dependency chain; column jj of the
// inverse is zero above the diagonal, so the terms p < jj of its sums add
// exact zeros and need no predicate.
static __device__ __noinline__ void csne_diag_factor(double* G, const CsneScratch& sc, int K, int kb) {
  const int lane = threadIdx.x & 31;
  const int o = 8 * kb;
  const int w = K - o < 8 ? K - o : 8;
  double* T = G + gtile(kb, kb);
  double row[8];
  const int ii = lane & 7;
#pragma unroll
  for (int k = 0; k < 8; ++k) row[k] = T[k * 8 + ii];
  bool ok = true;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    if (c < w) {
      const double d = __shfl_sync(0xffffffffu, row[c], c);
      ok = ok && d > 0.0;
      const double rs = rsqrt(d);
      row[c] = (ii == c) ? d * rs : (ii > c ? row[c] * rs : row[c]);   // L_cc = sqrt(d), L_ic
#pragma unroll
      for (int k = 1; k < 8; ++k) {
        if (k > c) {
          const double lkc = __shfl_sync(0xffffffffu, row[c], k);   // L_kc from lane k
          const double upd = row[k] - row[c] * lkc;
          row[k] = (ii >= k) ? upd : row[k];
        }
      }
    }
  }
  double rii = row[0];
#pragma unroll
  for (int k = 1; k < 8; ++k) rii = (k == ii) ? row[k] : rii;
  const double dii = (ii < w) ? __drcp_rn(rii) : 0.0;   // correctly rounded, as 1.0 / rii, off the DDIV path
  if (lane < 8) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k <= ii) T[k * 8 + ii] = row[k];    // lower part incl. diagonal
    sc.dinv[o + ii] = dii;
  }
  if (lane == 0 && !ok) sc.flag[0] = 0;
  __syncwarp();
  // inverse of L_kk (lower), column jj per lane
  double Lm[8][8], dv[8];
#pragma unroll
  for (int m = 1; m < 8; ++m) {
    dv[m] = sc.dinv[o + m];
#pragma unroll
    for (int p = 0; p < m; ++p) Lm[m][p] = T[p * 8 + m];
  }
  const int jj = ii;
  double x[8];
  x[0] = (jj == 0) ? dii : 0.0;
#pragma unroll
  for (int m = 1; m < 8; ++m) {
    double acc = 0.0;
#pragma unroll
    for (int p = 0; p < m; ++p) acc += Lm[m][p] * x[p];
    const double v = -acc * dv[m];
    x[m] = (m == jj) ? dii : ((m > jj && m < w) ? v : 0.0);
  }
  __syncwarp();
  if (lane < 8) {
#pragma unroll
    for (int m = 1; m < 8; ++m)
      if (m > jj) T[m * 8 + jj] = x[m];         // Linv[m][jj] at (row jj, col m)
  }
  __syncwarp();
}

// Solve min ||B s - y|| (layout above).  Returns 1 with s[0..K) on success, 0
// when a guard trips.  All threads call; ends synchronised.
// DCT = true: `dg` supplies the closed-form augmented Gram (no dictionary column is read for it).
template <bool DCT = false>
static __device__ __noinline__ int ls_csne(const double* B, int ld, int M, int K, double* s, const CsneScratch& sc,
                              long long* ph = nullptr, const DctGram* dg = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, W = blockDim.x >> 5;
  const int M4 = (M + 3) & ~3;
  const int nbA = csne_cols(K) >> 3;      // block rows incl. the y row
  const int nb = (K + 7) >> 3;            // pivot blocks
  double* G = sc.G;
  if (tid == 0) sc.flag[0] = 1;
  // ---- 1. augmented Gram, lower tiles, by DMMA ----------------------------------
  // Warp 0 computes tile (0, 0) and factorises it at once (the first step of
  // 2.) while the other warps take the remaining tiles from a shared counter
  // (flag[1], 1 on entry); warp 0 joins them when its factorisation is done.
  // Every tile is computed by the same instructions whichever warp takes it.
  const int ntiles = nbA * (nbA + 1) / 2;
  // the closed form's arguments in registers (dg points to shared memory)
  const bool closed = DCT && dg != nullptr;
  const double* dF = closed ? dg->F : nullptr;
  const double* dq = closed ? dg->q : nullptr;
  const uint8_t* dcols = closed ? dg->cols : nullptr;
  const int dN = closed ? dg->N : 0;
  const double ds0 = closed ? dg->s0 : 0.0, ds1 = closed ? dg->s1 : 0.0, dyty = closed ? dg->yty : 0.0;
  auto gentry = [&](int ci, int cj) -> double {   // dct_gram_entry on the register copies
    const int dm = ci > cj ? ci - cj : cj - ci, dp = ci + cj;
    const double fm = dF[dm];
    const double fp = dp < dN ? dF[dp] : (dp == dN ? 0.0 : -dF[2 * dN - dp]);
    return (0.5 * (ci ? ds1 : ds0) * (cj ? ds1 : ds0)) * (fm + fp);
  };
  auto gram_tile = [&](int t) {
    const int bi = tri_row(t);
    const int bj = t - bi * (bi + 1) / 2;
    if (closed) {
      // the DCT-II closed form for atom x atom entries; row / column K of the
      // augmented Gram is A^T y at the system's atoms, (K, K) is y^T y, the
      // padding beyond K is zero: no dictionary column is read
      const int i = lane >> 2, j0 = 2 * (lane & 3);
      const int r = 8 * bi + i, c = 8 * bj + j0;
      const int base = gtile(bi, bj) + i;
      // atom indices first (three independent loads), then the lookups
      const int ar = r < K ? dcols[r] : -1;
      const int ac0 = c < K ? dcols[c] : -1, ac1 = c + 1 < K ? dcols[c + 1] : -1;
      double v0 = 0.0, v1 = 0.0;
      if (ar >= 0) {
        if (ac0 >= 0) v0 = gentry(ar, ac0);
        else if (c == K) v0 = dq[ar];
        if (ac1 >= 0) v1 = gentry(ar, ac1);
        else if (c + 1 == K) v1 = dq[ar];
      } else if (r == K) {
        v0 = ac0 >= 0 ? dq[ac0] : (c == K ? dyty : 0.0);
        v1 = ac1 >= 0 ? dq[ac1] : (c + 1 == K ? dyty : 0.0);
      }
      G[base + j0 * 8] = v0;
      G[base + (j0 + 1) * 8] = v1;
      return;
    }
    const double* ca = B + (8 * bi + (lane >> 2)) * ld + (lane & 3);
    const double* cb = B + (8 * bj + (lane >> 2)) * ld + (lane & 3);
    double d0[2] = {0.0, 0.0}, d1[2] = {0.0, 0.0};
    int k0 = 0;
    for (; k0 + 4 < M4; k0 += 8) {
      dmma8x(d0, ca[k0], cb[k0]);
      dmma8x(d1, ca[k0 + 4], cb[k0 + 4]);
    }
    if (k0 < M4) dmma8x(d0, ca[k0], cb[k0]);
    const int base = gtile(bi, bj) + (lane >> 2);
    G[base + (2 * (lane & 3)) * 8] = d0[0] + d1[0];
    G[base + (2 * (lane & 3) + 1) * 8] = d0[1] + d1[1];
  };
  if (warp == 0) {
    gram_tile(0);
    __syncwarp();
    csne_diag_factor(G, sc, K, 0);
  }
  for (;;) {
    int t = 0;
    if (lane == 0) t = atomicAdd(&sc.flag[1], 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= ntiles) break;
    gram_tile(t);
  }
  __syncthreads();
  if (tid == 0) sc.flag[1] = 1;   // every warp is past the counter loop
  HCS_MARKP(ph, 4);
  // ---- 2. blocked right-looking Cholesky with look-ahead --------------------------
  // step kb: panel L_ik = G_ik L_kk^-T (all warps), then warp 0 updates the next
  // diagonal tile and factorises it while warps 1.. apply the rest of the
  // trailing update G_ij -= L_ik L_jk^T.  (The factorisation of tile 0 ran in 1.)
  HCS_MARKP(ph, 11);
  for (int kb = 0; kb < nb; ++kb) {
    const int o = 8 * kb;
    const int w = K - o < 8 ? K - o : 8;
    const int base = gtile(kb, kb);
    // (c) panel: L_ik = G_ik Linv^T for block rows below (incl. the y row)
    for (int bi = kb + 1 + warp; bi < nbA; bi += W) {
      const int bt = gtile(bi, kb);
      const int jj = lane >> 2;
      double a[2], lv[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = 4 * h + (lane & 3);
        a[h] = G[bt + m * 8 + jj];                  // A[ii = jj][m] = G_ik[ii][m]
        lv[h] = (m < jj && jj < w) ? G[base + jj * 8 + m] : (m == jj && jj < w ? sc.dinv[o + jj] : 0.0);
      }
      double dd[2] = {0.0, 0.0};
      dmma8x(dd, a[0], lv[0]);                      // B[m][n = jj] = Linv[jj][m]
      dmma8x(dd, a[1], lv[1]);
      __syncwarp();
      G[bt + (2 * (lane & 3)) * 8 + jj] = dd[0];
      G[bt + (2 * (lane & 3) + 1) * 8 + jj] = dd[1];
    }
    __syncthreads();
    HCS_MARKP(ph, 12);
    // (d) trailing update for step kb, tiles kb < bj <= bi < nbA (bj < nb)
    const int rem = nbA - kb - 1;
    const int ntr = rem * (rem + 1) / 2;
    if (warp == 0) {
      if (kb + 1 < nb) {
        csne_tile_update(G, kb + 1, kb + 1, kb);
        __syncwarp();
        csne_diag_factor(G, sc, K, kb + 1);
      }
    } else {
      for (int t = warp - 1; t < ntr; t += W - 1) {
        const int a = tri_row(t);
        const int bi = kb + 1 + a, bj = kb + 1 + (t - a * (a + 1) / 2);
        if (bj >= nb || (bi == kb + 1 && bj == kb + 1)) continue;
        csne_tile_update(G, bi, bj, kb);
      }
    }
    __syncthreads();
    HCS_MARKP(ph, 13);
  }
  HCS_MARKP(ph, 5);
  // ---- 3. guard, z = last row of L, back substitution ---------------------------
  if (warp == 0) {
    double dmax = 0.0, dmin = INFINITY;
    for (int i = lane; i < K; i += 32) {
      const double dv = fabs(G[gel(i, i)]);
      dmax = fmax(dmax, dv);
      dmin = fmin(dmin, dv);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, off));
      dmin = fmin(dmin, __shfl_xor_sync(0xffffffffu, dmin, off));
    }
    const bool ok = sc.flag[0] && M >= K && dmin > kCsneGuard * dmax;
    if (ok) {
      for (int j = lane; j < K; j += 32) sc.c[j] = G[gel(K, j)];   // z = L^-1 g
      __syncwarp();
      csne_backward(G, sc.dinv, sc.c, K);
    }
    if (lane == 0) sc.flag[0] = ok;
  }
  __syncthreads();
  if (!sc.flag[0]) return 0;
  for (int j = tid; j < K; j += blockDim.x) s[j] = sc.c[j];
  // ---- 4. one CSNE refinement step ------------------------------------------------
  __syncthreads();
  for (int rr = tid; rr < M; rr += blockDim.x) {   // r = y - B s
    double a0 = 0.0, a1 = 0.0;
    int c = 0;
    for (; c + 1 < K; c += 2) {
      a0 += B[c * ld + rr] * s[c];
      a1 += B[(c + 1) * ld + rr] * s[c + 1];
    }
    if (c < K) a0 += B[c * ld + rr] * s[c];
    sc.r[rr] = B[K * ld + rr] - (a0 + a1);
  }
  __syncthreads();
  for (int c = tid; c < K; c += blockDim.x) {     // B^T r, rows walked in a column-skewed order
    double a0 = 0.0, a1 = 0.0;
    int rr = c % M;
    for (int t = 0; t < M; ++t) {
      const double v = B[c * ld + rr] * sc.r[rr];
      if (t & 1) a1 += v; else a0 += v;
      if (++rr == M) rr = 0;
    }
    sc.c[c] = a0 + a1;
  }
  __syncthreads();
  if (warp == 0) {
    csne_forward(G, sc.dinv, sc.c, K);
    csne_backward(G, sc.dinv, sc.c, K);
    double ds = 0.0, ss = 0.0;
    for (int j = lane; j < K; j += 32) {
      ds += sc.c[j] * sc.c[j];
      ss += s[j] * s[j];
    }
    ds = warp_sum(ds);
    ss = warp_sum(ss);
    const bool ok = isfinite(ds) && ds <= kCsneStep * kCsneStep * ss;
    for (int j = lane; j < K; j += 32) s[j] += sc.c[j];
    if (lane == 0) sc.flag[0] = ok;
  }
  __syncthreads();
  HCS_MARKP(ph, 6);
  return sc.flag[0];
}

}  // namespace hcs
