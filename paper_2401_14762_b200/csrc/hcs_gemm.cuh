// hcs_gemm.cuh -- FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) tile GEMM used
// by the batched shared-basis solvers.
//
// One CTA owns a tile of kSlots = 32 pixel columns.  A GEMM computes
//     Out[n, s] = sum_k Mat[n, k] * In[k, s],   n, k < Np (N padded to 16)
// where Mat is Psi or Psi^T (N x N, shared by every pixel, L2-resident) and
// In is the CTA's 32 pixel vectors held in shared memory.  Warp w owns output
// one or two 8-row blocks for all 32 columns (warp_rows): up to 2 x 4 DMMA
// 8x8 accumulators.
//
// Mat is pre-arranged once per call ("fragment order") so that each warp's A
// fragments for one k-step are one coalesced load (see tile_gemm).
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

// Element coordinates of accumulator acc[rb][cb][i] held by `lane` of warp w
// (16-row warp tiles; used by the PSNR kernel).
__device__ __forceinline__ int acc_row(int w, int rb, int lane) { return 16 * w + 8 * rb + (lane >> 2); }
__device__ __forceinline__ int acc_col(int cb, int i, int lane) { return 8 * cb + 2 * (lane & 3) + i; }

// Out = Mat * In for a 32-column tile with 2 N_pad threads: warp w owns rows
// 16 w .. 16 w + 15 (two 8-row blocks, acc[rb][cb][i] at acc_row / acc_col).
// Mat[r][c] = basis[r N + c] (trans = false: Psi) or basis[c N + r] (trans =
// true: Psi^T), A fragments straight from the L2-resident row-major basis,
// prefetched 4 k-steps ahead (the streaming kernels: PSNR, sparsify/measure).
__device__ __forceinline__ void basis_tile_gemm(const double* __restrict__ basis, int N, int KS, bool trans,
                                                const double* In, double (&acc)[2][4][2]) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int rb = 0; rb < 2; ++rb)
#pragma unroll
    for (int cb = 0; cb < 4; ++cb) acc[rb][cb][0] = acc[rb][cb][1] = 0.0;
  const int r0 = 16 * w + (lane >> 2), r1 = r0 + 8;
  const bool v0 = r0 < N, v1 = r1 < N;
  const size_t st = trans ? (size_t)N : 1;                  // stride along k
  const double* p0 = basis + (trans ? (size_t)r0 : (size_t)r0 * N);
  const double* p1 = basis + (trans ? (size_t)r1 : (size_t)r1 * N);
  double a0[4], a1[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = 4 * i + (lane & 3);
    a0[i] = (v0 && c < N) ? __ldg(p0 + c * st) : 0.0;
    a1[i] = (v1 && c < N) ? __ldg(p1 + c * st) : 0.0;
  }
  for (int ks0 = 0; ks0 < KS; ks0 += 4) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double* b = In + ((ks0 + i) << 7) + lane;
      const double b0 = b[0], b1 = b[32], b2 = b[64], b3 = b[96];
      dmma(acc[0][0], a0[i], b0);
      dmma(acc[1][0], a1[i], b0);
      dmma(acc[0][1], a0[i], b1);
      dmma(acc[1][1], a1[i], b1);
      dmma(acc[0][2], a0[i], b2);
      dmma(acc[1][2], a1[i], b2);
      dmma(acc[0][3], a0[i], b3);
      dmma(acc[1][3], a1[i], b3);
      const int c = 4 * (ks0 + 4 + i) + (lane & 3);          // k-step ks0 + i + 4
      a0[i] = (v0 && c < N) ? __ldg(p0 + c * st) : 0.0;
      a1[i] = (v1 && c < N) ? __ldg(p1 + c * st) : 0.0;
    }
  }
}

// Balanced row-block map of the slot engine.  RB = Np / 8 row blocks of 8
// rows over min(RB, 16) warps: the first nd = RB - 16 warps own two blocks,
// the rest one.  The DMMA pipe is per SM sub-partition (warp w runs on
// sub-partition w % 4), so this spreads the blocks evenly: RB = 28 (N = 224)
// puts exactly 7 blocks on every sub-partition, where 14 warps of 16 rows
// would load two sub-partitions with 4 warps and two with 3 (87.5% cap).
__device__ __forceinline__ void warp_rows(int RB, int w, int& rb0, int& nrb) {
  const int nd = RB > 16 ? RB - 16 : 0;
  if (w < nd) { rb0 = 2 * w; nrb = 2; } else { rb0 = nd + w; nrb = 1; }
}
__host__ __device__ __forceinline__ int engine_warps(int Np) { return (Np >> 3) < 16 ? (Np >> 3) : 16; }

// A fragments of the first k-steps, loaded ahead of the GEMM (before the
// barrier that precedes it) so that their L2 latency is off the critical path.
// Two-block warps: a[i] = k-step i (both blocks); one-block warps:
// a[i].x = k-step i, a[i].y = k-step i + 4.
template <int NRB>
__device__ __forceinline__ void gemm_preload(const double* __restrict__ frag, int rb0, int KS, double2 (&a)[4]) {
  const int lane = threadIdx.x & 31;
  if (NRB == 2) {
    const double2* fa = reinterpret_cast<const double2*>(frag + (size_t)rb0 * KS * 32) + lane;
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = __ldg(fa + i * 32);
  } else {
    const double* fa = frag + (size_t)rb0 * KS * 32 + lane;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      a[i].x = __ldg(fa + i * 32);
      a[i].y = 4 + i < KS ? __ldg(fa + (4 + i) * 32) : 0.0;
    }
  }
}
__device__ __forceinline__ void gemm_preload(int nrb, const double* frag, int rb0, int KS, double2 (&a)[4]) {
  if (nrb == 2) gemm_preload<2>(frag, rb0, KS, a); else gemm_preload<1>(frag, rb0, KS, a);
}

// acc = Mat(row blocks rb0 .. rb0 + NRB - 1) * In.  KS = Np / 4 (a multiple of
// 4).  frag is the fragment-order matrix of prep_basis_kernel: the A
// fragments of row block rb start at double offset rb * KS * 32; a two-block
// warp's pair is interleaved (one 16-byte load per lane and k-step).  a holds
// the gemm_preload fragments on entry (consumed).
template <int NRB>
__device__ __forceinline__ void tile_gemm(const double* __restrict__ frag, int rb0, const double* In, int KS,
                                          double (&acc)[2][4][2], double2 (&a)[4]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int rb = 0; rb < NRB; ++rb)
#pragma unroll
    for (int cb = 0; cb < 4; ++cb) acc[rb][cb][0] = acc[rb][cb][1] = 0.0;
  if (NRB == 2) {
    const double2* fa = reinterpret_cast<const double2*>(frag + (size_t)rb0 * KS * 32) + lane;
    // a[i] is reloaded (4 k-steps ahead) right after its last use: prefetch
    // distance 4 at 16 registers
    for (int ks0 = 0; ks0 < KS; ks0 += 4) {
      const bool more = ks0 + 4 < KS;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double* b = In + ((ks0 + i) << 7) + lane;
        const double b0 = b[0], b1 = b[32], b2 = b[64], b3 = b[96];
        dmma(acc[0][0], a[i].x, b0);
        dmma(acc[1][0], a[i].y, b0);
        dmma(acc[0][1], a[i].x, b1);
        dmma(acc[1][1], a[i].y, b1);
        dmma(acc[0][2], a[i].x, b2);
        dmma(acc[1][2], a[i].y, b2);
        dmma(acc[0][3], a[i].x, b3);
        dmma(acc[1][3], a[i].y, b3);
        if (more) a[i] = __ldg(fa + (ks0 + 4 + i) * 32);
      }
    }
  } else {
    const double* fa = frag + (size_t)rb0 * KS * 32 + lane;
    // two 4-step halves: prefetch distance 8 k-steps (half the DMMAs per step)
    for (int ks0 = 0; ks0 < KS; ks0 += 8) {
      const bool more0 = ks0 + 8 < KS, more1 = ks0 + 12 < KS;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double* b = In + ((ks0 + i) << 7) + lane;
        dmma(acc[0][0], a[i].x, b[0]);
        dmma(acc[0][1], a[i].x, b[32]);
        dmma(acc[0][2], a[i].x, b[64]);
        dmma(acc[0][3], a[i].x, b[96]);
        if (more0) a[i].x = __ldg(fa + (ks0 + 8 + i) * 32);
      }
      if (ks0 + 4 >= KS) break;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double* b = In + ((ks0 + 4 + i) << 7) + lane;
        dmma(acc[0][0], a[i].y, b[0]);
        dmma(acc[0][1], a[i].y, b[32]);
        dmma(acc[0][2], a[i].y, b[64]);
        dmma(acc[0][3], a[i].y, b[96]);
        if (more1) a[i].y = __ldg(fa + (ks0 + 12 + i) * 32);
      }
    }
  }
}
__device__ __forceinline__ void tile_gemm(int nrb, const double* frag, int rb0, const double* In, int KS,
                                          double (&acc)[2][4][2], double2 (&a)[4]) {
  if (nrb == 2) tile_gemm<2>(frag, rb0, In, KS, acc, a); else tile_gemm<1>(frag, rb0, In, KS, acc, a);
}

// ---------------------------------------------------------------------------
// A fragments through a per-warp shared-memory ring (cp.async, kRing k-steps
// deep).  With the fragments loaded straight into registers (tile_gemm) ptxas
// puts every in-flight __ldg of the loop on one scoreboard, so the wait for the
// oldest fragment also waits for the youngest: the 4-k-step prefetch distance
// collapses to ~0 and a quarter of the GEMM's stall samples are long-scoreboard
// waits (profiles/ncu_admm_ring_r02.txt).  cp.async groups are counted
// (cp.async.wait_group kRing - 1 = DEPBAR.LE), so the ring really runs kRing - 1
// k-steps ahead of the DMMAs.  Each lane copies and reads back only its own
// 8 NRB bytes per k-step: no cross-lane synchronisation.  Stage st of a warp's
// ring is at byte st * 256 * NRB; the warp's ring base is ring_offset().
constexpr int kRing = 4;

// bytes of all rings of a 32-slot CTA / byte offset of warp w's ring
__host__ __device__ __forceinline__ int ring_bytes(int Np) {
  const int RB = Np >> 3, W = RB < 16 ? RB : 16, nd = RB > 16 ? RB - 16 : 0;
  return kRing * 256 * (2 * nd + (W - nd));
}
__device__ __forceinline__ int ring_offset(int RB, int w) {
  const int nd = RB > 16 ? RB - 16 : 0;
  return kRing * 256 * (w < nd ? 2 * w : nd + w);
}

template <int NRB>
__device__ __forceinline__ void ring_copy(unsigned dst, const double* src) {
  if (NRB == 2) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src));
}
// the same copy, ordered after the register `dep` is available (the ring
// stage's last read has landed before the stage is overwritten)
template <int NRB>
__device__ __forceinline__ void ring_copy_after(unsigned dst, const double* src, double dep) {
  if (NRB == 2) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src), "d"(dep));
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src), "d"(dep));
}
__device__ __forceinline__ void ring_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void ring_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
template <int NRB>
__device__ __forceinline__ double2 ring_read(unsigned src) {
  double2 v;
  if (NRB == 2) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(src));
  } else {
    asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v.x) : "r"(src));
    v.y = 0.0;
  }
  return v;
}

// first kRing k-steps of the next GEMM into the ring (issued before the barrier
// that precedes the GEMM); ring = shared-space byte address of this lane's
// slot in stage 0
template <int NRB>
__device__ __forceinline__ void ring_preload(const double* __restrict__ frag, int rb0, int KS, unsigned ring) {
  const int lane = threadIdx.x & 31;
  const double* src = frag + (size_t)rb0 * KS * 32 + lane * NRB;
#pragma unroll
  for (int st = 0; st < kRing; ++st) {
    ring_copy<NRB>(ring + st * 256 * NRB, src + (size_t)st * 32 * NRB);
    ring_commit();
  }
}

// acc = Mat(row blocks rb0 .. rb0 + NRB - 1) * In with the A fragments from the
// ring (ring_preload done).  KS is a multiple of 4 = kRing.  Same DMMA order
// per accumulator as tile_gemm: bitwise-identical results.
template <int NRB>
__device__ __forceinline__ void tile_gemm_ring(const double* __restrict__ frag, int rb0, const double* In, int KS,
                                               double (&acc)[2][4][2], unsigned ring) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int rb = 0; rb < NRB; ++rb)
#pragma unroll
    for (int cb = 0; cb < 4; ++cb) acc[rb][cb][0] = acc[rb][cb][1] = 0.0;
  const double* src = frag + (size_t)rb0 * KS * 32 + lane * NRB;
  ring_wait<kRing - 1>();
  double2 a = ring_read<NRB>(ring);
  for (int ks0 = 0; ks0 < KS; ks0 += kRing) {
#pragma unroll
    for (int i = 0; i < kRing; ++i) {
      const int ks = ks0 + i;
      const double* b = In + (ks << 7) + lane;
      const double b0 = b[0], b1 = b[32], b2 = b[64], b3 = b[96];
      dmma(acc[0][0], a.x, b0);
      if (NRB == 2) dmma(acc[1][0], a.y, b0);
      // stage i is in registers: refill it with k-step ks + kRing, then fetch
      // the next k-step's fragment (complete once <= kRing - 1 groups pend)
      if (ks + kRing < KS) ring_copy_after<NRB>(ring + i * 256 * NRB, src + (size_t)(ks + kRing) * 32 * NRB, a.x);
      ring_commit();
      ring_wait<kRing - 1>();
      double2 an = a;
      if (ks + 1 < KS) an = ring_read<NRB>(ring + ((i + 1) % kRing) * 256 * NRB);
      dmma(acc[0][1], a.x, b1);
      if (NRB == 2) dmma(acc[1][1], a.y, b1);
      dmma(acc[0][2], a.x, b2);
      if (NRB == 2) dmma(acc[1][2], a.y, b2);
      dmma(acc[0][3], a.x, b3);
      if (NRB == 2) dmma(acc[1][3], a.y, b3);
      a = an;
    }
  }
}

// Column sums of an accumulator-layout quantity: v[2 cb + i] is this lane's
// value for slot column 8 cb + 2 (lane & 3) + i (already summed over its row
// blocks).  Three transpose-and-add butterfly stages over the 8 lanes sharing
// a column (lane bits 2..4) leave each lane with the full 8-row sum of one
// column, col_of_reduced(lane): 7 double shuffles instead of 24.
__device__ __forceinline__ double col_reduce8(const double (&v)[8], int lane) {
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
__device__ __forceinline__ int col_of_reduced(int lane) {
  return 8 * (2 * ((lane >> 2) & 1) + ((lane >> 3) & 1)) + 2 * (lane & 3) + ((lane >> 4) & 1);
}


// acc = Mat(row blocks rb0 ..) * In over the k-steps set in kmask only (bit ks:
// rows 4 ks .. 4 ks + 3 of In are nonzero in some column).  The skipped
// k-steps multiply exact zeros, so the result is bitwise that of tile_gemm
// (products a * 0 are +-0 and leave every partial sum unchanged).  A fragments
// are loaded two active k-steps ahead.  FISTA's second GEMM (Psi x_{k+1}):
// x_{k+1} is soft-thresholded, and the converged supports of the benchmark
// cubes sit in the lowest 16 coefficients (12% of the k-steps are active per
// 32-pixel group, tools/support_stats.py).
template <int NRB>
__device__ __forceinline__ void tile_gemm_masked(const double* __restrict__ frag, int rb0, const double* In, int KS,
                                                 unsigned long long kmask, double (&acc)[2][4][2]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int rb = 0; rb < NRB; ++rb)
#pragma unroll
    for (int cb = 0; cb < 4; ++cb) acc[rb][cb][0] = acc[rb][cb][1] = 0.0;
  auto next = [&](unsigned long long& m) -> int {
    if (!m) return -1;
    const int ks = __ffsll((long long)m) - 1;
    m &= m - 1;
    return ks;
  };
  auto load = [&](int ks) -> double2 {
    double2 v = make_double2(0.0, 0.0);
    if (ks < 0) return v;
    if (NRB == 2) {
      v = __ldg(reinterpret_cast<const double2*>(frag + (size_t)rb0 * KS * 32) + lane + ks * 32);
    } else {
      v.x = __ldg(frag + (size_t)rb0 * KS * 32 + lane + ks * 32);
    }
    return v;
  };
  unsigned long long m = kmask;
  int k0 = next(m), k1 = next(m);
  double2 a0 = load(k0), a1 = load(k1);
  while (k0 >= 0) {
    const int k2 = next(m);
    const double2 a2 = load(k2);
    const double* b = In + (k0 << 7) + lane;
    const double b0 = b[0], b1 = b[32], b2 = b[64], b3 = b[96];
    dmma(acc[0][0], a0.x, b0);
    dmma(acc[0][1], a0.x, b1);
    dmma(acc[0][2], a0.x, b2);
    dmma(acc[0][3], a0.x, b3);
    if (NRB == 2) {
      dmma(acc[1][0], a0.y, b0);
      dmma(acc[1][1], a0.y, b1);
      dmma(acc[1][2], a0.y, b2);
      dmma(acc[1][3], a0.y, b3);
    }
    k0 = k1;
    a0 = a1;
    k1 = k2;
    a1 = a2;
  }
}
__device__ __forceinline__ void tile_gemm_masked(int nrb, const double* frag, int rb0, const double* In, int KS,
                                                 unsigned long long kmask, double (&acc)[2][4][2]) {
  if (nrb == 2) tile_gemm_masked<2>(frag, rb0, In, KS, kmask, acc);
  else tile_gemm_masked<1>(frag, rb0, In, KS, kmask, acc);
}

// ---------------------------------------------------------------------------
// Half-width engine (two CTAs per SM, 16 slots, 8 warps): the same GEMM with
// CB = 2 column blocks and up to 4 row blocks per warp, so that the two CTAs
// of an SM run out of phase and one CTA's epilogue / slot phase overlaps the
// other's DMMA work.  The matrix is read in the plain fragment order (row
// block rb, k-step ks at (rb KS + ks) * 32, prep_basis with interleave off);
// In holds 16 columns: in_idx16.
constexpr int kSlots16 = 16;

__device__ __forceinline__ int in_idx16(int k, int s) {
  return (((k >> 2) * 2 + (s >> 3)) << 5) + ((s & 7) << 2) + (k & 3);
}

// Contiguous balanced row-block map over W warps: warps w < RB % W own one
// more block.  With W = 8 the warp pairs (w, w + 4) share an SM sub-partition,
// so N = 224 (RB = 28) puts 4 + 3 = 7 blocks on each.
__device__ __forceinline__ void warp_rows16(int RB, int W, int w, int& rb0, int& nrb) {
  const int base = RB / W, extra = RB % W;
  nrb = base + (w < extra ? 1 : 0);
  rb0 = w * base + (w < extra ? w : extra);
}
__host__ __device__ __forceinline__ int engine_warps16(int Np) { return (Np >> 3) < 8 ? (Np >> 3) : 8; }

template <int NRB>
__device__ __forceinline__ void gemm_preload16(const double* __restrict__ frag, int rb0, int KS, double (&a)[4][4]) {
  const double* fa = frag + (size_t)rb0 * KS * 32 + (threadIdx.x & 31);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int rb = 0; rb < NRB; ++rb) a[i][rb] = __ldg(fa + ((size_t)rb * KS + i) * 32);
}
__device__ __forceinline__ void gemm_preload16(int nrb, const double* frag, int rb0, int KS, double (&a)[4][4]) {
  switch (nrb) {
    case 4: gemm_preload16<4>(frag, rb0, KS, a); break;
    case 3: gemm_preload16<3>(frag, rb0, KS, a); break;
    case 2: gemm_preload16<2>(frag, rb0, KS, a); break;
    default: gemm_preload16<1>(frag, rb0, KS, a); break;
  }
}

// acc[rb][cb] = Mat(row block rb0 + rb) * In(column block cb), rb < NRB, cb < 2;
// a holds the gemm_preload16 fragments (k-steps 0..3) on entry; each is
// reloaded 4 k-steps ahead right after its last use.
template <int NRB>
__device__ __forceinline__ void tile_gemm16(const double* __restrict__ frag, int rb0, const double* In, int KS,
                                            double (&acc)[4][2][2], double (&a)[4][4]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int rb = 0; rb < NRB; ++rb)
#pragma unroll
    for (int cb = 0; cb < 2; ++cb) acc[rb][cb][0] = acc[rb][cb][1] = 0.0;
  const double* fa = frag + (size_t)rb0 * KS * 32 + lane;
  for (int ks0 = 0; ks0 < KS; ks0 += 4) {
    const bool more = ks0 + 4 < KS;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double* b = In + ((ks0 + i) << 6) + lane;
      const double b0 = b[0], b1 = b[32];
#pragma unroll
      for (int rb = 0; rb < NRB; ++rb) {
        dmma(acc[rb][0], a[i][rb], b0);
        dmma(acc[rb][1], a[i][rb], b1);
      }
      if (more) {
#pragma unroll
        for (int rb = 0; rb < NRB; ++rb) a[i][rb] = __ldg(fa + ((size_t)rb * KS + ks0 + 4 + i) * 32);
      }
    }
  }
}
__device__ __forceinline__ void tile_gemm16(int nrb, const double* frag, int rb0, const double* In, int KS,
                                            double (&acc)[4][2][2], double (&a)[4][4]) {
  switch (nrb) {
    case 4: tile_gemm16<4>(frag, rb0, In, KS, acc, a); break;
    case 3: tile_gemm16<3>(frag, rb0, In, KS, acc, a); break;
    case 2: tile_gemm16<2>(frag, rb0, In, KS, acc, a); break;
    default: tile_gemm16<1>(frag, rb0, In, KS, acc, a); break;
  }
}

// Column sums for 16 slot columns: v[2 cb + i] is this lane's value for
// column 8 cb + 2 (lane & 3) + i.  Two transpose-and-add stages (lane bits 2,
// 3) and one plain stage (bit 4) leave the full 8-row sum of column
// col_of_reduced4(lane) in this lane (lanes l and l ^ 16 hold the same column).
__device__ __forceinline__ double col_reduce4(const double (&v)[4], int lane) {
  const bool b = (lane >> 2) & 1, c = (lane >> 3) & 1;
  double u[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double send = b ? v[k] : v[k + 2], keep = b ? v[k + 2] : v[k];
    u[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  const double send = c ? u[0] : u[1], keep = c ? u[1] : u[0];
  double q = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  return q + __shfl_xor_sync(0xffffffffu, q, 16);
}
__device__ __forceinline__ int col_of_reduced4(int lane) {
  return 8 * ((lane >> 2) & 1) + 2 * (lane & 3) + ((lane >> 3) & 1);
}

}  // namespace hcs
