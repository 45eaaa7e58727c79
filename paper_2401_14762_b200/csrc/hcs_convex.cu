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
#include <cstdlib>
#include <type_traits>

namespace hcs {

// slot states: kEmpty (to be refilled in the next slot phase), kActive, kDead
// (queue exhausted: never refilled again)
enum { kEmpty = 0, kActive = 1, kDead = 3 };

#ifdef HCS_PHASES
__device__ unsigned long long g_phase_cx[16];
#endif
// debug builds (-DHCS_TRACE): per-warp clock64 at the marks of ticks 200..203 of CTA 0
#ifdef HCS_TRACE
__device__ long long g_trace[4][16][12];
#define TMARK(k) do { if (blockIdx.x == 0 && tick >= 200 && tick < 204 && lane == 0) g_trace[tick - 200][w][k] = clock64(); } while (0)
#else
#define TMARK(k) do {} while (0)
#endif

template <int SL>
struct SlotState {
  long long pid[SL];
  long long rpid[SL];
  long long start[SL];
  long long npid[SL];     // staged next pixel of the slot (>= P: none)
  double slip[SL];        // its Lipschitz constant (fista)
  double t[SL], tn[SL], betan[SL];
  double inv_l[SL], thr[SL];
  int status[SL], iter[SL], flag[SL], rfail[SL], retired[SL], moff[SL], need_pf[SL];
  int nact[2];
  // per tick parity: slots whose pixel retired / slots refilled or emptied in
  // this tick's slot phase (their columns' iterates restart from zero)
  unsigned retmask[2], freshmask[2];
  int exhausted;
  long long np;           // pixels in the queue (P, or *plist_n)
  unsigned long long kmask[2];   // fista, per tick parity: k-steps of x_{k+1} with a nonzero in some slot
};

// Slot-column layout of the GEMM input buffers: 32 slots (one CTA per SM) or 16
// (two CTAs per SM, hcs_gemm.cuh)
template <int SL>
__device__ __forceinline__ int slot_idx(int k, int s) {
  if constexpr (SL == 32) return in_idx(k, s); else return in_idx16(k, s);
}

__host__ __device__ __forceinline__ int stage_mask_bytes(int M) { return ((M + 7) & ~7) + 8; }

// Row -> measurement map in thread order.  Thread (w, lane) of the engine owns
// the accumulator elements acc[rb][cb][i] = (row 8 (rb0 + rb) + lane / 4,
// slot 8 cb + 2 (lane % 4) + i); their 16 map entries (0xFF: row not measured)
// are the 16 bytes at pos + 16 (32 w + lane), entry (2 cb + i) MAXRB + rb, so an
// epilogue gets all of them with one 16-byte shared load per tick instead of a
// dependent byte load per element.  pos_addr is the inverse of warp_rows /
// warp_rows16 for element (row n, slot s); RB = Np / 8, W = engine warps.
template <int SL>
__device__ __forceinline__ int pos_addr(int RB, int W, int n, int s) {
  constexpr int MAXRB = (SL == 32) ? 2 : 4;
  const int g = n >> 3;
  int w, rbl;
  if constexpr (SL == 32) {
    const int nd = RB > 16 ? RB - 16 : 0;
    if (g < 2 * nd) { w = g >> 1; rbl = g & 1; } else { w = g - nd; rbl = 0; }
  } else {
    const int base = RB / W, extra = RB % W, cut = extra * (base + 1);
    if (g < cut) { w = g / (base + 1); rbl = g - w * (base + 1); }
    else { const int q = (g - cut) / base; w = extra + q; rbl = (g - cut) - q * base; }
  }
  const int ln = ((n & 7) << 2) + ((s & 7) >> 1);
  return (((w << 5) + ln) << 4) + ((s >> 3) * 2 + (s & 1)) * MAXRB + rbl;
}
// entry e of the 16 map bytes a thread loaded as one uint4
__device__ __forceinline__ int pos_entry(const uint4& pw, int e) {
  const unsigned v = e < 4 ? pw.x : e < 8 ? pw.y : e < 12 ? pw.z : pw.w;
  return (int)((v >> (8 * (e & 3))) & 0xFFu);
}

// Claim the slot's next pixel from the work queue and start copying its
// measurements, mask row and (fista) Lipschitz constant into the slot's
// staging area with cp.async: the refill that consumes it, usually many ticks
// later, finds the data in shared memory instead of waiting on HBM.  Called
// by the owning warp (cp.async completion is per thread).
template <int ALGO, int SL>
__device__ void prefetch_slot(const ConvexArgs& a, SlotState<SL>& ss, double* sy, uint8_t* sm, int s) {
  const int lane = threadIdx.x & 31;
  const int M = a.M, Mm = stage_mask_bytes(M);
  long long pid = 0;
  if (lane == 0) {
    const long long q = ss.exhausted ? ss.np : (long long)atomicAdd(a.counter, 1ull);
    if (q >= ss.np) {
      ss.exhausted = 1;
      pid = a.P;                       // none
    } else {
      pid = a.plist ? a.plist[q] : q;
    }
    ss.npid[s] = pid;
  }
  pid = __shfl_sync(0xffffffffu, pid, 0);
  if (pid >= a.P) return;
  for (int j = lane; j < M; j += 32) cp_async8(sy + s * M + j, a.y + pid * M + j);
  // mask row: the 8-byte aligned chunks covering it (plain loads when the
  // chunks would leave the array or the base is misaligned)
  const unsigned long long b0 = (unsigned long long)pid * M, a0 = b0 & ~7ull;
  int moff = (int)(b0 - a0);
  const int nch = (moff + M + 7) >> 3;
  if ((reinterpret_cast<uintptr_t>(a.mask) & 7) == 0 && a0 + 8ull * nch <= (unsigned long long)a.P * M) {
    for (int c = lane; c < nch; c += 32) cp_async8b(sm + s * Mm + 8 * c, a.mask + a0 + 8 * c);
  } else {
    for (int j = lane; j < M; j += 32) sm[s * Mm + j] = a.mask[b0 + j];
    moff = 0;
  }
  if (lane == 0) {
    if (ALGO == kFista) cp_async8(&ss.slip[s], a.lip + pid);
    ss.moff[s] = moff;
  }
}

// Take the slot's staged pixel (zero pixels retire on the spot,
// solvers.py:169-170 / 212-213) and set the slot up: measurements, residual
// r = y, the row -> measurement map pos, and the slot's column of the first
// GEMM's input (fista: g = A z - y = -y at the measured rows; admm: z - w = 0);
// the next pixel is staged right after the slot phase (need_pf), where the
// queue atomic's round trip overlaps the other warps' GEMM work.  Called by
// the owning warp.
template <int ALGO, int SL>
__device__ void refill_slot(const ConvexArgs& a, SlotState<SL>& ss, double* bufA, double* bufB, double* ys, double* r,
                            uint8_t* pos, double* sy, uint8_t* sm, int s) {
  const int lane = threadIdx.x & 31;
  const int M = a.M, N = a.N, Np = a.Np, Mm = stage_mask_bytes(M);
  const int RB = Np >> 3, W = blockDim.x >> 5;
  for (int n = lane; n < Np; n += 32) {
    bufA[slot_idx<SL>(n, s)] = 0.0;
    bufB[slot_idx<SL>(n, s)] = 0.0;   // fista: z_0 = 0; admm: u'_0 = 0 (r_0 = y - u'_0[mask] = y)
  }
  for (;;) {
    cp_async_wait_all();
    __syncwarp();
    const long long pid = ss.npid[s];
    if (pid >= a.P) {
      if (lane == 0) ss.status[s] = kDead;
      for (int n = lane; n < Np; n += 32) pos[pos_addr<SL>(RB, W, n, s)] = 0xFF;
      __syncwarp();
      return;
    }
    bool nz = false, bad = false;
    for (int j = lane; j < M; j += 32) {
      const double v = sy[s * M + j];
      ys[s * M + j] = v;
      if (ALGO == kFista) r[s * M + j] = v;
      nz |= (v != 0.0);
      bad |= !isfinite(v);
    }
    nz = __any_sync(0xffffffffu, nz);
    bad = __any_sync(0xffffffffu, bad);
    const double lip = (ALGO == kFista) ? ss.slip[s] : 0.0;
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
      __syncwarp();
      prefetch_slot<ALGO, SL>(a, ss, sy, sm, s);
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
      __syncwarp();
      prefetch_slot<ALGO, SL>(a, ss, sy, sm, s);
      continue;
    }
    for (int n = lane; n < Np; n += 32) pos[pos_addr<SL>(RB, W, n, s)] = 0xFF;
    __syncwarp();
    const uint8_t* mrow = sm + s * Mm + ss.moff[s];
    for (int j = lane; j < M; j += 32) {
      const int row = mrow[j];
      pos[pos_addr<SL>(RB, W, row, s)] = (uint8_t)j;
      if (ALGO == kFista) bufA[slot_idx<SL>(row, s)] = -ys[s * M + j];
    }
    if (lane == 0) {
      ss.pid[s] = pid;
      ss.start[s] = t0;
      ss.status[s] = kActive;
      ss.iter[s] = 0;
      ss.t[s] = 1.0;
      if (ALGO == kFista) {
        ss.inv_l[s] = 1.0 / lip;
        ss.thr[s] = __dmul_rn(a.prm.lam, ss.inv_l[s]);
      } else {
        ss.thr[s] = a.prm.lam / a.prm.alpha;
      }
    }
    if (lane == 0) ss.need_pf[s] = 1;   // staged after the barrier, off the slot phase
    __syncwarp();
    return;
  }
}

// Stop rule after an iteration (solvers.py:115-127 evaluated before the next
// pass) plus the non-finite check (solvers.py:155-157).  Lane 0 of the owner.
template <int SL>
__device__ __forceinline__ void finish_iteration(const ConvexArgs& a, SlotState<SL>& ss, int s, double delta,
                                                 bool admm, double gap2) {
  int it = ss.iter[s] + 1;
  ss.iter[s] = it;
  const bool failed = ss.flag[s] || !isfinite(delta);
  const int dec = failed ? kContinue : stop_decision(delta, it, ss.start[s], a.prm);
  const bool conv = dec == kConverged;
  if (failed || dec != kContinue) {
    long long pid = ss.pid[s];
    ss.status[s] = kEmpty;
    ss.retired[s] = 1;
    ss.rpid[s] = pid;
    ss.rfail[s] = failed;
    a.st.iterations[pid] = failed ? 0 : it;
    a.st.converged[pid] = conv ? 1 : 0;
    a.st.final_delta[pid] = failed ? __longlong_as_double(0x7ff8000000000000ll) : delta;
    a.st.failed_at[pid] = failed ? it : -1;
    if (admm && a.st.admm_gap)
      a.st.admm_gap[pid] = failed ? __longlong_as_double(0x7ff8000000000000ll) : sqrt(gap2);
    if (a.st.elapsed) a.st.elapsed[pid] = 1e-9 * (double)(now_ns() - ss.start[s]);
    if (a.st.work) a.st.work[pid] = 4.0 * (double)a.N * (double)a.N * (double)it;
  }
}

// One tick = one solver iteration of all SL slots:
//   slot phase: stop rule on the partial sums by one warp, a lane per slot | barrier
//     refills by the slots' owner warps (only in ticks that refill)       | barrier
//   (fista: results of retired slots;) GEMM 1 (reads A); epilogue 1 (writes B) | barrier
//   GEMM 2 (reads B); epilogue 2 (writes A for the next tick)             | barrier
// (admm: A = z - w, B = u'; each buffer is written only after every warp is
// done reading it, so no barrier sits between a GEMM and its epilogue.
// fista: A holds g, then x_{k+1}, then the next g, B holds z, two more
// barriers.)  Per-element iterates stay in registers in the accumulator
// layout: fista p0 = x_k; admm p1 = w (z goes to x_out every pass).
// Residual-delta and ADMM-gap sums are reduced per warp (col_reduce) into
// part[], summed in a fixed tree order by the slot warp: deterministic.
// SL = 32: one CTA per SM, up to 16 warps of 1-2 row blocks x 4 column blocks
// (<= 128 registers).  SL = 16: two CTAs per SM of 8 warps, up to 4 row blocks
// x 2 column blocks each; the two CTAs drift out of phase so that one's
// epilogues and slot phase overlap the other's GEMMs on the DMMA pipe.
// RING: A fragments through the per-warp cp.async ring of hcs_gemm.cuh (32-slot
// engine, when the ring fits in shared memory) instead of register prefetch.
template <int ALGO, int SL, int MAXT, int MINB, int RING>
__global__ void __launch_bounds__(MAXT, MINB) convex_kernel(ConvexArgs a) {
  if (*(volatile const int*)a.err & kErrMask) return;   // invalid masks (validate_masks_kernel)
  constexpr int CB = SL / 8;                  // 8-column blocks
  constexpr int MAXRB = (SL == 32) ? 2 : 4;   // row blocks per warp
  constexpr int NV = 2 * CB;                  // per-lane column partials
  extern __shared__ __align__(16) unsigned char smraw[];
  hcs_smem_poison(smraw, a.smem_bytes);
  const int Np = a.Np, M = a.M, N = a.N, KS = Np >> 2;
  const int W = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int rb0, nrb;
  if constexpr (SL == 32) warp_rows(Np >> 3, w, rb0, nrb); else warp_rows16(Np >> 3, W, w, rb0, nrb);
  const int row0 = 8 * rb0 + (lane >> 2);   // element row of acc[rb] is row0 + 8 rb
  // buffer index of this thread's element acc[rb][cb][i]: one base plus
  // compile-time offsets (slot_idx of row row0 + 8 rb, slot 8 cb + 2 (lane & 3) + i)
  const int ebase = slot_idx<SL>(row0, 2 * (lane & 3));
  auto eidx = [&](int rb, int cb, int i) { return ebase + rb * (2 * (SL / 8) * 32) + cb * 32 + i * 4; };
  double* bufA = reinterpret_cast<double*>(smraw);      // Np * SL: fista g / x_{k+1}, admm z - w
  double* bufB = bufA + Np * SL;                        // Np * SL: fista z, admm u'
  double* ys = bufB + Np * SL;                          // SL * M
  double* r = ys + SL * M;                              // SL * M (fista; admm's is y - u'[mask], in bufB)
  const double* ysq = ys + 2 * (lane & 3) * M;          // measurements of slot 2 (lane & 3); slot 8 cb + i: (8 cb + i) M further
  double* partD = r + (ALGO == kFista ? SL * M : 0);    // 16 * SL residual-delta partials
  double* partG = partD + 16 * SL;                      // 16 * SL admm gap partials (admm)
  double* sy = partG + (ALGO == kAdmm ? 16 * SL : 0);   // SL * M staged next measurements
  SlotState<SL>& ss = *reinterpret_cast<SlotState<SL>*>(sy + SL * M);
  // SL * 256: row -> measurement index in thread order (pos_addr), 16-byte aligned
  uint8_t* pos = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(&ss + 1) + 15) & ~(uintptr_t)15);
  uint8_t* sm = pos + SL * kMaxN;                       // SL * stage_mask_bytes(M) staged mask rows
  // this lane's slot in stage 0 of the warp's A-fragment ring (shared-space byte address)
  unsigned ring = 0;
  if constexpr (RING) {
    unsigned char* rg = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(sm + SL * stage_mask_bytes(M)) + 15) & ~(uintptr_t)15);
    ring = static_cast<unsigned>(__cvta_generic_to_shared(rg + ring_offset(Np >> 3, w))) + lane * 8 * nrb;
  }
  const int cred = (SL == 32) ? col_of_reduced(lane) : col_of_reduced4(lane);
  const bool use_kskip = (SL == 32) && ALGO == kFista && a.kskip;

  double p0[MAXRB][CB][2], p1[MAXRB][CB][2];
#pragma unroll
  for (int rb = 0; rb < MAXRB; ++rb)
#pragma unroll
    for (int cb = 0; cb < CB; ++cb)
#pragma unroll
      for (int i = 0; i < 2; ++i) p0[rb][cb][i] = p1[rb][cb][i] = 0.0;
  if (threadIdx.x < SL) {
    ss.status[threadIdx.x] = kEmpty;
    ss.retired[threadIdx.x] = 0;
    ss.need_pf[threadIdx.x] = 0;
  }
  if (threadIdx.x == 0) {
    ss.exhausted = 0;
    ss.nact[0] = ss.nact[1] = 0;
    ss.retmask[0] = ss.retmask[1] = ss.freshmask[0] = ss.freshmask[1] = 0u;
    ss.kmask[0] = ss.kmask[1] = 0ull;
    ss.np = a.plist ? (long long)*a.plist_n : a.P;
  }
  __syncthreads();
  // Slot phase: the stop rule (and fista's momentum) of all slots is run by one
  // warp with one lane per slot; refills and the staging of the next pixel stay
  // with the slot's owner warp, w + W k (cp.async completion is per thread).
  // Measured alternatives (profiles/convex_ring_r02.txt): two slots per warp
  // via half-warp shuffles (3.3k cycles per tick instead of 1.7k); all slot
  // work including refills in one warp (serialises 32 refills per tick when
  // pixels converge in one iteration); the slot phase under the other warps'
  // GEMM (its code runs 6-8x longer under DMMA contention).
  const int nown = W, ow = w;
  const bool slot_warp = w == W - 1;
  for (int s = ow; s < SL; s += nown) prefetch_slot<ALGO, SL>(a, ss, sy, sm, s);
  // GEMM 1 multiplies by Psi^T (fista) / Psi (admm), GEMM 2 by the other
  const double* mat1 = (ALGO == kFista) ? a.fragT : a.fragS;
  const double* mat2 = (ALGO == kFista) ? a.fragS : a.fragT;
  // A-fragment prefetch registers (the next GEMM's first k-steps)
  double2 af[4];
  double af16[4][4];
  auto preload = [&](const double* m) {
    if constexpr (RING) {
      if (nrb == 2) ring_preload<2>(m, rb0, KS, ring); else ring_preload<1>(m, rb0, KS, ring);
    } else if constexpr (SL == 32) {
      gemm_preload(nrb, m, rb0, KS, af);
    } else {
      gemm_preload16(nrb, m, rb0, KS, af16);
    }
  };
  double acc[MAXRB][CB][2];
  auto gemm = [&](const double* m, const double* in) {
    if constexpr (RING) {
      if (nrb == 2) tile_gemm_ring<2>(m, rb0, in, KS, acc, ring); else tile_gemm_ring<1>(m, rb0, in, KS, acc, ring);
    } else if constexpr (SL == 32) {
      tile_gemm(nrb, m, rb0, in, KS, acc, af);
    } else {
      tile_gemm16(nrb, m, rb0, in, KS, acc, af16);
    }
  };
  auto reduce = [&](const double (&v)[NV]) -> double {
    if constexpr (SL == 32) return col_reduce8(v, lane); else return col_reduce4(v, lane);
  };
  preload(mat1);

#ifdef HCS_PHASES
  long long cph[16] = {0};
  cph[15] = clock64();
#define CMARK(k) HCS_MARKP(cph, k)
#else
#define CMARK(k) do {} while (0)
#endif
  // admm: 1 / (d + alpha) for d = 0, 1 (Psi orthonormal: the factor's eigenvalues);
  // opaque to the optimiser, which otherwise rewrites x * (m ? inv1 : inv0) into
  // a division per element
  double inv0 = 1.0 / a.prm.alpha, inv1 = 1.0 / (1.0 + a.prm.alpha);
  asm volatile("" : "+d"(inv0), "+d"(inv1));
  for (int tick = 0;; ++tick) {
    const int par = tick & 1;
    TMARK(0);
    // ---- slot phase: stop rule of the last iteration, momentum, refill ----
    // one warp, one lane per slot: the partial sums in a fixed tree order,
    // masks and the active count by ballots (no atomics)
    if (slot_warp) {
      const int sl_ = lane;
      const bool valid = sl_ < SL;
      const int st0 = valid ? ss.status[sl_] : kDead;
      const bool was_active = st0 == kActive;
      double pd[16], pg[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        pd[i] = (was_active && i < W) ? partD[i * SL + sl_] : 0.0;
        pg[i] = (ALGO == kAdmm && was_active && i < W) ? partG[i * SL + sl_] : 0.0;
      }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1)
#pragma unroll
        for (int i = 0; i < o; ++i) {
          pd[i] += pd[i + o];
          if (ALGO == kAdmm) pg[i] += pg[i + o];
        }
      if (valid) {
        ss.retired[sl_] = 0;
        if (was_active) {
          if (ALGO == kFista) ss.t[sl_] = ss.tn[sl_];
          finish_iteration<SL>(a, ss, sl_, sqrt(pd[0]), ALGO == kAdmm, pg[0]);
        }
      }
      __syncwarp();
      const unsigned retb = __ballot_sync(0xffffffffu, valid && ss.retired[sl_]);
      unsigned failb = (ALGO == kAdmm) ? __ballot_sync(0xffffffffu, valid && ss.retired[sl_] && ss.rfail[sl_]) : 0u;
      while (failb) {   // NumericalFailure: x = 0
        const int sk = __ffs(failb) - 1;
        failb &= failb - 1;
        for (int n = lane; n < N; n += 32) a.x_out[ss.rpid[sk] * N + n] = 0.0;
      }
      const int st1 = valid ? ss.status[sl_] : kDead;
      const unsigned emptyb = __ballot_sync(0xffffffffu, st1 == kEmpty);
      if (valid && st1 != kEmpty) {
        if (st1 == kActive) {
          ss.flag[sl_] = 0;
          if (ALGO == kFista) {
            const double t = ss.t[sl_];
            const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));   // solvers.py:160-161
            ss.tn[sl_] = tn;
            ss.betan[sl_] = (t - 1.0) / tn;
          }
        } else {
          ss.inv_l[sl_] = 0.0;
          ss.thr[sl_] = 0.0;
          ss.betan[sl_] = 0.0;
        }
      }
      const unsigned actb = __ballot_sync(0xffffffffu, st1 == kActive);
      if (lane == 0) {
        ss.nact[par] = __popc(actb);   // the refills below add theirs
        ss.retmask[par] = retb;
        ss.freshmask[par] = emptyb;
      }
    }
    __syncthreads();
    // refills by the slots' owner warps (w + W k: the warp that staged the next
    // pixel), in parallel; the extra barrier only in ticks that refill
    if (const unsigned em = ss.freshmask[par]) {
      for (int sk = ow; sk < SL; sk += nown)
        if ((em >> sk) & 1u) {
          refill_slot<ALGO, SL>(a, ss, bufA, bufB, ys, r, pos, sy, sm, sk);
          if (lane == 0) {
            if (ss.status[sk] == kActive) {
              atomicAdd(&ss.nact[par], 1);
              ss.flag[sk] = 0;
              if (ALGO == kFista) {
                const double t = ss.t[sk];
                const double tn = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));   // solvers.py:160-161
                ss.tn[sk] = tn;
                ss.betan[sk] = (t - 1.0) / tn;
              }
            } else {
              ss.inv_l[sk] = 0.0;
              ss.thr[sk] = 0.0;
              ss.betan[sk] = 0.0;
            }
          }
        }
      __syncthreads();
    }
    CMARK(0);
    for (int s = ow; s < SL; s += nown)
      if (ss.need_pf[s]) {
        __syncwarp();
        if (lane == 0) ss.need_pf[s] = 0;
        prefetch_slot<ALGO, SL>(a, ss, sy, sm, s);
      }
    // masks of this tick's slot phase (written before the barriers above)
    unsigned retm = 0u, freshm = 0u;
    bool done = false;
    auto read_masks = [&]() {
      retm = ss.retmask[par];
      freshm = ss.freshmask[par];
      done = ss.nact[par] == 0;
      if (threadIdx.x == 0) {
        ss.nact[par ^ 1] = 0;
        ss.retmask[par ^ 1] = 0u;
        ss.freshmask[par ^ 1] = 0u;
        ss.kmask[par ^ 1] = 0ull;
      }
    };
    auto fista_results = [&]() {
      // result of the slots that retired (element layout); x_0 = 0 for the
      // refilled / emptied ones
      if (retm | freshm) {
#pragma unroll
        for (int cb = 0; cb < CB; ++cb)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int s = acc_col(cb, i, lane);
            if ((retm >> s) & 1u) {
              const long long pid = ss.rpid[s];
              const bool fail = ss.rfail[s];
#pragma unroll
              for (int rb = 0; rb < MAXRB; ++rb) {
                if (rb >= nrb) break;
                const int n = row0 + 8 * rb;
                if (n < N) a.x_out[pid * N + n] = fail ? 0.0 : p0[rb][cb][i];
              }
            }
            if ((freshm >> s) & 1u) {
#pragma unroll
              for (int rb = 0; rb < MAXRB; ++rb) p0[rb][cb][i] = 0.0;
            }
          }
      }
    };
    read_masks();
    if (ALGO == kFista) fista_results();
    if (done) break;
    CMARK(1);
    TMARK(1);
    // ---- GEMM 1 (fista: grad = Psi^T g; admm: v = Psi (z - w)) ------------
    gemm(mat1, bufA);
    TMARK(2);
    // fista: its epilogue overwrites the GEMM's input; admm's writes the other
    // buffer, so a warp runs on into its epilogue
    if (ALGO == kFista) __syncthreads();
    TMARK(3);
    CMARK(2);

    double part[NV];
    unsigned long long kbits = 0ull;   // fista: k-steps of this thread's nonzero x_{k+1}
    // this thread's 16 row -> measurement entries (refills are done: barrier above)
    const uint4 pw = *reinterpret_cast<const uint4*>(pos + 16 * threadIdx.x);
    // The epilogues run per column block: all shared loads of the block's
    // elements, then the arithmetic (independent chains the scheduler can
    // interleave; the soft threshold's division on the branch-free path of
    // soft_fast), then the stores.  NRB is the compile-time row-block count
    // of the warp (exact for the 32-slot engine; the 16-slot engine passes
    // its maximum and predicates on nrb).
    if (ALGO == kFista) {
      // ---- epilogue 1: prox-gradient + momentum ---------------------------
      auto epi1 = [&](auto nrbc) {
        constexpr int NRB = decltype(nrbc)::value;
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) {
          double z[2][NRB], xn[2][NRB], il[2], th[2], bn[2];
          int zi[2][NRB];
          bool ok = true;
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int s = acc_col(cb, i, lane);
            il[i] = ss.inv_l[s];
            th[i] = ss.thr[s];
            bn[i] = ss.betan[s];
#pragma unroll
            for (int rb = 0; rb < NRB; ++rb) {
              zi[i][rb] = eidx(rb, cb, i);
              z[i][rb] = (rb < nrb) ? bufB[zi[i][rb]] : 0.0;
            }
          }
          // (skipping the divisions of a block that shrinks to zero as a whole,
          // behind a warp vote, measured 2.6% slower)
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int rb = 0; rb < NRB; ++rb) {
              z[i][rb] = __dsub_rn(z[i][rb], __dmul_rn(il[i], acc[rb][cb][i]));   // aux, solvers.py:183
              xn[i][rb] = soft_fast(z[i][rb], th[i], ok);                          // solvers.py:185
            }
          if (!ok) {   // operands outside the fast division's range: the plain soft()
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
              for (int rb = 0; rb < NRB; ++rb) xn[i][rb] = soft(z[i][rb], th[i]);
          }
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            bool bad = false;
#pragma unroll
            for (int rb = 0; rb < NRB; ++rb) {
              if (rb >= nrb) continue;
              const double x = p0[rb][cb][i], v = xn[i][rb];
              bufB[zi[i][rb]] = __dadd_rn(v, __dmul_rn(bn[i], __dsub_rn(v, x)));          // solvers.py:189
              p0[rb][cb][i] = v;
              bad |= !isfinite(v);
              bufA[zi[i][rb]] = v;
              if (v != 0.0) kbits |= 1ull << ((row0 + 8 * rb) >> 2);
            }
            if (bad) ss.flag[acc_col(cb, i, lane)] = 1;
          }
        }
      };
      if constexpr (SL == 32) {
        if (nrb == 2) epi1(std::integral_constant<int, 2>{}); else epi1(std::integral_constant<int, 1>{});
      } else {
        epi1(std::integral_constant<int, MAXRB>{});
      }
      if (use_kskip) {
        const unsigned lo = __reduce_or_sync(0xffffffffu, (unsigned)kbits);
        const unsigned hi = __reduce_or_sync(0xffffffffu, (unsigned)(kbits >> 32));
        if (lane == 0 && (lo | hi)) atomicOr(&ss.kmask[par], ((unsigned long long)hi << 32) | lo);
      }
      preload(mat2);   // next GEMM's first k-steps (the dense path's)
      TMARK(4);
      __syncthreads();
      TMARK(5);
      CMARK(3);
      // ---- GEMM 2: F = Psi x_{k+1}; epilogue: residual, delta, next g -------
      // the masked loop only when at most half the k-steps are active (it
      // prefetches 2 steps ahead instead of 4: slower on a dense mask)
      if (use_kskip && 2 * __popcll(ss.kmask[par]) <= KS) {
        if constexpr (SL == 32) tile_gemm_masked(nrb, a.fragS, rb0, bufA, KS, ss.kmask[par], acc);
      } else {
        gemm(a.fragS, bufA);
      }
      TMARK(6);
      __syncthreads();
      TMARK(7);
      CMARK(4);
      auto epi2 = [&](auto nrbc) {
        constexpr int NRB = decltype(nrbc)::value;
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) {
          double yv[2][NRB], ro[2][NRB], rn[2][NRB], bn[2];
          int pj[2][NRB];
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int s = acc_col(cb, i, lane);
            bn[i] = ss.betan[s];
#pragma unroll
            for (int rb = 0; rb < NRB; ++rb) {
              const int e = pos_entry(pw, (2 * cb + i) * MAXRB + rb);
              pj[i][rb] = (rb < nrb && e != 0xFF) ? (2 * (lane & 3) + 8 * cb + i) * M + e : -1;
              yv[i][rb] = pj[i][rb] >= 0 ? ys[pj[i][rb]] : 0.0;
              ro[i][rb] = pj[i][rb] >= 0 ? r[pj[i][rb]] : 0.0;
            }
          }
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            double dd = 0.0;
#pragma unroll
            for (int rb = 0; rb < NRB; ++rb) {
              rn[i][rb] = yv[i][rb] - acc[rb][cb][i];   // measured row: r = y - A x (solvers.py:192-196)
              if (pj[i][rb] >= 0) {
                const double d = rn[i][rb] - ro[i][rb];
                dd = fma(d, d, dd);
              }
            }
            part[2 * cb + i] = dd;
          }
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int s = acc_col(cb, i, lane);
#pragma unroll
            for (int rb = 0; rb < NRB; ++rb) {
              if (rb >= nrb) continue;
              double g = 0.0;
              if (pj[i][rb] >= 0) {
                const double rnv = rn[i][rb], rov = ro[i][rb], bnv = bn[i];
                r[pj[i][rb]] = rnv;
                // next gradient input A z - y = -(1 + b) r + b r_prev
                g = (bnv == 0.0) ? -rnv : -(1.0 + bnv) * rnv + bnv * rov;
              }
              bufA[eidx(rb, cb, i)] = g;
            }
          }
        }
      };
      if constexpr (SL == 32) {
        if (nrb == 2) epi2(std::integral_constant<int, 2>{}); else epi2(std::integral_constant<int, 1>{});
      } else {
        epi2(std::integral_constant<int, MAXRB>{});
      }
      partD[w * SL + cred] = reduce(part);
      preload(mat1);   // next GEMM's first k-steps
      TMARK(8);
      __syncthreads();
      TMARK(9);
      CMARK(5);
    } else {
      // ---- GEMM 1: v = Psi (z - w); epilogue: u' = (yhat + alpha v) / (d + alpha),
      //      residual y - A x = y - u'[mask] of this iteration's x; the last
      //      residual is y - (the u' this epilogue overwrites)[mask] ----------
      const double alpha = a.prm.alpha;
      if (freshm) {   // slots refilled in this tick: a zero dual (and Psi times their zero input, exactly 0)
#pragma unroll
        for (int cb = 0; cb < CB; ++cb)
#pragma unroll
          for (int i = 0; i < 2; ++i)
            if ((freshm >> acc_col(cb, i, lane)) & 1u) {
#pragma unroll
              for (int rb = 0; rb < MAXRB; ++rb) acc[rb][cb][i] = p1[rb][cb][i] = 0.0;
            }
      }
      auto epi1 = [&](auto nrbc) {
        constexpr int NRB = decltype(nrbc)::value;
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) {
          double yh[2][NRB], upo[2][NRB], up[2][NRB];
          int idx[2][NRB];
          bool in_mask[2][NRB];
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int s = acc_col(cb, i, lane);
#pragma unroll
            for (int rb = 0; rb < NRB; ++rb) {
              const int e = pos_entry(pw, (2 * cb + i) * MAXRB + rb);
              in_mask[i][rb] = rb < nrb && e != 0xFF;
              idx[i][rb] = eidx(rb, cb, i);
              yh[i][rb] = in_mask[i][rb] ? ysq[(8 * cb + i) * M + e] : 0.0;
              upo[i][rb] = (rb < nrb) ? bufB[idx[i][rb]] : 0.0;
            }
          }
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            double dd = 0.0;
#pragma unroll
            for (int rb = 0; rb < NRB; ++rb) {
              up[i][rb] = (yh[i][rb] + alpha * acc[rb][cb][i]) * (in_mask[i][rb] ? inv1 : inv0);
              if (in_mask[i][rb]) {
                const double rn = yh[i][rb] - up[i][rb];
                const double d = rn - (yh[i][rb] - upo[i][rb]);
                dd = fma(d, d, dd);
              }
            }
            part[2 * cb + i] = dd;
          }
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int rb = 0; rb < NRB; ++rb)
              if (rb < nrb) bufB[idx[i][rb]] = up[i][rb];
        }
      };
      if constexpr (SL == 32) {
        if (nrb == 2) epi1(std::integral_constant<int, 2>{}); else epi1(std::integral_constant<int, 1>{});
      } else {
        epi1(std::integral_constant<int, MAXRB>{});
      }
      partD[w * SL + cred] = reduce(part);
      preload(mat2);   // next GEMM's first k-steps
      TMARK(4);
      __syncthreads();
      TMARK(5);
      CMARK(3);
      // ---- GEMM 2: x = Psi^T u'; epilogue: shrink, dual update, gap --------
      gemm(a.fragT, bufB);
      TMARK(6);
      TMARK(7);
      CMARK(4);
      auto epi2 = [&](auto nrbc) {
        constexpr int NRB = decltype(nrbc)::value;
#pragma unroll
        for (int cb = 0; cb < CB; ++cb) {
          double zn[2][NRB], th[2];
          bool ok = true;
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            th[i] = ss.thr[acc_col(cb, i, lane)];
#pragma unroll
            for (int rb = 0; rb < NRB; ++rb)
              zn[i][rb] = soft_fast(__dadd_rn(acc[rb][cb][i], p1[rb][cb][i]), th[i], ok);   // solvers.py:229
          }
          if (!ok) {   // operands outside the fast division's range: the plain soft()
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
              for (int rb = 0; rb < NRB; ++rb) zn[i][rb] = soft(__dadd_rn(acc[rb][cb][i], p1[rb][cb][i]), th[i]);
          }
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int s = acc_col(cb, i, lane);
            const bool act = ss.status[s] == kActive;
            double* xo = a.x_out + ss.pid[s] * N;
            bool bad = false;
            double g2 = 0.0;
#pragma unroll
            for (int rb = 0; rb < NRB; ++rb) {
              if (rb >= nrb) continue;
              const int n = row0 + 8 * rb;
              const double x = acc[rb][cb][i], wv = p1[rb][cb][i], z = zn[i][rb];
              const double wn = __dsub_rn(__dadd_rn(wv, x), z);            // solvers.py:231
              // z is the returned iterate: stored every pass (L2-absorbed), so
              // it needs no registers between passes
              if (act && n < N) xo[n] = z;
              p1[rb][cb][i] = wn;
              bufA[eidx(rb, cb, i)] = z - wn;                              // next GEMM 1 input
              const double dg = x - z;
              g2 = fma(dg, dg, g2);
              bad |= !isfinite(z);
            }
            part[2 * cb + i] = g2;
            if (bad) ss.flag[s] = 1;
          }
        }
      };
      if constexpr (SL == 32) {
        if (nrb == 2) epi2(std::integral_constant<int, 2>{}); else epi2(std::integral_constant<int, 1>{});
      } else {
        epi2(std::integral_constant<int, MAXRB>{});
      }
      partG[w * SL + cred] = reduce(part);
      preload(mat1);   // next GEMM's first k-steps
      TMARK(8);
      __syncthreads();
      TMARK(9);
      CMARK(5);
    }
  }
#ifdef HCS_PHASES
  if (threadIdx.x == 0)
    for (int k = 0; k < 15; ++k) atomicAdd(&g_phase_cx[k], (unsigned long long)cph[k]);
#endif
  hcs_smem_canary(smraw, a.smem_bytes, a.err);
}

// Fragment-order copies of Psi and Psi^T (layout of tile_gemm), and
// u0 = Psi * (1/sqrt(N)) 1.  Row block rb's fragment for k-step ks, lane l is
// Mat[8 rb + l/4][4 ks + l%4]; with `interleave` (the 32-slot engine) blocks
// owned in pairs by one warp (warp_rows) are interleaved as double2, else the
// order is plain (the 16-slot engine, tile_gemm16).
__global__ void prep_basis_kernel(const double* __restrict__ basis, int N, int Np, double* fragS, double* fragT,
                                  double* u0, int interleave) {
  const int KS = Np >> 2, RB = Np >> 3;
  const int nd = (interleave && RB > 16) ? RB - 16 : 0;
  const long long total = (long long)RB * KS * 32;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int lane = (int)(idx & 31);
    const long long t = idx >> 5;
    const int ks = (int)(t % KS);
    const int rb = (int)(t / KS);
    const int r = 8 * rb + (lane >> 2), c = 4 * ks + (lane & 3);
    const size_t dst = rb < 2 * nd ? ((size_t)((rb >> 1) * KS + ks) * 32 + lane) * 2 + (rb & 1)
                                   : ((size_t)rb * KS + ks) * 32 + lane;
    fragS[dst] = (r < N && c < N) ? basis[(size_t)r * N + c] : 0.0;
    fragT[dst] = (r < N && c < N) ? basis[(size_t)c * N + r] : 0.0;
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

// Lipschitz constants of every pixel's A (fista), one warp per pixel, ahead
// of the slot engine so that a refill never waits on the power iteration.
__global__ void lipschitz_prepass_kernel(long long P, int M, const uint8_t* __restrict__ mask,
                                         const double* __restrict__ u0, double* __restrict__ lip, const int* err) {
  if (*(volatile const int*)err & kErrMask) return;
  const int lane = threadIdx.x & 31;
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long p = gw; p < P; p += nw) {
    const double l = warp_lipschitz(u0, mask + p * M, M);
    if (lane == 0) lip[p] = l;
  }
}

cudaError_t launch_lipschitz_prepass(long long P, int M, const uint8_t* mask, const double* u0, double* lip,
                                     const int* err, int sms, cudaStream_t stream) {
  lipschitz_prepass_kernel<<<sms * 8, 256, 0, stream>>>(P, M, mask, u0, lip, err);
  return cudaGetLastError();
}

cudaError_t launch_prep_basis(const double* basis, int N, int Np, double* fragS, double* fragT, double* u0,
                              int slots, cudaStream_t stream) {
  prep_basis_kernel<<<64, 256, 0, stream>>>(basis, N, Np, fragS, fragT, u0, slots == 32 ? 1 : 0);
  return cudaGetLastError();
}

// ADMM while the shrinkage provably zeroes every coefficient (solvers.py:206-245
// with z = soft(x + w, lambda/alpha) = 0): with z = 0 the iteration is
// diagonal in the sample domain.  For orthonormal Psi and W = Psi w,
//     Psi x = u' = (yhat - alpha W) / (d + alpha),   w <- w + x  =>  W <- W + u',
// the residual y - A x = yhat - u' on the measured rows, ||x - z|| = ||u'||,
// and z = 0 is certified every pass by |x_i + w_i| <= ||x + w|| = ||u' + W||
// <= (1 - 1e-9) lambda/alpha (Parseval; the margin covers the rounding of the
// elementwise recurrence against the coefficient-domain one).  The same
// iterates, iteration count and stop decisions as the slot engine, at
// O(N) instead of 4 N^2 FLOP per iteration; a pixel whose certificate fails
// (or whose measurements are not finite) is appended to plist and solved from
// scratch by the slot engine.  One warp per pixel, rows n = lane + 32 k.
__global__ void __launch_bounds__(256) admm_zero_kernel(ConvexArgs a, long long* plist,
                                                        unsigned long long* plist_n) {
  if (*(volatile const int*)a.err & kErrMask) return;
  __shared__ double syw[8][kMaxN];
  __shared__ uint8_t smw[8][kMaxN];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int N = a.N, M = a.M;
  const double alpha = a.prm.alpha;
  const double inv0 = 1.0 / alpha, inv1 = 1.0 / (1.0 + alpha);
  const double bound = (a.prm.lam / alpha) * (1.0 - 1e-9);
  const double NaN = __longlong_as_double(0x7ff8000000000000ll);
  constexpr int R = kMaxN / 32;
  for (long long p = gw; p < a.P; p += nw) {
    for (int n = lane; n < kMaxN; n += 32) {
      syw[wl][n] = 0.0;
      smw[wl][n] = 0;
    }
    __syncwarp();
    bool nz = false, bad = false;
    for (int j = lane; j < M; j += 32) {
      const double v = a.y[p * M + j];
      const int row = a.mask[p * M + j];
      syw[wl][row] = v;
      smw[wl][row] = 1;
      nz |= (v != 0.0);
      bad |= !isfinite(v);
    }
    nz = __any_sync(0xffffffffu, nz);
    bad = __any_sync(0xffffffffu, bad);
    __syncwarp();
    const long long t0 = now_ns();
    if (bad) {   // cho_solve raises (solvers.py:227); the engine flags it
      if (lane == 0) plist[atomicAdd(plist_n, 1ull)] = p;
      continue;
    }
    double* xo = a.x_out + p * N;
    if (!nz) {   // y == 0: x = 0, 0 iterations, converged, delta 0, no admm_gap
      for (int n = lane; n < N; n += 32) xo[n] = 0.0;
      if (lane == 0) {
        a.st.iterations[p] = 0;
        a.st.converged[p] = 1;
        a.st.final_delta[p] = 0.0;
        a.st.failed_at[p] = -1;
        if (a.st.admm_gap) a.st.admm_gap[p] = NaN;
        if (a.st.lipschitz) a.st.lipschitz[p] = NaN;
        if (a.st.elapsed) a.st.elapsed[p] = 0.0;
        if (a.st.work) a.st.work[p] = 0.0;
      }
      continue;
    }
    int dec = stop_decision(1.0, 0, t0, a.prm);
    double yh[R], inv[R], W[R], rp[R];
    bool ms[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int n = lane + 32 * k;
      yh[k] = syw[wl][n];
      ms[k] = smw[wl][n] != 0;
      inv[k] = ms[k] ? inv1 : inv0;
      W[k] = 0.0;
      rp[k] = yh[k];                   // r_0 = y on the measured rows
    }
    int it = 0;
    double delta = 1.0, gap2 = 0.0;
    bool certified = true, failed = false;
    while (dec == kContinue) {
      double dd = 0.0, s2 = 0.0, g2 = 0.0;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if (lane + 32 * k >= N) break;
        const double up = (yh[k] + alpha * (-W[k])) * inv[k];
        if (ms[k]) {
          const double rn = yh[k] - up;
          const double d = rn - rp[k];
          dd = fma(d, d, dd);
          rp[k] = rn;
        }
        const double xw = up + W[k];
        s2 += xw * xw;
        g2 += up * up;
        W[k] += up;
      }
      dd = warp_sum(dd);
      s2 = warp_sum(s2);
      g2 = warp_sum(g2);
      if (!(sqrt(s2) <= bound)) { certified = false; break; }
      ++it;
      delta = sqrt(dd);
      gap2 = g2;
      if (!isfinite(delta)) { failed = true; break; }
      dec = stop_decision(delta, it, t0, a.prm);
    }
    if (!certified) {
      if (lane == 0) plist[atomicAdd(plist_n, 1ull)] = p;
      continue;
    }
    for (int n = lane; n < N; n += 32) xo[n] = 0.0;   // z = 0
    if (lane == 0) {
      a.st.iterations[p] = failed ? 0 : it;
      a.st.converged[p] = (!failed && dec == kConverged) ? 1 : 0;
      a.st.final_delta[p] = failed ? NaN : delta;
      a.st.failed_at[p] = failed ? it : -1;
      if (a.st.admm_gap) a.st.admm_gap[p] = failed ? NaN : (it == 0 ? 0.0 : sqrt(gap2));
      if (a.st.lipschitz) a.st.lipschitz[p] = NaN;
      if (a.st.elapsed) a.st.elapsed[p] = 1e-9 * (double)(now_ns() - t0);
      if (a.st.work) a.st.work[p] = 12.0 * (double)N * (double)it;   // the elementwise pass, not 4 N^2
    }
  }
}

cudaError_t launch_admm_zero(const ConvexArgs& args, long long* plist, unsigned long long* plist_n, int sms,
                             cudaStream_t stream) {
  admm_zero_kernel<<<sms * 8, 256, 0, stream>>>(args, plist, plist_n);
  return cudaGetLastError();
}

// without the A-fragment ring
static size_t convex_smem_base(int algo, int Np, int M, int slots) {
  const size_t sl = (size_t)slots;
  size_t b = sizeof(double) * (size_t)Np * sl * 2;                   // bufA, bufB
  b += sizeof(double) * sl * M * (algo == kFista ? 2 : 1);           // ys, r (fista)
  b += sizeof(double) * 16 * sl * (algo == kAdmm ? 2 : 1);           // partD, partG (admm)
  b += sizeof(double) * sl * M;                                      // sy
  b += slots == 32 ? sizeof(SlotState<32>) : sizeof(SlotState<16>);
  b += 16 + sl * kMaxN;                                              // pos (16-byte aligned)
  b += sl * stage_mask_bytes(M);                                     // sm
  return (b + 15) & ~(size_t)15;
}

// the 32-slot engine takes the A-fragment ring when it fits beside the rest
// (HCS_CONVEX_RING=0: register prefetch, for A/B runs)
bool convex_ring(int algo, int Np, int M, int slots) {
  if (slots != 32) return false;
  if (const char* ov = getenv("HCS_CONVEX_RING")) if (atoi(ov) == 0) return false;
  return convex_smem_base(algo, Np, M, slots) + 16 + ring_bytes(Np) + kSmemExtra <= (size_t)227 * 1024;
}

size_t convex_smem_bytes(int algo, int Np, int M, int slots) {
  const size_t b = convex_smem_base(algo, Np, M, slots);
  return convex_ring(algo, Np, M, slots) ? b + 16 + ring_bytes(Np) : b;
}

// Slot engine variant for (Np, M): 32 slots x one CTA per SM (default).  The
// 16-slot x two-CTAs-per-SM engine (HCS_CONVEX_SLOTS=16, experiments) runs
// the two CTAs out of phase, but on B200 the FP64 epilogue / slot-phase
// arithmetic shares the FP64 datapath with DMMA, so it queues behind the other
// CTA's tensor work instead of overlapping it: measured 15% slower (FISTA
// 62.6 -> 73.2 ms, ADMM 103.7 -> 120.6 ms on 100k Salinas pixels;
// epilogue cycles x5.6 per CTA; profiles/convex_slots_ab_r01.txt).
// Systems whose 32-slot layout exceeds the 227 KB of one CTA (N = 224 with
// M above ~116, i.e. sampling ratios above ~0.52) take the 16-slot engine, one
// or two CTAs per SM; 0 = not even 16 slots fit (HCS_EINVAL).
int convex_slots(int algo, int Np, int M) {
  constexpr size_t kCta = 227 * 1024;
  int want = 32;
  if (const char* ov = getenv("HCS_CONVEX_SLOTS")) want = atoi(ov) == 16 ? 16 : 32;
  if (want == 16 && 2 * (convex_smem_bytes(algo, Np, M, 16) + 1024) > 228 * 1024) want = 32;
  if (want == 32 && convex_smem_bytes(algo, Np, M, 32) > kCta) want = 16;
  if (want == 16 && convex_smem_bytes(algo, Np, M, 16) > kCta) return 0;
  return want;
}

int convex_ctas_per_sm(int algo, int Np, int M, int slots) {
  if (slots == 32) return 1;
  return 2 * (convex_smem_bytes(algo, Np, M, 16) + 1024) <= 228 * 1024 ? 2 : 1;
}

template <int ALGO, int SL, int MAXT, int MINB, int RING>
static cudaError_t launch_convex_t(const ConvexArgs& args, int grid, size_t smem, cudaStream_t stream) {
  cudaError_t e = cudaFuncSetAttribute(convex_kernel<ALGO, SL, MAXT, MINB, RING>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem + kSmemExtra));
  if (e != cudaSuccess) return e;
  const int warps = SL == 32 ? engine_warps(args.Np) : engine_warps16(args.Np);
  ConvexArgs ca = args;
  ca.smem_bytes = (unsigned)smem;
  convex_kernel<ALGO, SL, MAXT, MINB, RING><<<grid, 32 * warps, smem + kSmemExtra, stream>>>(ca);
  return cudaGetLastError();
}

cudaError_t launch_convex(int algo, const ConvexArgs& args, int slots, int grid, cudaStream_t stream) {
  const size_t smem = convex_smem_bytes(algo, args.Np, args.M, slots);
  if (slots == 32) {
    if (convex_ring(algo, args.Np, args.M, slots)) {
      if (algo == kFista) return launch_convex_t<kFista, 32, 512, 1, 1>(args, grid, smem, stream);
      return launch_convex_t<kAdmm, 32, 512, 1, 1>(args, grid, smem, stream);
    }
    if (algo == kFista) return launch_convex_t<kFista, 32, 512, 1, 0>(args, grid, smem, stream);
    return launch_convex_t<kAdmm, 32, 512, 1, 0>(args, grid, smem, stream);
  }
  if (algo == kFista) return launch_convex_t<kFista, 16, 256, 2, 0>(args, grid, smem, stream);
  return launch_convex_t<kAdmm, 16, 256, 2, 0>(args, grid, smem, stream);
}

}  // namespace hcs

// debug builds (-DHCS_TRACE): the per-warp tick timeline of CTA 0 (4 ticks x 16 warps x 12 marks)
extern "C" int hcs_debug_trace_cx(long long* out768) {
#ifdef HCS_TRACE
  return cudaMemcpyFromSymbol(out768, hcs::g_trace, sizeof(long long) * 4 * 16 * 12) == cudaSuccess ? 0 : 2;
#else
  (void)out768;
  return 1;
#endif
}

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
