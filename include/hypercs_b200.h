/*
 * hypercs_b200.h -- C ABI of the B200-native per-pixel compressive-sensing
 * recovery library (libhypercs_b200.so, sm_100a).
 *
 * This is the drop-in boundary for the reference's hot path, the per-pixel
 * solver API of `hypercs` (Python):
 *
 *   SOLVERS[name](y, dictionary, config) -> SolverResult
 *       /root/reference/pkg/src/hypercs/solvers.py:164-403
 *   recover_cube(measurements, dictionary, config, algorithm, jobs) -> (cube, RecoveryStats)
 *       /root/reference/pkg/src/hypercs/solvers.py:455-514
 *
 * The reference has no FFI of its own (it is pure Python); its callers bind
 * to the functions below through ctypes.  Conventions:
 *
 *   - every array pointer is a DEVICE pointer owned by the caller; arrays are
 *     pixel-major and row-major (pixel p of an (x, y) cube is p = ix * Y + iy,
 *     solvers.py:497);
 *   - `basis` is the N x N orthonormal synthesis matrix Psi (f = Psi c) and
 *     pixel p's dictionary is A_p = Psi[mask_p, :] (the reference's
 *     Dictionary.matrix, transform.py:267-281, with one mask per pixel);
 *   - N <= 256 (band indices are uint8), 1 <= M <= N;
 *   - masks: each pixel's M band indices strictly increasing and < N.  The
 *     library checks this on the device before any solver kernel reads a
 *     mask: a violation makes every solver kernel of the call exit without
 *     writing outputs and hcs_recover_status() return HCS_EINVAL;
 *   - `basis` must be orthonormal (Psi^T Psi = I): the FISTA / ADMM closed
 *     forms, the sample-domain Lipschitz constant and the coefficient-domain
 *     PSNR rely on it.  A non-orthonormal basis is UNDEFINED BEHAVIOUR (silently
 *     wrong results); hcs_check_basis() measures max |Psi^T Psi - I| once per
 *     basis (the Python Dictionary rejects > 1e-10, transform.py:170-173);
 *   - all calls are stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 *     default stream) and reentrant; no global mutable state;
 *   - return codes: HCS_OK, HCS_EINVAL (bad arguments: the Python layer raises
 *     ValueError, same preconditions as the reference), HCS_ECUDA (CUDA error),
 *     HCS_ENONFINITE (non-finite measurements where the reference raises
 *     ValueError from scipy's finiteness check, solvers.py:227 /
 *     kernels.py:61).  Per-pixel numerical failures never become error codes:
 *     they go to stats.failed_at (solvers.py:445-452).
 *     HCS_ENONFINITE is only known after the stream has executed, so it is
 *     reported by hcs_recover_status(), not by hcs_recover().
 */
#ifndef HYPERCS_B200_H
#define HYPERCS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HCS_OK 0
#define HCS_EINVAL 1
#define HCS_ECUDA 2
#define HCS_ENONFINITE 3

/* algorithm ids, in the order of SOLVERS (solvers.py:397-403) */
#define HCS_FISTA 0
#define HCS_ADMM 1
#define HCS_GOMP 2
#define HCS_BIHT 3
#define HCS_COSAMP 4

#define HCS_MAX_N 256

/* SolverConfig (solvers.py:40-85); max_iter <= 0 means no cap (None),
 * time_limit <= 0 means no wall-clock budget (None).  The budget is per pixel,
 * measured on the device from the moment the pixel is loaded (globaltimer),
 * and checked before every iteration with the reference's precedence
 * converged > timeout > cap (solvers.py:115-127). */
typedef struct {
  double lam;             /* l1 weight (fista, admm) */
  double mu;              /* biht gradient step */
  double alpha;           /* admm penalty rho */
  double epsilon;         /* residual-delta convergence threshold */
  int32_t kappa;          /* greedy target sparsity */
  int32_t atoms_per_iter; /* gomp G; <= 0 -> max(1, kappa / 5) */
  int32_t max_iter;       /* iteration cap; <= 0 -> unlimited */
  int32_t reserved;
  double time_limit;      /* seconds per pixel; <= 0 -> unlimited */
} hcs_params;

/* Per-pixel outputs (SolverResult fields, solvers.py:88-95).  Any pointer
 * may be NULL except iterations/converged/final_delta/failed_at. */
typedef struct {
  int32_t* iterations;   /* P */
  uint8_t* converged;    /* P */
  double* final_delta;   /* P */
  int32_t* failed_at;    /* P: -1 ok, else the NumericalFailure iteration */
  double* admm_gap;      /* P: ||x - z|| (admm only; NaN for zero pixels) */
  double* lipschitz;     /* P: power-iteration constant of A_p (fista) */
  double* elapsed;       /* P: seconds the pixel spent in the solver (device clock) */
  double* work;          /* P: algorithmic FLOPs executed for the pixel (SURVEY.md §8(d)
                            counts: 4N^2 per convex pass; 2NM correlation + LS(M,k)
                            + 2Mk residual per greedy pass), or NULL */
  uint64_t* trace;       /* optional selection trace (greedy): P x trace_calls x 4 words,
                            one 256-bit index bitmap per argmax_k call */
  int32_t* trace_len;    /* P: number of argmax_k calls recorded */
  int32_t trace_calls;   /* capacity per pixel */
  int32_t reserved;
} hcs_stats;

/* Version of the ABI (major * 100 + minor). */
int hcs_abi_version(void);

/* 1 for a bounds-checked build (-DHCS_CHECKS: shared-memory poison and
 * canaries, device index assertions; hcs_recover_status then reports a
 * failed check as HCS_ECUDA), else 0. */
int hcs_checked_build(void);

/* Human-readable message for the last error on this host thread. */
const char* hcs_last_error(void);

/* Device workspace hcs_recover needs for (algo, P, N, M), sized for the
 * device current at this call.  Layout (ABI 1.1; opaque to callers): a 256 B
 * header (work-queue counters, the error word hcs_recover_status reads, the
 * spill count of the warp-per-pixel gOMP kernel, and for the greedy solvers a
 * word that is 0 iff the basis was recognised on the device as the
 * orthonormal DCT-II, which lets BIHT / CoSaMP form their least-squares Gram
 * matrices in closed form; any other orthonormal basis takes the general
 * path); FISTA / ADMM: the basis in
 * DMMA fragment order (twice), a start vector, per-pixel Lipschitz constants
 * or the ADMM pixel list; gOMP / BIHT / CoSaMP: the transposed basis, a
 * P-entry spill list and per-CTA least-squares scratch (hcs_recover never
 * launches more CTAs than the workspace holds scratch for). */
size_t hcs_workspace_bytes(int algo, int64_t P, int32_t N, int32_t M);

/* Recover P pixels with one algorithm: the body of recover_cube
 * (solvers.py:455-514) for per-pixel dictionaries.  x_out is P x N. */
int hcs_recover(int algo, int64_t P, int32_t N, int32_t M, const double* basis,
                const double* y, const uint8_t* mask, const hcs_params* prm, double* x_out,
                const hcs_stats* stats, void* workspace, size_t workspace_bytes, void* stream);

/* Number of kernels one hcs_recover call with these arguments launches. */
int hcs_recover_launches(int algo, int32_t N, int32_t M, const hcs_params* prm);

/* After the stream has executed a hcs_recover call on `workspace`: HCS_OK,
 * HCS_EINVAL (a mask entry out of range or not strictly increasing; outputs
 * not written) or HCS_ENONFINITE (non-finite measurements); reads 4 bytes
 * from the workspace and synchronises `stream`. */
int hcs_recover_status(const void* workspace, void* stream);

/* max_ij |(Psi^T Psi - I)_ij| of the N x N basis (device pointer), written to
 * *max_dev_out (host); synchronises `stream`. */
int hcs_check_basis(int32_t N, const double* basis, double* max_dev_out, void* stream);

/* Batched kernels of hypercs.kernels (kernels.py:14-76). */
int hcs_soft_threshold(int64_t n, const double* v, double t, double* out, void* stream);
/* argmax_k (kernels.py:31-41) on P rows of length n: idx_out is P x k, ascending. */
int hcs_argmax_k(int64_t P, int32_t n, const double* v, int32_t k, int32_t* idx_out, void* stream);
/* least_squares (kernels.py:44-67) on P systems b_p (M x K row-major), y_p (M):
 * s_out P x K; path_out (optional) P: 0 = pivoted-QR solve, 1 = minimum-norm fallback. */
int hcs_least_squares(int64_t P, int32_t M, int32_t K, const double* b, const double* y,
                      double* s_out, int32_t* path_out, void* stream);
/* residual_delta (kernels.py:70-76) on P pairs of length n. */
int hcs_residual_delta(int64_t P, int32_t n, const double* r, const double* r_prev, double* out,
                       void* stream);
/* lipschitz_constant (transform.py:176-217) of A_p = basis[mask_p, :]. */
int hcs_lipschitz(int64_t P, int32_t N, int32_t M, const double* basis, const uint8_t* mask,
                  double* out, void* stream);

/* PSNR partial sums (metrics.py:30-55): sse_out[0] += sum (ref - basis @ x)^2
 * over P x N, absmax_out[0] = max(absmax_out[0], max |ref|).  Accumulates, so
 * the caller zeroes the two doubles once and may reduce them across ranks. */
int hcs_psnr_partials(int64_t P, int32_t N, const double* ref, const double* x,
                      const double* basis, double* sse_out, double* absmax_out, void* stream);

/* Coefficient-domain PSNR partial: sse_out[0] += sum over
 * P x N of (ref_coeffs - x)^2.  For an orthonormal basis this equals the
 * spectral-domain SSE of hcs_psnr_partials (Parseval) with no GEMM: an HBM
 * stream of 16 bytes per voxel.  The peak max|ref spectra| is input-derived
 * (hcs_psnr_partials or the caller's reduction). */
int hcs_sse_coeff_partials(int64_t P, int32_t N, const double* ref_coeffs, const double* x, double* sse_out,
                           void* stream);

/* ---- input side ------------------------------------------
 * Synthetic spectra of the frozen generator (synth.py v1) from host-drawn
 * parameters: f[p, b] = clip(sum_i amps[p, i] exp(-((b - centres[p, i]) /
 * widths[p, i])^2 / 2) + noise[p, b], 0, 1); centres/widths/amps are P x 4. */
int hcs_synth_spectra(int64_t P, int32_t N, const double* centres, const double* widths, const double* amps,
                      const double* noise, double* f_out, void* stream);

/* Sparsify + measure, the body of cli.run_sparsify / run_compress
 * (cli.py:97-139) for the DCT basis and per-pixel masks:
 *   c = basis^T f_p (to_sparse_domain, transform.py:40-45);
 *   rule HCS_SPARSIFY_MAXREL:  c_i = 0 where |c_i| < factor * max|c|  (BASELINE generator);
 *   rule HCS_SPARSIFY_MEANSTD: keep (|c_i| - mean|c|) >= factor * std|c| (transform.sparsify,
 *                              transform.py:73-97, population std);
 *   f_s = basis c (from_sparse_domain); y_p = f_s[mask_p] (measure, transform.py:168-173).
 * keys (P x N, optional): mask_p = the M smallest keys' band indices, sorted (written
 * to mask; ties to the lower index); without keys mask is an input.  coeffs_out,
 * spectra_out (P x N) and nzero_out (device counter, incremented by the number of
 * zeroed coefficients) may be NULL.  factor < 0 -> HCS_EINVAL (ValueError). */
#define HCS_SPARSIFY_MAXREL 0
#define HCS_SPARSIFY_MEANSTD 1
int hcs_sparsify_measure(int64_t P, int32_t N, int32_t M, const double* basis, const double* f, int32_t rule,
                         double factor, const double* keys, uint8_t* mask, double* coeffs_out, double* spectra_out,
                         double* y_out, uint64_t* nzero_out, void* stream);

/* FP64 tensor-core (DMMA m8n8k4) throughput of this GPU in TFLOP/s, best of 3
 * launches of `iters` iterations on the legacy default stream: the roofline
 * denominator for the FP64 GEMM phases (synchronises the device). */
int hcs_dmma_peak_tflops(double* tflops_out, int iters);

#ifdef __cplusplus
}
#endif
#endif /* HYPERCS_B200_H */
