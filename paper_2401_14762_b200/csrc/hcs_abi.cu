// hcs_abi.cu -- extern "C" entry points of libhypercs_b200.so (include/hypercs_b200.h).
//
// Host-side validation mirrors the reference's preconditions (solvers.py:67-85
// config checks are done by the Python SolverConfig; the per-solver checks of
// solvers.py:259-260, 306-307, 355-358 and the shape checks of :464-471 are
// repeated here so a C caller gets HCS_EINVAL for the same inputs).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/hypercs_b200.h"
#include "hcs_gemm.cuh"
#include "hcs_internal.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(HCS_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

constexpr size_t kHeader = 256;   // counter (u64) + error flag (int)

inline size_t align256(size_t b) { return (b + 255) & ~size_t(255); }
inline int pad16(int n) { return (n + 15) & ~15; }

int num_sms() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

bool greedy(int algo) { return algo == HCS_GOMP || algo == HCS_BIHT || algo == HCS_COSAMP; }


// LS matrices fit in shared memory up to this many bytes per CTA
constexpr size_t kGreedySmemCap = 200 * 1024;
constexpr int kMaxGreedyPerSm = 8;

// Greedy workspace (ABI 1.1): [header 256 B: queue counter, error flag,
// spill count, spill-queue counter][transposed basis N x N doubles][spill
// list P x int64][per-CTA LS scratch, greedy_ls_doubles(M) doubles per CTA]
struct GreedyWs {
  size_t basis_t, spill, scratch;
  long long slots;   // CTA scratch slots in a workspace of `bytes` bytes (0: not computed)
};

GreedyWs greedy_ws(int64_t P, int32_t N, int32_t M, size_t bytes) {
  GreedyWs w;
  w.basis_t = kHeader;
  w.spill = w.basis_t + align256(sizeof(double) * (size_t)N * N);
  w.scratch = w.spill + align256(sizeof(long long) * (size_t)(P > 0 ? P : 1));
  const size_t per = sizeof(double) * hcs::greedy_ls_doubles(M);
  w.slots = bytes > w.scratch ? (long long)((bytes - w.scratch) / per) : 0;
  return w;
}

}  // namespace

extern "C" {

int hcs_abi_version(void) { return 101; }

int hcs_checked_build(void) {
#ifdef HCS_CHECKS
  return 1;
#else
  return 0;
#endif
}

const char* hcs_last_error(void) { return g_err.c_str(); }

size_t hcs_workspace_bytes(int algo, int64_t P, int32_t N, int32_t M) {
  size_t b = kHeader;
  if (algo == HCS_FISTA || algo == HCS_ADMM) {
    const int Np = pad16(N);
    b += 2 * align256(sizeof(double) * (size_t)Np * Np);   // fragS, fragT
    b += align256(sizeof(double) * (size_t)Np);            // u0
    if (algo == HCS_FISTA && P > 0) b += align256(sizeof(double) * (size_t)P);   // Lipschitz constants
    if (algo == HCS_ADMM && P > 0) b += align256(sizeof(long long) * (size_t)P);  // uncertified-pixel list
  } else if (greedy(algo)) {
    b = greedy_ws(P, N, M, 0).scratch;
    // per-CTA global scratch for systems beyond the shared-memory region
    b += align256(sizeof(double) * hcs::greedy_ls_doubles(M) * (size_t)num_sms() * kMaxGreedyPerSm);
  }
  return b;
}

constexpr int kSmemPerBlock = 227 * 1024;

static int validate(int algo, int64_t P, int32_t N, int32_t M, const hcs_params* prm) {
  if (algo < HCS_FISTA || algo > HCS_COSAMP) return fail(HCS_EINVAL, "unknown algorithm");
  if (P < 0) return fail(HCS_EINVAL, "negative pixel count");
  if (N < 1 || N > HCS_MAX_N) return fail(HCS_EINVAL, "N must be in [1, 256]");
  if (M < 1 || M > N) return fail(HCS_EINVAL, "M must be in [1, N]");
  if (!prm) return fail(HCS_EINVAL, "null params");
  if (prm->lam < 0) return fail(HCS_EINVAL, "lam must be >= 0");
  if (prm->kappa < 1) return fail(HCS_EINVAL, "kappa must be >= 1");
  if (prm->mu <= 0) return fail(HCS_EINVAL, "mu must be > 0");
  if (prm->alpha <= 0) return fail(HCS_EINVAL, "alpha must be > 0");
  if (prm->epsilon <= 0) return fail(HCS_EINVAL, "epsilon must be > 0");
  const int G = prm->atoms_per_iter > 0 ? prm->atoms_per_iter : (prm->kappa / 5 > 1 ? prm->kappa / 5 : 1);
  if (G < 1 || G > prm->kappa) return fail(HCS_EINVAL, "atoms_per_iter must be in [1, kappa]");
  if (algo == HCS_GOMP && !(G <= prm->kappa && prm->kappa <= M))
    return fail(HCS_EINVAL, "need atoms_per_iter <= kappa <= " + std::to_string(M));
  if (algo == HCS_BIHT && prm->kappa > M) return fail(HCS_EINVAL, "kappa must be <= " + std::to_string(M));
  if (algo == HCS_COSAMP) {
    if (2 * prm->kappa > N) return fail(HCS_EINVAL, "need 2 * kappa <= " + std::to_string(N));
    if (prm->kappa > M) return fail(HCS_EINVAL, "kappa must be <= " + std::to_string(M));
  }
  return HCS_OK;
}

int hcs_recover(int algo, int64_t P, int32_t N, int32_t M, const double* basis, const double* y,
                const uint8_t* mask, const hcs_params* prm, double* x_out, const hcs_stats* stats,
                void* workspace, size_t workspace_bytes, void* stream_) {
  int v = validate(algo, P, N, M, prm);
  if (v != HCS_OK) return v;
  if (!stats || !stats->iterations || !stats->converged || !stats->final_delta || !stats->failed_at)
    return fail(HCS_EINVAL, "stats arrays iterations/converged/final_delta/failed_at are required");
  if (workspace_bytes < hcs_workspace_bytes(algo, P, N, M)) return fail(HCS_EINVAL, "workspace too small");
  if (P > 0 && (!basis || !y || !mask || !x_out || !workspace)) return fail(HCS_EINVAL, "null array");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  cudaError_t e = cudaMemsetAsync(ws, 0, kHeader, stream);
  if (e != cudaSuccess) return cuda_fail(e, "memset");
  if (P == 0) return HCS_OK;

  hcs::Stats st{stats->iterations, stats->converged, stats->final_delta, stats->failed_at, stats->admm_gap,
                stats->lipschitz, stats->elapsed, stats->work, stats->trace, stats->trace_len,
                stats->trace ? stats->trace_calls : 0};
  // the budget in whole nanoseconds, rounded down (elapsed >= limit, solvers.py:123)
  const long long limit_ns = prm->time_limit > 0 ? (long long)(prm->time_limit * 1e9) : -1;
  hcs::Params pr{prm->lam, prm->mu, prm->alpha, prm->epsilon, prm->kappa,
                 prm->atoms_per_iter > 0 ? prm->atoms_per_iter : (prm->kappa / 5 > 1 ? prm->kappa / 5 : 1),
                 prm->max_iter, algo, limit_ns};
  unsigned long long* counter = reinterpret_cast<unsigned long long*>(ws);
  int* err = reinterpret_cast<int*>(ws + 8);
  const int sms = num_sms();
  // masks: strictly increasing band indices < N, checked on the device before
  // any solver kernel reads one (HCS_EINVAL from hcs_recover_status)
  e = hcs::launch_validate_masks(P, M, N, mask, err, sms, stream);
  if (e != cudaSuccess) return cuda_fail(e, "validate_masks_kernel");

  if (algo == HCS_FISTA || algo == HCS_ADMM) {
    const int Np = pad16(N);
    const int calgo = algo == HCS_FISTA ? hcs::kFista : hcs::kAdmm;
    const int slots = hcs::convex_slots(calgo, Np, M);
    if (slots == 0)
      return fail(HCS_EINVAL, "convex solvers: 16 pixel slots of N = " + std::to_string(N) + ", M = " +
                                  std::to_string(M) + " exceed the 227 KB shared memory of one SM");
    double* fragS = reinterpret_cast<double*>(ws + kHeader);
    double* fragT = reinterpret_cast<double*>(ws + kHeader + align256(sizeof(double) * (size_t)Np * Np));
    double* u0 = reinterpret_cast<double*>(ws + kHeader + 2 * align256(sizeof(double) * (size_t)Np * Np));
    double* lip = reinterpret_cast<double*>(ws + kHeader + 2 * align256(sizeof(double) * (size_t)Np * Np) +
                                            align256(sizeof(double) * (size_t)Np));
    e = hcs::launch_prep_basis(basis, N, Np, fragS, fragT, u0, slots, stream);
    if (e != cudaSuccess) return cuda_fail(e, "prep_basis_kernel");
    if (algo == HCS_FISTA) {
      e = hcs::launch_lipschitz_prepass(P, M, mask, u0, lip, err, sms, stream);
      if (e != cudaSuccess) return cuda_fail(e, "lipschitz_prepass_kernel");
    }
    hcs::ConvexArgs args{(long long)P, N, Np, M, y, mask, fragT, fragS, u0, lip, x_out, st, pr, counter, err};
    if (const char* ov = getenv("HCS_CONVEX_KSKIP")) args.kskip = atoi(ov) != 0;   // A/B experiments
    if (algo == HCS_ADMM) {
      // pixels whose shrinkage is certified zero are solved by the O(N) pass;
      // the slot engine takes the rest from the list (admm_zero_kernel)
      long long* plist = reinterpret_cast<long long*>(lip);   // same offset as fista's Lipschitz array
      unsigned long long* plist_n = reinterpret_cast<unsigned long long*>(ws + 16);
      e = hcs::launch_admm_zero(args, plist, plist_n, sms, stream);
      if (e != cudaSuccess) return cuda_fail(e, "admm_zero_kernel");
      args.plist = plist;
      args.plist_n = plist_n;
    }
    // persistent: one CTA (32 slots) or two CTAs (16 slots each) per SM
    const long long tiles = (P + slots - 1) / slots;
    const long long ctas = (long long)sms * hcs::convex_ctas_per_sm(calgo, Np, M, slots);
    const int grid = (int)(tiles < ctas ? tiles : ctas);
    e = hcs::launch_convex(calgo, args, slots, grid, stream);
    if (e != cudaSuccess) return cuda_fail(e, "convex_kernel");
    return HCS_OK;
  }
  const int kalloc = hcs::greedy_kalloc_host(algo, M, prm->kappa, kGreedySmemCap);
  const size_t smem = hcs::greedy_smem_bytes(algo, M, kalloc);
  int per_sm = hcs::greedy_blocks_per_sm(algo, M, smem);
  if (const char* ov = getenv("HCS_GREEDY_PER_SM")) {   // diagnostics override
    const int v = atoi(ov);
    if (v >= 1 && v < per_sm) per_sm = v;
  }
  if (per_sm < 1) per_sm = 1;
  if (per_sm > kMaxGreedyPerSm) per_sm = kMaxGreedyPerSm;
  long long grid = (long long)sms * per_sm;
  // the CTA scratch slots the workspace holds (sized by hcs_workspace_bytes on
  // the device current at that call): never launch more CTAs than slots
  const GreedyWs gw = greedy_ws(P, N, M, workspace_bytes);
  if (grid > gw.slots) grid = gw.slots;
  double* basis_t = reinterpret_cast<double*>(ws + gw.basis_t);
  long long* spill_list = reinterpret_cast<long long*>(ws + gw.spill);
  double* gscratch = reinterpret_cast<double*>(ws + gw.scratch);
  int* notdct = reinterpret_cast<int*>(ws + 32);   // header word: 0 = DCT-II basis (closed-form CSNE Gram)
  e = hcs::launch_transpose_basis(basis, N, basis_t, notdct, stream);
  if (e != cudaSuccess) return cuda_fail(e, "transpose_basis_kernel");
  hcs::GreedyArgs args{(long long)P, N, M, kalloc, basis, y, mask, x_out, st, pr, counter, err, gscratch, basis_t};
  args.slots = gw.slots;
  args.notdct = notdct;
  if (const char* ov = getenv("HCS_DCT_GRAM")) {   // A/B experiments: 0 = always the DMMA Gram
    if (atoi(ov) == 0) args.notdct = nullptr;
  }
#ifdef HCS_CHECKS
  if (const char* ov = getenv("HCS_CHECK_SELFTEST")) args.selftest = atoi(ov);
#endif
  // gOMP solves by Householder QR (the reference's algorithm): its
  // iteration-2 selections are made on roundoff-level residuals, and CSNE's
  // more accurate solutions shift which noise columns win (2.5x the oracle's
  // 1-ulp tie rate and cube PSNR outside the oracle's 1-ulp band,
  // tools/gomp_rounding_study.py, profiles/gomp_ls_statistics_r02.txt);
  // BIHT / CoSaMP keep the CSNE fast path
  args.ls_mode = algo == HCS_GOMP ? 1 : 0;
  if (const char* ov = getenv("HCS_GREEDY_LS")) args.ls_mode = atoi(ov);   // A/B experiments
  bool warp_path = algo == HCS_GOMP && args.ls_mode == 1 && hcs::gomp_warp_supported(N, M, prm->kappa);
  if (const char* ov = getenv("HCS_GOMP_WARP")) warp_path = warp_path && atoi(ov) != 0;
  if (warp_path) {
    // warp-per-pixel Householder gOMP; the pixels it spills (supports beyond
    // 33 columns, rank guard) are re-solved from scratch by the CTA kernel
    unsigned long long* spill_n = reinterpret_cast<unsigned long long*>(ws + 16);
    e = hcs::launch_gomp_warp(args, hcs::GwSpill{spill_n, spill_list, gscratch, (long long)hcs::greedy_ls_doubles(M)},
                              sms, gw.slots, stream);
    if (e != cudaSuccess) return cuda_fail(e, "gomp_warp_kernel");
    args.counter = reinterpret_cast<unsigned long long*>(ws + 24);
    args.plist = spill_list;
    args.plist_n = spill_n;
  }
  e = hcs::launch_greedy(algo, args, (int)grid, smem, stream);
  if (e != cudaSuccess) return cuda_fail(e, "greedy_kernel");
  return HCS_OK;
}

int hcs_recover_launches(int algo, int32_t N, int32_t M, const hcs_params* prm) {
  if (!prm || algo < HCS_FISTA || algo > HCS_COSAMP) return 0;
  if (algo == HCS_FISTA || algo == HCS_ADMM) return 4;   // mask check + basis prep + (Lipschitz | zero pass) + slot engine
  bool warp_path = algo == HCS_GOMP && hcs::gomp_warp_supported(N, M, prm->kappa);
  if (const char* ov = getenv("HCS_GREEDY_LS")) warp_path = warp_path && atoi(ov) == 1;
  if (const char* ov = getenv("HCS_GOMP_WARP")) warp_path = warp_path && atoi(ov) != 0;
  return warp_path ? 4 : 3;   // mask check + basis transpose + (warp kernel +) CTA kernel
}

int hcs_check_basis(int32_t N, const double* basis, double* max_dev_out, void* stream_) {
  if (N < 1 || N > HCS_MAX_N) return fail(HCS_EINVAL, "N must be in [1, 256]");
  if (!basis || !max_dev_out) return fail(HCS_EINVAL, "null array");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return cuda_fail(e, "check_basis alloc");
  unsigned long long h = 0;
  e = cudaMemsetAsync(d, 0, sizeof(unsigned long long), stream);
  if (e == cudaSuccess) e = hcs::launch_basis_gram_dev(N, basis, d, stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, stream);
  cudaFreeAsync(d, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return cuda_fail(e, "check_basis");
  double dev;
  memcpy(&dev, &h, sizeof(dev));
  *max_dev_out = dev;
  return HCS_OK;
}

int hcs_recover_status(const void* workspace, void* stream_) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  int flag = 0;
  cudaError_t e = cudaMemcpyAsync(&flag, static_cast<const unsigned char*>(workspace) + 8, sizeof(int),
                                  cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  if (e != cudaSuccess) return cuda_fail(e, "status");
  if (flag & hcs::kErrMask) return fail(HCS_EINVAL, "mask entries must be strictly increasing band indices < N");
  if (flag & hcs::kErrCheck) {   // bounds-checked builds only
    int line = 0;
    cudaMemcpy(&line, static_cast<const unsigned char*>(workspace) + 48, sizeof(int), cudaMemcpyDeviceToHost);
    return fail(HCS_ECUDA, "device bounds check failed (source line " + std::to_string(line) +
                               "; 1 = shared-memory canary)");
  }
  if (flag) return fail(HCS_ENONFINITE, "array must not contain infs or NaNs");
  return HCS_OK;
}

int hcs_soft_threshold(int64_t n, const double* v, double t, double* out, void* stream) {
  if (t < 0) return fail(HCS_EINVAL, "threshold must be >= 0");
  if (n < 0) return fail(HCS_EINVAL, "negative length");
  if (n == 0) return HCS_OK;
  cudaError_t e = hcs::launch_soft(n, v, t, out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? HCS_OK : cuda_fail(e, "soft_threshold");
}

int hcs_argmax_k(int64_t P, int32_t n, const double* v, int32_t k, int32_t* idx_out, void* stream) {
  if (n < 1 || n > HCS_MAX_N) return fail(HCS_EINVAL, "n must be in [1, 256]");
  if (k < 1 || k > n) return fail(HCS_EINVAL, "k must be in [1, " + std::to_string(n) + "], got " + std::to_string(k));
  if (P <= 0) return HCS_OK;
  cudaError_t e = hcs::launch_argmax_k(P, n, v, k, idx_out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? HCS_OK : cuda_fail(e, "argmax_k");
}

int hcs_least_squares(int64_t P, int32_t M, int32_t K, const double* b, const double* y, double* s_out,
                      int32_t* path_out, void* stream) {
  if (M < 1 || K < 1 || M > HCS_MAX_N || K > HCS_MAX_N) return fail(HCS_EINVAL, "M and K must be in [1, 256]");
  if (P <= 0) return HCS_OK;
  cudaError_t e = hcs::launch_batched_ls(P, M, K, b, y, s_out, path_out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? HCS_OK : cuda_fail(e, "least_squares");
}

int hcs_residual_delta(int64_t P, int32_t n, const double* r, const double* r_prev, double* out, void* stream) {
  if (n < 1) return fail(HCS_EINVAL, "n must be >= 1");
  if (P <= 0) return HCS_OK;
  cudaError_t e = hcs::launch_rdelta(P, n, r, r_prev, out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? HCS_OK : cuda_fail(e, "residual_delta");
}

int hcs_lipschitz(int64_t P, int32_t N, int32_t M, const double* basis, const uint8_t* mask, double* out,
                  void* stream) {
  if (N < 1 || N > HCS_MAX_N || M < 1 || M > N) return fail(HCS_EINVAL, "bad N/M");
  if (P <= 0) return HCS_OK;
  cudaError_t e = hcs::launch_lipschitz(P, N, M, basis, mask, out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? HCS_OK : cuda_fail(e, "lipschitz");
}

int hcs_psnr_partials(int64_t P, int32_t N, const double* ref, const double* x, const double* basis, double* sse_out,
                      double* absmax_out, void* stream) {
  if (N < 1 || N > HCS_MAX_N) return fail(HCS_EINVAL, "N must be in [1, 256]");
  if (P <= 0) return HCS_OK;
  cudaError_t e = hcs::launch_psnr(P, N, ref, x, basis, sse_out, absmax_out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? HCS_OK : cuda_fail(e, "psnr_partials");
}

int hcs_sse_coeff_partials(int64_t P, int32_t N, const double* ref_coeffs, const double* x, double* sse_out,
                           void* stream) {
  if (P < 0) return fail(HCS_EINVAL, "negative pixel count");
  if (N < 1 || N > HCS_MAX_N) return fail(HCS_EINVAL, "N must be in [1, 256]");
  if (P == 0) return HCS_OK;
  if (!ref_coeffs || !x || !sse_out) return fail(HCS_EINVAL, "null array");
  cudaError_t e = hcs::launch_sse_coeff(P * (long long)N, ref_coeffs, x, sse_out, num_sms(),
                                        static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? HCS_OK : cuda_fail(e, "sse_coeff_partials");
}

int hcs_synth_spectra(int64_t P, int32_t N, const double* centres, const double* widths, const double* amps,
                      const double* noise, double* f_out, void* stream) {
  if (P < 0) return fail(HCS_EINVAL, "negative pixel count");
  if (N < 1 || N > HCS_MAX_N) return fail(HCS_EINVAL, "N must be in [1, 256]");
  if (P == 0) return HCS_OK;
  if (!centres || !widths || !amps || !noise || !f_out) return fail(HCS_EINVAL, "null array");
  cudaError_t e = hcs::launch_synth_spectra(P, N, centres, widths, amps, noise, f_out, num_sms(),
                                            static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? HCS_OK : cuda_fail(e, "synth_spectra");
}

int hcs_sparsify_measure(int64_t P, int32_t N, int32_t M, const double* basis, const double* f, int32_t rule,
                         double factor, const double* keys, uint8_t* mask, double* coeffs_out, double* spectra_out,
                         double* y_out, uint64_t* nzero_out, void* stream) {
  if (P < 0) return fail(HCS_EINVAL, "negative pixel count");
  if (N < 1 || N > HCS_MAX_N) return fail(HCS_EINVAL, "N must be in [1, 256]");
  if (M < 1 || M > N) return fail(HCS_EINVAL, "M must be in [1, N]");
  if (rule != HCS_SPARSIFY_MAXREL && rule != HCS_SPARSIFY_MEANSTD) return fail(HCS_EINVAL, "unknown threshold rule");
  if (!(factor >= 0)) return fail(HCS_EINVAL, "threshold factor must be >= 0");   // transform.py:85-86
  if (P == 0) return HCS_OK;
  if (!basis || !f || !mask || !y_out) return fail(HCS_EINVAL, "null array");
  cudaError_t e = hcs::launch_sparsify_measure(P, N, M, rule, factor, basis, f, keys, mask, coeffs_out, spectra_out,
                                               y_out, reinterpret_cast<unsigned long long*>(nzero_out), num_sms(),
                                               static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? HCS_OK : cuda_fail(e, "sparsify_measure");
}

}  // extern "C"
