// hcs_internal.cuh -- argument blocks and launchers shared by the translation
// units of libhypercs_b200.so (not part of the public C ABI).
#pragma once
#include "hcs_common.cuh"

namespace hcs {

enum { kFista = 0, kAdmm = 1, kGomp = 2, kBiht = 3, kCosamp = 4 };

struct ConvexArgs {
  long long P;
  int N, Np, M;
  const double* y;
  const uint8_t* mask;
  const double* fragT;    // Psi^T (analysis) in fragment order
  const double* fragS;    // Psi (synthesis) in fragment order
  const double* u0;       // Psi * (1/sqrt(N)) 1, for the Lipschitz constant
  double* lip;            // (P,) per-pixel Lipschitz constants (fista; lipschitz_prepass)
  double* x_out;
  Stats st;
  Params prm;
  unsigned long long* counter;
  int* err;
  // optional pixel list (the ADMM pixels the zero-shrinkage pass could not
  // certify): the engine works on plist[0 .. *plist_n) instead of 0 .. P-1
  const long long* plist = nullptr;
  const unsigned long long* plist_n = nullptr;
  int kskip = 1;          // fista: skip the all-zero k-steps of Psi x_{k+1} (bitwise-identical)
  unsigned smem_bytes = 0;   // dynamic shared bytes of the layout (checked builds: poison / canary)
};

struct GreedyArgs {
  long long P;
  int N, M, kalloc;      // kalloc: LS columns the shared-memory region holds
  const double* basis;   // Psi, N x N row-major
  const double* y;
  const uint8_t* mask;
  double* x_out;
  Stats st;
  Params prm;
  unsigned long long* counter;
  int* err;
  double* gscratch;      // per-CTA global LS scratch (systems beyond the shared-memory size)
  const double* basis_t;   // Psi transposed (basis_t[c N + r] = Psi[r][c]): column gathers read one column
  // least-squares method: 0 = CSNE fast path with the guarded pivoted-QR
  // fallback; 1 = pivoted Householder QR always (LAPACK dlaqp2 restatement,
  // the reference's own algorithm: its rounding statistics decide gOMP's
  // noise-level selections, tools/gomp_rounding_study.py)
  int ls_mode = 0;
  // optional pixel list (the pixels the warp-per-pixel gOMP kernel spilled):
  // the CTA kernel then works on plist[0 .. *plist_n) instead of 0 .. P-1
  const long long* plist = nullptr;
  const unsigned long long* plist_n = nullptr;
  unsigned smem_bytes = 0;   // dynamic shared bytes of the layout (checked builds: poison / canary)
  long long slots = 0;       // CTA scratch slots in gscratch
  int selftest = 0;          // checked builds: 1 = deliberately overrun the shared region (positive control)
  // *notdct == 0: the basis is the orthonormal DCT-II (checked by transpose_basis_kernel), so the CSNE
  // Gram takes the closed form of hcs_ls_csne.cuh (DctGram); nullptr: never
  const int* notdct = nullptr;
};

// spill list of the warp-per-pixel gOMP kernel
struct GwSpill {
  unsigned long long* count;
  long long* list;
  double* pre;            // per-warp pre-column scratch (the CTA scratch slots)
  long long pre_stride;   // doubles per slot
};

// hcs_convex.cu
cudaError_t launch_convex(int algo, const ConvexArgs& args, int slots, int grid, cudaStream_t stream);
size_t convex_smem_bytes(int algo, int Np, int M, int slots);
cudaError_t launch_admm_zero(const ConvexArgs& args, long long* plist, unsigned long long* plist_n, int sms,
                             cudaStream_t stream);
int convex_slots(int algo, int Np, int M);
int convex_ctas_per_sm(int algo, int Np, int M, int slots);
cudaError_t launch_lipschitz_prepass(long long P, int M, const uint8_t* mask, const double* u0, double* lip,
                                     const int* err, int sms, cudaStream_t stream);
cudaError_t launch_prep_basis(const double* basis, int N, int Np, double* fragS, double* fragT, double* u0,
                              int slots, cudaStream_t stream);
// hcs_greedy.cu
cudaError_t launch_greedy(int algo, const GreedyArgs& args, int grid, size_t smem, cudaStream_t stream);
size_t greedy_smem_bytes(int algo, int M, int kalloc);
int greedy_kalloc_host(int algo, int M, int kappa, size_t smem_cap);
size_t greedy_ls_doubles(int M);
cudaError_t launch_transpose_basis(const double* basis, int N, double* bt, int* notdct, cudaStream_t stream);
int greedy_blocks_per_sm(int algo, int M, size_t smem);
// hcs_gomp_warp.cu
bool gomp_warp_supported(int N, int M, int kappa);
cudaError_t launch_gomp_warp(const GreedyArgs& args, const GwSpill& sp, int sms, long long slots,
                             cudaStream_t stream);
// hcs_batched.cu
cudaError_t launch_basis_gram_dev(int N, const double* basis, unsigned long long* out, cudaStream_t stream);
cudaError_t launch_validate_masks(long long P, int M, int N, const uint8_t* mask, int* err, int sms,
                                  cudaStream_t stream);
cudaError_t launch_batched_ls(long long P, int M, int K, const double* b, const double* y, double* s,
                              int32_t* path, cudaStream_t stream);
cudaError_t launch_argmax_k(long long P, int n, const double* v, int k, int32_t* idx, cudaStream_t stream);
cudaError_t launch_soft(long long n, const double* v, double t, double* out, cudaStream_t stream);
cudaError_t launch_rdelta(long long P, int n, const double* r, const double* rp, double* out, cudaStream_t stream);
cudaError_t launch_lipschitz(long long P, int N, int M, const double* basis, const uint8_t* mask, double* out,
                             cudaStream_t stream);
cudaError_t launch_psnr(long long P, int N, const double* ref, const double* x, const double* basis, double* sse,
                        double* amax, cudaStream_t stream);
cudaError_t launch_sse_coeff(long long n, const double* a, const double* b, double* sse, int sms,
                             cudaStream_t stream);

// hcs_input.cu
cudaError_t launch_synth_spectra(long long P, int N, const double* centres, const double* widths, const double* amps,
                                 const double* noise, double* f, int sms, cudaStream_t stream);
cudaError_t launch_sparsify_measure(long long P, int N, int M, int rule, double factor, const double* basis,
                                    const double* f, const double* keys, uint8_t* mask, double* coeffs,
                                    double* spectra, double* y, unsigned long long* nzero, int sms,
                                    cudaStream_t stream);

}  // namespace hcs
