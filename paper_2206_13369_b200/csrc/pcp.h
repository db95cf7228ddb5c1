// Device state and plan for ML-PCP.
#pragma once
#include <utility>
#include <vector>

#include "kernels.h"

namespace mlr {

constexpr int kHistCols = 8;  // gap, objective, rank, sparsity, wall, mu, jacobi sweeps, nnz

// Device-resident solver state (one instance in device memory per plan).
struct PcpDev {
  double lam, rho, tol, d_norm, sigma1, scale;
  double mu;        // mu_k of the current iteration
  double tau;       // 1/mu_k
  double mu_last;   // mu of the last finalized iteration
  double mu_final;  // mu after the final `mu *= rho` (reference PcpState.mu)
  double nuclear;   // sum(sigma - tau)+ of the current SVT
  double time_budget;
  double jac_tol;
  double t0_ns;
  double m_global, n;
  int k;            // current iteration (1-based)
  int done;         // 0 running, 1 converged, 2 stopped, 3 error
  int status;       // 0 ok, 3 Jacobi did not converge
  int rank;
  int max_iters;
  int jac_sweeps;
  int trunc, sv, sv_cap;  // ialm_solve: keep only the top-sv triplets, adapt sv (pcp.py:157-165)
  int jac_skip;     // Jacobi not needed this iteration: done, or rank 0 certified (pcp_rank0_test)
  int r0_state;     // rank-0 test: 0 undecided, 1 rank > 0 (diagonal), 2 certified (power bound), 3 done
  int eig_skip;     // trd path: the Jacobi fallback is not needed (trd solved it, or jac_skip)
  int trd_ok;       // trd path: this iteration's eigenpairs came from the tridiagonal solver
};

struct LanczosDev {
  int k, done, kmax, stable;
  double theta, theta_prev, sigma1;
  double alpha[512];
  double beta[512];
};

// Scratch of the tridiagonal coarse eigensolver (trd.cu)
struct TrdBuf {
  double* hv;     // n x ldh (ldh = n rounded up to even): row j = Householder vector v_j (entries j+1..n-1)
  double* z;      // n x n: eigenvectors of T, vector c at z[c * n + i]
  double *beta, *dd, *ee, *lam;  // n each: reflector scalars, diag / off-diag of T, eigenvalues (descending)
  uint4 *pll, *rowll;            // flag-carrying publication buffers (2 x n each): p by step parity, rows by row parity
  uint4* sent;                   // per-CTA and row sentinels, one 128-byte line each
  double* scale;                 // power-of-two scale of T used by the bisection / vectors
  int* info;                     // [0] = k (eigenvalues above tau^2), [1] = failure, [2] = V columns in use
};

struct PcpPlan {
  PhaseTimer timer;
  ChainDev ch;
  bool f32;
  int64_t m_local, m_global;
  int max_iters;
  int row_blocks, gram_splits, lz_splits, lz_kmax;
  int lz_fused_ctas;  // > 0: one-pass D^T D q (n <= 2048)
  int lz_long_clusters;  // > 0: one-pass D^T D q for long FP32 rows (2-CTA clusters, TMA-staged rows)
  int coarse_ksplit;  // split-K of the n_p^3 coarse products (<= gram_splits)
  int lz_run_ctas;    // > 0: the whole Lanczos run in one cooperative kernel (one rank, n <= 4096)
  int eig_sort;       // sort the eigenpairs after each Jacobi (warm start of the next)
  int trd_on;         // coarse eigensolver: tridiagonal (trd.cu) with the Jacobi as fallback
  TrdBuf trd;
  double* lzRed;      // lz_run_ctas x (2 (kmax + 1) + 4) dot partials
  double jac_tol_host;
  double jac_floor_rel;
  int jac_max_sweeps;
  int trunc_sv0, trunc_cap;  // > 0: truncated SVT (full-width ialm_solve)
  // device buffers (carved from the caller's workspace)
  PcpDev* dev;
  LanczosDev* lz;
  double* hist;        // [max_iters][kHistCols]
  void* A;             // m_local x np (T)
  void* Z;             // m_local x np (T)
  double* gram_part;   // gram_splits x np x np
  double* row_part;    // row_blocks x 4
  double *T1, *Bm, *Xm, *Vm, *Wm;   // np x np: U, T, B~ (Jacobi), V (eigenvectors), W~ (W~^T on the tcgen05 path)
  bool tc_recon;                    // FP32: Z = A W~ by the 3xTF32 tcgen05 kernel (tc_gemm.cu)
  float *w_hi, *w_lo;               // np x np: TF32 hi / lo parts of W~^T
  TcRecon tc;
  double* qbuf;        // Jacobi per-pair rotations
  int* qflag;
  double *sig, *fw;    // np
  double* jac_off;     // 2
  int* jac_result;     // 4
  double *lzQ, *lzT, *lzW, *lzWork;
};

int trd_max_n();
bool trd_supported(int n);
size_t trd_bytes(int n);
void trd_carve(TrdBuf* b, char* base, int n);
int trd_eig(PcpDev* st, TrdBuf* b, double* Bm, double* V, int n, int np, const double* tau, const int* skip,
            cudaStream_t s);

int pcp_input_stats(PcpPlan* p, const void* D, int64_t ldd, double* out2, cudaStream_t st);
int matrix_stats(int64_t m, int n, bool f32, const void* D, int64_t ldd, double* part, int blocks, double* out3,
                 cudaStream_t st);
int pcp_lanczos_init(PcpPlan* p, cudaStream_t st);
int pcp_lanczos_matvec(PcpPlan* p, const void* D, int64_t ldd, double* wpart_out, cudaStream_t st);
int pcp_lanczos_update(PcpPlan* p, const double* w_reduced, double tol, cudaStream_t st);
int pcp_lanczos_run(PcpPlan* p, const void* D, int64_t ldd, double tol, cudaStream_t st);
int lanczos_run_ok(const PcpPlan* p);
int pcp_start(PcpPlan* p, const void* D, int64_t ldd, void* Y0, int64_t ldy, const double* in_stats, double lam,
              double mu0, double rho, double tol, int max_iters, double time_budget, double jac_tol,
              cudaStream_t st);
int pcp_gram(PcpPlan* p, double* red, int with_stats, cudaStream_t st);
int pcp_finalize(PcpPlan* p, const double* red, cudaStream_t st);
int pcp_svt(PcpPlan* p, const double* red, cudaStream_t st);
int pcp_update(PcpPlan* p, const void* D, int64_t ldd, const void* Yin, void* Yout, int64_t ldy, cudaStream_t st);
int pcp_outputs(PcpPlan* p, const void* D, int64_t ldd, const void* Yprev, int64_t ldy, void* L, void* S, int64_t ldo,
                cudaStream_t st);

}  // namespace mlr
