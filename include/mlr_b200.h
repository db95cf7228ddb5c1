/*
 * mlr_b200.h — C ABI of the B200-native multilevel PCP / CPCP hot path.
 *
 * The reference (mlrpca 0.1.0, pure Python) has no FFI: its boundary is the
 * Python API ml_ialm_solve / ml_fwt_solve.  This library exports the
 * per-iteration steps of those two loops as plain-C entry points over
 * caller-owned device buffers (the host loop in
 * paper_2206_13369_b200/pcp.py / cpcp.py binds them with ctypes; any other
 * FFI can bind them the same way — see INTEGRATION.md).
 *
 * Conventions
 *   - every function returns 0 on success, MLR_ERR_* otherwise; the message
 *     is available from mlr_last_error() (thread-local);
 *   - matrices are row-major with an explicit leading dimension (elements);
 *   - `f32` selects float storage/compute of the fine planes (1) or double (0);
 *   - `stream` is a cudaStream_t (NULL = legacy default stream); all calls
 *     are stream-ordered and return after enqueue, except *_state / *_history
 *     / *_lanczos_state which synchronise the stream and copy to host;
 *   - plans live in caller-provided device workspace of *_workspace_bytes();
 *     the library allocates only the small chain tables (mlr_chain_create).
 *
 * Reference interfaces replaced (paths under pkg/src/mlrpca/):
 *   mlr_chain_create      multilevel.build_chain + RestrictionChain.gram_cho
 *                         (multilevel.py:125-179, 97-102) — stencil upload
 *   mlr_restrict          multilevel.restrict (multilevel.py:212-219)
 *   mlr_prolong           multilevel.prolong  (multilevel.py:238-245)
 *   mlr_eigh_psd          the SVD inside svd_full (linalg.py:86-99) as used by
 *                         the SVT step (pcp.py:257-267), via Jacobi on M^T M
 *   mlr_pcp_*             pcp.ml_ialm_solve loop (pcp.py:213-309) incl. the
 *                         sigma_1 / dual init (pcp.py:95-115)
 *   mlr_cpcp_*            cpcp.ml_fwt_solve / _run_fwt (cpcp.py:326-515)
 */
#ifndef MLR_B200_H
#define MLR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MLR_OK 0
#define MLR_ERR_ARG 1
#define MLR_ERR_CUDA 2

int mlr_version(void);
const char* mlr_last_error(void);
int mlr_device_count(void);

/* ---------------------------------------------------------------- chain
 * Composite restriction R (n x nh) as a 2-tap stencil: fine column j has
 * weight w0[j] on coarse column c0[j] and w1[j] on c0[j]+1.  g_diag/g_off
 * are the tridiagonal of G_R = R^T R.  Host arrays; copied to the current
 * device. */
int mlr_chain_create(int n, int nh, const int32_t* c0, const double* w0, const double* w1, const double* g_diag,
                     const double* g_off, void** chain_out);
int mlr_chain_destroy(void* chain);
int mlr_chain_padded_width(void* chain); /* np = nh rounded up to 64 */

/* out (m x np, row-major, ld np) = X (m x n, ld ldx) R */
int mlr_restrict(void* chain, int64_t m, int f32, const void* X, int64_t ldx, void* out, void* stream);
/* out (m x n, ld ldo) = XH (m x np, ld np) R^T */
int mlr_prolong(void* chain, int64_t m, int f32, const void* XH, void* out, int64_t ldo, void* stream);

/* out3 = (||X||_F^2 over finite entries, max|X|, #non-finite entries) — the
 * as_matrix finiteness check (linalg.py:48-57) plus the norms the solvers
 * need; work holds mlr_matrix_stats_work_doubles() doubles. */
int64_t mlr_matrix_stats_work_doubles(void);
int mlr_matrix_stats(int64_t m, int n, int f32, const void* X, int64_t ldx, double* out3, double* work,
                     void* stream);

/* Eigen-decomposition of a symmetric PSD np x np matrix B (np % 64 == 0,
 * FP64, row-major) by one-sided block Jacobi; V (np x np) receives the
 * eigenvectors (columns), lam (np) the eigenvalues (unsorted).  work must
 * hold mlr_eigh_work_doubles(np) doubles.  info[0] = sweeps (>0 converged,
 * <=0 not converged). Synchronous. */
int64_t mlr_eigh_work_doubles(int np);
int mlr_eigh_psd(int np, const double* B, double* V, double* lam, double tol, int max_sweeps, double* work,
                 int* info, void* stream);

/* ---------------------------------------------------------------- ML-PCP */
int64_t mlr_pcp_workspace_bytes(void* chain, int64_t m_local, int f32, int max_iters);
int mlr_pcp_create(void* chain, int64_t m_local, int64_t m_global, int f32, int max_iters, void* workspace,
                   void** plan_out);
int mlr_pcp_destroy(void* plan);
int64_t mlr_pcp_red_doubles(void* plan); /* size of the all-reduce buffer */
int mlr_pcp_input_stats(void* plan, const void* D, int64_t ldd, double* out2, void* stream);
int mlr_pcp_lanczos_init(void* plan, void* stream);
int mlr_pcp_lanczos_matvec(void* plan, const void* D, int64_t ldd, double* w_part, void* stream);
int mlr_pcp_lanczos_update(void* plan, const double* w_reduced, double tol, void* stream);
int mlr_pcp_lanczos_state(void* plan, double* out4, void* stream); /* k, done, sigma1, theta */
int mlr_pcp_start(void* plan, const void* D, int64_t ldd, void* Y0, int64_t ldy, const double* in_stats, double lam,
                  double mu0, double rho, double tol, int max_iters, double time_budget, double jac_tol,
                  int jac_max_sweeps, void* stream);
int mlr_pcp_gram(void* plan, double* red, int with_stats, void* stream);
int mlr_pcp_finalize(void* plan, const double* red, void* stream);
int mlr_pcp_svt(void* plan, const double* red, void* stream);
int mlr_pcp_update(void* plan, const void* D, int64_t ldd, const void* Y_in, void* Y_out, int64_t ldy, void* stream);
int mlr_pcp_outputs(void* plan, const void* D, int64_t ldd, const void* Y_prev, int64_t ldy, void* L, void* S,
                    int64_t ldo, void* stream);
/* out16: k, done, status, rank, mu, mu_final, mu_last, nuclear, sigma1, d_norm, jac_sweeps, tau, scale, lam, 0, 0 */
int mlr_pcp_state(void* plan, double* out16, void* stream);
int mlr_pcp_history(void* plan, int count, double* out, void* stream); /* count x 8 */
/* Per-phase CUDA-event timing: phases gram, pre (B, X=BV), jacobi, post
 * (weights, P, W~), recon (Z = A W~), update (fused fine pass), finalize,
 * lanczos (sigma_1 estimate).  mlr_pcp_timing synchronises, returns total ms
 * and launch counts per phase (8 entries each) and resets the accumulators. */
/* Truncated SVT of the full-width baseline ialm_solve (reference pcp.py:118-197,
 * svd_truncated linalg.py:102-125): with sv0 > 0 only the top-sv singular values
 * of each iteration take part and sv adapts (pcp.py:160-165), capped at cap.
 * Call before mlr_pcp_start; sv0 = 0 restores the full SVT. */
int mlr_pcp_set_truncation(void* plan, int sv0, int cap);
int mlr_pcp_set_timing(void* plan, int enable);
int mlr_pcp_timing(void* plan, double* ms8, int* counts8);

/* ---------------------------------------------------------------- ML-CPCP
 * mask: bit-packed observation pattern, uint32 words, ldm words per row,
 * bit (j & 31) of word j >> 5; NULL = fully observed. */
int64_t mlr_cpcp_workspace_bytes(void* chain, int64_t m_local, int f32, int max_iters);
int mlr_cpcp_create(void* chain, int64_t m_local, int64_t m_global, int64_t row0, int f32, int max_iters, int world,
                    void* workspace, void** plan_out);
int mlr_cpcp_destroy(void* plan);
int64_t mlr_cpcp_red_doubles(void* plan);
int mlr_cpcp_start(void* plan, const void* D, int64_t ldd, const uint32_t* mask, int64_t ldm, void* S, int64_t lds,
                   double lambda_l, double lambda_s, double tol, double radius, int max_iters, double time_budget,
                   void* stream);
int mlr_cpcp_gram(void* plan, double* red, double* amax, void* stream);
int mlr_cpcp_begin(void* plan, const double* red, const double* amax_all, void* stream);
int mlr_cpcp_lmo(void* plan, const double* red, const double* amax_all, double* dots, void* stream);
int mlr_cpcp_update(void* plan, const void* D, int64_t ldd, const uint32_t* mask, int64_t ldm, void* S, int64_t lds,
                    const double* dots, void* stream);
int mlr_cpcp_finalize(void* plan, const double* red, void* stream);
int mlr_cpcp_outputs(void* plan, void* L, int64_t ldl, void* stream);
/* out32: k, done, status, t_l, t_s, u_l, u_s, sigma, passes, ga, gb, corner_l, corner_s, i_s, j_s, s2, ... */
int mlr_cpcp_state(void* plan, double* out32, void* stream);
int mlr_cpcp_history(void* plan, int count, double* out, double* objectives, void* stream); /* count x 8, count */
/* Per-phase CUDA-event timing (8 slots: gram, power, dots, qp, -, update, finalize, -). */
int mlr_cpcp_set_timing(void* plan, int enable);
int mlr_cpcp_timing(void* plan, double* ms8, int* counts8);

#ifdef __cplusplus
}
#endif
#endif /* MLR_B200_H */
