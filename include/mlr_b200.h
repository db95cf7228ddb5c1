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
 *                         sigma_1 / dual init (pcp.py:95-115); the coarse SVT
 *                         (pcp.py:257-267) inside mlr_pcp_svt runs a
 *                         tridiagonal eigensolver on M^T M (Householder
 *                         reduction, Sturm bisection, twisted-factorisation
 *                         vectors) with the block Jacobi as fallback
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

/* ---------------------------------------------------------------- NCCL
 * Communicator of the row-sharded solvers (the reference is
 * single-process and has no counterpart).  One rank per GPU: rank 0 calls
 * mlr_comm_unique_id, the 128-byte id is exchanged once out of band, every
 * rank calls mlr_comm_create.  The host loops then all-reduce the plan's
 * red buffer (mlr_pcp_gram / mlr_cpcp_gram layouts), all-gather the CPCP
 * arg-max records and all-reduce the QP dots / Lanczos vectors on the
 * plan's stream.  NCCL is dlopen'd at the first call (mlr_comm_available()
 * reports whether it could be).  dtype: 8 = float64, 4 = int64; op: 0 = sum,
 * 2 = max (NCCL's enum values). */
int mlr_comm_available(void);
int mlr_comm_unique_id(void* out128);
int mlr_comm_create(const void* id128, int nranks, int rank, int device, void** comm_out);
int mlr_comm_destroy(void* comm);
int mlr_comm_allreduce(void* comm, void* buf, int64_t count, int dtype, int op, void* stream);
int mlr_comm_allgather(void* comm, const void* in, void* out, int64_t count, int dtype, void* stream);
int mlr_comm_rank(void* comm);
int mlr_comm_size(void* comm);

/* ---------------------------------------------------------------- box QP
 * Test entry of the device box QP of every FW-T step (_solve_box_qp and
 * _coord_min, cpcp.py:195-231, evaluated in the reference's operation order):
 * for i < count, (out2[2i], out2[2i+1]) = (ga, gb) of in6[6i..6i+5] =
 * (aa, bb, ab, la, lb, fallback_gamma; NaN = None).  Device pointers. */
int mlr_box_qp_batch(const double* in6, double* out2, int count, void* stream);

/* ---------------------------------------------------------------- tensor cores
 * Test entry of the reconstruction kernel FP32 plans use for Z = A W~ (the
 * L_H = U_r diag(sigma_r - tau) V_r^T step, pcp.py:258-266): 3xTF32
 * tcgen05.mma with TMEM accumulators and TMA operand loads (tc_gemm.cu).
 * Z (m x np FP32, ld np) = A (m x np FP32, ld np) W (np x np FP64, row-major);
 * np % 64 == 0; work: np^2 doubles + 2 np^2 floats.  Synchronous. */
int mlr_tc_gemm_tf32x3(int64_t m, int np, const float* A, const double* W, float* Z, void* work, void* stream);

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
/* One rank: the whole Lanczos run (init state from mlr_pcp_lanczos_init) in one
 * cooperative launch, same steps and stopping rule as the matvec/update loop;
 * available when mlr_pcp_lanczos_run_available(plan) (n <= 4096). */
int mlr_pcp_lanczos_run(void* plan, const void* D, int64_t ldd, double tol, void* stream);
int mlr_pcp_lanczos_run_available(void* plan);
int mlr_pcp_start(void* plan, const void* D, int64_t ldd, void* Y0, int64_t ldy, const double* in_stats, double lam,
                  double mu0, double rho, double tol, int max_iters, double time_budget, double jac_tol,
                  int jac_max_sweeps, void* stream);
/* time_budget < 0 means none (reference None); 0 or more stops after the first
 * iteration whose wall time reaches it (pcp.py:295).
 * red layout after mlr_pcp_gram: [K = A^T A (n_p^2), res^2, sum|S|, nnz(S), budget
 * flag]; row-sharded runs all-reduce (sum) red[0 : n_p^2 + 4) before
 * mlr_pcp_finalize, so every rank takes the same time-budget decision. */
int mlr_pcp_gram(void* plan, double* red, int with_stats, void* stream);
int mlr_pcp_finalize(void* plan, const double* red, void* stream);
int mlr_pcp_svt(void* plan, const double* red, void* stream);
int mlr_pcp_update(void* plan, const void* D, int64_t ldd, const void* Y_in, void* Y_out, int64_t ldy, void* stream);
int mlr_pcp_outputs(void* plan, const void* D, int64_t ldd, const void* Y_prev, int64_t ldy, void* L, void* S,
                    int64_t ldo, void* stream);
/* out16: k, done, status, rank, mu, mu_final, mu_last, nuclear, sigma1, d_norm, jac_sweeps, tau, scale, lam, 0, 0
 * (jac_sweeps: Jacobi sweeps of the latest eigensolve, 0 when none ran, -1 when the tridiagonal solver ran) */
int mlr_pcp_state(void* plan, double* out16, void* stream);
/* Pipelined polling: mlr_pcp_snapshot enqueues an asynchronous copy of the
 * plan's device state (solver + Lanczos) into `host` (pinned, at least
 * mlr_pcp_snapshot_bytes()) and returns at once; after the caller has waited on
 * an event recorded behind it, mlr_pcp_snapshot_read decodes it into the
 * mlr_pcp_state / mlr_pcp_lanczos_state layouts (either output may be NULL).
 * The host can keep the next batch of steps queued while it waits. */
int64_t mlr_pcp_snapshot_bytes(void);
int mlr_pcp_snapshot(void* plan, void* host, void* stream);
int mlr_pcp_snapshot_read(const void* host, double* out16, double* lz4);
int mlr_pcp_history(void* plan, int count, double* out, void* stream); /* count x 8 */
/* Truncated SVT of the full-width baseline ialm_solve (reference pcp.py:118-197,
 * svd_truncated linalg.py:102-125): with sv0 > 0 only the top-sv singular values
 * of each iteration take part and sv adapts (pcp.py:160-165), capped at cap.
 * Call before mlr_pcp_start; sv0 = 0 restores the full SVT. */
int mlr_pcp_set_truncation(void* plan, int sv0, int cap);
/* Per-phase CUDA-event timing: phases gram, pre (B, X=BV), jacobi (the coarse eigensolve: tridiagonal or Jacobi, incl. the rank-0 certificate), post
 * (weights, P, W~), recon (Z = A W~), update (fused fine pass), finalize,
 * lanczos (sigma_1 estimate).  mlr_pcp_timing synchronises, returns total ms
 * and launch counts per phase (8 entries each) and resets the accumulators. */
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
/* time_budget < 0 means none (cpcp.py:451).  red layout after mlr_cpcp_gram:
 * [K_g (n_p^2), sum r^2, sum|S|, nnz, sum S^2, sum S r, budget flag];
 * all-reduce (sum) red[0 : n_p^2 + 6) across ranks. */
int mlr_cpcp_gram(void* plan, double* red, double* amax, void* stream);
int mlr_cpcp_begin(void* plan, const double* red, const double* amax_all, void* stream);
int mlr_cpcp_lmo(void* plan, const double* red, const double* amax_all, double* dots, void* stream);
int mlr_cpcp_update(void* plan, const void* D, int64_t ldd, const uint32_t* mask, int64_t ldm, void* S, int64_t lds,
                    const double* dots, void* stream);
int mlr_cpcp_finalize(void* plan, const double* red, void* stream);
int mlr_cpcp_outputs(void* plan, void* L, int64_t ldl, void* stream);
/* out32: k, done, status, t_l, t_s, u_l, u_s, sigma, passes, ga, gb, corner_l, corner_s, i_s, j_s, s2, ... */
int mlr_cpcp_state(void* plan, double* out32, void* stream);
/* pipelined polling, as mlr_pcp_snapshot / mlr_pcp_snapshot_read */
int64_t mlr_cpcp_snapshot_bytes(void);
int mlr_cpcp_snapshot(void* plan, void* host, void* stream);
int mlr_cpcp_snapshot_read(const void* host, double* out32);
int mlr_cpcp_history(void* plan, int count, double* out, double* objectives, void* stream); /* count x 8, count */
/* Per-phase CUDA-event timing (8 slots: gram, power, dots, qp, -, update, finalize, -). */
int mlr_cpcp_set_timing(void* plan, int enable);
int mlr_cpcp_timing(void* plan, double* ms8, int* counts8);

/* ---------------------------------------------------------------- telemetry
 * Numerical-rank telemetry of the reference (collect_rank, cpcp.py:434-439;
 * collect_diagnostics, pcp.py:298-306 with epsilon_bound multilevel.py:248-265).
 *
 * Spectrum plan: singular values of a row-sharded X (m_local x n, T = f32 ? float
 * : double), or of X C for a fixed n x n double factor C (NULL = identity), in two
 * passes accurate to ~eps * sigma_1 (one Gram eigensolve resolves only
 * ~sqrt(eps) * sigma_1, far above the reference's max(m, n) * eps threshold):
 *   gram   red  = X^T X (this rank's rows)              [allreduce red]
 *   rotate V1 = eig(C^T red C) (warm-started); B = X C V1; red2 = B^T B  [allreduce red2]
 *   finish sigma = sqrt(eig(red2)) sorted descending; rank = #{sigma > sigma_1 * rel};
 *          wsum = sum_{k < rank} sigma_k * pair_w[k] (pair_w may be NULL)
 * skip: optional device int; every step is a no-op while it is nonzero.
 * red / red2 hold mlr_spec_red_doubles(plan) doubles; outputs are device pointers. */
int64_t mlr_spec_workspace_bytes(int64_t m_local, int n);
int mlr_spec_create(int64_t m_local, int n, int f32, const double* C, int64_t ldc, const int* skip, void* workspace,
                    void** plan_out, void* stream);
int mlr_spec_destroy(void* plan);
int64_t mlr_spec_red_doubles(void* plan);
int mlr_spec_gram(void* plan, const void* X, int64_t ldx, double* red, void* stream);
int mlr_spec_rotate(void* plan, const void* X, int64_t ldx, const double* red, double* red2, void* stream);
int mlr_spec_finish(void* plan, const double* red2, double rel, double* sig_out, double* rank_out,
                    const double* pair_w, double* wsum_out, void* stream);
/* Dense lower Cholesky factor C of G_R = R^T R (n_H x n_H, C C^T = G_R): sigma(L_H R^T) = sigma(L_H C). */
int mlr_chain_cholesky(void* chain, double* C, int64_t ldc, void* stream);
/* ML-PCP coarse iterate L_H = Z (m_local x n_H, the plan's dtype) of the latest SVT step. */
int mlr_pcp_coarse_copy(void* plan, void* out, int64_t ldo, void* stream);
/* delta = <Z_k (G_R - I), Z_k - Z_f G_R> over this rank's rows (pcp.py:300-302);
 * work holds mlr_pcp_delta_work_doubles() doubles; out is one device double. */
int64_t mlr_pcp_delta_work_doubles(void);
int mlr_pcp_delta(void* plan, const void* Zk, const void* Zf, int64_t ldz, double* out, double* work, void* stream);
/* ML-CPCP rank binding: the coarse iterate L_H (m_local x n_p, ld n_p), the plan's
 * device stop flag (use as the spectrum plan's skip) and the device slot the
 * finalize step records as the iteration's rank_l (-1 unless written). */
int mlr_cpcp_rank_binding(void* plan, const void** lh, int64_t* ld, const int** done, double** rank_slot);
/* FP32 plans: apply this iteration's rank-1 update (cpcp.py:399-402) to an FP64
 * shadow L64 (m_local x n_H, ld >= n_H, zeroed before the first iteration) so the
 * rank is taken of the unrounded iterate, like the reference's float64 run.
 * Call after mlr_cpcp_update. */
int mlr_cpcp_rank_shadow(void* plan, double* L64, int64_t ld, void* stream);
/* track_oracle_atoms (cpcp.py:355-360): after mlr_cpcp_lmo, copy the iteration's
 * LMO factors (u: m_local doubles, v: n_H doubles); later expand one saved pair
 * into the dense atom M_L = -radius u (R v)^T (m_local x n float64, ld ldo). */
int mlr_cpcp_atom_copy(void* plan, double* u_out, double* v_out, void* stream);
int mlr_cpcp_atom_dense(void* plan, const double* u, const double* v, double* out, int64_t ldo, void* stream);

/* ---------------------------------------------------------------- frame stacks
 * Video pipeline layout (reference io.py:131-182).  frames: count 8-bit rasters
 * (height x width, row-major, frame j at frames + j*height*width), device memory.
 * x: the (height*width) x count solver matrix (row-major, ld ldx >= count), pixel
 * (row, col) of frame j at entry (row + col*height, j) (io.py:33-36).
 * to_matrix: x = u8 / 255.0 (float64, then rounded to float when f32) - ingest_frames.
 * to_frames: clamp to [0, 1] and floor(v * 255 + 0.5) - emit_frames' _quantize. */
int mlr_frames_to_matrix(const uint8_t* frames, int count, int height, int width, int f32, void* x, int64_t ldx,
                         void* stream);
int mlr_matrix_to_frames(const void* x, int64_t ldx, int f32, int count, int height, int width, uint8_t* frames,
                         void* stream);

/* ------------------------------------------------------------ observation mask
 * The reference's ObservationMask (cpcp.py:23-53) holds a boolean m x n array; the
 * ML-CPCP passes read it bit-packed (see mlr_cpcp_start).  observed: m x n bytes in
 * device memory (non-zero = observed, row stride ld_observed bytes); bits: m x ldm
 * uint32 words, bit j & 31 of word j >> 5, words past ceil(n / 32) zeroed. */
int mlr_mask_pack(const uint8_t* observed, int64_t ld_observed, int64_t m, int64_t n, uint32_t* bits, int64_t ldm,
                  void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MLR_B200_H */
