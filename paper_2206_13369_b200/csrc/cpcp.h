// Device state and plan for ML-CPCP (multilevel Frank-Wolfe thresholding).
#pragma once
#include "kernels.h"

namespace mlr {

constexpr int kCpHistCols = 8;  // gap, objective, rank, sparsity, wall, gamma_l, gamma_s, power passes
constexpr int kCpStats = 5;     // sum r^2, sum |S|, nnz(S), sum S^2, sum S*r

struct CpcpDev {
  double lam_l, lam_s, tol, radius, time_budget, t0_ns, m_global, n, rtol;
  double u_l, u_s, t_l, t_s, pd_norm;
  // stats of the latest fine pass (after reduction)
  double sq, l1, nnz, ss, sr;
  // LMO of the current iteration
  double s2, sigma, coef;   // coef = -radius * u_l if corner_l else 0
  int corner_l, corner_s, none, passes;
  double spike, r_is, s_is, v_tl, v_ts;
  long long idx_is;         // column-major global index of the arg-max (-1: none)
  long long i_s;            // global row of the arg-max
  int j_s;
  double ga, gb;
  int k, done, status, max_iters, max_passes;
  double rank_l;            // numerical rank of L (collect_rank), -1 when not collected
};

struct CpcpPlan {
  PhaseTimer timer;  // phases: gram, power, dots, qp, -, update, finalize
  ChainDev ch;
  bool f32;
  int64_t m_local, m_global, row0;
  int max_iters, row_blocks, gram_splits, world, cluster;
  CpcpDev* dev;
  double* hist;      // [max_iters][kCpHistCols]
  double* obj;       // [max_iters]
  void* LH;          // m_local x np (T)
  void* GH;          // m_local x np (T): r R
  void* SH;          // m_local x np (T): S R
  double* u;         // m_local
  double* v;         // np (warm start)
  double* vin;       // np
  double* gram_part; // gram_splits x np x np
  double* row_part;  // row_blocks x 8 (stats) + row_blocks x 4 (argmax)
  double* dots_part; // row_blocks x 3
  const uint32_t* mask_dev;  // bound at start (may be null: fully observed)
  int64_t ldm_dev;
  // segment-QP dots from coarse data (masked chain Gram per row, once per solve)
  bool coarse_dots;
  void* mgd;         // m_local x np (T): diagonal of M_i
  void* mgo;         // m_local x np (T): super-diagonal of M_i
  // full-width solve (identity chain, one rank): the LMO's power passes run as
  // matvecs on g_H = r instead of on the n x n Gram, which is never formed
  bool fine;
  int fine_ctas;
  double* ft;        // m_local: t = g v
  double* fz;        // np: z = g^T t
  double* fv0;       // np: v at LMO entry (restored when g v = 0)
  double* fzpart;    // fine_ctas x np
  double* fspart;    // fine_ctas x 2
};

int cpcp_start(CpcpPlan* p, const void* D, int64_t ldd, const uint32_t* mask, int64_t ldm, void* S, int64_t lds,
               double lam_l, double lam_s, double tol, double radius, int max_iters, double time_budget,
               cudaStream_t st);
int cpcp_gram(CpcpPlan* p, double* red, double* amax, cudaStream_t st);
int cpcp_begin(CpcpPlan* p, const double* red, const double* amax_all, cudaStream_t st);
int cpcp_lmo(CpcpPlan* p, const double* red, const double* amax_all, double* dots, cudaStream_t st);
int cpcp_update(CpcpPlan* p, const void* D, int64_t ldd, const uint32_t* mask, int64_t ldm, void* S, int64_t lds,
                const double* dots, cudaStream_t st);
int cpcp_finalize(CpcpPlan* p, const double* red, cudaStream_t st);
int cpcp_outputs(CpcpPlan* p, void* L, int64_t ldl, cudaStream_t st);
int cpcp_rank_shadow(CpcpPlan* p, double* L64, int64_t ld, cudaStream_t st);
int cpcp_atom_copy(CpcpPlan* p, double* u_out, double* v_out, cudaStream_t st);
int box_qp_batch(const double* in, double* out, int count, cudaStream_t st);
int cpcp_atom_dense(CpcpPlan* p, const double* u, const double* v, double* out, int64_t ldo, cudaStream_t st);

}  // namespace mlr
