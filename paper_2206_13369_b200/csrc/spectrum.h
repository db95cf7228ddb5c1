// Accurate singular values of a tall row-sharded matrix X (m x n), or of X C
// for a fixed n x n factor C, for the reference's numerical-rank telemetry:
//   cpcp.py:434-439   rank(L) of the FW-T iterate (collect_rank)
//   multilevel.py:248-265 epsilon_bound of the final ML-PCP coarse iterate
// Both count sigma_i > sigma_1 * max(m, n) * eps, a threshold far below what
// one Gram eigensolve resolves (eigenvalues of X^T X carry an absolute error
// ~eps sigma_1^2), so the values come from two passes:
//   1. K = (X C)^T (X C), Jacobi (warm-started from the previous call) -> V1;
//   2. B = X C V1 has nearly orthogonal columns; K2 = B^T B, Jacobi with the
//      purely relative stopping rule -> sigma_i = sqrt(lambda_i(K2)), accurate
//      to ~eps sigma_1 in absolute terms, like the reference's gesdd.
#pragma once
#include "kernels.h"

namespace mlr {

struct SpecPlan {
  int64_t m_local;
  int n, np, splits;
  bool f32, warm;
  const int* skip;   // optional device flag: every step is a no-op when set
  double* C;         // np x np (zero padded), null = identity
  double* V1;        // np x np: pass-1 basis (warm start)
  double* V2;        // np x np
  double* T1;        // np x np
  double* M1;        // np x np
  double* X2;        // m_local x np: B = X C V1
  double* gram_part; // splits x np x np
  double* qbuf;
  int* qflag;
  double* off;
  int* result;
  double* sig;       // np, sorted descending
};

int64_t spec_workspace_bytes(int64_t m_local, int n, int splits);
void spec_carve(SpecPlan& p, void* ws);
int spec_init(SpecPlan* p, const double* C, int64_t ldc, cudaStream_t st);
int spec_gram(SpecPlan* p, const void* X, int64_t ldx, double* red, cudaStream_t st);
int spec_rotate(SpecPlan* p, const void* X, int64_t ldx, const double* red, double* red2, cudaStream_t st);
int spec_finish(SpecPlan* p, const double* red2, double rel, double* sig_out, double* rank_out, const double* pair_w,
                double* wsum_out, cudaStream_t st);

// dense lower Cholesky factor of G_R = R^T R (n_H x n_H), from the chain's LDL^T
int chain_cholesky(const ChainDev& ch, double* C, int64_t ldc, cudaStream_t st);
// ML-PCP alignment error delta_k = <Z_k (G - I), Z_k - Z_f G> (pcp.py:298-306)
int pcp_delta(const ChainDev& ch, bool f32, int64_t m, const void* Zk, const void* Zf, int64_t ld, double* out,
              double* work, int blocks, cudaStream_t st);

}  // namespace mlr
