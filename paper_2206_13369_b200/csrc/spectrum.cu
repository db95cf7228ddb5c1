// Two-pass Gram/Jacobi singular values of a tall matrix (see spectrum.h).
#include "common.cuh"
#include "kernels.h"
#include "spectrum.h"

namespace mlr {

namespace {

struct Carve {
  char* base;
  size_t off = 0;
  template <typename P>
  P* take(size_t bytes) {
    off = (off + 255) & ~size_t(255);
    P* q = base ? reinterpret_cast<P*>(base + off) : nullptr;
    off += bytes;
    return q;
  }
};

void carve(SpecPlan& p, Carve& c) {
  const size_t nn = (size_t)p.np * p.np;
  p.C = c.take<double>(8 * nn);
  p.V1 = c.take<double>(8 * nn);
  p.V2 = c.take<double>(8 * nn);
  p.T1 = c.take<double>(8 * nn);
  p.M1 = c.take<double>(8 * nn);
  p.X2 = c.take<double>(8 * (size_t)std::max<int64_t>(p.m_local, 1) * p.np);
  p.gram_part = c.take<double>(8 * nn * p.splits);
  p.qbuf = c.take<double>(8 * (size_t)jacobi2_qbuf_elems(p.np));
  p.qflag = c.take<int>(4 * (size_t)jacobi2_qflag_elems(p.np));
  p.off = c.take<double>(8 * 4);
  p.result = c.take<int>(4 * 16);
  p.sig = c.take<double>(8 * (size_t)p.np);
}

__global__ void spec_eye(double* V, int np, const int* skip) {
  if (skip && *skip) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)np * np;
       e += (int64_t)gridDim.x * blockDim.x)
    V[e] = (e / np == e % np) ? 1.0 : 0.0;
}

__global__ void spec_copy(const double* __restrict__ src, double* __restrict__ dst, int64_t count, const int* skip) {
  if (skip && *skip) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = src[e];
}

// sigma_i = sqrt(lambda_i), sorted descending by counting (stable on ties);
// rank = #{sigma > sigma_1 * rel}; wsum = sum_{k < rank} sigma_(k) w_k
__global__ void __launch_bounds__(1024) spec_finish_kernel(const double* __restrict__ M, int np, double rel,
                                                           double* __restrict__ sv, double* __restrict__ sig_sorted,
                                                           double* __restrict__ sig_out, double* __restrict__ rank_out,
                                                           const double* __restrict__ pair_w,
                                                           double* __restrict__ wsum_out, const int* skip) {
  if (skip && *skip) return;
  __shared__ double scratch[2 * 32];
  __shared__ double wmax[32];
  __shared__ int rank_s;
  double mx = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) {
    const double s = sqrt(fmax(M[(int64_t)i * (np + 1)], 0.0));
    sv[i] = s;
    mx = fmax(mx, s);
  }
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) m = fmax(m, wmax[w]);
    wmax[0] = m;
  }
  __syncthreads();
  const double smax = wmax[0];
  const double thr = smax * rel;
  double rk = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) {
    const double s = sv[i];
    int pos = 0;
    for (int j = 0; j < np; ++j) {
      const double t = sv[j];
      pos += (t > s || (t == s && j < i)) ? 1 : 0;
    }
    sig_sorted[pos] = s;
    if (smax > 0.0 && s > thr) rk += 1.0;
  }
  double v[2] = {rk, 0.0};
  block_sum<2>(v, scratch);  // ends with __syncthreads: sig_sorted is complete
  if (threadIdx.x == 0) rank_s = (int)(v[0] + 0.5);
  __syncthreads();
  double ws = 0.0;
  for (int k = threadIdx.x; k < np; k += blockDim.x) {
    if (sig_out) sig_out[k] = sig_sorted[k];
    if (pair_w && k < rank_s) ws += sig_sorted[k] * pair_w[k];
  }
  double v2[2] = {ws, 0.0};
  block_sum<2>(v2, scratch);
  if (threadIdx.x == 0) {
    if (rank_out) *rank_out = (double)rank_s;
    if (wsum_out) *wsum_out = pair_w ? v2[0] : 0.0;
  }
}

int mm(SpecPlan* p, const double* A, bool ta, const double* B, bool tb, double* C, cudaStream_t st) {
  GemmSpec g{};
  g.M = p->np; g.N = p->np; g.K = p->np;
  g.A = A; g.lda = p->np; g.a_f32 = false; g.trans_a = ta;
  g.B = B; g.ldb = p->np; g.b_f32 = false; g.trans_b = tb;
  g.C = C; g.ldc = p->np; g.c_f32 = false; g.c_slice = 0; g.splits = 1; g.alpha = 1.0;
  g.kscale = nullptr; g.skip = p->skip;
  return gemm_f64(g, st);
}

// red (np x np) = sum over the local rows of op(X)^T op(X), X m_local x ncols
int gram(SpecPlan* p, const void* X, int64_t ldx, bool x_f32, int ncols, double* red, cudaStream_t st) {
  const int64_t nn = (int64_t)p->np * p->np;
  if (p->m_local > 0) {
    GemmSpec g{};
    g.M = ncols; g.N = ncols; g.K = (int)p->m_local;
    g.A = X; g.lda = ldx; g.a_f32 = x_f32; g.trans_a = true;
    g.B = X; g.ldb = ldx; g.b_f32 = x_f32; g.trans_b = false;
    g.C = p->gram_part; g.ldc = p->np; g.c_f32 = false; g.c_slice = nn; g.splits = p->splits; g.alpha = 1.0;
    g.kscale = nullptr; g.skip = p->skip; g.sym = true;
    int rc = gemm_f64(g, st);
    if (rc) return rc;
    return sum_slices(p->gram_part, nn, nn, p->splits, red, st);
  }
  MLR_CUDA(cudaMemsetAsync(red, 0, sizeof(double) * nn, st));
  return kOk;
}

constexpr double kEps = 2.220446049250313e-16;

}  // namespace

int64_t spec_workspace_bytes(int64_t m_local, int n, int splits) {
  SpecPlan p{};
  p.m_local = m_local;
  p.n = n;
  p.np = (int)round_up(n, 64);
  p.splits = splits;
  Carve c{nullptr};
  carve(p, c);
  return (int64_t)c.off + 256;
}

void spec_carve(SpecPlan& p, void* ws) {
  Carve c{(char*)ws};
  carve(p, c);
}

int spec_init(SpecPlan* p, const double* C, int64_t ldc, cudaStream_t st) {
  const int64_t nn = (int64_t)p->np * p->np;
  // the Gram partials are written for the n x n block only: zero the padding once
  MLR_CUDA(cudaMemsetAsync(p->gram_part, 0, sizeof(double) * nn * p->splits, st));
  MLR_CUDA(cudaMemsetAsync(p->X2, 0, sizeof(double) * std::max<int64_t>(p->m_local, 1) * p->np, st));
  if (C) {
    MLR_CUDA(cudaMemsetAsync(p->C, 0, sizeof(double) * nn, st));
    MLR_CUDA(cudaMemcpy2DAsync(p->C, sizeof(double) * p->np, C, sizeof(double) * ldc, sizeof(double) * p->n, p->n,
                               cudaMemcpyDeviceToDevice, st));
  } else {
    p->C = nullptr;
  }
  p->warm = false;
  return kOk;
}

int spec_gram(SpecPlan* p, const void* X, int64_t ldx, double* red, cudaStream_t st) {
  return gram(p, X, ldx, p->f32, p->n, red, st);
}

int spec_rotate(SpecPlan* p, const void* X, int64_t ldx, const double* red, double* red2, cudaStream_t st) {
  const int np = p->np;
  const int64_t nn = (int64_t)np * np;
  int rc;
  // pass 1 on M = C^T K C (warm: V1^T M V1, with V1 accumulating)
  const double* M = red;
  if (p->C) {
    if ((rc = mm(p, red, false, p->C, false, p->T1, st))) return rc;    // K C
    if ((rc = mm(p, p->C, true, p->T1, false, p->M1, st))) return rc;   // C^T K C
    M = p->M1;
  }
  if (p->warm) {
    if ((rc = mm(p, M, false, p->V1, false, p->T1, st))) return rc;     // M V1
    if ((rc = mm(p, p->V1, true, p->T1, false, p->M1, st))) return rc;  // V1^T M V1
  } else {
    if (M != p->M1) {
      spec_copy<<<256, 256, 0, st>>>(M, p->M1, nn, p->skip);
      MLR_LAUNCH_CHECK("spec_copy");
    }
    spec_eye<<<256, 256, 0, st>>>(p->V1, np, p->skip);
    MLR_LAUNCH_CHECK("spec_eye");
  }
  if ((rc = jacobi2_eig(false, p->M1, p->V1, np, np, 64 * kEps, 1e-17, 60, p->qbuf, p->qflag, p->off, p->result,
                        p->skip, st)))
    return rc;
  p->warm = true;
  // B = X (C V1): m_local x np, nearly orthogonal columns
  const double* W = p->V1;
  if (p->C) {
    if ((rc = mm(p, p->C, false, p->V1, false, p->T1, st))) return rc;
    W = p->T1;
  }
  if (p->m_local > 0) {
    GemmSpec z{};
    z.M = (int)p->m_local; z.N = np; z.K = p->n;
    z.A = X; z.lda = ldx; z.a_f32 = p->f32; z.trans_a = false;
    z.B = W; z.ldb = np; z.b_f32 = false; z.trans_b = false;
    z.C = p->X2; z.ldc = np; z.c_f32 = false; z.c_slice = 0; z.splits = 1; z.alpha = 1.0;
    z.kscale = nullptr; z.skip = p->skip;
    if ((rc = gemm_f64(z, st))) return rc;
  }
  return gram(p, p->X2, np, false, np, red2, st);
}

int spec_finish(SpecPlan* p, const double* red2, double rel, double* sig_out, double* rank_out, const double* pair_w,
                double* wsum_out, cudaStream_t st) {
  const int np = p->np;
  spec_copy<<<256, 256, 0, st>>>(red2, p->M1, (int64_t)np * np, p->skip);
  MLR_LAUNCH_CHECK("spec_copy");
  spec_eye<<<256, 256, 0, st>>>(p->V2, np, p->skip);
  MLR_LAUNCH_CHECK("spec_eye");
  // relative stopping rule, plus an absolute floor of 1e-4 * (rel sigma_1)^2:
  // an off-diagonal g moves an eigenvalue by at most |g| (Weyl), so values
  // near the rank threshold keep ~5e-5 relative accuracy (finer than the
  // reference's own SVD resolves there) while the block of numerically-zero
  // singular values, pure rounding noise, is not diagonalised for nothing.
  // rel = 0 (all singular values wanted) keeps the purely relative rule.
  int rc = jacobi2_eig(false, p->M1, p->V2, np, np, 64 * kEps, 1e-4 * rel * rel, 60, p->qbuf, p->qflag, p->off,
                       p->result, p->skip, st);
  if (rc) return rc;
  spec_finish_kernel<<<1, 1024, 0, st>>>(p->M1, np, rel, p->T1, p->sig, sig_out, rank_out, pair_w, wsum_out, p->skip);
  MLR_LAUNCH_CHECK("spec_finish_kernel");
  return kOk;
}

}  // namespace mlr

// ------------------------------------------------------------ ML-PCP diagnostics
namespace mlr {

// Dense lower Cholesky factor of G_R = R^T R from its LDL^T (C = L D^1/2,
// bidiagonal): C[j][j] = sqrt(d_j), C[j+1][j] = l_j sqrt(d_j).
__global__ void chain_chol_kernel(ChainDev ch, double* __restrict__ C, int64_t ldc) {
  const int nh = ch.nh;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)nh * nh;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / nh), j = (int)(e % nh);
    double v = 0.0;
    if (i == j) v = sqrt(ch.gd[j]);
    else if (i == j + 1) v = ch.gl[j] * sqrt(ch.gd[j]);
    C[(int64_t)i * ldc + j] = v;
  }
}

int chain_cholesky(const ChainDev& ch, double* C, int64_t ldc, cudaStream_t st) {
  chain_chol_kernel<<<256, 256, 0, st>>>(ch, C, ldc);
  MLR_LAUNCH_CHECK("chain_chol_kernel");
  return kOk;
}

// delta_k = <Z_k (G - I), Z_k - Z_f G> over the local rows (reference
// pcp.py:300-302: drift = R^T R - I, ref = restrict(L_final) = Z_f G).  G is
// tridiagonal: G[j][j] = d_j + l_{j-1}^2 d_{j-1}, G[j][j+1] = l_j d_j.
template <typename T>
__global__ void __launch_bounds__(256) pcp_delta_kernel(ChainDev ch, int64_t m, const T* __restrict__ Zk,
                                                        const T* __restrict__ Zf, int64_t ld,
                                                        double* __restrict__ part) {
  __shared__ double scratch[2 * 32];
  const int nh = ch.nh;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * nw + warp; i < m; i += (int64_t)gridDim.x * nw) {
    const T* zk = Zk + i * ld;
    const T* zf = Zf + i * ld;
    for (int j = lane; j < nh; j += 32) {
      const double gdj = ch.gd[j] + (j > 0 ? ch.gl[j - 1] * ch.gl[j - 1] * ch.gd[j - 1] : 0.0);
      const double glo = j > 0 ? ch.gl[j - 1] * ch.gd[j - 1] : 0.0;  // G[j-1][j]
      const double ghi = j + 1 < nh ? ch.gl[j] * ch.gd[j] : 0.0;     // G[j+1][j]
      const double zkj = (double)zk[j];
      const double zkg = zkj * gdj + (j > 0 ? (double)zk[j - 1] * glo : 0.0) +
                         (j + 1 < nh ? (double)zk[j + 1] * ghi : 0.0);
      const double zfg = (double)zf[j] * gdj + (j > 0 ? (double)zf[j - 1] * glo : 0.0) +
                         (j + 1 < nh ? (double)zf[j + 1] * ghi : 0.0);
      acc += (zkg - zkj) * (zkj - zfg);
    }
  }
  double v[2] = {acc, 0.0};
  block_sum<2>(v, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

__global__ void sum_parts_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double scratch[2 * 32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  double v[2] = {s, 0.0};
  block_sum<2>(v, scratch);
  if (threadIdx.x == 0) *out = v[0];
}

int pcp_delta(const ChainDev& ch, bool f32, int64_t m, const void* Zk, const void* Zf, int64_t ld, double* out,
              double* work, int blocks, cudaStream_t st) {
  if (m <= 0) {
    MLR_CUDA(cudaMemsetAsync(out, 0, sizeof(double), st));
    return kOk;
  }
  if (f32)
    pcp_delta_kernel<float><<<blocks, 256, 0, st>>>(ch, m, (const float*)Zk, (const float*)Zf, ld, work);
  else
    pcp_delta_kernel<double><<<blocks, 256, 0, st>>>(ch, m, (const double*)Zk, (const double*)Zf, ld, work);
  MLR_LAUNCH_CHECK("pcp_delta_kernel");
  sum_parts_kernel<<<1, 256, 0, st>>>(work, blocks, out);
  MLR_LAUNCH_CHECK("sum_parts_kernel");
  return kOk;
}

}  // namespace mlr
