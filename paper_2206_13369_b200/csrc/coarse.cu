// Coarse-level helpers: chain upload, tridiagonal solves with G_R = R^T R,
// SVT weights from the Jacobi eigenpairs.
//
// The reference forms M_H = (D - S + Y/mu) R (R^T R)^{-1} with cho_solve on
// the (bidiagonal) Cholesky factor of the tridiagonal G_R (pcp.py:251-255,
// multilevel.py:97-102).  Here the Gram is formed from A = W R and the
// inverse is applied on both sides with an LDL^T recurrence:
//   B = G_R^{-1} (A^T A) G_R^{-1} = M_H^T M_H.
#include "common.cuh"
#include "kernels.h"

namespace mlr {

// Solve G x = y for a single column (LDL^T, unit lower bidiagonal L).
__device__ __forceinline__ void ldl_solve_col(const double* __restrict__ gl, const double* __restrict__ gd,
                                              int nh, const double* in, int64_t in_stride, double* out,
                                              int64_t out_stride) {
  double prev = in[0];
  out[0] = prev;
  for (int k = 1; k < nh; ++k) {
    prev = in[k * in_stride] - gl[k - 1] * prev;
    out[k * out_stride] = prev;
  }
  double x = out[(nh - 1) * out_stride] / gd[nh - 1];
  out[(nh - 1) * out_stride] = x;
  for (int k = nh - 2; k >= 0; --k) {
    x = out[k * out_stride] / gd[k] - gl[k] * x;
    out[k * out_stride] = x;
  }
}

// out[:, c] = G^{-1} in[:, c] (trans_in=0) or G^{-1} in[c, :]^T (trans_in=1)
// for c < nh; rows/cols >= nh are zero-filled in out (np x np, row-major).
__global__ void ldl_solve_kernel(const int* __restrict__ skip, ChainDev ch, const double* __restrict__ in,
                                 double* __restrict__ out, int trans_in) {
  if (skip && *skip) return;
  const int np = ch.np, nh = ch.nh;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < np; c += gridDim.x * blockDim.x) {
    if (c >= nh) {
      for (int r = 0; r < np; ++r) out[(int64_t)r * np + c] = 0.0;
      continue;
    }
    if (trans_in)
      ldl_solve_col(ch.gl, ch.gd, nh, in + (int64_t)c * np, 1, out + c, np);
    else
      ldl_solve_col(ch.gl, ch.gd, nh, in + c, np, out + c, np);
    for (int r = nh; r < np; ++r) out[(int64_t)r * np + c] = 0.0;
  }
}

int ldl_solve(const int* skip, const ChainDev& ch, const double* in, double* out, int trans_in,
              cudaStream_t st) {
  int threads = 128, blocks = (int)ceil_div(ch.np, threads);
  ldl_solve_kernel<<<blocks, threads, 0, st>>>(skip, ch, in, out, trans_in);
  MLR_LAUNCH_CHECK("ldl_solve_kernel");
  return kOk;
}

// Eigenvalues lambda_i = v_i^T x_i of the converged Jacobi pair (X = B V);
// sigma_i = sqrt(lambda_i); SVT weight f_i = max(sigma_i - tau, 0)/sigma_i;
// rank = #{sigma_i > tau} (strict, pcp.py:258); nuclear = sum(sigma_i - tau)+
// (pcp.py:264-267).  One CTA; f feeds the k-scaled NT GEMM P = V diag(f) V^T.
template <typename T>
__global__ void svt_weights_kernel(const int* __restrict__ skip, int np, int nh, const T* __restrict__ Bd,
                                   const double* tau_p, double* __restrict__ sig_out,
                                   double* __restrict__ f_out, int* rank_out, double* nuclear_out) {
  if (skip && *skip) return;
  __shared__ double scratch[2 * 32];
  const double tau = *tau_p;
  double nuc = 0.0, rk = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) {
    double f = 0.0, s = 0.0;
    if (i < nh) {
      const double lam = (double)Bd[(int64_t)i * (np + 1)];  // diagonalised B~
      s = sqrt(fmax(lam, 0.0));
      if (s > tau) {
        f = (s - tau) / s;
        nuc += s - tau;
        rk += 1.0;
      }
    }
    if (sig_out) sig_out[i] = s;
    f_out[i] = f;
  }
  double v[2] = {nuc, rk};
  block_sum<2>(v, scratch);
  if (threadIdx.x == 0) {
    *nuclear_out = v[0];
    *rank_out = (int)(v[1] + 0.5);
  }
}

int svt_weights(const int* skip, int np, int nh, bool f32, const void* Bd, const double* tau, double* sig_out,
                double* f_out, int* rank_out, double* nuclear_out, cudaStream_t st) {
  if (f32)
    svt_weights_kernel<float><<<1, 1024, 0, st>>>(skip, np, nh, (const float*)Bd, tau, sig_out, f_out, rank_out,
                                                  nuclear_out);
  else
    svt_weights_kernel<double><<<1, 1024, 0, st>>>(skip, np, nh, (const double*)Bd, tau, sig_out, f_out, rank_out,
                                                   nuclear_out);
  MLR_LAUNCH_CHECK("svt_weights_kernel");
  return kOk;
}

}  // namespace mlr
