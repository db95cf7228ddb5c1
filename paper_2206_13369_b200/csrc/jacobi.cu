// One-sided block Jacobi eigensolver for the coarse SVT (replaces gesdd in
// svd_full, reference linalg.py:86-99, called at pcp.py:257).
//
// Problem: B = M_H^T M_H (n_p x n_p, symmetric PSD, FP64).  We run one-sided
// (Hestenes) Jacobi on X = B * V0 (V0 = previous iteration's eigenvectors,
// the warm start) and accumulate V = V0 * J.  At convergence the columns of
// X = B V are mutually orthogonal, so V holds eigenvectors of B and the
// Rayleigh quotients v_i^T x_i are its eigenvalues (sigma_i^2 of M_H).
//
// Parallel structure (one cooperative launch per eigensolve):
//   * columns are grouped into blocks of BW; a round-robin tournament pairs
//     blocks, npairs = nb/2 pairs per step, nb-1 steps per sweep;
//   * each pair is owned by `nchunks` CTAs, each holding RC rows of the
//     pair's 2*BW columns of X and V in shared memory;
//   * phase A: per-CTA partial Gram (2BW x 2BW) -> global;   grid barrier
//   * phase B: every CTA of the pair sums the partials (same order, so all
//     compute the identical Gram), runs one inner cyclic sweep of 2BW-1
//     parallel rounds on the Gram accumulating Q, then applies Q to its
//     X/V rows;                                                 grid barrier
//   * convergence: max_{i<j} |g_ij|/sqrt(g_ii g_jj) over a whole sweep <= tol.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace mlr {

constexpr int JRC = 64;        // rows per CTA chunk
constexpr int JTHREADS = 256;

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  // non-negative doubles order like their bit patterns
  atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

// circle-method tournament: m players (m odd) + 1 fixed player m; round t.
__device__ __forceinline__ void rr_pair(int t, int k, int m, int& a, int& b) {
  if (k == 0) {
    a = t;
    b = m;
  } else {
    a = (t + k) % m;
    b = (t - k + m) % m;
  }
}

template <int BW>
struct JacSmem {
  static constexpr int PW = 2 * BW;
  double G[PW][PW + 1];
  double Q[PW][PW + 1];
  double X[JRC][PW + 1];
  double V[JRC][PW + 1];
  double cs[PW / 2][2];
  int pr[PW / 2][2];
  int rotated;
};

template <int BW>
__global__ void __launch_bounds__(JTHREADS)
jacobi_kernel(double* __restrict__ X, double* __restrict__ V, int np, double tol, int max_sweeps,
              double* __restrict__ partials, double* __restrict__ off_slots, int* __restrict__ result,
              const int* __restrict__ skip) {
  if (skip && *skip) return;
  constexpr int PW = 2 * BW;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  JacSmem<BW>& S = *reinterpret_cast<JacSmem<BW>*>(smem_raw);
  cg::grid_group grid = cg::this_grid();

  const int nb = np / BW;
  const int m = nb - 1;
  const int nchunks = np / JRC;
  const int units = (nb / 2) * nchunks;
  const int tid = threadIdx.x;

  int sweep = 0;
  bool converged = false;
  for (; sweep < max_sweeps; ++sweep) {
    for (int t = 0; t < m; ++t) {
      // ---- phase A: partial Gram of each owned (pair, row-chunk) unit
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int pair = u / nchunks, r0 = (u % nchunks) * JRC;
        int pa, pb;
        rr_pair(t, pair, m, pa, pb);
        __syncthreads();
        for (int e = tid; e < JRC * PW; e += JTHREADS) {
          int r = e / PW, l = e % PW;
          int col = (l < BW) ? pa * BW + l : pb * BW + (l - BW);
          S.X[r][l] = X[(int64_t)(r0 + r) * np + col];
        }
        __syncthreads();
        double* part = partials + (int64_t)u * PW * PW;
        for (int e = tid; e < PW * PW; e += JTHREADS) {
          int i = e / PW, j = e % PW;
          double s = 0.0;
#pragma unroll 8
          for (int r = 0; r < JRC; ++r) s = fma(S.X[r][i], S.X[r][j], s);
          part[e] = s;
        }
      }
      grid.sync();
      if (t == 0 && blockIdx.x == 0 && tid == 0) off_slots[(sweep + 1) & 1] = 0.0;
      // ---- phase B: full Gram, inner sweep, apply to owned rows
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int pair = u / nchunks, chunk = u % nchunks, r0 = chunk * JRC;
        int pa, pb;
        rr_pair(t, pair, m, pa, pb);
        __syncthreads();
        const double* pp = partials + (int64_t)pair * nchunks * PW * PW;
        for (int e = tid; e < PW * PW; e += JTHREADS) {
          double s = 0.0;
          for (int c = 0; c < nchunks; ++c) s += pp[(int64_t)c * PW * PW + e];
          S.G[e / PW][e % PW] = s;
          S.Q[e / PW][e % PW] = (e / PW == e % PW) ? 1.0 : 0.0;
        }
        if (tid == 0) S.rotated = 0;
        __syncthreads();
        {
          double mx = 0.0;
          for (int e = tid; e < PW * PW; e += JTHREADS) {
            int i = e / PW, j = e % PW;
            if (i < j) {
              double a = S.G[i][i], b = S.G[j][j];
              if (a > 0.0 && b > 0.0) mx = fmax(mx, fabs(S.G[i][j]) / sqrt(a * b));
            }
          }
          mx = warp_max(mx);
          if ((tid & 31) == 0 && chunk == 0 && mx > 0.0) atomic_max_nonneg(&off_slots[sweep & 1], mx);
        }
        for (int rnd = 0; rnd < PW - 1; ++rnd) {
          if (tid < PW / 2) {
            int i, j;
            rr_pair(rnd, tid, PW - 1, i, j);
            double a = S.G[i][i], b = S.G[j][j], g = S.G[i][j];
            double c = 1.0, s = 0.0;
            if (a > 0.0 && b > 0.0 && fabs(g) > tol * sqrt(a * b)) {
              double z = (b - a) / (2.0 * g);
              double tt = (z >= 0.0 ? 1.0 : -1.0) / (fabs(z) + sqrt(1.0 + z * z));
              c = 1.0 / sqrt(1.0 + tt * tt);
              s = c * tt;
              S.rotated = 1;
            }
            S.cs[tid][0] = c;
            S.cs[tid][1] = s;
            S.pr[tid][0] = i;
            S.pr[tid][1] = j;
          }
          __syncthreads();
          for (int e = tid; e < (PW / 2) * (PW / 2); e += JTHREADS) {
            int p = e / (PW / 2), q = e % (PW / 2);
            int p1 = S.pr[p][0], p2 = S.pr[p][1], q1 = S.pr[q][0], q2 = S.pr[q][1];
            double cp = S.cs[p][0], sp = S.cs[p][1], cq = S.cs[q][0], sq = S.cs[q][1];
            double g11 = S.G[p1][q1], g12 = S.G[p1][q2], g21 = S.G[p2][q1], g22 = S.G[p2][q2];
            double t11 = cq * g11 - sq * g12, t12 = sq * g11 + cq * g12;
            double t21 = cq * g21 - sq * g22, t22 = sq * g21 + cq * g22;
            S.G[p1][q1] = cp * t11 - sp * t21;
            S.G[p1][q2] = cp * t12 - sp * t22;
            S.G[p2][q1] = sp * t11 + cp * t21;
            S.G[p2][q2] = sp * t12 + cp * t22;
          }
          for (int e = tid; e < PW * (PW / 2); e += JTHREADS) {
            int r = e / (PW / 2), q = e % (PW / 2);
            int q1 = S.pr[q][0], q2 = S.pr[q][1];
            double c = S.cs[q][0], s = S.cs[q][1];
            double a = S.Q[r][q1], b = S.Q[r][q2];
            S.Q[r][q1] = c * a - s * b;
            S.Q[r][q2] = s * a + c * b;
          }
          __syncthreads();
        }
        if (S.rotated) {
          for (int e = tid; e < JRC * PW; e += JTHREADS) {
            int r = e / PW, l = e % PW;
            int col = (l < BW) ? pa * BW + l : pb * BW + (l - BW);
            int64_t off = (int64_t)(r0 + r) * np + col;
            S.X[r][l] = X[off];
            S.V[r][l] = V[off];
          }
          __syncthreads();
          for (int e = tid; e < JRC * PW; e += JTHREADS) {
            int r = e / PW, l = e % PW;
            double sx = 0.0, sv = 0.0;
#pragma unroll 8
            for (int k = 0; k < PW; ++k) {
              sx = fma(S.X[r][k], S.Q[k][l], sx);
              sv = fma(S.V[r][k], S.Q[k][l], sv);
            }
            int col = (l < BW) ? pa * BW + l : pb * BW + (l - BW);
            int64_t off = (int64_t)(r0 + r) * np + col;
            X[off] = sx;
            V[off] = sv;
          }
        }
      }
      grid.sync();
    }
    double off = *((volatile double*)&off_slots[sweep & 1]);
    if (off <= tol) {
      converged = true;
      ++sweep;
      break;
    }
  }
  if (blockIdx.x == 0 && tid == 0) result[0] = converged ? sweep : -sweep;
}

template <int BW>
static int launch_jacobi(double* X, double* V, int np, double tol, int max_sweeps, double* partials,
                         double* off_slots, int* result, const int* skip, cudaStream_t st) {
  const int nb = np / BW;
  const int nchunks = np / JRC;
  const int units = (nb / 2) * nchunks;
  size_t smem = sizeof(JacSmem<BW>);
  auto kern = jacobi_kernel<BW>;
  MLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, nsm = 0, per_sm = 0;
  MLR_CUDA(cudaGetDevice(&dev));
  MLR_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  MLR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, JTHREADS, smem));
  if (per_sm < 1) {
    set_error("jacobi_eig: kernel does not fit on an SM");
    return kErrArg;
  }
  const int grid = std::min(units, nsm * per_sm);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(JTHREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MLR_CUDA(cudaLaunchKernelEx(&cfg, kern, X, V, np, tol, max_sweeps, partials, off_slots, result, skip));
  return kOk;
}

int jacobi_block_width(int np) { return np >= 1024 ? 32 : 16; }

int64_t jacobi_partials_doubles(int np) {
  int bw = jacobi_block_width(np);
  int64_t nb = np / bw, nchunks = np / JRC, pw = 2 * bw;
  return (nb / 2) * nchunks * pw * pw;
}

int jacobi_eig(double* X, double* V, int np, double tol, int max_sweeps, double* partials,
               double* off_slots, int* result, const int* skip, cudaStream_t st) {
  if (np % 64 != 0) {
    set_error("jacobi_eig: n_p must be a multiple of 64");
    return kErrArg;
  }
  MLR_CUDA(cudaMemsetAsync(off_slots, 0, 2 * sizeof(double), st));
  if (jacobi_block_width(np) == 32)
    return launch_jacobi<32>(X, V, np, tol, max_sweeps, partials, off_slots, result, skip, st);
  return launch_jacobi<16>(X, V, np, tol, max_sweeps, partials, off_slots, result, skip, st);
}

}  // namespace mlr
