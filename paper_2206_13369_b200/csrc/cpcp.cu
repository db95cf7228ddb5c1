// ML-CPCP: multilevel Frank-Wolfe thresholding (reference cpcp.py:326-515)
// on the device.
//
// State kept on the GPU per iteration:
//   S   (m_local x n, T)  — the sparse block, stored densely (supported on Q)
//   L_H (m_local x np, T) — L = L_H R^T always (L starts at 0 and only ever
//                           moves toward prolonged coarse atoms)
//   g_H = r R, s~ = S R (m_local x np) — restrictions of the residual and S
// The residual r = P[L + S - D] is recomputed exactly inside the single fine
// pass (the reference tracks it incrementally and refreshes every 64
// iterations, cpcp.py:423-427).  All five segment-QP dot products
// (cpcp.py:387-395) are evaluated from coarse quantities plus the mask bits
// (see cp_dots_kernel), so each iteration streams D, S and the bit-packed
// mask once and writes S once.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include <cstdlib>

#include "common.cuh"
#include "cpcp.h"
#include "kernels.h"
#include "rows.h"

namespace cg = cooperative_groups;

namespace mlr {

__device__ __forceinline__ double cp_now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return (double)t;
}

template <typename T>
struct CpStencil;
template <>
struct CpStencil<float> {
  static __device__ __forceinline__ const float* w0(const ChainDev& c) { return c.w0f; }
  static __device__ __forceinline__ const float* w1(const ChainDev& c) { return c.w1f; }
};
template <>
struct CpStencil<double> {
  static __device__ __forceinline__ const double* w0(const ChainDev& c) { return c.w0; }
  static __device__ __forceinline__ const double* w1(const ChainDev& c) { return c.w1; }
};

struct AmRec {
  double mag, val, sval;
  long long idx;
};

__device__ __forceinline__ void am_merge(AmRec& a, const AmRec& b) {
  if (argmax_better(b.mag, b.idx, a.mag, a.idx)) a = b;
}

__device__ __forceinline__ AmRec am_warp(AmRec a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    AmRec b;
    b.mag = __shfl_xor_sync(0xffffffffu, a.mag, o);
    b.val = __shfl_xor_sync(0xffffffffu, a.val, o);
    b.sval = __shfl_xor_sync(0xffffffffu, a.sval, o);
    b.idx = __shfl_xor_sync(0xffffffffu, a.idx, o);
    am_merge(a, b);
  }
  return a;
}

enum CpMode { kCpInit = 0, kCpUpdate = 1, kCpOutput = 2 };

// One fine pass (see file comment).  INIT: r = -P[D], S untouched (zero).
template <typename T, int MODE>
__global__ void __launch_bounds__(256)
cp_row_kernel(const CpcpDev* __restrict__ st, ChainDev ch, int64_t m, int64_t row0, int64_t m_global,
              const T* __restrict__ D, int64_t ldd, const uint32_t* __restrict__ mask, int64_t ldm,
              T* __restrict__ S, int64_t lds, T* __restrict__ LH, T* __restrict__ GH, T* __restrict__ SH,
              const double* __restrict__ u, const double* __restrict__ v, T* __restrict__ Lout, int64_t ldl,
              double* __restrict__ part) {
  if (MODE == kCpUpdate && st->done) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = ch.n, nh = ch.nh, np = ch.np;
  T* lrow = reinterpret_cast<T*>(smem_raw);  // np + 2
  T* rrow = lrow + np + 2;                   // n
  T* srow = rrow + n;                        // n
  __shared__ double scratch[5 * 32];
  __shared__ AmRec amw[32];
  const T* __restrict__ w0 = CpStencil<T>::w0(ch);
  const T* __restrict__ w1 = CpStencil<T>::w1(ch);
  const int* __restrict__ c0 = ch.c0;

  const double ga = MODE == kCpUpdate ? st->ga : 0.0;
  const double gb = MODE == kCpUpdate ? st->gb : 0.0;
  const double coef = MODE == kCpUpdate ? st->coef : 0.0;
  const T one_ga = (T)(1.0 - ga), one_gb = (T)(1.0 - gb);
  const T lam_s = (T)st->lam_s;
  const bool spike_on = MODE == kCpUpdate && st->corner_s;
  const long long i_s = st->i_s;
  const int j_s = st->j_s;
  const T spike_add = (T)(gb * st->spike);
  if (threadIdx.x < 2) lrow[np + threadIdx.x] = T(0);

  double a_sq = 0.0, a_l1 = 0.0, a_nnz = 0.0, a_ss = 0.0, a_sr = 0.0;
  AmRec best{0.0, 0.0, 0.0, -1};

  for (int64_t i = blockIdx.x; i < m; i += gridDim.x) {
    __syncthreads();
    T* lhrow = LH + i * np;
    if (MODE == kCpUpdate) {
      // coarse rank-1 update L_H <- (1-ga) L_H + ga * coef * u_i v^T  (cpcp.py:399-402)
      const double cu = ga * coef * u[i];
      for (int k = threadIdx.x; k < np; k += blockDim.x) {
        T val = k < nh ? (T)((double)one_ga * (double)lhrow[k] + cu * v[k]) : T(0);
        lrow[k] = val;
        lhrow[k] = val;
      }
    } else if (MODE == kCpOutput) {
      for (int k = threadIdx.x; k < np; k += blockDim.x) lrow[k] = lhrow[k];
    }
    __syncthreads();
    const T* drow = D + i * ldd;
    T* sro = S + i * lds;
    const uint32_t* mrow = mask ? mask + i * ldm : nullptr;
    const long long gi = row0 + i;
    const bool spike_row = spike_on && gi == i_s;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      if (MODE == kCpOutput) {
        const int c = c0[j];
        Lout[i * ldl + j] = w0[j] * lrow[c] + w1[j] * lrow[c + 1];
        continue;
      }
      const bool obs = mrow ? ((mrow[j >> 5] >> (j & 31)) & 1u) : true;
      T r = T(0), sn = T(0);
      if (MODE == kCpInit) {
        r = obs ? -drow[j] : T(0);
      } else {
        const int c = c0[j];
        const T l = w0[j] * lrow[c] + w1[j] * lrow[c + 1];
        T sh = one_gb * sro[j];
        if (spike_row && j == j_s) sh += spike_add;
        if (obs) {
          const T d = drow[j];
          const T rh = (l + sh) - d;                 // r after the segment step
          sn = soft_thr<T>(sh - rh, lam_s);         // cpcp.py:414-415
          r = (l + sn) - d;                          // r += P[S_new - S]
        } else {
          sn = soft_thr<T>(sh, lam_s);
        }
        sro[j] = sn;
      }
      rrow[j] = r;
      srow[j] = sn;
      const double rd = (double)r, sd = (double)sn;
      a_sq = fma(rd, rd, a_sq);
      a_l1 += fabs(sd);
      a_nnz += sn != T(0) ? 1.0 : 0.0;
      a_ss = fma(sd, sd, a_ss);
      a_sr = fma(sd, rd, a_sr);
      const double mg = fabs(rd);
      const long long idx = (long long)j * m_global + gi;
      if (argmax_better(mg, idx, best.mag, best.idx)) best = AmRec{mg, rd, sd, idx};
    }
    if (MODE == kCpOutput) continue;
    __syncthreads();
    // restrictions g_H = r R and s~ = S R for this row (gather stencil)
    T* grow = GH + i * np;
    T* shrow = SH + i * np;
    for (int k = threadIdx.x; k < np; k += blockDim.x) {
      T g = T(0), sg = T(0);
      if (k < nh) {
        const int lo = ch.lo[k], hi = ch.hi[k];
        for (int j = lo; j < hi; ++j) {
          const T w = c0[j] == k ? w0[j] : w1[j];
          g += rrow[j] * w;
          sg += srow[j] * w;
        }
      }
      grow[k] = g;
      shrow[k] = sg;
    }
  }
  if (MODE == kCpOutput) return;
  double vals[5] = {a_sq, a_l1, a_nnz, a_ss, a_sr};
  block_sum<5>(vals, scratch);
  best = am_warp(best);
  if ((threadIdx.x & 31) == 0) amw[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    AmRec b = amw[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) am_merge(b, amw[w]);
    double* p = part + 9 * blockIdx.x;
    for (int q = 0; q < 5; ++q) p[q] = vals[q];
    p[5] = b.mag;
    p[6] = b.val;
    p[7] = b.sval;
    p[8] = (double)b.idx;
  }
}

// Reduce per-CTA partials: stats -> out[0..5), arg-max record -> am[0..4)
// as (mag, val, sval, idx).
// Sum the per-CTA stats and merge the arg-max records (256 threads; fixed
// summation order; the arg-max merge is a total order, so order-free).
// out[kCpStats] is this rank's time-budget flag: summed by the stats
// all-reduce, so all ranks of a row-sharded solve stop together (cpcp.py:451).
__global__ void __launch_bounds__(256) cp_part_reduce(const double* __restrict__ part, int nparts,
                                                      double* __restrict__ out, double* __restrict__ am,
                                                      const CpcpDev* __restrict__ st) {
  __shared__ double scratch[kCpStats * 32];
  __shared__ AmRec amw[8];
  double v[kCpStats];
#pragma unroll
  for (int q = 0; q < kCpStats; ++q) v[q] = 0.0;
  AmRec b{0.0, 0.0, 0.0, -1};
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
    const double* p = part + 9 * i;
#pragma unroll
    for (int q = 0; q < kCpStats; ++q) v[q] += p[q];
    am_merge(b, AmRec{p[5], p[6], p[7], (long long)p[8]});
  }
  block_sum<kCpStats>(v, scratch);
  b = am_warp(b);
  if ((threadIdx.x & 31) == 0) amw[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < kCpStats; ++q) out[q] = v[q];
    const double wall = (cp_now_ns() - st->t0_ns) * 1e-9;
    out[kCpStats] = (st->time_budget >= 0.0 && wall >= st->time_budget) ? 1.0 : 0.0;
    AmRec r = amw[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) am_merge(r, amw[w]);
    am[0] = r.mag;
    am[1] = r.val;
    am[2] = r.sval;
    am[3] = (double)r.idx;
  }
}

__global__ void cp_start_scalars(CpcpDev* st, double lam_l, double lam_s, double tol, double radius, int max_iters,
                                 double time_budget, double m_global, double n) {
  st->lam_l = lam_l;
  st->lam_s = lam_s;
  st->tol = tol;
  st->radius = radius;
  st->time_budget = time_budget;
  st->m_global = m_global;
  st->n = n;
  st->rtol = 1e-6;        // _LeadingTriple value_rtol (cpcp.py:299)
  st->max_passes = 40;    // _LeadingTriple max_passes (cpcp.py:299)
  st->max_iters = max_iters;
  st->t_l = st->t_s = 0.0;
  st->ga = st->gb = 0.0;
  st->corner_l = st->corner_s = 0;
  st->coef = 0.0;
  st->spike = 0.0;
  st->i_s = -1;
  st->j_s = -1;
  st->k = 0;
  st->done = 0;
  st->status = 0;
  st->rank_l = -1.0;
  st->t0_ns = cp_now_ns();
}

// initial_bounds (cpcp.py:121-131) and the P[D] = 0 early exit (cpcp.py:348-350)
__global__ void cp_begin_kernel(CpcpDev* st, const double* __restrict__ stats, double* __restrict__ hist,
                                double* __restrict__ objh) {
  const double sq = stats[0];
  st->u_l = sq / (2.0 * st->lam_l);
  st->u_s = sq / (2.0 * st->lam_s);
  st->pd_norm = sqrt(sq);
  st->sq = sq;
  st->l1 = 0.0;
  st->nnz = 0.0;
  st->ss = 0.0;
  st->sr = 0.0;
  st->k = 1;
  if (st->u_l == 0.0) {
    st->done = 1;
    st->k = 1;
    double* h = hist;
    for (int q = 0; q < kCpHistCols; ++q) h[q] = 0.0;
    objh[0] = 0.0;
  }
}

// Warm-started power iteration on K_g = g_H^T g_H (exact restatement of
// _LeadingTriple, cpcp.py:304-323: s2 = v^T K v, w = K v / sqrt(s2),
// nw = |w|, v <- w / nw, stop when |s2 - s2_prev| <= rtol s2).  One cluster;
// CTA c owns rows [c*R, (c+1)*R) of K in shared memory when they fit.
constexpr int kPowThreads = 512;

__global__ void __launch_bounds__(kPowThreads)
cp_power_kernel(CpcpDev* __restrict__ st, const double* __restrict__ K, int np, double* __restrict__ v,
                double* __restrict__ vin, int rows_in_smem) {
  if (st->done) return;
  cg::cluster_group cluster = cg::this_cluster();
  const int cr = (int)cluster.block_rank();
  const int cs = (int)cluster.num_blocks();
  const int R = np / cs;
  extern __shared__ __align__(16) double psm[];
  double* vv = psm;            // np : current v
  double* kvb = vv + np;       // 2 x np : K v (full, gathered), double-buffered by pass parity
  double* red = kvb + 2 * np;  // 64
  double* krows = red + 64;    // R x np (optional)
  const int tid = threadIdx.x;
  for (int j = tid; j < np; j += kPowThreads) vv[j] = v[j];
  if (rows_in_smem)
    for (int e = tid; e < R * np; e += kPowThreads) krows[e] = K[(int64_t)cr * R * np + e];
  __syncthreads();
  const int lane = tid & 31, wid = tid >> 5, nw = kPowThreads / 32;
  double s2_prev = -1.0, s2 = 0.0, nwv = 0.0;
  int none = 0, pass = 0;
  const double rtol = st->rtol;
  const int maxp = st->max_passes;
  for (pass = 1; pass <= maxp; ++pass) {
    // local rows of K v, pushed to every CTA of the cluster.  kv alternates
    // between two buffers, so the one cluster barrier per pass also orders
    // the reuse (a CTA writes this buffer again only two passes later, after
    // every CTA has passed the barrier that follows its reads)
    double* kv = kvb + (pass & 1) * np;
    for (int rr = wid; rr < R; rr += nw) {
      const double* krow = rows_in_smem ? krows + (int64_t)rr * np : K + (int64_t)(cr * R + rr) * np;
      double s = 0.0;
      for (int j = lane; j < np; j += 32) s = fma(krow[j], vv[j], s);
      s = warp_sum(s);
      if (lane == 0) {
        for (int q = 0; q < cs; ++q) {
          double* dst = cluster.map_shared_rank(kv, q);
          dst[cr * R + rr] = s;
        }
      }
    }
    cluster.sync();
    // s2 = v . Kv, |Kv|^2 (identical in every CTA)
    double a = 0.0, b = 0.0;
    for (int j = tid; j < np; j += kPowThreads) {
      a = fma(vv[j], kv[j], a);
      b = fma(kv[j], kv[j], b);
    }
    a = warp_sum(a);
    b = warp_sum(b);
    if (lane == 0) {
      red[wid] = a;
      red[32 + wid] = b;
    }
    __syncthreads();
    if (tid == 0) {
      double sa = 0.0, sb = 0.0;
      for (int w = 0; w < nw; ++w) {
        sa += red[w];
        sb += red[32 + w];
      }
      red[62] = sa;
      red[63] = sb;
    }
    __syncthreads();
    s2 = red[62];
    const double kvn = sqrt(red[63]);
    if (s2 <= 0.0 || kvn == 0.0) {
      none = 1;
      break;
    }
    nwv = kvn / sqrt(s2);
    // vin <- v ; v <- Kv / |Kv|
    for (int j = tid; j < np; j += kPowThreads) {
      if (cr == 0) vin[j] = vv[j];
      vv[j] = kv[j] / kvn;
    }
    const bool stop = fabs(s2 - s2_prev) <= rtol * s2;
    s2_prev = s2;
    __syncthreads();  // vv complete before this CTA's next Kv rows read it
    if (stop) break;
  }
  if (pass > maxp) pass = maxp;
  if (cr == 0) {
    if (!none)
      for (int j = tid; j < np; j += kPowThreads) v[j] = vv[j];
    if (tid == 0) {
      st->none = none;
      st->s2 = none ? 0.0 : s2;
      st->sigma = none ? 0.0 : nwv;
      st->passes = pass;
    }
  }
}

// Full-width LMO (identity chain, one rank): the _LeadingTriple passes
// (cpcp.py:304-323) as matvecs on g = g_H (m x n_p, T), on a cooperative
// grid: t = g v (warp per row) | z partials = g^T t over row blocks |
// column-sliced fixed-order reduction of z, ||z||^2 | v <- z / ||z||.
// s2 = ||g v||^2 is the same Rayleigh quotient the Gram path forms as v^T K v.
constexpr int kFineThreads = 256;

__device__ __forceinline__ double fine_sum(const double* __restrict__ part, int stride, int count) {
  // fixed-order sum of count partials by one warp (identical in every CTA)
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int i = lane; i < count; i += 32) s += part[i * stride];
  return warp_sum(s);
}

template <typename T>
__global__ void __launch_bounds__(kFineThreads)
cp_power_fine_kernel(CpcpDev* __restrict__ st, const T* __restrict__ G, int64_t m, int np, double* __restrict__ v,
                     double* __restrict__ vin, double* __restrict__ t, double* __restrict__ z,
                     double* __restrict__ v0, double* __restrict__ zpart, double* __restrict__ spart) {
  if (st->done) return;  // uniform: every CTA reads the same flag
  cg::grid_group grid = cg::this_grid();
  const int P = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int W = kFineThreads / 32;
  __shared__ double red[W];
  __shared__ double bc[2];
  const double rtol = st->rtol;
  const int maxp = st->max_passes;
  const int cw = (np + P - 1) / P;  // column slice per CTA
  const int c0 = b * cw, c1 = min(np, c0 + cw);
  for (int j = c0 + tid; j < c1; j += kFineThreads) v0[j] = v[j];
  const int64_t rb = (m + P - 1) / P;
  const int64_t r0 = b * rb, r1 = min(m, r0 + rb);
  double s2_prev = -1.0, s2 = 0.0, nwv = 0.0;
  int none = 0, pass = 0;
  for (pass = 1; pass <= maxp; ++pass) {
    // t = g v and per-CTA partial of ||t||^2
    double ss = 0.0;
    for (int64_t i = (int64_t)b * W + wid; i < m; i += (int64_t)P * W) {
      const T* row = G + i * np;
      double acc = 0.0;
      for (int j = lane; j < np; j += 32) acc = fma((double)row[j], v[j], acc);
      acc = warp_sum(acc);
      if (lane == 0) {
        t[i] = acc;
        ss = fma(acc, acc, ss);
      }
    }
    if (lane == 0) red[wid] = ss;
    __syncthreads();
    if (tid == 0) {
      double q = 0.0;
      for (int w = 0; w < W; ++w) q += red[w];
      spart[2 * b] = q;
    }
    grid.sync();
    // z partials over this CTA's row block, 8 columns per thread
    for (int j0 = tid * 8; j0 < np; j0 += kFineThreads * 8) {
      double acc[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = 0.0;
      for (int64_t i = r0; i < r1; ++i) {
        const double ti = t[i];
        const T* row = G + i * np + j0;
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (j0 + e < np) acc[e] = fma((double)row[e], ti, acc[e]);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (j0 + e < np) zpart[(int64_t)b * np + j0 + e] = acc[e];
    }
    grid.sync();
    // z = sum of the partials (column slice), ||z||^2 partial
    double zz = 0.0;
    for (int j = c0 + tid; j < c1; j += kFineThreads) {
      double acc = 0.0;
      for (int q = 0; q < P; ++q) acc += zpart[(int64_t)q * np + j];
      z[j] = acc;
      zz = fma(acc, acc, zz);
    }
    zz = warp_sum(zz);
    if (lane == 0) red[wid] = zz;
    __syncthreads();
    if (tid == 0) {
      double q = 0.0;
      for (int w = 0; w < W; ++w) q += red[w];
      spart[2 * b + 1] = q;
    }
    grid.sync();
    if (wid == 0) {
      const double a = fine_sum(spart, 2, P);
      const double c = fine_sum(spart + 1, 2, P);
      if (lane == 0) {
        bc[0] = a;
        bc[1] = c;
      }
    }
    __syncthreads();
    s2 = bc[0];
    const double kvn = sqrt(bc[1]);
    if (s2 <= 0.0 || kvn == 0.0) {
      none = 1;
      break;
    }
    nwv = kvn / sqrt(s2);
    for (int j = c0 + tid; j < c1; j += kFineThreads) {
      vin[j] = v[j];
      v[j] = z[j] / kvn;
    }
    const bool stop = fabs(s2 - s2_prev) <= rtol * s2;
    s2_prev = s2;
    grid.sync();  // v complete before the next pass reads it
    if (stop) break;
  }
  if (pass > maxp) pass = maxp;
  if (none) {  // the reference keeps its previous right vector
    for (int j = c0 + tid; j < c1; j += kFineThreads) v[j] = v0[j];
  }
  if (b == 0 && tid == 0) {
    st->none = none;
    st->s2 = none ? 0.0 : s2;
    st->sigma = none ? 0.0 : nwv;
    st->passes = pass;
  }
}

// Corner selection (cpcp.py:361-368), arg-max pick across ranks.
__global__ void cp_lmo_scalars(CpcpDev* st, const double* __restrict__ am_all, int world) {
  if (st->done) return;
  AmRec b{0.0, 0.0, 0.0, -1};
  for (int q = 0; q < world; ++q) {
    const double* a = am_all + 4 * q;
    AmRec c{a[0], a[1], a[2], (long long)a[3]};
    am_merge(b, c);
  }
  if (b.idx < 0) b = AmRec{0.0, 0.0, 0.0, 0};  // all-zero residual: (0,0)
  const long long mg = (long long)st->m_global;
  st->idx_is = b.idx;
  st->j_s = (int)(b.idx / mg);
  st->i_s = b.idx % mg;
  st->r_is = b.val;
  st->s_is = b.sval;
  const double val_l = st->none ? 0.0 : -st->radius * st->sigma;
  const double val_s = -fabs(b.val);
  st->corner_l = st->lam_l < -val_l;
  st->corner_s = st->lam_s < -val_s;
  st->v_tl = st->corner_l ? st->u_l : 0.0;
  st->v_ts = st->corner_s ? st->u_s : 0.0;
  st->coef = st->corner_l ? -st->radius * st->u_l : 0.0;
  st->spike = st->corner_s ? -st->u_s * (b.val > 0.0 ? 1.0 : (b.val < 0.0 ? -1.0 : 0.0)) : 0.0;
}

// Masked chain Gram per row, once per solve: M_i = sum_j mask_ij R_j^T R_j is
// tridiagonal (R_j has two adjacent taps), so the segment-QP quadratic form
// aa = sum_ij mask_ij (E_i R_j^T)^2 = sum_i E_i M_i E_i^T needs no fine pass.
//   mgd[i][k] = sum_{j in [lo_k, hi_k)} mask_ij (weight of j on k)^2
//   mgo[i][k] = sum_{j : c0_j = k} mask_ij w0_j w1_j
template <typename T>
__global__ void __launch_bounds__(256) cp_maskgram_kernel(ChainDev ch, int64_t m, const uint32_t* __restrict__ mask,
                                                          int64_t ldm, T* __restrict__ mgd, T* __restrict__ mgo) {
  const int np = ch.np, nh = ch.nh;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * np; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / np;
    const int k = (int)(e % np);
    double d = 0.0, o = 0.0;
    if (k < nh) {
      const uint32_t* mrow = mask + i * ldm;
      for (int j = ch.lo[k]; j < ch.hi[k]; ++j) {
        if (!((__ldg(mrow + (j >> 5)) >> (j & 31)) & 1u)) continue;
        const bool own = ch.c0[j] == k;
        const double w = own ? ch.w0[j] : ch.w1[j];
        d = fma(w, w, d);
        if (own) o = fma(ch.w0[j], ch.w1[j], o);
      }
    }
    mgd[e] = (T)d;
    mgo[e] = (T)o;
  }
}

// Segment-QP dots from coarse data only (warp per row):
//   u_i = g_H[i] . vin / sqrt(s2), E_i = coef u_i v - L_H[i]
//   aa += E_i M_i E_i^T (M_i from cp_maskgram_kernel, or G_R when fully observed)
//   ab += -E_i . s~_i (+ spike * a_{i_s j_s}),  ar += E_i . g_H[i]
template <typename T>
__global__ void __launch_bounds__(256)
cp_dots_coarse_kernel(const CpcpDev* __restrict__ st, ChainDev ch, int64_t m, int64_t row0, const T* __restrict__ LH,
                      const T* __restrict__ GH, const T* __restrict__ SH, const T* __restrict__ mgd,
                      const T* __restrict__ mgo, const double* __restrict__ v, const double* __restrict__ vin,
                      double* __restrict__ u, double* __restrict__ part) {
  if (st->done) return;
  __shared__ double scratch[3 * 32];
  const int nh = ch.nh, np = ch.np;
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const int64_t wglob = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5);
  const int64_t wstride = (int64_t)gridDim.x * warps;
  const double coef = st->coef;
  const double rs2 = st->none ? 0.0 : 1.0 / sqrt(st->s2);
  const bool spike_on = st->corner_s;
  const long long i_s = st->i_s;
  const int j_s = st->j_s;
  const double spike = st->spike;
  double aa = 0.0, ab = 0.0, ar = 0.0;
  for (int64_t i = wglob; i < m; i += wstride) {
    const T* g = GH + i * np;
    const T* lh = LH + i * np;
    const T* sh = SH + i * np;
    double d = 0.0;
    for (int k = lane; k < nh; k += 32) d = fma((double)g[k], vin[k], d);
    d = warp_sum(d);
    const double ui = st->none ? 0.0 : d * rs2;
    if (lane == 0) u[i] = ui;
    const double cu = coef * ui;
    double e_ab = 0.0, e_ar = 0.0, e_aa = 0.0;
    for (int k = lane; k < nh; k += 32) {
      const double e = cu * v[k] - (double)lh[k];
      const double e1 = k + 1 < nh ? cu * v[k + 1] - (double)lh[k + 1] : 0.0;
      double dk, ok;
      if (mgd) {
        dk = (double)mgd[i * np + k];
        ok = (double)mgo[i * np + k];
      } else {  // fully observed: M_i = G_R = L D L^T (tridiagonal)
        dk = ch.gd[k] + (k > 0 ? ch.gl[k - 1] * ch.gl[k - 1] * ch.gd[k - 1] : 0.0);
        ok = k + 1 < nh ? ch.gl[k] * ch.gd[k] : 0.0;
      }
      e_aa = fma(e * dk, e, e_aa);
      e_aa = fma(2.0 * e * ok, e1, e_aa);
      e_ab = fma(e, (double)sh[k], e_ab);
      e_ar = fma(e, (double)g[k], e_ar);
    }
    ab -= e_ab;
    ar += e_ar;
    aa += e_aa;
    if (spike_on && (row0 + i) == i_s && lane == 0) {
      const int c = ch.c0[j_s];
      const double ec = cu * v[c] - (double)lh[c];
      const double ec1 = c + 1 < nh ? cu * v[c + 1] - (double)lh[c + 1] : 0.0;
      ab += spike * (ec * ch.w0[j_s] + ec1 * ch.w1[j_s]);
    }
  }
  double vals[3] = {aa, ab, ar};
  block_sum<3>(vals, scratch);
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x + 0] = vals[0];
    part[3 * blockIdx.x + 1] = vals[1];
    part[3 * blockIdx.x + 2] = vals[2];
  }
}

// FP32 masked variant of cp_dots_coarse_kernel: each lane owns 4 consecutive
// coarse columns and moves them as float4 (one 16-byte load per array per
// 128 columns instead of four 4-byte loads), and with n_p <= 128 (SEG1) all
// five coarse rows are loaded before the u_i reduction so their latency
// overlaps it.  E_i's right neighbour (the tridiagonal term) comes from the
// next lane by a shuffle.
template <bool SEG1>
__global__ void __launch_bounds__(256)
cp_dots_coarse_v4(const CpcpDev* __restrict__ st, ChainDev ch, int64_t m, int64_t row0, const float* __restrict__ LH,
                  const float* __restrict__ GH, const float* __restrict__ SH, const float* __restrict__ mgd,
                  const float* __restrict__ mgo, const double* __restrict__ v, const double* __restrict__ vin,
                  double* __restrict__ u, double* __restrict__ part) {
  if (st->done) return;
  __shared__ double scratch[3 * 32];
  const int nh = ch.nh, np = ch.np;
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const int64_t wglob = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5);
  const int64_t wstride = (int64_t)gridDim.x * warps;
  const double coef = st->coef;
  const double rs2 = st->none ? 0.0 : 1.0 / sqrt(st->s2);
  const bool spike_on = st->corner_s;
  const long long i_s = st->i_s;
  const int j_s = st->j_s;
  const double spike = st->spike;
  double aa = 0.0, ab = 0.0, ar = 0.0;
  auto ld4 = [](const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); };
  const int k1 = lane * 4;
  // SEG1: the next row's five coarse rows are in flight while this one is evaluated
  float4 n_g = make_float4(0.f, 0.f, 0.f, 0.f), n_l = n_g, n_s = n_g, n_d = n_g, n_o = n_g;
  auto prefetch = [&](int64_t r) {
    if (SEG1 && r < m && k1 < np) {
      n_g = ld4(GH + r * np + k1);
      n_l = ld4(LH + r * np + k1);
      n_s = ld4(SH + r * np + k1);
      n_d = ld4(mgd + r * np + k1);
      n_o = ld4(mgo + r * np + k1);
    }
  };
  prefetch(wglob);
  for (int64_t i = wglob; i < m; i += wstride) {
    const float* g = GH + i * np;
    const float* lh = LH + i * np;
    const float* sh = SH + i * np;
    const float* md = mgd + i * np;
    const float* mo = mgo + i * np;
    const float4 g4 = n_g, l4 = n_l, s4 = n_s, d4 = n_d, o4 = n_o;
    prefetch(i + wstride);
    double d = 0.0;
    for (int base = 0; base < np; base += 128) {
      const int k = base + k1;
      if (k >= np) break;
      const float4 gg = SEG1 ? g4 : ld4(g + k);
      const float gv[4] = {gg.x, gg.y, gg.z, gg.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (k + q < nh) d = fma((double)gv[q], vin[k + q], d);
    }
    d = warp_sum(d);
    const double ui = st->none ? 0.0 : d * rs2;
    if (lane == 0) u[i] = ui;
    const double cu = coef * ui;
    double e_ab = 0.0, e_ar = 0.0, e_aa = 0.0;
    for (int base = 0; base < np; base += 128) {  // uniform trip count (shuffles below)
      const int k = base + k1;
      const bool act = k < np;
      float4 gg = g4, ll = l4, ss = s4, dd = d4, oo = o4;
      if (!SEG1 && act) {
        gg = ld4(g + k);
        ll = ld4(lh + k);
        ss = ld4(sh + k);
        dd = ld4(md + k);
        oo = ld4(mo + k);
      }
      const float gv[4] = {gg.x, gg.y, gg.z, gg.w}, lv[4] = {ll.x, ll.y, ll.z, ll.w};
      const float sv[4] = {ss.x, ss.y, ss.z, ss.w}, dv[4] = {dd.x, dd.y, dd.z, dd.w};
      const float ov[4] = {oo.x, oo.y, oo.z, oo.w};
      double e[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) e[q] = (act && k + q < nh) ? cu * v[k + q] - (double)lv[q] : 0.0;
      double enext = __shfl_down_sync(0xffffffffu, e[0], 1);
      if (lane == 31) {  // first column of the next 128-column segment
        const int kn = base + 128;
        enext = kn < nh ? cu * v[kn] - (double)lh[kn] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double e1 = q < 3 ? e[q + 1] : enext;
        e_aa = fma(e[q] * (double)dv[q], e[q], e_aa);
        e_aa = fma(2.0 * e[q] * (double)ov[q], e1, e_aa);
        e_ab = fma(e[q], (double)sv[q], e_ab);
        e_ar = fma(e[q], (double)gv[q], e_ar);
      }
    }
    ab -= e_ab;
    ar += e_ar;
    aa += e_aa;
    if (spike_on && (row0 + i) == i_s && lane == 0) {
      const int c = ch.c0[j_s];
      const double ec = cu * v[c] - (double)lh[c];
      const double ec1 = c + 1 < nh ? cu * v[c + 1] - (double)lh[c + 1] : 0.0;
      ab += spike * (ec * ch.w0[j_s] + ec1 * ch.w1[j_s]);
    }
  }
  double vals[3] = {aa, ab, ar};
  block_sum<3>(vals, scratch);
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x + 0] = vals[0];
    part[3 * blockIdx.x + 1] = vals[1];
    part[3 * blockIdx.x + 2] = vals[2];
  }
}

// Per-row coarse evaluation of the segment-QP dots (warp per row):
//   u_i  = g_H[i] . vin / sqrt(s2)           (left vector of the triple)
//   E_i  = coef * u_i * v - L_H[i]          (a = P[E R^T])
//   aa  += sum_j mask_ij (E_i . R_j)^2
//   ab  += -E_i . s~_i  (+ spike * a_{i_s j_s})
//   ar  +=  E_i . g_H[i]
template <typename T>
__global__ void __launch_bounds__(256)
cp_dots_kernel(const CpcpDev* __restrict__ st, ChainDev ch, int64_t m, int64_t row0, const uint32_t* __restrict__ mask,
               int64_t ldm, const T* __restrict__ LH, const T* __restrict__ GH, const T* __restrict__ SH,
               const double* __restrict__ v, const double* __restrict__ vin, double* __restrict__ u,
               double* __restrict__ part) {
  if (st->done) return;
  __shared__ double scratch[3 * 32];
  const int n = ch.n, nh = ch.nh, np = ch.np;
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const int64_t wglob = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5);
  const int64_t wstride = (int64_t)gridDim.x * warps;
  const double coef = st->coef;
  const double rs2 = st->none ? 0.0 : 1.0 / sqrt(st->s2);
  const bool spike_on = st->corner_s;
  const long long i_s = st->i_s;
  const int j_s = st->j_s;
  const double spike = st->spike;
  const int* __restrict__ c0 = ch.c0;
  const double* __restrict__ w0 = ch.w0;
  const double* __restrict__ w1 = ch.w1;
  double aa = 0.0, ab = 0.0, ar = 0.0;
  for (int64_t i = wglob; i < m; i += wstride) {
    const T* g = GH + i * np;
    const T* lh = LH + i * np;
    const T* sh = SH + i * np;
    double d = 0.0;
    for (int k = lane; k < nh; k += 32) d = fma((double)g[k], vin[k], d);
    d = warp_sum(d);
    const double ui = st->none ? 0.0 : d * rs2;
    if (lane == 0) u[i] = ui;
    const double cu = coef * ui;
    double e_ab = 0.0, e_ar = 0.0;
    for (int k = lane; k < nh; k += 32) {
      const double e = cu * v[k] - (double)lh[k];
      e_ab = fma(e, (double)sh[k], e_ab);
      e_ar = fma(e, (double)g[k], e_ar);
    }
    ab -= e_ab;
    ar += e_ar;
    const uint32_t* mrow = mask ? mask + i * ldm : nullptr;
    double e_aa = 0.0;
    const bool srow = spike_on && (row0 + i) == i_s;
    for (int j = lane; j < n; j += 32) {
      const bool obs = mrow ? ((mrow[j >> 5] >> (j & 31)) & 1u) : true;
      if (!obs) continue;
      const int c = c0[j];
      const double ec = cu * v[c] - (double)lh[c];
      const double ec1 = c + 1 < nh ? cu * v[c + 1] - (double)lh[c + 1] : 0.0;
      const double a = ec * w0[j] + ec1 * w1[j];
      e_aa = fma(a, a, e_aa);
      if (srow && j == j_s) ab += spike * a;
    }
    aa += e_aa;
  }
  double vals[3] = {aa, ab, ar};
  block_sum<3>(vals, scratch);
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x + 0] = vals[0];
    part[3 * blockIdx.x + 1] = vals[1];
    part[3 * blockIdx.x + 2] = vals[2];
  }
}

__global__ void __launch_bounds__(256) cp_dots_reduce(const double* __restrict__ part, int nparts,
                                                      double* __restrict__ out, const CpcpDev* __restrict__ st) {
  if (st->done) return;
  __shared__ double scratch[3 * 32];
  double v[3] = {0.0, 0.0, 0.0};
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
    v[0] += part[3 * i];
    v[1] += part[3 * i + 1];
    v[2] += part[3 * i + 2];
  }
  block_sum<3>(v, scratch);
  if (threadIdx.x == 0) {
    out[0] = v[0];
    out[1] = v[1];
    out[2] = v[2];
  }
}

// _solve_box_qp / _coord_min (cpcp.py:195-231), FP64, evaluated in the
// reference's operation order with non-contractible intrinsics (no FMA
// fusion), so the step sizes are bit-identical to numpy's for the same
// inputs (tests/test_gpu_large.py::test_box_qp_bitwise).
__device__ double coord_min(double quad, double lin) {
  if (quad <= 0.0) return lin < 0.0 ? 1.0 : 0.0;
  return fmin(fmax(__ddiv_rn(-lin, quad), 0.0), 1.0);
}

__device__ void box_qp(double aa, double bb, double ab, double la, double lb, double fb, double& ga, double& gb) {
  // value(ga, gb) = .5*(aa*ga*ga + 2*ab*ga*gb + bb*gb*gb) + la*ga + lb*gb, left to right
  auto q = [&](double x, double y) {
    double s = __dadd_rn(__dmul_rn(__dmul_rn(aa, x), x), __dmul_rn(__dmul_rn(__dmul_rn(2.0, ab), x), y));
    s = __dadd_rn(s, __dmul_rn(__dmul_rn(bb, y), y));
    s = __dmul_rn(0.5, s);
    s = __dadd_rn(s, __dmul_rn(la, x));
    return __dadd_rn(s, __dmul_rn(lb, y));
  };
  const double det = __dsub_rn(__dmul_rn(aa, bb), __dmul_rn(ab, ab));
  bool have = false;
  if (det > 0.0) {
    const double x = __ddiv_rn(__dadd_rn(__dmul_rn(-la, bb), __dmul_rn(lb, ab)), det);
    const double y = __ddiv_rn(__dadd_rn(__dmul_rn(-lb, aa), __dmul_rn(la, ab)), det);
    if (x >= 0.0 && x <= 1.0 && y >= 0.0 && y <= 1.0) {
      ga = x;
      gb = y;
      have = true;
    }
  }
  if (!have) {
    double x = 0.0, y = 0.0;
    for (int it = 0; it < 200; ++it) {
      const double xn = coord_min(aa, __dadd_rn(la, __dmul_rn(ab, y)));
      const double yn = coord_min(bb, __dadd_rn(lb, __dmul_rn(ab, xn)));
      const bool stop = fabs(__dsub_rn(xn, x)) <= 1e-12 && fabs(__dsub_rn(yn, y)) <= 1e-12;
      x = xn;
      y = yn;
      if (stop) break;
    }
    ga = x;
    gb = y;
  }
  if (fb >= 0.0 || fb < 0.0) {  // fallback given (NaN = none, as the reference's None)
    const double gf = fmin(fmax(fb, 0.0), 1.0);
    if (q(gf, gf) < q(ga, gb)) {
      ga = gf;
      gb = gf;
    }
  }
}

// Test entry: out[2i], out[2i+1] = box_qp(in[6i .. 6i+5]) (aa, bb, ab, la, lb, fallback or NaN)
__global__ void box_qp_batch_kernel(const double* __restrict__ in, double* __restrict__ out, int count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const double* c = in + 6 * (int64_t)i;
  double ga = 0.0, gb = 0.0;
  box_qp(c[0], c[1], c[2], c[3], c[4], c[5], ga, gb);
  out[2 * (int64_t)i] = ga;
  out[2 * (int64_t)i + 1] = gb;
}

int box_qp_batch(const double* in, double* out, int count, cudaStream_t st) {
  if (count <= 0) return kOk;
  box_qp_batch_kernel<<<(count + 127) / 128, 128, 0, st>>>(in, out, count);
  MLR_LAUNCH_CHECK("box_qp_batch_kernel");
  return kOk;
}

__global__ void cp_qp_kernel(CpcpDev* st, const double* __restrict__ dots) {
  if (st->done) return;
  const double aa = dots[0], ab = dots[1], ar = dots[2];
  double bb = st->ss, br = -st->sr;
  if (st->corner_s) {
    bb += st->spike * st->spike - 2.0 * st->spike * st->s_is;
    br += st->spike * st->r_is;
  }
  const double la = ar + st->lam_l * (st->v_tl - st->t_l);
  const double lb = br + st->lam_s * (st->v_ts - st->t_s);
  double ga = 0.0, gb = 0.0;
  box_qp(aa, bb, ab, la, lb, 2.0 / (st->k + 2.0), ga, gb);
  st->ga = ga;
  st->gb = gb;
  st->t_l += ga * (st->v_tl - st->t_l);
  st->t_s += gb * (st->v_ts - st->t_s);
}

// Objective, bound update, history, 5-window convergence (cpcp.py:429-452).
__global__ void cp_finalize_kernel(CpcpDev* st, const double* __restrict__ stats, double* __restrict__ hist,
                                   double* __restrict__ objh) {
  if (st->done) return;
  const int k = st->k;
  st->sq = stats[0];
  st->l1 = stats[1];
  st->nnz = stats[2];
  st->ss = stats[3];
  st->sr = stats[4];
  st->t_s = st->l1;
  const double obj = 0.5 * st->sq + st->lam_l * st->t_l + st->lam_s * st->t_s;
  st->u_l = fmin(st->u_l, obj / st->lam_l);
  st->u_s = fmin(st->u_s, obj / st->lam_s);
  objh[k - 1] = obj;
  const double wall = (cp_now_ns() - st->t0_ns) * 1e-9;
  double* h = hist + (int64_t)(k - 1) * kCpHistCols;
  h[0] = sqrt(st->sq) / st->pd_norm;
  h[1] = obj;
  h[2] = st->rank_l;
  h[3] = st->nnz / (st->m_global * st->n);
  h[4] = wall;
  h[5] = st->ga;
  h[6] = st->gb;
  h[7] = (double)st->passes;
  bool conv = false;
  if (k > 5) {
    const double prev = objh[k - 6];
    conv = prev - obj <= st->tol * fmax(fabs(prev), 2.2250738585072014e-308);
  }
  if (conv) {
    st->done = 1;
  } else if (k >= st->max_iters || stats[kCpStats] > 0.0) {
    st->done = 2;
  } else {
    st->k = k + 1;
  }
}

// FP64 shadow of the coarse iterate for collect_rank on FP32 data: the same
// rank-1 update as the fused row pass (L_H <- (1-ga) L_H + ga coef u v^T,
// cpcp.py:399-402) without rounding to FP32, so the numerical rank sees the
// iterate the reference's float64 run holds rather than FP32 rounding noise.
__global__ void __launch_bounds__(256) cp_shadow_kernel(const CpcpDev* __restrict__ st, int64_t m, int nh,
                                                        const double* __restrict__ u, const double* __restrict__ v,
                                                        double* __restrict__ L64, int64_t ld) {
  if (st->done) return;
  const double ga = st->ga, one_ga = 1.0 - ga, gc = ga * st->coef;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * nh; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / nh;
    const int k = (int)(e % nh);
    double* p = L64 + i * ld + k;
    *p = one_ga * *p + (gc * u[i]) * v[k];
  }
}

// track_oracle_atoms (cpcp.py:355-360): the LMO atom of one iteration,
// M_L = -radius * u (R v)^T (cpcp.py:506-513; fwt_solve: -u v^T), from the
// factors saved after that iteration's LMO step.  Dense m_local x n, float64.
__global__ void __launch_bounds__(256) cp_atom_kernel(const CpcpDev* __restrict__ st, ChainDev ch, int64_t m,
                                                      const double* __restrict__ u, const double* __restrict__ v,
                                                      double* __restrict__ out, int64_t ldo) {
  const double nr = -st->radius;
  const int n = ch.n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n;
    const int j = (int)(e % n);
    const int c = ch.c0[j];
    // m_h[i][c] = (-radius) * (u_i v_c), then m_h @ R^T (two taps)
    double a = nr * (u[i] * v[c]) * ch.w0[j];
    if (ch.w1[j] != 0.0) a += nr * (u[i] * v[c + 1]) * ch.w1[j];
    out[i * ldo + j] = a;
  }
}

int cpcp_atom_copy(CpcpPlan* p, double* u_out, double* v_out, cudaStream_t st) {
  if (p->m_local > 0)
    MLR_CUDA(cudaMemcpyAsync(u_out, p->u, sizeof(double) * p->m_local, cudaMemcpyDeviceToDevice, st));
  MLR_CUDA(cudaMemcpyAsync(v_out, p->v, sizeof(double) * p->ch.nh, cudaMemcpyDeviceToDevice, st));
  return kOk;
}

int cpcp_atom_dense(CpcpPlan* p, const double* u, const double* v, double* out, int64_t ldo, cudaStream_t st) {
  if (p->m_local == 0) return kOk;
  const int blocks = (int)std::min<int64_t>(ceil_div(p->m_local * p->ch.n, 256), 148 * 16);
  cp_atom_kernel<<<blocks, 256, 0, st>>>(p->dev, p->ch, p->m_local, u, v, out, ldo);
  MLR_LAUNCH_CHECK("cp_atom_kernel");
  return kOk;
}

int cpcp_rank_shadow(CpcpPlan* p, double* L64, int64_t ld, cudaStream_t st) {
  if (p->m_local == 0) return kOk;
  const int blocks = (int)std::min<int64_t>(ceil_div(p->m_local * p->ch.nh, 256), 148 * 8);
  cp_shadow_kernel<<<blocks, 256, 0, st>>>(p->dev, p->m_local, p->ch.nh, p->u, p->v, L64, ld);
  MLR_LAUNCH_CHECK("cp_shadow_kernel");
  return kOk;
}

// ------------------------------------------------------------ host drivers
template <typename T, int MODE>
static int cp_row(CpcpPlan* p, const void* D, int64_t ldd, const uint32_t* mask, int64_t ldm, void* S, int64_t lds,
                  void* Lout, int64_t ldl, cudaStream_t st) {
  if (p->m_local == 0) return kOk;
  if (rows_warp_ok(p->ch, p->f32))  // streaming warp-per-row path (rows.cu)
    return cp_rows(p, MODE, D, ldd, mask, ldm, S, lds, Lout, ldl, st);
  size_t smem = sizeof(T) * (size_t)(p->ch.np + 2 + 2 * p->ch.n);
  if (smem > 200 * 1024) {
    set_error("cpcp row kernel: fine row does not fit in shared memory");
    return kErrArg;
  }
  auto kern = cp_row_kernel<T, MODE>;
  MLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<p->row_blocks, 256, smem, st>>>(p->dev, p->ch, p->m_local, p->row0, p->m_global, (const T*)D, ldd, mask,
                                         ldm, (T*)S, lds, (T*)p->LH, (T*)p->GH, (T*)p->SH, p->u, p->v, (T*)Lout, ldl,
                                         p->row_part);
  MLR_LAUNCH_CHECK("cp_row_kernel");
  return kOk;
}

int cpcp_start(CpcpPlan* p, const void* D, int64_t ldd, const uint32_t* mask, int64_t ldm, void* S, int64_t lds,
               double lam_l, double lam_s, double tol, double radius, int max_iters, double time_budget,
               cudaStream_t st) {
  const size_t tb = p->f32 ? 4 : 8;
  p->mask_dev = mask;
  p->ldm_dev = ldm;
  cp_start_scalars<<<1, 1, 0, st>>>(p->dev, lam_l, lam_s, tol, radius, max_iters, time_budget,
                                    (double)p->m_global, (double)p->ch.n);
  MLR_LAUNCH_CHECK("cp_start_scalars");
  const int np = p->ch.np;
  MLR_CUDA(cudaMemsetAsync(p->hist, 0, sizeof(double) * kCpHistCols * p->max_iters, st));
  if (p->m_local > 0 && p->coarse_dots && mask) {
    const int blocks = (int)std::min<int64_t>(ceil_div(p->m_local * np, 256), 148 * 16);
    if (p->f32)
      cp_maskgram_kernel<float><<<blocks, 256, 0, st>>>(p->ch, p->m_local, mask, ldm, (float*)p->mgd, (float*)p->mgo);
    else
      cp_maskgram_kernel<double><<<blocks, 256, 0, st>>>(p->ch, p->m_local, mask, ldm, (double*)p->mgd,
                                                         (double*)p->mgo);
    MLR_LAUNCH_CHECK("cp_maskgram_kernel");
  }
  if (p->m_local > 0) {
    MLR_CUDA(cudaMemsetAsync(p->LH, 0, tb * p->m_local * np, st));
    MLR_CUDA(cudaMemsetAsync(p->SH, 0, tb * p->m_local * np, st));
    MLR_CUDA(cudaMemset2DAsync(S, lds * tb, 0, tb * p->ch.n, p->m_local, st));
  }
  // warm start v = 1/sqrt(n_H) on the real coarse columns (cpcp.py:300)
  std::vector<double> v0(np, 0.0);
  for (int k = 0; k < p->ch.nh; ++k) v0[k] = 1.0 / std::sqrt((double)p->ch.nh);
  MLR_CUDA(cudaMemcpyAsync(p->v, v0.data(), sizeof(double) * np, cudaMemcpyHostToDevice, st));
  MLR_CUDA(cudaStreamSynchronize(st));
  return p->f32 ? cp_row<float, kCpInit>(p, D, ldd, mask, ldm, S, lds, nullptr, 0, st)
                : cp_row<double, kCpInit>(p, D, ldd, mask, ldm, S, lds, nullptr, 0, st);
}

int cpcp_gram(CpcpPlan* p, double* red, double* amax, cudaStream_t st) {
  const int np = p->ch.np;
  const int64_t nn = (int64_t)np * np;
  p->timer.begin(st);
  if (p->m_local > 0) {
    GemmSpec g{};
    g.M = np; g.N = np; g.K = (int)p->m_local;
    g.A = p->GH; g.lda = np; g.a_f32 = p->f32; g.trans_a = true;
    g.B = p->GH; g.ldb = np; g.b_f32 = p->f32; g.trans_b = false;
    g.C = p->gram_part; g.ldc = np; g.c_f32 = false; g.c_slice = nn; g.splits = p->gram_splits; g.alpha = 1.0;
    g.skip = &p->dev->done;
    g.sym = true;  // Gram: upper-triangle tiles, mirrored
    if (!p->fine) {  // full width: the LMO works on g_H directly
      int rc = gemm_f64(g, st);
      if (rc) return rc;
      rc = sum_slices(p->gram_part, nn, nn, p->gram_splits, red, st);
      if (rc) return rc;
    }
  } else {
    MLR_CUDA(cudaMemsetAsync(red, 0, sizeof(double) * nn, st));
  }
  // no rows: zero stats, an empty arg-max record (idx -1) and the budget flag
  cp_part_reduce<<<1, 256, 0, st>>>(p->row_part, p->m_local > 0 ? p->row_blocks : 0, red + nn, amax, p->dev);
  MLR_LAUNCH_CHECK("cp_part_reduce");
  p->timer.end(0, st);
  return kOk;
}

int cpcp_begin(CpcpPlan* p, const double* red, const double* amax_all, cudaStream_t st) {
  (void)amax_all;
  const int64_t nn = (int64_t)p->ch.np * p->ch.np;
  cp_begin_kernel<<<1, 1, 0, st>>>(p->dev, red + nn, p->hist, p->obj);
  MLR_LAUNCH_CHECK("cp_begin_kernel");
  return kOk;
}

int cpcp_lmo(CpcpPlan* p, const double* red, const double* amax_all, double* dots, cudaStream_t st) {
  const int np = p->ch.np;
  int cs = p->cluster;
  const int R = np / cs;
  const bool fit = (size_t)R * np * 8 + (3 * np + 64) * 8 <= 200 * 1024;
  size_t smem = (3 * (size_t)np + 64) * 8 + (fit ? (size_t)R * np * 8 : 0);
  MLR_CUDA(cudaFuncSetAttribute(cp_power_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (cs > 8) MLR_CUDA(cudaFuncSetAttribute(cp_power_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(kPowThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  p->timer.begin(st);
  if (p->fine) {
    cudaLaunchConfig_t fc = {};
    fc.gridDim = dim3(p->fine_ctas);
    fc.blockDim = dim3(kFineThreads);
    fc.stream = st;
    cudaLaunchAttribute fa[1];
    fa[0].id = cudaLaunchAttributeCooperative;
    fa[0].val.cooperative = 1;
    fc.attrs = fa;
    fc.numAttrs = 1;
    if (p->f32)
      MLR_CUDA(cudaLaunchKernelEx(&fc, cp_power_fine_kernel<float>, p->dev, (const float*)p->GH, p->m_local, np,
                                  p->v, p->vin, p->ft, p->fz, p->fv0, p->fzpart, p->fspart));
    else
      MLR_CUDA(cudaLaunchKernelEx(&fc, cp_power_fine_kernel<double>, p->dev, (const double*)p->GH, p->m_local, np,
                                  p->v, p->vin, p->ft, p->fz, p->fv0, p->fzpart, p->fspart));
  } else {
    MLR_CUDA(cudaLaunchKernelEx(&cfg, cp_power_kernel, p->dev, (const double*)red, np, p->v, p->vin, fit ? 1 : 0));
  }
  cp_lmo_scalars<<<1, 1, 0, st>>>(p->dev, amax_all, p->world);
  MLR_LAUNCH_CHECK("cp_lmo_scalars");
  p->timer.end(1, st);
  p->timer.begin(st);
  if (p->m_local > 0 && p->coarse_dots) {
    int blocks = p->row_blocks;
    const void* mgd = p->mask_dev ? p->mgd : nullptr;
    const void* mgo = p->mask_dev ? p->mgo : nullptr;
    const char* v4env = getenv("MLR_DOTS_V4");
    if (p->f32 && mgd && p->ch.np % 4 == 0 && !(v4env && v4env[0] == '0')) {
      auto kern = p->ch.np <= 128 ? cp_dots_coarse_v4<true> : cp_dots_coarse_v4<false>;
      int dev = 0, sms = 0, per = 0;  // one wave: every warp pipelines its rows
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 256, 0);
      blocks = std::max(1, std::min(blocks, sms * std::max(per, 1)));
      kern<<<blocks, 256, 0, st>>>(p->dev, p->ch, p->m_local, p->row0, (const float*)p->LH, (const float*)p->GH,
                                   (const float*)p->SH, (const float*)mgd, (const float*)mgo, p->v, p->vin, p->u,
                                   p->dots_part);
    } else if (p->f32)
      cp_dots_coarse_kernel<float><<<blocks, 256, 0, st>>>(p->dev, p->ch, p->m_local, p->row0, (const float*)p->LH,
                                                           (const float*)p->GH, (const float*)p->SH,
                                                           (const float*)mgd, (const float*)mgo, p->v, p->vin, p->u,
                                                           p->dots_part);
    else
      cp_dots_coarse_kernel<double><<<blocks, 256, 0, st>>>(p->dev, p->ch, p->m_local, p->row0,
                                                            (const double*)p->LH, (const double*)p->GH,
                                                            (const double*)p->SH, (const double*)mgd,
                                                            (const double*)mgo, p->v, p->vin, p->u, p->dots_part);
    MLR_LAUNCH_CHECK("cp_dots_coarse_kernel");
    cp_dots_reduce<<<1, 256, 0, st>>>(p->dots_part, blocks, dots, p->dev);
    MLR_LAUNCH_CHECK("cp_dots_reduce");
  } else if (p->m_local > 0 && (size_t)p->ch.np * 16 + 8 * (size_t)(p->ch.np + 2) * 8 <= 200 * 1024) {
    const int rc = cp_dots_rows(p, st);
    if (rc) return rc;
    cp_dots_reduce<<<1, 256, 0, st>>>(p->dots_part, p->row_blocks, dots, p->dev);
    MLR_LAUNCH_CHECK("cp_dots_reduce");
  } else if (p->m_local > 0) {
    const int blocks = p->row_blocks;
    if (p->f32)
      cp_dots_kernel<float><<<blocks, 256, 0, st>>>(p->dev, p->ch, p->m_local, p->row0, p->mask_dev, p->ldm_dev,
                                                    (const float*)p->LH, (const float*)p->GH, (const float*)p->SH,
                                                    p->v, p->vin, p->u, p->dots_part);
    else
      cp_dots_kernel<double><<<blocks, 256, 0, st>>>(p->dev, p->ch, p->m_local, p->row0, p->mask_dev, p->ldm_dev,
                                                     (const double*)p->LH, (const double*)p->GH,
                                                     (const double*)p->SH, p->v, p->vin, p->u, p->dots_part);
    MLR_LAUNCH_CHECK("cp_dots_kernel");
    cp_dots_reduce<<<1, 256, 0, st>>>(p->dots_part, blocks, dots, p->dev);
    MLR_LAUNCH_CHECK("cp_dots_reduce");
  } else {
    MLR_CUDA(cudaMemsetAsync(dots, 0, 3 * sizeof(double), st));
  }
  p->timer.end(2, st);
  return kOk;
}

int cpcp_update(CpcpPlan* p, const void* D, int64_t ldd, const uint32_t* mask, int64_t ldm, void* S, int64_t lds,
                const double* dots, cudaStream_t st) {
  p->timer.begin(st);
  cp_qp_kernel<<<1, 1, 0, st>>>(p->dev, dots);
  MLR_LAUNCH_CHECK("cp_qp_kernel");
  p->timer.end(3, st);
  p->timer.begin(st);
  int rc = p->f32 ? cp_row<float, kCpUpdate>(p, D, ldd, mask, ldm, S, lds, nullptr, 0, st)
                  : cp_row<double, kCpUpdate>(p, D, ldd, mask, ldm, S, lds, nullptr, 0, st);
  p->timer.end(5, st);
  return rc;
}

int cpcp_finalize(CpcpPlan* p, const double* red, cudaStream_t st) {
  const int64_t nn = (int64_t)p->ch.np * p->ch.np;
  p->timer.begin(st);
  cp_finalize_kernel<<<1, 1, 0, st>>>(p->dev, red + nn, p->hist, p->obj);
  MLR_LAUNCH_CHECK("cp_finalize_kernel");
  p->timer.end(6, st);
  return kOk;
}

int cpcp_outputs(CpcpPlan* p, void* L, int64_t ldl, cudaStream_t st) {
  return p->f32 ? cp_row<float, kCpOutput>(p, nullptr, 0, nullptr, 0, nullptr, 0, L, ldl, st)
                : cp_row<double, kCpOutput>(p, nullptr, 0, nullptr, 0, nullptr, 0, L, ldl, st);
}

}  // namespace mlr
