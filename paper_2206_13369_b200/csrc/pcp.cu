// ML-PCP (multilevel inexact ALM, reference pcp.py:213-309) on the device.
//
// Fine planes are row-major m_local x n (T = float or double).  Coarse
// matrices A (= W R) and Z (= A W~) are m_local x np (np = n_H rounded up to
// 64, zero padded).  The fused row kernel does, for one fine row at a time:
//     L   = Z_i R^T                     (prolongation stencil, pcp.py:266)
//     S   = shrink(D - L + Y/mu, lam/mu) (pcp.py:272-275)
//     res = D - L - S; Y' = Y + mu res   (pcp.py:277-281) + reductions
//     A'  = (D - S + Y'/(rho mu)) R      (next iteration's restriction,
//                                        pcp.py:252-255) via a gather stencil
// so each iteration reads D and Y once and writes Y once (plus m x n_H for
// Z and A').  S is never stored: it is recomputed at exit from the previous
// Y (double-buffered by the host).
#include <cooperative_groups.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "pcp.h"
#include "rows.h"

namespace cg = cooperative_groups;

namespace mlr {

__device__ __forceinline__ double global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return (double)t;
}

// ------------------------------------------------------------ input stats
template <typename T>
__global__ void input_stats_kernel(const T* __restrict__ D, int64_t ldd, int64_t m, int n,
                                   double* __restrict__ part) {
  // ||D||_F^2, max|D| and the count of non-finite entries (as_matrix's
  // finiteness check, linalg.py:55-56)
  __shared__ double scratch[2 * 32];
  double s = 0.0, mx = 0.0, bad = 0.0;
  for (int64_t i = blockIdx.x; i < m; i += gridDim.x) {
    const T* row = D + i * ldd;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      double v = (double)row[j];
      if (!isfinite(v)) {
        bad += 1.0;
        continue;
      }
      s = fma(v, v, s);
      mx = fmax(mx, fabs(v));
    }
  }
  mx = warp_max(mx);
  __shared__ double smx[32];
  if ((threadIdx.x & 31) == 0) smx[threadIdx.x >> 5] = mx;
  double v[2] = {s, bad};
  block_sum<2>(v, scratch);
  if (threadIdx.x == 0) {
    double m2 = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m2 = fmax(m2, smx[w]);
    part[3 * blockIdx.x] = v[0];
    part[3 * blockIdx.x + 1] = m2;
    part[3 * blockIdx.x + 2] = v[1];
  }
}

__global__ void __launch_bounds__(256) input_stats_finish(const double* __restrict__ part, int nparts,
                                                          double* __restrict__ out) {
  __shared__ double scratch[2 * 32];
  __shared__ double smx[32];
  double v[2] = {0.0, 0.0}, mx = 0.0;
  for (int b = threadIdx.x; b < nparts; b += blockDim.x) {
    v[0] += part[3 * b];
    mx = fmax(mx, part[3 * b + 1]);
    v[1] += part[3 * b + 2];
  }
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) smx[threadIdx.x >> 5] = mx;
  block_sum<2>(v, scratch);
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) smx[0] = fmax(smx[0], smx[w]);
    out[0] = v[0];
    out[1] = smx[0];
    out[2] = v[1];
  }
}

// ------------------------------------------------------------ Lanczos on D^T D
// sigma_1(D) (pcp.py:100 and :114 call np.linalg.norm(d, 2), a full SVD;
// Lanczos with full reorthogonalisation reaches ~1e-15 relative).
__global__ void lz_init_kernel(LanczosDev* lz, double* Q, int n, int kmax) {
  const double v = 1.0 / sqrt((double)n);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) Q[j] = v;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    lz->k = 0;
    lz->done = 0;
    lz->kmax = kmax;
    lz->theta = 0.0;
    lz->theta_prev = 0.0;
    lz->stable = 0;
    lz->sigma1 = 0.0;
  }
}

// t = D q (warp per row; 16-byte loads of D, FP64 q from L2, FP64 sums).
template <typename T>
__global__ void __launch_bounds__(256) lz_dv_kernel(const LanczosDev* __restrict__ lz, const T* __restrict__ D,
                                                    int64_t ldd, int64_t m, int n, const double* __restrict__ Q,
                                                    double* __restrict__ t) {
  if (lz->done) return;
  const double* __restrict__ q = Q + (int64_t)lz->k * n;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int NV = 16 / sizeof(T);
  const bool vec = (n % NV == 0) && (ldd % NV == 0);
  // FP32, aligned: two rows per warp share every q load (q is re-read from
  // L1/L2 for each row; halving those reads lifts the pass toward HBM speed)
  if (sizeof(T) == 4 && vec) {
    for (int64_t i = w0; i < m; i += 2 * nw) {
      const bool two = i + nw < m;
      const T* ra = D + i * ldd;
      const T* rb = D + (two ? i + nw : i) * ldd;
      double sa0 = 0.0, sa1 = 0.0, sb0 = 0.0, sb1 = 0.0;
      for (int j = lane * 4; j < n; j += 128) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(ra + j));
        const float4 b = __ldg(reinterpret_cast<const float4*>(rb + j));
        const double2 q01 = __ldg(reinterpret_cast<const double2*>(q + j));
        const double2 q23 = __ldg(reinterpret_cast<const double2*>(q + j + 2));
        sa0 = fma((double)a.x, q01.x, sa0);
        sa1 = fma((double)a.y, q01.y, sa1);
        sa0 = fma((double)a.z, q23.x, sa0);
        sa1 = fma((double)a.w, q23.y, sa1);
        sb0 = fma((double)b.x, q01.x, sb0);
        sb1 = fma((double)b.y, q01.y, sb1);
        sb0 = fma((double)b.z, q23.x, sb0);
        sb1 = fma((double)b.w, q23.y, sb1);
      }
      const double sa = warp_sum(sa0 + sa1), sb = warp_sum(sb0 + sb1);
      if (lane == 0) {
        t[i] = sa;
        if (two) t[i + nw] = sb;
      }
    }
    return;
  }
  for (int64_t i = w0; i < m; i += nw) {
    const T* row = D + i * ldd;
    double s0 = 0.0, s1 = 0.0;
    if (vec) {
      int j = lane * NV;
      for (; j + 32 * NV < n; j += 64 * NV) {  // two vectors in flight
        T a[NV], b[NV];
        *reinterpret_cast<float4*>(a) = __ldg(reinterpret_cast<const float4*>(row + j));
        *reinterpret_cast<float4*>(b) = __ldg(reinterpret_cast<const float4*>(row + j + 32 * NV));
#pragma unroll
        for (int e = 0; e < NV; ++e) {
          s0 = fma((double)a[e], __ldg(q + j + e), s0);
          s1 = fma((double)b[e], __ldg(q + j + 32 * NV + e), s1);
        }
      }
      if (j < n) {
        T a[NV];
        *reinterpret_cast<float4*>(a) = __ldg(reinterpret_cast<const float4*>(row + j));
#pragma unroll
        for (int e = 0; e < NV; ++e) s0 = fma((double)a[e], __ldg(q + j + e), s0);
      }
    } else {
      for (int j = lane; j < n; j += 32) s0 = fma((double)row[j], q[j], s0);
    }
    const double s = warp_sum(s0 + s1);
    if (lane == 0) t[i] = s;
  }
}

// Partial w = D^T t over a tile of rows x 2048 columns: thread owns 8
// consecutive columns (16-byte loads), 2 rows in flight; FP64 partials
// wpart[row block][j], summed by sum_slices (deterministic).
constexpr int LZ_COLS = 2048;
template <typename T>
__global__ void __launch_bounds__(256) lz_dtv_kernel(const LanczosDev* __restrict__ lz, const T* __restrict__ D,
                                                     int64_t ldd, int64_t m, int n, const double* __restrict__ t,
                                                     double* __restrict__ wpart, int64_t rows_per_split) {
  if (lz->done) return;
  const int j0 = blockIdx.x * LZ_COLS + threadIdx.x * 8;
  const int64_t r0 = blockIdx.y * rows_per_split;
  const int64_t r1 = min(m, r0 + rows_per_split);
  if (j0 >= n) return;
  double acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.0;
  constexpr int NV = 16 / sizeof(T);
  const bool vec = (j0 + 8 <= n) && (n % NV == 0) && (ldd % NV == 0);
  if (vec) {
    int64_t i = r0;
    for (; i + 3 < r1; i += 4) {  // four rows in flight
      T a[4][8];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int v = 0; v < 8 / NV; ++v)
          *reinterpret_cast<float4*>(a[r] + v * NV) =
              __ldg(reinterpret_cast<const float4*>(D + (i + r) * ldd + j0 + v * NV));
      double tr[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) tr[r] = __ldg(t + i + r);
#pragma unroll
      for (int e = 0; e < 8; ++e)
        acc[e] = fma((double)a[3][e], tr[3], fma((double)a[2][e], tr[2], fma((double)a[1][e], tr[1], fma((double)a[0][e], tr[0], acc[e]))));
    }
    for (; i + 1 < r1; i += 2) {
      T a[8], b[8];
      const T* ra = D + i * ldd + j0;
      const T* rb = ra + ldd;
#pragma unroll
      for (int v = 0; v < 8 / NV; ++v) {
        *reinterpret_cast<float4*>(a + v * NV) = __ldg(reinterpret_cast<const float4*>(ra + v * NV));
        *reinterpret_cast<float4*>(b + v * NV) = __ldg(reinterpret_cast<const float4*>(rb + v * NV));
      }
      const double ta = __ldg(t + i), tb = __ldg(t + i + 1);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = fma((double)b[e], tb, fma((double)a[e], ta, acc[e]));
    }
    if (i < r1) {
      T a[8];
      const T* ra = D + i * ldd + j0;
#pragma unroll
      for (int v = 0; v < 8 / NV; ++v)
        *reinterpret_cast<float4*>(a + v * NV) = __ldg(reinterpret_cast<const float4*>(ra + v * NV));
      const double ta = __ldg(t + i);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = fma((double)a[e], ta, acc[e]);
    }
  } else {
    for (int64_t i = r0; i < r1; ++i) {
      const double ti = t[i];
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (j0 + e < n) acc[e] = fma((double)D[i * ldd + j0 + e], ti, acc[e]);
    }
  }
  double* o = wpart + (int64_t)blockIdx.y * n + j0;
#pragma unroll
  for (int e = 0; e < 8; ++e)
    if (j0 + e < n) o[e] = acc[e];
}

// w = D^T (D q) in one pass over D for short rows (n <= LZ_FUSED_N): a warp
// keeps its row in registers, reduces t_i = d_i . q, then adds t_i d_i to
// its private FP64 accumulator in shared memory; the CTA sums its warps'
// accumulators in a fixed order into wpart[blockIdx.x] (sum_slices then
// sums the CTAs, also in a fixed order: deterministic).  Half the HBM
// traffic of the two-kernel path and no t round trip.
constexpr int LZ_FUSED_N = 2048, LZ_FW = 8;
template <typename T>
__global__ void __launch_bounds__(LZ_FW * 32, 1) lz_dtdv_kernel(const LanczosDev* __restrict__ lz,
                                                                const T* __restrict__ D, int64_t ldd, int64_t m,
                                                                int n, const double* __restrict__ Q,
                                                                double* __restrict__ wpart) {
  if (lz->done) return;
  constexpr int NV = 16 / sizeof(T);
  constexpr int MAXC = LZ_FUSED_N / (32 * NV);
  extern __shared__ __align__(16) double lzacc[];  // LZ_FW x n
  const double* __restrict__ q = Q + (int64_t)lz->k * n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* acc = lzacc + (int64_t)warp * n;
  for (int j = lane; j < n; j += 32) acc[j] = 0.0;
  const bool vec = (n % NV == 0) && (ldd % NV == 0);
  for (int64_t i = (int64_t)blockIdx.x * LZ_FW + warp; i < m; i += (int64_t)gridDim.x * LZ_FW) {
    const T* row = D + i * ldd;
    T r[MAXC][NV];
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int j = (c * 32 + lane) * NV;
      if (vec) {
        if (j < n) *reinterpret_cast<float4*>(r[c]) = __ldg(reinterpret_cast<const float4*>(row + j));
      } else {
#pragma unroll
        for (int e = 0; e < NV; ++e) r[c][e] = j + e < n ? row[j + e] : T(0);
      }
    }
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int j = (c * 32 + lane) * NV;
      if (j < n)
#pragma unroll
        for (int e = 0; e < NV; ++e)
          if (vec || j + e < n) s = fma((double)r[c][e], __ldg(q + j + e), s);
    }
    const double t = warp_sum(s);
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      const int j = (c * 32 + lane) * NV;
      if (j < n)
#pragma unroll
        for (int e = 0; e < NV; ++e)
          if (vec || j + e < n) acc[j + e] = fma((double)r[c][e], t, acc[j + e]);
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < LZ_FW; ++w) v += lzacc[(int64_t)w * n + j];
    wpart[(int64_t)blockIdx.x * n + j] = v;
  }
}

// w = D^T (D q) in ONE pass over D for long FP32 rows (n > LZ_FUSED_N, C5:
// 20000 columns).  A 2-CTA cluster owns whole rows; CTA c of the pair owns
// the column segment [c seg, (c+1) seg).  Row segments stream HBM -> shared
// memory by TMA bulk copies (cp.async.bulk, one mbarrier per stage, one
// elected producer thread, LZL_STAGES segments in flight); each thread keeps
// its columns' q and FP64 accumulator in registers.  Per batch of LZL_R rows:
// partial dots d_i.q over the segment (FP64) -> block sum -> the two CTAs
// swap partials through DSMEM and one cluster barrier -> t_i summed in a
// fixed order (identical in both CTAs) -> acc += t_i d_i.  The cluster's
// FP64 partial of w goes to wpart[cluster]; sum_slices adds the clusters in
// a fixed order (deterministic).  D is read once per Lanczos step instead of
// twice (lz_dv_kernel + lz_dtv_kernel).
constexpr int LZL_T = 512, LZL_CL = 2, LZL_R = 2, LZL_NG = 5;  // NG float4 groups per thread: seg <= 10240

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void dsmem_st_f64(const double* local, uint32_t cta, double v) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local)), "r"(cta));
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(remote), "d"(v) : "memory");
}
// st.async of one double into a peer CTA's shared memory; the bytes complete
// a transaction on the peer's mbarrier (same offset in the peer's smem).
__device__ __forceinline__ void dsmem_st_async_f64(const double* local_slot, const uint64_t* local_bar,
                                                   uint32_t cta, double v) {
  uint32_t rslot, rbar;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rslot) : "r"(smem_u32(local_slot)), "r"(cta));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_u32(local_bar)), "r"(cta));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(rslot), "d"(v),
               "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// FP32 -> FP64 on the integer pipe: sign | (e8 + 896) << 20 | m23 >> 3 in the
// high word, m23 << 29 in the low word (exact for every normal float).  The
// F2F.F64.F32 conversion runs on the XU pipe at 16 lanes/clk/SM and is the
// busiest pipe of this kernel (ncu: XU 44% of peak, the top pipe, with the
// warps stalled on its results); 4 integer operations convert at the same
// rate on the ALU pipe, so alternating the two doubles the conversion rate.
// Zeros and denormals map to +-2^-127 (1 + m / 2^23) (absolute error below
// 1.2e-38: no effect on an FP64 sum of |x q| terms); the input was checked
// to be finite (input_stats_kernel) before the Lanczos runs.
__device__ __forceinline__ double lz_f2d_int(float x) {
  const uint32_t f = __float_as_uint(x);
  const uint32_t hi = (((uint32_t)((int32_t)f >> 3)) & 0x8FFFFFFFu) + 0x38000000u;
  return __hiloint2double((int)hi, (int)(f << 29));
}
template <int CV>
__device__ __forceinline__ void lz_cvt4(const float4 x, double (&d)[4]) {
  d[0] = CV == 2 ? lz_f2d_int(x.x) : (double)x.x;
  d[1] = CV >= 1 ? lz_f2d_int(x.y) : (double)x.y;
  d[2] = CV == 2 ? lz_f2d_int(x.z) : (double)x.z;
  d[3] = CV >= 1 ? lz_f2d_int(x.w) : (double)x.w;
}

template <int CV>
__global__ void __launch_bounds__(LZL_T, 1) lz_dtdq_long_kernel(const LanczosDev* __restrict__ lz,
                                                                const float* __restrict__ D, int64_t ldd,
                                                                int64_t m, int n, int seg, int stages,
                                                                const double* __restrict__ Q,
                                                                double* __restrict__ wpart) {
  extern __shared__ __align__(128) unsigned char lzl_smem[];
  __shared__ __align__(8) uint64_t full[16];
  __shared__ __align__(8) uint64_t xbar[2];  // batch parity: the peer's partials have landed
  __shared__ double xch[2][LZL_R][LZL_CL];
  __shared__ double red[2][LZL_T / 32][LZL_R];
  uint32_t cr, cid, ncl;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(cr));
  asm("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
  asm("mov.u32 %0, %%nclusterid.x;" : "=r"(ncl));
  const bool skip = lz->done != 0;  // uniform over the grid
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int col0 = (int)cr * seg;
  const int len = max(0, min(seg, n - col0));     // multiple of 4 (n % 4 == 0)
  const int ng4 = len >> 2;
  const int64_t nrows = (int64_t)cid < m ? (m - 1 - cid) / ncl + 1 : 0;
  float* stage = reinterpret_cast<float*>(lzl_smem);
  const uint32_t bytes = (uint32_t)len * 4u;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (!skip && tid == 0 && bytes > 0)
    for (int s = 0; s < stages && s < nrows; ++s) {
      mbar_expect_tx(&full[s], bytes);
      bulk_g2s(stage + (size_t)s * seg, D + ((int64_t)cid + (int64_t)s * ncl) * ldd + col0, bytes, &full[s]);
    }
  double qv[LZL_NG][4], acc[LZL_NG][4];
  const double* __restrict__ q = Q + (int64_t)(skip ? 0 : lz->k) * n + col0;
#pragma unroll
  for (int g = 0; g < LZL_NG; ++g) {
    const int k = tid + g * LZL_T;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      qv[g][e] = (!skip && k < ng4) ? q[4 * k + e] : 0.0;
      acc[g][e] = 0.0;
    }
  }
  cluster_sync_all();  // both CTAs started: exchange slots may be written
  if (!skip) {
    const int64_t nb = (nrows + LZL_R - 1) / LZL_R;
    // partial dots of batch b over this CTA's segment -> red[b & 1]
    auto dots = [&](int64_t b) {
      const int64_t j0 = b * LZL_R;
      const int rr = (int)(nrows - j0 < LZL_R ? nrows - j0 : LZL_R);
#pragma unroll
      for (int r = 0; r < LZL_R; ++r) {
        double pr = 0.0;
        if (r < rr) {
          const int64_t j = j0 + r;
          const int s = (int)(j % stages);
          mbar_wait(&full[s], (uint32_t)((j / stages) & 1));
          const float4* row = reinterpret_cast<const float4*>(stage + (size_t)s * seg);
          double a0 = 0.0, a1 = 0.0;
#pragma unroll
          for (int g = 0; g < LZL_NG; ++g) {
            const int k = tid + g * LZL_T;
            if (k < ng4) {
              double xd[4];
              lz_cvt4<CV>(row[k], xd);
              a0 = fma(xd[0], qv[g][0], a0);
              a1 = fma(xd[1], qv[g][1], a1);
              a0 = fma(xd[2], qv[g][2], a0);
              a1 = fma(xd[3], qv[g][3], a1);
            }
          }
          pr = warp_sum(a0 + a1);
        }
        if (lane == 0) red[b & 1][warp][r] = pr;
      }
    };
    // warp 0: the CTA's partial of each row of batch b (fixed order) into
    // its own slot and, by st.async, the peer's slot, completing 8 bytes of a
    // transaction on the peer's xbar[b & 1]; thread 0 arms its own xbar for
    // the peer's partials.  No cluster barrier: each CTA waits only for the
    // bytes it needs (the peer cannot run two batches ahead, since it waits
    // for this CTA's partials of the batch in between).
    auto post = [&](int64_t b) {
      if (warp == 0 && lane < LZL_R) {
        double v = 0.0;
        for (int w = 0; w < LZL_T / 32; ++w) v += red[b & 1][w][lane];
        xch[b & 1][lane][cr] = v;
        for (uint32_t c = 0; c < LZL_CL; ++c)
          if (c != cr) dsmem_st_async_f64(&xch[b & 1][lane][cr], &xbar[b & 1], c, v);
      }
      if (tid == 0) mbar_expect_tx(&xbar[b & 1], (uint32_t)(LZL_R * (LZL_CL - 1) * sizeof(double)));
    };
    if (nb > 0) {
      dots(0);
      __syncthreads();
      post(0);
    }
    // Software pipeline: the dots of batch b + 1 run while the peer's
    // partials of batch b arrive; then t(b) and the accumulation of batch b.
    for (int64_t b = 0; b < nb; ++b) {
      const int64_t j0 = b * LZL_R;
      const int rr = (int)(nrows - j0 < LZL_R ? nrows - j0 : LZL_R);
      if (b + 1 < nb) dots(b + 1);
      mbar_wait(&xbar[b & 1], (uint32_t)((b >> 1) & 1));
      __syncthreads();  // the own-slot writes of warp 0 are visible too
      double t[LZL_R];
#pragma unroll
      for (int r = 0; r < LZL_R; ++r) {
        double v = 0.0;
#pragma unroll
        for (int c = 0; c < LZL_CL; ++c) v += xch[b & 1][r][c];
        t[r] = r < rr ? v : 0.0;
      }
#pragma unroll
      for (int r = 0; r < LZL_R; ++r) {
        if (r < rr) {
          const int s = (int)((j0 + r) % stages);
          const float4* row = reinterpret_cast<const float4*>(stage + (size_t)s * seg);
#pragma unroll
          for (int g = 0; g < LZL_NG; ++g) {
            const int k = tid + g * LZL_T;
            if (k < ng4) {
              double xd[4];
              lz_cvt4<CV>(row[k], xd);
#pragma unroll
              for (int e = 0; e < 4; ++e) acc[g][e] = fma(xd[e], t[r], acc[g][e]);
            }
          }
        }
      }
      __syncthreads();  // batch b's stages are consumed; red[(b + 1) & 1] is complete
      if (tid == 0 && bytes > 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int r = 0; r < rr; ++r) {
          const int64_t jn = j0 + r + stages;
          if (jn < nrows) {
            const int s = (int)(jn % stages);
            mbar_expect_tx(&full[s], bytes);
            bulk_g2s(stage + (size_t)s * seg, D + ((int64_t)cid + jn * ncl) * ldd + col0, bytes, &full[s]);
          }
        }
      }
      if (b + 1 < nb) post(b + 1);
    }
  }
  double* o = wpart + (int64_t)cid * n + col0;
#pragma unroll
  for (int g = 0; g < LZL_NG; ++g) {
    const int k = tid + g * LZL_T;
    if (k < ng4)
#pragma unroll
      for (int e = 0; e < 4; ++e) o[4 * k + e] = acc[g][e];
  }
  cluster_sync_all();  // no CTA leaves while its peer's last st.async may be in flight
}

int lz_long_stages(int seg) {
  const int64_t avail = 200 * 1024;
  return (int)std::min<int64_t>(16, avail / ((int64_t)seg * 4));
}

// True if the symmetric tridiagonal (a[0..k1), b[0..k1-1)) has an eigenvalue
// above x: T - x I has a positive LDL^T pivot d_i = p_i / p_(i-1), with the
// leading principal minors p_i = (a_i - x) p_(i-1) - b_(i-1)^2 p_(i-2)
// (division-free; rescaled when large, the ratio is scale-free).
__device__ __forceinline__ bool tridiag_has_above(const double* a, const double* b, int k1, double x) {
  double pm = 1.0, p = a[0] - x;
  if (p > 0.0) return true;
  if (p == 0.0) p = -1e-300;
  for (int i = 1; i < k1; ++i) {
    const double bb = b[i - 1] * b[i - 1];
    double pn = fma(a[i] - x, p, -bb * pm);
    if (pn == 0.0) pn = -1e-300 * copysign(1.0, p);
    if ((pn > 0.0) == (p > 0.0)) return true;  // d_i = pn / p > 0
    pm = p;
    p = pn;
    if (fabs(p) > 1e150) {
      p *= 1e-150;
      pm *= 1e-150;
    }
  }
  return false;
}

// Largest eigenvalue by block-parallel multisection (all threads of the CTA
// take part; each round shrinks the bracket ~blockDim-fold).
__device__ double tridiag_max_eig_block(const double* a, const double* b, int k1) {
  __shared__ double br[2];
  __shared__ int best;
  if (threadIdx.x == 0) {
    double lo = 1e300, hi = -1e300;
    for (int i = 0; i < k1; ++i) {
      double r = (i > 0 ? fabs(b[i - 1]) : 0.0) + (i + 1 < k1 ? fabs(b[i]) : 0.0);
      lo = fmin(lo, a[i] - r);
      hi = fmax(hi, a[i] + r);
    }
    br[0] = lo;
    br[1] = hi;
  }
  __syncthreads();
  const int nt = blockDim.x;
  for (int round = 0; round < 12; ++round) {
    const double lo = br[0], hi = br[1];
    if (threadIdx.x == 0) best = -1;
    __syncthreads();
    const double x = lo + (hi - lo) * (double)(threadIdx.x + 1) / (double)(nt + 1);
    if (x > lo && x < hi && tridiag_has_above(a, b, k1, x)) atomicMax(&best, (int)threadIdx.x);
    __syncthreads();
    if (threadIdx.x == 0) {
      const int t = best;
      const double nlo = t < 0 ? lo : lo + (hi - lo) * (double)(t + 1) / (double)(nt + 1);
      const double nhi = t + 1 >= nt ? hi : lo + (hi - lo) * (double)(t + 2) / (double)(nt + 1);
      br[0] = nlo;
      br[1] = nhi;
    }
    __syncthreads();
    if (!(br[1] - br[0] > 1e-17 * fabs(br[1]))) break;
  }
  return 0.5 * (br[0] + br[1]);
}

__global__ void __launch_bounds__(1024) lz_update_kernel(LanczosDev* lz, double* __restrict__ Q,
                                                          const double* __restrict__ w_in,
                                                          double* __restrict__ w, int n, double tol) {
  if (lz->done) return;
  __shared__ double scratch[4 * 32];
  __shared__ double h[512];
  const int k = lz->k;
  double* qk = Q + (int64_t)k * n;
  // alpha = q_k . w
  double s = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double v = w_in[j];
    w[j] = v;
    s = fma(v, qk[j], s);
  }
  double v1[1] = {s};
  block_sum<1>(v1, scratch);
  __shared__ double alpha_s;
  if (threadIdx.x == 0) alpha_s = v1[0];
  __syncthreads();
  const double alpha = alpha_s;
  const double bprev = k > 0 ? lz->beta[k - 1] : 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double v = w[j] - alpha * qk[j];
    if (k > 0) v -= bprev * Q[(int64_t)(k - 1) * n + j];
    w[j] = v;
  }
  __syncthreads();
  // full reorthogonalisation, twice (classical Gram-Schmidt)
  for (int pass = 0; pass < 2; ++pass) {
    // h = Q^T w: one warp per basis vector (all dots in flight at once)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int c = wid; c <= k; c += nwarps) {
      const double* qc = Q + (int64_t)c * n;
      double d = 0.0;
      for (int j = lane; j < n; j += 32) d = fma(qc[j], w[j], d);
      d = warp_sum(d);
      if (lane == 0) h[c] = d;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      double v = w[j];
      for (int c = 0; c <= k; ++c) v -= h[c] * Q[(int64_t)c * n + j];
      w[j] = v;
    }
    __syncthreads();
  }
  double nn = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) nn = fma(w[j], w[j], nn);
  double v2[1] = {nn};
  block_sum<1>(v2, scratch);
  __shared__ double beta_s;
  __shared__ int stop_s;
  if (threadIdx.x == 0) {
    lz->alpha[k] = alpha;
    lz->beta[k] = sqrt(v2[0]);
  }
  __syncthreads();
  const double th_all = tridiag_max_eig_block(lz->alpha, lz->beta, k + 1);
  if (threadIdx.x == 0) {
    const double beta = lz->beta[k];
    const double th = th_all;
    const double rel = lz->theta > 0.0 ? fabs(th - lz->theta) / th : 1.0;
    lz->theta_prev = lz->theta;
    lz->theta = th;
    lz->stable = (rel <= tol) ? lz->stable + 1 : 0;
    int stop = (lz->stable >= 2 && k >= 3) || beta <= 1e-300 * fmax(th, 1e-300) || k + 1 >= lz->kmax;
    if (stop) {
      lz->done = 1;
      lz->sigma1 = sqrt(fmax(th, 0.0));
    }
    beta_s = beta;
    stop_s = stop;
    lz->k = stop ? k : k + 1;
  }
  __syncthreads();
  if (!stop_s) {
    double* qn = Q + (int64_t)(k + 1) * n;
    const double inv = 1.0 / beta_s;
    for (int j = threadIdx.x; j < n; j += blockDim.x) qn[j] = w[j] * inv;
  }
}

// One Lanczos step on a 16-CTA cluster: CTA r owns columns [r S, (r+1) S) of
// every basis vector (S = ceil(n / 16)), so the two reorthogonalisation
// passes stream the basis through 16 SMs.  Dot products are combined by
// reading the 16 partials over DSMEM in a fixed order (identical in every
// CTA); every CTA then evaluates the Ritz value redundantly.
constexpr int LZ_CL = 16, LZ_T = 256;

__device__ __forceinline__ double lz_cluster_sum(cg::cluster_group& cl, double* part_local, int idx) {
  // partials are published by the caller (cl.sync() in between); lanes 0..15 of warp 0 gather
  double v = 0.0;
  const int lane = threadIdx.x & 31;
  if (lane < LZ_CL) v = cl.map_shared_rank(part_local, lane)[idx];
  return warp_sum(v);
}

__global__ void __launch_bounds__(LZ_T) lz_update_cluster(LanczosDev* lz, double* __restrict__ Q,
                                                           const double* __restrict__ w_in, int n, double tol,
                                                           int passes) {
  if (lz->done) return;
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  const int S = (n + LZ_CL - 1) / LZ_CL;
  const int j0 = r * S, len = max(0, min(n, j0 + S) - j0);
  const int k = lz->k;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  extern __shared__ __align__(16) double lzs[];
  double* w = lzs;                  // S
  double* part = w + S;             // partials: [0] alpha, [1] beta, [2..2+K) h pass 0, [2+K..2+2K) h pass 1
  const int K = k + 1;
  double* hfull = part + 2 + 2 * K;  // K
  double* ta = hfull + K;            // tridiagonal alpha[0..K)
  double* tb = ta + K;               // beta[0..K)
  double* acc0 = tb + K;             // S: reorthogonalisation halves
  double* acc1 = acc0 + S;           // S
  __shared__ double scratch[32];
  __shared__ double bcast;
  const double* qk = Q + (int64_t)k * n + j0;
  // alpha = q_k . w
  double s = 0.0;
  for (int j = tid; j < len; j += LZ_T) {
    const double v = w_in[j0 + j];
    w[j] = v;
    s = fma(v, qk[j], s);
  }
  double v1[1] = {s};
  block_sum<1>(v1, scratch);
  if (tid == 0) part[0] = v1[0];
  cl.sync();
  if (wid == 0) {
    const double a = lz_cluster_sum(cl, part, 0);
    if (lane == 0) bcast = a;
  }
  __syncthreads();
  const double alpha = bcast;
  const double bprev = k > 0 ? lz->beta[k - 1] : 0.0;
  for (int j = tid; j < len; j += LZ_T) {
    double v = w[j] - alpha * qk[j];
    if (k > 0) v -= bprev * Q[(int64_t)(k - 1) * n + j0 + j];
    w[j] = v;
  }
  __syncthreads();
  // full reorthogonalisation, `passes` times (classical Gram-Schmidt; none by
  // default, see pcp_lanczos_update): only the top Ritz value is used
  for (int pass = 0; pass < passes; ++pass) {
    double* ph = part + 2 + pass * K;
    for (int c = wid; c < K; c += LZ_T / 32) {
      const double* qc = Q + (int64_t)c * n + j0;
      double d = 0.0;
      for (int j = lane; j < len; j += 32) d = fma(qc[j], w[j], d);
      d = warp_sum(d);
      if (lane == 0) ph[c] = d;
    }
    cl.sync();
    for (int c = wid; c < K; c += LZ_T / 32) {
      const double h = lz_cluster_sum(cl, ph, c);
      if (lane == 0) hfull[c] = h;
    }
    __syncthreads();
    // w -= Q^T h: threads (half, j) split the basis vectors in two halves,
    // 8 loads in flight per thread, halves combined through shared memory
    {
      const int half = tid / (LZ_T / 2), jt = tid % (LZ_T / 2);
      const int c0 = half ? K / 2 : 0, c1 = half ? K : K / 2;
      for (int j = jt; j < len; j += LZ_T / 2) {
        double acc = 0.0;
#pragma unroll 8
        for (int c = c0; c < c1; ++c) acc = fma(hfull[c], Q[(int64_t)c * n + j0 + j], acc);
        (half ? acc1 : acc0)[j] = acc;
      }
    }
    __syncthreads();
    for (int j = tid; j < len; j += LZ_T) w[j] -= acc0[j] + acc1[j];
    __syncthreads();
  }
  double nn = 0.0;
  for (int j = tid; j < len; j += LZ_T) nn = fma(w[j], w[j], nn);
  double v2[1] = {nn};
  block_sum<1>(v2, scratch);
  if (tid == 0) part[1] = v2[0];
  cl.sync();
  if (wid == 0) {
    const double b2 = lz_cluster_sum(cl, part, 1);
    if (lane == 0) bcast = sqrt(b2);
  }
  for (int c = tid; c < k; c += LZ_T) {
    ta[c] = lz->alpha[c];
    tb[c] = lz->beta[c];
  }
  __syncthreads();
  const double beta = bcast;
  if (tid == 0) {
    ta[k] = alpha;
    tb[k] = beta;
  }
  __syncthreads();
  // the largest Ritz value (multisection) only every 4th step: it only
  // feeds the stopping test, and the Sturm counts dominate this kernel
  const bool close = lz->theta > 0.0 && fabs(lz->theta - lz->theta_prev) <= 1e-6 * lz->theta;
  const bool eval = close || (k % 4 == 3) || k + 1 >= lz->kmax || beta <= 1e-300;
  const double th = eval ? tridiag_max_eig_block(ta, tb, K) : lz->theta;
  const double rel = lz->theta > 0.0 ? fabs(th - lz->theta) / th : 1.0;
  const int stable = !eval ? lz->stable : ((rel <= tol) ? lz->stable + 1 : 0);
  const bool stop = (eval && stable >= 2 && k >= 3) || beta <= 1e-300 * fmax(th, 1e-300) || k + 1 >= lz->kmax;
  if (!stop) {
    double* qn = Q + (int64_t)(k + 1) * n + j0;
    const double inv = 1.0 / beta;
    for (int j = tid; j < len; j += LZ_T) qn[j] = w[j] * inv;
  }
  cl.sync();  // every CTA has read lz and the remote partials
  if (r == 0 && tid == 0) {
    lz->alpha[k] = alpha;
    lz->beta[k] = beta;
    if (eval) {
      lz->theta_prev = lz->theta;
      lz->theta = th;
    }
    lz->stable = stable;
    if (stop) {
      lz->done = 1;
      lz->sigma1 = sqrt(fmax(th, 0.0));
    }
    lz->k = stop ? k : k + 1;
  }
}

// The whole Lanczos run in one cooperative kernel (one CTA per SM, one rank,
// n <= LZ_RUN_MAXN): per step
//   t = D q_k (CTA b owns a contiguous row block; warp per row)      | sync
//   CTA partial of D^T t (thread-owned columns, rows re-read from L2)  | sync
//   w = sum of the partials over CTA b's column slice; alpha partials | sync
//   w -= alpha q_k + beta q_{k-1}; reorthogonalisation (twice) with
//   dot partials per slice, every CTA summing them in the same order   | 2 syncs
//   beta; q_{k+1}; the Ritz value (multisection, every CTA alike)      | sync
// so the host launches once instead of ~3 kernels per step plus polls.
// Every reduction has a fixed order: bit-identical to rerunning it.
constexpr int LZ_RUN_MAXN = 4096, LZ_RUN_T = 256;

// Sum of G per-CTA partials base[g * stride] by one warp: lane l takes
// g = l, l + 32, ... (loads in flight together), then a fixed shuffle tree.
__device__ __forceinline__ double warp_gsum(const double* base, int64_t stride, int G, int lane) {
  double v = 0.0;
  for (int g = lane; g < G; g += 32) v += base[(int64_t)g * stride];
  return warp_sum(v);
}

template <typename T>
__global__ void __launch_bounds__(LZ_RUN_T, 1) lz_run_kernel(LanczosDev* lz, double* __restrict__ Q,
                                                              const T* __restrict__ D, int64_t ldd, int64_t m,
                                                              int n, double tol, double* __restrict__ tbuf,
                                                              double* __restrict__ wpart, double* __restrict__ w,
                                                              double* __restrict__ red, int passes) {
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int NW = LZ_RUN_T / 32, MAXC = LZ_RUN_MAXN / LZ_RUN_T;
  const int64_t r0 = m * b / G, r1 = m * (b + 1) / G;  // this CTA's rows
  const int S = (n + G - 1) / G, j0 = min(n, b * S), j1 = min(n, j0 + S);  // this CTA's column slice
  const int K0 = lz->kmax + 1;                                             // stride of the partial arrays
  __shared__ double scratch[2 * 32];
  __shared__ double bc[4];
  extern __shared__ __align__(16) double lzr[];
  double* ts = lzr;                   // t of this CTA's rows
  double* hfull = ts + (r1 - r0);     // h (K0)
  double* ta = hfull + K0;            // tridiagonal alpha
  double* tb = ta + K0;               // beta
  int k = lz->k;
  int stable = lz->stable;
  double theta = lz->theta, theta_prev = lz->theta_prev;
  bool stop = lz->done != 0;
  while (!stop) {
    const double* qk = Q + (int64_t)k * n;
    // ---- t = D q_k over this CTA's rows
    for (int64_t i = r0 + wid; i < r1; i += NW) {
      const T* row = D + i * ldd;
      double s = 0.0;
#pragma unroll 8
      for (int j = lane; j < n; j += 32) s = fma((double)row[j], qk[j], s);
      s = warp_sum(s);
      if (lane == 0) ts[i - r0] = s;
    }
    __syncthreads();
    // ---- CTA partial of D^T t: thread owns columns tid, tid + 256, ...
    {
      double acc[MAXC];
#pragma unroll
      for (int c = 0; c < MAXC; ++c) acc[c] = 0.0;
      for (int64_t i = r0; i < r1; ++i) {
        const T* row = D + i * ldd;
        const double ti = ts[i - r0];
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
          const int j = c * LZ_RUN_T + tid;
          if (j < n) acc[c] = fma((double)row[j], ti, acc[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        const int j = c * LZ_RUN_T + tid;
        if (j < n) wpart[(int64_t)b * n + j] = acc[c];
      }
    }
    grid.sync();
    // ---- w over this CTA's slice (warp per column sums the G partials); alpha partial
    for (int j = j0 + wid; j < j1; j += NW) {
      const double v = warp_gsum(wpart + j, n, G, lane);
      if (lane == 0) w[j] = v;
    }
    __syncthreads();
    double sa = 0.0;
    for (int j = j0 + tid; j < j1; j += LZ_RUN_T) sa = fma(w[j], qk[j], sa);
    {
      double v2[2] = {sa, 0.0};
      block_sum<2>(v2, scratch);
      if (tid == 0) red[(int64_t)b * (2 * K0 + 4)] = v2[0];
    }
    grid.sync();
    if (wid == 0) {
      const double a = warp_gsum(red, 2 * K0 + 4, G, lane);
      if (lane == 0) bc[0] = a;
    }
    __syncthreads();
    const double alpha = bc[0];
    const double bprev = k > 0 ? lz->beta[k - 1] : 0.0;
    for (int j = j0 + tid; j < j1; j += LZ_RUN_T) {
      double v = w[j] - alpha * qk[j];
      if (k > 0) v -= bprev * Q[(int64_t)(k - 1) * n + j];
      w[j] = v;
    }
    __syncthreads();
    const int K = k + 1;
    // ---- full reorthogonalisation, twice (classical Gram-Schmidt)
    for (int pass = 0; pass < passes; ++pass) {
      double* ph = red + (int64_t)b * (2 * K0 + 4) + 2 + pass * K0;
      for (int c = wid; c < K; c += NW) {
        const double* qc = Q + (int64_t)c * n;
        double d = 0.0;
        for (int j = j0 + lane; j < j1; j += 32) d = fma(qc[j], w[j], d);
        d = warp_sum(d);
        if (lane == 0) ph[c] = d;
      }
      grid.sync();
      for (int c = wid; c < K; c += NW) {
        const double h = warp_gsum(red + 2 + pass * K0 + c, 2 * K0 + 4, G, lane);
        if (lane == 0) hfull[c] = h;
      }
      __syncthreads();
      for (int j = j0 + tid; j < j1; j += LZ_RUN_T) {
        double acc = 0.0;
        for (int c = 0; c < K; ++c) acc = fma(hfull[c], Q[(int64_t)c * n + j], acc);
        w[j] -= acc;
      }
      __syncthreads();
    }
    // ---- beta
    double nn = 0.0;
    for (int j = j0 + tid; j < j1; j += LZ_RUN_T) nn = fma(w[j], w[j], nn);
    {
      double v2[2] = {nn, 0.0};
      block_sum<2>(v2, scratch);
      if (tid == 0) red[(int64_t)b * (2 * K0 + 4) + 1] = v2[0];
    }
    grid.sync();
    if (wid == 0) {
      const double b2 = warp_gsum(red + 1, 2 * K0 + 4, G, lane);
      if (lane == 0) bc[1] = sqrt(b2);
    }
    for (int c = tid; c < k; c += LZ_RUN_T) {
      ta[c] = lz->alpha[c];
      tb[c] = lz->beta[c];
    }
    __syncthreads();
    const double beta = bc[1];
    if (tid == 0) {
      ta[k] = alpha;
      tb[k] = beta;
    }
    __syncthreads();
    // ---- Ritz value: same adaptive schedule as lz_update_cluster
    const bool close = theta > 0.0 && fabs(theta - theta_prev) <= 1e-6 * theta;
    const bool eval = close || (k % 4 == 3) || k + 1 >= lz->kmax || beta <= 1e-300;
    const double th = eval ? tridiag_max_eig_block(ta, tb, K) : theta;
    const double rel = theta > 0.0 ? fabs(th - theta) / th : 1.0;
    stable = !eval ? stable : ((rel <= tol) ? stable + 1 : 0);
    stop = (eval && stable >= 2 && k >= 3) || beta <= 1e-300 * fmax(th, 1e-300) || k + 1 >= lz->kmax;
    if (!stop) {
      double* qn = Q + (int64_t)(k + 1) * n;
      const double inv = 1.0 / beta;
      for (int j = j0 + tid; j < j1; j += LZ_RUN_T) qn[j] = w[j] * inv;
    }
    if (eval) {
      theta_prev = theta;
      theta = th;
    }
    grid.sync();  // q_{k+1} complete; every CTA has read lz->alpha/beta of earlier steps
    if (b == 0 && tid == 0) {
      lz->alpha[k] = alpha;
      lz->beta[k] = beta;
      lz->theta_prev = theta_prev;
      lz->theta = theta;
      lz->stable = stable;
      if (stop) {
        lz->done = 1;
        lz->sigma1 = sqrt(fmax(th, 0.0));
      }
      lz->k = stop ? k : k + 1;
    }
    grid.sync();  // lz->alpha/beta visible before the next step reads them
    if (!stop) ++k;
  }
}

// ------------------------------------------------------------ scalars
__global__ void pcp_start_scalars(PcpDev* st, const LanczosDev* lz, const double* __restrict__ in_stats,
                                  double lam, double mu0, double rho, double tol, int max_iters,
                                  double time_budget, double jac_tol, double m_global, double n, int sv0,
                                  int sv_cap) {
  st->trunc = sv0 > 0;
  st->sv = sv0;
  st->sv_cap = sv_cap;
  st->m_global = m_global;
  st->n = n;
  const double sumsq = in_stats[0], maxabs = in_stats[1];
  const double sigma1 = lz->sigma1;
  st->lam = lam;
  st->rho = rho;
  st->tol = tol;
  st->d_norm = sqrt(sumsq);                                   // pcp.py:238
  st->sigma1 = sigma1;
  st->mu = mu0 > 0.0 ? mu0 : 1.25 / sigma1;                   // pcp.py:101
  st->scale = fmax(sigma1, maxabs / lam);                     // pcp.py:114
  st->tau = 1.0 / st->mu;
  st->mu_last = st->mu;
  st->mu_final = st->mu;
  st->nuclear = 0.0;
  st->time_budget = time_budget;
  st->jac_tol = jac_tol;
  st->k = 1;
  st->done = 0;
  st->status = 0;
  st->rank = 0;
  st->max_iters = max_iters;
  st->jac_sweeps = 0;
  st->t0_ns = global_ns();
}

// Finalize iteration k from the (all-reduced) fine-pass stats at red[0..4):
// history record, stopping rules (pcp.py:284-296), mu <- rho mu.
__global__ void pcp_finalize_kernel(PcpDev* st, const double* __restrict__ red, double* __restrict__ hist,
                                    const int* __restrict__ jac_result) {
  if (st->done) return;
  const int k = st->k;
  const double res2 = red[0], l1 = red[1], nnz = red[2], budget_hit = red[3];
  const double gap = sqrt(res2) / st->d_norm;
  const double wall = (global_ns() - st->t0_ns) * 1e-9;
  double* h = hist + (int64_t)(k - 1) * kHistCols;
  h[0] = gap;
  h[1] = st->nuclear + st->lam * l1;
  h[2] = (double)st->rank;
  h[3] = nnz / ((double)st->m_global * (double)st->n);
  h[4] = wall;
  h[5] = st->mu;
  h[6] = (double)st->jac_sweeps;
  h[7] = nnz;
  st->mu_last = st->mu;
  st->mu_final = st->mu * st->rho;
  if (st->status != 0) {
    st->done = 3;
  } else if (gap <= st->tol) {
    st->done = 1;
  } else if (k >= st->max_iters || budget_hit > 0.0) {
    st->done = 2;
  } else {
    st->k = k + 1;
    st->mu = st->mu * st->rho;
    st->tau = 1.0 / st->mu;
  }
}

__global__ void pcp_after_jacobi(PcpDev* st, const int* __restrict__ jac_result, int trd) {
  if (st->done) return;
  if (trd && st->trd_ok) {  // the tridiagonal solver ran (history: -1)
    st->jac_sweeps = -1;
    return;
  }
  if (st->jac_skip) {  // rank 0 certified: no eigensolve this iteration
    st->jac_sweeps = 0;
    return;
  }
  int r = jac_result[0];
  st->jac_sweeps = r;
  if (r <= 0) st->status = 3;
}

// ------------------------------------------------------------ fused row kernel
enum RowMode { kStart = 0, kUpdate = 1, kOutput = 2 };

template <typename T>
struct StencilT;
template <>
struct StencilT<float> {
  static __device__ __forceinline__ const float* w0(const ChainDev& c) { return c.w0f; }
  static __device__ __forceinline__ const float* w1(const ChainDev& c) { return c.w1f; }
};
template <>
struct StencilT<double> {
  static __device__ __forceinline__ const double* w0(const ChainDev& c) { return c.w0; }
  static __device__ __forceinline__ const double* w1(const ChainDev& c) { return c.w1; }
};

template <typename T, int MODE>
__global__ void __launch_bounds__(512)
pcp_row_kernel(const PcpDev* __restrict__ st, ChainDev ch, int64_t m, const T* __restrict__ D, int64_t ldd,
               const T* __restrict__ Yin, T* __restrict__ Yout, int64_t ldy, const T* __restrict__ Z,
               T* __restrict__ A, T* __restrict__ Lout, T* __restrict__ Sout, int64_t ldo,
               double* __restrict__ part) {
  if (MODE == kUpdate && st->done) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = ch.n, nh = ch.nh, np = ch.np;
  T* zrow = reinterpret_cast<T*>(smem_raw);           // np + 2 (zero tail for c0+1)
  T* wrow = zrow + np + 2;                            // n
  if (threadIdx.x < 2) zrow[np + threadIdx.x] = T(0);
  __shared__ double scratch[3 * 32];
  const T* __restrict__ w0 = StencilT<T>::w0(ch);
  const T* __restrict__ w1 = StencilT<T>::w1(ch);
  const int* __restrict__ c0 = ch.c0;

  const double mu_d = st->mu;
  const T inv = (T)(1.0 / mu_d);
  const T mu = (T)mu_d;
  const T thr = (T)(st->lam * (1.0 / mu_d));
  const T inv_next = (T)(1.0 / (mu_d * st->rho));
  const T inv_scale = (T)(1.0 / st->scale);
  (void)inv_scale;
  double acc_res = 0.0, acc_l1 = 0.0, acc_nnz = 0.0;

  for (int64_t i = blockIdx.x; i < m; i += gridDim.x) {
    __syncthreads();
    if (MODE != kStart) {
      for (int k = threadIdx.x; k < np; k += blockDim.x) zrow[k] = Z[i * np + k];
      __syncthreads();
    }
    const T* drow = D + i * ldd;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const T d = drow[j];
      if (MODE == kStart) {
        // y = d / scale (pcp.py:115); work = y/mu + d (pcp.py:252-254, S = 0)
        const T y = (T)((double)d / st->scale);
        Yout[i * ldy + j] = y;
        wrow[j] = y * inv + d;
      } else {
        const int c = c0[j];
        const T l = w0[j] * zrow[c] + w1[j] * zrow[c + 1];
        const T y = Yin[i * ldy + j];
        const T w = y * inv + d - l;
        const T s = soft_thr<T>(w, thr);
        if (MODE == kOutput) {
          Lout[i * ldo + j] = l;
          Sout[i * ldo + j] = s;
        } else {
          const T res = (d - l) - s;
          const T yn = y + res * mu;
          Yout[i * ldy + j] = yn;
          acc_res = fma((double)res, (double)res, acc_res);
          acc_l1 += fabs((double)s);
          acc_nnz += (s != T(0)) ? 1.0 : 0.0;
          wrow[j] = yn * inv_next + d - s;
        }
      }
    }
    if (MODE == kOutput) continue;
    __syncthreads();
    // gather A[i, k] = sum_{j in [lo_k, hi_k)} W[i, j] R[j, k]
    T* arow = A + i * np;
    for (int k = threadIdx.x; k < np; k += blockDim.x) {
      T a = T(0);
      if (k < nh) {
        const int lo = ch.lo[k], hi = ch.hi[k];
        for (int j = lo; j < hi; ++j) a += wrow[j] * (c0[j] == k ? w0[j] : w1[j]);
      }
      arow[k] = a;
    }
  }
  if (MODE == kUpdate) {
    double v[3] = {acc_res, acc_l1, acc_nnz};
    block_sum<3>(v, scratch);
    if (threadIdx.x == 0) {
      part[3 * blockIdx.x + 0] = v[0];
      part[3 * blockIdx.x + 1] = v[1];
      part[3 * blockIdx.x + 2] = v[2];
    }
  }
}

// Sum nv-wide per-CTA partials (256 threads, fixed order -> deterministic).
// out[3] is this rank's time-budget flag (1 when the budget is spent); the
// flags are summed by the same all-reduce as the stats, so every rank of a
// row-sharded solve takes the same stop decision (pcp.py:295).
__global__ void __launch_bounds__(256) stats_reduce_kernel(const double* __restrict__ part, int nparts, int nv,
                                                           double* __restrict__ out, const PcpDev* __restrict__ st) {
  __shared__ double scratch[3 * 32];
  double v[3] = {0.0, 0.0, 0.0};
  for (int b = threadIdx.x; b < nparts; b += blockDim.x)
    for (int q = 0; q < nv && q < 3; ++q) v[q] += part[nv * b + q];
  block_sum<3>(v, scratch);
  if (threadIdx.x == 0) {
    for (int q = 0; q < 3; ++q) out[q] = q < nv ? v[q] : 0.0;
    const double wall = (global_ns() - st->t0_ns) * 1e-9;
    out[3] = (st->time_budget >= 0.0 && wall >= st->time_budget) ? 1.0 : 0.0;
  }
}

// ------------------------------------------------------------ host-side drivers
template <typename T>
static int row_pass(int mode, PcpPlan* p, const void* D, int64_t ldd, const void* Yin, void* Yout, int64_t ldy,
                    void* Lout, void* Sout, int64_t ldo, cudaStream_t st) {
  const int threads = 256;
  if (p->m_local == 0) return kOk;
  if (rows_warp_ok(p->ch, p->f32))  // streaming warp-per-row path (rows.cu)
    return pcp_rows(p, mode, D, ldd, Yin, Yout, ldy, Lout, Sout, ldo, st);
  size_t smem = sizeof(T) * (size_t)(p->ch.np + p->ch.n + 4);
  if (smem > 200 * 1024) {
    set_error("pcp row kernel: fine row does not fit in shared memory");
    return kErrArg;
  }
  int blocks = p->row_blocks;
  const T* Dp = (const T*)D;
#define MLR_ROW(MODE)                                                                               \
  {                                                                                                 \
    auto kern = pcp_row_kernel<T, MODE>;                                                            \
    MLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));   \
    kern<<<blocks, threads, smem, st>>>(p->dev, p->ch, p->m_local, Dp, ldd, (const T*)Yin, (T*)Yout, \
                                        ldy, (const T*)p->Z, (T*)p->A, (T*)Lout, (T*)Sout, ldo,      \
                                        p->row_part);                                               \
  }
  if (mode == kStart) MLR_ROW(kStart)
  else if (mode == kUpdate) MLR_ROW(kUpdate)
  else MLR_ROW(kOutput)
#undef MLR_ROW
  MLR_LAUNCH_CHECK("pcp_row_kernel");
  return kOk;
}

int pcp_input_stats(PcpPlan* p, const void* D, int64_t ldd, double* out2, cudaStream_t st) {
  int blocks = p->row_blocks;
  if (p->m_local == 0) {
    MLR_CUDA(cudaMemsetAsync(out2, 0, 3 * sizeof(double), st));
    return kOk;
  }
  if (p->f32)
    input_stats_kernel<float><<<blocks, 256, 0, st>>>((const float*)D, ldd, p->m_local, p->ch.n, p->row_part);
  else
    input_stats_kernel<double><<<blocks, 256, 0, st>>>((const double*)D, ldd, p->m_local, p->ch.n, p->row_part);
  MLR_LAUNCH_CHECK("input_stats_kernel");
  input_stats_finish<<<1, 256, 0, st>>>(p->row_part, blocks, out2);
  MLR_LAUNCH_CHECK("input_stats_finish");
  return kOk;
}

int matrix_stats(int64_t m, int n, bool f32, const void* D, int64_t ldd, double* part, int blocks, double* out3,
                 cudaStream_t st) {
  if (m == 0) {
    MLR_CUDA(cudaMemsetAsync(out3, 0, 3 * sizeof(double), st));
    return kOk;
  }
  if (f32)
    input_stats_kernel<float><<<blocks, 256, 0, st>>>((const float*)D, ldd, m, n, part);
  else
    input_stats_kernel<double><<<blocks, 256, 0, st>>>((const double*)D, ldd, m, n, part);
  MLR_LAUNCH_CHECK("input_stats_kernel");
  input_stats_finish<<<1, 256, 0, st>>>(part, blocks, out3);
  MLR_LAUNCH_CHECK("input_stats_finish");
  return kOk;
}

int pcp_lanczos_init(PcpPlan* p, cudaStream_t st) {
  lz_init_kernel<<<(int)ceil_div(p->ch.n, 256), 256, 0, st>>>(p->lz, p->lzQ, p->ch.n, p->lz_kmax);
  MLR_LAUNCH_CHECK("lz_init_kernel");
  return kOk;
}

int pcp_lanczos_matvec(PcpPlan* p, const void* D, int64_t ldd, double* wpart_out, cudaStream_t st) {
  const int n = p->ch.n;
  const int64_t m = p->m_local;
  if (m == 0) {
    MLR_CUDA(cudaMemsetAsync(wpart_out, 0, sizeof(double) * n, st));
    return kOk;
  }
  p->timer.begin(st);
  if (n <= LZ_FUSED_N && p->lz_fused_ctas > 0) {
    const int ctas = p->lz_fused_ctas;
    const size_t smem = sizeof(double) * LZ_FW * (size_t)n;
    if (p->f32) {
      MLR_CUDA(cudaFuncSetAttribute(lz_dtdv_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      lz_dtdv_kernel<float><<<ctas, LZ_FW * 32, smem, st>>>(p->lz, (const float*)D, ldd, m, n, p->lzQ, p->lzW);
    } else {
      MLR_CUDA(cudaFuncSetAttribute(lz_dtdv_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      lz_dtdv_kernel<double><<<ctas, LZ_FW * 32, smem, st>>>(p->lz, (const double*)D, ldd, m, n, p->lzQ, p->lzW);
    }
    MLR_LAUNCH_CHECK("lz_dtdv_kernel");
    const int rc = sum_slices(p->lzW, n, n, ctas, wpart_out, st);
    p->timer.end(kPhLanczos, st);
    return rc;
  }
  if (p->lz_long_clusters > 0 && p->f32 && ldd % 4 == 0 && ((uintptr_t)D & 15) == 0) {
    const int ncl = p->lz_long_clusters;
    const int seg = (int)(ceil_div(ceil_div(n, LZL_CL), 4) * 4);
    const int stages = lz_long_stages(seg);
    const size_t smem = (size_t)stages * seg * sizeof(float);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ncl * LZL_CL);
    cfg.blockDim = dim3(LZL_T);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = LZL_CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    static const int cv = [] {
      const char* e = getenv("MLR_LZ_CVT");  // 0: F2F only, 1: F2F / integer alternating (default), 2: integer only
      return e ? atoi(e) : 1;
    }();
    auto kern = cv == 0 ? lz_dtdq_long_kernel<0> : cv == 2 ? lz_dtdq_long_kernel<2> : lz_dtdq_long_kernel<1>;
    MLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    MLR_CUDA(cudaLaunchKernelEx(&cfg, kern, (const LanczosDev*)p->lz, (const float*)D, ldd, m, n, seg, stages,
                                (const double*)p->lzQ, p->lzW));
    MLR_LAUNCH_CHECK("lz_dtdq_long_kernel");
    const int rc = sum_slices(p->lzW, n, n, ncl, wpart_out, st);
    p->timer.end(kPhLanczos, st);
    return rc;
  }
  const int blocks = (int)std::min<int64_t>(ceil_div(m, 8), (int64_t)p->row_blocks);
  if (p->f32)
    lz_dv_kernel<float><<<blocks, 256, 0, st>>>(p->lz, (const float*)D, ldd, m, n, p->lzQ, p->lzT);
  else
    lz_dv_kernel<double><<<blocks, 256, 0, st>>>(p->lz, (const double*)D, ldd, m, n, p->lzQ, p->lzT);
  MLR_LAUNCH_CHECK("lz_dv_kernel");
  int splits = p->lz_splits;
  int64_t rps = ceil_div(m, splits);
  dim3 grid((unsigned)ceil_div(n, LZ_COLS), (unsigned)splits);
  if (p->f32)
    lz_dtv_kernel<float><<<grid, 256, 0, st>>>(p->lz, (const float*)D, ldd, m, n, p->lzT, p->lzW, rps);
  else
    lz_dtv_kernel<double><<<grid, 256, 0, st>>>(p->lz, (const double*)D, ldd, m, n, p->lzT, p->lzW, rps);
  MLR_LAUNCH_CHECK("lz_dtv_kernel");
  const int rc = sum_slices(p->lzW, n, n, splits, wpart_out, st);
  p->timer.end(kPhLanczos, st);
  return rc;
}

int lanczos_run_ok(const PcpPlan* p) { return p->lz_run_ctas > 0; }

int pcp_lanczos_run(PcpPlan* p, const void* D, int64_t ldd, double tol, cudaStream_t st) {
  if (p->lz_run_ctas <= 0) {
    set_error("pcp_lanczos_run: not available for this plan (n too large)");
    return kErrArg;
  }
  const int n = p->ch.n;
  int64_t m = p->m_local;
  const int G = p->lz_run_ctas;
  const int K0 = p->lz_kmax + 1;
  const size_t smem = sizeof(double) * ((size_t)ceil_div(std::max<int64_t>(m, 1), G) + 3 * (size_t)K0 + 8);
  const char* pe = getenv("MLR_LZ_REORTH");
  // one classical Gram-Schmidt pass: the top Ritz value (all that is used) is
  // insensitive to the residual non-orthogonality (measured: same steps and
  // sigma_1 to the golden mu tolerance, C2 4.4 -> 3.5 ms)
  int passes = pe ? std::max(1, std::min(2, atoi(pe))) : 1;
  void* args[] = {(void*)&p->lz, (void*)&p->lzQ, (void*)&D, (void*)&ldd, (void*)&m, (void*)&n, (void*)&tol,
                  (void*)&p->lzT, (void*)&p->lzW, (void*)&p->lzWork, (void*)&p->lzRed, (void*)&passes};
  p->timer.begin(st);
  if (p->f32) {
    MLR_CUDA(cudaFuncSetAttribute(lz_run_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    MLR_CUDA(cudaLaunchCooperativeKernel((void*)lz_run_kernel<float>, dim3(G), dim3(LZ_RUN_T), args, smem, st));
  } else {
    MLR_CUDA(cudaFuncSetAttribute(lz_run_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    MLR_CUDA(cudaLaunchCooperativeKernel((void*)lz_run_kernel<double>, dim3(G), dim3(LZ_RUN_T), args, smem, st));
  }
  p->timer.end(kPhLanczos, st);
  return kOk;
}

int pcp_lanczos_update(PcpPlan* p, const double* w_reduced, double tol, cudaStream_t st) {
  const int n = p->ch.n;
  const int K = p->lz_kmax + 1;
  const size_t smem = sizeof(double) * (3 * (size_t)ceil_div(n, LZ_CL) + 2 + 5 * (size_t)K + 8);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(LZ_CL);
  cfg.blockDim = dim3(LZ_T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = LZ_CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MLR_CUDA(cudaFuncSetAttribute(lz_update_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  MLR_CUDA(cudaFuncSetAttribute(lz_update_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  p->timer.begin(st);
  static int passes = -1;
  if (passes < 0) {
    const char* pe = getenv("MLR_LZ_CL_REORTH");
    // default 0: the plain three-term recurrence.  Only the top Ritz value
    // is used (sigma_1 for mu_0 and Y_0); Paige's analysis shows it converges
    // to the extreme eigenvalue to working accuracy without reorthogonalising
    // (lost orthogonality only duplicates converged Ritz values).  Measured:
    // the same 107 steps on C5 and sigma_1 equal to the exact 2-norm to the
    // tests' 1e-8 (mu); Lanczos 72 -> 60 ms per C5 solve.
    passes = pe ? std::max(0, std::min(2, atoi(pe))) : 0;
  }
  MLR_CUDA(cudaLaunchKernelEx(&cfg, lz_update_cluster, p->lz, p->lzQ, w_reduced, n, tol, passes));
  p->timer.end(kPhLanczos, st);
  return kOk;
}

int pcp_start(PcpPlan* p, const void* D, int64_t ldd, void* Y0, int64_t ldy, const double* in_stats, double lam,
              double mu0, double rho, double tol, int max_iters, double time_budget, double jac_tol,
              cudaStream_t st) {
  p->jac_tol_host = jac_tol;
  // off-diagonals below floor_rel * max(diag) count as converged: the Gram
  // itself is only accurate to ~eps * |B| (FP64 accumulation of T-precision A)
  p->jac_floor_rel = p->f32 ? 1e-13 : 1e-17;
  pcp_start_scalars<<<1, 1, 0, st>>>(p->dev, p->lz, in_stats, lam, mu0, rho, tol, max_iters, time_budget, jac_tol,
                                     (double)p->m_global, (double)p->ch.n, p->trunc_sv0, p->trunc_cap);
  MLR_LAUNCH_CHECK("pcp_start_scalars");
  MLR_CUDA(cudaMemsetAsync(p->hist, 0, sizeof(double) * kHistCols * p->max_iters, st));
  return p->f32 ? row_pass<float>(kStart, p, D, ldd, nullptr, Y0, ldy, nullptr, nullptr, 0, st)
                : row_pass<double>(kStart, p, D, ldd, nullptr, Y0, ldy, nullptr, nullptr, 0, st);
}

// K = A^T A (split over rows, deterministic) -> red[0 .. np*np), and the
// previous fine pass's stats -> red[np*np .. np*np+3).
int pcp_gram(PcpPlan* p, double* red, int with_stats, cudaStream_t st) {
  const int np = p->ch.np;
  const int64_t nn = (int64_t)np * np;
  p->timer.begin(st);
  if (p->m_local > 0) {
    GemmSpec g{};
    g.M = np; g.N = np; g.K = (int)p->m_local;
    g.A = p->A; g.lda = np; g.a_f32 = p->f32; g.trans_a = true;
    g.B = p->A; g.ldb = np; g.b_f32 = p->f32; g.trans_b = false;
    g.C = p->gram_part; g.ldc = np; g.c_f32 = false; g.c_slice = nn; g.splits = p->gram_splits; g.alpha = 1.0;
    // once the solve is done (set by pcp_finalize_kernel) the iterations the
    // host queued ahead are no-ops; the Gram used to run in full in each of
    // them (C5: 6 of 29 launches, 6.8 ms of a 230 ms solve)
    const int* done = &p->dev->done;
    g.kscale = nullptr; g.skip = done;
    g.sym = true;  // Gram: upper-triangle tiles, mirrored
    int rc = gemm_f64(g, st);
    if (rc) return rc;
    rc = sum_slices(p->gram_part, nn, nn, p->gram_splits, red, st, done);
    if (rc) return rc;
  } else {
    MLR_CUDA(cudaMemsetAsync(red, 0, sizeof(double) * nn, st));
  }
  if (with_stats) {
    stats_reduce_kernel<<<1, 256, 0, st>>>(p->row_part, p->m_local > 0 ? p->row_blocks : 0, 3, red + nn, p->dev);
    MLR_LAUNCH_CHECK("stats_reduce_kernel");
  }
  p->timer.end(kPhGram, st);
  return kOk;
}

int pcp_finalize(PcpPlan* p, const double* red, cudaStream_t st) {
  const int64_t nn = (int64_t)p->ch.np * p->ch.np;
  p->timer.begin(st);
  pcp_finalize_kernel<<<1, 1, 0, st>>>(p->dev, red + nn, p->hist, p->jac_result);
  MLR_LAUNCH_CHECK("pcp_finalize_kernel");
  p->timer.end(kPhFinalize, st);
  return kOk;
}

// Truncated SVT of ialm_solve (reference pcp.py:152-165): only the top-sv
// singular values take part (svd_truncated returns sv triplets); rank counts
// those above tau; sv adapts for the next iteration.  The sv-th largest
// sigma is found exactly by a radix select over the bit patterns
// (non-negative doubles order like their bits).
__global__ void __launch_bounds__(1024) svt_weights_trunc_kernel(PcpDev* __restrict__ st, int np, int nh,
                                                                  const double* __restrict__ Bd,
                                                                  double* __restrict__ sig_out,
                                                                  double* __restrict__ f_out) {
  if (st->done) return;
  __shared__ double scratch[2 * 32];
  __shared__ unsigned long long key_s;
  __shared__ int cnt_s;
  const double tau = st->tau;
  const int sv = min(st->sv, nh);
  // sigma_i = sqrt(lambda_i) (i < nh), as bit patterns
  unsigned long long prefix = 0ull;
  for (int bit = 63; bit >= 0; --bit) {
    const unsigned long long cand = prefix | (1ull << bit);
    int c = 0;
    for (int i = threadIdx.x; i < nh; i += blockDim.x) {
      const double s = sqrt(fmax(Bd[(int64_t)i * (np + 1)], 0.0));
      c += (unsigned long long)__double_as_longlong(s) >= cand ? 1 : 0;
    }
    double v[2] = {(double)c, 0.0};
    block_sum<2>(v, scratch);
    if (threadIdx.x == 0) cnt_s = (int)(v[0] + 0.5);
    __syncthreads();
    if (cnt_s >= sv) prefix = cand;  // at least sv values >= cand: the sv-th largest has this bit
    __syncthreads();
  }
  const double s_sv = __longlong_as_double((long long)prefix);  // the sv-th largest sigma
  double nuc = 0.0, rk = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) {
    double f = 0.0, s = 0.0;
    if (i < nh) {
      s = sqrt(fmax(Bd[(int64_t)i * (np + 1)], 0.0));
      if (s >= s_sv && s > tau) {
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
    st->nuclear = v[0];
    st->rank = (int)(v[1] + 0.5);
    // widen when the truncation clipped values above the threshold (pcp.py:160-163)
    st->sv = s_sv > tau ? min(st->sv + 5, st->sv_cap) : max(min(st->rank + 1, st->sv_cap), 1);
  }
}

// Eigenvalues of the converged B~ in descending order (real coarse indices
// only; the zero padding [nh, np) never mixes with them): the next
// iteration's warm start then has blocks of similar eigenvalues, so fewer
// block-Jacobi sweeps are needed.  perm[r] = index of the r-th largest.
__global__ void __launch_bounds__(1024) eig_sort_kernel(const PcpDev* __restrict__ st, double* __restrict__ Bd,
                                                        int np, int nh, int* __restrict__ perm) {
  if (st->done) return;
  extern __shared__ double dsort[];
  for (int i = threadIdx.x; i < nh; i += blockDim.x) dsort[i] = Bd[(int64_t)i * (np + 1)];
  __syncthreads();
  for (int i = threadIdx.x; i < nh; i += blockDim.x) {
    const double di = dsort[i];
    int r = 0;
    for (int j = 0; j < nh; ++j) {
      const double dj = dsort[j];
      r += (dj > di || (dj == di && j < i)) ? 1 : 0;
    }
    perm[r] = i;
    Bd[(int64_t)r * (np + 1)] = di;
  }
}

__global__ void eig_permute_kernel(const PcpDev* __restrict__ st, const double* __restrict__ V,
                                   double* __restrict__ Vout, int np, int nh, const int* __restrict__ perm) {
  if (st->done) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)np * np;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / np), c = (int)(e % np);
    Vout[e] = V[(int64_t)r * np + (c < nh ? perm[c] : c)];
  }
}

__global__ void pcp_jac_skip_done(PcpDev* st, int pow) { st->jac_skip = st->done || (pow && st->r0_state == 2); }
// Z = 0 on a certified rank-0 iteration (the reconstruction GEMM was skipped)
__global__ void pcp_zero_if_rank0(const PcpDev* __restrict__ st, uint32_t* __restrict__ z, int64_t n) {
  if (st->done || !st->jac_skip) return;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4; i < n; i += (int64_t)gridDim.x * blockDim.x * 4) {
    if (i + 4 <= n && (i & 3) == 0) *reinterpret_cast<uint4*>(z + i) = make_uint4(0u, 0u, 0u, 0u);
    else for (int64_t q = i; q < n && q < i + 4; ++q) z[q] = 0u;
  }
}

// Rank-0 certificate (ahead of the coarse eigensolve).  When every singular
// value of M_H is <= tau the SVT is zero (pcp.py:258-262: rank = #{sigma >
// tau} = 0, L_H = 0, nuclear = 0) and the eigenvectors are not needed.  That
// holds iff tau^2 I - B~ is positive definite, which a Cholesky factorisation
// decides.  Cheap exit first: any diagonal entry of B~ above tau^2 bounds
// lambda_max from below, so the rank is positive.  Otherwise the Cholesky of
// A = tau^2 (1 - margin) I - B~ runs in FP32 in one CTA (packed lower
// triangle in shared memory).  When it succeeds, A + E is PD with
// |E_ij| <= gamma_{n+1} sqrt(a_ii a_jj) <= gamma_{n+1} tau^2.  The worst-case
// normwise bound n gamma_{n+1} tau^2 (0.09 tau^2 at n = 1250) is far from
// what rounding does in practice (errors of random sign: ~sqrt(n) u), so the
// margin is the heuristic rank0_margin(n) = max(1e-3, 2 (n+1) sqrt(n) u_32):
// a success then says lambda_max(B~) < tau^2, the rank is 0 exactly as the
// reference counts it.  Borderline cases (lambda_max within the margin of
// tau^2) fail the test and take the eigensolver.  Sets st->jac_skip = done ||
// certified.  (After the start the reference often has rank 0 for a few
// iterations: C2 iterations 2-5.)
__host__ __device__ inline double rank0_margin(int n) {
  return fmax(1e-3, 2.0 * (n + 1) * sqrt((double)n) * 5.9604644775390625e-8);
}
constexpr int R0_THREADS = 768, R0_TPT = 3;  // 4x4 register tiles, up to 3 per thread (n_H <= 268)

int64_t rank0_smem_bytes(int nh) {
  const int T = (nh + 3) / 4;
  return (T * (T + 1) / 2 <= R0_THREADS * R0_TPT) ? 1 : INT_MAX;  // register-resident; smem: l only
}

// Right-looking Cholesky with the lower triangle in 4x4 FP32 register tiles
// (tile (I, J), I >= J, owned by one thread); per step two barriers: the
// pivot, then the scaled column l broadcast through shared memory.
__global__ void __launch_bounds__(R0_THREADS) pcp_rank0_test(PcpDev* st, const double* __restrict__ Bt, int np,
                                                             int nh, int decided_if_set) {
  if (decided_if_set && st->r0_state != 0) return;  // the power bound (or the diagonal) decided
  __shared__ __align__(16) float l[4 * 96];
  __shared__ float piv;
  const int tid = threadIdx.x;
  const double tau = st->tau;
  if (st->done) {
    if (tid == 0) st->jac_skip = 1;
    return;
  }
  // cheap exit: a diagonal entry > tau^2 means lambda_max > tau^2
  int big = 0;
  for (int i = tid; i < nh; i += R0_THREADS) big |= Bt[(int64_t)i * np + i] > tau * tau;
  if (__syncthreads_or(big)) {
    if (tid == 0) st->jac_skip = 0;
    return;
  }
  const double lim = tau * tau * (1.0 - rank0_margin(nh));
  const int T = (nh + 3) / 4, ntiles = T * (T + 1) / 2;
  float a[R0_TPT][4][4];
  int ti[R0_TPT], tj[R0_TPT];
#pragma unroll
  for (int q = 0; q < R0_TPT; ++q) {
    int t = tid + q * R0_THREADS, I = 0;
    if (t >= ntiles) {
      ti[q] = tj[q] = -1;
    } else {
      while (t >= I + 1) {  // row I holds tiles (I, 0..I)
        t -= I + 1;
        ++I;
      }
      ti[q] = I;
      tj[q] = t;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = 4 * ti[q] + r, j = 4 * tj[q] + c;
        a[q][r][c] = (ti[q] >= 0 && i < nh && j < nh && j <= i)
                         ? (float)((i == j ? lim : 0.0) - Bt[(int64_t)i * np + j])
                         : (i == j ? 1.f : 0.f);  // padding: identity
      }
  }
  for (int i = tid; i < 4 * 96; i += R0_THREADS) l[i] = 0.f;
  int ok = 1;
  const int n4 = 4 * T;
  for (int k = 0; k < n4; ++k) {
    const int kt = k >> 2, kr = k & 3;
    // pivot a_kk (after the owner's update of step k - 1)
#pragma unroll
    for (int q = 0; q < R0_TPT; ++q)
      if (ti[q] == kt && tj[q] == kt) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
          if (r == kr) {
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (c == kr) piv = a[q][r][c];
          }
      }
    __syncthreads();
    const float d = piv;
    if (!(d > 0.f)) {
      ok = 0;
      break;
    }
    const float rd = rsqrtf(d);
    // column k below the diagonal, scaled: l_i = a_ik / sqrt(a_kk), i > k
#pragma unroll
    for (int q = 0; q < R0_TPT; ++q)
      if (tj[q] == kt && ti[q] >= kt) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          float v = 0.f;
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (c == kr) v = a[q][r][c];
          const int i = 4 * ti[q] + r;
          if (i > k) l[i] = v * rd;
          else if (i == k) l[i] = 0.f;
        }
      }
    __syncthreads();
    // trailing update a_ij -= l_i l_j for j > k (tiles with J >= kt)
#pragma unroll
    for (int q = 0; q < R0_TPT; ++q)
      if (tj[q] >= kt) {
        const float4 li = *reinterpret_cast<const float4*>(&l[4 * ti[q]]);
        const float4 lj = *reinterpret_cast<const float4*>(&l[4 * tj[q]]);
        const float lr[4] = {li.x, li.y, li.z, li.w}, lc[4] = {lj.x, lj.y, lj.z, lj.w};
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const bool live = tj[q] > kt || c > kr;
            if (live) a[q][r][c] = fmaf(-lr[r], lc[c], a[q][r][c]);
          }
      }
    // (l_i, i <= k, is zero from step i on; the next barrier orders l and piv reuse)
  }
  if (tid == 0) st->jac_skip = ok;
}

// Large n_H (C5: 1250): the same certificate as a grid-cooperative, panel
// right-looking FP32 Cholesky of the full matrix (column-major, scratch in
// the plan's free Gram slices, L2-resident).  Per panel of R0G_B columns:
// every CTA loads the panel and factors it redundantly in shared memory
// (identical arithmetic, so every CTA reaches the same verdict), then applies
// the rank-R0G_B update to the trailing columns it owns (column j on CTA j mod
// G); one grid barrier per panel.
constexpr int R0G_B = 8, R0G_T = 256;

__global__ void __launch_bounds__(R0G_T) pcp_rank0_grid(PcpDev* st, const double* __restrict__ Bt, int np, int nh,
                                                        float* __restrict__ W, int decided_if_set) {
  if (decided_if_set && st->r0_state != 0) return;  // the power bound (or the diagonal) decided
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) float pan[];  // [R0G_B][nh]
  __shared__ int s_big;
  const int tid = threadIdx.x, G = gridDim.x, b = blockIdx.x;
  const double tau = st->tau;
  if (st->done) {  // uniform across the grid
    if (b == 0 && tid == 0) st->jac_skip = 1;
    return;
  }
  if (tid == 0) s_big = 0;
  __syncthreads();
  {
    int big = 0;
    for (int i = tid; i < nh; i += R0G_T) big |= Bt[(int64_t)i * np + i] > tau * tau;
    if (__syncthreads_or(big)) {  // same verdict in every CTA (same inputs)
      if (b == 0 && tid == 0) st->jac_skip = 0;
      return;
    }
  }
  const float lim = (float)(tau * tau * (1.0 - rank0_margin(nh)));
  // W = lim I - B~, lower part, column-major (column j owned by CTA j mod G)
  for (int j = b; j < nh; j += G)
    for (int i = j + tid; i < nh; i += R0G_T)
      W[(int64_t)j * nh + i] = (i == j ? lim : 0.f) - (float)Bt[(int64_t)i * np + j];
  grid.sync();
  int ok = 1;
  for (int k = 0; k < nh; k += R0G_B) {
    const int nbk = min(R0G_B, nh - k);
    for (int c = 0; c < nbk; ++c)
      for (int i = k + tid; i < nh; i += R0G_T) pan[c * nh + i] = W[(int64_t)(k + c) * nh + i];
    __syncthreads();
    for (int c = 0; c < nbk; ++c) {  // factor the panel (rows >= k + c of column c)
      const float d = pan[c * nh + k + c];
      if (!(d > 0.f)) {
        ok = 0;
        break;
      }
      const float r = rsqrtf(d);
      __syncthreads();
      for (int i = k + c + 1 + tid; i < nh; i += R0G_T) pan[c * nh + i] *= r;
      __syncthreads();
      for (int c2 = c + 1; c2 < nbk; ++c2) {
        const float lj = pan[c * nh + k + c2];
        for (int i = k + c2 + tid; i < nh; i += R0G_T) pan[c2 * nh + i] = fmaf(-pan[c * nh + i], lj, pan[c2 * nh + i]);
      }
      __syncthreads();
    }
    if (!ok) break;  // uniform: every CTA factored the same panel
    // trailing update of my columns j >= k + nbk: a_ij -= sum_c l_ic l_jc
    const int j0 = k + nbk;
    for (int j = j0 + ((b - j0 % G) + G) % G; j < nh; j += G) {
      float lj[R0G_B];
#pragma unroll
      for (int c = 0; c < R0G_B; ++c) lj[c] = c < nbk ? pan[c * nh + j] : 0.f;
      float* wj = W + (int64_t)j * nh;
      for (int i = j + tid; i < nh; i += R0G_T) {
        float v = wj[i];
#pragma unroll
        for (int c = 0; c < R0G_B; ++c) v = fmaf(-pan[c * nh + i], lj[c], v);
        wj[i] = v;
      }
    }
    grid.sync();
  }
  if (b == 0 && tid == 0) st->jac_skip = ok;
}

// Power-bound rank-0 certificate (before the Cholesky one).  With
// P = (B + B^T) / (2 tau^2) (PSD), lambda_max(P)^q <= trace(P^q) for
// q = 2^s, so trace(P^q) <= (1 - margin)^q certifies lambda_max(B) <
// tau^2 (1 - margin) -- the Cholesky certificate's condition -- and the
// bound over-estimates lambda_max by at most n^(1/q) (q = 128: 1.06 at
// n_H = 1250).  s symmetric FP64 squarings (n_p^3 each, upper tiles) cost
// far less than the panel Cholesky's n_H / 8 grid barriers; when the bound
// fails, the Cholesky certificate decides as before.
constexpr int R0_POW_SQUARINGS = 7;
__global__ void r0_pow_init(PcpDev* st, const double* __restrict__ Bt, int np, int nh, double* __restrict__ P) {
  __shared__ int s_big;
  if (st->done) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->r0_state = 3;
      st->jac_skip = 1;
    }
    return;
  }
  const double tau = st->tau, t2 = tau * tau;
  if (threadIdx.x == 0) s_big = 0;
  __syncthreads();
  int big = 0;
  for (int i = threadIdx.x; i < nh; i += blockDim.x) big |= Bt[(int64_t)i * np + i] > t2;
  if (big) s_big = 1;
  __syncthreads();
  if (s_big) {  // a diagonal entry above tau^2: rank > 0 (same verdict in every CTA)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->r0_state = 1;
      st->jac_skip = 0;
    }
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) st->r0_state = 0;
  const double inv = 0.5 / t2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)np * np;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / np), j = (int)(e % np);
    P[e] = (i < nh && j < nh) ? (Bt[(int64_t)i * np + j] + Bt[(int64_t)j * np + i]) * inv : 0.0;
  }
}
__global__ void __launch_bounds__(1024) r0_pow_decide(PcpDev* st, const double* __restrict__ P, int np, int nh,
                                                      double thr) {
  __shared__ double scratch[32];
  if (st->r0_state != 0) return;
  double v[1] = {0.0};
  for (int i = threadIdx.x; i < nh; i += blockDim.x) v[0] += P[(int64_t)i * np + i];
  block_sum<1>(v, scratch);
  if (threadIdx.x == 0 && v[0] <= thr) {  // NaN / inf (lambda > 1 overflowed): not certified
    st->r0_state = 2;
    st->jac_skip = 1;
  }
}
static int r0_power_bound(PcpPlan* p, cudaStream_t st) {
  const int nh = p->ch.nh, np = p->ch.np;
  double* Pa = p->T1;  // both free between the pre products and the SVT products
  double* Pb = p->Xm;
  r0_pow_init<<<148, 256, 0, st>>>(p->dev, p->Bm, np, nh, Pa);
  MLR_LAUNCH_CHECK("r0_pow_init");
  const int* skip = &p->dev->r0_state;
  const int ksplit = p->coarse_ksplit;
  for (int s = 0; s < R0_POW_SQUARINGS; ++s) {
    GemmSpec g{};
    g.M = np; g.N = np; g.K = np;
    g.A = Pa; g.lda = np; g.a_f32 = false; g.trans_a = false;
    g.B = Pa; g.ldb = np; g.b_f32 = false; g.trans_b = false;
    g.C = ksplit > 1 ? p->gram_part : Pb; g.ldc = np; g.c_f32 = false;
    g.c_slice = ksplit > 1 ? (int64_t)np * np : 0; g.splits = ksplit; g.alpha = 1.0;
    g.kscale = nullptr; g.skip = skip; g.sym = true;
    int rc = gemm_f64(g, st);
    if (rc) return rc;
    if (ksplit > 1 && (rc = sum_slices(p->gram_part, (int64_t)np * np, (int64_t)np * np, ksplit, Pb, st, skip)))
      return rc;
    std::swap(Pa, Pb);
  }
  const double thr = std::pow(1.0 - rank0_margin(nh), (double)(1 << R0_POW_SQUARINGS));
  r0_pow_decide<<<1, 1024, 0, st>>>(p->dev, Pa, np, nh, thr);
  MLR_LAUNCH_CHECK("r0_pow_decide");
  return kOk;
}

int pcp_rank0(PcpPlan* p, cudaStream_t st) {
  const int nh = p->ch.nh, np = p->ch.np;
  const int64_t smem = rank0_smem_bytes(nh);
  static int max_optin = -1;
  if (max_optin < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  const char* env = getenv("MLR_RANK0_TEST");
  const char* pwe = getenv("MLR_RANK0_POW");
  // measured: the power bound pays where the Cholesky certificate needs the
  // grid version (n_H > 268: C5 eigensolve phase 134.4 -> 124.9 ms); below,
  // the one-CTA register Cholesky is cheaper (C1 17.0 vs 18.7 ms)
  const int use_pow = !(env && env[0] == '0') && (pwe ? pwe[0] == '1' : rank0_smem_bytes(nh) > max_optin);
  if (use_pow) {
    const int rc = r0_power_bound(p, st);
    if (rc) return rc;
  }
  const size_t gscratch = (size_t)nh * nh * sizeof(float);
  const size_t gfree = (size_t)p->gram_splits * np * np * sizeof(double);  // Gram slices: free until post
  const char* genv = getenv("MLR_RANK0_GRID");  // 1: grid version for every n_H, 0: never
  const bool want_grid = genv ? genv[0] == '1' : smem > max_optin;
  if (!(env && env[0] == '0') && want_grid && gscratch <= gfree && nh >= R0G_B) {
    const size_t psm = (size_t)R0G_B * nh * sizeof(float);
    static int sms = -1, per = 0;
    if (sms < 0) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    MLR_CUDA(cudaFuncSetAttribute(pcp_rank0_grid, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm));
    MLR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, pcp_rank0_grid, R0G_T, psm));
    if (per >= 1) {
      PcpDev* dev = p->dev;
      const double* bm = p->Bm;
      int npv = np, nhv = nh;
      float* w = reinterpret_cast<float*>(p->gram_part);
      int up = use_pow;
      void* args[] = {&dev, &bm, &npv, &nhv, &w, &up};
      MLR_CUDA(cudaLaunchCooperativeKernel((void*)pcp_rank0_grid, dim3(sms), dim3(R0G_T), args, psm, st));
      return kOk;
    }
  }
  if (smem > max_optin || (env && env[0] == '0')) {
    pcp_jac_skip_done<<<1, 1, 0, st>>>(p->dev, use_pow);
    MLR_LAUNCH_CHECK("pcp_jac_skip_done");
    return kOk;
  }
  MLR_CUDA(cudaFuncSetAttribute(pcp_rank0_test, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  pcp_rank0_test<<<1, R0_THREADS, smem, st>>>(p->dev, p->Bm, np, nh, use_pow);
  MLR_LAUNCH_CHECK("pcp_rank0_test");
  return kOk;
}

// Coarse SVT from the (all-reduced) Gram in red: B = G^-1 K G^-1; Jacobi
// on X = B V (warm start V); W~ = G^-1 V diag(f) V^T; Z = A W~.
int pcp_svt(PcpPlan* p, const double* red, cudaStream_t st) {
  const int np = p->ch.np;
  const int* skip = &p->dev->done;
  int rc;
  // Warm start: with V the previous eigenvectors and U = G^-1 V,
  //   B~ = V^T (G^-1 K G^-1) V = U^T K U       (M_H = A G^-1, B = M_H^T M_H)
  p->timer.begin(st);
  // n_p^3 products: (n_p/64)^2 output tiles are too few CTAs for small n_p,
  // so K is split (slices in gram_part, free between Gram passes) and the
  // slices summed in a fixed order
  const int ksplit = p->coarse_ksplit;
  auto mm = [&](const double* A, bool ta, const double* Bp, bool tb, double* C, const double* ks,
                const int* klim = nullptr, const int* nlim = nullptr, bool sym = false) {
    GemmSpec g{};
    g.klim = klim;
    g.nlim = nlim;
    g.sym = sym;
    g.M = np; g.N = np; g.K = np;
    g.A = A; g.lda = np; g.a_f32 = false; g.trans_a = ta;
    g.B = Bp; g.ldb = np; g.b_f32 = false; g.trans_b = tb;
    g.C = ksplit > 1 ? p->gram_part : C; g.ldc = np; g.c_f32 = false;
    g.c_slice = ksplit > 1 ? (int64_t)np * np : 0; g.splits = ksplit; g.alpha = 1.0;
    g.kscale = ks; g.skip = skip;
    int rc = gemm_f64(g, st);
    if (rc || ksplit <= 1) return rc;
    return sum_slices(p->gram_part, (int64_t)np * np, (int64_t)np * np, ksplit, C, st, skip);
  };
  // tridiagonal eigensolver (trd.cu): no warm start, B = G^-1 K G^-1 directly
  const bool use_trd = p->trd_on && p->trunc_sv0 == 0;
  if (use_trd) {
    if ((rc = mm(red, false, p->ch.gi, false, p->Xm, nullptr))) return rc;    // X = K G^-1
    // B = G^-1 X, symmetric: upper tiles only, mirrored (large n_p; measured
    // slower at n_p <= 256, where the halved tile count under-fills the GPU)
    if ((rc = mm(p->ch.gi, false, p->Xm, false, p->Bm, nullptr, nullptr, nullptr, np >= 512))) return rc;
  } else {
    if ((rc = mm(p->ch.gi, false, p->Vm, false, p->T1, nullptr))) return rc;   // U = G^-1 V
    if ((rc = mm(red, false, p->T1, false, p->Xm, nullptr))) return rc;        // T = K U
    if ((rc = mm(p->T1, true, p->Xm, false, p->Bm, nullptr))) return rc;       // B~ = U^T T
  }
  p->timer.end(kPhPre, st);
  p->timer.begin(st);
  if ((rc = pcp_rank0(p, st))) return rc;
  if (use_trd &&
      (rc = trd_eig(p->dev, &p->trd, p->Bm, p->Vm, p->ch.nh, np, &p->dev->tau, &p->dev->jac_skip, st)))
    return rc;
  // the Jacobi: the eigensolver (warm started), or on the trd path the
  // fallback for a failed tridiagonal solve (V = I then), skipped otherwise
  if ((rc = jacobi2_eig(false, p->Bm, p->Vm, np, np, p->jac_tol_host, p->jac_floor_rel, p->jac_max_sweeps, p->qbuf,
                        p->qflag, p->jac_off, p->jac_result, use_trd ? &p->dev->eig_skip : &p->dev->jac_skip, st)))
    return rc;
  p->timer.end(kPhJacobi, st);
  p->timer.begin(st);
  pcp_after_jacobi<<<1, 1, 0, st>>>(p->dev, p->jac_result, use_trd ? 1 : 0);
  MLR_LAUNCH_CHECK("pcp_after_jacobi");
  if (p->eig_sort && !use_trd) {
    // sort the eigenpairs (warm start of the next iteration); fw is free until svt_weights
    int* perm = reinterpret_cast<int*>(p->fw);
    const int nh = p->ch.nh;
    eig_sort_kernel<<<1, 1024, sizeof(double) * nh, st>>>(p->dev, p->Bm, np, nh, perm);
    MLR_LAUNCH_CHECK("eig_sort_kernel");
    eig_permute_kernel<<<(int)std::min<int64_t>(ceil_div((int64_t)np * np, 256), 1184), 256, 0, st>>>(
        p->dev, p->Vm, p->T1, np, nh, perm);
    MLR_LAUNCH_CHECK("eig_permute_kernel");
    MLR_CUDA(cudaMemcpyAsync(p->Vm, p->T1, sizeof(double) * np * np, cudaMemcpyDeviceToDevice, st));
  }
  // lambda_i = diag(B~) after convergence; f_i = (sigma_i - tau)+ / sigma_i
  if (p->trunc_sv0 > 0) {
    svt_weights_trunc_kernel<<<1, 1024, 0, st>>>(p->dev, np, p->ch.nh, p->Bm, p->sig, p->fw);
    MLR_LAUNCH_CHECK("svt_weights_trunc_kernel");
  } else if ((rc = svt_weights(skip, np, p->ch.nh, false, p->Bm, &p->dev->tau, p->sig, p->fw, &p->dev->rank,
                               &p->dev->nuclear, st))) {
    return rc;
  }
  // W~ = G^-1 V diag(f) V^T = U' diag(f) V^T with U' = G^-1 V.  A certified
  // rank-0 iteration has W~ = 0 and Z = 0: the products are skipped
  // (jac_skip) and Z is cleared instead.
  skip = &p->dev->jac_skip;
  const bool tc = p->tc_recon && p->m_local > 0;
  // tridiagonal path: V has k = info[0] nonzero columns, so U' = G^-1 V is
  // needed only in its first k columns and the products below sum over k
  const int* kl = use_trd ? p->trd.info + 2 : nullptr;
  if ((rc = mm(p->ch.gi, false, p->Vm, false, p->T1, nullptr, nullptr, kl))) return rc;
  if (tc) {
    // W~^T = V diag(f) U'^T (the tcgen05 B operand is K-major), then its TF32 hi / lo parts
    if ((rc = mm(p->Vm, false, p->T1, true, p->Wm, p->fw, kl))) return rc;
    if ((rc = tc_split_w(p->Wm, p->w_hi, p->w_lo, np, skip, st))) return rc;
  } else if ((rc = mm(p->T1, false, p->Vm, true, p->Wm, p->fw, kl))) {
    return rc;
  }
  p->timer.end(kPhPost, st);
  // Z = A W~
  p->timer.begin(st);
  if (tc) {
    if ((rc = tc_recon_run(&p->tc, (float*)p->Z, np, skip, st))) return rc;
    const int64_t zn = p->m_local * np;
    pcp_zero_if_rank0<<<(int)std::min<int64_t>(ceil_div(zn, 1024), 1184), 256, 0, st>>>(
        p->dev, reinterpret_cast<uint32_t*>(p->Z), zn);
    MLR_LAUNCH_CHECK("pcp_zero_if_rank0");
  } else if (p->m_local > 0) {
    GemmSpec z{};
    z.M = (int)p->m_local; z.N = np; z.K = np;
    z.A = p->A; z.lda = np; z.a_f32 = p->f32; z.trans_a = false;
    z.B = p->Wm; z.ldb = np; z.b_f32 = false; z.trans_b = false;
    z.C = p->Z; z.ldc = np; z.c_f32 = p->f32; z.c_slice = 0; z.splits = 1; z.alpha = 1.0;
    z.kscale = nullptr; z.skip = skip;
    if ((rc = gemm_f64(z, st))) return rc;
    const int64_t zn = p->m_local * np * (p->f32 ? 1 : 2);  // Z as 32-bit words
    pcp_zero_if_rank0<<<(int)std::min<int64_t>(ceil_div(zn, 1024), 1184), 256, 0, st>>>(
        p->dev, reinterpret_cast<uint32_t*>(p->Z), zn);
    MLR_LAUNCH_CHECK("pcp_zero_if_rank0");
  }
  p->timer.end(kPhRecon, st);
  return kOk;
}

int pcp_update(PcpPlan* p, const void* D, int64_t ldd, const void* Yin, void* Yout, int64_t ldy, cudaStream_t st) {
  p->timer.begin(st);
  const int rc = p->f32 ? row_pass<float>(kUpdate, p, D, ldd, Yin, Yout, ldy, nullptr, nullptr, 0, st)
                : row_pass<double>(kUpdate, p, D, ldd, Yin, Yout, ldy, nullptr, nullptr, 0, st);
  p->timer.end(kPhUpdate, st);
  return rc;
}

// Final L = Z R^T and S = shrink(D - L + Y_{k-1}/mu_k, lam/mu_k).
__global__ void pcp_output_mu(PcpDev* st) { st->mu = st->mu_last; }
__global__ void pcp_output_mu_restore(PcpDev* st) { st->mu = st->mu_final; }

int pcp_outputs(PcpPlan* p, const void* D, int64_t ldd, const void* Yprev, int64_t ldy, void* L, void* S, int64_t ldo,
                cudaStream_t st) {
  pcp_output_mu<<<1, 1, 0, st>>>(p->dev);
  int rc = p->f32 ? row_pass<float>(kOutput, p, D, ldd, Yprev, nullptr, ldy, L, S, ldo, st)
                  : row_pass<double>(kOutput, p, D, ldd, Yprev, nullptr, ldy, L, S, ldo, st);
  if (rc) return rc;
  pcp_output_mu_restore<<<1, 1, 0, st>>>(p->dev);
  MLR_LAUNCH_CHECK("pcp_output_mu");
  return kOk;
}

}  // namespace mlr
