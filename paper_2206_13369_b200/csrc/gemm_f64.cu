// FP64-accumulating GEMMs for the coarse level (Gram, reconstruction, small
// n_H x n_H products) on the DMMA tensor path (mma.sync m8n8k4 .f64).
//
// C[M x N] = op(A)[M x K] * op(B)[K x N], row-major storage, inputs float or
// double (converted to double when staged into shared memory), output float
// or double.  gridDim.z > 1 splits K; slice z writes C + z * c_slice and a
// separate deterministic reduction sums the slices.
//
// Replaces the reference's numpy GEMMs / LAPACK calls:
//   Gram K = A^T A          (stands in for gesdd inside svd_full, linalg.py:86-99)
//   Z = A * W               (reconstruction, pcp.py:259-266)
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace mlr {

constexpr int GBM = 64, GBN = 64, GBK = 16, GPAD = 8;
constexpr int GTHREADS = 128;  // 4 warps, 2x2, each 32x32

__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

template <typename TA, typename TB, typename TC, bool TRANS_A, bool TRANS_B>
__global__ void __launch_bounds__(GTHREADS)
gemm_f64_kernel(int M, int N, int K, const TA* __restrict__ A, int64_t lda,
                const TB* __restrict__ B, int64_t ldb, TC* __restrict__ C, int64_t ldc,
                int64_t c_slice, int k_chunk, double alpha, const double* __restrict__ kscale,
                const int* __restrict__ skip, int sym_tiles, const int* __restrict__ klim,
                const int* __restrict__ nlim) {
  if (skip && *skip) return;
  __shared__ double As[2][GBK][GBM + GPAD];
  __shared__ double Bs[2][GBK][GBN + GPAD];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  int bm = blockIdx.y, bn = blockIdx.x;
  if (sym_tiles > 0) {  // blockIdx.x enumerates the tiles bm <= bn of a symmetric result
    int t = blockIdx.x;
    bm = 0;
    while (t >= sym_tiles - bm) {
      t -= sym_tiles - bm;
      ++bm;
    }
    bn = bm + t;
  }
  const int m0 = bm * GBM, n0 = bn * GBN;
  if (nlim && n0 >= *nlim) return;  // columns >= *nlim of C are not wanted (uniform per CTA)
  const int kb = blockIdx.z * k_chunk;
  const int ke = min(klim ? min(K, *klim) : K, kb + k_chunk);
  C += (int64_t)blockIdx.z * c_slice;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // Each thread stages 8 elements of A and 8 of B per K-tile (64x16 = 1024).
  double ra[8], rb[8];
  auto load_tile = [&](int k0) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      int idx = tid + e * GTHREADS;  // 0..1023
      int kk, mm;
      if (TRANS_A) {  // A stored K x M: coalesce along m
        kk = idx >> 6; mm = idx & 63;
      } else {        // A stored M x K: coalesce along k
        mm = idx >> 4; kk = idx & 15;
      }
      int gk = k0 + kk, gm = m0 + mm;
      double v = 0.0;
      if (gk < ke && gm < M) {
        v = TRANS_A ? (double)A[(int64_t)gk * lda + gm] : (double)A[(int64_t)gm * lda + gk];
        if (kscale) v *= kscale[gk];
      }
      ra[e] = v;
      int nn;
      if (TRANS_B) { nn = idx >> 4; kk = idx & 15; }   // B stored N x K
      else { kk = idx >> 6; nn = idx & 63; }           // B stored K x N
      gk = k0 + kk;
      int gn = n0 + nn;
      double w = 0.0;
      if (gk < ke && gn < N) w = TRANS_B ? (double)B[(int64_t)gn * ldb + gk] : (double)B[(int64_t)gk * ldb + gn];
      rb[e] = w;
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      int idx = tid + e * GTHREADS;
      int kk, mm, nn;
      if (TRANS_A) { kk = idx >> 6; mm = idx & 63; } else { mm = idx >> 4; kk = idx & 15; }
      As[buf][kk][mm] = ra[e];
      if (TRANS_B) { nn = idx >> 4; kk = idx & 15; } else { kk = idx >> 6; nn = idx & 63; }
      Bs[buf][kk][nn] = rb[e];
    }
  };

  int ntiles = (ke - kb + GBK - 1) / GBK;
  if (ntiles <= 0) ntiles = 0;
  if (ntiles > 0) {
    load_tile(kb);
    store_tile(0);
  }
  __syncthreads();
  for (int t = 0; t < ntiles; ++t) {
    const int buf = t & 1;
    if (t + 1 < ntiles) load_tile(kb + (t + 1) * GBK);
#pragma unroll
    for (int k4 = 0; k4 < GBK; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[buf][k4 + (lane & 3)][wm + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs[buf][k4 + (lane & 3)][wn + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if (t + 1 < ntiles) store_tile(buf ^ 1);
    __syncthreads();
  }
  // epilogue
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int gm = m0 + wm + i * 8 + (lane >> 2);
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int gn = n0 + wn + j * 8 + (lane & 3) * 2;
      if (gn < N) C[(int64_t)gm * ldc + gn] = (TC)(alpha * acc[i][j][0]);
      if (gn + 1 < N) C[(int64_t)gm * ldc + gn + 1] = (TC)(alpha * acc[i][j][1]);
      if (sym_tiles > 0 && bm != bn) {  // mirror into the lower triangle
        if (gn < N) C[(int64_t)gn * ldc + gm] = (TC)(alpha * acc[i][j][0]);
        if (gn + 1 < N) C[(int64_t)(gn + 1) * ldc + gm] = (TC)(alpha * acc[i][j][1]);
      }
    }
  }
}

// Tall-skinny Gram C = X^T X (X: K x N row-major, N % 128 == 0) on the FP64
// DMMA path, for the coarse Grams of both solvers (K_H = A^T A, K_g = g_H^T g_H).
// CTA = one 128 x 128 block (bm <= bn) of C over a K slice, one launch for
// all blocks; warp = one 32 x 32 subtile (diagonal blocks: the 10 upper
// subtiles, the other 6 warps only help stage the tiles).  X tiles of KT rows stream through a 3-stage
// cp.async ring in their storage type and are widened to FP64 when the MMA
// fragments are read.  Each slice z writes the full square (subtiles and
// their mirrors) at C + z * c_slice; sum_slices adds the slices in a fixed order.
constexpr int GR_STAGES = 3;
template <typename T>
struct GramCfg {
  static constexpr int KT = sizeof(T) == 4 ? 32 : 16;  // rows per stage
  static constexpr int LD = 128 + (sizeof(T) == 4 ? 8 : 4);  // padded row (conflict-free fragment reads)
  static constexpr size_t STAGE = (size_t)KT * LD * sizeof(T);
};

__device__ __forceinline__ void gr_cp16(void* smem, const void* gmem, int bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gmem), "r"(bytes) : "memory");
}

template <typename T>
__global__ void __launch_bounds__(512)
gram128_kernel(int N, int K, const T* __restrict__ X, int64_t ldx, double* __restrict__ C, int64_t ldc,
               int64_t c_slice, int k_chunk, const int* __restrict__ skip, int nb) {
  if (skip && *skip) return;
  using G = GramCfg<T>;
  constexpr int KT = G::KT, LD = G::LD, NT = 512;
  constexpr int V = 16 / sizeof(T);  // elements per 16-byte copy
  extern __shared__ __align__(16) unsigned char gr_smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // block (bm, bn), bm <= bn, enumerated row by row
  int bm = 0, bn;
  {
    int t = blockIdx.x;
    while (t >= nb - bm) {
      t -= nb - bm;
      ++bm;
    }
    bn = bm + t;
  }
  const bool DIAG = bm == bn;
  T* sa = reinterpret_cast<T*>(gr_smem);                               // [stages][KT][LD] block bm
  T* sb = DIAG ? sa : sa + (size_t)GR_STAGES * KT * LD;                 // block bn
  // warp subtile: all 16 off the diagonal, the 10 upper ones on it
  int wi = warp >> 2, wj = warp & 3;
  bool work = true;
  if (DIAG) {
    int t = warp;
    wi = 0;
    while (wi < 4 && t >= 4 - wi) {
      t -= 4 - wi;
      ++wi;
    }
    wj = wi + t;
    work = warp < 10;
  }
  const int kb = blockIdx.y * k_chunk, ke = min(K, kb + k_chunk);
  const int ntiles = ke > kb ? (ke - kb + KT - 1) / KT : 0;
  C += (int64_t)blockIdx.y * c_slice;
  const T* xa = X + (int64_t)bm * 128;
  const T* xb = X + (int64_t)bn * 128;
  constexpr int CPR = 128 / V;  // 16-byte copies per row
  auto issue = [&](int t) {
    if (t < ntiles) {
      const int r0 = kb + t * KT, st = t % GR_STAGES;
      for (int e = tid; e < KT * CPR; e += NT) {
        const int r = e / CPR, c = (e % CPR) * V;
        const bool in = r0 + r < ke;
        const int64_t off = (int64_t)(in ? r0 + r : kb) * ldx + c;
        gr_cp16(sa + ((size_t)st * KT + r) * LD + c, xa + off, in ? 16 : 0);
        if (!DIAG) gr_cp16(sb + ((size_t)st * KT + r) * LD + c, xb + off, in ? 16 : 0);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int q = 0; q < GR_STAGES - 1; ++q) issue(q);
  const int ma = wi * 32 + (lane >> 2), nb0 = wj * 32 + (lane >> 2), kk = lane & 3;
  for (int t = 0; t < ntiles; ++t) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(GR_STAGES - 2) : "memory");
    __syncthreads();       // stage t visible; stage t - 1 fully consumed
    issue(t + GR_STAGES - 1);
    const T* A = sa + (size_t)(t % GR_STAGES) * KT * LD;
    const T* B = sb + (size_t)(t % GR_STAGES) * KT * LD;
    if (!work) continue;
#pragma unroll
    for (int k4 = 0; k4 < KT; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = (double)A[(k4 + kk) * LD + ma + 8 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = (double)B[(k4 + kk) * LD + nb0 + 8 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  if (!work) return;
  // epilogue: subtile and (off the diagonal) its mirror
  const bool mirror = bm != bn || wi != wj;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = bm * 128 + wi * 32 + i * 8 + (lane >> 2);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = bn * 128 + wj * 32 + j * 8 + (lane & 3) * 2;
      *reinterpret_cast<double2*>(C + (int64_t)gm * ldc + gn) = make_double2(acc[i][j][0], acc[i][j][1]);
      if (mirror) {
        C[(int64_t)gn * ldc + gm] = acc[i][j][0];
        C[(int64_t)(gn + 1) * ldc + gm] = acc[i][j][1];
      }
    }
  }
  (void)N;
}

bool gram128_ok(int n) {
  const char* e = getenv("MLR_GRAM128");
  return n % 128 == 0 && !(e && e[0] == '0');
}

template <typename T>
static int gram128_launch(const GemmSpec& g, cudaStream_t st) {
  using G = GramCfg<T>;
  const int nb = g.N / 128;
  const int chunk = (int)round_up(ceil_div(g.K, g.splits), G::KT);
  const size_t smem = (nb > 1 ? 2 : 1) * GR_STAGES * G::STAGE;
  MLR_CUDA(cudaFuncSetAttribute(gram128_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  gram128_kernel<T><<<dim3(nb * (nb + 1) / 2, g.splits), 512, smem, st>>>(
      g.N, g.K, (const T*)g.A, g.lda, (double*)g.C, g.ldc, g.c_slice, chunk, g.skip, nb);
  MLR_LAUNCH_CHECK("gram128_kernel");
  return kOk;
}

// Deterministic sum of `slices` partial matrices (contiguous, stride `slice`).
__global__ void sum_slices_kernel(const double* __restrict__ P, int64_t count, int64_t slice,
                                  int slices, double* __restrict__ out, const int* __restrict__ skip) {
  if (skip && *skip) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    // fixed summation order; loads batched 8 deep so the chain is not
    // one L2 round trip per slice
    double s = 0.0;
    int z = 0;
    for (; z + 8 <= slices; z += 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = P[(int64_t)(z + q) * slice + i];
#pragma unroll
      for (int q = 0; q < 8; ++q) s += v[q];
    }
    for (; z < slices; ++z) s += P[(int64_t)z * slice + i];
    out[i] = s;
  }
}

template <typename TA, typename TB, typename TC, bool TA_, bool TB_>
static int launch(int M, int N, int K, const void* A, int64_t lda, const void* B, int64_t ldb,
                  void* C, int64_t ldc, int64_t c_slice, int splits, double alpha, const double* kscale,
                  const int* skip, bool sym, const int* klim, const int* nlim, cudaStream_t st) {
  const int tn = (N + GBN - 1) / GBN, tm = (M + GBM - 1) / GBM;
  const int sym_tiles = (sym && M == N) ? tn : 0;
  dim3 grid(sym_tiles ? tn * (tn + 1) / 2 : tn, sym_tiles ? 1 : tm, splits);
  int chunk = (int)round_up(ceil_div(K, splits), GBK);
  gemm_f64_kernel<TA, TB, TC, TA_, TB_><<<grid, GTHREADS, 0, st>>>(
      M, N, K, (const TA*)A, lda, (const TB*)B, ldb, (TC*)C, ldc, c_slice, chunk, alpha, kscale, skip, sym_tiles,
      klim, nlim);
  MLR_LAUNCH_CHECK("gemm_f64_kernel");
  return kOk;
}

int gemm_f64(GemmSpec g, cudaStream_t st) {
  // symmetric Gram X^T X with 128-multiple width: the blocked DMMA Gram
  if (g.sym && g.trans_a && !g.trans_b && g.A == g.B && g.lda == g.ldb && g.a_f32 == g.b_f32 && g.M == g.N &&
      !g.c_f32 && g.alpha == 1.0 && !g.kscale && gram128_ok(g.N) && g.lda % 4 == 0 && g.ldc % 2 == 0)
    return g.a_f32 ? gram128_launch<float>(g, st) : gram128_launch<double>(g, st);
  // dispatch on (A type, B type, C type, transA, transB)
#define MLR_G(TA, TB, TC, XA, XB)                                                              \
  if (g.a_f32 == std::is_same<TA, float>::value && g.b_f32 == std::is_same<TB, float>::value && \
      g.c_f32 == std::is_same<TC, float>::value && g.trans_a == XA && g.trans_b == XB)            \
    return launch<TA, TB, TC, XA, XB>(g.M, g.N, g.K, g.A, g.lda, g.B, g.ldb, g.C, g.ldc,         \
                                      g.c_slice, g.splits, g.alpha, g.kscale, g.skip, g.sym, g.klim, g.nlim, st);
#define MLR_G_TYPES(XA, XB)                 \
  MLR_G(float, float, float, XA, XB)        \
  MLR_G(float, float, double, XA, XB)       \
  MLR_G(float, double, float, XA, XB)       \
  MLR_G(float, double, double, XA, XB)      \
  MLR_G(double, float, float, XA, XB)       \
  MLR_G(double, float, double, XA, XB)      \
  MLR_G(double, double, float, XA, XB)      \
  MLR_G(double, double, double, XA, XB)
  MLR_G_TYPES(false, false)
  MLR_G_TYPES(true, false)
  MLR_G_TYPES(false, true)
#undef MLR_G_TYPES
#undef MLR_G
  set_error("gemm_f64: unsupported type/transpose combination");
  return kErrArg;
}

int sum_slices(const double* P, int64_t count, int64_t slice, int slices, double* out,
               cudaStream_t st, const int* skip) {
  int blocks = (int)std::min<int64_t>(ceil_div(count, 256), 148 * 8);
  if (blocks < 1) blocks = 1;
  sum_slices_kernel<<<blocks, 256, 0, st>>>(P, count, slice, slices, out, skip);
  MLR_LAUNCH_CHECK("sum_slices_kernel");
  return kOk;
}

}  // namespace mlr
