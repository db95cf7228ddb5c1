// Warp-per-row streaming kernels: the fine-level hot path of both solvers.
//
// One warp owns one fine row at a time and streams it in chunks of
// CH = 32 lanes x 16 bytes (128 floats / 64 doubles): D / Y / S and the
// stencil (c0, w0, w1) move as 16-byte vectors and a row needs only
// __syncwarp.  The restriction x_H[k] = sum_j x_j R[j, k] never stages the
// fine row: fine j contributes w0_j x_j to key c0_j and w1_j x_j to key
// c0_j + 1, and c0 is non-decreasing, so both sums are segmented reductions
// over runs of equal c0.  They are formed in registers (in-lane scan, then a
// 5-step shuffle scan across the warp, carried across chunks) and folded
// into a per-warp ring of 2*CH coarse keys in shared memory, each key being
// written to HBM once its run has ended.  Deterministic (fixed order, no
// atomics), no bank-conflicted gathers, ~2 KB of shared memory per warp.
// Requires ChainDev::keys_dense (c0 takes every value 0..nh-2).
//
//   pcp_rows_warp<T, MODE> : ML-PCP  start (Y0, A1) / update / output passes
//                            (pcp.py:252-282, 112-115)
//   cp_rows_warp<T, MODE>  : ML-CPCP init / update / output passes
//                            (cpcp.py:352-354, 399-427)
//   cp_dots_warp<T>        : ML-CPCP segment-QP dots from coarse data (cpcp.py:387-395)
#include <climits>

#include "common.cuh"
#include "cpcp.h"
#include "kernels.h"
#include "pcp.h"
#include "rows.h"

namespace mlr {

constexpr int RW_THREADS = 256, RW_WARPS = RW_THREADS / 32;
constexpr unsigned kFull = 0xffffffffu;

template <typename T>
struct Vec;
template <>
struct Vec<float> {
  using V = float4;
  using I = int4;
  static constexpr int N = 4;
  static __device__ __forceinline__ void unpack(const V& v, float (&o)[4]) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
  static __device__ __forceinline__ V pack(const float (&o)[4]) { return make_float4(o[0], o[1], o[2], o[3]); }
  static __device__ __forceinline__ void unpacki(const I& v, int (&o)[4]) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
};
template <>
struct Vec<double> {
  using V = double2;
  using I = int2;
  static constexpr int N = 2;
  static __device__ __forceinline__ void unpack(const V& v, double (&o)[2]) { o[0] = v.x; o[1] = v.y; }
  static __device__ __forceinline__ V pack(const double (&o)[2]) { return make_double2(o[0], o[1]); }
  static __device__ __forceinline__ void unpacki(const I& v, int (&o)[2]) { o[0] = v.x; o[1] = v.y; }
};

template <typename T>
__device__ __forceinline__ const T* stencil_w0(const ChainDev& ch) {
  if constexpr (std::is_same<T, float>::value) return ch.w0f; else return ch.w0;
}
template <typename T>
__device__ __forceinline__ const T* stencil_w1(const ChainDev& ch) {
  if constexpr (std::is_same<T, float>::value) return ch.w1f; else return ch.w1;
}

// Load NV consecutive values starting at j (vectorised when the whole vector
// is in range and aligned), zero past n.
template <typename T, int NV>
__device__ __forceinline__ void load_vec(const T* __restrict__ p, int j, int n, bool vec, T (&o)[NV]) {
  using VT = Vec<T>;
  if (vec && j + NV <= n) {
    VT::unpack(__ldg(reinterpret_cast<const typename VT::V*>(p + j)), o);
  } else {
#pragma unroll
    for (int e = 0; e < NV; ++e) o[e] = j + e < n ? p[j + e] : T(0);
  }
}
template <typename T, int NV>
__device__ __forceinline__ void load_vec_rw(const T* p, int j, int n, bool vec, T (&o)[NV]) {
  using VT = Vec<T>;
  if (vec && j + NV <= n) {
    VT::unpack(*reinterpret_cast<const typename VT::V*>(p + j), o);
  } else {
#pragma unroll
    for (int e = 0; e < NV; ++e) o[e] = j + e < n ? p[j + e] : T(0);
  }
}
template <typename T, int NV>
__device__ __forceinline__ void store_vec(T* p, int j, int n, bool vec, const T (&o)[NV]) {
  using VT = Vec<T>;
  if (vec && j + NV <= n) {
    *reinterpret_cast<typename VT::V*>(p + j) = VT::pack(o);
  } else {
#pragma unroll
    for (int e = 0; e < NV; ++e)
      if (j + e < n) p[j + e] = o[e];
  }
}

// Stencil of NV consecutive fine columns; key = INT_MAX past n.
template <typename T, int NV>
struct StencilVec {
  int key[NV];
  T w0[NV], w1[NV];
  __device__ __forceinline__ void load(const ChainDev& ch, int j) {
    using VT = Vec<T>;
    const int n = ch.n;
    if (j + NV <= n) {
      VT::unpacki(__ldg(reinterpret_cast<const typename VT::I*>(ch.c0 + j)), key);
      VT::unpack(__ldg(reinterpret_cast<const typename VT::V*>(stencil_w0<T>(ch) + j)), w0);
      VT::unpack(__ldg(reinterpret_cast<const typename VT::V*>(stencil_w1<T>(ch) + j)), w1);
    } else {
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        const bool in = j + e < n;
        key[e] = in ? __ldg(ch.c0 + j + e) : INT_MAX;
        w0[e] = in ? __ldg(stencil_w0<T>(ch) + j + e) : T(0);
        w1[e] = in ? __ldg(stencil_w1<T>(ch) + j + e) : T(0);
      }
    }
  }
};

// Streaming restriction of NB fine quantities x (one row) onto coarse keys.
// Call chunk() once per chunk with every lane's NV values, then finish().
template <typename T, int NB, int NV>
struct SegRestrict {
  static constexpr int RK = 64 * NV;  // key ring (2 * CH)
  T* acc;                             // NB * RK, zero on entry and exit
  int carry_key, kflush;
  T carry0[NB], carry1[NB];

  __device__ __forceinline__ void begin(T* ring) {
    acc = ring;
    carry_key = INT_MAX - 1;
    kflush = -1;
#pragma unroll
    for (int b = 0; b < NB; ++b) carry0[b] = carry1[b] = T(0);
  }

  // next_key: c0 of the first fine column after this chunk (INT_MAX at the row end).
  __device__ __forceinline__ void chunk(const StencilVec<T, NV>& sv, const T (&x)[NB][NV], int next_key,
                                        T* const (&out)[NB], int nh, int lane) {
    const int(&key)[NV] = sv.key;
    T t0[NB][NV], t1[NB][NV];
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        t0[b][e] = sv.w0[e] * x[b][e];
        t1[b][e] = sv.w1[e] * x[b][e];
      }
    // in-lane segmented inclusive scan
#pragma unroll
    for (int e = 1; e < NV; ++e)
      if (key[e] == key[e - 1])
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          t0[b][e] += t0[b][e - 1];
          t1[b][e] += t1[b][e - 1];
        }
    // warp segmented inclusive scan of the lane tails (keys are monotone, so
    // equal tail keys imply every lane in between is one run)
    const int kt = key[NV - 1];
    T s0[NB], s1[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      s0[b] = t0[b][NV - 1];
      s1[b] = t1[b][NV - 1];
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int kk = __shfl_up_sync(kFull, kt, o);
      const bool take = lane >= o && kk == kt;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const T a = __shfl_up_sync(kFull, s0[b], o);
        const T c = __shfl_up_sync(kFull, s1[b], o);
        if (take) {
          s0[b] += a;
          s1[b] += c;
        }
      }
    }
    if (kt == carry_key)
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        s0[b] += carry0[b];
        s1[b] += carry1[b];
      }
    // exclusive prefix for the lane's head run
    int kp = __shfl_up_sync(kFull, kt, 1);
    T p0[NB], p1[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      p0[b] = __shfl_up_sync(kFull, s0[b], 1);
      p1[b] = __shfl_up_sync(kFull, s1[b], 1);
    }
    if (lane == 0) {
      kp = carry_key;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        p0[b] = carry0[b];
        p1[b] = carry1[b];
      }
    }
    if (kp == key[0])
#pragma unroll
      for (int e = 0; e < NV; ++e)
        if (key[e] == key[0])
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            t0[b][e] += p0[b];
            t1[b][e] += p1[b];
          }
    // run ends
    int knext = __shfl_down_sync(kFull, key[0], 1);
    if (lane == 31) knext = next_key;
    bool end[NV];
    int kmax = -1;
#pragma unroll
    for (int e = 0; e < NV; ++e) {
      const int nk = e < NV - 1 ? key[e + 1] : knext;
      end[e] = key[e] != INT_MAX && nk != key[e];
      if (end[e]) kmax = key[e];
    }
    carry_key = __shfl_sync(kFull, kt, 31);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      carry0[b] = __shfl_sync(kFull, s0[b], 31);
      carry1[b] = __shfl_sync(kFull, s1[b], 31);
    }
    // fold: w0 runs into their key, then w1 runs into key + 1, then flush
#pragma unroll
    for (int e = 0; e < NV; ++e)
      if (end[e])
#pragma unroll
        for (int b = 0; b < NB; ++b) acc[b * RK + key[e] % RK] += t0[b][e];
    __syncwarp();
#pragma unroll
    for (int e = 0; e < NV; ++e)
      if (end[e] && key[e] + 1 < nh)
#pragma unroll
        for (int b = 0; b < NB; ++b) acc[b * RK + (key[e] + 1) % RK] += t1[b][e];
    __syncwarp();
#pragma unroll
    for (int e = 0; e < NV; ++e)
      if (end[e])
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          T* slot = acc + b * RK + key[e] % RK;
          out[b][key[e]] = *slot;
          *slot = T(0);
        }
    kflush = max(kflush, __reduce_max_sync(kFull, kmax));
    __syncwarp();
  }

  // Flush the keys after the last w0 run (they hold w1 runs only) and zero
  // the padded tail [nh, np).
  __device__ __forceinline__ void finish(T* const (&out)[NB], int nh, int np, int lane) {
    for (int k = kflush + 1 + lane; k < np; k += 32)
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        if (k < nh) {
          T* slot = acc + b * RK + k % RK;
          out[b][k] = *slot;
          *slot = T(0);
        } else {
          out[b][k] = T(0);
        }
      }
    __syncwarp();
  }
};

// -------------------------------------------------------------------- ML-PCP
enum RowModeW { kWStart = 0, kWUpdate = 1, kWOutput = 2 };

template <typename T, int MODE>
__global__ void __launch_bounds__(RW_THREADS)
pcp_rows_warp(const PcpDev* __restrict__ st, ChainDev ch, int64_t m, const T* __restrict__ D, int64_t ldd,
              const T* __restrict__ Yin, T* __restrict__ Yout, int64_t ldy, const T* __restrict__ Z,
              T* __restrict__ A, T* __restrict__ Lout, T* __restrict__ Sout, int64_t ldo, double* __restrict__ part) {
  if (MODE == kWUpdate && st->done) return;
  using SR = SegRestrict<T, 1, Vec<T>::N>;
  constexpr int NV = Vec<T>::N, CH = 32 * NV;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = ch.n, nh = ch.nh, np = ch.np;
  const int zlen = round_up_dev(np + 2, 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* zrow = reinterpret_cast<T*>(smem_raw) + warp * (zlen + SR::RK);
  T* ring = zrow + zlen;
  for (int k = lane; k < SR::RK; k += 32) ring[k] = T(0);
  __syncwarp();

  const double mu_d = st->mu;
  const T inv = (T)(1.0 / mu_d);
  const T mu = (T)mu_d;
  const T thr = (T)(st->lam * (1.0 / mu_d));
  const T inv_next = (T)(1.0 / (mu_d * st->rho));
  const double scale = st->scale;
  double acc_res = 0.0, acc_l1 = 0.0, acc_nnz = 0.0;
  const bool vec = (ldd % NV == 0) && (ldy % NV == 0) && (MODE != kWOutput || ldo % NV == 0);
  SR sr;

  for (int64_t i = (int64_t)blockIdx.x * RW_WARPS + warp; i < m; i += (int64_t)gridDim.x * RW_WARPS) {
    if (MODE != kWStart) {
      for (int k = lane; k < zlen; k += 32) zrow[k] = k < np ? Z[i * np + k] : T(0);
      __syncwarp();
    }
    const T* drow = D + i * ldd;
    sr.begin(ring);
    T* const outp[1] = {A + i * np};
    for (int cbase = 0; cbase < n; cbase += CH) {
      const int j = cbase + lane * NV;
      StencilVec<T, NV> sv;
      sv.load(ch, j);
      T dv[NV], yv[NV];
      load_vec<T, NV>(drow, j, n, vec, dv);
      if (MODE != kWStart) load_vec<T, NV>(Yin + i * ldy, j, n, vec, yv);
      T x[1][NV], yo[NV], lo_v[NV], so_v[NV];
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        const T d = dv[e];
        if (MODE == kWStart) {
          // y = d / scale (pcp.py:115); work = y/mu + d (pcp.py:252-254, S = 0)
          const T y = (T)((double)d / scale);
          yo[e] = y;
          x[0][e] = y * inv + d;
        } else {
          const int c = min(sv.key[e], np);
          const T l = sv.w0[e] * zrow[c] + sv.w1[e] * zrow[c + 1];
          const T y = yv[e];
          const T w = y * inv + d - l;
          const T s = soft_thr<T>(w, thr);
          lo_v[e] = l;
          so_v[e] = s;
          if (MODE == kWUpdate) {
            const T res = (d - l) - s;
            const T yn = y + res * mu;
            yo[e] = yn;
            if (j + e < n) {
              acc_res = fma((double)res, (double)res, acc_res);
              acc_l1 += fabs((double)s);
              acc_nnz += s != T(0) ? 1.0 : 0.0;
            }
            x[0][e] = yn * inv_next + d - s;
          }
        }
      }
      if (MODE == kWOutput) {
        store_vec<T, NV>(Lout + i * ldo, j, n, vec, lo_v);
        store_vec<T, NV>(Sout + i * ldo, j, n, vec, so_v);
        continue;
      }
      store_vec<T, NV>(Yout + i * ldy, j, n, vec, yo);
      sr.chunk(sv, x, cbase + CH < n ? __ldg(ch.c0 + cbase + CH) : INT_MAX, outp, nh, lane);
    }
    if (MODE != kWOutput) sr.finish(outp, nh, np, lane);
    __syncwarp();
  }
  if (MODE == kWUpdate) {
    __shared__ double scratch[3 * 32];
    double v[3] = {acc_res, acc_l1, acc_nnz};
    block_sum<3>(v, scratch);
    if (threadIdx.x == 0) {
      part[3 * blockIdx.x + 0] = v[0];
      part[3 * blockIdx.x + 1] = v[1];
      part[3 * blockIdx.x + 2] = v[2];
    }
  }
}

bool rows_warp_ok(const ChainDev& ch, bool) { return ch.keys_dense != 0; }

int pcp_rows(PcpPlan* p, int mode, const void* D, int64_t ldd, const void* Yin, void* Yout, int64_t ldy, void* Lout,
             void* Sout, int64_t ldo, cudaStream_t st) {
  const size_t tb = p->f32 ? 4 : 8;
  const int nv = p->f32 ? 4 : 2;
  const size_t smem = RW_WARPS * ((size_t)round_up(p->ch.np + 2, 4) + 64 * nv) * tb;
  const int blocks = p->row_blocks;
#define MLR_LAUNCH(T, MODE)                                                                                     \
  {                                                                                                             \
    auto kern = pcp_rows_warp<T, MODE>;                                                                         \
    MLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));               \
    kern<<<blocks, RW_THREADS, smem, st>>>(p->dev, p->ch, p->m_local, (const T*)D, ldd, (const T*)Yin, (T*)Yout, \
                                           ldy, (const T*)p->Z, (T*)p->A, (T*)Lout, (T*)Sout, ldo, p->row_part); \
  }
  if (p->f32) {
    if (mode == kWStart) MLR_LAUNCH(float, kWStart) else if (mode == kWUpdate) MLR_LAUNCH(float, kWUpdate) else MLR_LAUNCH(float, kWOutput)
  } else {
    if (mode == kWStart) MLR_LAUNCH(double, kWStart) else if (mode == kWUpdate) MLR_LAUNCH(double, kWUpdate) else MLR_LAUNCH(double, kWOutput)
  }
#undef MLR_LAUNCH
  MLR_LAUNCH_CHECK("pcp_rows_warp");
  return kOk;
}

// -------------------------------------------------------------------- ML-CPCP
struct AmRecW {
  double mag, val, sval;
  long long idx;
};
__device__ __forceinline__ void am_merge_w(AmRecW& a, const AmRecW& b) {
  if (argmax_better(b.mag, b.idx, a.mag, a.idx)) a = b;
}

enum CpModeW { kCWInit = 0, kCWUpdate = 1, kCWOutput = 2 };

template <typename T, int MODE>
__global__ void __launch_bounds__(RW_THREADS)
cp_rows_warp(const CpcpDev* __restrict__ st, ChainDev ch, int64_t m, int64_t row0, int64_t m_global,
             const T* __restrict__ D, int64_t ldd, const uint32_t* __restrict__ mask, int64_t ldm, T* __restrict__ S,
             int64_t lds, T* __restrict__ LH, T* __restrict__ GH, T* __restrict__ SH, const double* __restrict__ u,
             const double* __restrict__ vg, T* __restrict__ Lout, int64_t ldl, double* __restrict__ part) {
  if (MODE == kCWUpdate && st->done) return;
  using SR = SegRestrict<T, 2, Vec<T>::N>;
  constexpr int NV = Vec<T>::N, CH = 32 * NV;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = ch.n, nh = ch.nh, np = ch.np;
  const int zlen = round_up_dev(np + 2, 4);
  double* vs = reinterpret_cast<double*>(smem_raw);  // v (np), CTA-shared
  unsigned char* p = smem_raw + round_up_dev(np * 8, 16);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* lrow = reinterpret_cast<T*>(p) + warp * (zlen + 2 * SR::RK);
  T* ring = lrow + zlen;
  if (MODE == kCWUpdate)
    for (int k = threadIdx.x; k < np; k += blockDim.x) vs[k] = vg[k];
  for (int k = lane; k < 2 * SR::RK; k += 32) ring[k] = T(0);
  __syncthreads();

  const double ga = MODE == kCWUpdate ? st->ga : 0.0;
  const double gb = MODE == kCWUpdate ? st->gb : 0.0;
  const double coef = MODE == kCWUpdate ? st->coef : 0.0;
  const T one_ga = (T)(1.0 - ga), one_gb = (T)(1.0 - gb);
  const T lam_s = (T)st->lam_s;
  const bool spike_on = MODE == kCWUpdate && st->corner_s;
  const long long i_s = st->i_s;
  const int j_s = st->j_s;
  const T spike_add = (T)(gb * st->spike);
  double a_sq = 0.0, a_l1 = 0.0, a_nnz = 0.0, a_ss = 0.0, a_sr = 0.0;
  AmRecW best{0.0, 0.0, 0.0, -1};
  const bool vec = (ldd % NV == 0) && (lds % NV == 0) && (MODE != kCWOutput || ldl % NV == 0);
  SR sr;

  for (int64_t i = (int64_t)blockIdx.x * RW_WARPS + warp; i < m; i += (int64_t)gridDim.x * RW_WARPS) {
    T* lhrow = LH + i * np;
    if (MODE == kCWUpdate) {
      // coarse rank-1 update L_H <- (1-ga) L_H + ga * coef * u_i v^T (cpcp.py:399-402)
      const double cu = ga * coef * u[i];
      for (int k = lane; k < zlen; k += 32) {
        const T val = k < nh ? (T)((double)one_ga * (double)lhrow[k] + cu * vs[k]) : T(0);
        lrow[k] = val;
        if (k < np) lhrow[k] = val;
      }
    } else if (MODE == kCWOutput) {
      for (int k = lane; k < zlen; k += 32) lrow[k] = k < np ? lhrow[k] : T(0);
    }
    __syncwarp();
    const T* drow = D + i * ldd;
    T* sro = S + i * lds;
    const uint32_t* mrow = mask ? mask + i * ldm : nullptr;
    const long long gi = row0 + i;
    const bool spike_row = spike_on && gi == i_s;
    sr.begin(ring);
    T* const outs[2] = {GH + i * np, SH + i * np};
    for (int cbase = 0; cbase < n; cbase += CH) {
      const int j = cbase + lane * NV;
      StencilVec<T, NV> sv;
      sv.load(ch, j);
      if (MODE == kCWOutput) {
        T lv[NV];
#pragma unroll
        for (int e = 0; e < NV; ++e) {
          const int c = min(sv.key[e], np);
          lv[e] = sv.w0[e] * lrow[c] + sv.w1[e] * lrow[c + 1];
        }
        store_vec<T, NV>(Lout + i * ldl, j, n, vec, lv);
        continue;
      }
      T dv[NV], sv_old[NV];
      load_vec<T, NV>(drow, j, n, vec, dv);
      if (MODE == kCWUpdate) load_vec_rw<T, NV>(sro, j, n, vec, sv_old);
      const uint32_t bits = mrow && j < n ? (__ldg(mrow + (j >> 5)) >> (j & 31)) : 0xffffffffu;
      T x[2][NV];
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        const int jj = j + e;
        const bool obs = (bits >> e) & 1u;
        const T d = dv[e];
        T r = T(0), sn = T(0);
        if (MODE == kCWInit) {
          r = obs ? -d : T(0);
        } else {
          const int c = min(sv.key[e], np);
          const T l = sv.w0[e] * lrow[c] + sv.w1[e] * lrow[c + 1];
          T sh = one_gb * sv_old[e];
          if (spike_row && jj == j_s) sh += spike_add;
          if (obs) {
            const T rh = (l + sh) - d;         // r after the segment step
            sn = soft_thr<T>(sh - rh, lam_s);  // cpcp.py:414-415
            r = (l + sn) - d;
          } else {
            sn = soft_thr<T>(sh, lam_s);
          }
        }
        if (jj >= n) r = sn = T(0);
        x[0][e] = r;
        x[1][e] = sn;
        if (jj < n) {
          const double rd = (double)r, sd = (double)sn;
          a_sq = fma(rd, rd, a_sq);
          a_l1 += fabs(sd);
          a_nnz += sn != T(0) ? 1.0 : 0.0;
          a_ss = fma(sd, sd, a_ss);
          a_sr = fma(sd, rd, a_sr);
          const double mg = fabs(rd);
          const long long idx = (long long)jj * m_global + gi;
          if (argmax_better(mg, idx, best.mag, best.idx)) best = AmRecW{mg, rd, sd, idx};
        }
      }
      if (MODE == kCWUpdate) store_vec<T, NV>(sro, j, n, vec, x[1]);
      sr.chunk(sv, x, cbase + CH < n ? __ldg(ch.c0 + cbase + CH) : INT_MAX, outs, nh, lane);
    }
    if (MODE != kCWOutput) sr.finish(outs, nh, np, lane);
    __syncwarp();
  }
  if (MODE == kCWOutput) return;
  __shared__ double scratch[5 * 32];
  __shared__ AmRecW amw[RW_WARPS];
  double vals[5] = {a_sq, a_l1, a_nnz, a_ss, a_sr};
  block_sum<5>(vals, scratch);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    AmRecW b;
    b.mag = __shfl_xor_sync(kFull, best.mag, o);
    b.val = __shfl_xor_sync(kFull, best.val, o);
    b.sval = __shfl_xor_sync(kFull, best.sval, o);
    b.idx = __shfl_xor_sync(kFull, best.idx, o);
    am_merge_w(best, b);
  }
  if (lane == 0) amw[warp] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    AmRecW b = amw[0];
    for (int w = 1; w < RW_WARPS; ++w) am_merge_w(b, amw[w]);
    double* o = part + 9 * blockIdx.x;
    for (int q = 0; q < 5; ++q) o[q] = vals[q];
    o[5] = b.mag;
    o[6] = b.val;
    o[7] = b.sval;
    o[8] = (double)b.idx;
  }
}

int cp_rows(CpcpPlan* p, int mode, const void* D, int64_t ldd, const uint32_t* mask, int64_t ldm, void* S,
            int64_t lds, void* Lout, int64_t ldl, cudaStream_t st) {
  const size_t tb = p->f32 ? 4 : 8;
  const int nv = p->f32 ? 4 : 2;
  const size_t smem = (size_t)round_up(p->ch.np * 8, 16) +
                      RW_WARPS * ((size_t)round_up(p->ch.np + 2, 4) + 2 * 64 * nv) * tb;
  const int blocks = p->row_blocks;
#define MLR_LAUNCH(T, MODE)                                                                                     \
  {                                                                                                             \
    auto kern = cp_rows_warp<T, MODE>;                                                                          \
    MLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));               \
    kern<<<blocks, RW_THREADS, smem, st>>>(p->dev, p->ch, p->m_local, p->row0, p->m_global, (const T*)D, ldd,    \
                                           mask, ldm, (T*)S, lds, (T*)p->LH, (T*)p->GH, (T*)p->SH, p->u, p->v, \
                                           (T*)Lout, ldl, p->row_part);                                         \
  }
  if (p->f32) {
    if (mode == kCWInit) MLR_LAUNCH(float, kCWInit) else if (mode == kCWUpdate) MLR_LAUNCH(float, kCWUpdate) else MLR_LAUNCH(float, kCWOutput)
  } else {
    if (mode == kCWInit) MLR_LAUNCH(double, kCWInit) else if (mode == kCWUpdate) MLR_LAUNCH(double, kCWUpdate) else MLR_LAUNCH(double, kCWOutput)
  }
#undef MLR_LAUNCH
  MLR_LAUNCH_CHECK("cp_rows_warp");
  return kOk;
}

// Segment-QP dots from coarse data (see cpcp.cu cp_dots_kernel): E_i in
// per-warp shared memory; each lane evaluates a_ij = E_i R_j^T for NV
// consecutive fine columns with vectorised stencil loads and 4 mask bits.
template <typename T>
__global__ void __launch_bounds__(RW_THREADS)
cp_dots_warp(const CpcpDev* __restrict__ st, ChainDev ch, int64_t m, int64_t row0, const uint32_t* __restrict__ mask,
             int64_t ldm, const T* __restrict__ LH, const T* __restrict__ GH, const T* __restrict__ SH,
             const double* __restrict__ vg, const double* __restrict__ ving, double* __restrict__ u,
             double* __restrict__ part) {
  if (st->done) return;
  constexpr int NV = 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = ch.n, nh = ch.nh, np = ch.np;
  double* vs = reinterpret_cast<double*>(smem_raw);
  double* vins = vs + np;
  double* E0 = vins + np;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* E = E0 + warp * (np + 2);
  for (int k = threadIdx.x; k < np; k += blockDim.x) {
    vs[k] = vg[k];
    vins[k] = ving[k];
  }
  __syncthreads();
  const double coef = st->coef;
  const double rs2 = st->none ? 0.0 : 1.0 / sqrt(st->s2);
  const bool spike_on = st->corner_s;
  const long long i_s = st->i_s;
  const int j_s = st->j_s;
  const double spike = st->spike;
  double aa = 0.0, ab = 0.0, ar = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * RW_WARPS + warp; i < m; i += (int64_t)gridDim.x * RW_WARPS) {
    const T* g = GH + i * np;
    const T* lh = LH + i * np;
    const T* sh = SH + i * np;
    double d = 0.0;
    for (int k = lane; k < nh; k += 32) d = fma((double)g[k], vins[k], d);
    d = warp_sum(d);
    const double ui = st->none ? 0.0 : d * rs2;
    if (lane == 0) u[i] = ui;
    const double cu = coef * ui;
    double e_ab = 0.0, e_ar = 0.0;
    for (int k = lane; k < np + 2; k += 32) {
      const double e = k < nh ? cu * vs[k] - (double)lh[k] : 0.0;
      E[k] = e;
      if (k < nh) {
        e_ab = fma(e, (double)sh[k], e_ab);
        e_ar = fma(e, (double)g[k], e_ar);
      }
    }
    ab -= e_ab;
    ar += e_ar;
    __syncwarp();
    const uint32_t* mrow = mask ? mask + i * ldm : nullptr;
    const bool srow = spike_on && (row0 + i) == i_s;
    double e_aa = 0.0;
    for (int j = lane * NV; j < n; j += 32 * NV) {
      int c[NV];
      double w0[NV], w1[NV];
      if (j + NV <= n) {
        const int4 cc = __ldg(reinterpret_cast<const int4*>(ch.c0 + j));
        const double2 a0 = __ldg(reinterpret_cast<const double2*>(ch.w0 + j));
        const double2 a1 = __ldg(reinterpret_cast<const double2*>(ch.w0 + j + 2));
        const double2 b0 = __ldg(reinterpret_cast<const double2*>(ch.w1 + j));
        const double2 b1 = __ldg(reinterpret_cast<const double2*>(ch.w1 + j + 2));
        c[0] = cc.x; c[1] = cc.y; c[2] = cc.z; c[3] = cc.w;
        w0[0] = a0.x; w0[1] = a0.y; w0[2] = a1.x; w0[3] = a1.y;
        w1[0] = b0.x; w1[1] = b0.y; w1[2] = b1.x; w1[3] = b1.y;
      } else {
#pragma unroll
        for (int e = 0; e < NV; ++e) {
          const bool in = j + e < n;
          c[e] = in ? ch.c0[j + e] : 0;
          w0[e] = in ? ch.w0[j + e] : 0.0;
          w1[e] = in ? ch.w1[j + e] : 0.0;
        }
      }
      const uint32_t bits = mrow ? (__ldg(mrow + (j >> 5)) >> (j & 31)) : 0xffffffffu;
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        if (j + e >= n || !((bits >> e) & 1u)) continue;
        const double a = E[c[e]] * w0[e] + E[c[e] + 1] * w1[e];
        e_aa = fma(a, a, e_aa);
        if (srow && j + e == j_s) ab += spike * a;
      }
    }
    aa += e_aa;
    __syncwarp();
  }
  __shared__ double scratch[3 * 32];
  double vals[3] = {aa, ab, ar};
  block_sum<3>(vals, scratch);
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x + 0] = vals[0];
    part[3 * blockIdx.x + 1] = vals[1];
    part[3 * blockIdx.x + 2] = vals[2];
  }
}

int cp_dots_rows(CpcpPlan* p, cudaStream_t st) {
  const size_t smem = (size_t)p->ch.np * 16 + RW_WARPS * (size_t)(p->ch.np + 2) * 8 + 64;
  const int blocks = p->row_blocks;
  if (p->f32) {
    MLR_CUDA(cudaFuncSetAttribute(cp_dots_warp<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cp_dots_warp<float><<<blocks, RW_THREADS, smem, st>>>(p->dev, p->ch, p->m_local, p->row0, p->mask_dev,
                                                          p->ldm_dev, (const float*)p->LH, (const float*)p->GH,
                                                          (const float*)p->SH, p->v, p->vin, p->u, p->dots_part);
  } else {
    MLR_CUDA(cudaFuncSetAttribute(cp_dots_warp<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cp_dots_warp<double><<<blocks, RW_THREADS, smem, st>>>(p->dev, p->ch, p->m_local, p->row0, p->mask_dev,
                                                           p->ldm_dev, (const double*)p->LH, (const double*)p->GH,
                                                           (const double*)p->SH, p->v, p->vin, p->u, p->dots_part);
  }
  MLR_LAUNCH_CHECK("cp_dots_warp");
  return kOk;
}

}  // namespace mlr
