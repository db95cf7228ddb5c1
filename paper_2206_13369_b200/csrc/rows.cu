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
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <initializer_list>
#include <type_traits>

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

// Per-lane asynchronous staging of the row chunks a warp will process
// (cp.async, 16 bytes per lane per stream, RING_ST chunks deep, continuing
// across the warp's rows): several chunks of D / Y / S and the mask word are
// in flight without holding registers.  Each lane reads back only the bytes
// it copied, so cp.async.wait_group alone orders the data.
constexpr int RING_ST = 4;
constexpr int RING_BYTES = RING_ST * (2 * 512 + 128);  // per warp: 2 streams + the mask word

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int src_bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

struct LaneRing {
  unsigned char* base;
  __device__ __forceinline__ unsigned char* slot(int s, int q, int lane) const {
    return base + ((s * 2 + q) * 32 + lane) * 16;
  }
  __device__ __forceinline__ uint32_t* mslot(int s, int lane) const {
    return reinterpret_cast<uint32_t*>(base + RING_ST * 1024 + (s * 32 + lane) * 4);
  }
};

// Stencil of NV consecutive fine columns; key = INT_MAX past n.
template <typename T, int NV>
struct StencilVec {
  int key[NV];
  T w0[NV], w1[NV];
  // weights only (regular chains compute the keys): zero past n
  __device__ __forceinline__ void loadw(const T* __restrict__ w0p, const T* __restrict__ w1p, int n, int j) {
    using VT = Vec<T>;
    if (j + NV <= n) {
      VT::unpack(__ldg(reinterpret_cast<const typename VT::V*>(w0p + j)), w0);
      VT::unpack(__ldg(reinterpret_cast<const typename VT::V*>(w1p + j)), w1);
    } else {
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        const bool in = j + e < n;
        w0[e] = in ? __ldg(w0p + j + e) : T(0);
        w1[e] = in ? __ldg(w1p + j + e) : T(0);
      }
    }
  }
  __device__ __forceinline__ void load(const int* __restrict__ c0, const T* __restrict__ w0p,
                                       const T* __restrict__ w1p, int n, int j) {
    using VT = Vec<T>;
    if (j + NV <= n) {
      VT::unpacki(__ldg(reinterpret_cast<const typename VT::I*>(c0 + j)), key);
      VT::unpack(__ldg(reinterpret_cast<const typename VT::V*>(w0p + j)), w0);
      VT::unpack(__ldg(reinterpret_cast<const typename VT::V*>(w1p + j)), w1);
    } else {
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        const bool in = j + e < n;
        key[e] = in ? __ldg(c0 + j + e) : INT_MAX;
        w0[e] = in ? __ldg(w0p + j + e) : T(0);
        w1[e] = in ? __ldg(w1p + j + e) : T(0);
      }
    }
  }
};

// Streaming restriction of NB fine quantities x (one row) onto coarse keys.
// Call chunk() once per chunk with every lane's NV values, then finish().
// Per chunk: an in-lane then a warp segmented scan (`steps` shuffle steps
// suffice when no run of equal c0 spans more than 2^steps lanes) gives every
// run's w0 and w1 sums; runs that end in the chunk are ranked with ballots
// and staged, and since keys are dense (run K ends before run K + 1), lane p
// writes key K_p = T1(run K_p - 1) + T0(run K_p) straight to HBM (coalesced).
template <typename T, int NB, int NV>
struct SegRestrict {
  static constexpr int MAXE = 32 * NV;  // run ends per chunk (at most one per element)
  static constexpr int STAGE_BYTES = MAXE * 4 + 2 * NB * MAXE * (int)sizeof(T);
  int* skey;
  T* st0;  // NB x MAXE
  T* st1;  // NB x MAXE
  int carry_key, last_key;
  T carry0[NB], carry1[NB], prev1[NB];

  __device__ __forceinline__ void begin(unsigned char* stage) {
    skey = reinterpret_cast<int*>(stage);
    st0 = reinterpret_cast<T*>(stage + MAXE * 4);
    st1 = st0 + NB * MAXE;
    carry_key = INT_MAX - 1;
    last_key = -1;
#pragma unroll
    for (int b = 0; b < NB; ++b) carry0[b] = carry1[b] = prev1[b] = T(0);
  }

  // next_key: c0 of the first fine column after this chunk (INT_MAX at the row end).
  __device__ __forceinline__ void chunk(const StencilVec<T, NV>& sv, const T (&x)[NB][NV], int next_key,
                                        T* const (&out)[NB], int lane, int steps) {
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
    for (int e = 1; e < NV; ++e) {
      const bool same = key[e] == key[e - 1];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        t0[b][e] += same ? t0[b][e - 1] : T(0);
        t1[b][e] += same ? t1[b][e - 1] : T(0);
      }
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
    for (int st = 0; st < 5; ++st) {
      if (st >= steps) break;
      const int o = 1 << st;
      const int kk = __shfl_up_sync(kFull, kt, o);
      const bool take = lane >= o && kk == kt;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const T a = __shfl_up_sync(kFull, s0[b], o);
        const T c = __shfl_up_sync(kFull, s1[b], o);
        s0[b] += take ? a : T(0);
        s1[b] += take ? c : T(0);
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
    const bool head = kp == key[0];
#pragma unroll
    for (int e = 0; e < NV; ++e) {
      const bool add = head && key[e] == key[0];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        t0[b][e] += add ? p0[b] : T(0);
        t1[b][e] += add ? p1[b] : T(0);
      }
    }
    // run ends, ranked across the warp
    int knext = __shfl_down_sync(kFull, key[0], 1);
    if (lane == 31) knext = next_key;
    carry_key = __shfl_sync(kFull, kt, 31);
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      carry0[b] = __shfl_sync(kFull, s0[b], 31);
      carry1[b] = __shfl_sync(kFull, s1[b], 31);
    }
    const unsigned lt = (1u << lane) - 1u;
    int r = 0, total = 0;
    bool end[NV];
#pragma unroll
    for (int e = 0; e < NV; ++e) {
      const int nk = e < NV - 1 ? key[e + 1] : knext;
      end[e] = key[e] != INT_MAX && nk != key[e];
      const unsigned bal = __ballot_sync(kFull, end[e]);
      r += __popc(bal & lt);
      total += __popc(bal);
    }
#pragma unroll
    for (int e = 0; e < NV; ++e)
      if (end[e]) {
        skey[r] = key[e];
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          st0[b * MAXE + r] = t0[b][e];
          st1[b * MAXE + r] = t1[b][e];
        }
        ++r;
      }
    __syncwarp();
    for (int q = lane; q < total; q += 32) {
      const int K = skey[q];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const T pv = q > 0 ? st1[b * MAXE + q - 1] : prev1[b];
        out[b][K] = pv + st0[b * MAXE + q];
      }
    }
    if (total > 0) {
      last_key = skey[total - 1];
#pragma unroll
      for (int b = 0; b < NB; ++b) prev1[b] = st1[b * MAXE + total - 1];
    }
    __syncwarp();
  }

  // key last_key + 1 holds only the final run's w1 sum; the rest of [.., np) is zero
  __device__ __forceinline__ void finish(T* const (&out)[NB], int nh, int np, int lane) {
    for (int k = last_key + 1 + lane; k < np; k += 32)
#pragma unroll
      for (int b = 0; b < NB; ++b) out[b][k] = (k == last_key + 1 && k < nh) ? prev1[b] : T(0);
  }
};

// Restriction for regular chains (repeated halving, n = n_H * P, P = 2^lgp,
// c0[j] = max(0, (j+1)/P - 1)).  Fine columns [pP, pP + P) are one group of
// L = P/NV lanes: their w1 parts and the w0 part of the group's last column
// (the first column of run p, whose w1 is zero) belong to coarse key p ("B"),
// the other w0 parts to key p - 1 ("A"; key 0 for the row's first group).
// Key p = B_p + A_{p+1}: a butterfly over the group, one shuffle from the
// next group, and a carry across chunks.  No keys, ballots or staging;
// fixed summation order (deterministic).
template <typename T, int NB, int NV>
struct RegRestrict {
  T carry[NB];
  bool have;
  __device__ __forceinline__ void begin() { have = false; }

  __device__ __forceinline__ void chunk(const T (&w0)[NV], const T (&w1)[NV], const T (&x)[NB][NV], int cbase,
                                        T* const (&out)[NB], int lane, int lgp) {
    constexpr int CH = 32 * NV;
    const int L = (1 << lgp) / NV;  // lanes per group (1..32)
    const bool last_lane = (lane & (L - 1)) == L - 1;
    const bool first_group = cbase == 0 && lane < L;
    const int pbase = cbase >> lgp;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      T a = T(0), bb = T(0);
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        const T p0 = w0[e] * x[b][e];
        if (e == NV - 1 && last_lane) bb += p0; else a += p0;
        bb = fma(w1[e], x[b][e], bb);
      }
      if (first_group) {
        bb += a;
        a = T(0);
      }
#pragma unroll
      for (int st = 0; st < 5; ++st) {
        const int o = 1 << st;
        if (o >= L) break;
        a += __shfl_xor_sync(kFull, a, o);
        bb += __shfl_xor_sync(kFull, bb, o);
      }
      const T an = L < 32 ? __shfl_down_sync(kFull, a, L) : T(0);
      if ((lane & (L - 1)) == 0 && lane + L < 32) out[b][pbase + (lane >> (lgp - (NV == 8 ? 3 : NV == 4 ? 2 : 1)))] = bb + an;
      if (lane == 0 && have) out[b][pbase - 1] = carry[b] + a;
      carry[b] = __shfl_sync(kFull, bb, 31);
    }
    have = true;
    (void)CH;
  }

  // the last group of the row's last chunk has no successor; zero the rest of [.., np)
  __device__ __forceinline__ void finish(T* const (&out)[NB], int n, int np, int lane, int lgp) {
    constexpr int CH = 32 * NV;
    const int plast = (((n + CH - 1) / CH) * CH >> lgp) - 1;
    for (int k = plast + lane; k < np; k += 32)
#pragma unroll
      for (int b = 0; b < NB; ++b) out[b][k] = k == plast ? carry[b] : T(0);
  }
};

__host__ __device__ __forceinline__ int seg_scan_steps(int max_run, int nv) {
  const int lanes = min(32, (max_run + 2 * nv - 2) / nv);  // lanes one run can touch
  int s = 0;
  while ((1 << s) < lanes) ++s;
  return s;
}

// -------------------------------------------------------------------- ML-PCP
enum RowModeW { kWStart = 0, kWUpdate = 1, kWOutput = 2 };

template <typename T, int MODE, bool RING, int RG>
__global__ void __launch_bounds__(RW_THREADS, 3)
pcp_rows_warp(const PcpDev* __restrict__ st, ChainDev ch, int64_t m, const T* __restrict__ D, int64_t ldd,
              const T* __restrict__ Yin, T* __restrict__ Yout, int64_t ldy, const T* __restrict__ Z,
              T* __restrict__ A, T* __restrict__ Lout, T* __restrict__ Sout, int64_t ldo, double* __restrict__ part) {
  if (MODE == kWUpdate && st->done) return;
  constexpr bool REG = RG > 0;  // regular chain; RG == 2: stencil weights held in registers (long rows)
  using SR = SegRestrict<T, 1, Vec<T>::N>;
  constexpr int NV = Vec<T>::N, CH = 32 * NV;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = ch.n, nh = ch.nh, np = ch.np;
  const int* __restrict__ c0p = ch.c0;
  const T* __restrict__ w0p = stencil_w0<T>(ch);
  const T* __restrict__ w1p = stencil_w1<T>(ch);
  const int steps = seg_scan_steps(ch.max_run, NV);
  const int zlen = round_up_dev(np + 2, 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int STAGE = REG ? 0 : SR::STAGE_BYTES;
  const int lgp = ch.reg_lgp;
  unsigned char* wbase = smem_raw + (size_t)warp * (zlen * sizeof(T) + STAGE + (RING ? RING_BYTES : 0));
  T* zrow = reinterpret_cast<T*>(wbase);
  unsigned char* stage = wbase + zlen * sizeof(T);
  const LaneRing ring{stage + STAGE};

  const double mu_d = st->mu;
  const T inv = (T)(1.0 / mu_d);
  const T mu = (T)mu_d;
  const T thr = (T)(st->lam * (1.0 / mu_d));
  const T inv_next = (T)(1.0 / (mu_d * st->rho));
  const double scale = st->scale;
  double acc_res = 0.0, acc_l1 = 0.0, acc_nnz = 0.0;
  const bool vec = (ldd % NV == 0) && (ldy % NV == 0) && (MODE != kWOutput || ldo % NV == 0);
  const bool pipe = RING && vec;
  SR sr;
  RegRestrict<T, 1, NV> rr;
  // regular chains: a lane's stencil weights depend only on its position in
  // the chunk (the phase (j+1) mod P) except in chunk 0, so they are loaded
  // once per kernel instead of once per chunk
  T rw0[NV], rw1[NV];
  constexpr bool wreg = RG == 2;
  if (wreg) {
#pragma unroll
    for (int e = 0; e < NV; ++e) {
      rw0[e] = __ldg(w0p + CH + lane * NV + e);
      rw1[e] = __ldg(w1p + CH + lane * NV + e);
    }
  }
  const int nc = (n + CH - 1) / CH;
  const int64_t first = (int64_t)blockIdx.x * RW_WARPS + warp, stride = (int64_t)gridDim.x * RW_WARPS;
  // prefetch cursor: (row, chunk, ring slot) of the next chunk to stage
  int64_t irow = first;
  int ic = 0, isl = 0;
  auto issue = [&]() {
    if (irow < m) {
      const int jq = ic * CH + lane * NV;
      const int bytes = jq < n ? min(16, (n - jq) * (int)sizeof(T)) : 0;
      cp_async16(ring.slot(isl, 0, lane), D + irow * ldd + (bytes ? jq : 0), bytes);
      if (MODE != kWStart) cp_async16(ring.slot(isl, 1, lane), Yin + irow * ldy + (bytes ? jq : 0), bytes);
    }
    cp_commit();
    isl = (isl + 1) & (RING_ST - 1);
    if (++ic == nc) {
      ic = 0;
      irow += stride;
    }
  };
  if (pipe)
    for (int q = 0; q < RING_ST - 1; ++q) issue();
  int csl = 0;  // ring slot of the chunk being processed

  for (int64_t i = first; i < m; i += stride) {
    if (MODE != kWStart) {
      for (int k = lane; k < zlen; k += 32) zrow[k] = k < np ? Z[i * np + k] : T(0);
      __syncwarp();
    }
    const T* drow = D + i * ldd;
    const T* yrow = Yin + i * ldy;
    if (REG) rr.begin(); else sr.begin(stage);
    T* const outp[1] = {A + i * np};
    T dn[NV], yn[NV];  // register path: one chunk in flight
    if (!pipe) {
      load_vec<T, NV>(drow, lane * NV, n, vec, dn);
      if (MODE != kWStart) load_vec<T, NV>(yrow, lane * NV, n, vec, yn);
    }
    for (int c = 0; c < nc; ++c) {
      const int cbase = c * CH;
      const int j = cbase + lane * NV;
      T dv[NV], yv[NV];
      if (pipe) {
        issue();
        cp_wait<RING_ST - 1>();
        const int sl = csl;
        csl = (csl + 1) & (RING_ST - 1);
        Vec<T>::unpack(*reinterpret_cast<const typename Vec<T>::V*>(ring.slot(sl, 0, lane)), dv);
        if (MODE != kWStart)
          Vec<T>::unpack(*reinterpret_cast<const typename Vec<T>::V*>(ring.slot(sl, 1, lane)), yv);
        else
#pragma unroll
          for (int e = 0; e < NV; ++e) yv[e] = T(0);
      } else {
#pragma unroll
        for (int e = 0; e < NV; ++e) {
          dv[e] = dn[e];
          yv[e] = MODE != kWStart ? yn[e] : T(0);
        }
        if (cbase + CH < n) {
          load_vec<T, NV>(drow, j + CH, n, vec, dn);
          if (MODE != kWStart) load_vec<T, NV>(yrow, j + CH, n, vec, yn);
        }
      }
      StencilVec<T, NV> sv;
      if (wreg && cbase > 0) {
#pragma unroll
        for (int e = 0; e < NV; ++e) {
          sv.w0[e] = j + e < n ? rw0[e] : T(0);
          sv.w1[e] = j + e < n ? rw1[e] : T(0);
        }
      } else if (REG) {
        sv.loadw(w0p, w1p, n, j);
      } else {
        sv.load(c0p, w0p, w1p, n, j);
      }
      T x[1][NV], yo[NV], lo_v[NV], so_v[NV];
      T c_res = T(0), c_l1 = T(0);
      int c_nnz = 0;
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        const T d = dv[e];
        if (MODE == kWStart) {
          // y = d / scale (pcp.py:115); work = y/mu + d (pcp.py:252-254, S = 0)
          const T y = (T)((double)d / scale);
          yo[e] = y;
          x[0][e] = y * inv + d;
        } else {
          const int c = REG ? max(0, ((j + e + 1) >> lgp) - 1) : min(sv.key[e], np);
          const T l = sv.w0[e] * zrow[c] + sv.w1[e] * zrow[c + 1];
          const T y = yv[e];
          const T w = y * inv + d - l;
          const T s = soft_thr<T>(w, thr);
          lo_v[e] = l;
          so_v[e] = s;
          if (MODE == kWUpdate) {
            const T res = (d - l) - s;  // zero past n (d = l = s = 0 there)
            const T ynew = y + res * mu;
            yo[e] = ynew;
            c_res = fma(res, res, c_res);
            c_l1 += fabs(s);
            c_nnz += s != T(0) ? 1 : 0;
            x[0][e] = ynew * inv_next + d - s;
          }
        }
      }
      if (MODE == kWUpdate) {
        acc_res += (double)c_res;
        acc_l1 += (double)c_l1;
        acc_nnz += (double)c_nnz;
      }
      if (MODE == kWOutput) {
        store_vec<T, NV>(Lout + i * ldo, j, n, vec, lo_v);
        store_vec<T, NV>(Sout + i * ldo, j, n, vec, so_v);
        continue;
      }
      store_vec<T, NV>(Yout + i * ldy, j, n, vec, yo);
      if (REG)
        rr.chunk(sv.w0, sv.w1, x, cbase, outp, lane, lgp);
      else
        sr.chunk(sv, x, cbase + CH < n ? __ldg(c0p + cbase + CH) : INT_MAX, outp, lane, steps);
    }
    if (MODE != kWOutput) {
      if (REG) rr.finish(outp, n, np, lane, lgp); else sr.finish(outp, nh, np, lane);
    }
    __syncwarp();
  }
  cp_wait<0>();
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

// ------------------------------------------------- FP32 regular-chain fast path
// The update passes of both solvers specialised for what every BASELINE
// config has: FP32, a regular chain with P = 2^LGP fine columns per coarse
// column (compile-time, so the lane-group butterflies unroll), n % 4 == 0,
// 16-byte aligned rows.  Same per-element arithmetic (and so the same
// results) as the general kernels; what goes is the per-chunk overhead the
// general ones pay: bounds checks and stencil loads on interior chunks (the
// weights are periodic after chunk 0 and sit in registers), 64-bit index
// arithmetic in the prefetch ring, runtime-bounded shuffle loops, a branchy
// arg-max.  The last, partial chunk of a row takes the checked path.  The
// next row's coarse row (Z, or L_H for ML-CPCP) rides in the prefetch ring
// when a row has at least RING_ST chunks and the double buffer fits (ZPF).
// Grid = the resident CTAs (one wave); unused partial-result slots up to the
// plan's row_blocks are written empty.
#ifndef FAST_RING
#define FAST_RING 4
#endif
// per warp: FAST_RING slots of two streams (VB = 4 NV bytes per lane each) + the mask word
__host__ __device__ constexpr int fast_ring_bytes(int nv) { return FAST_RING * (2 * 32 * 4 * nv + 128); }
template <int ST, int VB>
struct LaneRingT {
  unsigned char* base;
  __device__ __forceinline__ unsigned char* slot(int s, int q, int lane) const {
    return base + ((s * 2 + q) * 32 + lane) * VB;
  }
  __device__ __forceinline__ uint32_t* mslot(int s, int lane) const {
    return reinterpret_cast<uint32_t*>(base + ST * 64 * VB + (s * 32 + lane) * 4);
  }
};
// NV consecutive floats of one lane: ring slot <-> registers, global row <- registers
template <int NV>
__device__ __forceinline__ void ring_unpack(const unsigned char* slot, float (&o)[NV]) {
#pragma unroll
  for (int v = 0; v < NV / 4; ++v) {
    const float4 q = reinterpret_cast<const float4*>(slot)[v];
    o[4 * v] = q.x;
    o[4 * v + 1] = q.y;
    o[4 * v + 2] = q.z;
    o[4 * v + 3] = q.w;
  }
}
template <int NV, bool FULL>
__device__ __forceinline__ void row_store(float* row, int j, int n, const float (&o)[NV]) {
#pragma unroll
  for (int v = 0; v < NV / 4; ++v)
    if (FULL || j + 4 * v < n)
      *reinterpret_cast<float4*>(row + j + 4 * v) = make_float4(o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
}
// lane-strided cp.async of NV floats of a fine row (n % 4 == 0; zero-filled past n)
template <int NV>
__device__ __forceinline__ void ring_issue(unsigned char* slot, const float* row, int jq, int n) {
#pragma unroll
  for (int v = 0; v < NV / 4; ++v) {
    const bool in = jq + 4 * v < n;
    cp_async16(slot + 16 * v, row + (in ? jq + 4 * v : 0), in ? 16 : 0);
  }
}
#ifndef FAST_MINB
#define FAST_MINB 2
#endif

// lane-strided cp.async of one coarse row (np floats, np % 4 == 0) into smem
__device__ __forceinline__ void copy_coarse_row(float* dst, const float* src, int np, int lane) {
  for (int k = lane * 4; k < np; k += 128) cp_async16(dst + k, src + k, 16);
}

template <int LGP, bool ZPF, int NV>
__global__ void __launch_bounds__(RW_THREADS, FAST_MINB)
pcp_update_fast(const PcpDev* __restrict__ st, ChainDev ch, int m, const float* __restrict__ D, int64_t ldd,
                const float* __restrict__ Yin, float* __restrict__ Yout, int64_t ldy, const float* __restrict__ Z,
                float* __restrict__ A, double* __restrict__ part, int part_slots) {
  if (st->done) return;
  constexpr int CH = 32 * NV, VB = 4 * NV;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = ch.n, np = ch.np;
  const int zlen = round_up_dev(np + 2, 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wbase = smem_raw + (size_t)warp * ((ZPF ? 2 : 1) * zlen * 4 + fast_ring_bytes(NV));
  float* zbuf = reinterpret_cast<float*>(wbase);
  const LaneRingT<FAST_RING, VB> ring{wbase + (ZPF ? 2 : 1) * zlen * 4};
  if (blockIdx.x == 0)
    for (int b = gridDim.x + threadIdx.x; b < part_slots; b += blockDim.x)
      part[3 * b] = part[3 * b + 1] = part[3 * b + 2] = 0.0;

  const double mu_d = st->mu;
  const float inv = (float)(1.0 / mu_d);
  const float mu = (float)mu_d;
  const float thr = (float)(st->lam * (1.0 / mu_d));
  const float inv_next = (float)(1.0 / (mu_d * st->rho));
  double acc_res = 0.0, acc_l1 = 0.0;
  long long i_nnz = 0;
  const float* __restrict__ w0p = ch.w0f;
  const float* __restrict__ w1p = ch.w1f;
  // chunk 0 weights are reloaded (L1) per row; interior chunks share rw
  float rw0[NV], rw1[NV];
#pragma unroll
  for (int e = 0; e < NV; ++e) {
    const int j1 = CH + lane * NV + e;
    rw0[e] = j1 < n ? __ldg(w0p + j1) : 0.f;
    rw1[e] = j1 < n ? __ldg(w1p + j1) : 0.f;
  }
  const int nfull = n / CH, nc = (n + CH - 1) / CH;
  const int first = blockIdx.x * RW_WARPS + warp, stride = gridDim.x * RW_WARPS;
  int irow = first, ic = 0, isl = 0;
  const float* dnext = D + (int64_t)first * ldd;
  const float* ynext = Yin + (int64_t)first * ldy;
  auto issue = [&]() {
    if (irow < m) {
      const int jq = ic * CH + lane * NV;
      ring_issue<NV>(ring.slot(isl, 0, lane), dnext, jq, n);
      ring_issue<NV>(ring.slot(isl, 1, lane), ynext, jq, n);
    }
    cp_commit();
    isl = (isl + 1) & (FAST_RING - 1);
    if (++ic == nc) {
      ic = 0;
      irow += stride;
      dnext += (int64_t)stride * ldd;
      ynext += (int64_t)stride * ldy;
    }
  };
  if (ZPF && first < m) copy_coarse_row(zbuf, Z + (int64_t)first * np, np, lane);
#pragma unroll
  for (int q = 0; q < FAST_RING - 1; ++q) issue();
  int csl = 0, zb = 0;
  RegRestrict<float, 1, NV> rr;

  for (int i = first; i < m; i += stride) {
    float* zrow = zbuf + (ZPF ? zb * zlen : 0);
    if (ZPF) {
      // this row's Z went out with the ring group of the previous row's chunk 0
      // (>= FAST_RING groups ago) or, for the first row, with the first group
      cp_wait<FAST_RING - 2>();
      __syncwarp();
      if (lane < zlen - np) zrow[np + lane] = 0.f;
      if (i + stride < m) copy_coarse_row(zbuf + (zb ^ 1) * zlen, Z + (int64_t)(i + stride) * np, np, lane);
      zb ^= 1;
    } else {
      for (int k = lane; k < zlen; k += 32) zrow[k] = k < np ? Z[(int64_t)i * np + k] : 0.f;
    }
    __syncwarp();
    float* yrow = Yout + (int64_t)i * ldy;
    rr.begin();
    float* const outp[1] = {A + (int64_t)i * np};

    auto chunk = [&](int c, const float(&w0)[NV], const float(&w1)[NV], auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
      const int cbase = c * CH;
      const int j = cbase + lane * NV;
      issue();
      cp_wait<FAST_RING - 1>();
      const int sl = csl;
      csl = (csl + 1) & (FAST_RING - 1);
      float dv[NV], yv[NV];
      ring_unpack<NV>(ring.slot(sl, 0, lane), dv);
      ring_unpack<NV>(ring.slot(sl, 1, lane), yv);
      // coarse keys of the lane's NV columns: k0 for e < NV - 1, k3 for the last (P >= NV)
      int k0 = max(0, (j >> LGP) - 1), k3 = max(0, ((j + NV) >> LGP) - 1);
      if (!FULL) {
        k0 = min(k0, zlen - 2);
        k3 = min(k3, zlen - 2);
      }
      const float z0 = zrow[k0], z1 = zrow[k0 + 1], z3a = zrow[k3], z3b = zrow[k3 + 1];
      float x[1][NV], yo[NV];
      float c_res = 0.f, c_l1 = 0.f;
      int c_nnz = 0;
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        const float za = e < NV - 1 ? z0 : z3a, zb_ = e < NV - 1 ? z1 : z3b;
        const float l = w0[e] * za + w1[e] * zb_;
        const float d = dv[e], y = yv[e];
        const float w = y * inv + d - l;
        const float s = soft_thr<float>(w, thr);
        const float res = (d - l) - s;  // zero past n (d = l = s = 0 there)
        const float ynew = y + res * mu;
        yo[e] = ynew;
        c_res = fmaf(res, res, c_res);
        c_l1 += fabsf(s);
        c_nnz += s != 0.f ? 1 : 0;
        x[0][e] = ynew * inv_next + d - s;
      }
      acc_res += (double)c_res;
      acc_l1 += (double)c_l1;
      i_nnz += c_nnz;
      row_store<NV, FULL>(yrow, j, n, yo);
      rr.chunk(w0, w1, x, cbase, outp, lane, LGP);
    };
    if (nfull > 0) {
      float cw0[NV], cw1[NV];
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        cw0[e] = __ldg(w0p + lane * NV + e);
        cw1[e] = __ldg(w1p + lane * NV + e);
      }
      chunk(0, cw0, cw1, std::true_type{});
      for (int c = 1; c < nfull; ++c) chunk(c, rw0, rw1, std::true_type{});
    }
    if (nfull < nc) {
      float t0[NV], t1[NV];
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        const int jt = nfull * CH + lane * NV + e;
        const bool in = jt < n;
        t0[e] = in ? (nfull == 0 ? __ldg(w0p + jt) : rw0[e]) : 0.f;
        t1[e] = in ? (nfull == 0 ? __ldg(w1p + jt) : rw1[e]) : 0.f;
      }
      chunk(nfull, t0, t1, std::false_type{});
    }
    rr.finish(outp, n, np, lane, LGP);
    __syncwarp();
  }
  cp_wait<0>();
  __shared__ double scratch[3 * 32];
  double v[3] = {acc_res, acc_l1, (double)i_nnz};
  block_sum<3>(v, scratch);
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x + 0] = v[0];
    part[3 * blockIdx.x + 1] = v[1];
    part[3 * blockIdx.x + 2] = v[2];
  }
}

// fast path applicability (both solvers): FP32, regular chain with 4 <= P <= 32,
// periodic weights after chunk 0, n % 4 == 0, 16-byte aligned leading dimensions
static bool fast_ok(const ChainDev& ch, bool f32, std::initializer_list<int64_t> lds) {
  if (!f32 || ch.reg_lgp < 2 || ch.reg_lgp > 5 || !ch.reg_periodic || ch.n % 4 != 0 || ch.np % 4 != 0) return false;
  for (int64_t l : lds)
    if (l % 4 != 0) return false;
  const char* env = getenv("MLR_FAST_ROWS");
  return !(env && env[0] == '0');
}

template <typename K>
static int fast_grid(K kern, size_t smem, int want) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, RW_THREADS, smem);
  return std::max(1, std::min(want, sms * std::max(per, 1)));
}

// Columns per lane.  8 (when a coarse group spans >= 8) halves the per-chunk
// overhead; measured (B200): ML-CPCP C4 -10%, C3 -15%, but ML-PCP C2 +8% and
// C5 +12% (its larger ring no longer leaves room for two CTAs' coarse rows).
static int fast_nv(const ChainDev& ch, bool cpcp) {
  const char* env = getenv("MLR_FAST_NV");
  if (env && (env[0] == '4' || env[0] == '8')) return ch.reg_lgp >= 3 ? env[0] - '0' : 4;
  return cpcp && ch.reg_lgp >= 3 ? 8 : 4;
}

// double-buffer the coarse row when a row has >= FAST_RING chunks and 2 CTAs still fit
static bool fast_zpf(const ChainDev& ch, size_t fixed, int nv) {
  const size_t zl = (size_t)round_up(ch.np + 2, 4) * 4;
  return (ch.n + 32 * nv - 1) / (32 * nv) >= FAST_RING &&
         fixed + RW_WARPS * (2 * zl + fast_ring_bytes(nv)) <= 110 * 1024;
}

template <int LGP, int NV>
static int pcp_fast_launch(PcpPlan* p, const void* D, int64_t ldd, const void* Yin, void* Yout, int64_t ldy,
                           cudaStream_t st) {
  const bool zpf = fast_zpf(p->ch, 0, NV);
  const size_t smem = RW_WARPS * ((zpf ? 2 : 1) * (size_t)round_up(p->ch.np + 2, 4) * 4 + fast_ring_bytes(NV));
  auto kern = zpf ? pcp_update_fast<LGP, true, NV> : pcp_update_fast<LGP, false, NV>;
  MLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = fast_grid(kern, smem, p->row_blocks);
  kern<<<grid, RW_THREADS, smem, st>>>(p->dev, p->ch, (int)p->m_local, (const float*)D, ldd, (const float*)Yin,
                                       (float*)Yout, ldy, (const float*)p->Z, (float*)p->A, p->row_part,
                                       p->row_blocks);
  MLR_LAUNCH_CHECK("pcp_update_fast");
  return kOk;
}

bool rows_warp_ok(const ChainDev& ch, bool) { return ch.keys_dense != 0; }
// regular chains whose groups are whole lanes and fit a chunk
static bool rows_reg_ok(const ChainDev& ch, bool f32) {
  const int nv = f32 ? 4 : 2, P = 1 << ch.reg_lgp;
  return ch.reg_lgp > 0 && P >= nv && P <= 32 * nv;
}

int pcp_rows(PcpPlan* p, int mode, const void* D, int64_t ldd, const void* Yin, void* Yout, int64_t ldy, void* Lout,
             void* Sout, int64_t ldo, cudaStream_t st) {
  const size_t tb = p->f32 ? 4 : 8;
  const bool reg = rows_reg_ok(p->ch, p->f32);
  if (mode == kWUpdate && fast_ok(p->ch, p->f32, {ldd, ldy}) && p->m_local < INT_MAX) {
    const bool v8 = fast_nv(p->ch, false) == 8;
    switch (p->ch.reg_lgp) {
      case 2: return pcp_fast_launch<2, 4>(p, D, ldd, Yin, Yout, ldy, st);
      case 3: return v8 ? pcp_fast_launch<3, 8>(p, D, ldd, Yin, Yout, ldy, st)
                        : pcp_fast_launch<3, 4>(p, D, ldd, Yin, Yout, ldy, st);
      case 4: return v8 ? pcp_fast_launch<4, 8>(p, D, ldd, Yin, Yout, ldy, st)
                        : pcp_fast_launch<4, 4>(p, D, ldd, Yin, Yout, ldy, st);
      default: return v8 ? pcp_fast_launch<5, 8>(p, D, ldd, Yin, Yout, ldy, st)
                         : pcp_fast_launch<5, 4>(p, D, ldd, Yin, Yout, ldy, st);
    }
  }
  const size_t stage = reg ? 0 : (p->f32 ? SegRestrict<float, 1, 4>::STAGE_BYTES : SegRestrict<double, 1, 2>::STAGE_BYTES);
  // the cp.async ring only while 3 CTAs per SM still fit (occupancy first)
  const size_t base = RW_WARPS * ((size_t)round_up(p->ch.np + 2, 4) * tb + stage);
  const bool ring = base + RW_WARPS * RING_BYTES <= 80 * 1024;
  const size_t smem = base + (ring ? RW_WARPS * RING_BYTES : 0);
  const int blocks = p->row_blocks;
  // weights in registers pay off on long rows only (measured: C5 -13%, C2 +7%)
  const int rg = reg ? (p->ch.n >= 16 * 32 * (p->f32 ? 4 : 2) ? 2 : 1) : 0;
#define MLR_LAUNCH(T, MODE)                                                                                     \
  {                                                                                                             \
    auto kern = rg == 2 ? (ring ? pcp_rows_warp<T, MODE, true, 2> : pcp_rows_warp<T, MODE, false, 2>)            \
              : rg == 1 ? (ring ? pcp_rows_warp<T, MODE, true, 1> : pcp_rows_warp<T, MODE, false, 1>)            \
                        : (ring ? pcp_rows_warp<T, MODE, true, 0> : pcp_rows_warp<T, MODE, false, 0>);           \
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

template <typename T, int MODE, bool RING, bool REG>
__global__ void __launch_bounds__(RW_THREADS, 3)
cp_rows_warp(const CpcpDev* __restrict__ st, ChainDev ch, int64_t m, int64_t row0, int64_t m_global,
             const T* __restrict__ D, int64_t ldd, const uint32_t* __restrict__ mask, int64_t ldm, T* __restrict__ S,
             int64_t lds, T* __restrict__ LH, T* __restrict__ GH, T* __restrict__ SH, const double* __restrict__ u,
             const double* __restrict__ vg, T* __restrict__ Lout, int64_t ldl, double* __restrict__ part) {
  if (MODE == kCWUpdate && st->done) return;
  using SR = SegRestrict<T, 2, Vec<T>::N>;
  constexpr int NV = Vec<T>::N, CH = 32 * NV;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = ch.n, nh = ch.nh, np = ch.np;
  const int* __restrict__ c0p = ch.c0;
  const T* __restrict__ w0p = stencil_w0<T>(ch);
  const T* __restrict__ w1p = stencil_w1<T>(ch);
  const int steps = seg_scan_steps(ch.max_run, NV);
  const int zlen = round_up_dev(np + 2, 4);
  double* vs = reinterpret_cast<double*>(smem_raw);  // v (np), CTA-shared
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int STAGE = REG ? 0 : SR::STAGE_BYTES;
  const int lgp = ch.reg_lgp;
  unsigned char* wbase =
      smem_raw + round_up_dev(np * 8, 16) + (size_t)warp * (zlen * sizeof(T) + STAGE + (RING ? RING_BYTES : 0));
  T* lrow = reinterpret_cast<T*>(wbase);
  unsigned char* stage = wbase + zlen * sizeof(T);
  const LaneRing ring{stage + STAGE};
  if (MODE == kCWUpdate)
    for (int k = threadIdx.x; k < np; k += blockDim.x) vs[k] = vg[k];
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
  // arg-max |r| (ties: smallest column-major index); the index is formed only on ties
  T bm = T(-1), bval = T(0), bsv = T(0);
  long long bidx = -1;
  const bool vec = (ldd % NV == 0) && (lds % NV == 0) && (MODE != kCWOutput || ldl % NV == 0);
  SR sr;
  RegRestrict<T, 2, NV> rr;
  const int nc = (n + CH - 1) / CH;
  const int64_t first = (int64_t)blockIdx.x * RW_WARPS + warp, stride = (int64_t)gridDim.x * RW_WARPS;
  const bool pipe = RING && vec && MODE != kCWOutput;
  int64_t irow = first;
  int ic = 0, isl = 0;
  auto issue = [&]() {  // stage the next chunk of this warp's (row, chunk) sequence
    if (irow < m) {
      const int jq = ic * CH + lane * NV;
      const int bytes = jq < n ? min(16, (n - jq) * (int)sizeof(T)) : 0;
      cp_async16(ring.slot(isl, 0, lane), D + irow * ldd + (bytes ? jq : 0), bytes);
      if (MODE == kCWUpdate) cp_async16(ring.slot(isl, 1, lane), S + irow * lds + (bytes ? jq : 0), bytes);
      if (mask) cp_async4(ring.mslot(isl, lane), mask + irow * ldm + (jq < n ? (jq >> 5) : 0), jq < n ? 4 : 0);
    }
    cp_commit();
    isl = (isl + 1) & (RING_ST - 1);
    if (++ic == nc) {
      ic = 0;
      irow += stride;
    }
  };
  if (pipe)
    for (int q = 0; q < RING_ST - 1; ++q) issue();
  int csl = 0;

  for (int64_t i = first; i < m; i += stride) {
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
    if (REG) rr.begin(); else sr.begin(stage);
    T* const outs[2] = {GH + i * np, SH + i * np};
    T dn[NV], sn_[NV];  // register path: one chunk in flight
    uint32_t bitn = 0xffffffffu;
    if (!pipe && MODE != kCWOutput) {
      load_vec<T, NV>(drow, lane * NV, n, vec, dn);
      if (MODE == kCWUpdate) load_vec_rw<T, NV>(sro, lane * NV, n, vec, sn_);
      bitn = mrow ? (lane * NV < n ? __ldg(mrow + ((lane * NV) >> 5)) >> ((lane * NV) & 31) : 0u) : 0xffffffffu;
    }
    for (int c = 0; c < nc; ++c) {
      const int cbase = c * CH;
      const int j = cbase + lane * NV;
      StencilVec<T, NV> sv;
      // (per-lane weights in registers, as in pcp_rows_warp, spill here)
      if (REG) sv.loadw(w0p, w1p, n, j); else sv.load(c0p, w0p, w1p, n, j);
      if (MODE == kCWOutput) {
        T lv[NV];
#pragma unroll
        for (int e = 0; e < NV; ++e) {
          const int c = REG ? max(0, ((j + e + 1) >> lgp) - 1) : min(sv.key[e], np);
          lv[e] = sv.w0[e] * lrow[c] + sv.w1[e] * lrow[c + 1];
        }
        store_vec<T, NV>(Lout + i * ldl, j, n, vec, lv);
        continue;
      }
      T dv[NV], sold[NV];
      uint32_t bits = 0xffffffffu;
      if (pipe) {
        issue();
        cp_wait<RING_ST - 1>();
        const int sl = csl;
        csl = (csl + 1) & (RING_ST - 1);
        Vec<T>::unpack(*reinterpret_cast<const typename Vec<T>::V*>(ring.slot(sl, 0, lane)), dv);
        if (MODE == kCWUpdate)
          Vec<T>::unpack(*reinterpret_cast<const typename Vec<T>::V*>(ring.slot(sl, 1, lane)), sold);
        else
#pragma unroll
          for (int e = 0; e < NV; ++e) sold[e] = T(0);
        if (mrow) bits = j < n ? (*ring.mslot(sl, lane) >> (j & 31)) : 0u;
      } else {
#pragma unroll
        for (int e = 0; e < NV; ++e) {
          dv[e] = dn[e];
          sold[e] = MODE == kCWUpdate ? sn_[e] : T(0);
        }
        bits = bitn;
        if (cbase + CH < n) {
          load_vec<T, NV>(drow, j + CH, n, vec, dn);
          if (MODE == kCWUpdate) load_vec_rw<T, NV>(sro, j + CH, n, vec, sn_);
          bitn = mrow ? (j + CH < n ? __ldg(mrow + ((j + CH) >> 5)) >> ((j + CH) & 31) : 0u) : 0xffffffffu;
        }
      }
      T x[2][NV];
      if (MODE == kCWInit) {
#pragma unroll
        for (int e = 0; e < NV; ++e) {
          x[0][e] = ((bits >> e) & 1u) ? -dv[e] : T(0);  // r = -P[D]; zero past n
          x[1][e] = T(0);
        }
      } else {
        T sh[NV];
#pragma unroll
        for (int e = 0; e < NV; ++e) sh[e] = one_gb * sold[e];
        if (spike_row) {
#pragma unroll
          for (int e = 0; e < NV; ++e)
            if (j + e == j_s) sh[e] += spike_add;
        }
#pragma unroll
        for (int e = 0; e < NV; ++e) {
          const int c = REG ? max(0, ((j + e + 1) >> lgp) - 1) : min(sv.key[e], np);
          const T l = sv.w0[e] * lrow[c] + sv.w1[e] * lrow[c + 1];
          const T d = dv[e];
          const bool obs = (bits >> e) & 1u;
          const T rh = (l + sh[e]) - d;                       // r after the segment step
          const T sn = soft_thr<T>(obs ? sh[e] - rh : sh[e], lam_s);  // cpcp.py:414-415
          x[0][e] = obs ? (l + sn) - d : T(0);
          x[1][e] = sn;
        }
      }
      // statistics (per-chunk partials in T, then FP64) and the arg-max
      T c_sq = T(0), c_l1 = T(0), c_ss = T(0), c_sr = T(0);
      int c_nnz = 0;
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        const T r = x[0][e], sn = x[1][e];
        c_sq = fma(r, r, c_sq);
        c_l1 += fabs(sn);
        c_nnz += sn != T(0) ? 1 : 0;
        c_ss = fma(sn, sn, c_ss);
        c_sr = fma(sn, r, c_sr);
        const T mg = fabs(r);
        if (mg >= bm && j + e < n) {
          const long long idx = (long long)(j + e) * m_global + gi;
          if (mg > bm || idx < bidx) {
            bm = mg;
            bval = r;
            bsv = sn;
            bidx = idx;
          }
        }
      }
      a_sq += (double)c_sq;
      a_l1 += (double)c_l1;
      a_nnz += (double)c_nnz;
      a_ss += (double)c_ss;
      a_sr += (double)c_sr;
      if (MODE == kCWUpdate) store_vec<T, NV>(sro, j, n, vec, x[1]);
      if (REG)
        rr.chunk(sv.w0, sv.w1, x, cbase, outs, lane, lgp);
      else
        sr.chunk(sv, x, cbase + CH < n ? __ldg(c0p + cbase + CH) : INT_MAX, outs, lane, steps);
    }
    if (MODE != kCWOutput) {
      if (REG) rr.finish(outs, n, np, lane, lgp); else sr.finish(outs, nh, np, lane);
    }
    __syncwarp();
  }
  cp_wait<0>();
  if (MODE == kCWOutput) return;
  __shared__ double scratch[5 * 32];
  __shared__ AmRecW amw[RW_WARPS];
  double vals[5] = {a_sq, a_l1, a_nnz, a_ss, a_sr};
  block_sum<5>(vals, scratch);
  AmRecW best{bidx >= 0 ? (double)bm : 0.0, (double)bval, (double)bsv, bidx};
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

// ML-CPCP update pass, FP32 regular-chain fast path (see pcp_update_fast)
template <int LGP, bool ZPF, int NV>
__global__ void __launch_bounds__(RW_THREADS, FAST_MINB)
cp_update_fast(const CpcpDev* __restrict__ st, ChainDev ch, int m, int64_t row0, int64_t m_global,
               const float* __restrict__ D, int64_t ldd, const uint32_t* __restrict__ mask, int64_t ldm,
               float* __restrict__ S, int64_t lds, float* __restrict__ LH, float* __restrict__ GH,
               float* __restrict__ SH, const double* __restrict__ u, const double* __restrict__ vg,
               double* __restrict__ part, int part_slots) {
  if (st->done) return;
  constexpr int CH = 32 * NV, VB = 4 * NV;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = ch.n, nh = ch.nh, np = ch.np;
  const int zlen = round_up_dev(np + 2, 4);
  double* vs = reinterpret_cast<double*>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wbase = smem_raw + round_up_dev(np * 8, 16) + (size_t)warp * ((ZPF ? 2 : 1) * zlen * 4 + fast_ring_bytes(NV));
  float* lbuf = reinterpret_cast<float*>(wbase);
  const LaneRingT<FAST_RING, VB> ring{wbase + (ZPF ? 2 : 1) * zlen * 4};
  for (int k = threadIdx.x; k < np; k += blockDim.x) vs[k] = vg[k];
  if (blockIdx.x == 0)  // empty partial-result slots past the grid
    for (int b = gridDim.x + threadIdx.x; b < part_slots; b += blockDim.x) {
      double* o = part + 9 * b;
      for (int q = 0; q < 8; ++q) o[q] = 0.0;
      o[8] = -1.0;
    }
  __syncthreads();

  const double ga = st->ga, gb = st->gb, coef = st->coef;
  const float one_ga = (float)(1.0 - ga), one_gb = (float)(1.0 - gb);
  const float lam_s = (float)st->lam_s;
  const bool spike_on = st->corner_s;
  const long long i_s = st->i_s;
  const int j_s = st->j_s;
  const float spike_add = (float)(gb * st->spike);
  const float* __restrict__ w0p = ch.w0f;
  const float* __restrict__ w1p = ch.w1f;
  // stencil weights: chunk 0 (the first coarse group differs) and the
  // periodic interior chunks, held for the whole kernel
  float rw0[NV], rw1[NV];  // chunk 0 weights are reloaded (L1) per row
#pragma unroll
  for (int e = 0; e < NV; ++e) {
    const int j1 = CH + lane * NV + e;
    rw0[e] = j1 < n ? __ldg(w0p + j1) : 0.f;
    rw1[e] = j1 < n ? __ldg(w1p + j1) : 0.f;
  }
  double a_sq = 0.0, a_l1 = 0.0, a_ss = 0.0, a_sr = 0.0;
  long long i_nnz = 0;  // exact, as the per-chunk FP64 sum of the general kernel
  float bm = -1.f, bval = 0.f, bsv = 0.f;
  int bj = INT_MAX, brow = -1;
  const int nfull = n / CH;
  const int nc = (n + CH - 1) / CH;
  const int first = blockIdx.x * RW_WARPS + warp, stride = gridDim.x * RW_WARPS;
  struct {
    int irow, ic, isl;
  } cur{first, 0, 0};
  const float* dnext = D + (int64_t)first * ldd;
  const float* snext = S + (int64_t)first * lds;
  const uint32_t* mnext = mask + (int64_t)first * ldm;
  auto issue = [&]() {
    if (cur.irow < m) {
      const int jq = cur.ic * CH + lane * NV;
      const bool in = jq < n;
      ring_issue<NV>(ring.slot(cur.isl, 0, lane), dnext, jq, n);
      ring_issue<NV>(ring.slot(cur.isl, 1, lane), snext, jq, n);
      cp_async4(ring.mslot(cur.isl, lane), mnext + (in ? (jq >> 5) : 0), in ? 4 : 0);
    }
    cp_commit();
    cur.isl = (cur.isl + 1) & (FAST_RING - 1);
    if (++cur.ic == nc) {
      cur.ic = 0;
      cur.irow += stride;
      dnext += (int64_t)stride * ldd;
      snext += (int64_t)stride * lds;
      mnext += (int64_t)stride * ldm;
    }
  };
  if (ZPF && first < m) copy_coarse_row(lbuf, LH + (int64_t)first * np, np, lane);
#pragma unroll
  for (int q = 0; q < FAST_RING - 1; ++q) issue();
  int csl = 0, lb = 0;
  RegRestrict<float, 2, NV> rr;

  for (int i = first; i < m; i += stride) {
    float* lhrow = LH + (int64_t)i * np;
    float* lrow = lbuf + (ZPF ? lb * zlen : 0);
    if (ZPF) {  // this row's L_H arrived with an earlier ring group (see pcp_update_fast)
      cp_wait<FAST_RING - 2>();
      __syncwarp();
    }
    {
      // coarse rank-1 update L_H <- (1-ga) L_H + ga * coef * u_i v^T (cpcp.py:399-402)
      const double cu = ga * coef * u[i];
      for (int k = lane; k < zlen; k += 32) {
        const float old = k < nh ? (ZPF ? lrow[k] : lhrow[k]) : 0.f;
        const float val = k < nh ? (float)((double)one_ga * (double)old + cu * vs[k]) : 0.f;
        lrow[k] = val;
        if (k < np) lhrow[k] = val;
      }
    }
    if (ZPF) {
      if (i + stride < m) copy_coarse_row(lbuf + (lb ^ 1) * zlen, LH + (int64_t)(i + stride) * np, np, lane);
      lb ^= 1;
    }
    __syncwarp();
    float* sro = S + (int64_t)i * lds;
    const long long gi = row0 + i;
    const bool spike_row = spike_on && gi == i_s;
    rr.begin();
    float* const outs[2] = {GH + (int64_t)i * np, SH + (int64_t)i * np};

    auto chunk = [&](int c, const float(&w0)[NV], const float(&w1)[NV], auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
      const int cbase = c * CH;
      const int j = cbase + lane * NV;
      issue();
      cp_wait<FAST_RING - 1>();
      const int sl = csl;
      csl = (csl + 1) & (FAST_RING - 1);
      float dv[NV], sold[NV];
      ring_unpack<NV>(ring.slot(sl, 0, lane), dv);
      ring_unpack<NV>(ring.slot(sl, 1, lane), sold);
      const uint32_t bits = (FULL || j < n) ? (*ring.mslot(sl, lane) >> (j & 31)) : 0u;
      float sh[NV];
#pragma unroll
      for (int e = 0; e < NV; ++e) sh[e] = one_gb * sold[e];
      if (spike_row) {
#pragma unroll
        for (int e = 0; e < NV; ++e)
          if (j + e == j_s) sh[e] += spike_add;
      }
      // coarse keys of the lane's NV columns: k0 for e < NV - 1, k3 for the last (P >= NV)
      int k0 = max(0, (j >> LGP) - 1), k3 = max(0, ((j + NV) >> LGP) - 1);
      if (!FULL) {
        k0 = min(k0, zlen - 2);
        k3 = min(k3, zlen - 2);
      }
      const float z0 = lrow[k0], z1 = lrow[k0 + 1], z3a = lrow[k3], z3b = lrow[k3 + 1];
      float x[2][NV];
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        const float za = e < NV - 1 ? z0 : z3a, zb = e < NV - 1 ? z1 : z3b;
        const float l = w0[e] * za + w1[e] * zb;
        const float d = dv[e];
        const bool obs = (bits >> e) & 1u;
        const float rh = (l + sh[e]) - d;
        const float sn = soft_thr<float>(obs ? sh[e] - rh : sh[e], lam_s);  // cpcp.py:414-415
        x[0][e] = obs ? (l + sn) - d : 0.f;
        x[1][e] = sn;
      }
      float c_sq = 0.f, c_l1 = 0.f, c_ss = 0.f, c_sr = 0.f;
      int c_nnz = 0;
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        const float r = x[0][e], sn = x[1][e];
        c_sq = fmaf(r, r, c_sq);
        c_l1 += fabsf(sn);
        c_nnz += sn != 0.f ? 1 : 0;
        c_ss = fmaf(sn, sn, c_ss);
        c_sr = fmaf(sn, r, c_sr);
      }
      // arg-max |r|, ties to the smallest column-major index: within a lane
      // rows only grow and columns grow within a row, so on a tie the new
      // entry wins iff its column is smaller.  Chunks whose largest |r| is
      // below the running best (nearly all) skip the per-element test.
      float m4 = fabsf(x[0][0]);
#pragma unroll
      for (int e = 1; e < NV; ++e) m4 = fmaxf(m4, fabsf(x[0][e]));
      if (m4 >= bm) {
#pragma unroll
        for (int e = 0; e < NV; ++e) {
          const float r = x[0][e], mg = fabsf(r);
          const bool take = (FULL || j + e < n) && (mg > bm || (mg == bm && j + e < bj));
          bm = take ? mg : bm;
          bval = take ? r : bval;
          bsv = take ? x[1][e] : bsv;
          bj = take ? j + e : bj;
          brow = take ? i : brow;
        }
      }
      a_sq += (double)c_sq;
      a_l1 += (double)c_l1;
      i_nnz += c_nnz;
      a_ss += (double)c_ss;
      a_sr += (double)c_sr;
      row_store<NV, FULL>(sro, j, n, x[1]);
      rr.chunk(w0, w1, x, cbase, outs, lane, LGP);
    };
    if (nfull > 0) {
      float cw0[NV], cw1[NV];
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        cw0[e] = __ldg(w0p + lane * NV + e);
        cw1[e] = __ldg(w1p + lane * NV + e);
      }
      chunk(0, cw0, cw1, std::true_type{});
      for (int c = 1; c < nfull; ++c) chunk(c, rw0, rw1, std::true_type{});
    }
    if (nfull < nc) {
      float t0[NV], t1[NV];
#pragma unroll
      for (int e = 0; e < NV; ++e) {
        const int jt = nfull * CH + lane * NV + e;
        const bool in = jt < n;
        t0[e] = in ? (nfull == 0 ? __ldg(w0p + jt) : rw0[e]) : 0.f;
        t1[e] = in ? (nfull == 0 ? __ldg(w1p + jt) : rw1[e]) : 0.f;
      }
      chunk(nfull, t0, t1, std::false_type{});
    }
    rr.finish(outs, n, np, lane, LGP);
    __syncwarp();
  }
  cp_wait<0>();
  __shared__ double scratch[5 * 32];
  __shared__ AmRecW amw[RW_WARPS];
  double vals[5] = {a_sq, a_l1, (double)i_nnz, a_ss, a_sr};
  block_sum<5>(vals, scratch);
  const long long bidx = brow >= 0 ? (long long)bj * m_global + row0 + brow : -1;
  AmRecW best{bidx >= 0 ? (double)bm : 0.0, (double)bval, (double)bsv, bidx};
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
  const bool reg = rows_reg_ok(p->ch, p->f32);
  if (mode == kCWUpdate && mask && fast_ok(p->ch, p->f32, {ldd, lds}) && p->m_local < INT_MAX) {
    const int nv = fast_nv(p->ch, true);
    const size_t fixed = (size_t)round_up(p->ch.np * 8, 16);
    const bool zpf = fast_zpf(p->ch, fixed, nv);
    const size_t smem = fixed + RW_WARPS * ((zpf ? 2 : 1) * (size_t)round_up(p->ch.np + 2, 4) * 4 + fast_ring_bytes(nv));
    auto pick = [&](auto lgp, auto v) {
      constexpr int L = decltype(lgp)::value, V = decltype(v)::value;
      return zpf ? cp_update_fast<L, true, V> : cp_update_fast<L, false, V>;
    };
    using I4 = std::integral_constant<int, 4>;
    using I8 = std::integral_constant<int, 8>;
    const int lg = p->ch.reg_lgp;
    auto kern = lg == 2   ? pick(std::integral_constant<int, 2>{}, I4{})
                : lg == 3 ? (nv == 8 ? pick(std::integral_constant<int, 3>{}, I8{}) : pick(std::integral_constant<int, 3>{}, I4{}))
                : lg == 4 ? (nv == 8 ? pick(std::integral_constant<int, 4>{}, I8{}) : pick(std::integral_constant<int, 4>{}, I4{}))
                          : (nv == 8 ? pick(std::integral_constant<int, 5>{}, I8{}) : pick(std::integral_constant<int, 5>{}, I4{}));
    MLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = fast_grid(kern, smem, p->row_blocks);
    kern<<<grid, RW_THREADS, smem, st>>>(p->dev, p->ch, (int)p->m_local, p->row0, p->m_global, (const float*)D, ldd,
                                         mask, ldm, (float*)S, lds, (float*)p->LH, (float*)p->GH, (float*)p->SH, p->u,
                                         p->v, p->row_part, p->row_blocks);
    MLR_LAUNCH_CHECK("cp_update_fast");
    return kOk;
  }
  const size_t stage = reg ? 0 : (p->f32 ? SegRestrict<float, 2, 4>::STAGE_BYTES : SegRestrict<double, 2, 2>::STAGE_BYTES);
  const size_t base = (size_t)round_up(p->ch.np * 8, 16) + RW_WARPS * ((size_t)round_up(p->ch.np + 2, 4) * tb + stage);
  const bool ring = base + RW_WARPS * RING_BYTES <= 80 * 1024;
  const size_t smem = base + (ring ? RW_WARPS * RING_BYTES : 0);
  const int blocks = p->row_blocks;
#define MLR_LAUNCH(T, MODE)                                                                                     \
  {                                                                                                             \
    auto kern = reg ? (ring ? cp_rows_warp<T, MODE, true, true> : cp_rows_warp<T, MODE, false, true>)            \
                    : (ring ? cp_rows_warp<T, MODE, true, false> : cp_rows_warp<T, MODE, false, false>);         \
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
