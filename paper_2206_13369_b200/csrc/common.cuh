// Shared device utilities for the multilevel PCP/CPCP hot path (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

namespace mlr {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);

#define MLR_CUDA(call)                                          \
  do {                                                          \
    cudaError_t e_ = (call);                                    \
    if (e_ != cudaSuccess) return ::mlr::cuda_fail(e_, #call);  \
  } while (0)

#define MLR_LAUNCH_CHECK(where)                                 \
  do {                                                          \
    cudaError_t e_ = cudaGetLastError();                        \
    if (e_ != cudaSuccess) return ::mlr::cuda_fail(e_, where);  \
  } while (0)

constexpr int kOk = 0;
constexpr int kErrArg = 1;
constexpr int kErrCuda = 2;

inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
__host__ __device__ __forceinline__ int round_up_dev(int x, int a) { return (x + a - 1) / a * a; }
inline int64_t ceil_div(int64_t x, int64_t a) { return (x + a - 1) / a; }

// ---------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_sumf(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum of NV doubles (deterministic order). `scratch` must hold
// NV * 32 doubles. Result valid in thread 0 only.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = warp_sum(v[q]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) scratch[q * 32 + wid] = v[q];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += scratch[q * 32 + w];
      v[q] = s;
    }
  }
  __syncthreads();
}

// Arg-max record for the l1 oracle: largest |value|, ties broken by the
// smallest column-major index (reference cpcp.py:155-161).
struct ArgMax {
  double mag;     // |r|
  long long idx;  // column-major index j*m + i (global); -1 = empty
  double val;     // signed r at that entry
  double sval;    // S at that entry (needed for the spike terms)
};

__device__ __forceinline__ bool argmax_better(double m1, long long i1, double m2, long long i2) {
  // true if (m1,i1) beats (m2,i2)
  if (i2 < 0) return i1 >= 0;
  if (i1 < 0) return false;
  if (m1 != m2) return m1 > m2;
  return i1 < i2;
}

template <typename T>
__device__ __forceinline__ T soft_thr(T x, T tau) {
  T a = fabs(x) - tau;
  a = a > T(0) ? a : T(0);
  return copysign(a, x);
}

}  // namespace mlr
