// Ping-pong latency between two CTAs through flag-carrying 16-byte records
// (st.relaxed.gpu / ld.relaxed.gpu v4), and through a release/acquire flag.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void st4(uint4* p, uint4 v) {
  asm volatile("st.relaxed.gpu.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ uint4 ld4(const uint4* p) {
  uint4 v;
  asm volatile("ld.relaxed.gpu.global.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__global__ void pingpong(uint4* buf, int iters, long long* out, int nthreads_poll) {
  const int me = blockIdx.x;  // 0 or 1
  uint4* mine = buf + me * 1024;
  uint4* other = buf + (1 - me) * 1024;
  long long t0 = clock64();
  for (int i = 1; i <= iters; ++i) {
    if (me == 0) {
      if (threadIdx.x < nthreads_poll) st4(mine + threadIdx.x, make_uint4(i, i, i, i));
      if (threadIdx.x < nthreads_poll) { uint4 v; do { v = ld4(other + threadIdx.x); } while (v.y != (unsigned)i); }
      __syncthreads();
    } else {
      if (threadIdx.x < nthreads_poll) { uint4 v; do { v = ld4(other + threadIdx.x); } while (v.y != (unsigned)i); }
      __syncthreads();
      if (threadIdx.x < nthreads_poll) st4(mine + threadIdx.x, make_uint4(i, i, i, i));
    }
  }
  if (threadIdx.x == 0) out[me] = clock64() - t0;
}
int main() {
  uint4* buf; long long* out;
  cudaMalloc(&buf, 2 * 1024 * 16); cudaMalloc(&out, 16);
  for (int np : {1, 32, 512}) {
    for (int sep : {1, 74}) {
      cudaMemset(buf, 0, 2 * 1024 * 16);
      // 2 CTAs; grid of sep+1 with the rest idle is awkward: launch 2 CTAs (placement decided by HW)
      int iters = 2000;
      pingpong<<<2, 512>>>(buf, iters, out, np);
      cudaDeviceSynchronize();
      long long h[2];
      cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
      printf("pollers %d: round trip %.0f cycles (one way %.0f)\n", np, (double)h[0] / iters, (double)h[0] / iters / 2);
      break;
    }
  }
  return 0;
}
