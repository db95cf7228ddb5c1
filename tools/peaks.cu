// Peak-throughput microbenchmarks for the roofline denominators that
// MEASURED_PEAKS.json does not carry: FP64 tensor-core MMA (the
// mma.sync.m8n8k4.f64 path the Gram / reconstruction / coarse products use),
// FP32 FFMA and FP64 DFMA SIMT.  Prints one JSON object.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks tools/peaks.cu && tools/peaks
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));    \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

constexpr int kIters = 4096;
constexpr int kAcc = 8;  // independent accumulator chains per warp / thread

__global__ void dmma_kernel(double* out, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = seed - threadIdx.x * 1e-3;
  double c[kAcc][2];
#pragma unroll
  for (int q = 0; q < kAcc; ++q) c[q][0] = c[q][1] = 0.0;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int q = 0; q < kAcc; ++q)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[q][0]), "+d"(c[q][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < kAcc; ++q) s += c[q][0] + c[q][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dfma_kernel(double* out, double seed) {
  double x[kAcc];
#pragma unroll
  for (int q = 0; q < kAcc; ++q) x[q] = seed + q;
  const double m = 0.999999, add = 1e-7;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int q = 0; q < kAcc; ++q) x[q] = fma(x[q], m, add);
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < kAcc; ++q) s += x[q];
  if (s == 12345.678) out[0] = s;
}

__global__ void ffma_kernel(float* out, float seed) {
  float x[kAcc];
#pragma unroll
  for (int q = 0; q < kAcc; ++q) x[q] = seed + q;
  const float m = 0.999999f, add = 1e-7f;
  for (int it = 0; it < kIters; ++it)
#pragma unroll
    for (int q = 0; q < kAcc; ++q) x[q] = fmaf(x[q], m, add);
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < kAcc; ++q) s += x[q];
  if (s == 12345.678f) out[0] = s;
}

// tcgen05.mma.kind::tf32 issue-bound loop: one elected thread per CTA
// issues M128 N256 K8 MMAs on fixed (zero) shared-memory operands into one
// TMEM accumulator, then commits; 2 x 128 x 256 x 8 flops per MMA.
constexpr int kTcIters = 8192;
__global__ void __launch_bounds__(128, 1) tc_tf32_kernel(float* out) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < (128 + 256) * 32; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  const uint32_t s_a = (uint32_t)__cvta_generic_to_shared(sm), s_b = s_a + 128 * 32 * 4;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    auto desc = [](uint32_t a) {
      return (uint64_t)((a & 0x3FFFF) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
    };
    const uint64_t da = desc(s_a), db = desc(s_b);
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (32u << 17) | (8u << 24);
    for (int it = 0; it < kTcIters; ++it)
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tbase),
          "l"(da + 2 * (it & 3)), "l"(db + 2 * (it & 3)), "r"(idesc), "r"(it > 0 ? 1u : 0u));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile(
        "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&bar)));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
  }
  if (threadIdx.x == 0 && out) out[blockIdx.x] = 0.f;
}

template <typename K>
float time_ms(K launch, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  double* d;
  CK(cudaMalloc(&d, 64));
  const int sms = p.multiProcessorCount;
  // DMMA: 512 flops per warp instruction
  double best_dmma = 0.0;
  for (int warps = 4; warps <= 32; warps *= 2) {
    const int blocks = sms * 2, threads = 32 * warps / 2;
    float ms = time_ms([&] { dmma_kernel<<<blocks, threads>>>(d, 1.0); }, 5);
    double flops = (double)blocks * (threads / 32) * kIters * kAcc * 512.0;
    double tf = flops / (ms * 1e-3) / 1e12;
    if (tf > best_dmma) best_dmma = tf;
  }
  CK(cudaGetLastError());
  double best_dfma = 0.0, best_ffma = 0.0;
  for (int threads = 256; threads <= 1024; threads *= 2) {
    const int blocks = sms * (2048 / threads);
    float ms = time_ms([&] { dfma_kernel<<<blocks, threads>>>(d, 1.0); }, 5);
    double tf = (double)blocks * threads * kIters * kAcc * 2.0 / (ms * 1e-3) / 1e12;
    if (tf > best_dfma) best_dfma = tf;
    ms = time_ms([&] { ffma_kernel<<<blocks, threads>>>((float*)d, 1.f); }, 5);
    tf = (double)blocks * threads * kIters * kAcc * 2.0 / (ms * 1e-3) / 1e12;
    if (tf > best_ffma) best_ffma = tf;
  }
  CK(cudaGetLastError());
  const size_t tsm = (128 + 256) * 32 * 4 + 1024;
  CK(cudaFuncSetAttribute(tc_tf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
  float tms = time_ms([&] { tc_tf32_kernel<<<sms, 128, tsm>>>((float*)d); }, 5);
  CK(cudaGetLastError());
  const double tf32 = (double)sms * kTcIters * 2.0 * 128 * 256 * 8 / (tms * 1e-3) / 1e12;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"max_sm_mhz\": %d, \"fp64_mma_tflops\": %.2f, "
         "\"fp64_dfma_tflops\": %.2f, \"fp32_ffma_tflops\": %.2f, \"tf32_tc_tflops\": %.1f, \"method\": "
         "\"tools/peaks.cu: %d-deep independent chains per warp/thread, best over occupancies; tcgen05 kind::tf32 "
         "M128 N256 K8 issue loop, one CTA per SM; CUDA events\"}\n",
         p.name, sms, clk / 1000, best_dmma, best_dfma, best_ffma, tf32, kAcc);
  return 0;
}
