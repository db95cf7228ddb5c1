// Micro-benchmark: dependent-chain latency (cycles) of one Jacobi rotation
// (c, s, t from a, b, g) for several formulations, one thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_jrot ubench_jrot.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float rcp_approx(float x) { float r; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
__device__ __forceinline__ float sqrt_approx(float x) { float r; asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
__device__ __forceinline__ float rsqrt_approx(float x) { float r; asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }

template <int V>
__device__ __forceinline__ void rot(double a, double b, double g, double& c, double& s, double& t) {
  if (V == 0) {  // FP64 library
    const double d = b - a, g2 = 2.0 * g;
    const double h = sqrt(fma(d, d, g2 * g2));
    t = g2 / (d >= 0.0 ? d + h : d - h);
    c = rsqrt(fma(t, t, 1.0));
    s = c * t;
  } else {  // FP32 approx seed + FP64 Newton
    const double d = b - a;
    const float df = (float)d, gf = (float)g;
    float hf, tf, rf;
    if (V == 1) {
      hf = sqrtf(fmaf(df, df, 4.f * gf * gf));
      tf = (2.f * gf) / (df >= 0.f ? df + hf : df - hf);
      rf = __frcp_rn(fmaf(2.f * gf, tf, df));
    } else {
      hf = sqrt_approx(fmaf(df, df, 4.f * gf * gf));
      tf = (2.f * gf) * rcp_approx(df >= 0.f ? df + hf : df - hf);
      rf = rcp_approx(fmaf(2.f * gf, tf, df));
    }
    double t0 = (double)tf;
    const double f = fma(g * t0, t0, fma(d, t0, -g));
    t0 = fma(-f, (double)rf, t0);
    if (V == 3) {  // second Newton step
      const double f2 = fma(g * t0, t0, fma(d, t0, -g));
      t0 = fma(-f2, (double)rf, t0);
    }
    t = t0;
    const double x = fma(t0, t0, 1.0);
    double y = (double)(V == 1 ? rsqrtf((float)x) : rsqrt_approx((float)x));
    y = y * fma(-0.5 * x * y, y, 1.5);
    y = y * fma(-0.5 * x * y, y, 1.5);
    c = y;
    s = y * t0;
  }
}

template <int V>
__global__ void chain(double a0, double b0, double g0, int n, long long* cyc, double* out) {
  double a = a0, b = b0, g = g0, acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double c, s, t;
    rot<V>(a, b, g, c, s, t);
    acc += c;
    g = g0 + 1e-30 * s;  // dependence
    a = a0 + 1e-30 * t;
  }
  long long t1 = clock64();
  cyc[0] = t1 - t0;
  out[0] = acc;
}

template <int V>
void run(const char* name) {
  long long* dc; double* dout; cudaMalloc(&dc, 8); cudaMalloc(&dout, 8);
  chain<V><<<1, 1>>>(1.0, 2.5, 0.3, 100, dc, dout);
  chain<V><<<1, 1>>>(1.0, 2.5, 0.3, 10000, dc, dout);
  long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  // accuracy vs the FP64 library on a sweep of inputs
  printf("%-40s %6.0f cycles/rotation\n", name, c / 10000.0);
}

template <int V>
__global__ void acc_kernel(double* err) {
  double e = 0, eo = 0;
  for (int i = 0; i < 4096; ++i) {
    const double a = 1.0 + i * 0.37, b = 0.5 + (i % 97) * 1.3, g = (i % 13 - 6) * 1e-3 * (1 + i % 5);
    if (g == 0.0) continue;
    double c0, s0, t0, c, s, t;
    rot<0>(a, b, g, c0, s0, t0);
    rot<V>(a, b, g, c, s, t);
    e = fmax(e, fabs(t - t0) / fabs(t0));
    eo = fmax(eo, fabs(c * c + s * s - 1.0));
  }
  err[0] = e; err[1] = eo;
}
template <int V>
void acc(const char* name) {
  double* d; cudaMalloc(&d, 16); acc_kernel<V><<<1, 1>>>(d); double h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("%-40s rel err t %.2e  |c^2+s^2-1| %.2e\n", name, h[0], h[1]);
}

int main() {
  run<0>("FP64 sqrt/div/rsqrt");
  run<1>("FP32 IEEE seed + FP64 Newton");
  run<2>("FP32 approx seed + FP64 Newton");
  run<3>("FP32 approx seed + 2 FP64 Newton");
  acc<1>("FP32 IEEE seed + FP64 Newton");
  acc<2>("FP32 approx seed + FP64 Newton");
  acc<3>("FP32 approx seed + 2 FP64 Newton");
  return 0;
}
