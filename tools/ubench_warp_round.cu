// Micro-benchmark: cycles per Jacobi cross round on a 32x32 FP64 tile.
//   variant 0: 16 threads compute the rotations, 2 barriers per round
//   variant 1: every thread recomputes the 2 rotations it needs, 1 barrier
//   variant 2: as 1 with the FP32-seeded / FP64-Newton rotation
// and the max deviation from the reference rotation (variant 0).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_warp_round ubench_warp_round.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int PW = 32, BW = 16, LD = 33;

__device__ __forceinline__ void jrot_lib(double a, double b, double g, double& c, double& s, double& t) {
  const double d = b - a, g2 = 2.0 * g;
  const double h = sqrt(fma(d, d, g2 * g2));
  t = g2 / (d >= 0.0 ? d + h : d - h);
  c = rsqrt(fma(t, t, 1.0));
  s = c * t;
}

// t solves g t^2 + d t - g = 0 (smaller root); FP32 seed, one FP64 Newton
// step with an FP32 reciprocal of f'; c = (1+t^2)^-1/2 by FP32 seed + 2 FP64
// Newton steps.
__device__ __forceinline__ void jrot_fast(double a, double b, double g, double& c, double& s, double& t) {
  const double d = b - a;
  const float df = (float)d, gf = (float)g;
  const float hf = sqrtf(fmaf(df, df, 4.f * gf * gf));
  const float tf = (2.f * gf) / (df >= 0.f ? df + hf : df - hf);
  double t0 = (double)tf;
  const double f = fma(g * t0, t0, fma(d, t0, -g));
  const float fp = fmaf(2.f * gf, tf, df);
  t0 = fma(-f, (double)__frcp_rn(fp), t0);
  t = t0;
  const double x = fma(t0, t0, 1.0);
  double y = (double)rsqrtf((float)x);
  y = y * fma(-0.5 * x * y, y, 1.5);
  y = y * fma(-0.5 * x * y, y, 1.5);
  c = y;
  s = y * t0;
}

template <int V>
__device__ __forceinline__ void jrot(double a, double b, double g, double& c, double& s, double& t) {
  c = 1.0; s = 0.0; t = 0.0;
  if (!(fabs(g) > 1e-300 && g * g > 1e-28 * fabs(a * b))) return;
  if (V == 2) jrot_fast(a, b, g, c, s, t); else jrot_lib(a, b, g, c, s, t);
}

template <int V, int NT>
__global__ void rounds(const double* Gin, int nrounds, long long* cycles, double* out) {
  __shared__ double G[PW][LD];
  __shared__ double2 cs[16];
  __shared__ double tt[16];
  const int tid = threadIdx.x;
  for (int e = tid; e < PW * PW; e += NT) G[e >> 5][e & 31] = Gin[e];
  __syncthreads();
  long long t0 = clock64();
  for (int rnd = 0; rnd < nrounds; ++rnd) {
    const int q = tid & 15;
    const int q1 = q, q2 = BW + ((q + rnd) & 15);
    double cq, sq, tq;
    if (V == 0) {
      if (tid < 16) {
        const int i = tid, j = BW + ((tid + rnd) & 15);
        double c, s, t;
        jrot<0>(G[i][i], G[j][j], G[i][j], c, s, t);
        cs[tid] = make_double2(c, s);
        tt[tid] = t;
      }
      __syncthreads();
      cq = cs[q].x; sq = cs[q].y; tq = tt[q];
    } else {
      jrot<V>(G[q1][q1], G[q2][q2], G[q1][q2], cq, sq, tq);
    }
    double o[16 / (2 * (NT / 32))][4];
#pragma unroll
    for (int u = 0; u < 16 / (2 * (NT / 32)); ++u) {
      const int pp = (tid >> 4) + 2 * (NT / 32) * u;
      const int p1 = pp, p2 = BW + ((pp + rnd) & 15);
      double cp, sp, tp;
      if (V == 0) { cp = cs[pp].x; sp = cs[pp].y; tp = tt[pp]; }
      else jrot<V>(G[p1][p1], G[p2][p2], G[p1][p2], cp, sp, tp);
      const double g11 = G[p1][q1], g12 = G[p1][q2], g21 = G[p2][q1], g22 = G[p2][q2];
      if (pp == q && tp != 0.0) {
        o[u][0] = g11 - tp * g12; o[u][3] = g22 + tp * g12; o[u][1] = 0.0; o[u][2] = 0.0;
      } else {
        const double t11 = cq * g11 - sq * g12, t12 = sq * g11 + cq * g12;
        const double t21 = cq * g21 - sq * g22, t22 = sq * g21 + cq * g22;
        o[u][0] = cp * t11 - sp * t21; o[u][1] = cp * t12 - sp * t22;
        o[u][2] = sp * t11 + cp * t21; o[u][3] = sp * t12 + cp * t22;
      }
    }
    if (V != 0) __syncthreads();  // everyone has read G for this round
#pragma unroll
    for (int u = 0; u < 16 / (2 * (NT / 32)); ++u) {
      const int pp = (tid >> 4) + 2 * (NT / 32) * u;
      const int p1 = pp, p2 = BW + ((pp + rnd) & 15);
      G[p1][q1] = o[u][0]; G[p1][q2] = o[u][1]; G[p2][q1] = o[u][2]; G[p2][q2] = o[u][3];
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cycles[blockIdx.x] = t1 - t0;
  for (int e = tid; e < PW * PW; e += NT) out[e] = G[e >> 5][e & 31];
}

template <int V, int NT>
void run(const double* dG, long long* dc, double* dout, double* ref, int nr) {
  rounds<V, NT><<<1, NT>>>(dG, 16, dc, dout);
  rounds<V, NT><<<1, NT>>>(dG, nr, dc, dout);
  long long c;
  double h[PW * PW];
  cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(h, dout, sizeof(h), cudaMemcpyDeviceToHost);
  double dev = 0;
  if (ref) for (int e = 0; e < PW * PW; ++e) dev = fmax(dev, fabs(h[e] - ref[e]));
  else for (int e = 0; e < PW * PW; ++e) ref ? 0 : 0;
  printf("variant %d threads %d: %.0f cycles/round  max|G - G_ref| %.2e\n", V, NT, (double)c / nr, dev);
}

int main() {
  double h[PW * PW], ref[PW * PW];
  for (int i = 0; i < PW; ++i)
    for (int j = 0; j < PW; ++j) h[i * PW + j] = (i == j) ? 10.0 + i : 1e-2 / (1 + i + j);
  double *dG, *dout;
  long long* dc;
  cudaMalloc(&dG, sizeof(h)); cudaMalloc(&dout, sizeof(h)); cudaMalloc(&dc, 64);
  cudaMemcpy(dG, h, sizeof(h), cudaMemcpyHostToDevice);
  const int nr = 1600;
  run<0, 256>(dG, dc, dout, nullptr, nr);
  cudaMemcpy(ref, dout, sizeof(ref), cudaMemcpyDeviceToHost);
  run<0, 128>(dG, dc, dout, ref, nr);
  run<1, 256>(dG, dc, dout, ref, nr);
  run<1, 128>(dG, dc, dout, ref, nr);
  run<2, 256>(dG, dc, dout, ref, nr);
  run<2, 128>(dG, dc, dout, ref, nr);
  return 0;
}
