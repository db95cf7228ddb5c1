// Micro-benchmark: latency of one Jacobi inner round (params + 2x2 block
// update of a 32x32 FP64 Gram + Q update) in one CTA, for several variants.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench ubench_rounds.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int PW = 32, BW = 16, LD = 36, T = 256;

template <int MODE>
__device__ __forceinline__ void rot(double a, double b, double g, double& c, double& s, double& t) {
  if (MODE == 0) {  // FP64 sqrt/div/rsqrt
    const double d = b - a, g2 = 2.0 * g;
    const double h = sqrt(fma(d, d, g2 * g2));
    t = g2 / (d >= 0.0 ? d + h : d - h);
    c = rsqrt(fma(t, t, 1.0));
    s = c * t;
  } else if (MODE == 1) {  // FP32 math only
    const float d = (float)(b - a), g2 = (float)(2.0 * g);
    const float h = sqrtf(fmaf(d, d, g2 * g2));
    const float tf = __fdividef(g2, d >= 0.f ? d + h : d - h);
    const float cf = rsqrtf(fmaf(tf, tf, 1.f));
    t = tf;
    c = cf;
    s = cf * tf;
  } else {  // no math
    t = 1e-3 * g;
    c = 1.0;
    s = t;
  }
}

template <int MODE>
__global__ void rounds_kernel(const double* Gin, int nrounds, long long* cycles, double* sink) {
  __shared__ double G[PW][LD], Q[PW][LD], cs[16][3];
  __shared__ int pr[16][2];
  const int tid = threadIdx.x;
  for (int e = tid; e < PW * PW; e += T) {
    G[e >> 5][e & 31] = Gin[e];
    Q[e >> 5][e & 31] = (e >> 5) == (e & 31);
  }
  __syncthreads();
  long long t0 = clock64();
  for (int rnd = 0; rnd < nrounds; ++rnd) {
    if (tid < 16) {
      const int i = tid, j = BW + ((tid + rnd) & 15);
      const double a = G[i][i], b = G[j][j], g = G[i][j];
      double c = 1.0, s = 0.0, t = 0.0;
      if (fabs(g) > 1e-300 && g * g > 1e-28 * fabs(a * b)) rot<MODE>(a, b, g, c, s, t);
      cs[tid][0] = c; cs[tid][1] = s; cs[tid][2] = t;
      pr[tid][0] = i; pr[tid][1] = j;
    }
    __syncthreads();
    {
      const int p = tid >> 4, q = tid & 15;
      const int p1 = pr[p][0], p2 = pr[p][1], q1 = pr[q][0], q2 = pr[q][1];
      const double cp = cs[p][0], sp = cs[p][1], cq = cs[q][0], sq = cs[q][1];
      const double g11 = G[p1][q1], g12 = G[p1][q2], g21 = G[p2][q1], g22 = G[p2][q2];
      if (p == q && cs[p][2] != 0.0) {
        const double t = cs[p][2];
        G[p1][p1] = g11 - t * g12; G[p2][p2] = g22 + t * g12; G[p1][p2] = 0.0; G[p2][p1] = 0.0;
      } else {
        const double t11 = cq * g11 - sq * g12, t12 = sq * g11 + cq * g12;
        const double t21 = cq * g21 - sq * g22, t22 = sq * g21 + cq * g22;
        G[p1][q1] = cp * t11 - sp * t21; G[p1][q2] = cp * t12 - sp * t22;
        G[p2][q1] = sp * t11 + cp * t21; G[p2][q2] = sp * t12 + cp * t22;
      }
    }
#pragma unroll
    for (int q4 = 0; q4 < 2; ++q4) {
      const int e = tid + q4 * T;
      const int r = e >> 4, q = e & 15;
      const int q1 = pr[q][0], q2 = pr[q][1];
      const double c = cs[q][0], s = cs[q][1];
      const double a = Q[r][q1], b = Q[r][q2];
      Q[r][q1] = c * a - s * b; Q[r][q2] = s * a + c * b;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cycles[blockIdx.x] = t1 - t0;
  if (tid == 0) sink[blockIdx.x] = G[3][5] + Q[7][9];
}

// Single-barrier round: thread (p, q) recomputes the rotations of pairs p
// and q itself, reads G/Q from buffer `cur` and writes buffer `cur^1`.
template <int MODE>
__global__ void rounds1_kernel(const double* Gin, int nrounds, long long* cycles, double* sink) {
  __shared__ double G[2][PW][LD], Q[2][PW][LD];
  const int tid = threadIdx.x;
  for (int e = tid; e < PW * PW; e += T) {
    G[0][e >> 5][e & 31] = Gin[e];
    Q[0][e >> 5][e & 31] = (e >> 5) == (e & 31);
  }
  __syncthreads();
  const int p = tid >> 4, q = tid & 15;
  long long t0 = clock64();
  int cur = 0;
  for (int rnd = 0; rnd < nrounds; ++rnd) {
    const int p1 = p, p2 = BW + ((p + rnd) & 15), q1 = q, q2 = BW + ((q + rnd) & 15);
    const double (*g)[LD] = G[cur];
    const double ap = g[p1][p1], bp = g[p2][p2], gp = g[p1][p2];
    const double aq = g[q1][q1], bq = g[q2][q2], gq = g[q1][q2];
    const double g11 = g[p1][q1], g12 = g[p1][q2], g21 = g[p2][q1], g22 = g[p2][q2];
    const double (*qq)[LD] = Q[cur];
    const double x11 = qq[p1][q1], x12 = qq[p1][q2], x21 = qq[p2][q1], x22 = qq[p2][q2];
    double cp = 1.0, sp = 0.0, tp = 0.0, cq = 1.0, sq = 0.0, tq = 0.0;
    if (fabs(gp) > 1e-300 && gp * gp > 1e-28 * fabs(ap * bp)) rot<MODE>(ap, bp, gp, cp, sp, tp);
    if (fabs(gq) > 1e-300 && gq * gq > 1e-28 * fabs(aq * bq)) rot<MODE>(aq, bq, gq, cq, sq, tq);
    double (*gn)[LD] = G[cur ^ 1];
    if (p == q && tp != 0.0) {
      gn[p1][p1] = g11 - tp * g12; gn[p2][p2] = g22 + tp * g12; gn[p1][p2] = 0.0; gn[p2][p1] = 0.0;
    } else {
      const double t11 = cq * g11 - sq * g12, t12 = sq * g11 + cq * g12;
      const double t21 = cq * g21 - sq * g22, t22 = sq * g21 + cq * g22;
      gn[p1][q1] = cp * t11 - sp * t21; gn[p1][q2] = cp * t12 - sp * t22;
      gn[p2][q1] = sp * t11 + cp * t21; gn[p2][q2] = sp * t12 + cp * t22;
    }
    double (*qn)[LD] = Q[cur ^ 1];
    qn[p1][q1] = cq * x11 - sq * x12; qn[p1][q2] = sq * x11 + cq * x12;
    qn[p2][q1] = cq * x21 - sq * x22; qn[p2][q2] = sq * x21 + cq * x22;
    cur ^= 1;
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cycles[blockIdx.x] = t1 - t0;
  if (tid == 0) sink[blockIdx.x] = G[cur][3][5] + Q[cur][7][9];
}

// Barrier-only and FP32-data variants of the 2-sync round (cost attribution).
template <typename TT, int WORK>
__global__ void rounds2_kernel(const double* Gin, int nrounds, long long* cycles, double* sink) {
  __shared__ TT G[PW][LD], Q[PW][LD];
  __shared__ TT cs[16][2];
  const int tid = threadIdx.x;
  for (int e = tid; e < PW * PW; e += T) {
    G[e >> 5][e & 31] = (TT)Gin[e];
    Q[e >> 5][e & 31] = (e >> 5) == (e & 31);
  }
  __syncthreads();
  long long t0 = clock64();
  for (int rnd = 0; rnd < nrounds; ++rnd) {
    if (WORK && tid < 16) {
      const int i = tid, j = BW + ((tid + rnd) & 15);
      const TT a = G[i][i], b = G[j][j], g = G[i][j];
      cs[tid][0] = a * (TT)0.999 + g * (TT)1e-3;
      cs[tid][1] = b * (TT)1e-3;
    }
    __syncthreads();
    if (WORK) {
      const int p = tid >> 4, q = tid & 15;
      const int p1 = p, p2 = BW + ((p + rnd) & 15), q1 = q, q2 = BW + ((q + rnd) & 15);
      const TT cp = cs[p][0], sp = cs[p][1], cq = cs[q][0], sq = cs[q][1];
      const TT g11 = G[p1][q1], g12 = G[p1][q2], g21 = G[p2][q1], g22 = G[p2][q2];
      const TT x11 = Q[p1][q1], x12 = Q[p1][q2], x21 = Q[p2][q1], x22 = Q[p2][q2];
      const TT t11 = cq * g11 - sq * g12, t12 = sq * g11 + cq * g12;
      const TT t21 = cq * g21 - sq * g22, t22 = sq * g21 + cq * g22;
      G[p1][q1] = cp * t11 - sp * t21; G[p1][q2] = cp * t12 - sp * t22;
      G[p2][q1] = sp * t11 + cp * t21; G[p2][q2] = sp * t12 + cp * t22;
      Q[p1][q1] = cq * x11 - sq * x12; Q[p1][q2] = sq * x11 + cq * x12;
      Q[p2][q1] = cq * x21 - sq * x22; Q[p2][q2] = sq * x21 + cq * x22;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cycles[blockIdx.x] = t1 - t0;
  if (tid == 0) sink[blockIdx.x] = (double)(G[3][5] + Q[7][9]);
}

int main() {
  double hG[PW * PW];
  for (int i = 0; i < PW; ++i)
    for (int j = 0; j < PW; ++j) hG[i * PW + j] = (i == j) ? 10.0 + i : 1.0 / (1.0 + i + j);
  double *dG, *sink;
  long long* cyc;
  cudaMalloc(&dG, sizeof(hG));
  cudaMalloc(&sink, 8 * 8);
  cudaMalloc(&cyc, 8 * 8);
  cudaMemcpy(dG, hG, sizeof(hG), cudaMemcpyHostToDevice);
  const int n = 160;
  long long h = 0;
  for (int rep = 0; rep < 2; ++rep) {
    rounds_kernel<0><<<1, T>>>(dG, n, cyc, sink);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("FP64 params   : %.1f cycles/round\n", (double)h / n);
    rounds_kernel<1><<<1, T>>>(dG, n, cyc, sink);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("FP32 params   : %.1f cycles/round\n", (double)h / n);
    rounds_kernel<2><<<1, T>>>(dG, n, cyc, sink);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("no-math params: %.1f cycles/round\n", (double)h / n);
    rounds1_kernel<0><<<1, T>>>(dG, n, cyc, sink);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("1-sync FP64   : %.1f cycles/round\n", (double)h / n);
    rounds1_kernel<1><<<1, T>>>(dG, n, cyc, sink);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("1-sync FP32   : %.1f cycles/round\n", (double)h / n);
    rounds1_kernel<2><<<1, T>>>(dG, n, cyc, sink);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("1-sync nomath : %.1f cycles/round\n", (double)h / n);
    rounds2_kernel<double, 0><<<1, T>>>(dG, n, cyc, sink);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("2 barriers only: %.1f cycles/round\n", (double)h / n);
    rounds2_kernel<double, 1><<<1, T>>>(dG, n, cyc, sink);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("2-sync fp64 data, trivial params: %.1f cycles/round\n", (double)h / n);
    rounds2_kernel<float, 1><<<1, T>>>(dG, n, cyc, sink);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("2-sync fp32 data, trivial params: %.1f cycles/round\n", (double)h / n);
  }
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
