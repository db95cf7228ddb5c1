// Two-sided block Jacobi eigensolver for the coarse SVT (replaces gesdd in
// svd_full, reference linalg.py:86-99, as called by pcp.py:257).
//
// Input: B (np x np, symmetric PSD, row-major, FP64) already rotated into
// the previous iteration's eigenbasis (B~ = V0^T B V0, the warm start) and
// V = V0.  Output: B diagonal (eigenvalues on the diagonal) and V = V0 J.
//
// Columns are grouped in blocks of 16; a round-robin tournament over the
// nb = np/16 blocks pairs them, npairs = nb/2 pairs per step.  Step 0 of a
// sweep pairs (2k, 2k+1) and runs a full cyclic inner sweep (31 rounds of 16
// disjoint 2x2 rotations) on each 32x32 diagonal sub-block, which also
// clears the intra-block pairs; steps 1..nb-1 run the 16 cross rounds
// (i, 16+(i+r)%16).  Each step:
//   phase A  pair owner k: load the 32x32 sub-block G of B; rotate; rotated
//            pairs are zeroed exactly with the classical diagonal update
//            (a - t g, b + t g) so tiny eigenvalues next to large ones do not
//            stagnate; publish Q_k and the rotated G_k              -- barrier
//   phase B  all CTAs: B[pq_k1, pq_k2] <- Q_k1^T B[..] Q_k2 (k1 < k2, plus
//            the mirror), B[pq_k, pq_k] <- G_k, V[rows, pq_k] <- V[rows, pq_k] Q_k
//                                                                   -- barrier
// Barriers are cluster barriers when the solve fits one 16-CTA cluster
// (np <= 512), grid barriers (cooperative launch) otherwise.
// Convergence: over a sweep every inspected pair has |g_ij| <= abs_floor or
// |g_ij| <= tol * sqrt(|g_ii g_jj|).
#include <cooperative_groups.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace mlr {

constexpr int J2_BW = 16, J2_PW = 32, J2_THREADS = 256, J2_LD = J2_PW + 4;

struct J2Smem {
  double G[J2_PW][J2_LD];
  double Q[J2_PW][J2_LD];
  double X[J2_PW][J2_LD];
  double Y[J2_PW][J2_LD];
  double Q2[J2_PW][J2_LD];
  double G2[J2_PW][J2_LD];       // ping-pong partner of G in the pipelined rounds
  double2 csb[2][J2_PW / 2];     // (c, s) of rounds rnd, rnd + 1
  double ttb[2][J2_PW / 2];      // t of rounds rnd, rnd + 1
  double cs[J2_PW / 2][3];  // c, s, t
  double2 csl[J2_PW][J2_PW / 2];  // rotation log of the inner rounds, replayed into Q
  int pr[J2_PW / 2][2];
  int rotated;
  int active;             // any pair of this block above tolerance
  int round_rot[J2_PW];   // per inner round: any rotation applied
  int qf[2];
  double red[32];
};

// Rotation (c, s, t) that annihilates g in [[a, g], [g, b]]:
// z = (b - a) / 2g, t = sign(z) / (|z| + sqrt(1 + z^2)), c = 1/sqrt(1+t^2).
// FP32 estimates refined by Newton steps in FP64; c and s share t, so the
// rotation is orthogonal to FP64 precision.
// Written without z = (b-a)/2g: with d = b - a and h = sqrt(d^2 + 4 g^2),
// t = 2g / (d + sign(d) h) — one sqrt, one division, one rsqrt on the
// critical path of every inner round.
__device__ __forceinline__ void jac_rot(double a, double b, double g, double& c, double& s, double& t) {
  const double d = b - a, g2 = 2.0 * g;
  const double h = sqrt(fma(d, d, g2 * g2));
  t = g2 / (d >= 0.0 ? d + h : d - h);
  c = rsqrt(fma(t, t, 1.0));
  s = c * t;
}

// One 2x2 block of G <- J^T G J: rows {p1, p2} rotated by (cp, sp), columns
// {q1, q2} by (cq, sq).  Explicit FMAs: the pipelined rounds recompute some
// of these entries in the rotation warp and must match bit for bit.
struct Blk {
  double o11, o12, o21, o22;
};
__device__ __forceinline__ Blk j2_block(double cp, double sp, double cq, double sq, double g11, double g12,
                                        double g21, double g22) {
  const double t11 = fma(cq, g11, -sq * g12), t12 = fma(sq, g11, cq * g12);
  const double t21 = fma(cq, g21, -sq * g22), t22 = fma(sq, g21, cq * g22);
  return Blk{fma(cp, t11, -sp * t21), fma(cp, t12, -sp * t22), fma(sp, t11, cp * t21), fma(sp, t12, cp * t22)};
}
// classical diagonal update of the rotated pair itself
__device__ __forceinline__ double j2_diag_lo(double t, double g, double a) { return fma(-t, g, a); }
__device__ __forceinline__ double j2_diag_hi(double t, double g, double b) { return fma(t, g, b); }

__device__ __forceinline__ void j2_pair(int step, int k, int nb, int& pa, int& pb) {
  if (step == 0) {
    pa = 2 * k;
    pb = 2 * k + 1;
    return;
  }
  const int m = nb - 1, t = step - 1;
  if (k == 0) {
    pa = t;
    pb = m;
  } else {
    pa = (t + k) % m;
    pb = (t - k + m) % m;
  }
}

__device__ __forceinline__ int j2_col(int l, int pa, int pb) {
  return l < J2_BW ? pa * J2_BW + l : pb * J2_BW + (l - J2_BW);
}

__device__ __forceinline__ void atomic_max_nonneg2(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

constexpr int J2_DF_MAXB = 128;  // dflow limit on the number of 16-blocks

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <bool CLUSTER>
__device__ __forceinline__ void j2_sync() {
  if (CLUSTER) cg::this_cluster().sync();
  else cg::this_grid().sync();
}

// Load a 32x32 tile whose rows/cols are the two 16-blocks of a pair.
__device__ __forceinline__ void load_pair_tile(double (*dst)[J2_LD], const double* __restrict__ src, int np,
                                               int ra, int rb, int ca, int cb) {
  double v[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = threadIdx.x + q * J2_THREADS;
    const int i = e >> 5, j = e & 31;
    v[q] = src[(int64_t)j2_col(i, ra, rb) * np + j2_col(j, ca, cb)];
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = threadIdx.x + q * J2_THREADS;
    dst[e >> 5][e & 31] = v[q];
  }
}

__device__ __forceinline__ void load_dense_tile(double (*dst)[J2_LD], const double* __restrict__ src) {
  double v[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) v[q] = src[threadIdx.x + q * J2_THREADS];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = threadIdx.x + q * J2_THREADS;
    dst[e >> 5][e & 31] = v[q];
  }
}

__device__ __forceinline__ void j2_dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// 32x32 tile product op(A) * B on the FP64 DMMA path (mma.sync m8n8k4):
// warp w owns rows 8*(w>>1)..+8 and columns 16*(w&1)..+16 (two 8x8 tiles).
// Output element q (0..3) of the calling thread sits at (tm_row(), tm_col(q)).
__device__ __forceinline__ int tm_row() { return 8 * ((threadIdx.x >> 5) >> 1) + ((threadIdx.x & 31) >> 2); }
__device__ __forceinline__ int tm_col(int q) {
  return 16 * ((threadIdx.x >> 5) & 1) + 8 * (q >> 1) + 2 * (threadIdx.x & 3) + (q & 1);
}

template <bool TA>
__device__ __forceinline__ void tile_mm(const double (*A)[J2_LD], const double (*B)[J2_LD], double (&o)[4]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r = 8 * (w >> 1) + (lane >> 2);  // A fragment row
  const int kk = lane & 3;
  const int c0 = 16 * (w & 1) + (lane >> 2);  // B fragment column (tile 0)
  o[0] = o[1] = o[2] = o[3] = 0.0;
#pragma unroll
  for (int k4 = 0; k4 < J2_PW; k4 += 4) {
    const double a = TA ? A[k4 + kk][r] : A[r][k4 + kk];
    const double b0 = B[k4 + kk][c0], b1 = B[k4 + kk][c0 + 8];
    j2_dmma(o[0], o[1], a, b0);
    j2_dmma(o[2], o[3], a, b1);
  }
}

template <typename Smem>
__device__ __forceinline__ void j2_item_compute(Smem& S, double* __restrict__ B, int np, int a1, int b1, int a2,
                                                int b2, bool ra, bool rb, bool store, int skipmask,
                                                const int* wait0, const int* wait1, int waitval, int* loaded0,
                                                int* loaded1);

// One off-diagonal pair-block item: out = Q_A^T X Q_B with X = B[pair
// (a1, b1) columns, pair (a2, b2) columns]; ra / rb say whether Q_A / Q_B are
// non-identity.  Leaves out in S.X (and its transpose in S.Q2); writes both
// orientations back to B when `store` (the caller ensures ra || rb there).
// Uses S.X, S.Y, S.Q, S.Q2; all threads; starts and ends with a barrier.
template <typename Smem>
__device__ __forceinline__ void j2_item(Smem& S, double* __restrict__ B, int np, int a1, int b1, int a2, int b2,
                                        const double* __restrict__ QA, const double* __restrict__ QB, bool ra,
                                        bool rb, bool store, int skipmask = 0, const int* wait0 = nullptr,
                                        const int* wait1 = nullptr, int waitval = 0, int* loaded0 = nullptr,
                                        int* loaded1 = nullptr) {
  const int tid = threadIdx.x;
  double xr[4], qa[4], qb[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {  // all three tiles in flight at once
    const int e = tid + u * J2_THREADS;
    xr[u] = B[(int64_t)j2_col(e >> 5, a1, b1) * np + j2_col(e & 31, a2, b2)];
    qa[u] = ra ? QA[e] : 0.0;
    qb[u] = rb ? QB[e] : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int e = tid + u * J2_THREADS;
    S.X[e >> 5][e & 31] = xr[u];
    if (ra) S.Q[e >> 5][e & 31] = qa[u];
    if (rb) S.Q2[e >> 5][e & 31] = qb[u];
  }
  __syncthreads();
  j2_item_compute(S, B, np, a1, b1, a2, b2, ra, rb, store, skipmask, wait0, wait1, waitval, loaded0, loaded1);
}

// Second half of j2_item: X (and Q_A in S.Q, Q_B in S.Q2 when rotated) are in
// shared memory, visible to all threads.
template <typename Smem>
__device__ __forceinline__ void j2_item_compute(Smem& S, double* __restrict__ B, int np, int a1, int b1, int a2,
                                                int b2, bool ra, bool rb, bool store, int skipmask,
                                                const int* wait0, const int* wait1, int waitval, int* loaded0,
                                                int* loaded1) {
  const int tid = threadIdx.x;
  if (tid == 0) {  // X is read: its next-step owners may now overwrite their quadrants
    if (loaded0) st_release(loaded0, waitval);
    if (loaded1) st_release(loaded1, waitval);
  }
  const int rr = tm_row();
  double o[4];
  if (!rb) {
#pragma unroll
    for (int u = 0; u < 4; ++u) o[u] = S.X[rr][tm_col(u)];
  } else {
    tile_mm<false>(S.X, S.Q2, o);  // Y = X Q_B
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) S.Y[rr][tm_col(u)] = o[u];
  __syncthreads();
  if (!ra) {
#pragma unroll
    for (int u = 0; u < 4; ++u) o[u] = S.Y[rr][tm_col(u)];
  } else {
    tile_mm<true>(S.Q, S.Y, o);  // Q_A^T Y
  }
  __syncthreads();  // everyone done reading S.X / S.Q2
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    S.X[rr][tm_col(u)] = o[u];
    S.Q2[tm_col(u)][rr] = o[u];
  }
  if (tid == 0) {  // next-step owners read this item's X before we overwrite it
    if (wait0)
      while (ld_acquire(wait0) < waitval) __nanosleep(20);
    if (wait1)
      while (ld_acquire(wait1) < waitval) __nanosleep(20);
  }
  __syncthreads();
  if (store) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = tid + u * J2_THREADS;
      const int i = e >> 5, j = e & 31;
      if ((skipmask >> (((i >> 4) << 1) | (j >> 4))) & 1) continue;  // a next-step owner writes it
      B[(int64_t)j2_col(i, a1, b1) * np + j2_col(j, a2, b2)] = S.X[i][j];
      B[(int64_t)j2_col(i, a2, b2) * np + j2_col(j, a1, b1)] = S.Q2[i][j];
    }
  }
}

// The 16x16 quadrant (rows hr.., cols hc.. of the 32x32 result) of an item,
// Q_A[:, hr..]^T X Q_B[:, hc..]: half of the first product, a quarter of the
// second.  Leaves the quadrant in S.Y[32 + i][j]?  No: in S.X[i][j], i, j < 16.
// Calls `loaded()` (thread 0, after a barrier) once X has been read.
template <typename Smem, typename F>
__device__ __forceinline__ void j2_quadrant(Smem& S, const double* __restrict__ B, int np, int a1, int b1, int a2,
                                            int b2, const double* __restrict__ QA, const double* __restrict__ QB,
                                            bool ra, bool rb, int hr, int hc, F loaded) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  double xr[4], qa[4], qb[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int e = tid + u * J2_THREADS;
    xr[u] = B[(int64_t)j2_col(e >> 5, a1, b1) * np + j2_col(e & 31, a2, b2)];
    qa[u] = ra ? QA[e] : 0.0;
    qb[u] = rb ? QB[e] : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int e = tid + u * J2_THREADS;
    S.X[e >> 5][e & 31] = xr[u];
    if (ra) S.Q[e >> 5][e & 31] = qa[u];
    if (rb) S.Q2[e >> 5][e & 31] = qb[u];
  }
  __syncthreads();
  if (tid == 0) loaded();
  // Y (32 x 16) = X Q_B[:, hc..hc+16): warp w -> rows 8(w>>1).., cols 8(w&1)..
  {
    const int r = 8 * (w >> 1) + (lane >> 2), kk = lane & 3, c = 8 * (w & 1) + (lane >> 2);
    double d0 = 0.0, d1 = 0.0;
    if (rb) {
#pragma unroll
      for (int k4 = 0; k4 < J2_PW; k4 += 4) j2_dmma(d0, d1, S.X[r][k4 + kk], S.Q2[k4 + kk][hc + c]);
    } else {
      d0 = S.X[r][hc + 8 * (w & 1) + 2 * kk];
      d1 = S.X[r][hc + 8 * (w & 1) + 2 * kk + 1];
    }
    S.Y[r][8 * (w & 1) + 2 * kk] = d0;
    S.Y[r][8 * (w & 1) + 2 * kk + 1] = d1;
  }
  __syncthreads();
  // quadrant (16 x 16) = Q_A[:, hr..hr+16)^T Y: warps 0..3
  if (w < 4) {
    const int r = 8 * (w >> 1) + (lane >> 2), kk = lane & 3, c = 8 * (w & 1) + (lane >> 2);
    double d0 = 0.0, d1 = 0.0;
    if (ra) {
#pragma unroll
      for (int k4 = 0; k4 < J2_PW; k4 += 4) j2_dmma(d0, d1, S.Q[k4 + kk][hr + r], S.Y[k4 + kk][c]);
    } else {
      d0 = S.Y[hr + r][8 * (w & 1) + 2 * kk];
      d1 = S.Y[hr + r][8 * (w & 1) + 2 * kk + 1];
    }
    S.X[r][8 * (w & 1) + 2 * kk] = d0;
    S.X[r][8 * (w & 1) + 2 * kk + 1] = d1;
  }
  __syncthreads();
}

// Cycle breakdown of CTA 0 (phase A load+measure, inner rounds, barrier 1,
// phase B, barrier 2, steps) — read with mlr_debug_j2prof.
__device__ unsigned long long g_j2prof[16];

// the same for the last CTA (a phase-B worker in split mode): slot 12 barrier
// wait, 13 ticket grabs / setup, 14 item compute, 15 items processed
__device__ unsigned long long g_j2prof2[8];
// Debug trace (mlr_debug_j2trace, tools/gpu/jacobi_trace.py): for global
// steps [g0, g0 + n), per CTA, %globaltimer at [0] the step barrier arrival,
// [1] its release, [3] the step start, [4] an owner's tile / quadrant
// loaded, [5] its rounds + Q done, [6] its wflag wait done; [2] phase-B
// items processed.  Off unless a buffer is set.
__device__ unsigned long long* g_j2trace = nullptr;
__device__ int g_j2trace_g0 = 0, g_j2trace_n = 0;
__device__ __forceinline__ unsigned long long j2_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void j2_trace(int g, int me, int nctas, int slot, unsigned long long v) {
  if (g_j2trace && g >= g_j2trace_g0 && g < g_j2trace_g0 + g_j2trace_n)
    g_j2trace[(((int64_t)(g - g_j2trace_g0) * nctas) + me) * 8 + slot] = v;
}
// slot 7: the SM the CTA runs on (placement of owners vs workers)
__device__ __forceinline__ void j2_trace_sm(int g, int me, int nctas) {
  if (g_j2trace && g >= g_j2trace_g0 && g < g_j2trace_g0 + g_j2trace_n) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_j2trace[(((int64_t)(g - g_j2trace_g0) * nctas) + me) * 8 + 7] = smid;
  }
}
__device__ __forceinline__ void j2_wmark2(int slot, long long& t0) {
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
    const long long t = clock64();
    atomicAdd(&g_j2prof2[slot], (unsigned long long)(t - t0));
    t0 = t;
  }
}
__device__ __forceinline__ void j2_wmark(int slot, long long& t0) {
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
    const long long t = clock64();
    atomicAdd(&g_j2prof[slot], (unsigned long long)(t - t0));
    t0 = t;
  }
}

__device__ __forceinline__ void j2_mark(int slot, long long& t0) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const long long t = clock64();
    atomicAdd(&g_j2prof[slot], (unsigned long long)(t - t0));
    t0 = t;
  }
}

// Per-CTA schedule built once per launch: the pair table of every step and
// this CTA's phase-B items (so the step loop does no integer div/mod).
struct J2Item {
  short kA, kB;  // pairs (kA == kB for V items)
  short r0;      // V row chunk start (-1 for B items)
  short pad;
};

template <bool CLUSTER>
__global__ void __launch_bounds__(J2_THREADS, 2)
jacobi2_kernel(double* __restrict__ B, double* __restrict__ V, int np, int nrows_v, double tol,
               double abs_floor_rel, int max_sweeps, double* __restrict__ Qlog, int cap,
               int* __restrict__ qflag_log, double* __restrict__ off_slots, int* __restrict__ result,
               const int* __restrict__ skip, int cache_q, double early_off, int vlog, int dflow, int tickets) {
  if (skip && *skip) return;
  if (result[7] != 0) return;  // converged or out of sweeps in an earlier launch
  extern __shared__ __align__(16) unsigned char smem_raw[];
  J2Smem& S = *reinterpret_cast<J2Smem*>(smem_raw);
  const int tid = threadIdx.x;
  const int nb = np / J2_BW;
  const int npairs = nb / 2;
  const int nctas = CLUSTER ? (int)cg::this_cluster().num_blocks() : (int)gridDim.x;
  const int me = CLUSTER ? (int)cg::this_cluster().block_rank() : (int)blockIdx.x;
  const int nbitems = npairs * (npairs - 1) / 2;  // off-diagonal pair blocks k1 < k2
  const int vchunks = (nrows_v + J2_PW - 1) / J2_PW;
  const int nitems = nbitems + (vlog ? 0 : npairs * vchunks);  // V items only without the log
  // Dataflow steps (dflow, requires the rotation log): phase-B items run on
  // the CTAs that own no pair when there are enough of them ("split"), the
  // items holding a next-step pair's off-diagonal block first; each of those
  // releases a per-pair flag that the next step's owner waits on instead of
  // a cluster/grid barrier, so phase A of step t+1 overlaps phase B of step t.
  const bool split = dflow && 2 * (nctas - npairs) >= npairs && dflow != 2;  // dflow 2: no owner/worker split
  const int nworkers = split ? nctas - npairs : nctas;
  const int widx = split ? me - npairs : me;  // < 0: owner only
  const int my_items = (dflow || widx < 0) ? 0 : (nitems - widx + nworkers - 1) / nworkers;
  int* cflag = qflag_log + cap * npairs;  // per next-step pair: step + 1 whose item is done
  int* tctr = cflag + npairs;             // dflow item-queue ticket counters (2, by step parity)
  int* wflag = tctr + 2;                  // per next-step pair: step whose critical item has read X
  // dynamic smem: [J2Smem][Qcache npairs x 32 x LD (optional)][sched nb*npairs int][items][qslot npairs int]
  unsigned char* p = smem_raw + ((sizeof(J2Smem) + 127) & ~size_t(127));
  double(*Qall)[J2_PW][J2_LD] = reinterpret_cast<double(*)[J2_PW][J2_LD]>(p);
  if (cache_q) p += (size_t)npairs * J2_PW * J2_LD * sizeof(double);
  int* sched = reinterpret_cast<int*>(p);
  p += (size_t)nb * npairs * sizeof(int);
  J2Item* items = reinterpret_cast<J2Item*>(p);
  p += (size_t)my_items * sizeof(J2Item);
  int* qslot = reinterpret_cast<int*>(p);  // my needed pairs -> cache slot (or -1)
  __shared__ int qf_all[64];
  __shared__ short cur_pair[J2_DF_MAXB], nxt_pair[J2_DF_MAXB], nxt_partner[J2_DF_MAXB];
  __shared__ int s_ticket;
  const double tol2 = tol * tol;

  for (int e = tid; e < nb * npairs; e += J2_THREADS) {
    const int step = e / npairs, k = e % npairs;
    int pa, pb;
    j2_pair(step, k, nb, pa, pb);
    sched[e] = pa | (pb << 16);
  }
  for (int q = tid; q < my_items; q += J2_THREADS) {
    const int it = widx + q * nworkers;
    J2Item x;
    if (it < nbitems) {
      int k1 = 0, rem = it;
      while (rem >= npairs - 1 - k1) {
        rem -= npairs - 1 - k1;
        ++k1;
      }
      x.kA = (short)k1;
      x.kB = (short)(k1 + 1 + rem);
      x.r0 = -1;
    } else {
      const int v = it - nbitems;
      x.kA = x.kB = (short)(v / vchunks);
      x.r0 = (short)((v % vchunks) * J2_PW);
    }
    x.pad = 0;
    items[q] = x;
  }
  __syncthreads();
  if (tid == 0) {  // compact list of the rotations this CTA reads
    for (int k = 0; k < npairs; ++k) qslot[k] = -1;
    for (int q = 0; q < my_items; ++q) {
      qslot[items[q].kA] = 0;
      qslot[items[q].kB] = 0;
    }
    int s = 0;
    for (int k = 0; k < npairs; ++k)
      if (qslot[k] == 0) qslot[k] = s++;
  }
  // absolute floor: abs_floor_rel * max_i |B_ii| (identical in every CTA)
  double dmax = 0.0;
  for (int i = tid; i < np; i += J2_THREADS) dmax = fmax(dmax, fabs(B[(int64_t)i * (np + 1)]));
  dmax = warp_max(dmax);
  if ((tid & 31) == 0) S.red[tid >> 5] = dmax;
  __syncthreads();
  if (tid == 0)
    for (int w = 1; w < J2_THREADS / 32; ++w) S.red[0] = fmax(S.red[0], S.red[w]);
  __syncthreads();
  // resume state (result[4..6]): sweep, next global step, first step not yet applied to V
  int sweep = result[4];
  int g = result[5];
  const int g_applied = result[6];
  const int g_start = g;
  const double abs_floor = g_start == 0 ? abs_floor_rel * S.red[0] : off_slots[2];
  // dflow: the critical items of every step (see phase B), once per launch:
  // thread st builds step st's list in next-step pair order, each item once
  short* crit_count = reinterpret_cast<short*>(items);
  short* crit_list = crit_count + ((nb + 7) & ~7);
  if (dflow) {
    __syncthreads();  // qslot (which shares this region) is no longer read
    for (int st = tid; st < nb; st += J2_THREADS) {
      int cnt = 0;
      if (st + 1 < nb) {
        short bp[J2_DF_MAXB];
        for (int k = 0; k < npairs; ++k) {
          const int x = sched[st * npairs + k];
          bp[x & 0xffff] = (short)k;
          bp[x >> 16] = (short)k;
        }
        for (int k2 = 0; k2 < npairs; ++k2) {
          const int nx = sched[(st + 1) * npairs + k2];
          const int ka = bp[nx & 0xffff], kb = bp[nx >> 16];
          if (ka == kb) continue;
          const int lo = min(ka, kb), hi = max(ka, kb);
          const int it = lo * (2 * npairs - lo - 1) / 2 + (hi - lo - 1);
          bool dup = false;
          for (int j = 0; j < cnt; ++j) dup |= crit_list[st * npairs + j] == it;
          if (!dup) crit_list[st * npairs + cnt++] = (short)it;
        }
      }
      crit_count[st] = (short)cnt;
    }
    __syncthreads();
  }
  bool converged = false;
  for (; sweep < max_sweeps; ++sweep) {
    if (vlog && g + nb > g_applied + cap) break;  // rotation log full: pause, V catches up, resume
    for (int step = 0; step < nb; ++step, ++g) {
      const int slot = g % cap;
      double* Qbuf = Qlog + (int64_t)slot * npairs * J2_PW * J2_PW;
      int* qflag = qflag_log + slot * npairs;
      long long tw = clock64();
      long long t0 = clock64();
      if (tid == 0) j2_trace(g, me, nctas, 3, j2_gtime());
      if (tid == 0) j2_trace_sm(g, me, nctas);
      if (blockIdx.x == 0 && tid == 0) atomicAdd(&g_j2prof[5], 1ull);
      const int* srow = sched + step * npairs;
      // ------------------------------------------------ phase A: pair owners
      for (int k = me; k < npairs; k += nctas) {
        const int pa = srow[k] & 0xffff, pb = srow[k] >> 16;
        // dflow: the off-diagonal block (pa, pb) comes from a phase-B item of
        // the previous step (unless pa, pb were paired then) that may still run
        bool loaded = false;
        bool crit_quad = false;
        if (dflow && step > 0 && cur_pair[pa] != cur_pair[pb]) {
          // (pa, pb) is one quadrant of the previous step's item (kA, kB):
          // compute just that quadrant (the workers compute and store the
          // rest, after this CTA has read the item's X: flag cflag[k] = g)
          const int k0a = cur_pair[pa], k0b = cur_pair[pb];
          const int kA = min(k0a, k0b), kB = max(k0a, k0b);
          int first = k;
          for (int k2 = 0; k2 < k; ++k2) {
            const int x = srow[k2];
            const int c1 = cur_pair[x & 0xffff], c2 = cur_pair[x >> 16];
            if (min(c1, c2) == kA && max(c1, c2) == kB) {
              first = k2;
              break;
            }
          }
          if (!split) {
            // owners are workers too: the first pair needing the item
            // computes all of it (workers skip it), a second one waits
            if (first == k) {
              const int* prow = sched + (step - 1) * npairs;
              const int a1 = prow[kA] & 0xffff, b1 = prow[kA] >> 16;
              const int a2 = prow[kB] & 0xffff, b2 = prow[kB] >> 16;
              const int pslot = (g - 1) % cap;
              const double* Qp = Qlog + (int64_t)pslot * npairs * J2_PW * J2_PW;
              const int* qfp = qflag_log + pslot * npairs;
              const bool ra = qfp[kA] != 0, rb = qfp[kB] != 0;
              const double da = B[(int64_t)(pa * J2_BW + (tid >> 4)) * np + pa * J2_BW + (tid & 15)];
              const double db = B[(int64_t)(pb * J2_BW + (tid >> 4)) * np + pb * J2_BW + (tid & 15)];
              j2_item(S, B, np, a1, b1, a2, b2, Qp + (int64_t)kA * J2_PW * J2_PW, Qp + (int64_t)kB * J2_PW * J2_PW, ra,
                      rb, ra || rb);
              S.G[tid >> 4][tid & 15] = da;
              S.G[J2_BW + (tid >> 4)][J2_BW + (tid & 15)] = db;
              const bool pa_row = cur_pair[pa] == kA;
              const int hr = (pa_row ? (pa == a1 ? 0 : 1) : (pb == a1 ? 0 : 1)) * J2_BW;
              const int hc = (pa_row ? (pb == a2 ? 0 : 1) : (pa == a2 ? 0 : 1)) * J2_BW;
              for (int e = tid; e < J2_BW * J2_BW; e += J2_THREADS) {
                const int i = e >> 4, j = e & 15;
                const double v = pa_row ? S.X[hr + i][hc + j] : S.X[hr + j][hc + i];  // B[pa + i][pb + j]
                S.G[i][J2_BW + j] = v;
                S.G[J2_BW + j][i] = v;
              }
              loaded = true;
              bool dup = false;
              for (int k2 = k + 1; k2 < npairs; ++k2) {
                const int x = srow[k2];
                const int c1 = cur_pair[x & 0xffff], c2 = cur_pair[x >> 16];
                if (min(c1, c2) == kA && max(c1, c2) == kB) dup = true;
              }
              if (dup) {
                __syncthreads();
                if (tid == 0) {
                  __threadfence();
                  for (int k2 = k + 1; k2 < npairs; ++k2) {
                    const int x = srow[k2];
                    const int c1 = cur_pair[x & 0xffff], c2 = cur_pair[x >> 16];
                    if (min(c1, c2) == kA && max(c1, c2) == kB) st_release(cflag + k2, g + 1);
                  }
                }
              }
            } else if (tid == 0) {
              while (ld_acquire(cflag + k) < g + 1) __nanosleep(20);
            }
          } else {
            const int* prow = sched + (step - 1) * npairs;
            const int a1 = prow[kA] & 0xffff, b1 = prow[kA] >> 16;
            const int a2 = prow[kB] & 0xffff, b2 = prow[kB] >> 16;
            const int pslot = (g - 1) % cap;
            const double* Qp = Qlog + (int64_t)pslot * npairs * J2_PW * J2_PW;
            const int* qfp = qflag_log + pslot * npairs;
            const bool ra = qfp[kA] != 0, rb = qfp[kB] != 0;
            const double da = B[(int64_t)(pa * J2_BW + (tid >> 4)) * np + pa * J2_BW + (tid & 15)];
            const double db = B[(int64_t)(pb * J2_BW + (tid >> 4)) * np + pb * J2_BW + (tid & 15)];
            // my off-diagonal block is one quadrant of the item
            const bool pa_row = cur_pair[pa] == kA;  // pa indexes the item's rows
            const int hr = (pa_row ? (pa == a1 ? 0 : 1) : (pb == a1 ? 0 : 1)) * J2_BW;
            const int hc = (pa_row ? (pb == a2 ? 0 : 1) : (pa == a2 ? 0 : 1)) * J2_BW;
            j2_quadrant(S, B, np, a1, b1, a2, b2, Qp + (int64_t)kA * J2_PW * J2_PW, Qp + (int64_t)kB * J2_PW * J2_PW,
                        ra, rb, hr, hc, [&]() { st_release(cflag + k, g); });
            crit_quad = true;
            S.G[tid >> 4][tid & 15] = da;
            S.G[J2_BW + (tid >> 4)][J2_BW + (tid & 15)] = db;
            {
              const int i = tid >> 4, j = tid & 15;
              const double v = pa_row ? S.X[i][j] : S.X[j][i];  // B[pa + i][pb + j]
              S.G[i][J2_BW + j] = v;
              S.G[J2_BW + j][i] = v;
            }
            loaded = true;
          }
        }
        __syncthreads();
        if (!loaded) load_pair_tile(S.G, B, np, pa, pb, pa, pb);
        if (tid == 0) {
          S.active = 0;
        }
        __syncthreads();
        if (step == 0 && k == 0 && tid == 0) off_slots[(sweep + 1) & 1] = 0.0;
        {
          double mx = 0.0;
          for (int e = tid; e < J2_PW * J2_PW; e += J2_THREADS) {
            const int i = e >> 5, j = e & 31;
            if (i < j && (step == 0 || (i < J2_BW && j >= J2_BW))) {
              const double g = fabs(S.G[i][j]);
              if (g > abs_floor) {
                const double d = fabs(S.G[i][i] * S.G[j][j]);
                mx = fmax(mx, d > 0.0 ? g * rsqrt(d) : 1e300);
              }
            }
          }
          mx = warp_max(mx);
          if ((tid & 31) == 0 && mx > 0.0) atomic_max_nonneg2(&off_slots[sweep & 1], mx);
          // a block whose inspected pairs are all below tolerance would not
          // rotate in any round: skip the rounds entirely
          if ((tid & 31) == 0 && mx > tol) S.active = 1;
        }
        __syncthreads();
        if (tid == 0) j2_trace(g, me, nctas, 4, j2_gtime());
        j2_mark(0, t0);
        const int rounds = !S.active ? 0 : (step == 0 ? J2_PW - 1 : J2_BW);
        // pair k of inner round rnd: circle method on 32 players for step 0,
        // cross pairs (k, 16 + (k + rnd) % 16) otherwise (computed, not loaded)
        auto pair_of = [&](int k, int rnd, int& i, int& j) {
          if (step == 0) {
            const int m = J2_PW - 1;
            if (k == 0) { i = rnd; j = m; } else { i = (rnd + k) % m; j = (rnd - k + m) % m; }
          } else {
            i = k;
            j = J2_BW + ((k + rnd) & (J2_BW - 1));
          }
        };
        double2* cs2 = reinterpret_cast<double2*>(&S.cs[0][0]);  // (c, s) per pair
        double* tt = &S.cs[0][0] + J2_PW;                         // t per pair
        unsigned rmask = 0;  // inner rounds that rotated (uniform: from __syncthreads_or)
        double(*Gfin)[J2_LD] = S.G;  // where the rotated tile ends up
        auto needs_rot = [&](double a, double b, double g) {
          return fabs(g) > abs_floor && g * g > tol2 * fabs(a * b);
        };
        if (step == 0) {
          // circle-method rounds: rotations, barrier, update, barrier
          for (int rnd = 0; rnd < rounds; ++rnd) {
            int rot_here = 0;
            if (tid < J2_PW / 2) {
              int i, j;
              pair_of(tid, rnd, i, j);
              const double a = S.G[i][i], b = S.G[j][j], g = S.G[i][j];
              double c = 1.0, s = 0.0, t = 0.0;
              if (needs_rot(a, b, g)) {
                jac_rot(a, b, g, c, s, t);
                rot_here = 1;
              }
              cs2[tid] = make_double2(c, s);
              S.csl[rnd][tid] = make_double2(c, s);
              tt[tid] = t;
            }
            if (!__syncthreads_or(rot_here)) continue;  // identity round: nothing to apply
            rmask |= 1u << rnd;
            {
              // thread (pp, q) owns rows {p1,p2} x cols {q1,q2} of G <- J^T G J
              const int pp = tid >> 4, q = tid & 15;
              int p1, p2, q1, q2;
              pair_of(pp, rnd, p1, p2);
              pair_of(q, rnd, q1, q2);
              const double2 csp = cs2[pp], csq = cs2[q];
              const double g11 = S.G[p1][q1], g12 = S.G[p1][q2], g21 = S.G[p2][q1], g22 = S.G[p2][q2];
              if (pp == q && tt[pp] != 0.0) {
                // the rotated pair itself: exact zero + classical diagonal update
                const double t = tt[pp];
                S.G[p1][p1] = j2_diag_lo(t, g12, g11);
                S.G[p2][p2] = j2_diag_hi(t, g12, g22);
                S.G[p1][p2] = 0.0;
                S.G[p2][p1] = 0.0;
              } else {
                const Blk o = j2_block(csp.x, csp.y, csq.x, csq.y, g11, g12, g21, g22);
                S.G[p1][q1] = o.o11;
                S.G[p1][q2] = o.o12;
                S.G[p2][q1] = o.o21;
                S.G[p2][q2] = o.o22;
              }
            }
            __syncthreads();
          }
        } else if (rounds > 0) {
          // Cross rounds, pipelined: pair i = (i, 16 + (i + rnd) % 16).  Warp
          // 0 (lanes 0..15, one pair each) computes the rotations of round
          // rnd + 1 while warps 1..7 apply round rnd from Gin into Gout: the
          // entries round rnd + 1 needs after round rnd are its own diagonal
          // update, that of pair i + 1 (whose second index j' becomes i's
          // partner) and the (i, j') element of block (pair i, pair i + 1),
          // all recomputed with the update's exact FMAs.  One barrier per round.
          double(*Gin)[J2_LD] = S.G;
          double(*Gout)[J2_LD] = S.G2;
          const int lane = tid & 31;
          double ra = 0.0, rb = 0.0, rg = 0.0, rc = 1.0, rs = 0.0, rt = 0.0;  // rotation warp: round rnd
          int rot_here = 0;
          if (tid < J2_BW) {
            const int i = tid, j = J2_BW + i;
            ra = Gin[i][i];
            rb = Gin[j][j];
            rg = Gin[i][j];
            if (needs_rot(ra, rb, rg)) {
              jac_rot(ra, rb, rg, rc, rs, rt);
              rot_here = 1;
            }
            S.csb[0][i] = make_double2(rc, rs);
            S.ttb[0][i] = rt;
            S.csl[0][i] = make_double2(rc, rs);
          }
          int any = __syncthreads_or(rot_here);
          // Q = J_0 J_1 ... replayed inside the rounds by warps 1-4 (they have
          // slack while warp 0 runs the rotation chain): 4 lanes per row of Q,
          // pairs kk = sq + 4h; x = Q[r][kk] stays, y = Q[r][partner] moves to
          // pair kk - 1 after every round (shuffle within the row's 4 lanes)
          const bool replay = tid >= 32 && tid < 160;
          const int rq = (tid - 32) >> 2, sq = (tid - 32) & 3;
          double qx[4], qy[4];
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            qx[h] = rq == sq + 4 * h ? 1.0 : 0.0;
            qy[h] = rq == J2_BW + sq + 4 * h ? 1.0 : 0.0;
          }
          const int qsrc = (lane & ~3) | ((sq + 1) & 3);
          for (int rnd = 0; rnd < rounds; ++rnd) {
            const int par = rnd & 1;
            if (any) rmask |= 1u << rnd;
            int rot_next = 0;
            if (tid < 32) {
              // ---- rotation warp: round rnd + 1
              const int i = lane & (J2_BW - 1);
              const int i1 = (i + 1) & (J2_BW - 1);
              const int src = (lane & 16) | i1;
              const double qc = __shfl_sync(0xffffffffu, rc, src), qs = __shfl_sync(0xffffffffu, rs, src);
              const double qt = __shfl_sync(0xffffffffu, rt, src), qb = __shfl_sync(0xffffffffu, rb, src);
              const double qg = __shfl_sync(0xffffffffu, rg, src);
              if (lane < J2_BW && rnd + 1 < rounds) {
                const int j = J2_BW + ((i + rnd) & (J2_BW - 1));       // partner in round rnd
                const int jn = J2_BW + ((i + rnd + 1) & (J2_BW - 1));  // partner in round rnd + 1
                double a2, b2, g2;
                if (any) {
                  a2 = rt != 0.0 ? j2_diag_lo(rt, rg, ra) : ra;
                  b2 = qt != 0.0 ? j2_diag_hi(qt, qg, qb) : qb;
                  const Blk o = j2_block(rc, rs, qc, qs, Gin[i][i1], Gin[i][jn], Gin[j][i1], Gin[j][jn]);
                  g2 = o.o12;
                } else {
                  a2 = ra;
                  b2 = qb;
                  g2 = Gin[i][jn];
                }
                ra = a2;
                rb = b2;
                rg = g2;
                rc = 1.0;
                rs = 0.0;
                rt = 0.0;
                if (needs_rot(ra, rb, rg)) {
                  jac_rot(ra, rb, rg, rc, rs, rt);
                  rot_next = 1;
                }
                S.csb[par ^ 1][i] = make_double2(rc, rs);
                S.ttb[par ^ 1][i] = rt;
                S.csl[rnd + 1][i] = make_double2(rc, rs);
              }
            } else {
              // ---- update warps: the 256 2x2 blocks of round rnd, Gin -> Gout
              for (int bi = any ? tid - 32 : J2_BW * J2_BW; bi < J2_BW * J2_BW; bi += J2_THREADS - 32) {
                const int pp = bi >> 4, q = bi & 15;
                const int p1 = pp, p2 = J2_BW + ((pp + rnd) & (J2_BW - 1));
                const int q1 = q, q2 = J2_BW + ((q + rnd) & (J2_BW - 1));
                const double2 csp = S.csb[par][pp], csq = S.csb[par][q];
                const double g11 = Gin[p1][q1], g12 = Gin[p1][q2], g21 = Gin[p2][q1], g22 = Gin[p2][q2];
                const double tp = S.ttb[par][pp];
                if (pp == q && tp != 0.0) {
                  Gout[p1][p1] = j2_diag_lo(tp, g12, g11);
                  Gout[p2][p2] = j2_diag_hi(tp, g12, g22);
                  Gout[p1][p2] = 0.0;
                  Gout[p2][p1] = 0.0;
                } else {
                  const Blk o = j2_block(csp.x, csp.y, csq.x, csq.y, g11, g12, g21, g22);
                  Gout[p1][q1] = o.o11;
                  Gout[p1][q2] = o.o12;
                  Gout[p2][q1] = o.o21;
                  Gout[p2][q2] = o.o22;
                }
              }
              if (replay) {
                if (any) {
#pragma unroll
                  for (int h = 0; h < 4; ++h) {
                    const double2 c2 = S.csb[par][sq + 4 * h];
                    const double a = qx[h], b = qy[h];
                    qx[h] = c2.x * a - c2.y * b;
                    qy[h] = c2.y * a + c2.x * b;
                  }
                }
                double v[4];
#pragma unroll
                for (int h = 0; h < 4; ++h) v[h] = __shfl_sync(0xffffffffu, qy[h], qsrc);
#pragma unroll
                for (int h = 0; h < 4; ++h) qy[h] = sq < 3 ? v[h] : v[(h + 1) & 3];
              }
            }
            const int any_next = __syncthreads_or(rot_next);
            if (any) {
              double(*tmp)[J2_LD] = Gin;
              Gin = Gout;
              Gout = tmp;
            }
            any = any_next;
          }
          Gfin = Gin;
          if (replay) {
            double* qo = Qbuf + (int64_t)k * J2_PW * J2_PW;
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const int kk = sq + 4 * h;
              qo[rq * J2_PW + kk] = qx[h];
              qo[rq * J2_PW + J2_BW + ((kk + rounds) & (J2_BW - 1))] = qy[h];
            }
          }
        }
        j2_mark(7, t0);
        // Q = J_0 J_1 ... : row r of Q evolves independently; 8 lanes own a
        // row, two pairs (kk = sub, sub + 8) each, and replay the log
        double* qo = Qbuf + (int64_t)k * J2_PW * J2_PW;
        const bool rot = rmask != 0;
        {
          const int r = tid >> 3, sub = tid & 7;
          if (step == 0) {  // circle-method pairs: replay in shared memory
            for (int e = sub; e < J2_PW; e += 8) S.Q[r][e] = (r == e) ? 1.0 : 0.0;
            __syncwarp();
            for (int rnd = 0; rnd < rounds; ++rnd) {
              if (!((rmask >> rnd) & 1u)) continue;
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int kk = sub + 8 * h;
                int i, j;
                pair_of(kk, rnd, i, j);
                const double2 c2 = S.csl[rnd][kk];
                const double a = S.Q[r][i], b = S.Q[r][j];
                S.Q[r][i] = c2.x * a - c2.y * b;
                S.Q[r][j] = c2.y * a + c2.x * b;
              }
              __syncwarp();
            }
            for (int e = sub; e < J2_PW; e += 8) qo[r * J2_PW + e] = S.Q[r][e];
          }
        }
        if (tid == 0) j2_trace(g, me, nctas, 5, j2_gtime());
        j2_mark(1, t0);
        // split mode: the worker taking my critical item must have read its X
        // (which contains my off-diagonal block) before I overwrite that block
        if (rot && crit_quad) {
          if (tid == 0)
            while (ld_acquire(wflag + k) < g) __nanosleep(20);
          if (tid == 0) j2_trace(g, me, nctas, 6, j2_gtime());
          __syncthreads();
        }
        // the rotated diagonal block goes straight back into B
        if (rot)
          for (int e = tid; e < J2_PW * J2_PW; e += J2_THREADS) {
            const int i = e >> 5, j = e & 31;
            B[(int64_t)j2_col(i, pa, pb) * np + j2_col(j, pa, pb)] = Gfin[i][j];
          }
        if (tid == 0) qflag[k] = rot ? 1 : 0;
      }
      if (!CLUSTER) __threadfence();  // barrier.cluster.arrive/wait are release/acquire
      j2_mark(6, t0);
      if (blockIdx.x == gridDim.x - 1 && tid == 0) tw = clock64();
      if (tid == 0) j2_trace(g, me, nctas, 0, j2_gtime());
      j2_sync<CLUSTER>();
      if (tid == 0) j2_trace(g, me, nctas, 1, j2_gtime());
      j2_mark(2, t0);
      j2_wmark(12, tw);
      // ------------------------------------------------ phase B: apply
      long long tw2 = tw;
      if (!dflow || widx >= 0)
        for (int k = tid; k < npairs; k += J2_THREADS) qf_all[k] = qflag[k];
      const bool last_step = step == nb - 1;
      if (dflow) {
        // block -> pair maps of this step and the next (within the sweep)
        for (int k = tid; k < npairs; k += J2_THREADS) {
          const int pa = srow[k] & 0xffff, pb = srow[k] >> 16;
          cur_pair[pa] = (short)k;
          cur_pair[pb] = (short)k;
          if (!last_step) {
            const int nx = sched[(step + 1) * npairs + k];
            const int na = nx & 0xffff, nbk = nx >> 16;
            nxt_pair[na] = (short)k;
            nxt_pair[nbk] = (short)k;
            nxt_partner[na] = (short)nbk;
            nxt_partner[nbk] = (short)na;
          }
        }
      }
      __syncthreads();
      __syncthreads();
      if (cache_q) {  // the rotations my items read (rotated pairs only), via cp.async
        for (int e2 = tid; e2 < npairs * J2_PW * J2_PW / 2; e2 += J2_THREADS) {
          const int e = 2 * e2;
          const int k = e >> 10;
          const int slot = qslot[k];
          if (slot >= 0 && qf_all[k]) {
            const unsigned dst = (unsigned)__cvta_generic_to_shared(&Qall[slot][(e >> 5) & 31][e & 31]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(Qbuf + e));
          }
        }
        asm volatile("cp.async.commit_group;\n" ::);
        asm volatile("cp.async.wait_group 0;\n" ::);
      }
      auto live = [&](int q) {
        const J2Item x = items[q];
        return x.r0 >= 0 ? qf_all[x.kA] != 0 : (qf_all[x.kA] || qf_all[x.kB]);
      };
      auto fetch = [&](int q, double (&reg)[4]) {
        const J2Item x = items[q];
        const int a1 = srow[x.kA] & 0xffff, b1 = srow[x.kA] >> 16;
        const int a2 = srow[x.kB] & 0xffff, b2 = srow[x.kB] >> 16;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int e = tid + u * J2_THREADS;
          const int i = e >> 5, j = e & 31;
          if (x.r0 >= 0)
            reg[u] = (x.r0 + i < nrows_v) ? V[(int64_t)(x.r0 + i) * np + j2_col(j, a1, b1)] : 0.0;
          else
            reg[u] = B[(int64_t)j2_col(i, a1, b1) * np + j2_col(j, a2, b2)];
        }
      };
      double cur[4], nxt[4];
      int q = 0;
      while (q < my_items && !live(q)) ++q;
      if (q < my_items) fetch(q, cur);
      while (q < my_items) {
        int q2 = q + 1;
        while (q2 < my_items && !live(q2)) ++q2;
        __syncthreads();
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int e = tid + u * J2_THREADS;
          S.X[e >> 5][e & 31] = cur[u];
        }
        if (q2 < my_items) fetch(q2, nxt);
        const J2Item x = items[q];
        const double(*QA)[J2_LD] = cache_q ? Qall[qslot[x.kA]] : S.Q;
        const double(*QB)[J2_LD] = cache_q ? Qall[qslot[x.kB]] : S.Q2;
        if (!cache_q) {
          load_dense_tile(S.Q, Qbuf + (int64_t)x.kA * J2_PW * J2_PW);
          load_dense_tile(S.Q2, Qbuf + (int64_t)x.kB * J2_PW * J2_PW);
        }
        __syncthreads();
        const int a1 = srow[x.kA] & 0xffff, b1 = srow[x.kA] >> 16;
        const int a2 = srow[x.kB] & 0xffff, b2 = srow[x.kB] >> 16;
        const int rr = tm_row();
        double o[4];
        if (x.r0 >= 0) {
          tile_mm<false>(S.X, QA, o);  // V rows * Q_k
#pragma unroll
          for (int u = 0; u < 4; ++u) S.Y[rr][tm_col(u)] = o[u];
          __syncthreads();
#pragma unroll
          for (int u = 0; u < 4; ++u) {  // coalesced 128-byte row segments
            const int e = tid + u * J2_THREADS;
            const int i = e >> 5, j = e & 31;
            if (x.r0 + i < nrows_v) V[(int64_t)(x.r0 + i) * np + j2_col(j, a1, b1)] = S.Y[i][j];
          }
        } else {
          // identity rotations were not cached: substitute I on the fly
          if (!qf_all[x.kB]) {
#pragma unroll
            for (int u = 0; u < 4; ++u) o[u] = S.X[rr][tm_col(u)];
          } else {
            tile_mm<false>(S.X, QB, o);  // Y = X Q_k2
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) S.Y[rr][tm_col(u)] = o[u];
          __syncthreads();
          if (!qf_all[x.kA]) {
#pragma unroll
            for (int u = 0; u < 4; ++u) o[u] = S.Y[rr][tm_col(u)];
          } else {
            tile_mm<true>(QA, S.Y, o);  // Q_k1^T Y
          }
          // stage the tile and its transpose, then write both orientations
          // with coalesced row segments
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            S.X[rr][tm_col(u)] = o[u];
            S.Q2[tm_col(u)][rr] = o[u];
          }
          __syncthreads();
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int e = tid + u * J2_THREADS;
            const int i = e >> 5, j = e & 31;
            B[(int64_t)j2_col(i, a1, b1) * np + j2_col(j, a2, b2)] = S.X[i][j];
            B[(int64_t)j2_col(i, a2, b2) * np + j2_col(j, a1, b1)] = S.Q2[i][j];
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) cur[u] = nxt[u];
        q = q2;
      }
      if (dflow && widx >= 0) {
        // Dynamic item queue over the items that no next-step owner computes
        // (see phase A).  Worker w's first ticket is w, the rest come from an
        // atomic counter offset by nworkers; each worker ends with exactly
        // one failing grab and the grab completing the count resets it.
        j2_wmark2(0, tw2);
        // Critical items (those holding a next-step pair's off-diagonal
        // block; computed for every step of the schedule at kernel start):
        // tickets 0 .. ncrit-1, in next-step pair order, each once.  An item
        // is critical iff a next-step pair joins one of its row blocks with
        // one of its column blocks (checked on the fly with nxt_partner).
        const short* dcrit = crit_list + (int64_t)step * npairs;
        int* ctr = tctr + (g & 1);
        auto is_crit = [&](int a1, int b1, int a2, int b2) {
          if (last_step) return false;
          const int p1 = nxt_partner[a1], p2 = nxt_partner[b1];
          return p1 == a2 || p1 == b2 || p2 == a2 || p2 == b2;
        };
        if (tid == 0) s_ticket = crit_count[step];
        __syncthreads();
        j2_wmark2(1, tw2);
        const int ncrit = s_ticket;
        __syncthreads();
        const int total = ncrit + nbitems;
        const int grabs = (total > nworkers ? total - nworkers : 0) + nworkers;
        auto grab = [&]() {
          if (tid == 0) s_ticket = atomicAdd(ctr, 1);
          __syncthreads();
          const int v = s_ticket;
          __syncthreads();
          return v;
        };
        // Static round-robin (default): worker w takes tickets w, w + nworkers, ...
        // (the critical items are tickets 0 .. ncrit-1, so they still come
        // first); items cost the same, and the contended atomic ticket counter
        // (~3 grabs per worker per step, 256 workers on one address) measured
        // ~12k cycles per step on a worker at C5.  tickets != 0: the queue.
        int tk = widx, last_v = -1;
        for (;;) {
          if (tk >= total) {
            if (tickets && last_v < 0) {  // the pre-assigned ticket was past the end: make the failing grab
              last_v = grab();
              tk = nworkers + last_v;
              continue;
            }
            break;
          }
          const int it = tk < ncrit ? dcrit[tk] : tk - ncrit;
          int kA = 0, rem = it;
          while (rem >= npairs - 1 - kA) {
            rem -= npairs - 1 - kA;
            ++kA;
          }
          const int kB = kA + 1 + rem;
          const bool crit = is_crit(srow[kA] & 0xffff, srow[kA] >> 16, srow[kB] & 0xffff, srow[kB] >> 16);
          if (tk >= ncrit && crit) {  // already taken as a critical item
          } else {
            // non-split: a next-step owner computes the whole item itself
            if ((qf_all[kA] || qf_all[kB]) && !(crit && !split)) {
              const int a1 = srow[kA] & 0xffff, b1 = srow[kA] >> 16;
              const int a2 = srow[kB] & 0xffff, b2 = srow[kB] >> 16;
              // quadrants that are a next-step pair's off-diagonal block are
              // written by that pair's owner; wait until it has read X
              int skipmask = 0;
              const int* w0 = nullptr;
              const int* w1 = nullptr;
              int* l0 = nullptr;
              int* l1 = nullptr;
              if (crit) {
                const int xs[2] = {a1, b1}, ys[2] = {a2, b2};
                for (int qx = 0; qx < 2; ++qx)
                  for (int qy = 0; qy < 2; ++qy)
                    if (nxt_partner[xs[qx]] == ys[qy]) {
                      skipmask |= 1 << (qx * 2 + qy);
                      const int kn = nxt_pair[xs[qx]];
                      if (!w0) {
                        w0 = cflag + kn;
                        l0 = wflag + kn;
                      } else {
                        w1 = cflag + kn;
                        l1 = wflag + kn;
                      }
                    }
              }
              j2_wmark(13, tw);
              j2_wmark2(2, tw2);
              j2_item(S, B, np, a1, b1, a2, b2, Qbuf + (int64_t)kA * J2_PW * J2_PW,
                      Qbuf + (int64_t)kB * J2_PW * J2_PW, qf_all[kA] != 0, qf_all[kB] != 0, true, skipmask, w0,
                      w1, g + 1, l0, l1);
              j2_wmark(14, tw);
              if (blockIdx.x == gridDim.x - 1 && tid == 0) atomicAdd(&g_j2prof[15], 1ull);
              if (tid == 0 && g_j2trace && g >= g_j2trace_g0 && g < g_j2trace_g0 + g_j2trace_n)
                g_j2trace[(((int64_t)(g - g_j2trace_g0) * nctas) + me) * 8 + 2] += 1;
            } else if (split && crit && tid == 0) {
              // identity critical item: nothing to read, release its owners
              const int xs[2] = {srow[kA] & 0xffff, srow[kA] >> 16};
              for (int qx = 0; qx < 2; ++qx) {
                const int y = nxt_partner[xs[qx]];
                if (cur_pair[y] == kB) st_release(wflag + nxt_pair[xs[qx]], g + 1);
              }
            }
          }
          if (tickets) {
            last_v = grab();
            tk = nworkers + last_v;
          } else {
            tk += nworkers;
          }
        }
        if (tickets && tid == 0 && last_v == grabs - 1) atomicExch(ctr, 0);
      }
      if (!CLUSTER && (!dflow || last_step)) __threadfence();
      j2_mark(3, t0);
      if (!dflow || last_step) j2_sync<CLUSTER>();  // sweep end: convergence check, pause
      j2_mark(4, t0);
    }
    const double off = *((volatile double*)&off_slots[sweep & 1]);
    // converged: nothing above tol this sweep, or (quadratic convergence)
    // everything was already so small that this sweep's rotations pushed
    // the off-diagonal below tol
    if (off <= tol || off <= early_off) {
      converged = true;
      ++sweep;
      break;
    }
  }
  if (me == 0 && tid == 0) {
    result[0] = converged ? sweep : -sweep;
    result[4] = sweep;
    result[5] = g;
    result[7] = converged ? 1 : (sweep >= max_sweeps ? 2 : 0);
    if (g_start == 0) off_slots[2] = abs_floor;
  }
}

// ------------------------------------------------------------------ V update
// The rotations of every step are logged (Qlog slot g % cap); V is updated
// off the critical path by j2_vapply_kernel after the Jacobi launch: CTA b
// keeps rows [16b, 16b+16) of V in shared memory and applies the logged
// steps in order, V[rows, pair k cols] <- V[rows, pair k cols] Q_k, warp w
// taking pairs w, w+16, ... with FP64 DMMA.  B fragments come straight from
// L2 (each one feeds both 8-row groups); 16 warps keep enough loads in
// flight to cover the L2 latency.
constexpr int VA_THREADS = 512, VA_WARPS = VA_THREADS / 32;

template <int VA_R>  // rows of V per CTA: 16, or 8 when a 16-row tile does not fit
__global__ void __launch_bounds__(VA_THREADS)
j2_vapply_kernel(double* __restrict__ V, int np, int nrows_v, const double* __restrict__ Qlog, int cap,
                 const int* __restrict__ qflag_log, int* __restrict__ result, const int* __restrict__ skip) {
  if (skip && *skip) return;
  const int g0 = result[6], g1 = result[5];
  const int nb = np / J2_BW, npairs = nb / 2;
  const int ldt = np + 2;
  extern __shared__ __align__(16) double va_smem[];
  double* T = va_smem;  // VA_R x ldt
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int r0 = blockIdx.x * VA_R;
  if (g1 > g0 && r0 < nrows_v) {
    for (int e = tid; e < VA_R * np; e += VA_THREADS) {
      const int r = e / np, c = e - r * np;
      T[r * ldt + c] = r0 + r < nrows_v ? V[(int64_t)(r0 + r) * np + c] : 0.0;
    }
    for (int g = g0; g < g1; ++g) {
      __syncthreads();  // step g-1 (or the tile load) complete
      const int slot = g % cap, st = g % nb;
      for (int k = w; k < npairs; k += VA_WARPS) {
        if (!qflag_log[slot * npairs + k]) continue;
        const double* q = Qlog + ((int64_t)slot * npairs + k) * J2_PW * J2_PW;
        double b[8][4];
#pragma unroll
        for (int k4 = 0; k4 < 8; ++k4)
#pragma unroll
          for (int ct = 0; ct < 4; ++ct) b[k4][ct] = __ldg(q + (k4 * 4 + (lane & 3)) * J2_PW + ct * 8 + (lane >> 2));
        int pa, pb;
        j2_pair(st, k, nb, pa, pb);
#pragma unroll
        for (int rg = 0; rg < VA_R / 8; ++rg) {
          double* trow = T + (rg * 8 + (lane >> 2)) * ldt;
          double o[4][2] = {};
#pragma unroll
          for (int k4 = 0; k4 < 8; ++k4) {
            const double a = trow[j2_col(k4 * 4 + (lane & 3), pa, pb)];
#pragma unroll
            for (int ct = 0; ct < 4; ++ct) j2_dmma(o[ct][0], o[ct][1], a, b[k4][ct]);
          }
          __syncwarp();
#pragma unroll
          for (int ct = 0; ct < 4; ++ct)
#pragma unroll
            for (int e = 0; e < 2; ++e) trow[j2_col(ct * 8 + 2 * (lane & 3) + e, pa, pb)] = o[ct][e];
        }
      }
    }
    __syncthreads();
    for (int e = tid; e < VA_R * np; e += VA_THREADS) {
      const int r = e / np, c = e - r * np;
      if (r0 + r < nrows_v) V[(int64_t)(r0 + r) * np + c] = T[r * ldt + c];
    }
  }
  // the last CTA to finish marks the logged range as applied
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(&result[8], 1) + 1 == (int)gridDim.x) {
      result[6] = g1;
      result[8] = 0;
      __threadfence();
    }
  }
}

// 16-row tiles while that still gives ~32+ CTAs; 8-row tiles otherwise (more
// CTAs for small n_p, or a 16-row tile no longer fits shared memory)
static int vapply_rows(int np) {
  const char* e = getenv("MLR_VA_ROWS");
  if (e) return atoi(e) == 16 ? 16 : 8;
  return (size_t)16 * (np + 2) * sizeof(double) <= 200 * 1024 && np / 16 >= 32 ? 16 : 8;
}
static size_t vapply_smem(int np) { return (size_t)vapply_rows(np) * (np + 2) * sizeof(double); }

// Rotation-log capacity in steps: whole sweeps, up to 60, within ~128 MB.
int jacobi2_log_steps(int np) {
  const int nb = np / J2_BW, npairs = nb / 2;
  if (npairs < 1) return 1;
  const int64_t per_step = (int64_t)npairs * J2_PW * J2_PW * 8;
  int64_t steps = ((int64_t)128 << 20) / per_step;
  steps = std::min<int64_t>(steps, 60 * (int64_t)nb);
  steps = std::max<int64_t>(steps / nb * nb, nb);
  return (int)steps;
}
static bool j2_use_log(int np) { return vapply_smem(np) <= 200 * 1024; }

int64_t jacobi2_qbuf_elems(int np) {
  const int npairs = std::max(np / J2_BW / 2, 1);
  return (int64_t)(j2_use_log(np) ? jacobi2_log_steps(np) : 1) * npairs * J2_PW * J2_PW;
}
int64_t jacobi2_qflag_elems(int np) {  // log flags + the dataflow pair flags
  const int npairs = std::max(np / J2_BW / 2, 1);
  return (int64_t)(j2_use_log(np) ? jacobi2_log_steps(np) : 1) * npairs + 2 * npairs + 2;
}

static int launch_j2(double* B, double* V, int np, int nrows_v, double tol, double abs_floor_rel, int max_sweeps,
                     double* Qlog, int cap, int* qflag_log, double* off_slots, int* result, const int* skip,
                     int vlog, cudaStream_t st) {
  const int nb = np / J2_BW;
  const int npairs = nb / 2;
  const bool cluster = np <= 512;
  int nctas = 16;
  if (!cluster) {
    int dev = 0, nsm = 0;
    MLR_CUDA(cudaGetDevice(&dev));
    MLR_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    nctas = std::max(1, std::min(std::max(npairs, npairs * (npairs + 1) / 4), nsm));
  }
  int grid_per_sm = 1;  // cooperative path: a second CTA per SM doubles the phase-B workers
  const int vchunks = (nrows_v + J2_PW - 1) / J2_PW;
  const int nitems = npairs * (npairs - 1) / 2 + (vlog ? 0 : npairs * vchunks);
  // dataflow steps (see jacobi2_kernel) when the per-CTA item lists fit
  int dflow = 0;
  if (vlog && nb <= J2_DF_MAXB) dflow = 1;
  if (const char* e = getenv("MLR_J2_DFLOW")) dflow = !dflow ? 0 : (e[0] == '0' ? 0 : (e[0] == '2' ? 2 : 1));
  int tickets = 0;  // 1: dynamic phase-B item queue (atomic counter) instead of static round-robin
  if (const char* e = getenv("MLR_J2_TICKETS")) tickets = e[0] == '1';
  const int max_items = dflow ? 0 : (nitems + nctas - 1) / nctas;
  // dflow: per-step critical-item counts and lists (shorts); else the item list
  const size_t item_bytes =
      dflow ? 2 * (size_t)((nb + 7) & ~7) + 2 * (size_t)nb * npairs + 64 : (size_t)max_items * 8;
  const size_t sched = (size_t)nb * npairs * sizeof(int) + item_bytes + (size_t)npairs * sizeof(int) + 64;
  const size_t qcache = (size_t)npairs * J2_PW * J2_LD * sizeof(double);
  const int cache_q = (!dflow && sizeof(J2Smem) + qcache + sched <= 200 * 1024) ? 1 : 0;
  const size_t smem = ((sizeof(J2Smem) + 127) & ~size_t(127)) + (cache_q ? qcache : 0) + sched;
  if (smem > 220 * 1024) {
    set_error("jacobi2: schedule does not fit in shared memory");
    return kErrArg;
  }
  // quadratic convergence: a sweep that started with every pair below
  // ~sqrt(tol) leaves the off-diagonal ~ below tol, no verification sweep
  const double early_off = 0.03 * std::sqrt(tol);
  if (!cluster && dflow) {
    MLR_CUDA(cudaFuncSetAttribute(jacobi2_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0, dev = 0, nsm = 0;
    MLR_CUDA(cudaGetDevice(&dev));
    MLR_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    MLR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, jacobi2_kernel<false>, J2_THREADS, smem));
    grid_per_sm = std::max(1, std::min(occ, 2));
    const int want = std::max(npairs, npairs * (npairs + 1) / 4);
    if (const char* e = getenv("MLR_J2_PER_SM")) grid_per_sm = std::max(1, std::min(occ, atoi(e)));
    nctas = std::max(1, std::min(want, nsm * grid_per_sm));
  }
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(J2_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.gridDim = dim3(nctas);
  cudaLaunchAttribute attr[1];
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cluster) {
    auto kern = jacobi2_kernel<true>;
    MLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    MLR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = nctas;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
  } else {
    MLR_CUDA(cudaFuncSetAttribute(jacobi2_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
  }
  const size_t vsm = vapply_smem(np);
  const int var = vapply_rows(np);
  if (vlog) {
    MLR_CUDA(cudaFuncSetAttribute(j2_vapply_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vsm));
    MLR_CUDA(cudaFuncSetAttribute(j2_vapply_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vsm));
  }
  // the log holds cap / nb sweeps: enough (jacobi, V) launch pairs for max_sweeps;
  // launches after convergence return immediately
  const int per_launch = vlog ? std::max(1, cap / nb) : max_sweeps;
  const int launches = (max_sweeps + per_launch - 1) / per_launch;
  for (int l = 0; l < std::max(launches, 1); ++l) {
    if (cluster)
      MLR_CUDA(cudaLaunchKernelEx(&cfg, jacobi2_kernel<true>, B, V, np, nrows_v, tol, abs_floor_rel, max_sweeps,
                                  Qlog, cap, qflag_log, off_slots, result, skip, cache_q, early_off, vlog, dflow,
                                  tickets));
    else
      MLR_CUDA(cudaLaunchKernelEx(&cfg, jacobi2_kernel<false>, B, V, np, nrows_v, tol, abs_floor_rel, max_sweeps,
                                  Qlog, cap, qflag_log, off_slots, result, skip, cache_q, early_off, vlog, dflow,
                                  tickets));
    if (vlog) {
      if (var == 16)
        j2_vapply_kernel<16><<<(nrows_v + 15) / 16, VA_THREADS, vsm, st>>>(V, np, nrows_v, Qlog, cap, qflag_log,
                                                                          result, skip);
      else
        j2_vapply_kernel<8><<<(nrows_v + 7) / 8, VA_THREADS, vsm, st>>>(V, np, nrows_v, Qlog, cap, qflag_log,
                                                                        result, skip);
      MLR_LAUNCH_CHECK("j2_vapply_kernel");
    }
  }
  return kOk;
}

int jacobi2_debug_trace(unsigned long long* buf, int g0, int n) {
  MLR_CUDA(cudaMemcpyToSymbol(g_j2trace, &buf, sizeof(buf)));
  MLR_CUDA(cudaMemcpyToSymbol(g_j2trace_g0, &g0, sizeof(int)));
  MLR_CUDA(cudaMemcpyToSymbol(g_j2trace_n, &n, sizeof(int)));
  return kOk;
}

int jacobi2_debug_prof2(unsigned long long* out8) {
  MLR_CUDA(cudaMemcpyFromSymbol(out8, g_j2prof2, sizeof(unsigned long long) * 8));
  unsigned long long z[8] = {};
  MLR_CUDA(cudaMemcpyToSymbol(g_j2prof2, z, sizeof(z)));
  return kOk;
}

int jacobi2_debug_prof(unsigned long long* out8) {
  MLR_CUDA(cudaMemcpyFromSymbol(out8, g_j2prof, sizeof(unsigned long long) * 16));
  unsigned long long z[16] = {};
  MLR_CUDA(cudaMemcpyToSymbol(g_j2prof, z, sizeof(z)));
  return kOk;
}

// Qbuf: the rotation log (jacobi2_qbuf_elems doubles); qflag:
// jacobi2_qflag_elems ints; off_slots: 4 doubles; result: 16 ints
// (result[0] = sweeps, negative when not converged).
int jacobi2_eig(bool f32, void* B, void* V, int np, int nrows_v, double tol, double abs_floor_rel, int max_sweeps,
                void* Qbuf, int* qflag, double* off_slots, int* result, const int* skip, cudaStream_t st) {
  (void)f32;  // the coarse eigenproblem is always solved in FP64
  if (np % 64 != 0) {
    set_error("jacobi2_eig: n_p must be a multiple of 64");
    return kErrArg;
  }
  MLR_CUDA(cudaMemsetAsync(off_slots, 0, 4 * sizeof(double), st));
  MLR_CUDA(cudaMemsetAsync(result, 0, 16 * sizeof(int), st));
  MLR_CUDA(cudaMemsetAsync(qflag, 0, sizeof(int) * jacobi2_qflag_elems(np), st));
  const int vlog = j2_use_log(np) ? 1 : 0;
  const int cap = vlog ? jacobi2_log_steps(np) : 1;
  return launch_j2((double*)B, (double*)V, np, nrows_v, tol, abs_floor_rel, max_sweeps, (double*)Qbuf, cap, qflag,
                   off_slots, result, skip, vlog, st);
}

}  // namespace mlr
