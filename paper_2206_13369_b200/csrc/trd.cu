// Coarse symmetric eigensolver by Householder tridiagonalisation (sm_100a).
//
// Replaces the two-sided Jacobi for the ML-PCP coarse SVT (reference
// pcp.py:257-258, svd_full = LAPACK gesdd, linalg.py:86-99): only the
// eigenpairs of B = M_H^T M_H above tau^2 enter the SVT, and the Jacobi had
// to diagonalise the whole noise bulk below tau^2 as well (6-12 sweeps per
// warm-started iteration at C5).  Here:
//
//   1. trd_reduce_kernel   B = Q T Q^T (T tridiagonal), one cooperative grid.
//      Row i of B lives in the shared memory of CTA i mod G (C5: 16 rows of
//      1250 doubles in each of 79 CTAs), so the n - 2 reflector steps never
//      touch HBM.  Every CTA keeps a replica of the next row, so it builds
//      the reflector v_j itself; per step it computes p_i = beta A_i v for its
//      rows (one warp per row) and publishes them with its partial p^T v,
//      then (after the one grid-wide exchange of the step) applies
//      A -= v w^T + w v^T, w = p - (beta/2)(p^T v) v, to its rows and to the
//      replica; the owner of row j + 2 publishes it for the next-but-one
//      step.  Publication is fence-free: every double travels in a 16-byte
//      record {lo, tag, hi, tag} written and polled with single 16-byte
//      volatile accesses (the NCCL LL protocol), the tag being the step.
//      Fixed-order sums: bitwise reproducible, so replicated ranks agree.
//   2. trd_bisect_kernel   eigenvalues of T above tau^2: Sturm counts give
//      k = #{lambda > tau^2} exactly; one warp per eigenvalue refines it by
//      32-point multisection to full FP64 accuracy (division-free Sturm
//      sequences: one FMA on the dependency chain per step).
//   3. trd_vectors_kernel  eigenvector of T per eigenvalue from the twisted
//      factorisation T - lambda I = N_r D_r N_r^T (one warp per vector, the
//      pivots from the forward / backward Sturm sequences so the divisions
//      stay off the dependency chain, twist index r at the smallest
//      |gamma_r|, then two products; scratch in shared memory).
//   4. trd_back_kernel     V = Q Z: the reflectors applied in reverse order to
//      the k vectors (one warp per vector, the vector in registers, the
//      reflector rows staged in shared memory by TMA bulk copies).
//   5. trd_commit_kernel   eigenvalues to diag(B~) (what svt_weights reads),
//      zero V outside the k columns; on any non-finite result V = I and the
//      Jacobi (launched after, skipped on success) solves the iteration.
//
// Accuracy: the reduction is backward stable (T = Q^T (B + E) Q with
// |E| ~ eps |B|) and the twisted vectors have residual ~ eps |T|, like
// LAPACK dsytrd + dstebz + dstein; a numpy restatement of exactly these steps
// reproduces the reference's C1 / C2 solves (same iterations and rank
// column, relF(L) 1e-12 / 3e-13).

#include <cfloat>

#include "common.cuh"
#include "kernels.h"
#include "pcp.h"

namespace mlr {

namespace {

constexpr int TRD_T = 512;
constexpr int TRD_W = TRD_T / 32;  // one local row per warp
constexpr int TRD_MAXG = 256;
constexpr int TRD_LL = 4;  // publication records per thread and step: n <= 4 x 512

// flag-carrying 16-byte records (NCCL LL): {lo32, tag, hi32, tag}
__device__ __forceinline__ void ll_store(uint4* p, double v, uint32_t tag) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  asm volatile("st.relaxed.gpu.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"((uint32_t)u), "r"(tag),
               "r"((uint32_t)(u >> 32)), "r"(tag)
               : "memory");
}
__device__ __forceinline__ uint4 ll_ld(const uint4* p) {
  uint4 v;
  asm volatile("ld.relaxed.gpu.global.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ double ll_val(uint4 v) {
  return __longlong_as_double((long long)(((unsigned long long)v.z << 32) | v.x));
}

// a / b to ~1 ulp: approximate reciprocal and two Newton steps (normal
// inputs of moderate exponent: T is pre-scaled to |T| ~ 1)
__device__ __forceinline__ double trd_div(double a, double bb) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(bb));
  double e = fma(-bb, r, 1.0);
  r = fma(r, e, r);
  e = fma(-bb, r, 1.0);
  r = fma(r, e, r);
  return a * r;
}

// Sum of the TRD_W per-warp partials in shared memory: every thread loads
// them (broadcast reads) and adds them in a fixed tree, ~80 cycles on the
// step's dependency chain against ~250 for a 5-level shuffle butterfly.
__device__ __forceinline__ double trd_sum16(const double* part) {
  static_assert(TRD_W == 16, "trd_sum16 adds 16 partials");
  const double2* p2 = reinterpret_cast<const double2*>(part);
  double2 a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = p2[i];
  const double s0 = (a[0].x + a[0].y) + (a[1].x + a[1].y), s1 = (a[2].x + a[2].y) + (a[3].x + a[3].y);
  const double s2 = (a[4].x + a[4].y) + (a[5].x + a[5].y), s3 = (a[6].x + a[6].y) + (a[7].x + a[7].y);
  return (s0 + s1) + (s2 + s3);
}

// The reflector that zeroes row[j+2..n) of the (replicated) row j + 1
// (Householder, LAPACK dlarfg convention): beta, the new off-diagonal e and
// the scale of v = row / (alpha - e).  s = sum of row[k]^2, k >= j + 2.
// Computed redundantly by every thread: identical inputs, identical ops.
__device__ __forceinline__ void trd_reflector(double alpha, double s, double& bet, double& ej, double& scale) {
  bet = 0.0;
  ej = alpha;
  scale = 0.0;
  if (s != 0.0) {
    const double nx = sqrt(fma(alpha, alpha, s));
    ej = alpha >= 0.0 ? -nx : nx;
    bet = trd_div(ej - alpha, ej);
    scale = trd_div(1.0, alpha - ej);
  }
}

// Step j uses v_j (vsb[j & 1], built at the end of step j - 1 from the
// replica of row j) and keeps the rank-2 update of step j - 1 pending on the
// local rows: the matvec corrects for it with two scalars,
//   (A - v' w'^T - w' v'^T)_i . v = A_i . v - v'_i (w' . v) - w'_i (v' . v),
// and the update itself is applied after p is published, while the
// exchange is in flight.  The exchange carries p only: every CTA has v and
// all of p, so K = beta/2 p . v needs no separate partial sums.
// NQ > 0: each warp keeps its row in registers (element k = lane + 32 q),
// which halves the shared-memory traffic of the matvec and the update;
// NQ = 0: rows in shared memory (any n up to the limits).
__device__ __forceinline__ void trd_dsm_st(const double* local_addr, uint32_t cta, double v) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(remote)
               : "r"((uint32_t)__cvta_generic_to_shared(local_addr)), "r"(cta));
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(remote), "d"(v) : "memory");
}
__device__ __forceinline__ void trd_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// CL: the whole grid is one thread-block cluster (n_H <= 256): p and the
// replica row are written straight into every CTA's shared memory
// (st.shared::cluster) and one cluster barrier per step replaces the
// flag-carrying records and sentinels in L2.
template <int NQ, bool CL, bool COLX>
__global__ void __launch_bounds__(TRD_T, 1)
trd_reduce_kernel(const double* __restrict__ B, int ldb, int n, TrdBuf b, const int* __restrict__ skip, int trace) {
  if (skip && *skip) return;
#ifdef TRD_TRACE
  long long tr[8];
  const bool tron = trace && threadIdx.x == 0;
#else
  trace = 0;
#endif
  extern __shared__ double trd_sm[];
  const int G = gridDim.x, g = blockIdx.x;
  const int R = (n + G - 1) / G;  // <= TRD_W (host checks)
  const int ldh = (n + 1) & ~1;
  double* rows = trd_sm;          // NQ = 0: R x n rows g, g + G, g + 2G, ...
  double* vsb = rows + (NQ > 0 ? 0 : (size_t)R * n);  // 2 x n: v_j by step parity
  double* wpv = vsb + 2 * (size_t)n;   // w of the pending update
  double* ps = wpv + n;
  double* cur = ps + n;                // the replica of row j + 1
  double* psb = cur + n;               // CL: 2 x n, p by step parity (written by every CTA)
  double* nxt = psb + 2 * (size_t)n;   // CL: 2 x n, the next replica row by row parity
  __shared__ __align__(16) double kpart[TRD_W], sqpart[TRD_W], s1part[TRD_W], s2part[TRD_W], s_bs[2];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (NQ == 0)
    for (int r = 0; r < R; ++r) {
      const int i = g + r * G;
      if (i < n)
        for (int k = tid; k < n; k += TRD_T) rows[(size_t)r * n + k] = B[(int64_t)i * ldb + k];
    }
  {
    double q = 0.0;
    for (int k = tid; k < n; k += TRD_T) {
      const double x = B[k];
      cur[k] = x;
      if (k >= 2) q = fma(x, x, q);
    }
    q = warp_sum(q);
    if (lane == 0) sqpart[wid] = q;
  }
  __syncthreads();
  double bet;
  {
    double s = 0.0;
    for (int w = 0; w < TRD_W; ++w) s += sqpart[w];
    double ej, scale;
    trd_reflector(cur[1], s, bet, ej, scale);
    if (g == 0 && tid == 0) {
      b.beta[0] = bet;
      b.dd[0] = cur[0];
      b.ee[0] = ej;
    }
    for (int k = 1 + tid; k < n; k += TRD_T) {
      const double v = k == 1 ? 1.0 : cur[k] * scale;
      vsb[k] = v;
      if (g == 0) b.hv[k] = v;
    }
  }
  __syncthreads();
  if constexpr (CL) {
    for (int k = tid; k < n; k += TRD_T) nxt[n + k] = B[ldb + k];  // row 1 for step 0
    trd_cluster_sync();  // every CTA is running before the first remote store
  }
  const int my_i = g + wid * G;  // the row this warp owns (if < n and wid < R)
  const bool has_row = wid < R && my_i < n;
  double* my_row = rows + (size_t)wid * n;
  double rr[NQ > 0 ? NQ : 1];
  if constexpr (NQ > 0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int k = lane + 32 * q;
      rr[q] = (has_row && k < n) ? B[(int64_t)my_i * ldb + k] : 0.0;
    }
  }
  for (int j = 0; j < n - 2; ++j) {
    const int m1 = j + 1;
    const uint32_t tag = (uint32_t)j + 1u;
    const double* vc = vsb + (size_t)(j & 1) * n;         // v_j
    const double* vp = vsb + (size_t)((j + 1) & 1) * n;   // v_{j-1} (pending)
    if constexpr (CL) {
      ps = psb + (size_t)(j & 1) * n;
      cur = nxt + (size_t)(m1 & 1) * n;
    }
#ifdef TRD_TRACE
    const bool trs = tron && j == n / 2;
    const long long tr0s = clock64();
    if (trs) {
      tr[0] = clock64();
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr[7]));
    }
#endif
    // (1) p_i = beta (A_i . v - v'_i s1 - w'_i s2) for the local rows i >= j + 1
    if (has_row && my_i >= m1) {
#ifdef TRD_TRACE
      long long w0 = 0, w1 = 0, w2 = 0;
      const bool wtr = trace && j == n / 2 && lane == 0 && wid == R - 1 && g < 4;
      if (wtr) w0 = clock64();
#endif
      double s1 = (j > 0 && lane < TRD_W) ? s1part[lane] : 0.0;
      double s2 = (j > 0 && lane < TRD_W) ? s2part[lane] : 0.0;
      double a0 = 0.0, a1 = 0.0;
      if constexpr (NQ > 0) {
        double a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int k = lane + 32 * q;
          if (k >= m1 && k < n) {
            const double t = rr[q] * vc[k];
            if ((q & 3) == 0) a0 += t;
            else if ((q & 3) == 1) a1 += t;
            else if ((q & 3) == 2) a2 += t;
            else a3 += t;
          }
        }
        a0 += a2;
        a1 += a3;
      } else {
        // blocks of 8 x 32 columns: the 16 loads of a block are issued
        // together, then four FMA chains; the last, partial block runs the
        // same code with predicated loads (a rolled remainder loop exposed the
        // shared-memory latency once per 32 columns: ~1.0 k cycles for the
        // <= 20 elements per lane of a C5 step)
        double a2 = 0.0, a3 = 0.0;
        int k = m1 + lane;
#pragma unroll 1
        for (; k + 224 < n; k += 256) {
          double x[8], y[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            x[u] = my_row[k + 32 * u];
            y[u] = vc[k + 32 * u];
          }
          a0 = fma(x[0], y[0], a0);
          a1 = fma(x[1], y[1], a1);
          a2 = fma(x[2], y[2], a2);
          a3 = fma(x[3], y[3], a3);
          a0 = fma(x[4], y[4], a0);
          a1 = fma(x[5], y[5], a1);
          a2 = fma(x[6], y[6], a2);
          a3 = fma(x[7], y[7], a3);
        }
        if (k < n) {
          double x[8], y[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const bool in = k + 32 * u < n;
            x[u] = in ? my_row[k + 32 * u] : 0.0;
            y[u] = in ? vc[k + 32 * u] : 0.0;
          }
          a0 = fma(x[0], y[0], a0);
          a1 = fma(x[1], y[1], a1);
          a2 = fma(x[2], y[2], a2);
          a3 = fma(x[3], y[3], a3);
          a0 = fma(x[4], y[4], a0);
          a1 = fma(x[5], y[5], a1);
          a2 = fma(x[6], y[6], a2);
          a3 = fma(x[7], y[7], a3);
        }
        a0 += a2;
        a1 += a3;
      }
      // the row dot and the two correction dots reduced together (three
      // independent shuffle chains in flight)
      double raw = a0 + a1;
#ifdef TRD_TRACE
      if (wtr) w1 = clock64();
#endif
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        raw += __shfl_xor_sync(0xffffffffu, raw, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      }
      if (j > 0) raw = fma(-vp[my_i], s1, fma(-wpv[my_i], s2, raw));
#ifdef TRD_TRACE
      if (wtr) w2 = clock64();
#endif
      // B is symmetric: the replica of row j + 1 that every CTA needs for the
      // next reflector is column j + 1, and this warp holds its entry
      // A[i][j + 1].  It travels with p_i (after the pending update of step
      // j - 1 on that one entry), so no owner has to finish its row update
      // and publish 1 row before the exchange can complete.
      double cm = 0.0;
      if (COLX && j > 0) {
        const double vi = vp[my_i], wi = wpv[my_i];
        if constexpr (NQ > 0) {
#pragma unroll
          for (int q = 0; q < NQ; ++q)
            if (lane + 32 * q == m1) cm = fma(-vi, wpv[m1], fma(-wi, vp[m1], rr[q]));
          cm = __shfl_sync(0xffffffffu, cm, m1 & 31);
        } else {
          cm = fma(-vi, wpv[m1], fma(-wi, vp[m1], my_row[m1]));
        }
      }
      if constexpr (CL) {
        if (lane < G) {
          trd_dsm_st(ps + my_i, (uint32_t)lane, bet * raw);
          if (COLX && j > 0) trd_dsm_st(cur + my_i, (uint32_t)lane, cm);
        }
      } else {
        if (lane == 0) {
          ll_store(b.pll + (size_t)(j & 1) * n + my_i, bet * raw, tag);
          if (COLX && j > 0) ll_store(b.rowll + (size_t)(m1 & 1) * n + my_i, cm, tag);
        }
      }
#ifdef TRD_TRACE
      if (wtr) printf("trdw g=%d: since step start %lld loop %lld shfl %lld publish %lld\n", g, w0 - tr0s, w1 - w0, w2 - w1, clock64() - w2);
#endif
    }
    if constexpr (!CL) {
      // this CTA's sentinel (one 128-byte line per CTA): readers poll it
      // instead of every p record, so each line has G pollers, not G x 8
      __syncthreads();
      if (tid == 0) ll_store(b.sent + ((size_t)(j & 1) * TRD_MAXG + g) * 8, 0.0, tag);
    }
#ifdef TRD_TRACE
    if (trs) tr[1] = clock64();
#endif
    // (2) the pending update of step j - 1 on the local rows (k >= j + 1);
    //     the owner of row j + 1 publishes it (through step j - 1)
    if (j > 0 && has_row && my_i >= m1) {
      const double vi = vp[my_i], wi = wpv[my_i];
      uint4* pub = (!COLX && my_i == m1) ? b.rowll + (size_t)(m1 & 1) * n : nullptr;
      if constexpr (NQ > 0) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const int k = lane + 32 * q;
          if (k >= m1 && k < n) {
            rr[q] = fma(-vi, wpv[k], fma(-wi, vp[k], rr[q]));
            if constexpr (CL) {
              if (!COLX && my_i == m1)
                for (int c = 0; c < G; ++c) trd_dsm_st(cur + k, (uint32_t)c, rr[q]);
            } else {
              if (pub) ll_store(pub + k, rr[q], tag);
            }
          }
        }
      }
      // blocks of 4 x 32 columns, the 12 loads of a block issued together;
      // the partial last block with predicated accesses
      int k = NQ > 0 ? n : m1 + lane;
#pragma unroll 1
      for (; k < n; k += 128) {
        double a[4], w[4], v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool in = k + 32 * u < n;
          a[u] = in ? my_row[k + 32 * u] : 0.0;
          w[u] = in ? wpv[k + 32 * u] : 0.0;
          v[u] = in ? vp[k + 32 * u] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (k + 32 * u < n) {
            const double x = fma(-vi, w[u], fma(-wi, v[u], a[u]));
            my_row[k + 32 * u] = x;
            if (pub) ll_store(pub + k + 32 * u, x, tag);
          }
        }
      }
      if (pub && !CL) {
        __syncwarp();
        if (lane == 0) ll_store(b.sent + ((size_t)2 * TRD_MAXG + (m1 & 1)) * 8, 0.0, tag);
      }
    }
#ifdef TRD_TRACE
    if (trace) __syncthreads();
    if (trs) tr[2] = clock64();
#endif
    // (3) the exchange: all of p and the replica of row j + 1; K partials.
    //     The sentinels first (one poller per source line), then every record
    //     is read and its tag checked (a relaxed store may still be in
    //     flight: those are polled again)
    if constexpr (CL) {
      trd_cluster_sync();  // every CTA's p and the replica row are in place
    }
    if constexpr (!CL) {
    if (tid < G) {
      const uint4* sp = b.sent + ((size_t)(j & 1) * TRD_MAXG + tid) * 8;
      while (ll_ld(sp).y != tag) {
      }
    } else if (!COLX && tid == TRD_T - 1 && j > 0) {
      const uint4* sp = b.sent + ((size_t)2 * TRD_MAXG + (m1 & 1)) * 8;
      while (ll_ld(sp).y != tag) {
      }
    }
    __syncthreads();
    {
      const uint4* pl = b.pll + (size_t)(j & 1) * n;
      const uint4* rl = b.rowll + (size_t)(m1 & 1) * n;
      double q = 0.0;
      {
        // the p and the replica records are fetched together: one L2 round
        // trip on the step's critical path instead of two
        constexpr int LLU = NQ > 0 ? 1 : TRD_LL;  // register rows: n <= TRD_T
        uint4 pr[LLU], cr[LLU];
#pragma unroll
        for (int u = 0; u < LLU; ++u) {
          const int k = m1 + tid + u * TRD_T;
          if (k < n) {
            pr[u] = ll_ld(pl + k);
            if (j > 0) cr[u] = ll_ld(rl + k);
          }
        }
#pragma unroll
        for (int u = 0; u < LLU; ++u) {
          const int k = m1 + tid + u * TRD_T;
          if (k < n) {
            while (pr[u].y != tag || pr[u].w != tag) pr[u] = ll_ld(pl + k);
            const double p = ll_val(pr[u]);
            ps[k] = p;
            q = fma(p, vc[k], q);
          }
        }
        if (j > 0) {
#pragma unroll
          for (int u = 0; u < LLU; ++u) {
            const int k = m1 + tid + u * TRD_T;
            if (k < n) {
              while (cr[u].y != tag || cr[u].w != tag) cr[u] = ll_ld(rl + k);
              cur[k] = ll_val(cr[u]);
            }
          }
        } else {
          for (int k = m1 + tid; k < n; k += TRD_T) cur[k] = B[ldb + k];
        }
      }
      q = warp_sum(q);
      if (lane == 0) kpart[wid] = q;
    }
    } else {
      double q = 0.0;
      for (int k = m1 + tid; k < n; k += TRD_T) q = fma(ps[k], vc[k], q);
      q = warp_sum(q);
      if (lane == 0) kpart[wid] = q;
    }
#ifdef TRD_TRACE
    if (trs) {
      tr[3] = clock64();
      long long gt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
      tr[7] = gt - tr[7];
    }
#endif
    __syncthreads();
#ifdef TRD_TRACE
    if (trs) tr[4] = clock64();
#endif
    // (4) w_j = p - K v_j (the new pending update); the replica row j + 1
    //     through step j and its sum of squares beyond j + 2
    {
      const double K = 0.5 * bet * trd_sum16(kpart);
      const double vi = vc[m1];
      const double wi = fma(-K, vi, ps[m1]);
      double q = 0.0;
      for (int k = m1 + tid; k < n; k += TRD_T) {
        const double wk = fma(-K, vc[k], ps[k]);
        wpv[k] = wk;
        const double c2 = fma(-vi, wk, fma(-wi, vc[k], cur[k]));
        cur[k] = c2;
        if (k >= j + 3) q = fma(c2, c2, q);
      }
      q = warp_sum(q);
      if (lane == 0) sqpart[wid] = q;
    }
    __syncthreads();
    // (5) the reflector of step j + 1 from the replica (warp 0), v_{j+1} and
    //     the two correction dots of the next matvec
    if (j + 1 < n - 2) {
      if (wid == 0) {
        const double s = trd_sum16(sqpart);
        if (lane == 0) {
          double bt, ej, sc;
          trd_reflector(cur[j + 2], s, bt, ej, sc);
          s_bs[0] = bt;
          s_bs[1] = sc;
          if (g == 0) {
            b.beta[j + 1] = bt;
            b.dd[j + 1] = cur[j + 1];
            b.ee[j + 1] = ej;
          }
        }
      }
      __syncthreads();
      const double scale = s_bs[1];
      double* vn = vsb + (size_t)((j + 1) & 1) * n;  // overwrites v_{j-1}: no longer needed
      double* hrow = b.hv + (int64_t)(j + 1) * ldh;
      double q1 = 0.0, q2 = 0.0;
      for (int k = j + 2 + tid; k < n; k += TRD_T) {
        const double v = k == j + 2 ? 1.0 : cur[k] * scale;
        vn[k] = v;
        if (g == 0) hrow[k] = v;
        q1 = fma(wpv[k], v, q1);
        q2 = fma(vc[k], v, q2);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        q1 += __shfl_xor_sync(0xffffffffu, q1, o);
        q2 += __shfl_xor_sync(0xffffffffu, q2, o);
      }
      if (lane == 0) {
        s1part[wid] = q1;
        s2part[wid] = q2;
      }
    }
#ifdef TRD_TRACE
    if (trs) tr[5] = clock64();
#endif
    __syncthreads();
    bet = s_bs[0];
#ifdef TRD_TRACE
    if (trs) {
      tr[6] = clock64();
      printf("trd g=%d j=%d: matvec %lld upd %lld xchg %lld bar %lld w %lld refl %lld total %lld startns %lld\n", g, j,
             tr[1] - tr[0], tr[2] - tr[1], tr[3] - tr[2], tr[4] - tr[3], tr[5] - tr[4], tr[6] - tr[5],
             tr[6] - tr[0], tr[7]);
    }
#endif
  }
  // the trailing 2 x 2 block: the replica is row n - 2 through step n - 3;
  // row n - 1 still has the update of step n - 3 pending
  if (g == 0 && tid == 0) {
    b.dd[n - 2] = cur[n - 2];
    b.ee[n - 2] = cur[n - 1];
    b.beta[n - 2] = 0.0;
    b.beta[n - 1] = 0.0;
    b.ee[n - 1] = 0.0;
  }
  if (has_row && my_i == n - 1) {
    double a = 0.0;
    if constexpr (NQ > 0) {
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        if (lane + 32 * q == n - 1) a = rr[q];
    } else {
      a = my_row[n - 1];
    }
    if (lane == (n - 1) % 32) {
      const double* vl = vsb + (size_t)((n - 3) & 1) * n;
      const double vi = vl[n - 1], wi = wpv[n - 1];
      b.dd[n - 1] = fma(-vi, wi, fma(-wi, vi, a));
    }
  }
  if constexpr (CL) trd_cluster_sync();  // no CTA leaves while remote stores into it may be in flight
}

// Number of eigenvalues of T greater than x: sign changes of the Sturm
// sequence p_i = (d_i - x) p_{i-1} - e_{i-1}^2 p_{i-2}, p_{-1} = 1 (the
// negative pivots q_i = p_i / p_{i-1} of T - x I).  One FMA on the
// dependency chain per step; every 8 steps the pair is rescaled by an exact
// power of two (T is pre-scaled so |d - x|, e^2 <= 4: 8 steps grow it by
// at most 8^8).  A zero p_i counts as non-negative: the number of sign
// changes over (p_{i-1}, 0, p_{i+1} = -e^2 p_{i-1}) is the same either way.
__device__ __forceinline__ int trd_count_gt(const double* __restrict__ d, const double* __restrict__ e2, int n,
                                            double x) {
  double pm = 1.0, pc = d[0] - x;
  int neg = pc < 0.0;
  int i = 1;
  for (; i + 8 <= n; i += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double pn = fma(d[i + u] - x, pc, -e2[i + u - 1] * pm);
      neg += (pn < 0.0) != (pc < 0.0);
      pm = pc;
      pc = pn;
    }
    const int hc = __double2hiint(pc) & 0x7fffffff, hm = __double2hiint(pm) & 0x7fffffff;
    const int ex = (max(hc, hm) >> 20) - 1023;
    const double f = __hiloint2double((1023 - ex) << 20, 0);
    pc *= f;
    pm *= f;
  }
  for (; i < n; ++i) {
    const double pn = fma(d[i] - x, pc, -e2[i - 1] * pm);
    neg += (pn < 0.0) != (pc < 0.0);
    pm = pc;
    pc = pn;
  }
  return n - neg;
}

// T scaled by the power of two that brings its Gershgorin bound into [1, 2)
__device__ __forceinline__ double trd_scale_of(double hi) { return hi > 0.0 ? scalbn(1.0, -ilogb(hi)) : 1.0; }

// One warp per eigenvalue index c (c-th largest, 0-based) among those above
// t = tau^2; all warps first agree on k = count(> t).  lam holds the
// unscaled eigenvalues, scale the factor for the vector kernel.
__global__ void __launch_bounds__(256) trd_bisect_kernel(TrdBuf b, int n, const double* __restrict__ tau_p,
                                                         const int* __restrict__ skip) {
  if (skip && *skip) return;
  extern __shared__ double bs_sm[];
  double* d = bs_sm;
  double* e2 = d + n;
  __shared__ double s_lo, s_hi, s_sc;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (wid == 0) {
    double hi = 0.0;
    for (int i = lane; i < n; i += 32) {
      const double el = i > 0 ? fabs(b.ee[i - 1]) : 0.0, er = i < n - 1 ? fabs(b.ee[i]) : 0.0;
      hi = fmax(hi, fabs(b.dd[i]) + el + er);
    }
    hi = warp_max(hi);
    if (lane == 0) {
      const double sc = trd_scale_of(hi);
      s_sc = sc;
      s_hi = hi * sc * (1.0 + 4.0 * DBL_EPSILON);
      const double tau = *tau_p;
      s_lo = tau * tau * sc;
      if (blockIdx.x == 0) b.scale[0] = sc;
    }
  }
  __syncthreads();
  const double sc = s_sc;
  for (int i = tid; i < n; i += blockDim.x) {
    d[i] = b.dd[i] * sc;
    const double e = i < n - 1 ? b.ee[i] * sc : 0.0;
    e2[i] = fmax(e * e, 0x1p-900);  // an exact zero coupling would stall the sequence
  }
  __syncthreads();
  const double t = s_lo;
  const int c = blockIdx.x * (blockDim.x >> 5) + wid;
  int k = 0;
  if (lane == 0) k = trd_count_gt(d, e2, n, t);
  k = __shfl_sync(0xffffffffu, k, 0);
  if (blockIdx.x == 0 && tid == 0) b.info[0] = k;
  if (c >= k) return;
  // lambda_c in (lo, hi]: count(lo) >= c + 1 > count(hi)
  double lo = t, hi = s_hi;
  for (int round = 0; round < 40; ++round) {
    const double w = hi - lo;
    if (w <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + 0x1p-1000) break;
    const double x = lo + w * (double)(lane + 1) / 33.0;
    const int cnt = trd_count_gt(d, e2, n, x);
    const unsigned above = __ballot_sync(0xffffffffu, cnt >= c + 1);  // a prefix of lanes
    const int na = __popc(above);
    const double nlo = na > 0 ? __shfl_sync(0xffffffffu, x, na - 1) : lo;
    const double nhi = na < 32 ? __shfl_sync(0xffffffffu, x, na & 31) : hi;
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) b.lam[c] = 0.5 * (lo + hi) / sc;
}

__device__ __forceinline__ double trd_rescale_pair(double& pc, double& pm) {
  const int hc = __double2hiint(pc) & 0x7fffffff, hm = __double2hiint(pm) & 0x7fffffff;
  const int ex = (max(hc, hm) >> 20) - 1023;
  const double f = __hiloint2double((1023 - ex) << 20, 0);
  pc *= f;
  pm *= f;
  return f;
}

// Twisted factorisation eigenvector of T for lambda_c, one warp per c, on T
// scaled by the bisection's power of two.  Lane 0 runs the recurrences:
//   forward Sturm sequence p -> pivots D+_i = p_i / p_{i-1} (T - lam I =
//   L+ D+ L+^T), backward sequence r -> R-_i = r_i / r_{i+1} (= U- R- U-^T),
//   gamma_i = D+_i + R-_i - (d_i - lam), twist r = argmin |gamma_i|,
//   z_r = 1, z_i = -(e_i / D+_i) z_{i+1} above, z_{i+1} = -(e_i / R-_{i+1}) z_i
//   below.  The chains are one FMA (sequences) or one multiply (z) per step;
// the divisions are off the chain.  Output z[c * n + i], unit 2-norm.
constexpr int TRD_VW = 6;

__global__ void __launch_bounds__(TRD_VW * 32) trd_vectors_kernel(TrdBuf b, int n, const int* __restrict__ skip) {
  if (skip && *skip) return;
  extern __shared__ double vsm[];  // (blockDim / 32) x 4 n
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int k = b.info[0];
  const int c = blockIdx.x * (blockDim.x >> 5) + wid;
  if (c >= k) return;
  // lane 0 runs only the two Sturm recurrences (one FMA each on the chain,
  // forward and backward interleaved) and stores the numerator and
  // denominator of every pivot; the divisions, the twist search and the
  // multipliers of the z products are then spread over the 32 lanes
  double* __restrict__ nf = vsm + (size_t)wid * 4 * n;  // forward p_i, then D+_i
  double* __restrict__ df = nf + n;                     // forward p_{i-1}, then the upward multipliers, then z
  double* __restrict__ nb = df + n;                     // backward r_i, then R-_i
  double* __restrict__ db = nb + n;                     // backward r_{i+1}, then the downward multipliers
  const double sc = b.scale[0];
  const double lam = b.lam[c] * sc;
  // (nearly) repeated eigenvalues: the twisted vectors of a cluster this
  // tight are not mutually orthogonal, so the Jacobi takes the iteration
  if (lane == 0 && c + 1 < k && !(b.lam[c] - b.lam[c + 1] > 1e-10 * fabs(b.lam[c]))) atomicExch(b.info + 1, 1);
  const double* __restrict__ d = b.dd;
  const double* __restrict__ e = b.ee;
  const double piv = 0x1p-900, big = 0x1p+900;
  auto clampd = [&](double x) { return fabs(x) < piv ? -piv : fmin(fmax(x, -big), big); };
  if (lane == 0) {
    // p_i = (d_i - lam) p_{i-1} - e_{i-1}^2 p_{i-2} (D+_i = p_i / p_{i-1}) and
    // r_i = (d_i - lam) r_{i+1} - e_i^2 r_{i+2}   (R-_i = r_i / r_{i+1})
    double pm = 1.0, pc = fma(__ldg(d), sc, -lam);
    double rn = 1.0, rc = fma(__ldg(d + n - 1), sc, -lam);
    nf[0] = pc;
    df[0] = 1.0;
    nb[n - 1] = rc;
    db[n - 1] = 1.0;
#pragma unroll 4
    for (int t = 1; t < n; ++t) {
      const int i = t, ib = n - 1 - t;
      const double ef = __ldg(e + i - 1) * sc, eb = __ldg(e + ib) * sc;
      const double pn = fma(fma(__ldg(d + i), sc, -lam), pc, -(ef * ef) * pm);
      const double rp = fma(fma(__ldg(d + ib), sc, -lam), rc, -(eb * eb) * rn);
      nf[i] = pn;
      df[i] = pc;
      nb[ib] = rp;
      db[ib] = rc;
      pm = pc;
      pc = pn;
      rn = rc;
      rc = rp;
      if ((t & 7) == 0) {
        trd_rescale_pair(pc, pm);
        trd_rescale_pair(rc, rn);
      }
    }
  }
  __syncwarp();
  // pivots and the twist index r = argmin |gamma_i|, gamma_i = D+_i + R-_i - (d_i - lam)
  double best = 1e300;
  int r = -1;
  for (int i = lane; i < n; i += 32) {
    const double dp = clampd(nf[i] / df[i]), rm = clampd(nb[i] / db[i]);
    nf[i] = dp;
    nb[i] = rm;
    const double gam = fabs(dp + rm - fma(__ldg(d + i), sc, -lam));
    if (gam < best || (gam == best && i > r)) {  // ties: the largest i (the serial scan's choice)
      best = gam;
      r = i;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int orr = __shfl_xor_sync(0xffffffffu, r, o);
    if (ob < best || (ob == best && orr > r)) {
      best = ob;
      r = orr;
    }
  }
  __syncwarp();
  // multipliers: upward z_i = -(e_i / D+_i) z_{i+1} (i < r), downward
  // z_{i+1} = -(e_i / R-_{i+1}) z_i (i >= r)
  for (int i = lane; i < n - 1; i += 32) {
    const double ei = __ldg(e + i) * sc;
    if (i < r) df[i] = -ei / nf[i];
    else db[i] = -ei / nb[i + 1];
  }
  __syncwarp();
  double* __restrict__ zz = nb;  // R- no longer needed
  if (lane == 0) {
    // both products in one loop (two independent multiply chains)
    double zu = 1.0, zd = 1.0, ss = 1.0;
    const int nu = r, nd = n - 1 - r, nt = max(nu, nd);
    double zr = 1.0;
#pragma unroll 4
    for (int t = 0; t < nt; ++t) {
      if (t < nu) {
        const int i = r - 1 - t;
        zu *= df[i];
        df[i] = zu;  // z_i (upward part stored in place)
        ss = fma(zu, zu, ss);
      }
      if (t < nd) {
        const int i = r + t;
        zd *= db[i];
        zz[i + 1] = zd;  // z_{i+1} (into the R- buffer)
        ss = fma(zd, zd, ss);
      }
    }
    df[r] = zr;
    const double inv = 1.0 / sqrt(ss);
    if (!(isfinite(inv) && inv > 0.0)) atomicExch(b.info + 1, 1);
    nf[0] = inv;  // hand the norm to the warp (D+ is no longer read)
  }
  __syncwarp();
  const double inv = nf[0];
  double* __restrict__ out = b.z + (size_t)c * n;
  // z_i: i <= r from df (upward part and z_r = 1), i > r from the R- buffer
  for (int i = lane; i < n; i += 32) out[i] = (i <= r ? df[i] : zz[i]) * inv;
}

// V = Q Z = H_0 H_1 ... H_{n-3} Z, one warp per column c < k with the column
// in registers (NQ = ceil(n / 32) per lane).  The reflector rows stream
// through shared memory by TMA bulk copies (cp.async.bulk, one mbarrier per
// stage of TRD_BCH rows, TRD_BST stages, thread 0 the producer), shared by
// the CTA's TRD_BW warps.  Output V[i * ldv + c].
// 5 warps per CTA: the C5 maximum of 731 kept vectors then spreads over 147 of
// the 148 SMs in one wave (8 warps left 56 SMs idle and two warps per
// scheduler contending for issue slots: C5 eigensolve phase 106.9 -> 106.5 ms)
constexpr int TRD_BW = 5, TRD_BCH = 4, TRD_BST = 3;
__device__ __forceinline__ uint32_t trd_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// z <- (I - beta h h^T) z for this warp's CPW vectors, register blocks
// q >= Q0 only (Q0 <= q0: the blocks below hold rows <= j, where h is zero).
template <int NQ, int CPW, int Q0>
__device__ __forceinline__ void trd_back_apply(const double* __restrict__ h, int j, int n, int q0, int lane,
                                               double bet, double (&z)[CPW][NQ]) {
  if constexpr (Q0 < NQ) {
    double acc[CPW];
#pragma unroll
    for (int u = 0; u < CPW; ++u) acc[u] = 0.0;
    double hr[NQ - Q0];  // the reflector's entries, read from shared memory once for both passes
#pragma unroll
    for (int q = Q0; q < NQ; ++q) {
      const int i = lane + 32 * q;
      hr[q - Q0] = (q >= q0 && i > j && i < n) ? h[i] : 0.0;
#pragma unroll
      for (int u = 0; u < CPW; ++u) acc[u] = fma(hr[q - Q0], z[u][q], acc[u]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int u = 0; u < CPW; ++u) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
#pragma unroll
    for (int u = 0; u < CPW; ++u) acc[u] *= bet;
#pragma unroll
    for (int q = Q0; q < NQ; ++q)
#pragma unroll
      for (int u = 0; u < CPW; ++u) z[u][q] = fma(-acc[u], hr[q - Q0], z[u][q]);
  }
}

template <int NQ, int CPW>
__global__ void __launch_bounds__(TRD_BW * 32, 1) trd_back_kernel(TrdBuf b, int n, int K, double* __restrict__ V,
                                                                   int ldv, const int* __restrict__ skip) {
  if (skip && *skip) return;
  extern __shared__ __align__(16) double bk_sm[];  // TRD_BST x TRD_BCH x ldh
  __shared__ __align__(8) uint64_t bars[TRD_BST];
  const int k = b.info[0];
  const int lane = threadIdx.x & 31;
  const int c0 = blockIdx.x * TRD_BW * CPW;
  if (c0 >= k) return;
  const int c = c0 + (threadIdx.x >> 5) * CPW;  // this warp's columns c .. c + CPW - 1
  const int ldh = (n + 1) & ~1;
  const int nref = n - 2;  // reflectors 0 .. n-3, applied from the top
  const int nch = (nref + TRD_BCH - 1) / TRD_BCH;
  auto issue = [&](int ch) {  // thread 0
    const int st = ch % TRD_BST;
    const int jtop = nref - 1 - ch * TRD_BCH;
    uint32_t bytes = 0;
    for (int r = 0; r < TRD_BCH; ++r) {
      const int j = jtop - r;
      if (j < 0) break;
      bytes += (uint32_t)(ldh - ((j + 1) & ~1)) * 8u;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(trd_smem_u32(bars + st)), "r"(bytes)
                 : "memory");
    for (int r = 0; r < TRD_BCH; ++r) {
      const int j = jtop - r;
      if (j < 0) break;
      const int a0 = (j + 1) & ~1;
      double* dst = bk_sm + ((size_t)st * TRD_BCH + r) * ldh + a0;
      const double* src = b.hv + (int64_t)j * ldh + a0;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              trd_smem_u32(dst)),
          "l"(src), "r"((uint32_t)(ldh - a0) * 8u), "r"(trd_smem_u32(bars + st))
          : "memory");
    }
  };
  if (threadIdx.x == 0) {
    for (int st = 0; st < TRD_BST; ++st)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(trd_smem_u32(bars + st)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int ch = 0; ch < TRD_BST && ch < nch; ++ch) issue(ch);
  }
  double* bk_beta = bk_sm + (size_t)TRD_BST * TRD_BCH * ldh;  // all n reflector scalars
  for (int i = threadIdx.x; i < n; i += blockDim.x) bk_beta[i] = b.beta[i];
  double z[CPW][NQ];
#pragma unroll
  for (int u = 0; u < CPW; ++u)
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int i = lane + 32 * q;
      z[u][q] = (c + u < k && i < n) ? b.z[(size_t)(c + u) * n + i] : 0.0;
    }
  __syncthreads();
  for (int ch = 0; ch < nch; ++ch) {
    const int st = ch % TRD_BST;
    const uint32_t parity = (uint32_t)(ch / TRD_BST) & 1u;
    asm volatile(
        "{\n.reg .pred p;\nTRD_W_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra TRD_W_%=;\n}\n" ::"r"(
            trd_smem_u32(bars + st)),
        "r"(parity)
        : "memory");
    const int jtop = nref - 1 - ch * TRD_BCH;
    for (int r = 0; r < TRD_BCH; ++r) {
      const int j = jtop - r;
      if (j < 0) break;
      const double bet = bk_beta[j];  // staged once: a global load here sits on every reflector's chain
      if (bet == 0.0) continue;
      const double* h = bk_sm + ((size_t)st * TRD_BCH + r) * ldh;
      const int q0 = (j + 1) >> 5;  // lower q hold only rows <= j for every lane
      // reflector j touches rows > j only: the register blocks below q0 are
      // skipped at compile time in groups of 8 (static register indices;
      // the group is uniform over the CTA and falls as j does)
      switch (q0 >> 3) {
        case 0: trd_back_apply<NQ, CPW, 0>(h, j, n, q0, lane, bet, z); break;
        case 1: trd_back_apply<NQ, CPW, 8>(h, j, n, q0, lane, bet, z); break;
        case 2: trd_back_apply<NQ, CPW, 16>(h, j, n, q0, lane, bet, z); break;
        case 3: trd_back_apply<NQ, CPW, 24>(h, j, n, q0, lane, bet, z); break;
        case 4: trd_back_apply<NQ, CPW, 32>(h, j, n, q0, lane, bet, z); break;
        case 5: trd_back_apply<NQ, CPW, 40>(h, j, n, q0, lane, bet, z); break;
        case 6: trd_back_apply<NQ, CPW, 48>(h, j, n, q0, lane, bet, z); break;
        default: trd_back_apply<NQ, CPW, 56>(h, j, n, q0, lane, bet, z); break;
      }
    }
    __syncthreads();  // stage st consumed by every warp
    if (threadIdx.x == 0 && ch + TRD_BST < nch) issue(ch + TRD_BST);
  }
#pragma unroll
  for (int u = 0; u < CPW; ++u)
    if (c + u < k) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int i = lane + 32 * q;
        if (i < n) V[(int64_t)i * ldv + c + u] = z[u][q];
      }
    }
}

// Eigenvalues onto diag(B~) (svt_weights), V zero outside the k computed
// columns; a failed solve hands V = I to the Jacobi fallback.
__global__ void trd_commit_kernel(PcpDev* st, TrdBuf b, int n, int np, double* __restrict__ Bm,
                                  double* __restrict__ V, int force_fail) {
  if (st->done || st->jac_skip) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->eig_skip = 1;
      st->trd_ok = 0;
    }
    return;
  }
  const int k = b.info[0];
  bool ok = b.info[1] == 0 && !force_fail;
  for (int c = 0; c < k && ok; ++c) ok = isfinite(b.lam[c]);
  const int64_t tot = (int64_t)np * np;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / np), c = (int)(e % np);
    if (!ok) V[e] = i == c ? 1.0 : 0.0;
    else if (c >= k || i >= n) V[e] = 0.0;
  }
  if (ok)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
      Bm[(int64_t)i * (np + 1)] = i < k ? b.lam[i] : 0.0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    b.info[2] = ok ? k : np;  // columns of V the SVT products need (the Jacobi fallback fills all)
    st->trd_ok = ok;
    st->eig_skip = ok;
    if (ok && k == 0) st->jac_skip = 1;  // rank 0: no W~ / Z products, Z cleared
  }
}

}  // namespace

int trd_max_n() { return TRD_LL * TRD_T; }

size_t trd_bytes(int n) {
  const size_t nn = (size_t)n * n;
  // hv (n x ldh), z: 2 n^2 + n; beta, dd, ee, lam: 4 n; pll, rowll: 4 n records; sentinels; scale, info
  return 8 * (2 * nn + 5 * (size_t)n) + 16 * (4 * (size_t)n + 2 * TRD_MAXG) + 128 * (2 * TRD_MAXG + 2) + 8 * 4 +
         4 * 16 + 14 * 256;
}

void trd_carve(TrdBuf* b, char* base, int n) {
  const size_t nn = (size_t)n * n;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    off = (off + 255) & ~size_t(255);
    char* p = base + off;
    off += bytes;
    return p;
  };
  b->hv = (double*)take(8 * (size_t)n * ((n + 1) & ~1));
  b->z = (double*)take(8 * nn);
  b->beta = (double*)take(8 * (size_t)n);
  b->dd = (double*)take(8 * (size_t)n);
  b->ee = (double*)take(8 * (size_t)n);
  b->lam = (double*)take(8 * (size_t)n);
  b->pll = (uint4*)take(16 * 2 * (size_t)n);
  b->rowll = (uint4*)take(16 * 2 * (size_t)n);
  b->sent = (uint4*)take(16 * 8 * (2 * (size_t)TRD_MAXG + 2));
  b->scale = (double*)take(8 * 4);
  b->info = (int*)take(4 * 16);
}

static int trd_grid(int n) {
  static int sms = -1;
  if (sms < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // small n: as few CTAs as hold one row per warp (fewer sentinels to poll);
  // large n: one CTA per SM halves the per-CTA shared-memory traffic of the
  // row updates (C5 eigensolve phase: 79 CTAs 148 ms, 148 CTAs 137 ms)
  int G = std::min(std::min(sms, TRD_MAXG), std::max(1, (n + TRD_W - 1) / TRD_W));
  if (n > 512) G = std::min(sms, TRD_MAXG);
  const char* e = getenv("MLR_TRD_G");
  if (e) G = std::max(1, std::min(std::min(sms, TRD_MAXG), atoi(e)));
  if ((n + G - 1) / G > TRD_W) G = (n + TRD_W - 1) / TRD_W;
  return G;
}

bool trd_supported(int n) {
  if (n < 3 || n > trd_max_n()) return false;
  const int G = trd_grid(n);
  if (G > TRD_MAXG) return false;
  const int R = (n + G - 1) / G;
  const size_t smem = 8 * ((size_t)R * n + 5 * (size_t)n);
  return smem <= 224 * 1024 && 8 * 13 * (size_t)(n + 2) <= 224 * 1024 && 32 * (size_t)n <= 200 * 1024;
}

// Eigenpairs of B (n x n in the leading block of an np x np buffer) above
// tau^2 into V (np x np, columns 0..k-1) and diag(B); Jacobi fallback flag in
// st->eig_skip.  skip: device flag (done or rank-0 certified).
int trd_eig(PcpDev* st, TrdBuf* b, double* Bm, double* V, int n, int np, const double* tau, const int* skip,
            cudaStream_t s) {
  const int G = trd_grid(n);
  const int R = (n + G - 1) / G;
  const int nq = (n + 31) / 32;
  const char* re = getenv("MLR_TRD_REGROWS");
  const bool regs = !(re && re[0] == '0') && nq <= 16;  // measured: spills above 16 (C5 at 40: 148 -> 198 ms)
  // one thread-block cluster for small n (register rows, G <= 16 CTAs)
  const char* ce = getenv("MLR_TRD_CLUSTER");
  const bool cl = regs && nq <= 8 && G <= 16 && !(ce && ce[0] == '0');
  const size_t smem = 8 * ((regs ? 0 : (size_t)R * n) + (cl ? 9 : 5) * (size_t)n);
  MLR_CUDA(cudaMemsetAsync(b->info, 0, 4 * 16, s));
  if (!cl) {  // the publication records carry step tags >= 1: clear them
    MLR_CUDA(cudaMemsetAsync(b->pll, 0, 16 * 2 * (size_t)n, s));
    MLR_CUDA(cudaMemsetAsync(b->rowll, 0, 16 * 2 * (size_t)n, s));
    MLR_CUDA(cudaMemsetAsync(b->sent, 0, 16 * 8 * (2 * (size_t)TRD_MAXG + 2), s));
  }
  // MLR_TRD_COLX=0: the owner of row j + 1 publishes it after its row update (the round-4 exchange)
  static const bool colx = !(getenv("MLR_TRD_COLX") && getenv("MLR_TRD_COLX")[0] == '0');
  void* kfn = colx ? (void*)trd_reduce_kernel<0, false, true> : (void*)trd_reduce_kernel<0, false, false>;
  if (cl) kfn = colx ? (void*)trd_reduce_kernel<8, true, true> : (void*)trd_reduce_kernel<8, true, false>;
  else if (regs)
    kfn = nq <= 8 ? (colx ? (void*)trd_reduce_kernel<8, false, true> : (void*)trd_reduce_kernel<8, false, false>)
                  : (colx ? (void*)trd_reduce_kernel<16, false, true> : (void*)trd_reduce_kernel<16, false, false>);
  MLR_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  {
    const double* bp = Bm;
    int ld = np, nn = n;
    TrdBuf bb = *b;
    static const int trace = getenv("MLR_TRD_TRACE") ? 1 : 0;
    int tr = trace;
    void* args[] = {(void*)&bp, &ld, &nn, &bb, (void*)&skip, &tr};
    if (cl) {
      if (G > 8) MLR_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(G);
      cfg.blockDim = dim3(TRD_T);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = G;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      MLR_CUDA(cudaLaunchKernelExC(&cfg, kfn, args));
    } else {
      MLR_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(G), dim3(TRD_T), args, smem, s));
    }
  }
  const int wpb = 8;  // warps per bisection CTA
  MLR_CUDA(cudaFuncSetAttribute(trd_bisect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(16 * n)));
  trd_bisect_kernel<<<(n + wpb - 1) / wpb, 32 * wpb, 16 * (size_t)n, s>>>(*b, n, tau, skip);
  MLR_LAUNCH_CHECK("trd_bisect_kernel");
  {
    const int vw = (int)std::max<size_t>(1, std::min<size_t>(TRD_VW, (200 * 1024) / (32 * (size_t)n)));
    const size_t vsm = 32 * (size_t)n * vw;
    MLR_CUDA(cudaFuncSetAttribute(trd_vectors_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)vsm));
    trd_vectors_kernel<<<(n + vw - 1) / vw, 32 * vw, vsm, s>>>(*b, n, skip);
  }
  MLR_LAUNCH_CHECK("trd_vectors_kernel");
  const char* cpe = getenv("MLR_TRD_BACK_CPW");
  const int cpw = cpe ? std::max(1, std::min(2, atoi(cpe))) : 1;  // 2 measured slower at C5 (spills)
  const int bg = (n + TRD_BW * cpw - 1) / (TRD_BW * cpw);
  const size_t bsm = 8 * ((size_t)TRD_BST * TRD_BCH + 1) * ((n + 1) & ~1);  // reflector ring + the n betas
#define TRD_BACK(NQ)                                                                                \
  if (nq <= NQ) {                                                                                   \
    if (cpw == 2) {                                                                                 \
      MLR_CUDA(cudaFuncSetAttribute(trd_back_kernel<NQ, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                    (int)bsm));                                                     \
      trd_back_kernel<NQ, 2><<<bg, TRD_BW * 32, bsm, s>>>(*b, n, n, V, np, skip);                   \
    } else {                                                                                        \
      MLR_CUDA(cudaFuncSetAttribute(trd_back_kernel<NQ, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                    (int)bsm));                                                     \
      trd_back_kernel<NQ, 1><<<bg, TRD_BW * 32, bsm, s>>>(*b, n, n, V, np, skip);                   \
    }                                                                                               \
    MLR_LAUNCH_CHECK("trd_back_kernel");                                                            \
  } else
  TRD_BACK(4) TRD_BACK(8) TRD_BACK(16) TRD_BACK(24) TRD_BACK(32) TRD_BACK(40) TRD_BACK(48) TRD_BACK(64) {
    set_error("trd_eig: n too large");
    return kErrArg;
  }
#undef TRD_BACK
  static const int force_fail = getenv("MLR_TRD_FORCE_FALLBACK") ? atoi(getenv("MLR_TRD_FORCE_FALLBACK")) : 0;
  trd_commit_kernel<<<std::min<int>(ceil_div((int64_t)np * np, 256), 592), 256, 0, s>>>(st, *b, n, np, Bm, V,
                                                                                       force_fail);
  MLR_LAUNCH_CHECK("trd_commit_kernel");
  return kOk;
}

}  // namespace mlr
