// Internal (C++) interfaces between the ABI layer and the kernel files.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <utility>
#include <vector>
#include <string>
#include <type_traits>

namespace mlr {

void set_error(const std::string& msg);

// ---------------------------------------------------------------- gemm
struct GemmSpec {
  int M, N, K;
  const void* A; int64_t lda; bool a_f32; bool trans_a;
  const void* B; int64_t ldb; bool b_f32; bool trans_b;
  void* C; int64_t ldc; bool c_f32;
  int64_t c_slice;  // elements between split-K slices of C
  int splits;
  double alpha;
  const double* kscale;  // optional: op(A)[:, k] *= kscale[k]
  const int* skip;       // optional device flag: kernel is a no-op when *skip != 0
  bool sym;              // C = op(A) op(B) is symmetric (Gram): upper-triangle tiles, mirrored
  const int* klim;       // optional device value: only k < *klim contributes (op(A) columns beyond are zero)
  const int* nlim;       // optional device value: columns >= *nlim of C are not computed (left as they are)
};
int gemm_f64(GemmSpec g, cudaStream_t st);
bool gram128_ok(int n);  // the blocked Gram kernel handles width n (gemm_f64.cu)

// frame-stack layout (frames.cu)
int frames_to_matrix(const uint8_t* frames, int count, int H, int W, bool f32, void* x, int64_t ldx, cudaStream_t st);
int mask_pack(const uint8_t* obs, int64_t ldo, int64_t m, int n, uint32_t* bits, int64_t ldm, cudaStream_t st);
int matrix_to_frames(const void* x, int64_t ldx, bool f32, int count, int H, int W, uint8_t* frames,
                     cudaStream_t st);
int sum_slices(const double* P, int64_t count, int64_t slice, int slices, double* out, cudaStream_t st,
               const int* skip = nullptr);

// 3xTF32 tcgen05 reconstruction Z = A W~ (tc_gemm.cu): TMA tensor maps of A
// and the TF32 hi / lo parts of W~^T, built once per plan
struct TcRecon {
  CUtensorMap mapA, mapBhi, mapBlo;
  int64_t M;
  int np, bn;
  bool ready;
};
int tc_recon_bn(int np);
int tc_recon_setup(TcRecon* r, const float* A, int64_t M, int np, const float* Whi, const float* Wlo);
int tc_recon_run(const TcRecon* r, float* Z, int64_t ldz, const int* skip, cudaStream_t st);
int tc_split_w(const double* Wt, float* hi, float* lo, int np, const int* skip, cudaStream_t st);

// ---------------------------------------------------------------- jacobi

// ---------------------------------------------------------------- chain
// Composite restriction R (n x n_h) in stencil form.  Fine column j has
// weight w0[j] on coarse column c0[j] and w1[j] on c0[j]+1 (w1 may be 0);
// coarse column k gathers fine columns [lo[k], hi[k]).
struct ChainDev {
  int n, nh, np;        // np = n_h rounded up to 64
  int* c0;              // [n]
  double* w0; double* w1;
  float* w0f; float* w1f;
  int* lo; int* hi;     // [nh]
  double* gl;           // LDL^T of G_R = R^T R: multipliers l[k], k < nh-1
  double* gd;           // pivots d[k]
  double* gi;           // dense G_R^{-1}, np x np (zero padded)
  int max_span;         // max hi-lo
  int keys_dense;       // c0 starts at 0, steps by <= 1 and reaches nh-2 (segmented restriction valid)
  int max_run;          // longest run of equal c0
  int reg_lgp;          // > 0: regular chain, c0[j] = max(0, (j+1)/P - 1) with P = 2^reg_lgp, n = n_H * P
  int reg_periodic;     // FP32 weights repeat with period 128 after the first 128 columns (rows.cu fast path)
};

int ldl_solve(const int* skip, const ChainDev& ch, const double* in, double* out, int trans_in,
              cudaStream_t st);
int svt_weights(const int* skip, int np, int nh, bool f32, const void* Bd, const double* tau, double* sig_out,
                double* f_out, int* rank_out, double* nuclear_out, cudaStream_t st);
int64_t jacobi2_qbuf_elems(int np);   // rotation log (doubles)
int64_t jacobi2_qflag_elems(int np);  // rotation-log flags (ints)
int jacobi2_debug_prof(unsigned long long* out8);
int jacobi2_debug_prof2(unsigned long long* out8);
int jacobi2_debug_trace(unsigned long long* buf, int g0, int n);
int jacobi2_eig(bool f32, void* B, void* V, int np, int nrows_v, double tol, double abs_floor_rel, int max_sweeps,
                void* Qbuf, int* qflag, double* off_slots, int* result, const int* skip, cudaStream_t st);

// Optional per-phase CUDA-event timing (enabled by mlr_pcp_set_timing):
// every launch of a phase is bracketed by an event pair on its stream.
enum PcpPhase { kPhGram = 0, kPhPre, kPhJacobi, kPhPost, kPhRecon, kPhUpdate, kPhFinalize, kPhLanczos, kPhCount };

struct PhaseTimer {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[kPhCount];
  std::vector<cudaEvent_t> pool;
  cudaEvent_t open = nullptr;
  cudaEvent_t take() {
    cudaEvent_t e;
    if (!pool.empty()) {
      e = pool.back();
      pool.pop_back();
    } else {
      cudaEventCreate(&e);
    }
    return e;
  }
  void begin(cudaStream_t st) {
    if (!on) return;
    open = take();
    cudaEventRecord(open, st);
  }
  void end(int phase, cudaStream_t st) {
    if (!on || !open) return;
    cudaEvent_t e = take();
    cudaEventRecord(e, st);
    ev[phase].push_back({open, e});
    open = nullptr;
  }
  // total ms and launch count per phase; recycles the events
  void collect(double* ms, int* cnt) {
    for (int ph = 0; ph < kPhCount; ++ph) {
      double s = 0.0;
      for (auto& pr : ev[ph]) {
        float t = 0.f;
        cudaEventSynchronize(pr.second);
        cudaEventElapsedTime(&t, pr.first, pr.second);
        s += t;
        pool.push_back(pr.first);
        pool.push_back(pr.second);
      }
      ms[ph] = s;
      cnt[ph] = (int)ev[ph].size();
      ev[ph].clear();
    }
  }
  ~PhaseTimer() {
    for (auto& v : ev)
      for (auto& pr : v) {
        cudaEventDestroy(pr.first);
        cudaEventDestroy(pr.second);
      }
    for (auto e : pool) cudaEventDestroy(e);
  }
};

}  // namespace mlr
