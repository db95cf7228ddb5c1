// extern "C" boundary (include/mlr_b200.h): chain upload, plan creation over
// caller workspace, and thin wrappers over the pcp.cu / cpcp.cu drivers.
#include <climits>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mlr_b200.h"
#include <cstdlib>

#include "common.cuh"
#include "cpcp.h"
#include "kernels.h"
#include "pcp.h"
#include "spectrum.h"

namespace mlr {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
int cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e);
  return kErrCuda;
}

struct Chain {
  ChainDev d;
  std::vector<void*> allocs;
};

static int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}
static int spec_splits(int64_t m_local, int n) {
  const int64_t t = round_up(n, 64) / 64;
  int64_t splits = ceil_div(2 * sm_count(), t * (t + 1) / 2);
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, m_local / 64));
  return (int)std::max<int64_t>(1, splits);
}

// ------------------------------------------------------------ restrict / prolong
template <typename T>
__global__ void restrict_kernel(ChainDev ch, int64_t m, const T* __restrict__ X, int64_t ldx, T* __restrict__ out) {
  const T* w0 = nullptr;
  const T* w1 = nullptr;
  if constexpr (std::is_same<T, float>::value) { w0 = ch.w0f; w1 = ch.w1f; } else { w0 = ch.w0; w1 = ch.w1; }
  for (int64_t i = blockIdx.x; i < m; i += gridDim.x) {
    const T* row = X + i * ldx;
    for (int k = threadIdx.x; k < ch.np; k += blockDim.x) {
      T a = T(0);
      if (k < ch.nh)
        for (int j = ch.lo[k]; j < ch.hi[k]; ++j) a += row[j] * (ch.c0[j] == k ? w0[j] : w1[j]);
      out[i * ch.np + k] = a;
    }
  }
}

template <typename T>
__global__ void prolong_kernel(ChainDev ch, int64_t m, const T* __restrict__ XH, T* __restrict__ out, int64_t ldo) {
  const T* w0 = nullptr;
  const T* w1 = nullptr;
  if constexpr (std::is_same<T, float>::value) { w0 = ch.w0f; w1 = ch.w1f; } else { w0 = ch.w0; w1 = ch.w1; }
  for (int64_t i = blockIdx.x; i < m; i += gridDim.x) {
    const T* row = XH + i * ch.np;
    for (int j = threadIdx.x; j < ch.n; j += blockDim.x) {
      const int c = ch.c0[j];
      T v = w0[j] * row[c];
      if (c + 1 < ch.np) v += w1[j] * row[c + 1];
      out[i * ldo + j] = v;
    }
  }
}

__global__ void eye_kernel(double* V, int np) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)np * np;
       e += (int64_t)gridDim.x * blockDim.x)
    V[e] = (e / np == e % np) ? 1.0 : 0.0;
}

__global__ void diag_kernel(int np, const double* __restrict__ X, double* __restrict__ lam) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < np) lam[i] = X[(int64_t)i * (np + 1)];
}

// ------------------------------------------------------------ workspace carving
struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(void* b) : base((char*)b) {}
  template <typename P>
  P* take(size_t bytes) {
    off = (off + 255) & ~size_t(255);
    P* p = base ? reinterpret_cast<P*>(base + off) : nullptr;
    off += bytes;
    return p;
  }
};

static void carve_pcp(PcpPlan& p, Carver& c) {
  const int np = p.ch.np, n = p.ch.n;
  const size_t tb = p.f32 ? 4 : 8;
  const size_t nn = (size_t)np * np;
  p.dev = c.take<PcpDev>(sizeof(PcpDev));
  p.lz = c.take<LanczosDev>(sizeof(LanczosDev));
  p.hist = c.take<double>(sizeof(double) * kHistCols * p.max_iters);
  p.A = c.take<void>(tb * (size_t)p.m_local * np);
  p.Z = c.take<void>(tb * (size_t)p.m_local * np);
  p.gram_part = c.take<double>(sizeof(double) * nn * p.gram_splits);
  p.row_part = c.take<double>(sizeof(double) * 4 * p.row_blocks);
  p.T1 = c.take<double>(8 * nn);
  p.Bm = c.take<double>(8 * nn);
  p.Xm = c.take<double>(8 * nn);
  p.Vm = c.take<double>(8 * nn);
  p.Wm = c.take<double>(8 * nn);
  if (p.tc_recon) {
    p.w_hi = c.take<float>(4 * nn);
    p.w_lo = c.take<float>(4 * nn);
  }
  p.sig = c.take<double>(8 * np);
  p.fw = c.take<double>(8 * np);
  p.qbuf = c.take<double>(8 * (size_t)jacobi2_qbuf_elems(np));
  p.qflag = c.take<int>(4 * (size_t)jacobi2_qflag_elems(np));
  p.jac_off = c.take<double>(8 * 4);
  p.jac_result = c.take<int>(4 * 16);
  p.lzQ = c.take<double>(8 * (size_t)n * (p.lz_kmax + 1));
  p.lzT = c.take<double>(8 * (size_t)std::max<int64_t>(p.m_local, 1));
  p.lzW = c.take<double>(8 * (size_t)n *
                         std::max(std::max(std::max(p.lz_splits, p.lz_fused_ctas), p.lz_run_ctas), p.lz_long_clusters));
  p.lzRed = c.take<double>(8 * (size_t)std::max(p.lz_run_ctas, 1) * (2 * ((size_t)p.lz_kmax + 1) + 4));
  p.lzWork = c.take<double>(8 * (size_t)n);
  if (p.trd_on) trd_carve(&p.trd, c.take<char>(trd_bytes(p.ch.nh)), p.ch.nh);
}

// K slices of the blocked 128x128 Gram (one CTA per SM).  Small Grams (few
// blocks) take one wave of sms / blocks slices; large ones (C5: 55 blocks)
// the slice count whose CTA count best fills whole waves (C5: 8 slices ->
// 440 CTAs = 2.97 waves of 148; the old one-wave rule gave 2 slices -> 110
// CTAs on 148 SMs).
static int64_t gram128_splits(int64_t b128, int sms, int64_t m_local) {
  if (4 * b128 <= sms) return std::max<int64_t>(1, sms / b128);
  int64_t best = 1;
  double best_e = 0.0;
  for (int64_t s = 1; s <= 16; ++s) {
    if (s > 1 && m_local / s < 512) break;
    const int64_t ctas = b128 * s;
    const double e = (double)ctas / (double)(ceil_div(ctas, (int64_t)sms) * sms);
    if (e > best_e + 0.02) {
      best_e = e;
      best = s;
    }
  }
  const char* env = getenv("MLR_GRAM_SPLITS");
  return env ? std::max(1, atoi(env)) : best;
}

static void pcp_params(PcpPlan& p, const ChainDev& ch, int64_t m_local, int64_t m_global, int f32, int max_iters) {
  p = PcpPlan{};
  p.ch = ch;
  p.f32 = f32 != 0;
  p.m_local = m_local;
  p.m_global = m_global;
  p.max_iters = max_iters;
  const int sms = sm_count();
  p.row_blocks = (int)std::max<int64_t>(1, std::min<int64_t>(m_local, (int64_t)sms * 8));
  const int64_t tiles = (int64_t)(ch.np / 64) * (ch.np / 64 + 1) / 2;  // symmetric Gram: upper-triangle tiles
  int64_t splits = ceil_div(2 * sms, tiles);
  if (gram128_ok(ch.np)) {  // blocked Gram (gemm_f64.cu): about one CTA per SM
    const int64_t b128 = (int64_t)(ch.np / 128) * (ch.np / 128 + 1) / 2;
    splits = gram128_splits(b128, sms, m_local);
  }
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, m_local / 64));
  p.gram_splits = (int)std::max<int64_t>(1, splits);
  {
    // coarse n_p^3 products: about one CTA per SM, K chunks of >= 32
    const int64_t t2 = (int64_t)(ch.np / 64) * (ch.np / 64);
    int64_t ks = std::min<int64_t>(ceil_div(sms, t2), ch.np / 32);
    const char* e = getenv("MLR_COARSE_KSPLIT");
    if (e) ks = atoi(e);
    p.coarse_ksplit = (int)std::max<int64_t>(1, std::min<int64_t>(ks, p.gram_splits));
  }
  const int64_t col_blocks = ceil_div(ch.n, 2048);  // lz_dtv_kernel tiles: row blocks x 2048 columns
  int64_t ls = ceil_div(2 * sms, col_blocks);
  ls = std::min<int64_t>(ls, std::max<int64_t>(1, m_local / 32));
  p.lz_splits = (int)std::max<int64_t>(1, ls);
  {
    const char* e = getenv("MLR_LZ_FUSED");
    const bool fused = ch.n <= 2048 && !(e && e[0] == '0');
    p.lz_fused_ctas = fused ? (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(std::max<int64_t>(m_local, 1), 8), sms))
                            : 0;
    const char* lg = getenv("MLR_LZ_LONG");
    // n <= 2 CTAs x 512 threads x 5 float4 groups (20480); seg x 4 B per stage, >= 4 stages
    p.lz_long_clusters = (f32 && ch.n > 2048 && ch.n % 4 == 0 && ch.n <= 20480 && !(lg && lg[0] == '0'))
                             ? sms / 2 : 0;
    const char* r = getenv("MLR_LZ_RUN");
    p.lz_run_ctas = (ch.n <= 4096 && m_local > 0 && !(r && r[0] == '0')) ? sms : 0;
    const char* rc = getenv("MLR_LZ_RUN_CTAS");
    if (p.lz_run_ctas && rc) p.lz_run_ctas = std::max(1, std::min(sms, atoi(rc)));
  }
  p.lz_kmax = std::min(500, std::max(8, ch.n));
  {
    const char* e = getenv("MLR_TC_RECON");
    p.tc_recon = f32 && tc_recon_bn(ch.np) > 0 && !(e && e[0] == '0');
  }
  {
    const char* e = getenv("MLR_EIG_SORT");
    p.eig_sort = e ? atoi(e) : 1;  // measured: C2 Jacobi -7%, C5 -6%
  }
  p.jac_tol_host = 1e-14;
  p.jac_max_sweeps = 60;
  {
    // coarse eigensolver: the tridiagonal solver (trd.cu) unless MLR_EIG=jacobi
    // (the warm-started block Jacobi).  Measured on B200 (eigensolve phase per
    // solve, trd vs Jacobi): C1 17.8 vs 24.9 ms, C2 26.7 vs 29.5 ms, C5 145 vs
    // 257 ms
    const char* e = getenv("MLR_EIG");
    const bool want = !(e && std::string(e) == "jacobi");
    p.trd_on = want && trd_supported(ch.nh);
  }
}

static void carve_cpcp(CpcpPlan& p, Carver& c) {
  const int np = p.ch.np;
  const size_t tb = p.f32 ? 4 : 8;
  const size_t nn = (size_t)np * np;
  p.dev = c.take<CpcpDev>(sizeof(CpcpDev));
  p.hist = c.take<double>(sizeof(double) * kCpHistCols * p.max_iters);
  p.obj = c.take<double>(sizeof(double) * p.max_iters);
  p.LH = c.take<void>(tb * (size_t)p.m_local * np);
  p.GH = c.take<void>(tb * (size_t)p.m_local * np);
  p.SH = c.take<void>(tb * (size_t)p.m_local * np);
  p.u = c.take<double>(8 * (size_t)std::max<int64_t>(p.m_local, 1));
  p.v = c.take<double>(8 * np);
  p.vin = c.take<double>(8 * np);
  p.gram_part = c.take<double>(8 * (p.fine ? 1 : nn * p.gram_splits));
  p.row_part = c.take<double>(8 * 9 * (size_t)p.row_blocks);
  p.dots_part = c.take<double>(8 * 3 * (size_t)p.row_blocks);
  if (p.coarse_dots) {
    p.mgd = c.take<void>(tb * (size_t)std::max<int64_t>(p.m_local, 1) * np);
    p.mgo = c.take<void>(tb * (size_t)std::max<int64_t>(p.m_local, 1) * np);
  }
  if (p.fine) {
    p.ft = c.take<double>(8 * (size_t)std::max<int64_t>(p.m_local, 1));
    p.fz = c.take<double>(8 * np);
    p.fv0 = c.take<double>(8 * np);
    p.fzpart = c.take<double>(8 * (size_t)p.fine_ctas * np);
    p.fspart = c.take<double>(8 * 2 * (size_t)p.fine_ctas);
  }
}

static void cpcp_params(CpcpPlan& p, const ChainDev& ch, int64_t m_local, int64_t m_global, int64_t row0, int f32,
                        int max_iters, int world) {
  p = CpcpPlan{};
  p.ch = ch;
  p.f32 = f32 != 0;
  p.m_local = m_local;
  p.m_global = m_global;
  p.row0 = row0;
  p.max_iters = max_iters;
  p.world = world;
  const int sms = sm_count();
  p.row_blocks = (int)std::max<int64_t>(1, std::min<int64_t>(m_local, (int64_t)sms * 8));
  const int64_t tiles = (int64_t)(ch.np / 64) * (ch.np / 64 + 1) / 2;  // symmetric Gram: upper-triangle tiles
  int64_t splits = ceil_div(2 * sms, tiles);
  if (gram128_ok(ch.np)) {  // blocked Gram (gemm_f64.cu): about one CTA per SM
    const int64_t b128 = (int64_t)(ch.np / 128) * (ch.np / 128 + 1) / 2;
    splits = gram128_splits(b128, sms, m_local);
  }
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, m_local / 64));
  p.gram_splits = (int)std::max<int64_t>(1, splits);
  p.cluster = ch.np >= 256 ? 16 : 8;
  // full width (identity chain) on one rank: matvec power passes, no Gram
  const char* e = getenv("MLR_CPCP_FINE");
  p.fine = ch.nh == ch.n && world == 1 && !(e && e[0] == '0');
  p.fine_ctas = sms;
  const char* cd = getenv("MLR_CPCP_COARSE_DOTS");
  p.coarse_dots = !(cd && cd[0] == '0');
}

}  // namespace mlr

using namespace mlr;

extern "C" {

int mlr_version(void) { return 1; }

// debug: cycle breakdown of the Jacobi kernel (CTA 0); resets the counters
int mlr_debug_j2prof(unsigned long long* out8) { return mlr::jacobi2_debug_prof(out8); }
int mlr_box_qp_batch(const double* in6, double* out2, int count, void* stream) {
  return mlr::box_qp_batch(in6, out2, count, (cudaStream_t)stream);
}
int mlr_debug_j2prof2(unsigned long long* out8) { return mlr::jacobi2_debug_prof2(out8); }
int mlr_debug_j2trace(unsigned long long* buf, int g0, int n) { return mlr::jacobi2_debug_trace(buf, g0, n); }
const char* mlr_last_error(void) { return g_err.c_str(); }
int mlr_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int mlr_chain_create(int n, int nh, const int32_t* c0, const double* w0, const double* w1, const double* g_diag,
                     const double* g_off, void** chain_out) {
  if (n < 1 || nh < 1 || nh > n || !c0 || !w0 || !w1 || !g_diag || !chain_out) {
    set_error("mlr_chain_create: invalid arguments");
    return kErrArg;
  }
  const int np = (int)round_up(nh, 64);
  std::vector<int> lo(nh, n), hi(nh, 0);
  for (int j = 0; j < n; ++j) {
    const int c = c0[j];
    if (c < 0 || c >= nh || (w1[j] != 0.0 && c + 1 >= nh)) {
      set_error("mlr_chain_create: stencil index out of range");
      return kErrArg;
    }
    if (j > 0 && c < c0[j - 1]) {
      set_error("mlr_chain_create: stencil columns must be non-decreasing");
      return kErrArg;
    }
    lo[c] = std::min(lo[c], j);
    hi[c] = std::max(hi[c], j + 1);
    if (w1[j] != 0.0) {
      lo[c + 1] = std::min(lo[c + 1], j);
      hi[c + 1] = std::max(hi[c + 1], j + 1);
    }
  }
  int span = 0;
  for (int k = 0; k < nh; ++k) {
    if (hi[k] <= lo[k]) {
      lo[k] = 0;
      hi[k] = 0;
    }
    span = std::max(span, hi[k] - lo[k]);
  }
  // LDL^T of the SPD tridiagonal G_R
  std::vector<double> gl(std::max(nh - 1, 1), 0.0), gd(nh);
  gd[0] = g_diag[0];
  for (int k = 1; k < nh; ++k) {
    gl[k - 1] = g_off[k - 1] / gd[k - 1];
    gd[k] = g_diag[k] - gl[k - 1] * g_off[k - 1];
  }
  for (int k = 0; k < nh; ++k)
    if (!(gd[k] > 0.0)) {
      set_error("mlr_chain_create: R^T R is not positive definite");
      return kErrArg;
    }
  std::vector<float> w0f(n), w1f(n);
  for (int j = 0; j < n; ++j) {
    w0f[j] = (float)w0[j];
    w1f[j] = (float)w1[j];
  }
  Chain* ch = new Chain();
  ChainDev& d = ch->d;
  d.n = n;
  d.nh = nh;
  d.np = np;
  d.max_span = span;
  {
    bool dense = n > 0 && c0[0] == 0 && c0[n - 1] >= nh - 2;
    for (int j = 1; j < n && dense; ++j) dense = c0[j] - c0[j - 1] <= 1;
    d.keys_dense = dense ? 1 : 0;
    int run = 0, best = 0;
    for (int j = 0; j < n; ++j) {
      run = (j > 0 && c0[j] == c0[j - 1]) ? run + 1 : 1;
      best = std::max(best, run);
    }
    d.max_run = best;
    // regular chain (repeated halving, n = n_H * 2^L): c0[j] = max(0, (j+1)/P - 1)
    // and no w1 weight on the first fine column of a run; the row kernels then
    // restrict with fixed lane groups instead of the general segmented scan
    d.reg_lgp = 0;
    const char* env = getenv("MLR_REG_CHAIN");
    if (nh >= 2 && n % nh == 0 && !(env && env[0] == '0')) {
      const int P = n / nh;
      int lg = 0;
      while ((1 << lg) < P) ++lg;
      bool reg = (1 << lg) == P && P >= 2 && P <= 64;
      for (int j = 0; j < n && reg; ++j) {
        reg = c0[j] == std::max(0, (j + 1) / P - 1);
        if ((j + 1) % P == 0 || j < P - 1) reg = reg && w1[j] == 0.0;
      }
      if (reg) d.reg_lgp = lg;
    }
    // FP32 stencil weights of column j >= 128 equal those of 128 + j % 128
    d.reg_periodic = 0;
    if (d.reg_lgp > 0) {
      bool per = true;
      for (int j = 256; j < n && per; ++j) per = w0f[j] == w0f[128 + j % 128] && w1f[j] == w1f[128 + j % 128];
      d.reg_periodic = per ? 1 : 0;
    }
  }
  auto up = [&](void** dst, const void* src, size_t bytes) -> int {
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(bytes, 8));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(chain)");
    ch->allocs.push_back(p);
    e = cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(chain)");
    *dst = p;
    return kOk;
  };
  int rc = 0;
  std::vector<int> c0v(c0, c0 + n);
  rc |= up((void**)&d.c0, c0v.data(), sizeof(int) * n);
  rc |= up((void**)&d.w0, w0, sizeof(double) * n);
  rc |= up((void**)&d.w1, w1, sizeof(double) * n);
  rc |= up((void**)&d.w0f, w0f.data(), sizeof(float) * n);
  rc |= up((void**)&d.w1f, w1f.data(), sizeof(float) * n);
  rc |= up((void**)&d.lo, lo.data(), sizeof(int) * nh);
  rc |= up((void**)&d.hi, hi.data(), sizeof(int) * nh);
  rc |= up((void**)&d.gl, gl.data(), sizeof(double) * gl.size());
  rc |= up((void**)&d.gd, gd.data(), sizeof(double) * nh);
  {
    // G_R^{-1} column by column from the LDL^T factors (cond(G_R) <= 5)
    std::vector<double> gi((size_t)np * np, 0.0), col(nh);
    for (int c = 0; c < nh; ++c) {
      for (int k = 0; k < nh; ++k) col[k] = (k == c) ? 1.0 : 0.0;
      for (int k = 1; k < nh; ++k) col[k] -= gl[k - 1] * col[k - 1];
      col[nh - 1] /= gd[nh - 1];
      for (int k = nh - 2; k >= 0; --k) col[k] = col[k] / gd[k] - gl[k] * col[k + 1];
      for (int k = 0; k < nh; ++k) gi[(size_t)k * np + c] = col[k];
    }
    rc |= up((void**)&d.gi, gi.data(), sizeof(double) * gi.size());
  }
  if (rc) {
    for (void* p : ch->allocs) cudaFree(p);
    delete ch;
    return kErrCuda;
  }
  *chain_out = ch;
  return kOk;
}

int mlr_chain_destroy(void* chain) {
  if (!chain) return kOk;
  Chain* ch = (Chain*)chain;
  for (void* p : ch->allocs) cudaFree(p);
  delete ch;
  return kOk;
}

int mlr_chain_padded_width(void* chain) { return chain ? ((Chain*)chain)->d.np : 0; }

int mlr_restrict(void* chain, int64_t m, int f32, const void* X, int64_t ldx, void* out, void* stream) {
  if (!chain || m < 0) { set_error("mlr_restrict: invalid arguments"); return kErrArg; }
  if (m == 0) return kOk;
  const ChainDev& ch = ((Chain*)chain)->d;
  int blocks = (int)std::min<int64_t>(m, sm_count() * 8);
  if (f32) restrict_kernel<float><<<blocks, 256, 0, (cudaStream_t)stream>>>(ch, m, (const float*)X, ldx, (float*)out);
  else restrict_kernel<double><<<blocks, 256, 0, (cudaStream_t)stream>>>(ch, m, (const double*)X, ldx, (double*)out);
  MLR_LAUNCH_CHECK("restrict_kernel");
  return kOk;
}

int mlr_prolong(void* chain, int64_t m, int f32, const void* XH, void* out, int64_t ldo, void* stream) {
  if (!chain || m < 0) { set_error("mlr_prolong: invalid arguments"); return kErrArg; }
  if (m == 0) return kOk;
  const ChainDev& ch = ((Chain*)chain)->d;
  int blocks = (int)std::min<int64_t>(m, sm_count() * 8);
  if (f32) prolong_kernel<float><<<blocks, 256, 0, (cudaStream_t)stream>>>(ch, m, (const float*)XH, (float*)out, ldo);
  else prolong_kernel<double><<<blocks, 256, 0, (cudaStream_t)stream>>>(ch, m, (const double*)XH, (double*)out, ldo);
  MLR_LAUNCH_CHECK("prolong_kernel");
  return kOk;
}

int64_t mlr_matrix_stats_work_doubles(void) { return 3 * 148 * 8 + 64; }

int mlr_matrix_stats(int64_t m, int n, int f32, const void* D, int64_t ldd, double* out3, double* work,
                     void* stream) {
  int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(m, 148 * 8));
  return matrix_stats(m, n, f32 != 0, D, ldd, work, blocks, out3, (cudaStream_t)stream);
}

int64_t mlr_eigh_work_doubles(int np) {
  return (int64_t)np * np + jacobi2_qbuf_elems(np) + jacobi2_qflag_elems(np) / 2 + 64;
}

int mlr_eigh_psd(int np, const double* B, double* V, double* lam, double tol, int max_sweeps, double* work,
                 int* info, void* stream) {
  if (np <= 0 || np % 64) { set_error("mlr_eigh_psd: np must be a positive multiple of 64"); return kErrArg; }
  cudaStream_t st = (cudaStream_t)stream;
  double* X = work;
  double* qbuf = X + (int64_t)np * np;
  double* off = qbuf + jacobi2_qbuf_elems(np);
  int* res = (int*)(off + 4);
  int* qflag = res + 16;
  MLR_CUDA(cudaMemcpyAsync(X, B, sizeof(double) * np * np, cudaMemcpyDeviceToDevice, st));
  eye_kernel<<<256, 256, 0, st>>>(V, np);
  MLR_LAUNCH_CHECK("eye_kernel");
  int rc = jacobi2_eig(false, X, V, np, np, tol, 1e-17, max_sweeps, qbuf, qflag, off, res, nullptr, st);
  if (rc) return rc;
  diag_kernel<<<(np + 127) / 128, 128, 0, st>>>(np, X, lam);
  MLR_LAUNCH_CHECK("diag_kernel");
  MLR_CUDA(cudaMemcpyAsync(info, res, sizeof(int), cudaMemcpyDeviceToHost, st));
  MLR_CUDA(cudaStreamSynchronize(st));
  return kOk;
}

// ---------------------------------------------------------------- PCP
int64_t mlr_pcp_workspace_bytes(void* chain, int64_t m_local, int f32, int max_iters) {
  if (!chain) return -1;
  PcpPlan p;
  pcp_params(p, ((Chain*)chain)->d, m_local, m_local, f32, max_iters);
  Carver c(nullptr);
  carve_pcp(p, c);
  return (int64_t)c.off + 256;
}

int mlr_pcp_create(void* chain, int64_t m_local, int64_t m_global, int f32, int max_iters, void* workspace,
                   void** plan_out) {
  if (!chain || !workspace || !plan_out || m_local < 0 || m_global < 1 || max_iters < 1) {
    set_error("mlr_pcp_create: invalid arguments");
    return kErrArg;
  }
  PcpPlan* p = new PcpPlan();
  pcp_params(*p, ((Chain*)chain)->d, m_local, m_global, f32, max_iters);
  Carver c(workspace);
  carve_pcp(*p, c);
  if (p->tc_recon && m_local > 0) {
    const int rc = tc_recon_setup(&p->tc, (const float*)p->A, m_local, p->ch.np, p->w_hi, p->w_lo);
    if (rc) {
      delete p;
      return rc;
    }
  }
  eye_kernel<<<256, 256>>>(p->Vm, p->ch.np);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    delete p;
    return cuda_fail(e, "mlr_pcp_create");
  }
  *plan_out = p;
  return kOk;
}

int mlr_pcp_destroy(void* plan) {
  delete (PcpPlan*)plan;
  return kOk;
}

int64_t mlr_pcp_red_doubles(void* plan) {
  PcpPlan* p = (PcpPlan*)plan;
  return std::max<int64_t>((int64_t)p->ch.np * p->ch.np + 8, p->ch.n + 8);
}

#define PLAN ((PcpPlan*)plan)
#define STREAM ((cudaStream_t)stream)

int mlr_pcp_input_stats(void* plan, const void* D, int64_t ldd, double* out2, void* stream) {
  return pcp_input_stats(PLAN, D, ldd, out2, STREAM);
}
int mlr_pcp_lanczos_init(void* plan, void* stream) { return pcp_lanczos_init(PLAN, STREAM); }
int mlr_pcp_lanczos_matvec(void* plan, const void* D, int64_t ldd, double* w_part, void* stream) {
  return pcp_lanczos_matvec(PLAN, D, ldd, w_part, STREAM);
}
int mlr_pcp_lanczos_update(void* plan, const double* w, double tol, void* stream) {
  return pcp_lanczos_update(PLAN, w, tol, STREAM);
}
int mlr_pcp_lanczos_run(void* plan, const void* D, int64_t ldd, double tol, void* stream) {
  return pcp_lanczos_run(PLAN, D, ldd, tol, STREAM);
}
int mlr_pcp_lanczos_run_available(void* plan) { return lanczos_run_ok(PLAN); }
int mlr_pcp_lanczos_state(void* plan, double* out4, void* stream) {
  LanczosDev h;
  MLR_CUDA(cudaMemcpyAsync(&h, PLAN->lz, sizeof(LanczosDev), cudaMemcpyDeviceToHost, STREAM));
  MLR_CUDA(cudaStreamSynchronize(STREAM));
  out4[0] = h.k;
  out4[1] = h.done;
  out4[2] = h.sigma1;
  out4[3] = h.theta;
  return kOk;
}
int mlr_pcp_start(void* plan, const void* D, int64_t ldd, void* Y0, int64_t ldy, const double* in_stats, double lam,
                  double mu0, double rho, double tol, int max_iters, double time_budget, double jac_tol,
                  int jac_max_sweeps, void* stream) {
  if (max_iters > PLAN->max_iters) {
    set_error("mlr_pcp_start: max_iters exceeds the plan's history capacity");
    return kErrArg;
  }
  PLAN->jac_max_sweeps = jac_max_sweeps;
  return pcp_start(PLAN, D, ldd, Y0, ldy, in_stats, lam, mu0, rho, tol, max_iters, time_budget, jac_tol, STREAM);
}
int mlr_pcp_gram(void* plan, double* red, int with_stats, void* stream) {
  return pcp_gram(PLAN, red, with_stats, STREAM);
}
int mlr_pcp_finalize(void* plan, const double* red, void* stream) { return pcp_finalize(PLAN, red, STREAM); }
int mlr_pcp_svt(void* plan, const double* red, void* stream) { return pcp_svt(PLAN, red, STREAM); }
int mlr_pcp_update(void* plan, const void* D, int64_t ldd, const void* Y_in, void* Y_out, int64_t ldy, void* stream) {
  return pcp_update(PLAN, D, ldd, Y_in, Y_out, ldy, STREAM);
}
int mlr_pcp_outputs(void* plan, const void* D, int64_t ldd, const void* Y_prev, int64_t ldy, void* L, void* S,
                    int64_t ldo, void* stream) {
  return pcp_outputs(PLAN, D, ldd, Y_prev, ldy, L, S, ldo, STREAM);
}
static void pcp_state_values(const PcpDev& h, double* out16) {
  double v[16] = {(double)h.k, (double)h.done, (double)h.status, (double)h.rank, h.mu, h.mu_final, h.mu_last,
                  h.nuclear, h.sigma1, h.d_norm, (double)h.jac_sweeps, h.tau, h.scale, h.lam, 0.0, 0.0};
  std::memcpy(out16, v, sizeof(v));
}
int mlr_pcp_state(void* plan, double* out16, void* stream) {
  PcpDev h;
  MLR_CUDA(cudaMemcpyAsync(&h, PLAN->dev, sizeof(PcpDev), cudaMemcpyDeviceToHost, STREAM));
  MLR_CUDA(cudaStreamSynchronize(STREAM));
  pcp_state_values(h, out16);
  return kOk;
}
int64_t mlr_pcp_snapshot_bytes(void) { return (int64_t)(sizeof(PcpDev) + sizeof(LanczosDev)); }
int mlr_pcp_snapshot(void* plan, void* host, void* stream) {
  if (!host) {
    set_error("mlr_pcp_snapshot: null buffer");
    return kErrArg;
  }
  MLR_CUDA(cudaMemcpyAsync(host, PLAN->dev, sizeof(PcpDev), cudaMemcpyDeviceToHost, STREAM));
  MLR_CUDA(cudaMemcpyAsync((char*)host + sizeof(PcpDev), PLAN->lz, sizeof(LanczosDev), cudaMemcpyDeviceToHost,
                           STREAM));
  return kOk;
}
int mlr_pcp_snapshot_read(const void* host, double* out16, double* lz4) {
  PcpDev h;
  LanczosDev z;
  std::memcpy(&h, host, sizeof(PcpDev));
  std::memcpy(&z, (const char*)host + sizeof(PcpDev), sizeof(LanczosDev));
  if (out16) pcp_state_values(h, out16);
  if (lz4) {
    lz4[0] = z.k;
    lz4[1] = z.done;
    lz4[2] = z.sigma1;
    lz4[3] = z.theta;
  }
  return kOk;
}
int mlr_pcp_set_truncation(void* plan, int sv0, int cap) {
  if (sv0 < 0 || (sv0 > 0 && cap < 1)) {
    set_error("mlr_pcp_set_truncation: invalid arguments");
    return kErrArg;
  }
  PLAN->trunc_sv0 = sv0 > 0 ? std::min(sv0, cap) : 0;
  PLAN->trunc_cap = cap;
  return kOk;
}
int mlr_pcp_set_timing(void* plan, int enable) {
  PLAN->timer.on = enable != 0;
  return kOk;
}
int mlr_pcp_timing(void* plan, double* ms, int* counts) {
  PLAN->timer.collect(ms, counts);
  return kOk;
}
int mlr_pcp_history(void* plan, int count, double* out, void* stream) {
  if (count < 0 || count > PLAN->max_iters) { set_error("mlr_pcp_history: bad count"); return kErrArg; }
  MLR_CUDA(cudaMemcpyAsync(out, PLAN->hist, sizeof(double) * kHistCols * count, cudaMemcpyDeviceToHost, STREAM));
  MLR_CUDA(cudaStreamSynchronize(STREAM));
  return kOk;
}
#undef PLAN

// ---------------------------------------------------------------- CPCP
#define PLAN ((CpcpPlan*)plan)
int64_t mlr_cpcp_workspace_bytes(void* chain, int64_t m_local, int f32, int max_iters) {
  if (!chain) return -1;
  CpcpPlan p;
  cpcp_params(p, ((Chain*)chain)->d, m_local, m_local, 0, f32, max_iters, 1);
  Carver c(nullptr);
  carve_cpcp(p, c);
  return (int64_t)c.off + 256;
}
int mlr_cpcp_create(void* chain, int64_t m_local, int64_t m_global, int64_t row0, int f32, int max_iters, int world,
                    void* workspace, void** plan_out) {
  if (!chain || !workspace || !plan_out || m_local < 0 || m_global < 1 || max_iters < 1 || world < 1) {
    set_error("mlr_cpcp_create: invalid arguments");
    return kErrArg;
  }
  CpcpPlan* p = new CpcpPlan();
  cpcp_params(*p, ((Chain*)chain)->d, m_local, m_global, row0, f32, max_iters, world);
  if (p->ch.np % p->cluster) {
    delete p;
    set_error("mlr_cpcp_create: coarse width not divisible by the cluster size");
    return kErrArg;
  }
  Carver c(workspace);
  carve_cpcp(*p, c);
  *plan_out = p;
  return kOk;
}
int mlr_cpcp_destroy(void* plan) {
  delete (CpcpPlan*)plan;
  return kOk;
}
int64_t mlr_cpcp_red_doubles(void* plan) { return (int64_t)PLAN->ch.np * PLAN->ch.np + 8; }
int mlr_cpcp_start(void* plan, const void* D, int64_t ldd, const uint32_t* mask, int64_t ldm, void* S, int64_t lds,
                   double lambda_l, double lambda_s, double tol, double radius, int max_iters, double time_budget,
                   void* stream) {
  if (max_iters > PLAN->max_iters) {
    set_error("mlr_cpcp_start: max_iters exceeds the plan's history capacity");
    return kErrArg;
  }
  return cpcp_start(PLAN, D, ldd, mask, ldm, S, lds, lambda_l, lambda_s, tol, radius, max_iters, time_budget,
                    STREAM);
}
int mlr_cpcp_gram(void* plan, double* red, double* amax, void* stream) { return cpcp_gram(PLAN, red, amax, STREAM); }
int mlr_cpcp_begin(void* plan, const double* red, const double* amax_all, void* stream) {
  return cpcp_begin(PLAN, red, amax_all, STREAM);
}
int mlr_cpcp_lmo(void* plan, const double* red, const double* amax_all, double* dots, void* stream) {
  return cpcp_lmo(PLAN, red, amax_all, dots, STREAM);
}
int mlr_cpcp_update(void* plan, const void* D, int64_t ldd, const uint32_t* mask, int64_t ldm, void* S, int64_t lds,
                    const double* dots, void* stream) {
  return cpcp_update(PLAN, D, ldd, mask, ldm, S, lds, dots, STREAM);
}
int mlr_cpcp_finalize(void* plan, const double* red, void* stream) { return cpcp_finalize(PLAN, red, STREAM); }
int mlr_cpcp_outputs(void* plan, void* L, int64_t ldl, void* stream) { return cpcp_outputs(PLAN, L, ldl, STREAM); }
static void cpcp_state_values(const CpcpDev& h, double* out32) {
  double v[32] = {(double)h.k, (double)h.done, (double)h.status, h.t_l, h.t_s, h.u_l, h.u_s, h.sigma,
                  (double)h.passes, h.ga, h.gb, (double)h.corner_l, (double)h.corner_s, (double)h.i_s,
                  (double)h.j_s, h.s2, h.pd_norm, h.sq, h.l1, h.nnz, h.ss, h.sr, h.r_is, h.s_is, h.spike,
                  (double)h.none, h.coef, 0, 0, 0, 0, 0};
  std::memcpy(out32, v, sizeof(v));
}
int mlr_cpcp_state(void* plan, double* out32, void* stream) {
  CpcpDev h;
  MLR_CUDA(cudaMemcpyAsync(&h, PLAN->dev, sizeof(CpcpDev), cudaMemcpyDeviceToHost, STREAM));
  MLR_CUDA(cudaStreamSynchronize(STREAM));
  cpcp_state_values(h, out32);
  return kOk;
}
int64_t mlr_cpcp_snapshot_bytes(void) { return (int64_t)sizeof(CpcpDev); }
int mlr_cpcp_snapshot(void* plan, void* host, void* stream) {
  if (!host) {
    set_error("mlr_cpcp_snapshot: null buffer");
    return kErrArg;
  }
  MLR_CUDA(cudaMemcpyAsync(host, PLAN->dev, sizeof(CpcpDev), cudaMemcpyDeviceToHost, STREAM));
  return kOk;
}
int mlr_cpcp_snapshot_read(const void* host, double* out32) {
  CpcpDev h;
  std::memcpy(&h, host, sizeof(CpcpDev));
  cpcp_state_values(h, out32);
  return kOk;
}
int mlr_cpcp_set_timing(void* plan, int enable) {
  PLAN->timer.on = enable != 0;
  return kOk;
}
int mlr_cpcp_timing(void* plan, double* ms, int* counts) {
  PLAN->timer.collect(ms, counts);
  return kOk;
}
int mlr_cpcp_history(void* plan, int count, double* out, double* objectives, void* stream) {
  if (count < 0 || count > PLAN->max_iters) { set_error("mlr_cpcp_history: bad count"); return kErrArg; }
  MLR_CUDA(cudaMemcpyAsync(out, PLAN->hist, sizeof(double) * kCpHistCols * count, cudaMemcpyDeviceToHost, STREAM));
  if (objectives)
    MLR_CUDA(cudaMemcpyAsync(objectives, PLAN->obj, sizeof(double) * count, cudaMemcpyDeviceToHost, STREAM));
  MLR_CUDA(cudaStreamSynchronize(STREAM));
  return kOk;
}

// ------------------------------------------------------------ spectrum / telemetry
int64_t mlr_spec_workspace_bytes(int64_t m_local, int n) {
  if (m_local < 0 || n < 1) return -1;
  return spec_workspace_bytes(m_local, n, spec_splits(m_local, n));
}
int mlr_spec_create(int64_t m_local, int n, int f32, const double* C, int64_t ldc, const int* skip, void* workspace,
                    void** plan_out, void* stream) {
  if (m_local < 0 || n < 1 || !workspace || !plan_out || (C && ldc < n)) {
    set_error("mlr_spec_create: invalid arguments");
    return kErrArg;
  }
  SpecPlan* p = new SpecPlan();
  p->m_local = m_local;
  p->n = n;
  p->np = (int)round_up(n, 64);
  p->splits = spec_splits(m_local, n);
  p->f32 = f32 != 0;
  p->skip = skip;
  spec_carve(*p, workspace);
  int rc = spec_init(p, C, ldc, (cudaStream_t)stream);
  if (rc) {
    delete p;
    return rc;
  }
  *plan_out = p;
  return kOk;
}
int mlr_spec_destroy(void* plan) {
  delete (SpecPlan*)plan;
  return kOk;
}
int64_t mlr_spec_red_doubles(void* plan) { return (int64_t)((SpecPlan*)plan)->np * ((SpecPlan*)plan)->np; }
int mlr_spec_gram(void* plan, const void* X, int64_t ldx, double* red, void* stream) {
  return spec_gram((SpecPlan*)plan, X, ldx, red, (cudaStream_t)stream);
}
int mlr_spec_rotate(void* plan, const void* X, int64_t ldx, const double* red, double* red2, void* stream) {
  return spec_rotate((SpecPlan*)plan, X, ldx, red, red2, (cudaStream_t)stream);
}
int mlr_spec_finish(void* plan, const double* red2, double rel, double* sig_out, double* rank_out,
                    const double* pair_w, double* wsum_out, void* stream) {
  return spec_finish((SpecPlan*)plan, red2, rel, sig_out, rank_out, pair_w, wsum_out, (cudaStream_t)stream);
}
int mlr_frames_to_matrix(const uint8_t* frames, int count, int height, int width, int f32, void* x, int64_t ldx,
                         void* stream) {
  if (!frames || !x || count < 1 || height < 1 || width < 1 || ldx < count || height > 65535 || count > 65535 * 32) {
    set_error("mlr_frames_to_matrix: invalid arguments");
    return kErrArg;
  }
  return frames_to_matrix(frames, count, height, width, f32 != 0, x, ldx, (cudaStream_t)stream);
}
int mlr_matrix_to_frames(const void* x, int64_t ldx, int f32, int count, int height, int width, uint8_t* frames,
                         void* stream) {
  if (!frames || !x || count < 1 || height < 1 || width < 1 || ldx < count || height > 65535 || count > 65535 * 32) {
    set_error("mlr_matrix_to_frames: invalid arguments");
    return kErrArg;
  }
  return matrix_to_frames(x, ldx, f32 != 0, count, height, width, frames, (cudaStream_t)stream);
}
int mlr_mask_pack(const uint8_t* observed, int64_t ld_observed, int64_t m, int64_t n, uint32_t* bits, int64_t ldm,
                  void* stream) {
  if (!observed || !bits || m < 0 || n < 1 || n > INT_MAX - 32 || ld_observed < n || ldm < (n + 31) / 32) {
    set_error("mlr_mask_pack: invalid arguments");
    return kErrArg;
  }
  return mask_pack(observed, ld_observed, m, (int)n, bits, ldm, (cudaStream_t)stream);
}
int mlr_chain_cholesky(void* chain, double* C, int64_t ldc, void* stream) {
  if (!chain || !C || ldc < ((Chain*)chain)->d.nh) {
    set_error("mlr_chain_cholesky: invalid arguments");
    return kErrArg;
  }
  return chain_cholesky(((Chain*)chain)->d, C, ldc, (cudaStream_t)stream);
}
int mlr_pcp_coarse_copy(void* plan, void* out, int64_t ldo, void* stream) {
  PcpPlan* p = (PcpPlan*)plan;
  if (!out || ldo < p->ch.nh) {
    set_error("mlr_pcp_coarse_copy: invalid arguments");
    return kErrArg;
  }
  if (p->m_local == 0) return kOk;
  const size_t tb = p->f32 ? 4 : 8;
  MLR_CUDA(cudaMemcpy2DAsync(out, tb * ldo, p->Z, tb * p->ch.np, tb * p->ch.nh, p->m_local, cudaMemcpyDeviceToDevice,
                             (cudaStream_t)stream));
  return kOk;
}
int64_t mlr_pcp_delta_work_doubles(void) { return 148 * 8 + 8; }
int mlr_pcp_delta(void* plan, const void* Zk, const void* Zf, int64_t ldz, double* out, double* work, void* stream) {
  PcpPlan* p = (PcpPlan*)plan;
  if (!Zk || !Zf || !out || !work || ldz < p->ch.nh) {
    set_error("mlr_pcp_delta: invalid arguments");
    return kErrArg;
  }
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(p->m_local, 8), 148 * 8));
  return pcp_delta(p->ch, p->f32, p->m_local, Zk, Zf, ldz, out, work, blocks, (cudaStream_t)stream);
}
int mlr_cpcp_rank_shadow(void* plan, double* L64, int64_t ld, void* stream) {
  CpcpPlan* p = (CpcpPlan*)plan;
  if (!L64 || ld < p->ch.nh) {
    set_error("mlr_cpcp_rank_shadow: invalid arguments");
    return kErrArg;
  }
  return cpcp_rank_shadow(p, L64, ld, (cudaStream_t)stream);
}
int mlr_cpcp_atom_copy(void* plan, double* u_out, double* v_out, void* stream) {
  if (!u_out || !v_out) {
    set_error("mlr_cpcp_atom_copy: invalid arguments");
    return kErrArg;
  }
  return cpcp_atom_copy((CpcpPlan*)plan, u_out, v_out, (cudaStream_t)stream);
}
int mlr_cpcp_atom_dense(void* plan, const double* u, const double* v, double* out, int64_t ldo, void* stream) {
  CpcpPlan* p = (CpcpPlan*)plan;
  if (!u || !v || !out || ldo < p->ch.n) {
    set_error("mlr_cpcp_atom_dense: invalid arguments");
    return kErrArg;
  }
  return cpcp_atom_dense(p, u, v, out, ldo, (cudaStream_t)stream);
}
int mlr_cpcp_rank_binding(void* plan, const void** lh, int64_t* ld, const int** done, double** rank_slot) {
  CpcpPlan* p = (CpcpPlan*)plan;
  if (!lh || !ld || !done || !rank_slot) {
    set_error("mlr_cpcp_rank_binding: invalid arguments");
    return kErrArg;
  }
  *lh = p->LH;
  *ld = p->ch.np;
  *done = &p->dev->done;
  *rank_slot = &p->dev->rank_l;
  return kOk;
}

}  // extern "C"
