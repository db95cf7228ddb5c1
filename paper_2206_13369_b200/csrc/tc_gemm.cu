// Reconstruction Z = A W~ of the FP32 ML-PCP plans on the 5th-generation
// tensor cores (replaces the FP64-DMMA gemm_f64 call for Z; reference
// pcp.py:258-266: L_H = U_r diag(sigma_r - tau) V_r^T, which the GPU
// formulation writes as L_H = A W~).
//
// 3xTF32: Z = A_hi W_hi + A_hi W_lo + A_lo W_hi with every operand an exact
// TF32 value (hi = low 13 mantissa bits cleared, lo = x - hi, exact in FP32),
// accumulated in FP32 in TMEM.  The dropped A_lo W_lo term and the TF32
// rounding of the lo parts are ~2^-21 relative per product, the FP32
// accumulation over K = n_p terms ~sqrt(K) 2^-24: FP32-class accuracy, which
// is all Z (stored as FP32) carries anyway.  The Gram K = A^T A stays FP64
// DMMA: its eigenvalues are needed down to tau^2 ~ 3e-8 lambda_max (C5),
// below what FP32 accumulation resolves.
//
// Per CTA: one 128 x BN tile of Z (BN = 256 when n_p % 256 == 0).  Warp
// roles (256 threads):
//   warp 0 lane 0   TMA producer: A (128 x 32 FP32, 128B-swizzled K-major)
//                   and the W~^T hi / lo tiles (BN x 32) per K block, one
//                   mbarrier per stage with the transaction byte count;
//   warp 1 lane 0   MMA issuer: 3 x (32 / 8) tcgen05.mma.kind::tf32 per K
//                   block into a 128 x BN FP32 accumulator in TMEM;
//                   tcgen05.commit releases the stage;
//   warp 2          TMEM allocator (BN columns);
//   warps 4-7       splitters: A -> (A_hi in place, A_lo) in shared memory
//                   (elementwise, so the swizzled layout is preserved), then
//                   the epilogue: tcgen05.ld 32 lanes x 32 columns per warp
//                   -> float4 stores of Z.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace mlr {

constexpr int TC_BM = 128, TC_BK = 32, TC_STAGES = 2, TC_THREADS = 256;

__device__ __forceinline__ uint32_t tc_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tc_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc_smem(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void tc_mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc_smem(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tc_mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc_smem(bar)) : "memory");
}
__device__ __forceinline__ void tc_mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "TC_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra TC_WAIT_%=;\n"
      "}\n" ::"r"(tc_smem(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tc_tma_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          tc_smem(dst)),
      "l"(map), "r"(x), "r"(y), "r"(tc_smem(bar))
      : "memory");
}

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row core
// groups 1024 bytes apart (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t tc_desc(const void* p) {
  const uint64_t a = tc_smem(p);
  return ((a & 0x3FFFF) >> 4) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

__device__ __forceinline__ void tc_mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(tc_smem(bar))
               : "memory");
}

template <int BN>
struct TcSmem {
  float a[TC_STAGES][TC_BM * TC_BK];    // TMA target, then A_hi in place
  float alo[TC_STAGES][TC_BM * TC_BK];  // A_lo (same swizzled layout)
  float bhi[TC_STAGES][BN * TC_BK];
  float blo[TC_STAGES][BN * TC_BK];
  uint64_t full[TC_STAGES], split[TC_STAGES], empty[TC_STAGES], tfull;
  uint32_t tmem_base;
};

template <int BN>
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_recon_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBhi,
                    const __grid_constant__ CUtensorMap tmBlo, int64_t M, int K, float* __restrict__ Z,
                    int64_t ldz, const int* __restrict__ skip) {
  if (skip && *skip) return;
  extern __shared__ __align__(1024) unsigned char tc_raw[];
  TcSmem<BN>& S = *reinterpret_cast<TcSmem<BN>*>((reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN;
  const int64_t m0 = (int64_t)blockIdx.y * TC_BM;
  const int KB = K / TC_BK;
  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_STAGES; ++s) {
      tc_mbar_init(&S.full[s], 1);
      tc_mbar_init(&S.split[s], 4);
      tc_mbar_init(&S.empty[s], 1);
    }
    tc_mbar_init(&S.tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem(&S.tmem_base)),
                 "r"((uint32_t)BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = S.tmem_base;

  if (warp == 0) {
    if (lane == 0) {  // ---------------------------------------------- TMA producer
      const uint32_t bytes = (uint32_t)(TC_BM + 2 * BN) * TC_BK * 4;
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % TC_STAGES;
        if (kb >= TC_STAGES) tc_mbar_wait(&S.empty[s], ((kb / TC_STAGES) - 1) & 1);
        tc_mbar_expect_tx(&S.full[s], bytes);
        tc_tma_2d(S.a[s], &tmA, kb * TC_BK, (int)m0, &S.full[s]);
        tc_tma_2d(S.bhi[s], &tmBhi, kb * TC_BK, n0, &S.full[s]);
        tc_tma_2d(S.blo[s], &tmBlo, kb * TC_BK, n0, &S.full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------------------------------------- MMA issuer
      // kind::tf32, D F32, A/B TF32 K-major, N = BN, M = 128
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(TC_BM >> 4) << 24);
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % TC_STAGES;
        tc_mbar_wait(&S.split[s], (kb / TC_STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t dah = tc_desc(S.a[s]), dal = tc_desc(S.alo[s]);
        const uint64_t dbh = tc_desc(S.bhi[s]), dbl = tc_desc(S.blo[s]);
#pragma unroll
        for (int k = 0; k < TC_BK / 8; ++k) {  // 8 TF32 = 32 bytes per MMA: +2 in the (addr >> 4) field
          const uint64_t o = 2ull * k;
          tc_mma_tf32(tmem, dah + o, dbh + o, idesc, (kb | k) ? 1u : 0u);
          tc_mma_tf32(tmem, dah + o, dbl + o, idesc, 1u);
          tc_mma_tf32(tmem, dal + o, dbh + o, idesc, 1u);
        }
        tc_commit(&S.empty[s]);  // stage free once these MMAs have read it
      }
      tc_commit(&S.tfull);
    }
  } else if (warp >= 4) {
    const int q = warp - 4;  // TMEM lanes 32 q .. 32 q + 31
    const int t = threadIdx.x - 128;
    // ---------------------------------------------------------------- splitters
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % TC_STAGES;
      tc_mbar_wait(&S.full[s], (kb / TC_STAGES) & 1);
      float4* a4 = reinterpret_cast<float4*>(S.a[s]);
      float4* l4 = reinterpret_cast<float4*>(S.alo[s]);
#pragma unroll
      for (int j = 0; j < TC_BM * TC_BK / 4 / 128; ++j) {
        const int i = t + 128 * j;
        float4 v = a4[i], lo;
        float4 hi;
        hi.x = __uint_as_float(__float_as_uint(v.x) & 0xffffe000u);
        hi.y = __uint_as_float(__float_as_uint(v.y) & 0xffffe000u);
        hi.z = __uint_as_float(__float_as_uint(v.z) & 0xffffe000u);
        hi.w = __uint_as_float(__float_as_uint(v.w) & 0xffffe000u);
        lo.x = v.x - hi.x;
        lo.y = v.y - hi.y;
        lo.z = v.z - hi.z;
        lo.w = v.w - hi.w;
        a4[i] = hi;
        l4[i] = lo;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) tc_mbar_arrive(&S.split[s]);
    }
    // ---------------------------------------------------------------- epilogue
    tc_mbar_wait(&S.tfull, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int64_t row = m0 + 32 * q + lane;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t r[32];
      const uint32_t addr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(32 * c);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
            "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
            "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(addr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (row < M) {
        float4* out = reinterpret_cast<float4*>(Z + row * ldz + n0 + 32 * c);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          out[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                               __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)BN));
  }
}

// W~^T (FP64, n_p x n_p, row-major) -> exact TF32 hi / lo parts in FP32
// (hi = W rounded to TF32 by truncation of the FP32 value, lo = TF32 of the
// FP64 remainder).
__global__ void tc_split_w_kernel(const double* __restrict__ Wt, float* __restrict__ hi, float* __restrict__ lo,
                                  int64_t count, const int* __restrict__ skip) {
  if (skip && *skip) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const double w = Wt[i];
    const float h = __uint_as_float(__float_as_uint((float)w) & 0xffffe000u);
    const float l = __uint_as_float(__float_as_uint((float)(w - (double)h)) & 0xffffe000u);
    hi[i] = h;
    lo[i] = l;
  }
}

static PFN_cuTensorMapEncodeTiled encode_fn() {
  static PFN_cuTensorMapEncodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled)p;
  }
  return fn;
}

static int make_map(CUtensorMap* map, const float* base, int64_t rows, int cols, int box_rows) {
  PFN_cuTensorMapEncodeTiled enc = encode_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return kErrCuda;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed");
    return kErrCuda;
  }
  return kOk;
}

int tc_recon_bn(int np) { return np % 256 == 0 ? 256 : (np % 128 == 0 ? 128 : (np % 64 == 0 ? 64 : 0)); }

template <int BN>
static int tc_launch(const CUtensorMap& a, const CUtensorMap& bh, const CUtensorMap& bl, int64_t M, int np, float* Z,
                     int64_t ldz, const int* skip, cudaStream_t st) {
  const size_t smem = sizeof(TcSmem<BN>) + 1024;
  MLR_CUDA(cudaFuncSetAttribute(tc_recon_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid(np / BN, (unsigned)ceil_div(M, (int64_t)TC_BM));
  tc_recon_kernel<BN><<<grid, TC_THREADS, smem, st>>>(a, bh, bl, M, np, Z, ldz, skip);
  MLR_LAUNCH_CHECK("tc_recon_kernel");
  return kOk;
}

int tc_recon_setup(TcRecon* r, const float* A, int64_t M, int np, const float* Whi, const float* Wlo) {
  r->bn = tc_recon_bn(np);
  r->M = M;
  r->np = np;
  if (!r->bn || np % TC_BK) {
    set_error("tc_recon_setup: n_p must be a multiple of 64");
    return kErrArg;
  }
  int rc;
  if ((rc = make_map(&r->mapA, A, M, np, TC_BM))) return rc;
  if ((rc = make_map(&r->mapBhi, Whi, np, np, r->bn))) return rc;
  if ((rc = make_map(&r->mapBlo, Wlo, np, np, r->bn))) return rc;
  r->ready = true;
  return kOk;
}

int tc_recon_run(const TcRecon* r, float* Z, int64_t ldz, const int* skip, cudaStream_t st) {
  if (r->M == 0) return kOk;
  switch (r->bn) {
    case 256: return tc_launch<256>(r->mapA, r->mapBhi, r->mapBlo, r->M, r->np, Z, ldz, skip, st);
    case 128: return tc_launch<128>(r->mapA, r->mapBhi, r->mapBlo, r->M, r->np, Z, ldz, skip, st);
    default: return tc_launch<64>(r->mapA, r->mapBhi, r->mapBlo, r->M, r->np, Z, ldz, skip, st);
  }
}

int tc_split_w(const double* Wt, float* hi, float* lo, int np, const int* skip, cudaStream_t st) {
  const int64_t count = (int64_t)np * np;
  tc_split_w_kernel<<<(int)std::min<int64_t>(ceil_div(count, 256), 1184), 256, 0, st>>>(Wt, hi, lo, count, skip);
  MLR_LAUNCH_CHECK("tc_split_w_kernel");
  return kOk;
}

}  // namespace mlr

using namespace mlr;

extern "C" {

/* Test entry: Z (m x np FP32, ld np) = A (m x np FP32) W (np x np FP64,
 * row-major) by the 3xTF32 tcgen05 kernel.  work: 2 np^2 floats + np^2
 * doubles.  Synchronous. */
int mlr_tc_gemm_tf32x3(int64_t m, int np, const float* A, const double* W, float* Z, void* work, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  double* Wt = reinterpret_cast<double*>(work);
  float* hi = reinterpret_cast<float*>(Wt + (int64_t)np * np);
  float* lo = hi + (int64_t)np * np;
  // W^T (B operand K-major: row n holds W[:, n])
  std::vector<double> h((size_t)np * np), t((size_t)np * np);
  MLR_CUDA(cudaMemcpyAsync(h.data(), W, sizeof(double) * np * np, cudaMemcpyDeviceToHost, st));
  MLR_CUDA(cudaStreamSynchronize(st));
  for (int i = 0; i < np; ++i)
    for (int j = 0; j < np; ++j) t[(size_t)j * np + i] = h[(size_t)i * np + j];
  MLR_CUDA(cudaMemcpyAsync(Wt, t.data(), sizeof(double) * np * np, cudaMemcpyHostToDevice, st));
  int rc = tc_split_w(Wt, hi, lo, np, nullptr, st);
  if (rc) return rc;
  TcRecon r{};
  if ((rc = tc_recon_setup(&r, A, m, np, hi, lo))) return rc;
  if ((rc = tc_recon_run(&r, Z, np, nullptr, st))) return rc;
  MLR_CUDA(cudaStreamSynchronize(st));
  return kOk;
}

}  // extern "C"
