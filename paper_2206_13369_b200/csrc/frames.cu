// Frame-stack layout kernels for the video pipeline (reference io.py:131-182).
//
// A stack of `count` 8-bit frames (height x width, row-major raster, frame j
// at frames + j*H*W) maps to the m x count solver matrix (m = H*W, row-major
// with leading dimension ldx): pixel (row, col) of frame j is matrix entry
// (row + col*H, j) (io.py:33-36, column-major within the frame).  In index
// terms this is the axis reversal (j, row, col) -> (col, row, j): for each
// row a 2-D transpose between frames and columns, done in 32 x 32 tiles
// through shared memory so both sides are coalesced.  Pure byte/streaming
// work (HBM-bound): 1 byte read + sizeof(T) written per pixel on ingest.
#include <algorithm>

#include "common.cuh"

namespace mlr {

constexpr int FT = 32, FR = 8;  // tile edge, thread rows

// ingest_frames (io.py:131-150): x = u8 / 255.0 in float64 (then rounded to T)
template <typename T>
__global__ void __launch_bounds__(FT * FR) frames_to_matrix_kernel(const uint8_t* __restrict__ frames, int count,
                                                                  int H, int W, T* __restrict__ x, int64_t ldx) {
  __shared__ uint8_t tile[FT][FT + 4];
  const int row = blockIdx.y, col0 = blockIdx.x * FT, j0 = blockIdx.z * FT;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t plane = (int64_t)H * W;
  for (int jj = ty; jj < FT; jj += FR) {
    const int j = j0 + jj, col = col0 + tx;
    tile[jj][tx] = (j < count && col < W) ? frames[j * plane + (int64_t)row * W + col] : 0;
  }
  __syncthreads();
  for (int cc = ty; cc < FT; cc += FR) {
    const int col = col0 + cc, j = j0 + tx;
    if (col < W && j < count) x[((int64_t)row + (int64_t)col * H) * ldx + j] = (T)((double)tile[tx][cc] / 255.0);
  }
}

// emit_frames' _quantize (io.py:153-158): clamp to [0, 1], floor(v*255 + 0.5)
template <typename T>
__global__ void __launch_bounds__(FT * FR) matrix_to_frames_kernel(const T* __restrict__ x, int64_t ldx, int count,
                                                                  int H, int W, uint8_t* __restrict__ frames) {
  __shared__ uint8_t tile[FT][FT + 4];
  const int row = blockIdx.y, col0 = blockIdx.x * FT, j0 = blockIdx.z * FT;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t plane = (int64_t)H * W;
  for (int cc = ty; cc < FT; cc += FR) {
    const int col = col0 + cc, j = j0 + tx;
    uint8_t q = 0;
    if (col < W && j < count) {
      double v = (double)x[((int64_t)row + (int64_t)col * H) * ldx + j];
      v = fmin(fmax(v, 0.0), 1.0);
      q = (uint8_t)floor(v * 255.0 + 0.5);
    }
    tile[cc][tx] = q;
  }
  __syncthreads();
  for (int jj = ty; jj < FT; jj += FR) {
    const int j = j0 + jj, col = col0 + tx;
    if (j < count && col < W) frames[j * plane + (int64_t)row * W + col] = tile[tx][jj];
  }
}

int frames_to_matrix(const uint8_t* frames, int count, int H, int W, bool f32, void* x, int64_t ldx,
                     cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(W, FT), (unsigned)H, (unsigned)ceil_div(count, FT)), block(FT, FR);
  if (f32)
    frames_to_matrix_kernel<float><<<grid, block, 0, st>>>(frames, count, H, W, (float*)x, ldx);
  else
    frames_to_matrix_kernel<double><<<grid, block, 0, st>>>(frames, count, H, W, (double*)x, ldx);
  MLR_LAUNCH_CHECK("frames_to_matrix_kernel");
  return kOk;
}

int matrix_to_frames(const void* x, int64_t ldx, bool f32, int count, int H, int W, uint8_t* frames,
                     cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(W, FT), (unsigned)H, (unsigned)ceil_div(count, FT)), block(FT, FR);
  if (f32)
    matrix_to_frames_kernel<float><<<grid, block, 0, st>>>((const float*)x, ldx, count, H, W, frames);
  else
    matrix_to_frames_kernel<double><<<grid, block, 0, st>>>((const double*)x, ldx, count, H, W, frames);
  MLR_LAUNCH_CHECK("matrix_to_frames_kernel");
  return kOk;
}

// Observation mask (reference cpcp.py:23-53: a boolean m x n array) -> the
// bit-packed rows the ML-CPCP passes read: uint32 words, bit j & 31 of word
// j >> 5, ldm words per row.  One warp per word: 32 coalesced byte loads, one
// ballot, one store.  The host path it replaces (numpy packbits of the whole
// mask on every solve) cost 31 ms of a 154 ms C4 solve.
__global__ void __launch_bounds__(256) mask_pack_kernel(const uint8_t* __restrict__ obs, int64_t ldo, int64_t m,
                                                        int n, uint32_t* __restrict__ bits, int64_t ldm) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int words = (n + 31) >> 5;
  const int64_t items = m * (int64_t)ldm;
  for (int64_t it = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); it < items; it += warps) {
    const int64_t row = it / ldm;
    const int w = (int)(it - row * ldm);
    const int j = w * 32 + lane;
    const bool on = w < words && j < n && obs[row * ldo + j] != 0;
    const uint32_t word = __ballot_sync(0xffffffffu, on);
    if (lane == 0) bits[it] = word;
  }
}

int mask_pack(const uint8_t* obs, int64_t ldo, int64_t m, int n, uint32_t* bits, int64_t ldm, cudaStream_t st) {
  const int64_t items = m * ldm;
  const int grid = (int)std::min<int64_t>((items + 7) / 8, 148 * 16);
  if (grid > 0) mask_pack_kernel<<<grid, 256, 0, st>>>(obs, ldo, m, n, bits, ldm);
  MLR_LAUNCH_CHECK("mask_pack_kernel");
  return kOk;
}

}  // namespace mlr
