// Auxiliary GEMV kernels: explicit-LUT TL1/TL2 path and the unpacked references
// (pkg/src/ternpack/kernels.py:59-72, 109-157).
#include "common.cuh"

namespace tb {

// --------------------------------------------------------------------------
// LUT-driven GEMV for a caller-supplied TL1/TL2 LUT (kernels.py:109-157).
// lane = row; each warp walks a slice of one row tile's chunks.
// --------------------------------------------------------------------------
template <int FMT>
__global__ void gemv_lut_kernel(const uint8_t *__restrict__ tiled,
                                const uint8_t *__restrict__ tiled_sign, int N, int C,
                                const int16_t *__restrict__ lut, int64_t groups,
                                int chunks_per_warp, int32_t *__restrict__ acc_out) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int splits = (C + chunks_per_warp - 1) / chunks_per_warp;
  const int64_t t = wid / splits;
  const int cb = (int)(wid % splits) * chunks_per_warp;
  const int64_t T = (N + kRowTile - 1) / kRowTile;
  if (t >= T) return;
  const int row = (int)(t * kRowTile + lane);
  int32_t acc = 0;
  const int ce = min(C, cb + chunks_per_warp);
  for (int c = cb; c < ce; ++c) {
    const uint8_t *src = tiled + ((t * C + c) * kRowTile + lane) * 16;
    uint32_t X[5] = {0, 0, 0, 0, 0};
    if (FMT == TB_TL2) {  // the row's five tile words (common.cuh tl2_bit)
      const uint4 m = *reinterpret_cast<const uint4 *>(src);
      X[0] = m.x, X[1] = m.y, X[2] = m.z, X[3] = m.w;
      X[4] = *reinterpret_cast<const uint32_t *>(tiled_sign + ((t * C + c) * kRowTile + lane) * 4);
    }
    for (int b = 0; b < 16; ++b) {
      const uint32_t byte = src[b];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t g = (int64_t)c * 32 + 2 * b + h;  // pair / triple index
        // TL1 tiles hold 2-bit codes (pack.cu repack): pair h = codes 2h, 2h+1
        const uint32_t idx = FMT == TB_TL1 ? 3u * ((byte >> (4 * h)) & 3u) + ((byte >> (4 * h + 2)) & 3u)
                                           : (h ? (byte >> 4) : (byte & 15));
        if (g >= groups) continue;
        if (FMT == TB_TL1) {
          if (idx <= 8) acc += lut[g * 9 + idx];
        } else {
          // tiled TL2 holds v = 13 + signed index (pack.cu)
          const int v = (int)tl2_tile_value(X, 2 * b + h);
          const int d = v - 13;
          const int32_t e = lut[g * 14 + (d < 0 ? -d : d)];
          acc += d < 0 ? -e : e;
        }
      }
    }
  }
  if (row < N && acc != 0) atomicAdd(acc_out + row, acc);
}

__global__ void gemv_ref_int32_kernel(const int8_t *__restrict__ v, int64_t rows, int64_t cols,
                                      const int8_t *__restrict__ a, int32_t *__restrict__ out) {
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  int32_t s = 0;
  for (int64_t k = lane; k < cols; k += 32) s += (int32_t)v[r * cols + k] * (int32_t)a[k];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[r] = s;
}

__global__ void gemv_f32_ref_kernel(const int8_t *__restrict__ v, int64_t rows, int64_t cols,
                                    float ws, const float *__restrict__ x,
                                    float *__restrict__ out) {
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  float s = 0.f;
  for (int64_t k = lane; k < cols; k += 32) s += (static_cast<float>(v[r * cols + k]) * ws) * x[k];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[r] = s;
}

}  // namespace tb

using namespace tb;

extern "C" int tb_gemv_lut(int fmt, const uint8_t *tiled, const uint8_t *tiled_sign,
                           int64_t rows, int64_t cols, const int16_t *lut, int64_t groups,
                           int32_t *acc_out, void *stream) {
  if (!tiled || !lut || !acc_out || rows < 1 || cols < 1 || groups < 1 ||
      (fmt != TB_TL1 && fmt != TB_TL2) || (fmt == TB_TL2 && !tiled_sign))
    return TB_ERR_ARGUMENT;
  const int64_t C = ceil_div(ref_row_bytes(fmt, cols), kChunkBytes);
  const int64_t T = ceil_div(rows, kRowTile);
  const int cpw = 8;
  const int64_t warps = T * ceil_div(C, cpw);
  const int64_t blocks = ceil_div(warps * 32, 256);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (fmt == TB_TL1)
    gemv_lut_kernel<TB_TL1><<<(unsigned)blocks, 256, 0, s>>>(tiled, tiled_sign, (int)rows, (int)C,
                                                             lut, groups, cpw, acc_out);
  else
    gemv_lut_kernel<TB_TL2><<<(unsigned)blocks, 256, 0, s>>>(tiled, tiled_sign, (int)rows, (int)C,
                                                             lut, groups, cpw, acc_out);
  TB_CHECK_LAUNCH();
  return TB_OK;
}

extern "C" int tb_gemv_ref_int32(const int8_t *values, int64_t rows, int64_t cols,
                                 const int8_t *act, int32_t *acc_out, void *stream) {
  if (!values || !act || !acc_out || rows < 1 || cols < 1) return TB_ERR_ARGUMENT;
  gemv_ref_int32_kernel<<<(unsigned)ceil_div(rows * 32, 256), 256, 0,
                          static_cast<cudaStream_t>(stream)>>>(values, rows, cols, act, acc_out);
  TB_CHECK_LAUNCH();
  return TB_OK;
}

extern "C" int tb_gemv_f32_ref(const int8_t *values, int64_t rows, int64_t cols, float w_scale,
                               const float *x, float *out, void *stream) {
  if (!values || !x || !out || rows < 1 || cols < 1) return TB_ERR_ARGUMENT;
  gemv_f32_ref_kernel<<<(unsigned)ceil_div(rows * 32, 256), 256, 0,
                        static_cast<cudaStream_t>(stream)>>>(values, rows, cols, w_scale, x, out);
  TB_CHECK_LAUNCH();
  return TB_OK;
}
