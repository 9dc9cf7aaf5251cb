// Decode GEMV (M <= 16) on the tiled I2_S / TL1 / TL2 layouts.
//
// Replaces kernels.gemv_i2s / gemv_tl1 / gemv_tl2 / gemv_parallel
// (pkg/src/ternpack/kernels.py:86-157, 189-268) and the numba byte-table
// gathers (_fast.py:25-95).  The reference gathers one int32 table entry per
// packed byte; here the packed bytes are decoded in registers to 2-bit codes
// c = w + 1 in {0,1,2} (four per 32-bit word, one per byte lane) and
// contracted with dp4a against a byte-transposed copy of the int8 activations
// held in shared memory.  sum_k w_k a_k = sum_k c_k a_k - sum_k a_k, so the
// per-chunk activation sums are subtracted once per chunk.  Integer results
// are exact, hence bit-identical to the reference's LUT/byte-table kernels.
//
// Data movement: a persistent grid (one CTA per SM); each CTA owns a
// contiguous range of (row tile, chunk) units -- a contiguous byte range of
// the tiled layout -- and one producer thread streams it HBM -> SMEM with
// cp.async.bulk into a 6-stage mbarrier ring.  Eight consumer warps decode:
// lane = row of the 32-row tile, so activation reads are warp broadcasts and
// weight reads are conflict-free 16-byte LDS.  Partial sums of a row tile are
// combined with red.global.add in a self-cleaning int32 workspace; the warp
// that retires the tile's last chunk applies the scales (core.py:99-101).
#include <algorithm>

#include "common.cuh"

namespace tb {

constexpr int kConsumerWarps = 8;
constexpr int kThreads = 32 * (1 + kConsumerWarps);
constexpr int kStageChunks = 16;
constexpr int kStages = 6;
constexpr int64_t kActSmemBudget = 120 * 1024;

struct GemvParams {
  const uint8_t *wmain;
  const uint8_t *wsign;
  const int8_t *act;
  int64_t ld_act;
  int64_t act_len;
  const double *a_scale;
  double w_scale;
  int32_t *ws_acc;  // [16][Npad]
  int32_t *ws_cnt;  // [T]
  int32_t *acc_out;
  double *out64;
  float *out32;
  int64_t total;  // T * Cs units in this pass
  int N, Npad, T, C, c0, Cs, M;
};

template <int FMT>
struct Fmt {
  static constexpr int kActWords = FMT == TB_TL2 ? 24 : 16;  // permuted act words / chunk
  static constexpr int kSignBytes = FMT == TB_TL2 ? kTileSignBytes : 0;
  static constexpr int kStageBytes = kStageChunks * (kTileChunkBytes + kSignBytes);
};

template <int FMT>
static size_t gemv_smem_bytes(int M, int Cs) {
  size_t stages = (size_t)kStages * Fmt<FMT>::kStageBytes;
  size_t bars = 2 * kStages * sizeof(uint64_t);
  size_t acts = (size_t)M * Cs * (Fmt<FMT>::kActWords * 4 + 4);
  return stages + bars + acts;
}

__device__ __forceinline__ uint32_t byte_of(const uint8_t *buf, int i) { return buf[i]; }

// Build the byte-transposed activation words of one chunk.
//   I2_S / TL1 (64 acts): word 4i+s = (a[16i+s], a[16i+4+s], a[16i+8+s], a[16i+12+s])
//   TL2        (96 acts): word 6i+s = (a[24i+s], a[24i+6+s], a[24i+12+s], a[24i+18+s])
template <int FMT>
__device__ void stage_activation_chunk(const int8_t *arow, int64_t act_len, int64_t k0,
                                       uint32_t *dst, int32_t *sum_out) {
  constexpr int W = FMT == TB_TL2 ? 96 : 64;
  constexpr int G = FMT == TB_TL2 ? 6 : 4;  // stride between bytes of one word
  alignas(16) uint8_t buf[W];
  if (k0 + W <= act_len && (reinterpret_cast<uintptr_t>(arow + k0) & 15) == 0) {
#pragma unroll
    for (int v = 0; v < W / 16; ++v)
      reinterpret_cast<uint4 *>(buf)[v] = __ldg(reinterpret_cast<const uint4 *>(arow + k0) + v);
  } else {
    for (int b = 0; b < W; ++b) buf[b] = (k0 + b < act_len) ? (uint8_t)arow[k0 + b] : 0;
  }
  int32_t sum = 0;
#pragma unroll
  for (int b = 0; b < W; ++b) sum += (int8_t)buf[b];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int s = 0; s < G; ++s) {
      const int base = i * 4 * G + s;
      dst[i * G + s] = byte_of(buf, base) | (byte_of(buf, base + G) << 8) |
                       (byte_of(buf, base + 2 * G) << 16) | (byte_of(buf, base + 3 * G) << 24);
    }
  }
  *sum_out = sum;
}

template <int FMT, int MT>
struct Acc {
  // I2_S keeps one accumulator per 2-bit slot (scaled by 4^s, see decode);
  // TL1 / TL2 decode straight to unscaled codes.
  static constexpr int kSlots = FMT == TB_I2S ? 4 : 1;
  int32_t v[MT][kSlots];
  int32_t csum[MT];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int m = 0; m < MT; ++m) {
#pragma unroll
      for (int s = 0; s < kSlots; ++s) v[m][s] = 0;
      csum[m] = 0;
    }
  }
  __device__ __forceinline__ int32_t total(int m) const {
    if (FMT == TB_I2S)
      return v[m][0] + (v[m][1] >> 2) + (v[m][2] >> 4) + (v[m][3] >> 6) - csum[m];
    return v[m][0] - csum[m];
  }
};

// One 16-byte chunk of one row (this lane's row) against MT activation rows.
template <int FMT, int MT>
__device__ __forceinline__ void process_chunk(const uint4 w4, const uint32_t sgn,
                                              const uint32_t *__restrict__ a_chunk,
                                              int64_t act_tok_stride, int M, Acc<FMT, MT> &acc) {
  const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t W = w[i];
    if constexpr (FMT == TB_I2S) {
      // byte b of (W & (3 << 2s)) = code of weight 16i + 4b + s, times 4^s
      const uint32_t x0 = W & 0x03030303u, x1 = W & 0x0C0C0C0Cu;
      const uint32_t x2 = W & 0x30303030u, x3 = W & 0xC0C0C0C0u;
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        if (m < M) {
          const uint4 A = *reinterpret_cast<const uint4 *>(a_chunk + m * act_tok_stride + 4 * i);
          acc.v[m][0] = dp4a_us(x0, A.x, acc.v[m][0]);
          acc.v[m][1] = dp4a_us(x1, A.y, acc.v[m][1]);
          acc.v[m][2] = dp4a_us(x2, A.z, acc.v[m][2]);
          acc.v[m][3] = dp4a_us(x3, A.w, acc.v[m][3]);
        }
      }
    } else if constexpr (FMT == TB_TL1) {
      // nibble n = 3*c0 + c1 (packing.py:56-60): c0 = n/3 = (11n)>>5 for n <= 8
      const uint32_t lo = W & 0x0F0F0F0Fu, hi = (W >> 4) & 0x0F0F0F0Fu;
      const uint32_t qlo = ((lo * 11u) >> 5) & 0x03030303u, rlo = lo - 3u * qlo;
      const uint32_t qhi = ((hi * 11u) >> 5) & 0x03030303u, rhi = hi - 3u * qhi;
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        if (m < M) {
          const uint4 A = *reinterpret_cast<const uint4 *>(a_chunk + m * act_tok_stride + 4 * i);
          int32_t t = acc.v[m][0];
          t = dp4a_us(qlo, A.x, t);
          t = dp4a_us(rlo, A.y, t);
          t = dp4a_us(qhi, A.z, t);
          t = dp4a_us(rhi, A.w, t);
          acc.v[m][0] = t;
        }
      }
    } else {
      // TL2 (packing.py:63-74): d = 13 + idx (sign 0) or 13 - idx (sign 1) is
      // the base-3 number of the triple's codes (c0 c1 c2).
      const uint32_t S = (sgn >> (8 * i)) & 0xFFu;
      const uint32_t lo = W & 0x0F0F0F0Fu, hi = (W >> 4) & 0x0F0F0F0Fu;
      // byte-wide sign masks: even sign bits -> low-nibble triples, odd -> high
      const uint32_t mlo = prmt((S & 0x55u) * 0x02082080u, 0u, 0xBA98u);
      const uint32_t mhi = prmt((S & 0xAAu) * 0x01041040u, 0u, 0xBA98u);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t x = h ? hi : lo;
        const uint32_t msk = h ? mhi : mlo;
        const uint32_t d = lop3_sel(x + 0x0D0D0D0Du, 0x0D0D0D0Du - x, msk);
        const uint32_t c0 = ((d * 7u + 0x07070707u) >> 6) & 0x03030303u;  // d / 9
        const uint32_t r = d - 9u * c0;                                      // d % 9
        const uint32_t c1 = ((r * 11u) >> 5) & 0x03030303u;                  // r / 3
        const uint32_t c2 = r - 3u * c1;                                     // r % 3
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          if (m < M) {
            const uint32_t *A = a_chunk + m * act_tok_stride + 6 * i + 3 * h;
            int32_t t = acc.v[m][0];
            t = dp4a_us(c0, A[0], t);
            t = dp4a_us(c1, A[1], t);
            t = dp4a_us(c2, A[2], t);
            acc.v[m][0] = t;
          }
        }
      }
    }
  }
}

template <int FMT, int MT>
__device__ __forceinline__ void flush_tile(const GemvParams &p, int t, int nch,
                                           const Acc<FMT, MT> &acc, int lane) {
  const int row = t * kRowTile + lane;
#pragma unroll
  for (int m = 0; m < MT; ++m)
    if (m < p.M) red_add_s32(p.ws_acc + (int64_t)m * p.Npad + row, acc.total(m));
  __threadfence();
  __syncwarp();
  int last = 0;
  if (lane == 0) {
    int old = atomicAdd(p.ws_cnt + t, nch);
    last = (old + nch == p.C);
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  __threadfence();
#pragma unroll
  for (int m = 0; m < MT; ++m) {
    if (m < p.M) {
      const int32_t v = atomicExch(p.ws_acc + (int64_t)m * p.Npad + row, 0);
      if (row < p.N) {
        const int64_t o = (int64_t)m * p.N + row;
        if (p.acc_out) p.acc_out[o] = v;
        if (p.out64 || p.out32) {
          const double y = static_cast<double>(v) * p.w_scale * p.a_scale[m];
          if (p.out64) p.out64[o] = y;
          if (p.out32) p.out32[o] = static_cast<float>(y);
        }
      }
    }
  }
  if (lane == 0) p.ws_cnt[t] = 0;
}

template <int FMT, int MT>
__global__ void __launch_bounds__(kThreads, 1) tgemv_kernel(const GemvParams p) {
  using F = Fmt<FMT>;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t *st_main = smem;
  uint8_t *st_sign = smem + kStages * kStageChunks * kTileChunkBytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kStages * F::kStageBytes);
  uint64_t *empty = full + kStages;
  uint32_t *s_act = reinterpret_cast<uint32_t *>(empty + kStages);
  int32_t *s_csum = reinterpret_cast<int32_t *>(s_act + (int64_t)p.M * p.Cs * F::kActWords);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t G = gridDim.x;
  const int64_t g0 = p.total * blockIdx.x / G;
  const int64_t g1 = p.total * (blockIdx.x + 1) / G;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t g = g0; g < g1; g += kStageChunks) {
        const int n = (int)imin64(kStageChunks, g1 - g);
        mbar_wait(empty + stage, phase ^ 1);
        mbar_arrive_expect_tx(full + stage, n * (kTileChunkBytes + F::kSignBytes));
        int done = 0;
        int64_t gg = g;
        while (done < n) {
          const int64_t t = gg / p.Cs;
          const int64_t cc = gg - t * p.Cs;
          const int run = (int)imin64(n - done, p.Cs - cc);
          const int64_t src = t * p.C + p.c0 + cc;  // chunk index in the tiled layout
          bulk_g2s(st_main + (stage * kStageChunks + done) * kTileChunkBytes,
                   p.wmain + src * kTileChunkBytes, run * kTileChunkBytes, full + stage);
          if (FMT == TB_TL2)
            bulk_g2s(st_sign + (stage * kStageChunks + done) * kTileSignBytes,
                     p.wsign + src * kTileSignBytes, run * kTileSignBytes, full + stage);
          done += run;
          gg += run;
        }
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }

  // ---------------------------------------------------------------- consumers
  const int ctid = threadIdx.x - 32;
  for (int64_t it = ctid; it < (int64_t)p.M * p.Cs; it += kConsumerWarps * 32) {
    const int m = (int)(it / p.Cs), c = (int)(it % p.Cs);
    stage_activation_chunk<FMT>(p.act + m * p.ld_act, p.act_len,
                                (int64_t)(p.c0 + c) * chunk_weights(FMT),
                                s_act + it * F::kActWords, s_csum + it);
  }
  named_bar_sync(1, kConsumerWarps * 32);

  const int cw = warp - 1;
  const int64_t act_tok_stride = (int64_t)p.Cs * F::kActWords;
  Acc<FMT, MT> acc;
  acc.zero();
  int cur_t = -1, nch = 0;
  int stage = 0;
  uint32_t phase = 0;
  for (int64_t g = g0; g < g1; g += kStageChunks) {
    const int n = (int)imin64(kStageChunks, g1 - g);
    mbar_wait(full + stage, phase);
    for (int j = cw; j < n; j += kConsumerWarps) {
      const int64_t gg = g + j;
      const int t = (int)(gg / p.Cs);
      const int c = (int)(gg - (int64_t)t * p.Cs);
      if (t != cur_t) {
        if (cur_t >= 0) flush_tile<FMT, MT>(p, cur_t, nch, acc, lane);
        cur_t = t;
        nch = 0;
        acc.zero();
      }
      const int slot = stage * kStageChunks + j;
      const uint4 w4 = *reinterpret_cast<const uint4 *>(st_main + slot * kTileChunkBytes + lane * 16);
      uint32_t sg = 0;
      if (FMT == TB_TL2)
        sg = *reinterpret_cast<const uint32_t *>(st_sign + slot * kTileSignBytes + lane * 4);
      process_chunk<FMT, MT>(w4, sg, s_act + (int64_t)c * F::kActWords, act_tok_stride, p.M, acc);
#pragma unroll
      for (int m = 0; m < MT; ++m)
        if (m < p.M) acc.csum[m] += s_csum[(int64_t)m * p.Cs + c];
      ++nch;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + stage);
    if (++stage == kStages) {
      stage = 0;
      phase ^= 1;
    }
  }
  if (cur_t >= 0) flush_tile<FMT, MT>(p, cur_t, nch, acc, lane);
}

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
    uint32_t sg = 0;
    if (FMT == TB_TL2)
      sg = *reinterpret_cast<const uint32_t *>(tiled_sign + ((t * C + c) * kRowTile + lane) * 4);
    for (int b = 0; b < 16; ++b) {
      const uint32_t byte = src[b];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t g = (int64_t)c * 32 + 2 * b + h;  // pair / triple index
        const uint32_t idx = h ? (byte >> 4) : (byte & 15);
        if (g >= groups) continue;
        if (FMT == TB_TL1) {
          if (idx <= 8) acc += lut[g * 9 + idx];
        } else {
          if (idx <= 13) {
            const int32_t e = lut[g * 14 + idx];
            acc += ((sg >> (2 * b + h)) & 1) ? -e : e;
          }
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

// --------------------------------------------------------------------------
// host side
// --------------------------------------------------------------------------
template <int FMT, int MT>
static int launch_tgemv(const GemvParams &p, cudaStream_t s, int grid) {
  static bool configured = false;
  const size_t smem = gemv_smem_bytes<FMT>(p.M, p.Cs);
  if (!configured) {
    if (cudaFuncSetAttribute(tgemv_kernel<FMT, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024) != cudaSuccess)
      return TB_ERR_CUDA;
    configured = true;
  }
  tgemv_kernel<FMT, MT><<<grid, kThreads, smem, s>>>(p);
  TB_CHECK_LAUNCH();
  return TB_OK;
}

template <int FMT>
static int dispatch_m(const GemvParams &p, cudaStream_t s, int grid) {
  if (p.M <= 1) return launch_tgemv<FMT, 1>(p, s, grid);
  if (p.M <= 2) return launch_tgemv<FMT, 2>(p, s, grid);
  if (p.M <= 4) return launch_tgemv<FMT, 4>(p, s, grid);
  if (p.M <= 8) return launch_tgemv<FMT, 8>(p, s, grid);
  return launch_tgemv<FMT, 16>(p, s, grid);
}

}  // namespace tb

using namespace tb;

extern "C" int64_t tb_gemv_workspace_bytes(int fmt, int64_t rows, int64_t cols) {
  if (rows < 1 || cols < 1 || fmt < TB_I2S || fmt > TB_TL2) return -1;
  const int64_t T = ceil_div(rows, kRowTile);
  return (16 * T * kRowTile + T) * (int64_t)sizeof(int32_t);
}

extern "C" int tb_gemv(int fmt, const uint8_t *tiled, const uint8_t *tiled_sign, int64_t rows,
                       int64_t cols, const int8_t *act, int64_t M, int64_t ld_act,
                       int64_t act_len, const double *a_scale, double w_scale, void *workspace,
                       int32_t *acc_out, double *out64, float *out32, void *stream) {
  if (!tiled || !act || !workspace || rows < 1 || cols < 1 || M < 1 || M > 16 || ld_act < 1 ||
      act_len < 0 || act_len > ld_act || (fmt == TB_TL2 && !tiled_sign) ||
      ((out64 || out32) && !a_scale) || fmt < TB_I2S || fmt > TB_TL2)
    return TB_ERR_ARGUMENT;
  if (rows > (int64_t)1 << 30) return TB_ERR_UNSUPPORTED;
  const int64_t C = ceil_div(ref_row_bytes(fmt, cols), kChunkBytes);
  const int64_t T = ceil_div(rows, kRowTile);
  const int act_words = fmt == TB_TL2 ? 24 : 16;
  // split K into passes so the staged activations fit the SMEM budget
  const int64_t per_chunk = M * (act_words * 4 + 4);
  const int64_t passes = ceil_div(C * per_chunk, kActSmemBudget);
  const int64_t Cs_nom = ceil_div(C, passes);
  GemvParams p{};
  p.wmain = tiled;
  p.wsign = tiled_sign;
  p.act = act;
  p.ld_act = ld_act;
  p.act_len = act_len;
  p.a_scale = a_scale;
  p.w_scale = w_scale;
  p.ws_acc = static_cast<int32_t *>(workspace);
  p.ws_cnt = p.ws_acc + 16 * T * kRowTile;
  p.acc_out = acc_out;
  p.out64 = out64;
  p.out32 = out32;
  p.N = (int)rows;
  p.Npad = (int)(T * kRowTile);
  p.T = (int)T;
  p.C = (int)C;
  p.M = (int)M;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int64_t c0 = 0; c0 < C; c0 += Cs_nom) {
    p.c0 = (int)c0;
    p.Cs = (int)std::min<int64_t>(Cs_nom, C - c0);
    p.total = T * p.Cs;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(sm_count_cached(), p.total));
    int st;
    if (fmt == TB_I2S) st = dispatch_m<TB_I2S>(p, s, grid);
    else if (fmt == TB_TL1) st = dispatch_m<TB_TL1>(p, s, grid);
    else st = dispatch_m<TB_TL2>(p, s, grid);
    if (st != TB_OK) return st;
  }
  return TB_OK;
}

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
