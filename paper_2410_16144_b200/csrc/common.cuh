// Shared device helpers for the sm_100a ternary kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ternary_b200.h"

#define TB_CHECK_LAUNCH()                                   \
  do {                                                      \
    cudaError_t _e = cudaGetLastError();                    \
    if (_e != cudaSuccess) return TB_ERR_CUDA;              \
  } while (0)

namespace tb {

constexpr int kRowTile = 32;     // rows per tile == lanes per warp
constexpr int kChunkBytes = 16;  // bytes of one row's stream per chunk
constexpr int kTileChunkBytes = kRowTile * kChunkBytes;  // 512 B
constexpr int kTileSignBytes = kRowTile * 4;             // 128 B (TL2)

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t pad_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }
__host__ __device__ inline int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

// reference row bytes (packing.py:42-53)
__host__ __device__ inline int64_t ref_row_bytes(int fmt, int64_t cols) {
  if (fmt == TB_I2S) return pad_up(cols, 4) / 4;
  if (fmt == TB_TL1) return ceil_div(pad_up(cols, 2) / 2, 2);
  return pad_up(cols, 6) / 6;  // TL2 index plane
}
__host__ __device__ inline int64_t ref_sign_row_bytes(int64_t cols) {
  return ceil_div(pad_up(cols, 6) / 3, 8);
}
// weights covered by one 16-byte chunk
__host__ __device__ inline int chunk_weights(int fmt) { return fmt == TB_TL2 ? 96 : 64; }
// byte used to pad a row's stream (a run of zero weights)
__host__ __device__ inline uint8_t zero_byte(int fmt) {
  return fmt == TB_I2S ? 0x55 : (fmt == TB_TL1 ? 0x44 : 0x00);
}

// ---------------------------------------------------------------- PTX bits

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// CTA-local variant: make mbarrier.init (generic proxy) visible to the async
// proxy (cp.async.bulk complete_tx) without a cluster-scope release.
__device__ __forceinline__ void fence_mbar_init_cta() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// Pure polling (mbarrier.test_wait never suspends the thread): lowest
// hand-off latency for the tight producer / MMA / unpack rings of the GEMM.
__device__ __forceinline__ bool mbar_test_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_spin(uint64_t *bar, uint32_t parity) {
  while (!mbar_test_wait(bar, parity)) {
  }
}

// 1-D bulk async copy global -> shared, completion via mbarrier tx count.
// (cp.async.bulk: SASS UBLKCP; src/dst 16-B aligned, size multiple of 16.)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void red_add_s32(int32_t *p, int32_t v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// dot of 4 unsigned bytes (codes) with 4 signed bytes (activations)
__device__ __forceinline__ int dp4a_us(uint32_t codes, uint32_t act, int acc) {
  int r;
  asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(codes), "r"(act), "r"(acc));
  return r;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// Tiled TL2 (one row of a 96-weight chunk = 32 triples = 160 bits: four
// "main" words X0..X3 and the "sign" word X4).  Triple t = 8 i + 2 b + h
// (index byte 4 i + b of the chunk, nibble h) is lane b of group j = 2 i + h;
// its 5-bit value v (pack.cu tl2_to_v) is laid out so the decode gets a
// group's four values in the byte lanes of one register with masks and a
// shift or two -- no nibble split, no per-group sign merge:
//   groups 0..4: bits 0-4 of byte lane b of X_j             (one mask)
//   group 5: v bits 0-2 = bits 5-7 of X0, bits 3-4 = bits 5-6 of X1
//   group 6: v bits 0-2 = bits 5-7 of X2, bits 3-4 = bits 5-6 of X3
//   group 7: v bits 0-2 = bits 5-7 of X4, bit 3 = bit 7 of X1, bit 4 = bit 7 of X3
// (19 logic ops per 32 triples; the nibble + sign-plane form took 27.)
// tl2_bit(t, k): (word, bit) of bit k of triple t's value.
struct Tl2Bit {
  int word, bit;
};
__host__ __device__ __forceinline__ Tl2Bit tl2_bit(int t, int k) {
  const int i = t >> 3, b = (t >> 1) & 3, h = t & 1, j = 2 * i + h;
  if (j < 5) return Tl2Bit{j, 8 * b + k};
  if (j == 5) return k < 3 ? Tl2Bit{0, 8 * b + 5 + k} : Tl2Bit{1, 8 * b + 2 + k};
  if (j == 6) return k < 3 ? Tl2Bit{2, 8 * b + 5 + k} : Tl2Bit{3, 8 * b + 2 + k};
  return k < 3 ? Tl2Bit{4, 8 * b + 5 + k} : (k == 3 ? Tl2Bit{1, 8 * b + 7} : Tl2Bit{3, 8 * b + 7});
}
// value v = 9 c0 + 3 c1 + c2 of triple t from a row's five words (the tile
// stores v + 1: the decode's two divisions then need no bias add)
__host__ __device__ __forceinline__ uint32_t tl2_tile_value(const uint32_t X[5], int t) {
  uint32_t v = 0;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const Tl2Bit p = tl2_bit(t, k);
    v |= ((X[p.word] >> p.bit) & 1u) << k;
  }
  return v - 1u;
}
// the eight groups' byte-lane registers (group j: lane b = v + 1 of triple 8 (j/2) + 2 b + j%2)
__device__ __forceinline__ void tl2_tile_groups(const uint32_t X0, const uint32_t X1,
                                                const uint32_t X2, const uint32_t X3,
                                                const uint32_t X4, uint32_t v[8]) {
  v[0] = X0 & 0x1F1F1F1Fu;
  v[1] = X1 & 0x1F1F1F1Fu;
  v[2] = X2 & 0x1F1F1F1Fu;
  v[3] = X3 & 0x1F1F1F1Fu;
  v[4] = X4 & 0x1F1F1F1Fu;
  v[5] = ((X0 >> 5) & 0x07070707u) | ((X1 >> 2) & 0x18181818u);
  v[6] = ((X2 >> 5) & 0x07070707u) | ((X3 >> 2) & 0x18181818u);
  v[7] = ((X4 >> 5) & 0x07070707u) | ((X1 >> 4) & 0x08080808u) | ((X3 >> 3) & 0x10101010u);
}

__device__ __forceinline__ uint32_t lop3_sel(uint32_t p, uint32_t q, uint32_t m) {
  // (p & ~m) | (q & m)
  return (p & ~m) | (q & m);
}

// Round half away from zero in float64 exactly as core.py:24-27.
__device__ __forceinline__ double rha(double v) { return trunc(v + copysign(0.5, v)); }

// int8 code of one activation, bit-identical to clip(rha(x / s), -127, 127)
// in float64 (core.py:24-27, 128-130) without a division per element: v' =
// x * (1/s) is within a few ulp of the correctly rounded x / s, which decides
// the same code unless v' sits within 1e-9 of a rounding tie (k + 0.5) -- then
// the exact quotient is evaluated.  (|v| <= 127, so 1e-9 >> the few-ulp error.)
// The exact division is a real call (never if-converted: a float64 divide per
// element would otherwise be paid on every element, not just near ties).
static __device__ __noinline__ double div_exact(double x, double s) { return x / s; }

__device__ __forceinline__ int quantize_one(double x, double s, double inv_s) {
  const double v1 = x * inv_s;
  const double a = fabs(v1);
  const double f = a - floor(a);
  double v = v1;
  if (fabs(f - 0.5) <= 1e-9) v = div_exact(x, s);
  double y = rha(v);
  y = fmin(fmax(y, -127.0), 127.0);
  return static_cast<int>(y);
}

static __device__ __noinline__ int quantize_one_call(double x, double s, double inv_s) {
  return quantize_one(x, s, inv_s);
}

// float32 input, float32 fast path: v = x * inv_s in fp32 is within 1.6e-5
// of the exact quotient x / s (|v| <= 127, two roundings of 2^-24 relative).
// If v is more than 4e-5 away from a rounding tie (|v - rint(v)| < 0.49996),
// the exact quotient rounds -- half away from zero or not -- to rint(v), the
// float64 reference's code (|v| <= 127 needs no clamp).  Otherwise defer to
// quantize_one (float64, exact division at ties).
__device__ __forceinline__ int quantize_fast(float x, float inv_sf, double s, double inv_s) {
  const float v = x * inv_sf;
  const float r = rintf(v);
  if (fabsf(v - r) < 0.49996f) return static_cast<int>(r);
  return quantize_one_call(static_cast<double>(x), s, inv_s);  // rare: near a tie
}

int sm_count_cached();

}  // namespace tb
