// Packing codecs, validation, tile repack and activation LUTs
// (reference: pkg/src/ternpack/packing.py:42-277, lut.py:52-84).
#include <climits>

#include "common.cuh"

namespace tb {

__device__ __forceinline__ int val_at(const int8_t *v, int64_t r, int64_t c, int64_t cols) {
  return c < cols ? v[r * cols + c] : 0;  // zero weights pad every format
}

// ---- encoders: one thread per output byte --------------------------------

__global__ void encode_i2s_kernel(const int8_t *v, int64_t rows, int64_t cols, uint8_t *out) {
  const int64_t bpr = ref_row_bytes(TB_I2S, cols);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * bpr;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / bpr, j = i % bpr;
    uint32_t b = 0;
#pragma unroll
    for (int s = 0; s < 4; ++s) b |= (uint32_t)(val_at(v, r, 4 * j + s, cols) + 1) << (2 * s);
    out[i] = (uint8_t)b;
  }
}

__global__ void encode_tl1_kernel(const int8_t *v, int64_t rows, int64_t cols, uint8_t *out) {
  const int64_t bpr = ref_row_bytes(TB_TL1, cols);
  const int64_t groups = pad_up(cols, 2) / 2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * bpr;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / bpr, j = i % bpr;
    uint32_t b = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int64_t g = 2 * j + h;
      uint32_t idx = 4;  // filler (0, 0) pair for an odd group count (packing.py:35)
      if (g < groups)
        idx = 3 * (val_at(v, r, 2 * g, cols) + 1) + (val_at(v, r, 2 * g + 1, cols) + 1);
      b |= idx << (4 * h);
    }
    out[i] = (uint8_t)b;
  }
}

__device__ __forceinline__ void tl2_code_of(const int8_t *v, int64_t r, int64_t g, int64_t cols,
                                            uint32_t &sign, uint32_t &idx) {
  int d = 9 * (val_at(v, r, 3 * g, cols) + 1) + 3 * (val_at(v, r, 3 * g + 1, cols) + 1) +
          (val_at(v, r, 3 * g + 2, cols) + 1) - 13;
  sign = d < 0;
  idx = d < 0 ? -d : d;
}

__global__ void encode_tl2_kernel(const int8_t *v, int64_t rows, int64_t cols, uint8_t *out,
                                  uint8_t *sign_out) {
  const int64_t ibpr = ref_row_bytes(TB_TL2, cols);
  const int64_t sbpr = ref_sign_row_bytes(cols);
  const int64_t groups = pad_up(cols, 6) / 3;
  const int64_t total = rows * (ibpr + sbpr);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < rows * ibpr) {
      int64_t r = i / ibpr, j = i % ibpr;
      uint32_t s0, i0, s1, i1;
      tl2_code_of(v, r, 2 * j, cols, s0, i0);
      tl2_code_of(v, r, 2 * j + 1, cols, s1, i1);
      out[i] = (uint8_t)(i0 | (i1 << 4));
    } else {
      int64_t k = i - rows * ibpr;
      int64_t r = k / sbpr, j = k % sbpr;
      uint32_t b = 0;
      for (int t = 0; t < 8; ++t) {
        int64_t g = 8 * j + t;
        if (g >= groups) break;
        uint32_t s, idx;
        tl2_code_of(v, r, g, cols, s, idx);
        b |= s << t;
      }
      sign_out[k] = (uint8_t)b;
    }
  }
}

// ---- decoders / validators -------------------------------------------------
// bad kinds: 1 = invalid code, 2 = TL2 non-canonical zero

__device__ __forceinline__ int tl2_sign_bit(const uint8_t *sign, int64_t r, int64_t sbpr,
                                            int64_t g) {
  return (sign[r * sbpr + (g >> 3)] >> (g & 7)) & 1;
}

__device__ __forceinline__ int tl2_nibble(const uint8_t *idx, int64_t r, int64_t ibpr,
                                          int64_t g) {
  uint8_t b = idx[r * ibpr + (g >> 1)];
  return (g & 1) ? (b >> 4) : (b & 15);
}

__global__ void decode_kernel(int fmt, const uint8_t *data, const uint8_t *sign, int64_t rows,
                              int64_t cols, int8_t *vals, int32_t *bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * cols;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / cols, c = i % cols;
    int w = 0;
    if (fmt == TB_I2S) {
      const int64_t bpr = ref_row_bytes(TB_I2S, cols);
      int code = (data[r * bpr + c / 4] >> (2 * (c & 3))) & 3;
      if (code == 3) atomicOr(bad, 1);
      w = code - 1;
    } else if (fmt == TB_TL1) {
      const int64_t bpr = ref_row_bytes(TB_TL1, cols);
      int64_t g = c / 2;
      uint8_t b = data[r * bpr + g / 2];
      int nib = (g & 1) ? (b >> 4) : (b & 15);
      if (nib > 8) atomicOr(bad, 1);
      w = (c & 1) ? (nib % 3 - 1) : (nib / 3 - 1);
    } else {
      const int64_t ibpr = ref_row_bytes(TB_TL2, cols), sbpr = ref_sign_row_bytes(cols);
      int64_t g = c / 3;
      int nib = tl2_nibble(data, r, ibpr, g);
      int s = tl2_sign_bit(sign, r, sbpr, g);
      if (nib > 13) atomicOr(bad, 1);
      else if (s && nib == 0) atomicOr(bad, 2);
      int d = nib * (1 - 2 * s) + 13;
      int p = c % 3;
      w = (p == 0 ? d / 9 : (p == 1 ? (d / 3) % 3 : d % 3)) - 1;
    }
    vals[i] = (int8_t)w;
  }
  // the reference also rejects invalid codes in the padding region
  if (fmt == TB_I2S || fmt == TB_TL1) {
    const int64_t bpr = ref_row_bytes(fmt, cols);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * bpr;
         i += (int64_t)gridDim.x * blockDim.x) {
      uint8_t b = data[i];
      bool badb = fmt == TB_I2S ? ((b & 3) == 3 || ((b >> 2) & 3) == 3 || ((b >> 4) & 3) == 3 ||
                                   (b >> 6) == 3)
                                : ((b & 15) > 8 || (b >> 4) > 8);
      if (badb) atomicOr(bad, 1);
    }
  } else {
    const int64_t ibpr = ref_row_bytes(TB_TL2, cols), sbpr = ref_sign_row_bytes(cols);
    const int64_t groups = pad_up(cols, 6) / 3;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * groups;
         i += (int64_t)gridDim.x * blockDim.x) {
      int64_t r = i / groups, g = i % groups;
      int nib = tl2_nibble(data, r, ibpr, g);
      int s = tl2_sign_bit(sign, r, sbpr, g);
      if (nib > 13) atomicOr(bad, 1);
      else if (s && nib == 0) atomicOr(bad, 2);
    }
  }
}

__global__ void validate_kernel(int fmt, const uint8_t *data, const uint8_t *sign, int64_t rows,
                                int64_t cols, int32_t *first_bad) {
  if (fmt == TB_I2S || fmt == TB_TL1) {
    const int64_t bpr = ref_row_bytes(fmt, cols);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * bpr;
         i += (int64_t)gridDim.x * blockDim.x) {
      uint8_t b = data[i];
      bool badb = fmt == TB_I2S ? ((b & 3) == 3 || ((b >> 2) & 3) == 3 || ((b >> 4) & 3) == 3 ||
                                   (b >> 6) == 3)
                                : ((b & 15) > 8 || (b >> 4) > 8);
      if (badb) atomicMin(&first_bad[0], (int32_t)(i / bpr));
    }
  } else {
    const int64_t ibpr = ref_row_bytes(TB_TL2, cols), sbpr = ref_sign_row_bytes(cols);
    const int64_t groups = pad_up(cols, 6) / 3;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * groups;
         i += (int64_t)gridDim.x * blockDim.x) {
      int64_t r = i / groups, g = i % groups;
      int nib = tl2_nibble(data, r, ibpr, g);
      int s = tl2_sign_bit(sign, r, sbpr, g);
      if (nib > 13) atomicMin(&first_bad[0], (int32_t)r);
      if (s && nib == 0) atomicMin(&first_bad[1], (int32_t)r);
    }
  }
}

// ---- tile repack: reference rows -> [tile][chunk][row][16 B] -------------
// TL1 bytes are re-encoded on the way: a pair index n = 3a + b (packing.py:
// 56-60; a = w0 + 1, b = w1 + 1) becomes the two 2-bit codes (a, b), so a TL1
// byte (pairs 2j, 2j+1 = weights 4j..4j+3) turns into the I2_S byte of the
// same four weights.  Same 4 bits per pair, lossless for valid indices (the
// only kind that reaches a kernel: validate() runs first), and the decode
// GEMV / GEMM run one inner loop for both formats.  tb_unrepack inverts it.

__device__ __forceinline__ uint8_t tl1_to_codes(uint32_t byte) {
  const uint32_t lo = byte & 15u, hi = byte >> 4;
  const uint32_t alo = (lo * 11u) >> 5, ahi = (hi * 11u) >> 5;  // n / 3 for n <= 8
  return (uint8_t)(alo | ((lo - 3u * alo) << 2) | (ahi << 4) | ((hi - 3u * ahi) << 6));
}

__device__ __forceinline__ uint8_t codes_to_tl1(uint32_t c) {
  const uint32_t lo = 3u * (c & 3u) + ((c >> 2) & 3u), hi = 3u * ((c >> 4) & 3u) + ((c >> 6) & 3u);
  return (uint8_t)(lo | (hi << 4));
}

// TL2 triples are re-encoded on the way to the tiled layout: (sign s, index
// idx) -> v = 13 + (s ? -idx : idx) = 9 c0 + 3 c1 + c2 (c = w + 1, the
// base-3 number of the triple, packing.py:63-74): the same 5 bits per triple,
// a bijection (zero is v = 13), so the decode takes the digits straight from
// v; the bits are placed for a cheap byte-lane extraction (common.cuh
// tl2_bit).  tb_unrepack inverts it.
// idx16 / sgn32: the chunk row's 16 reference index bytes and 32 sign bits
// -> the five tile words (common.cuh tl2_bit)
__device__ __forceinline__ void tl2_to_tile(const uint8_t *idx16, uint32_t sgn32, uint32_t X[5]) {
#pragma unroll
  for (int k = 0; k < 5; ++k) X[k] = 0;
#pragma unroll
  for (int t = 0; t < 32; ++t) {
    const uint32_t nib = (idx16[t >> 1] >> (4 * (t & 1))) & 15u;
    const uint32_t s = (sgn32 >> t) & 1u;
    const uint32_t v = (s ? 13u - nib : 13u + nib) + 1u;  // stored biased: 1..27 (tl2_tile_value)
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const Tl2Bit p = tl2_bit(t, k);
      X[p.word] |= ((v >> k) & 1u) << p.bit;
    }
  }
}
__device__ __forceinline__ void tile_to_tl2(const uint32_t X[5], uint8_t *idx16, uint32_t &sgn32) {
  uint32_t out = 0;
#pragma unroll
  for (int b = 0; b < 16; ++b) idx16[b] = 0;
#pragma unroll
  for (int t = 0; t < 32; ++t) {
    const uint32_t v = tl2_tile_value(X, t);
    const uint32_t s = v < 13u ? 1u : 0u;
    const uint32_t nib = s ? 13u - v : v - 13u;
    idx16[t >> 1] |= (uint8_t)(nib << (4 * (t & 1)));
    out |= s << t;
  }
  sgn32 = out;
}

__global__ void repack_kernel(int fmt, const uint8_t *ref, const uint8_t *ref_sign, int64_t rows,
                              int64_t cols, uint8_t *tiled, uint8_t *tiled_sign, int64_t C,
                              int64_t T) {
  const int64_t rb = ref_row_bytes(fmt, cols);
  const int64_t sbpr = fmt == TB_TL2 ? ref_sign_row_bytes(cols) : 0;
  const uint8_t zb = zero_byte(fmt);
  const int64_t total = T * C * kRowTile;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r_in = i % kRowTile;
    int64_t c = (i / kRowTile) % C;
    int64_t t = i / (kRowTile * C);
    int64_t r = t * kRowTile + r_in;
    uint8_t buf[16];
#pragma unroll
    for (int b = 0; b < 16; ++b) {
      int64_t j = 16 * c + b;
      buf[b] = (r < rows && j < rb) ? ref[r * rb + j] : zb;
      if (fmt == TB_TL1) buf[b] = tl1_to_codes(buf[b]);
    }
    uint32_t sv = 0;
    if (fmt == TB_TL2) {
      uint8_t sb[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        int64_t j = 4 * c + b;
        sb[b] = (r < rows && j < sbpr) ? ref_sign[r * sbpr + j] : 0;
      }
      memcpy(&sv, sb, 4);
      uint32_t X[5];
      tl2_to_tile(buf, sv, X);
      reinterpret_cast<uint32_t *>(tiled_sign)[i] = X[4];
      reinterpret_cast<uint4 *>(tiled)[i] = make_uint4(X[0], X[1], X[2], X[3]);
      continue;
    }
    uint4 v;
    memcpy(&v, buf, 16);
    reinterpret_cast<uint4 *>(tiled)[i] = v;
  }
}

__global__ void unrepack_kernel(int fmt, const uint8_t *tiled, const uint8_t *tiled_sign,
                                int64_t rows, int64_t cols, uint8_t *ref, uint8_t *ref_sign,
                                int64_t C) {
  const int64_t rb = ref_row_bytes(fmt, cols);
  const int64_t sbpr = fmt == TB_TL2 ? ref_sign_row_bytes(cols) : 0;
  const int64_t total = rows * (rb + sbpr);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < rows * rb) {
      int64_t r = i / rb, j = i % rb;
      int64_t t = r / kRowTile, rin = r % kRowTile, c = j / 16, b = j % 16;
      const int64_t q = (t * C + c) * kRowTile + rin;
      if (fmt == TB_TL2) {  // the chunk's triples back to (sign, index)
        uint8_t idx16[16];
        uint32_t X[5], bits;
        memcpy(X, tiled + q * 16, 16);
        X[4] = reinterpret_cast<const uint32_t *>(tiled_sign)[q];
        tile_to_tl2(X, idx16, bits);
        ref[i] = idx16[b];
      } else {
        const uint8_t v = tiled[q * 16 + b];
        ref[i] = fmt == TB_TL1 ? codes_to_tl1(v) : v;
      }
    } else {
      int64_t k = i - rows * rb;
      int64_t r = k / sbpr, j = k % sbpr;
      int64_t t = r / kRowTile, rin = r % kRowTile, c = j / 4, b = j % 4;
      const int64_t q = (t * C + c) * kRowTile + rin;
      uint8_t idx16[16];
      uint32_t X[5], bits;
      memcpy(X, tiled + q * 16, 16);
      X[4] = reinterpret_cast<const uint32_t *>(tiled_sign)[q];
      tile_to_tl2(X, idx16, bits);
      ref_sign[k] = (uint8_t)(bits >> (8 * b));
    }
  }
}

// ---- activation LUTs: entry = pattern . (activation group) ----------------

__global__ void lut_kernel(int fmt, const int8_t *act, int64_t len, int64_t groups,
                           int16_t *entries) {
  const int width = fmt == TB_TL1 ? 2 : 3;
  const int npat = fmt == TB_TL1 ? 9 : 14;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < groups * npat;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t g = i / npat;
    int p = (int)(i % npat);
    int a[3];
    for (int j = 0; j < width; ++j) {
      int64_t k = g * width + j;
      a[j] = k < len ? act[k] : 0;
    }
    int e;
    if (fmt == TB_TL1) {
      e = (p / 3 - 1) * a[0] + (p % 3 - 1) * a[1];  // lut.py:20
    } else {
      int d = p + 13;  // lut.py:23-26: canonical triple with base-3 value p+13
      e = (d / 9 - 1) * a[0] + ((d / 3) % 3 - 1) * a[1] + (d % 3 - 1) * a[2];
    }
    entries[i] = (int16_t)e;
  }
}

static int grid_for(int64_t n, int threads) {
  int64_t g = ceil_div(n, threads);
  int64_t cap = (int64_t)sm_count_cached() * 16;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace tb

using namespace tb;

extern "C" int64_t tb_ref_row_bytes(int fmt, int64_t cols) {
  if (cols < 1 || fmt < TB_I2S || fmt > TB_TL2) return -1;
  return ref_row_bytes(fmt, cols);
}
extern "C" int64_t tb_ref_sign_row_bytes(int64_t cols) {
  return cols < 1 ? -1 : ref_sign_row_bytes(cols);
}
extern "C" int64_t tb_tiled_chunks(int fmt, int64_t cols) {
  if (cols < 1 || fmt < TB_I2S || fmt > TB_TL2) return -1;
  return ceil_div(ref_row_bytes(fmt, cols), kChunkBytes);
}
extern "C" int64_t tb_tiled_bytes(int fmt, int64_t rows, int64_t cols) {
  if (rows < 1) return -1;
  int64_t C = tb_tiled_chunks(fmt, cols);
  return C < 0 ? -1 : ceil_div(rows, kRowTile) * C * kTileChunkBytes;
}
extern "C" int64_t tb_tiled_sign_bytes(int fmt, int64_t rows, int64_t cols) {
  if (fmt != TB_TL2) return 0;
  if (rows < 1) return -1;
  int64_t C = tb_tiled_chunks(fmt, cols);
  return C < 0 ? -1 : ceil_div(rows, kRowTile) * C * kTileSignBytes;
}

extern "C" int tb_encode(int fmt, const int8_t *values, int64_t rows, int64_t cols, uint8_t *out,
                         uint8_t *sign, void *stream) {
  if (!values || !out || rows < 1 || cols < 1) return TB_ERR_ARGUMENT;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int64_t n = rows * ref_row_bytes(fmt, cols);
  if (fmt == TB_I2S) {
    encode_i2s_kernel<<<grid_for(n, 256), 256, 0, s>>>(values, rows, cols, out);
  } else if (fmt == TB_TL1) {
    encode_tl1_kernel<<<grid_for(n, 256), 256, 0, s>>>(values, rows, cols, out);
  } else if (fmt == TB_TL2) {
    if (!sign) return TB_ERR_ARGUMENT;
    n += rows * ref_sign_row_bytes(cols);
    encode_tl2_kernel<<<grid_for(n, 256), 256, 0, s>>>(values, rows, cols, out, sign);
  } else {
    return TB_ERR_ARGUMENT;
  }
  TB_CHECK_LAUNCH();
  return TB_OK;
}

extern "C" int tb_decode(int fmt, const uint8_t *data, const uint8_t *sign, int64_t rows,
                         int64_t cols, int8_t *values, int32_t *bad, void *stream) {
  if (!data || !values || !bad || rows < 1 || cols < 1 || fmt < TB_I2S || fmt > TB_TL2 ||
      (fmt == TB_TL2 && !sign))
    return TB_ERR_ARGUMENT;
  decode_kernel<<<grid_for(rows * cols, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      fmt, data, sign, rows, cols, values, bad);
  TB_CHECK_LAUNCH();
  return TB_OK;
}

extern "C" int tb_validate(int fmt, const uint8_t *data, const uint8_t *sign, int64_t rows,
                           int64_t cols, int32_t *first_bad, void *stream) {
  if (!data || !first_bad || rows < 1 || cols < 1 || fmt < TB_I2S || fmt > TB_TL2 ||
      (fmt == TB_TL2 && !sign))
    return TB_ERR_ARGUMENT;
  int64_t n = fmt == TB_TL2 ? rows * (pad_up(cols, 6) / 3) : rows * ref_row_bytes(fmt, cols);
  validate_kernel<<<grid_for(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      fmt, data, sign, rows, cols, first_bad);
  TB_CHECK_LAUNCH();
  return TB_OK;
}

extern "C" int tb_repack(int fmt, const uint8_t *ref, const uint8_t *ref_sign, int64_t rows,
                         int64_t cols, uint8_t *tiled, uint8_t *tiled_sign, void *stream) {
  if (!ref || !tiled || rows < 1 || cols < 1 || fmt < TB_I2S || fmt > TB_TL2 ||
      (fmt == TB_TL2 && (!ref_sign || !tiled_sign)))
    return TB_ERR_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(tiled) & 15) || (fmt == TB_TL2 && (reinterpret_cast<uintptr_t>(tiled_sign) & 3)))
    return TB_ERR_ARGUMENT;
  int64_t C = tb_tiled_chunks(fmt, cols), T = ceil_div(rows, kRowTile);
  repack_kernel<<<grid_for(T * C * kRowTile, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      fmt, ref, ref_sign, rows, cols, tiled, tiled_sign, C, T);
  TB_CHECK_LAUNCH();
  return TB_OK;
}

extern "C" int tb_unrepack(int fmt, const uint8_t *tiled, const uint8_t *tiled_sign, int64_t rows,
                           int64_t cols, uint8_t *ref, uint8_t *ref_sign, void *stream) {
  if (!ref || !tiled || rows < 1 || cols < 1 || fmt < TB_I2S || fmt > TB_TL2 ||
      (fmt == TB_TL2 && (!ref_sign || !tiled_sign)))
    return TB_ERR_ARGUMENT;
  int64_t C = tb_tiled_chunks(fmt, cols);
  int64_t n = rows * (ref_row_bytes(fmt, cols) + (fmt == TB_TL2 ? ref_sign_row_bytes(cols) : 0));
  unrepack_kernel<<<grid_for(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      fmt, tiled, tiled_sign, rows, cols, ref, ref_sign, C);
  TB_CHECK_LAUNCH();
  return TB_OK;
}

extern "C" int tb_build_lut(int fmt, const int8_t *act, int64_t len, int64_t groups,
                            int16_t *entries, void *stream) {
  if (!act || !entries || len < 0 || groups < 1 || (fmt != TB_TL1 && fmt != TB_TL2))
    return TB_ERR_ARGUMENT;
  int64_t n = groups * (fmt == TB_TL1 ? 9 : 14);
  lut_kernel<<<grid_for(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(fmt, act, len,
                                                                               groups, entries);
  TB_CHECK_LAUNCH();
  return TB_OK;
}
