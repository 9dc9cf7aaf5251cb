/*
 * tern_oracle.c -- C restatement of the reference's CPU hot path.
 * TEST / BASELINE INFRASTRUCTURE ONLY (see oracle/ternpack_oracle.py header):
 * used by tests/ as a second checker and by bench.py's cpu_baseline and
 * `--impl reference` legs as the "port" of the reference CPU implementation.
 * Never linked into the product.
 *
 * Algorithm = the reference's byte-table gather kernels:
 *   quantize            pkg/src/ternpack/core.py:116-134
 *   LUT build           lut.py:65-84
 *   I2_S byte table     kernels.py:75-83 + _fast.py:98-129
 *   TL1 byte table      kernels.py:97-106 + _fast.py:115-129
 *   TL2 signed table    kernels.py:129-137 + _fast.py:132-147
 *   byte_gemv           _fast.py:25-51
 *   tl2_byte_gemv       _fast.py:54-95
 * Row ranges are split across OpenMP threads like gemv_parallel's row chunks
 * (kernels.py:176-186); integer results are identical for any thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static double rha(double v) { return trunc(v + copysign(0.5, v)); }

int to_quantize_f32(const float *x, int64_t K, int64_t kpad, int8_t *q, double *scale) {
  double amax = 0.0;
  for (int64_t k = 0; k < K; ++k) {
    double v = fabs((double)x[k]);
    if (!isfinite(v)) return 1;
    if (v > amax) amax = v;
  }
  double s = amax > 0.0 ? amax / 127.0 : 1.0;
  for (int64_t k = 0; k < kpad; ++k) {
    if (k < K) {
      double v = rha((double)x[k] / s);
      if (v > 127.0) v = 127.0;
      if (v < -127.0) v = -127.0;
      q[k] = (int8_t)v;
    } else {
      q[k] = 0;
    }
  }
  *scale = s;
  return 0;
}

void to_lut_tl1(const int8_t *a, int64_t len, int64_t groups, int16_t *e) {
  for (int64_t g = 0; g < groups; ++g) {
    int a0 = 2 * g < len ? a[2 * g] : 0, a1 = 2 * g + 1 < len ? a[2 * g + 1] : 0;
    for (int i = 0; i < 9; ++i) e[g * 9 + i] = (int16_t)((i / 3 - 1) * a0 + (i % 3 - 1) * a1);
  }
}

void to_lut_tl2(const int8_t *a, int64_t len, int64_t groups, int16_t *e) {
  for (int64_t g = 0; g < groups; ++g) {
    int av[3];
    for (int j = 0; j < 3; ++j) av[j] = 3 * g + j < len ? a[3 * g + j] : 0;
    for (int i = 0; i < 14; ++i) {
      int d = i + 13;
      e[g * 14 + i] = (int16_t)((d / 9 - 1) * av[0] + (d / 3 % 3 - 1) * av[1] + (d % 3 - 1) * av[2]);
    }
  }
}

/* t[j][b] = sum_s ((b >> 2s) & 3) - 1) * a[4j+s] */
void to_i2s_byte_table(const int8_t *a, int64_t len, int64_t bc, int32_t *t) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < bc; ++j) {
    int av[4];
    for (int s = 0; s < 4; ++s) av[s] = 4 * j + s < len ? a[4 * j + s] : 0;
    int32_t lo[16], hi[16];
    for (int n = 0; n < 16; ++n) {
      lo[n] = ((n & 3) - 1) * av[0] + ((n >> 2) - 1) * av[1];
      hi[n] = ((n & 3) - 1) * av[2] + ((n >> 2) - 1) * av[3];
    }
    for (int b = 0; b < 256; ++b) t[j * 256 + b] = lo[b & 15] + hi[b >> 4];
  }
}

/* t[j][b] = lut[2j][b & 15] + lut[2j+1][b >> 4]  (zero past 9 entries / groups) */
void to_tl1_byte_table(const int16_t *lut, int64_t groups, int64_t bc, int32_t *t) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < bc; ++j) {
    int32_t lo[16] = {0}, hi[16] = {0};
    for (int n = 0; n < 9; ++n) {
      if (2 * j < groups) lo[n] = lut[(2 * j) * 9 + n];
      if (2 * j + 1 < groups) hi[n] = lut[(2 * j + 1) * 9 + n];
    }
    for (int b = 0; b < 256; ++b) t[j * 256 + b] = lo[b & 15] + hi[b >> 4];
  }
}

/* 1024-entry tables: index = (sign pair << 8) | byte, signs applied */
void to_tl2_signed_table(const int16_t *lut, int64_t groups, int32_t *t) {
  const int64_t bc = groups / 2;
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < bc; ++j) {
    int32_t lo[16] = {0}, hi[16] = {0};
    for (int n = 0; n < 14; ++n) {
      lo[n] = lut[(2 * j) * 14 + n];
      hi[n] = lut[(2 * j + 1) * 14 + n];
    }
    for (int s = 0; s < 4; ++s) {
      int fl = 1 - 2 * (s & 1), fh = 1 - 2 * (s >> 1);
      for (int b = 0; b < 256; ++b) t[j * 1024 + (s << 8) + b] = fh * hi[b >> 4] + fl * lo[b & 15];
    }
  }
}

void to_byte_gemv(const uint8_t *packed, int64_t rows, int64_t bc, const int32_t *t, int32_t *out,
                  int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < rows; ++i) {
    const uint8_t *p = packed + i * bc;
    int32_t acc = 0;
    for (int64_t j = 0; j < bc; ++j) acc += t[j * 256 + p[j]];
    out[i] = acc;
  }
}

void to_tl2_byte_gemv(const uint8_t *idx, const uint8_t *sign, int64_t rows, int64_t bc,
                      int64_t sbc, const int32_t *t, int32_t *out, int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < rows; ++i) {
    const uint8_t *p = idx + i * bc, *sg = sign + i * sbc;
    int32_t acc = 0;
    for (int64_t j = 0; j < bc; ++j) {
      int s = (sg[j >> 2] >> ((j & 3) * 2)) & 3;
      acc += t[j * 1024 + (s << 8) + p[j]];
    }
    out[i] = acc;
  }
}

void to_gemv_ref_int32(const int8_t *v, int64_t rows, int64_t cols, const int8_t *a, int32_t *out,
                       int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < rows; ++i) {
    int32_t acc = 0;
    for (int64_t k = 0; k < cols; ++k) acc += (int32_t)v[i * cols + k] * (int32_t)a[k];
    out[i] = acc;
  }
}

int to_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
