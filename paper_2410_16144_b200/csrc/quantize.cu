// Activation quantisation, weight ternarisation and output scaling
// (reference: pkg/src/ternpack/core.py:24-27, 99-101, 104-113, 116-134).
#include <cfloat>

#include "common.cuh"

namespace tb {

// ----------------------------------------------------------------------------
// quantize_activations: one CTA per token.  Float64 arithmetic end to end so
// the int8 codes and the scale are bit-identical to NumPy's (an fp32 divide
// mismatches ~1 element in 0.9M).
// ----------------------------------------------------------------------------
template <typename T, int kThreads>
__global__ void __launch_bounds__(kThreads) quantize_kernel(const T *__restrict__ x, int64_t K,
                                                            int64_t ldx, int8_t *__restrict__ q,
                                                            int64_t ldq, double *__restrict__ scale,
                                                            int32_t *nonfinite) {
  const int64_t m = blockIdx.x;
  const T *row = x + m * ldx;
  int8_t *qrow = q + m * ldq;
  double amax = 0.0;
  bool bad = false;
  for (int64_t k = threadIdx.x; k < K; k += kThreads) {
    double v = static_cast<double>(row[k]);
    bad |= !isfinite(v);
    amax = fmax(amax, fabs(v));
  }
  __shared__ double red[kThreads / 32];
  __shared__ double s_scale;
  for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
  if (bad && nonfinite) atomicOr(nonfinite, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) a = fmax(a, red[i]);
    double s = a > 0.0 ? a / 127.0 : 1.0;
    s_scale = s;
    scale[m] = s;
  }
  __syncthreads();
  const double s = s_scale;
  const double inv_s = 1.0 / s;
  const float inv_sf = static_cast<float>(inv_s);
  for (int64_t k = threadIdx.x; k < ldq; k += kThreads) {
    int q = 0;
    if (k < K) {
      if constexpr (sizeof(T) == 4) q = quantize_fast(row[k], inv_sf, s, inv_s);
      else q = quantize_one(static_cast<double>(row[k]), s, inv_s);
    }
    qrow[k] = static_cast<int8_t>(q);
  }
}

// ----------------------------------------------------------------------------
// NumPy pairwise summation of |w| (numpy/core/src/umath/loops_utils.h
// pairwise_sum, PW_BLOCKSIZE 128, 8-way unrolled leaves), evaluated over one
// subtree per thread in the exact association order NumPy uses.
// ----------------------------------------------------------------------------
template <typename T>
__device__ double pairwise_abs(const T *a, int64_t n, bool &bad) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      double v = fabs(static_cast<double>(a[i]));
      bad |= !isfinite(v);
      res += v;
    }
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      r[j] = fabs(static_cast<double>(a[j]));
      bad |= !isfinite(r[j]);
    }
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        double v = fabs(static_cast<double>(a[i + j]));
        bad |= !isfinite(v);
        r[j] += v;
      }
    }
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) {
      double v = fabs(static_cast<double>(a[i]));
      bad |= !isfinite(v);
      res += v;
    }
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  double left = pairwise_abs(a, n2, bad);
  return left + pairwise_abs(a + n2, n - n2, bad);
}

template <typename T>
__global__ void pairwise_sums_kernel(const T *__restrict__ w, const int64_t *__restrict__ off,
                                     const int64_t *__restrict__ len, int64_t nsub,
                                     double *__restrict__ sums, int32_t *nonfinite) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nsub) return;
  bool bad = false;
  sums[i] = pairwise_abs(w + off[i], len[i], bad);
  if (bad && nonfinite) atomicOr(nonfinite, 1);
}

template <typename T>
__global__ void ternarize_apply_kernel(const T *__restrict__ w, int64_t n, double scale,
                                       int8_t *__restrict__ q) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = rha(static_cast<double>(w[i]) / scale);
    q[i] = static_cast<int8_t>(v > 1.0 ? 1 : (v < -1.0 ? -1 : static_cast<int>(v)));
  }
}

__global__ void scale_outputs_kernel(const int32_t *__restrict__ acc, int64_t M, int64_t N,
                                     double w_scale, const double *__restrict__ a_scale,
                                     double *__restrict__ out64, float *__restrict__ out32) {
  int64_t total = M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = static_cast<double>(acc[i]) * w_scale * a_scale[i / N];
    if (out64) out64[i] = v;
    if (out32) out32[i] = static_cast<float>(v);
  }
}

static int grid_for(int64_t n, int threads) {
  int64_t g = ceil_div(n, threads);
  int64_t cap = (int64_t)sm_count_cached() * 8;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

template <typename T>
static int quantize_impl(const T *x, int64_t M, int64_t K, int64_t ldx, int8_t *q, int64_t ldq,
                         double *scale, int32_t *flag, void *stream) {
  if (!x || !q || !scale || M < 0 || K < 1 || ldx < K || ldq < K) return TB_ERR_ARGUMENT;
  if (M == 0) return TB_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (K <= 8192)
    quantize_kernel<T, 512><<<(unsigned)M, 512, 0, s>>>(x, K, ldx, q, ldq, scale, flag);
  else
    quantize_kernel<T, 1024><<<(unsigned)M, 1024, 0, s>>>(x, K, ldx, q, ldq, scale, flag);
  TB_CHECK_LAUNCH();
  return TB_OK;
}

template <typename T>
static int sums_impl(const T *w, const int64_t *off, const int64_t *len, int64_t nsub,
                     double *sums, int32_t *flag, void *stream) {
  if (!w || !off || !len || !sums || nsub < 0) return TB_ERR_ARGUMENT;
  if (nsub == 0) return TB_OK;
  pairwise_sums_kernel<T><<<(unsigned)ceil_div(nsub, 128), 128, 0,
                            static_cast<cudaStream_t>(stream)>>>(w, off, len, nsub, sums, flag);
  TB_CHECK_LAUNCH();
  return TB_OK;
}

template <typename T>
static int apply_impl(const T *w, int64_t n, double scale, int8_t *q, void *stream) {
  if (!w || !q || n < 0 || !(scale > 0.0)) return TB_ERR_ARGUMENT;
  if (n == 0) return TB_OK;
  ternarize_apply_kernel<T><<<grid_for(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      w, n, scale, q);
  TB_CHECK_LAUNCH();
  return TB_OK;
}

}  // namespace tb

using namespace tb;

extern "C" int tb_quantize_f32(const float *x, int64_t M, int64_t K, int64_t ldx, int8_t *q,
                               int64_t ldq, double *scale, int32_t *flag, void *stream) {
  return quantize_impl(x, M, K, ldx, q, ldq, scale, flag, stream);
}
extern "C" int tb_quantize_f64(const double *x, int64_t M, int64_t K, int64_t ldx, int8_t *q,
                               int64_t ldq, double *scale, int32_t *flag, void *stream) {
  return quantize_impl(x, M, K, ldx, q, ldq, scale, flag, stream);
}
extern "C" int tb_abs_pairwise_sums_f32(const float *w, const int64_t *off, const int64_t *len,
                                        int64_t nsub, double *sums, int32_t *flag, void *stream) {
  return sums_impl(w, off, len, nsub, sums, flag, stream);
}
extern "C" int tb_abs_pairwise_sums_f64(const double *w, const int64_t *off, const int64_t *len,
                                        int64_t nsub, double *sums, int32_t *flag, void *stream) {
  return sums_impl(w, off, len, nsub, sums, flag, stream);
}
extern "C" int tb_ternarize_apply_f32(const float *w, int64_t n, double scale, int8_t *q,
                                      void *stream) {
  return apply_impl(w, n, scale, q, stream);
}
extern "C" int tb_ternarize_apply_f64(const double *w, int64_t n, double scale, int8_t *q,
                                      void *stream) {
  return apply_impl(w, n, scale, q, stream);
}
extern "C" int tb_scale_outputs(const int32_t *acc, int64_t M, int64_t N, double w_scale,
                                const double *a_scale, double *out64, float *out32,
                                void *stream) {
  if (!acc || !a_scale || M < 0 || N < 0) return TB_ERR_ARGUMENT;
  if (M * N == 0 || (!out64 && !out32)) return TB_OK;
  scale_outputs_kernel<<<grid_for(M * N, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      acc, M, N, w_scale, a_scale, out64, out32);
  TB_CHECK_LAUNCH();
  return TB_OK;
}
