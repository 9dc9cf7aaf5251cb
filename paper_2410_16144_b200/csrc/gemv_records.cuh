// Activation records + per-chunk decode/contract for the decode GEMV (see gemv.cu).
#pragma once
#include "common.cuh"

namespace tb {

constexpr int kStageChunks = 4;  // chunks per ring stage (per warp)

template <int FMT>
struct Fmt {
  static constexpr int kGroup = FMT == TB_TL2 ? 6 : 4;          // byte stride inside a word
  static constexpr int kWeights = 16 * kGroup;                   // weights per chunk (64 / 96)
  static constexpr int kActWords = 4 * kGroup;                   // transposed words per chunk
  static constexpr int kRecBytes = FMT == TB_TL2 ? 112 : 80;     // words + sum, 16-B multiple
  static constexpr int kSignBytes = FMT == TB_TL2 ? kTileSignBytes : 0;
  static constexpr int kSlots = FMT == TB_I2S ? 4 : 6;
};


// ---------------------------------------------------------------------------
// activation records
//   I2_S / TL1 (64 acts / chunk): word 4i+s = (a[16i+s], a[16i+4+s], a[16i+8+s], a[16i+12+s])
//   TL2        (96 acts / chunk): word 6i+s = (a[24i+s], a[24i+6+s], a[24i+12+s], a[24i+18+s])
//   word kActWords = sum of the chunk's activations
// One thread per (token, chunk, group i); the 4 group threads are adjacent lanes.
// ---------------------------------------------------------------------------
template <int FMT>
__device__ __forceinline__ void write_group(uint8_t *rec_chunk, int i, const uint32_t (&r)[Fmt<FMT>::kGroup],
                                            int32_t gsum, bool on) {
  using F = Fmt<FMT>;
  // chunk sum over the 4 adjacent group lanes (all 32 lanes shuffle)
  gsum += __shfl_xor_sync(0xffffffffu, gsum, 1);
  gsum += __shfl_xor_sync(0xffffffffu, gsum, 2);
  if (!on) return;
  uint32_t *dst = reinterpret_cast<uint32_t *>(rec_chunk) + i * F::kGroup;
  if constexpr (FMT == TB_TL2) {
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      uint32_t word = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int b = 6 * j + s;
        word |= ((r[b >> 2] >> (8 * (b & 3))) & 0xFFu) << (8 * j);
      }
      dst[s] = word;
    }
  } else {  // 4x4 byte transpose
    const uint32_t t0 = prmt(r[0], r[1], 0x5140u), t1 = prmt(r[0], r[1], 0x7362u);
    const uint32_t t2 = prmt(r[2], r[3], 0x5140u), t3 = prmt(r[2], r[3], 0x7362u);
    uint4 o;
    o.x = prmt(t0, t2, 0x5410u);
    o.y = prmt(t0, t2, 0x7632u);
    o.z = prmt(t1, t3, 0x5410u);
    o.w = prmt(t1, t3, 0x7632u);
    reinterpret_cast<uint4 *>(dst)[0] = o;
  }
  if (i == 0) *reinterpret_cast<int4 *>(rec_chunk + F::kActWords * 4) = make_int4(gsum, 0, 0, 0);
}

template <int FMT>
__global__ void act_prep_kernel(const int8_t *__restrict__ act, int M, int64_t ld, int64_t act_len,
                                int C, uint8_t *__restrict__ rec) {
  using F = Fmt<FMT>;
  const int lane = threadIdx.x & 31;
  const int64_t n4 = (int64_t)M * C * 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x - lane); base < n4;
       base += stride) {  // warp-uniform trip count (shuffles inside)
    const int64_t idx = base + lane;
    const bool on = idx < n4;
    const int64_t rc = on ? idx >> 2 : 0;
    const int i = (int)(idx & 3);
    const int m = (int)(rc / C), c = (int)(rc % C);
    const int64_t k0 = (int64_t)c * F::kWeights + i * 4 * F::kGroup;
    const int8_t *arow = act + m * ld;
    uint32_t r[F::kGroup];
#pragma unroll
    for (int v = 0; v < F::kGroup; ++v) {
      uint32_t word = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int64_t k = k0 + 4 * v + b;
        word |= (on && k < act_len ? (uint32_t)(uint8_t)arow[k] : 0u) << (8 * b);
      }
      r[v] = word;
    }
    int32_t s = 0;
#pragma unroll
    for (int v = 0; v < F::kGroup; ++v) s = __dp4a((int)r[v], 0x01010101, s);
    write_group<FMT>(rec + rc * F::kRecBytes, i, r, s, on);
  }
}

// quantize_activations (core.py:116-134) fused with record construction:
// one CTA per token, float64 absmax / divide / round-half-away, optional
// natural int8 output (the reference's QuantizedActivations.data).
// One thread-block CLUSTER per token (`ncta` CTAs of one cluster, this one
// being `rank`): each CTA owns a contiguous chunk range, the per-token absmax
// is combined through distributed shared memory, so a 14336-wide token is
// quantised by 8 SMs instead of one.  Called by every thread of the CTA.
template <int FMT, typename T, int kThreads>
__device__ __forceinline__ void quantize_token(
    const T *__restrict__ x, int64_t K, int64_t ldx, int8_t *__restrict__ qnat, int64_t ldq,
    double *__restrict__ scale, int C, uint8_t *__restrict__ rec, int32_t *nonfinite, int m,
    int rank, int ncta) {
  using F = Fmt<FMT>;
  const int cb = (int)((int64_t)C * rank / ncta), ce = (int)((int64_t)C * (rank + 1) / ncta);
  const T *row = x + m * ldx;
  const int lane = threadIdx.x & 31;
  const int64_t kb = (int64_t)cb * F::kWeights;
  const int64_t ke = min((int64_t)ce * F::kWeights, K);
  double amax = 0.0;
  bool bad = false;
  for (int64_t k = kb + threadIdx.x; k < ke; k += kThreads) {
    const double v = static_cast<double>(row[k]);
    bad |= !isfinite(v);
    amax = fmax(amax, fabs(v));
  }
  __shared__ double red[kThreads / 32];
  __shared__ double s_part;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if (lane == 0) red[threadIdx.x >> 5] = amax;
  if (bad && nonfinite) atomicOr(nonfinite, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) a = fmax(a, red[i]);
    s_part = a;
  }
  // cluster-wide max: every CTA reads every CTA's partial through DSMEM
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  double a = 0.0;
  {
    const uint32_t local = smem_u32(&s_part);
    for (int r = 0; r < ncta; ++r) {
      uint32_t remote;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(r));
      double v;
      asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(remote));
      a = fmax(a, v);
    }
  }
  // keep every CTA's shared memory alive until all remote reads are done
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  const double s = a > 0.0 ? a / 127.0 : 1.0;
  const double inv_s = 1.0 / s;
  if (rank == 0 && threadIdx.x == 0) scale[m] = s;
  const int64_t n4 = (int64_t)(ce - cb) * 4;
  for (int64_t base = threadIdx.x - lane; base < n4; base += kThreads) {
    const int64_t idx = base + lane;
    const bool on = idx < n4;
    const int c = cb + (int)(idx >> 2), i = (int)(idx & 3);
    const int64_t k0 = (int64_t)c * F::kWeights + i * 4 * F::kGroup;
    uint32_t r[F::kGroup];
    int32_t gs = 0;
#pragma unroll
    for (int v = 0; v < F::kGroup; ++v) {
      uint32_t word = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int64_t k = k0 + 4 * v + b;
        int q = 0;
        if (on && k < K) q = quantize_one(static_cast<double>(row[k]), s, inv_s);
        if (on && qnat && k < ldq) qnat[m * ldq + k] = static_cast<int8_t>(q);
        gs += q;
        word |= (uint32_t)(q & 0xFF) << (8 * b);
      }
      r[v] = word;
    }
    write_group<FMT>(rec + ((int64_t)m * C + (on ? c : 0)) * F::kRecBytes, i, r, gs, on);
  }
  // natural padding beyond the record coverage (only when ldq > C * kWeights)
  if (qnat && rank == ncta - 1)
    for (int64_t k = (int64_t)C * F::kWeights + threadIdx.x; k < ldq; k += kThreads)
      qnat[m * ldq + k] = 0;
}

// Stand-alone launch form: grid (ncta, M), cluster (ncta, 1, 1).
template <int FMT, typename T, int kThreads>
__global__ void __launch_bounds__(kThreads) quantize_records_kernel(
    const T *__restrict__ x, int64_t K, int64_t ldx, int8_t *__restrict__ qnat, int64_t ldq,
    double *__restrict__ scale, int C, uint8_t *__restrict__ rec, int32_t *nonfinite) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // x may come from the previous kernel
  quantize_token<FMT, T, kThreads>(x, K, ldx, qnat, ldq, scale, C, rec, nonfinite, blockIdx.y,
                                   blockIdx.x, gridDim.x);
}

// ---------------------------------------------------------------------------
// decode GEMV
// ---------------------------------------------------------------------------
template <int FMT, int MT>
struct Acc {
  static constexpr int kSlots = Fmt<FMT>::kSlots;
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
    if constexpr (FMT == TB_I2S) {
      // slot s accumulated codes * 4^s (masks without shifts): exact divisions
      return v[m][0] + (v[m][1] >> 2) + (v[m][2] >> 4) + (v[m][3] >> 6) - csum[m];
    } else if constexpr (FMT == TB_TL1) {
      // n*x1 (lo) + a*x0 - 3*a*x1 (lo) + 16*n*x1 / 16 (hi) + a*x0 - 3*a*x1 (hi)
      return v[m][0] + v[m][1] - 3 * v[m][2] + (v[m][3] >> 4) + v[m][4] - 3 * v[m][5] - csum[m];
    } else {
      int32_t s = -csum[m];
#pragma unroll
      for (int k = 0; k < kSlots; ++k) s += v[m][k];
      return s;
    }
  }
};

// One 16-byte chunk of this lane's row against MT activation records.
template <int FMT, int MT>
__device__ __forceinline__ void process_chunk(const uint4 w4, const uint32_t sgn,
                                              const uint8_t *__restrict__ rec0, int M,
                                              Acc<FMT, MT> &acc) {
  using F = Fmt<FMT>;
  constexpr int kTokStride = kStageChunks * F::kRecBytes;  // record stride between tokens
#ifdef TB_NO_COMPUTE  // profiling variant: data movement only
  acc.v[0][0] += (int32_t)(w4.x ^ w4.w);
  return;
#endif
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
          const uint4 A = *reinterpret_cast<const uint4 *>(rec0 + m * kTokStride + 16 * i);
          acc.v[m][0] = dp4a_us(x0, A.x, acc.v[m][0]);
          acc.v[m][1] = dp4a_us(x1, A.y, acc.v[m][1]);
          acc.v[m][2] = dp4a_us(x2, A.z, acc.v[m][2]);
          acc.v[m][3] = dp4a_us(x3, A.w, acc.v[m][3]);
        }
      }
    } else if constexpr (FMT == TB_TL1) {
      // nibble n = 3a + b (packing.py:56-60), codes a = w0+1, b = w1+1:
      //   a*x0 + b*x1 = n*x1 + a*x0 - 3*a*x1,   a = n/3 = (11n) >> 5 for n <= 8.
      // The high nibbles are used in place (16n): the same umulhi trick with
      // a 16x smaller constant, and a 16x-scaled accumulator for n*x1.
      const uint32_t lo = W & 0x0F0F0F0Fu, hi16 = W & 0xF0F0F0F0u;
      const uint32_t alo = __umulhi(lo, 11u << 27) & 0x03030303u;
      const uint32_t ahi = __umulhi(hi16, 11u << 23) & 0x03030303u;
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        if (m < M) {
          const uint4 A = *reinterpret_cast<const uint4 *>(rec0 + m * kTokStride + 16 * i);
          acc.v[m][0] = dp4a_us(lo, A.y, acc.v[m][0]);
          acc.v[m][1] = dp4a_us(alo, A.x, acc.v[m][1]);
          acc.v[m][2] = dp4a_us(alo, A.y, acc.v[m][2]);
          acc.v[m][3] = dp4a_us(hi16, A.w, acc.v[m][3]);
          acc.v[m][4] = dp4a_us(ahi, A.z, acc.v[m][4]);
          acc.v[m][5] = dp4a_us(ahi, A.w, acc.v[m][5]);
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
      uint32_t code[6];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t x = h ? hi : lo;
        const uint32_t msk = h ? mhi : mlo;
        const uint32_t d = lop3_sel(x + 0x0D0D0D0Du, 0x0D0D0D0Du - x, msk);
        const uint32_t c0 = ((d * 7u + 0x07070707u) >> 6) & 0x03030303u;  // d / 9
        const uint32_t r = d - 9u * c0;                                      // d % 9
        const uint32_t c1 = __umulhi(r, 11u << 27) & 0x03030303u;           // r / 3
        code[3 * h + 0] = c0;
        code[3 * h + 1] = c1;
        code[3 * h + 2] = r - 3u * c1;  // r % 3
      }
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        if (m < M) {
          const uint2 *A = reinterpret_cast<const uint2 *>(rec0 + m * kTokStride + 24 * i);
          const uint2 a01 = A[0], a23 = A[1], a45 = A[2];
          const uint32_t a[6] = {a01.x, a01.y, a23.x, a23.y, a45.x, a45.y};
#pragma unroll
          for (int q = 0; q < 6; ++q) acc.v[m][q] = dp4a_us(code[q], a[q], acc.v[m][q]);
        }
      }
    }
  }
#pragma unroll
  for (int m = 0; m < MT; ++m)
    if (m < M) acc.csum[m] += *reinterpret_cast<const int32_t *>(rec0 + m * kTokStride + F::kActWords * 4);
}


}  // namespace tb
