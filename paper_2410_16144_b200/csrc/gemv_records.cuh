// Activation records + per-chunk decode/contract for the decode GEMV (see gemv.cu).
#pragma once
#include "common.cuh"

namespace tb {

#ifndef TB_STAGE_CHUNKS
#define TB_STAGE_CHUNKS 4
#endif
constexpr int kStageChunks = TB_STAGE_CHUNKS;  // chunks per ring stage (per warp)

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
//   word kActWords = sum of the chunk's activations (TL2: + the sum over the
//   triples' third members, see write_group)
// One thread per (token, chunk, group i); the 4 group threads are adjacent lanes.
// ---------------------------------------------------------------------------
// Distributed shared memory (thread-block clusters): the fused step's CTAs
// of one cluster quantise disjoint slices of the inputs and write every
// record into all ranks' tables.
__device__ __forceinline__ uint32_t mapa_rank(uint32_t saddr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// split barrier: every rank arrives at entry and waits before its first
// DSMEM store, so no CTA writes into a peer that has not started yet
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}

template <int FMT>
__device__ __forceinline__ void write_group(uint8_t *rec_chunk, int i, const uint32_t (&r)[Fmt<FMT>::kGroup],
                                            int32_t gsum, bool on, int Q = 1) {
  using F = Fmt<FMT>;
  uint32_t wv[FMT == TB_TL2 ? 6 : 1];
  if constexpr (FMT == TB_TL2) {
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      uint32_t word = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int b = 6 * j + s;
        word |= ((r[b >> 2] >> (8 * (b & 3))) & 0xFFu) << (8 * j);
      }
      wv[s] = word;
    }
    // The TL2 decode keeps a triple's third digit as c2 + 1 (it saves the
    // subtraction): the chunk "sum" the contraction subtracts is therefore
    // sum(a) + sum(a over the third members) -- words 2 and 5 of the group.
    gsum = __dp4a((int)wv[2], 0x01010101, gsum);
    gsum = __dp4a((int)wv[5], 0x01010101, gsum);
  }
  // chunk sum over the 4 adjacent group lanes (all 32 lanes shuffle)
  gsum += __shfl_xor_sync(0xffffffffu, gsum, 1);
  gsum += __shfl_xor_sync(0xffffffffu, gsum, 2);
  if (!on) return;
  uint32_t *dst = reinterpret_cast<uint32_t *>(rec_chunk) + i * F::kGroup;
  if constexpr (FMT == TB_TL2) {
    if (Q == 1) {
#pragma unroll
      for (int s = 0; s < 6; ++s) dst[s] = wv[s];
    } else {
      for (int p = 0; p < Q; ++p) {
        const uint32_t a = mapa_rank(smem_u32(dst), p);
#pragma unroll
        for (int s = 0; s < 6; ++s) st_cluster_u32(a + 4 * s, wv[s]);
      }
    }
  } else {  // 4x4 byte transpose
    const uint32_t t0 = prmt(r[0], r[1], 0x5140u), t1 = prmt(r[0], r[1], 0x7362u);
    const uint32_t t2 = prmt(r[2], r[3], 0x5140u), t3 = prmt(r[2], r[3], 0x7362u);
    uint4 o;
    o.x = prmt(t0, t2, 0x5410u);
    o.y = prmt(t0, t2, 0x7632u);
    o.z = prmt(t1, t3, 0x5410u);
    o.w = prmt(t1, t3, 0x7632u);
    if (Q == 1) {
      reinterpret_cast<uint4 *>(dst)[0] = o;
    } else {
      for (int p = 0; p < Q; ++p) st_cluster_v4(mapa_rank(smem_u32(dst), p), o);
    }
  }
  if (i == 0) {
    // the sum in all four tail words: readers of different tokens pick
    // different words (token records 320 B apart put every even token's
    // tail in the same bank; one word each would be a 4-way conflict)
    const int4 sv = make_int4(gsum, gsum, gsum, gsum);
    int4 *sp = reinterpret_cast<int4 *>(rec_chunk + F::kActWords * 4);
    if (Q == 1) {
      *sp = sv;
    } else {
      const uint32_t u = (uint32_t)gsum;
      for (int p = 0; p < Q; ++p) st_cluster_v4(mapa_rank(smem_u32(sp), p), make_uint4(u, u, u, u));
    }
  }
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
  const float inv_sf = static_cast<float>(inv_s);
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
        if (on && k < K) {
          if constexpr (sizeof(T) == 4) q = quantize_fast(row[k], inv_sf, s, inv_s);
          else q = quantize_one(static_cast<double>(row[k]), s, inv_s);
        }
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
// CTA-local quantisation (the fused decode step of gemv.cu): every CTA of the
// GEMV grid quantises the whole input vector itself -- absmax over K floats
// (L2-resident after the first CTA) and the records of every chunk into its
// own shared memory -- so no separate quantise launch and no grid-wide
// dependency precede the weight stream.  Results are identical in every CTA.
// ---------------------------------------------------------------------------
template <int kThreads>
__device__ __forceinline__ float cta_absmax_f32(const float *__restrict__ x, int K, bool &bad,
                                                float *red) {
  float amax = 0.f;
  bool nf = false;
  const int lane = threadIdx.x & 31;
  if ((reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    const int K4 = K >> 2;
    const float4 *x4 = reinterpret_cast<const float4 *>(x);
    for (int i = threadIdx.x; i < K4; i += kThreads) {
      const float4 v = __ldcg(x4 + i);
      nf |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
      amax = fmaxf(amax, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
    for (int k = (K4 << 2) + threadIdx.x; k < K; k += kThreads) {
      const float v = __ldcg(x + k);
      nf |= !isfinite(v);
      amax = fmaxf(amax, fabsf(v));
    }
  } else {
    for (int k = threadIdx.x; k < K; k += kThreads) {
      const float v = __ldcg(x + k);
      nf |= !isfinite(v);
      amax = fmaxf(amax, fabsf(v));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  nf = __syncthreads_or(nf);
  if (lane == 0) red[threadIdx.x >> 5] = amax;
  __syncthreads();
  float a = 0.f;
#pragma unroll
  for (int i = 0; i < kThreads / 32; ++i) a = fmaxf(a, red[i]);
  __syncthreads();  // red may be reused
  bad = nf;
  return a;  // |x| max in float32 is exact, as is its float64 widening
}

// Records of every chunk of one token into `rtab` ([C][kRecBytes], shared).
template <int FMT, int kThreads>
__device__ __forceinline__ void cta_build_records(const float *__restrict__ x, int K, int C,
                                                  double s, uint8_t *rtab) {
  using F = Fmt<FMT>;
  const int lane = threadIdx.x & 31;
  const double inv_s = 1.0 / s;
  const float inv_sf = static_cast<float>(inv_s);
  const int n4 = C * 4;
  const bool vec = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  for (int base = threadIdx.x - lane; base < n4; base += kThreads) {  // warp-uniform
    const int idx = base + lane;
    const bool on = idx < n4;
    const int c = on ? idx >> 2 : 0, i = idx & 3;
    const int k0 = c * F::kWeights + i * 4 * F::kGroup;
    uint32_t r[F::kGroup];
    int32_t gs = 0;
#pragma unroll
    for (int v = 0; v < F::kGroup; ++v) {
      const int kv = k0 + 4 * v;
      float xv[4];
      if (on && vec && kv + 3 < K) {
        const float4 t = __ldcg(reinterpret_cast<const float4 *>(x + kv));
        xv[0] = t.x, xv[1] = t.y, xv[2] = t.z, xv[3] = t.w;
      } else {
#pragma unroll
        for (int b = 0; b < 4; ++b) xv[b] = (on && kv + b < K) ? __ldcg(x + kv + b) : 0.f;
      }
      uint32_t word = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int q = quantize_fast(xv[b], inv_sf, s, inv_s);  // 0.f -> 0
        gs += q;
        word |= (uint32_t)(q & 0xFF) << (8 * b);
      }
      r[v] = word;
    }
    write_group<FMT>(rtab + c * F::kRecBytes, i, r, gs, on);
  }
}

// All inputs of a step at once, values held in registers: every thread loads
// its record groups (group g = 4 * chunk + i of the concatenated inputs,
// g = tid + r * kThreads) in ONE round of independent loads -- issued before
// the weight prefetch so they do not queue behind it -- then the per-input
// absmax is reduced through shared memory and the records are quantised from
// the registers.  fits() is false when the inputs exceed kMaxG groups per
// thread (the caller then uses the looped cta_absmax / cta_build_records).
template <int FMT, int kThreads, int kMaxG>
struct RegQuant {
  using F = Fmt<FMT>;
  float4 xr[kMaxG][F::kGroup];
  // Only the inputs this CTA's jobs contract are quantised (`need`, bit v):
  // they occupy compact slots 0.. in input order; vmap holds slot -> input.
  int gb1, gb2, gb3;  // first global group of slots 1..3 (INT_MAX past the last)
  int G;
  int lo, hi, per;  // this CTA's groups [lo, hi) of the G (cluster rank r of Q: per each)
  int vmap;
  const float *const *xs_;

  __device__ __forceinline__ int slot_of(int g) const { return (g >= gb1) + (g >= gb2) + (g >= gb3); }
  __device__ __forceinline__ int base_of(int c) const {
    return c == 0 ? 0 : (c == 1 ? gb1 : (c == 2 ? gb2 : gb3));
  }
  __device__ __forceinline__ int vid(int c) const { return (vmap >> (4 * c)) & 15; }
  // every rank of a cluster decides alike (per is rank-independent)
  __device__ __forceinline__ bool fits() const { return per <= kMaxG * kThreads; }

  __device__ __forceinline__ void load(const float *const *xs, const int *Ks, const int *Cs, int n,
                                       int need, int rank = 0, int Q = 1) {
    // Every parameter at a fixed offset, loaded up front: kernel parameters are
    // cold in the constant cache at each launch, so a chain of dependent
    // (indexed) constant loads costs one L2 round trip per link (measured
    // ~1.4 us before the first input load went out).
    const float *xv[4];
    int Kv[4], Cv[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      xv[v] = xs[v];
      Kv[v] = Ks[v];
      Cv[v] = Cs[v];
    }
    int acc = 0, gbv[4] = {0x7fffffff, 0x7fffffff, 0x7fffffff, 0x7fffffff}, ns = 0;
    vmap = 0;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      if (v < n && ((need >> v) & 1)) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c == ns) gbv[c] = acc;
        vmap |= v << (4 * ns);
        ++ns;
        acc += 4 * Cv[v];
      }
    }
    gb1 = gbv[1], gb2 = gbv[2], gb3 = gbv[3];
    G = acc;
    xs_ = xs;
    // whole chunks (4 groups) per rank: a chunk's sum is a 4-lane shuffle
    per = (((G + Q - 1) / Q) + 3) & ~3;
    lo = min(G, rank * per);
    hi = min(G, lo + per);
    if (!fits()) return;
#pragma unroll
    for (int r = 0; r < kMaxG; ++r) {
      const int g = lo + threadIdx.x + r * kThreads;
      const int c = g < hi ? slot_of(g) : 0;
      const int v = vid(c);
      const int local = g - base_of(c);
      const int k0 = (local >> 2) * F::kWeights + (local & 3) * 4 * F::kGroup;
      const float *x = xv[0];
      int K = Kv[0];
#pragma unroll
      for (int vv = 1; vv < 4; ++vv)
        if (v == vv) x = xv[vv], K = Kv[vv];
      const bool vec = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
#pragma unroll
      for (int u = 0; u < F::kGroup; ++u) {
        const int kv = k0 + 4 * u;
        float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
        if (g < hi) {
          if (vec && kv + 3 < K) {
            t = __ldcg(reinterpret_cast<const float4 *>(x + kv));
          } else {  // L2 loads: x may have been written by a copy engine (ready flags)
            if (kv < K) t.x = __ldcg(x + kv);
            if (kv + 1 < K) t.y = __ldcg(x + kv + 1);
            if (kv + 2 < K) t.z = __ldcg(x + kv + 2);
            if (kv + 3 < K) t.w = __ldcg(x + kv + 3);
          }
        }
        xr[r][u] = t;
      }
    }
  }

  float amx[4], invf[4];  // per-input absmax and 127 / absmax (after reduce)

  // Every thread of the CTA.  Writes s_scale[v] (thread v) and returns the
  // non-finite mask (bit v) in every thread.  The absmax is an integer max of
  // the |x| bit patterns: for finite floats it orders like the values, and
  // any Inf / NaN lands at or above 0x7F800000 (the non-finite verdict).
  // Q > 1: the CTA's partial maxima go to every rank's cl[rank][v] (DSMEM)
  // and the cluster barrier makes the full absmax visible everywhere.
  __device__ __forceinline__ int reduce(int n, double *s_scale,
                                        float *red /* [kThreads/32][4] */,
                                        uint32_t *cl /* [Q][4] */, int rank, int Q) {
    constexpr int kW = kThreads / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t am[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int r = 0; r < kMaxG; ++r) {
      const int g = lo + threadIdx.x + r * kThreads;
      const int v = g < hi ? vid(slot_of(g)) : 0;
      uint32_t m = 0u;
#pragma unroll
      for (int u = 0; u < F::kGroup; ++u) {
        const float4 t = xr[r][u];
        m = max(m, max(max(__float_as_uint(t.x) & 0x7FFFFFFFu, __float_as_uint(t.y) & 0x7FFFFFFFu),
                       max(__float_as_uint(t.z) & 0x7FFFFFFFu, __float_as_uint(t.w) & 0x7FFFFFFFu)));
      }
#pragma unroll
      for (int vv = 0; vv < 4; ++vv)
        if (vv == v) am[vv] = max(am[vv], m);
    }
    uint32_t *ured = reinterpret_cast<uint32_t *>(red);
#pragma unroll
    for (int vv = 0; vv < 4; ++vv) {
      const uint32_t w = __reduce_max_sync(0xffffffffu, am[vv]);
      if (lane == 0) ured[warp * 4 + vv] = w;
    }
    __syncthreads();
    if (Q > 1) {
      cluster_wait();  // pairs with the entry arrive: every peer is running
      if (threadIdx.x < 4) {
        uint32_t a = 0u;
#pragma unroll
        for (int w = 0; w < kW; ++w) a = max(a, ured[w * 4 + threadIdx.x]);
        const uint32_t dst = smem_u32(cl + rank * 4 + threadIdx.x);
        for (int p = 0; p < Q; ++p) st_cluster_u32(mapa_rank(dst, p), a);
      }
      cluster_sync();
    }
    int badmask = 0;
    // per-input absmax; the scale itself (float64, core.py:128-130) is only
    // needed by thread v (output) and on the rare near-tie path
#pragma unroll
    for (int vv = 0; vv < 4; ++vv) {
      uint32_t a = 0u;
      if (Q > 1) {
        for (int p = 0; p < Q; ++p) a = max(a, cl[p * 4 + vv]);
      } else {
#pragma unroll
        for (int w = 0; w < kW; ++w) a = max(a, ured[w * 4 + vv]);
      }
      if (a >= 0x7F800000u) badmask |= 1 << vv;
      amx[vv] = __uint_as_float(a);
      invf[vv] = a > 0u ? 127.0f / amx[vv] : 1.0f;  // within 2^-24 of 1/s: quantize_fast's bound
    }
#pragma unroll
    for (int vv = 0; vv < 4; ++vv)
      if (threadIdx.x == vv && vv < n)
        s_scale[vv] = amx[vv] > 0.f ? static_cast<double>(amx[vv]) / 127.0 : 1.0;
    return badmask;
  }

  // Records of this thread's groups from the registers (after reduce()).
  // q = x * (127 / amax) is rounded by ONE fma with 1.5 * 2^23 (its low
  // mantissa byte is rint(q) in two's complement, |q| <= 127); a second fma
  // gives the exact rounding residue, and elements within 4e-5 of a .5 tie
  // are redone in float64 (core.py:24-27, 128-130).
  // Q > 1: every record goes to the same offset in all Q ranks' tables.
  __device__ __forceinline__ void records(const int *offs, uint8_t *rtab, int Q = 1) {
    const int lane = threadIdx.x & 31;
    constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
#pragma unroll
    for (int r = 0; r < kMaxG; ++r) {
      const int gw = lo + (threadIdx.x - lane) + r * kThreads;  // warp-uniform
      if (gw < hi) {
        const int g = gw + lane;
        const bool on = g < hi;
        const int c = on ? slot_of(g) : 0;
        const int v = vid(c);
        const int local = on ? g - base_of(c) : 0;
        float inv = invf[0], am = amx[0];
#pragma unroll
        for (int vv = 1; vv < 4; ++vv)
          if (vv == v) inv = invf[vv], am = amx[vv];
        uint32_t words[F::kGroup];
        bool near = false;  // some element within 4e-5 of a rounding tie
#pragma unroll
        for (int u = 0; u < F::kGroup; ++u) {
          const float4 t = xr[r][u];
          const float e[4] = {t.x, t.y, t.z, t.w};
          uint32_t tb[4];
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const float m = __fmaf_rn(e[b], inv, kMagic);
            const float d = __fmaf_rn(e[b], inv, kMagic - m);  // q - rint(q)
            near |= !(fabsf(d) < 0.49996f);
            tb[b] = __float_as_uint(m);
          }
          words[u] = prmt(prmt(tb[0], tb[1], 0x0040u), prmt(tb[2], tb[3], 0x0040u), 0x5410u);
        }
        uint32_t tie = 0;  // bit 4u+b: element within 4e-5 of a rounding tie
        if (near) {
#pragma unroll
          for (int u = 0; u < F::kGroup; ++u) {
            const float4 t = xr[r][u];
            const float e[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              const float m = __fmaf_rn(e[b], inv, kMagic);
              if (!(fabsf(__fmaf_rn(e[b], inv, kMagic - m)) < 0.49996f)) tie |= 1u << (4 * u + b);
            }
          }
        }
        if (tie) {  // rare: redo the flagged elements in float64 (exact at ties)
          const double s = am > 0.f ? static_cast<double>(am) / 127.0 : 1.0;
          const double inv_s = 1.0 / s;
          const int k0 = (local >> 2) * F::kWeights + (local & 3) * 4 * F::kGroup;
#pragma unroll 1
          while (tie) {
            const int bit = __ffs(tie) - 1;
            tie &= tie - 1;
            const float xv = xs_[v][k0 + bit];  // the element itself (cached)
            const uint32_t qb = (uint32_t)quantize_one(static_cast<double>(xv), s, inv_s) & 0xFFu;
            const int sh = 8 * (bit & 3);
#pragma unroll
            for (int u = 0; u < F::kGroup; ++u)
              if (u == (bit >> 2)) words[u] = (words[u] & ~(0xFFu << sh)) | (qb << sh);
          }
        }
        int32_t gs = 0;
#pragma unroll
        for (int u = 0; u < F::kGroup; ++u) gs = __dp4a((int)words[u], 0x01010101, gs);
        write_group<FMT>(rtab + offs[v] + (local >> 2) * F::kRecBytes, local & 3, words, gs, on, Q);
      }
    }
  }
};

// ---------------------------------------------------------------------------
// decode GEMV
// ---------------------------------------------------------------------------
// TL1 runs as I2_S: its tiles hold the same 2-bit codes (pack.cu repack).
#ifndef TB_I2S_DP4A
#ifndef TB_MMA_M1
#define TB_MMA_M1 0
#endif
template <int MT>
constexpr bool kI2sMma = MT >= 2 || TB_MMA_M1;  // M = 1 stays on dp4a (measured faster there)
#else
template <int MT>
constexpr bool kI2sMma = false;
#endif
#ifndef TB_TL2_LIN
#define TB_TL2_LIN 1  // one-token TL2: third digit by linearity (see process_chunk)
#endif
constexpr bool kTl2Lin = TB_TL2_LIN != 0;
template <int FMT, int MT, bool kMma = (FMT == TB_I2S && kI2sMma<MT>)>
struct Acc {
  static_assert(FMT != TB_TL1, "TL1 tiles are decoded by the I2_S path");
#ifndef TB_DP4A_SPLIT
#define TB_DP4A_SPLIT 1
#endif
  // M = 1 I2_S: two accumulator sets (even / odd words) halve the dp4a chains
  static constexpr int kSets = (FMT == TB_I2S && MT == 1) ? 1 + TB_DP4A_SPLIT : 1;
  static constexpr int kSlots = Fmt<FMT>::kSlots * kSets;
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
      int32_t r = -csum[m];
#pragma unroll
      for (int q = 0; q < kSets; ++q)
        r += v[m][4 * q] + (v[m][4 * q + 1] >> 2) + (v[m][4 * q + 2] >> 4) + (v[m][4 * q + 3] >> 6);
      return r;
    } else {
      if constexpr (MT == 1 && kTl2Lin)  // process_chunk's one-token TL2 slots
        return v[m][0] + v[m][3] + ((v[m][1] + v[m][4]) >> 5) + v[m][2] - 3 * (v[m][5] >> 5) - csum[m];
      int32_t s = -csum[m];
#pragma unroll
      for (int k = 0; k < kSlots; ++k) s += v[m][k];
      return s;
    }
  }
};

// ---------------------------------------------------------------------------
// I2_S / TL1 on the legacy int8 tensor-core path (mma.sync m16n8k32 u8 x s8).
// The warp's 32-row x 16-byte weight chunk is read with ldmatrix.x4, so lane
// (g = lane/4, t = lane%4) holds word t of rows g, g+8, g+16, g+24; each
// masked code plane of a word is a 4-byte K-slice of the MMA's A fragment.
//  - M <= 2 ("plane columns"): planes are masked without shifts (codes x 4^s,
//    u8) and every plane gets its own D column: P0 = planes 0|1 -> columns 0|1,
//    P1 = planes 2|3 -> columns 2|3 (token 1: columns 4..7).  B lane g holds
//    activation word 4t + (g&3) of token g>>2 (b0 for even g, b1 for odd), so
//    one LDS per lane feeds both MMAs; the cross terms land in columns that
//    are never read.  4 MMAs per chunk, 16 LOPs.
//  - M >= 4 ("token columns"): planes are shifted down to codes 0..2 and
//    column n = token n of an 8-token block: 4 MMAs per chunk and 8 tokens.
// The per-row result is Sum codes*a - Sum a, exact in int32 like the dp4a
// path (4^s scaling divided out exactly at the end).  A dp4a issue slot holds
// 128 weight MACs, an IMMA 512 (plane columns) -- the decode loop was
// issue-bound.
// ---------------------------------------------------------------------------
#ifndef TB_I2S_DP4A
#define TB_I2S_MMA 1
template <int MT>
struct Acc<TB_I2S, MT, true> {
  static constexpr bool kPlaneCols = MT <= 2;
  // P0/P1 (twice for M = 1: even / odd chunks, shorter MMA chains) or 8-token blocks
  static constexpr int kSets = kPlaneCols ? (MT == 1 ? 4 : 2) : (MT + 7) / 8;
  // Token columns, one 8-token block (M = 3..8): the planes stay UNSHIFTED
  // (codes x 4^s, one LOP per A register instead of a shift and a mask) and
  // every plane accumulates in its own fragment, folded exactly at the end;
  // an MMA then contracts plane s of TWO consecutive chunks (its two K
  // halves), so it is still 4 MMAs per chunk but 16 ALU ops instead of 28
  // (ncu had the ALU pipe at 71 % with the GEMV at 0.7 of HBM).
  // Off by default: bit-exact, but 115 registers instead of 79 (no room for a
  // glue CTA beside two table CTAs) and no faster -- the chains are latency
  // bound, not ALU-throughput bound (cfg4 M = 8 layer 75.2 vs 73.8 us).
#ifndef TB_MMA_UNSHIFT
#define TB_MMA_UNSHIFT 0
#endif
  static constexpr bool kUnshift = TB_MMA_UNSHIFT && !kPlaneCols && kSets == 1;
  static constexpr int kFrags = kUnshift ? 4 : kSets;
  int32_t d[2][kFrags][4];  // [row half h][set, or plane when kUnshift][fragment reg]
  __device__ __forceinline__ int32_t val(int h, int nb, int r) const {
    if constexpr (kUnshift)
      return d[h][0][r] + (d[h][1][r] >> 2) + (d[h][2][r] >> 4) + (d[h][3][r] >> 6);
    else
      return d[h][nb][r];
  }
  // Activation sums of this lane's own fragment columns only (plane columns:
  // token t/2; token columns: tokens 8nb + 2t, 8nb + 2t + 1); total() fetches
  // a token's sum from the lane that holds it.
  static constexpr int kCs = kPlaneCols ? 1 : 2 * kSets;
  int32_t csum[kCs];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int q = 0; q < kFrags; ++q)
#pragma unroll
        for (int r = 0; r < 4; ++r) d[h][q][r] = 0;
#pragma unroll
    for (int m = 0; m < kCs; ++m) csum[m] = 0;
  }
  // Row (lane) total of token m; every lane of the warp must call it.
  __device__ __forceinline__ int32_t total(int m) const {
    const int lane = threadIdx.x & 31;
    int32_t R[4];  // this lane's rows g, g+8, g+16, g+24 (of its fragment column pair)
    int src;
    int32_t cs;  // token m's activation sum, valid in lane src
    if constexpr (kPlaneCols) {
      cs = csum[0];
      const bool odd = lane & 1;  // t odd: planes 2|3 of set P1, else planes 0|1 of P0
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int32_t e[4], o[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          e[r] = d[h][0][r] + (kSets == 4 ? d[h][2][r] : 0);
          o[r] = d[h][1][r] + (kSets == 4 ? d[h][3][r] : 0);
        }
        const int32_t lo = odd ? (o[0] >> 4) + (o[1] >> 6) : e[0] + (e[1] >> 2);
        const int32_t hi = odd ? (o[2] >> 4) + (o[3] >> 6) : e[2] + (e[3] >> 2);
        R[2 * h] = lo + __shfl_xor_sync(0xffffffffu, lo, 1);
        R[2 * h + 1] = hi + __shfl_xor_sync(0xffffffffu, hi, 1);
      }
      src = 4 * (lane & 7) + 2 * m;  // lane t = 2m holds token m
    } else {
      const int nb = m >> 3, c = m & 7, which = c & 1;
      cs = csum[0];
#pragma unroll
      for (int q = 1; q < kCs; ++q)
        if (q == 2 * nb + which) cs = csum[q];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        R[2 * h] = which ? val(h, nb, 1) : val(h, nb, 0);
        R[2 * h + 1] = which ? val(h, nb, 3) : val(h, nb, 2);
      }
      src = 4 * (lane & 7) + (c >> 1);
    }
    // lane L wants row L: rows g + 8q live in R[q] of lane 4*(L%8) + t
    int32_t out = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int32_t v = __shfl_sync(0xffffffffu, R[q], src);
      if ((lane >> 3) == q) out = v;
    }
    return out - __shfl_sync(0xffffffffu, cs, src);
  }
  // Publish every token's row sums of this tile straight from the fragment
  // layout (REDs into ws[token][row0 + row]): token columns need no shuffles
  // at all, plane columns one (the plane pairs of a row sit in lanes t, t^1).
  __device__ __forceinline__ void red_all(int32_t *ws, int npad, int row0, int M) const {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    if constexpr (kPlaneCols) {
      const bool odd = lane & 1;
      const int tok = t >> 1;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int32_t e[4], o[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          e[r] = d[h][0][r] + (kSets == 4 ? d[h][2][r] : 0);
          o[r] = d[h][1][r] + (kSets == 4 ? d[h][3][r] : 0);
        }
        int32_t lo = odd ? (o[0] >> 4) + (o[1] >> 6) : e[0] + (e[1] >> 2);
        int32_t hi = odd ? (o[2] >> 4) + (o[3] >> 6) : e[2] + (e[3] >> 2);
        lo += __shfl_xor_sync(0xffffffffu, lo, 1);
        hi += __shfl_xor_sync(0xffffffffu, hi, 1);
        if (!odd && (tok == 0 || tok < M)) {
          int32_t *w = ws + (int64_t)tok * npad + row0 + g + 16 * h;
          red_add_s32(w, lo - csum[0]);
          red_add_s32(w + 8, hi - csum[0]);
        }
      }
    } else {
#pragma unroll
      for (int nb = 0; nb < kSets; ++nb)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int tok = 8 * nb + 2 * t + (r & 1);
            if (tok < M)
              red_add_s32(ws + (int64_t)tok * npad + row0 + g + 8 * (r >> 1) + 16 * h,
                          val(h, nb, r) - csum[2 * nb + (r & 1)]);
          }
    }
  }
};

__device__ __forceinline__ uint4 ldsm_x4(const void *p) {
  uint4 r;
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(smem_u32(p)));
  return r;
}

__device__ __forceinline__ void imma_u8s8(int32_t (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                          uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
#endif

// The warp's view of one 32-row x 16-byte chunk in shared memory: lane = row
// (dp4a paths), or the ldmatrix fragment of the tensor-core I2_S path.
template <int FMT, int MT>
__device__ __forceinline__ uint4 load_wchunk(const uint8_t *chunk, int lane) {
#ifdef TB_I2S_MMA
  if constexpr (FMT == TB_I2S && kI2sMma<MT>) return ldsm_x4(chunk + lane * 16);
#endif
  return *reinterpret_cast<const uint4 *>(chunk + lane * 16);
}

// Whether the fast path contracts chunks in pairs (process_chunk_pair).
#ifdef TB_I2S_MMA
template <int FMT, int MT>
constexpr bool kPairChunks = FMT == TB_I2S && kI2sMma<MT> && Acc<TB_I2S, MT, true>::kUnshift;
#else
template <int FMT, int MT>
constexpr bool kPairChunks = false;
#endif

#ifdef TB_I2S_MMA
// Two consecutive chunks (same row tile) on the unshifted-plane token-column
// path: MMA s contracts plane s of chunk A (K half 0) and chunk B (K half 1);
// the records' word s of lane t holds exactly that plane's 4 activations.
template <int MT, bool kNoCsum = false>
__device__ __forceinline__ void process_chunk_pair(const uint4 wa, const uint4 wb,
                                                   const uint8_t *__restrict__ recA,
                                                   const uint8_t *__restrict__ recB, int M,
                                                   Acc<TB_I2S, MT> &acc) {
  using F = Fmt<TB_I2S>;
  constexpr int kTokStride = kStageChunks * F::kRecBytes;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#ifdef TB_NO_COMPUTE
  acc.csum[0] += (int32_t)(wa.x ^ wb.w);
  return;
#endif
  uint4 ba = make_uint4(0u, 0u, 0u, 0u), bb = ba;
  if (g < M) {
    ba = *reinterpret_cast<const uint4 *>(recA + g * kTokStride + 16 * t);
    bb = *reinterpret_cast<const uint4 *>(recB + g * kTokStride + 16 * t);
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t ra = h ? wa.z : wa.x, rb = h ? wa.w : wa.y;
    const uint32_t rc = h ? wb.z : wb.x, rd = h ? wb.w : wb.y;
    imma_u8s8(acc.d[h][0], ra & 0x03030303u, rb & 0x03030303u, rc & 0x03030303u,
              rd & 0x03030303u, ba.x, bb.x);
    imma_u8s8(acc.d[h][1], ra & 0x0C0C0C0Cu, rb & 0x0C0C0C0Cu, rc & 0x0C0C0C0Cu,
              rd & 0x0C0C0C0Cu, ba.y, bb.y);
    imma_u8s8(acc.d[h][2], ra & 0x30303030u, rb & 0x30303030u, rc & 0x30303030u,
              rd & 0x30303030u, ba.z, bb.z);
    imma_u8s8(acc.d[h][3], ra & 0xC0C0C0C0u, rb & 0xC0C0C0C0u, rc & 0xC0C0C0C0u,
              rd & 0xC0C0C0C0u, ba.w, bb.w);
  }
  // the two chunks' activation sums of this lane's token columns (2t, 2t + 1)
  if constexpr (!kNoCsum)
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int tok = 2 * t + q;
    if (tok < M)
      acc.csum[q] += *reinterpret_cast<const int32_t *>(recA + tok * kTokStride +
                                                       (F::kActWords + ((tok >> 1) & 3)) * 4) +
                     *reinterpret_cast<const int32_t *>(recB + tok * kTokStride +
                                                       (F::kActWords + ((tok >> 1) & 3)) * 4);
  }
}
#endif

// One 16-byte chunk of this lane's row against MT activation records.
// kNoCsum: the caller takes the activation sums from a prefix table instead
// (records-table mode: set_csum_from_prefix at the flush).
template <int FMT, int MT, bool kNoCsum = false>
__device__ __forceinline__ void process_chunk(const uint4 w4, const uint32_t sgn,
                                              const uint8_t *__restrict__ rec0, int M,
                                              Acc<FMT, MT> &acc, int par = 0) {
  using F = Fmt<FMT>;
  constexpr int kTokStride = kStageChunks * F::kRecBytes;  // record stride between tokens
#ifdef TB_NO_COMPUTE  // profiling variant: data movement only
  acc.csum[0] += (int32_t)(w4.x ^ w4.w);
  return;
#endif
#ifdef TB_I2S_MMA
  if constexpr (FMT == TB_I2S && kI2sMma<MT>) {
    using A = Acc<TB_I2S, MT>;
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    if constexpr (A::kPlaneCols) {
      const int tok = g >> 2;
      uint32_t v = 0;
      if (tok == 0 || tok < M)
        v = *reinterpret_cast<const uint32_t *>(rec0 + tok * kTokStride + 4 * (4 * t + (g & 3)));
      const uint32_t b0 = (g & 1) ? 0u : v, b1 = (g & 1) ? v : 0u;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t ra = h ? w4.z : w4.x, rb = h ? w4.w : w4.y;
        const int q = A::kSets == 4 ? 2 * (par & 1) : 0;
        imma_u8s8(acc.d[h][q], ra & 0x03030303u, rb & 0x03030303u, ra & 0x0C0C0C0Cu,
                  rb & 0x0C0C0C0Cu, b0, b1);
        imma_u8s8(acc.d[h][q + 1], ra & 0x30303030u, rb & 0x30303030u, ra & 0xC0C0C0C0u,
                  rb & 0xC0C0C0C0u, b0, b1);
      }
    } else if constexpr (A::kUnshift) {
      // a lone chunk (tile ends, odd stage tails): the second K half is empty
      const uint4 bq = g < M ? *reinterpret_cast<const uint4 *>(rec0 + g * kTokStride + 16 * t)
                             : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t ra = h ? w4.z : w4.x, rb = h ? w4.w : w4.y;
        imma_u8s8(acc.d[h][0], ra & 0x03030303u, rb & 0x03030303u, 0u, 0u, bq.x, 0u);
        imma_u8s8(acc.d[h][1], ra & 0x0C0C0C0Cu, rb & 0x0C0C0C0Cu, 0u, 0u, bq.y, 0u);
        imma_u8s8(acc.d[h][2], ra & 0x30303030u, rb & 0x30303030u, 0u, 0u, bq.z, 0u);
        imma_u8s8(acc.d[h][3], ra & 0xC0C0C0C0u, rb & 0xC0C0C0C0u, 0u, 0u, bq.w, 0u);
      }
    } else {
      uint4 bq[A::kSets];
#pragma unroll
      for (int nb = 0; nb < A::kSets; ++nb) {
        const int tok = 8 * nb + g;
        bq[nb] = tok < M ? *reinterpret_cast<const uint4 *>(rec0 + tok * kTokStride + 16 * t)
                         : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t ra = h ? w4.z : w4.x, rb = h ? w4.w : w4.y;
        const uint32_t a0 = ra & 0x03030303u, b0c = rb & 0x03030303u;
        const uint32_t a1 = (ra >> 2) & 0x03030303u, b1c = (rb >> 2) & 0x03030303u;
        const uint32_t a2 = (ra >> 4) & 0x03030303u, b2c = (rb >> 4) & 0x03030303u;
        const uint32_t a3 = (ra >> 6) & 0x03030303u, b3c = (rb >> 6) & 0x03030303u;
#pragma unroll
        for (int nb = 0; nb < A::kSets; ++nb) {
          imma_u8s8(acc.d[h][nb], a0, b0c, a1, b1c, bq[nb].x, bq[nb].y);
          imma_u8s8(acc.d[h][nb], a2, b2c, a3, b3c, bq[nb].z, bq[nb].w);
        }
      }
    }
    if constexpr (kNoCsum) {
    } else if constexpr (A::kPlaneCols) {
      const int tok = t >> 1;
      if (tok == 0 || tok < M)
        acc.csum[0] += *reinterpret_cast<const int32_t *>(rec0 + tok * kTokStride + F::kActWords * 4);
    } else {
#pragma unroll
      for (int q = 0; q < A::kCs; ++q) {
        const int tok = 8 * (q >> 1) + 2 * t + (q & 1);
        if (tok < M)
          acc.csum[q] += *reinterpret_cast<const int32_t *>(rec0 + tok * kTokStride +
                                                          (F::kActWords + ((tok >> 1) & 3)) * 4);
      }
    }
    return;
  }
#endif
  const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
  uint4 tq[3];  // TL2, one token: activation words of the current word pair
  (void)tq;
  uint32_t tv[8];  // TL2: the eight groups' byte-lane values (common.cuh tl2_tile_groups)
  (void)tv;
  if constexpr (FMT == TB_TL2) tl2_tile_groups(w4.x, w4.y, w4.z, w4.w, sgn, tv);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t W = w[i];
    (void)W;
    if constexpr (FMT == TB_I2S) {
#ifdef TB_I2S_MMA
      if constexpr (!kI2sMma<MT>) {
#endif
      // byte b of (W & (3 << 2s)) = code of weight 16i + 4b + s, times 4^s
      const uint32_t x0 = W & 0x03030303u, x1 = W & 0x0C0C0C0Cu;
      const uint32_t x2 = W & 0x30303030u, x3 = W & 0xC0C0C0C0u;
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        if (m == 0 || m < M) {  // token 0 always exists: no branch for MT == 1
          const uint4 A = *reinterpret_cast<const uint4 *>(rec0 + m * kTokStride + 16 * i);
          constexpr int kS = Acc<FMT, MT>::kSets;
          const int o = kS > 1 ? 4 * (i % kS) : 0;
          acc.v[m][o + 0] = dp4a_us(x0, A.x, acc.v[m][o + 0]);
          acc.v[m][o + 1] = dp4a_us(x1, A.y, acc.v[m][o + 1]);
          acc.v[m][o + 2] = dp4a_us(x2, A.z, acc.v[m][o + 2]);
          acc.v[m][o + 3] = dp4a_us(x3, A.w, acc.v[m][o + 3]);
        }
      }
#ifdef TB_I2S_MMA
      }
#endif
    } else {
      // TL2 (packing.py:63-74): the tiled layout holds v = 13 + signed index =
      // the base-3 number 9 c0 + 3 c1 + c2 of the triple's codes (c = w + 1),
      // its bits placed for byte-lane extraction (common.cuh tl2_tile_groups).
      // Groups 2i (low nibbles of reference word i) and 2i + 1 (high nibbles):
      const uint32_t vlo = tv[2 * i], vhi = tv[2 * i + 1];
      if constexpr (MT == 1 && kTl2Lin) {
        // One token: the second digit stays unshifted (c1s = 32 c1, one mask)
        // and the third is never formed: with r = 3 c1 + (c2 + 1),
        //   sum (c2 + 1) a2 = sum r a2 - 3 sum c1 a2,
        // so the group costs a fourth dp4a (c1s against the a2 word) instead of
        // a shift and a multiply-subtract: 10 instructions per four triples
        // instead of 11, the FMA pipe's share unchanged.  Slots: 0/3 c0 a0
        // (low / high nibble groups), 1/4 c1s a1, 2 r a2, 5 c1s a2;
        // Acc::total folds them exactly (c1s sums are multiples of 32).
        if ((i & 1) == 0) {
          const uint4 *Q = reinterpret_cast<const uint4 *>(rec0 + 24 * i);
          tq[0] = Q[0];
          tq[1] = Q[1];
          tq[2] = Q[2];
        }
        const uint32_t a[6] = {(i & 1) ? tq[1].z : tq[0].x, (i & 1) ? tq[1].w : tq[0].y,
                               (i & 1) ? tq[2].x : tq[0].z, (i & 1) ? tq[2].y : tq[0].w,
                               (i & 1) ? tq[2].z : tq[1].x, (i & 1) ? tq[2].w : tq[1].y};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t d = h ? vhi : vlo;
          const uint32_t c0 = ((d * 7u) >> 6) & 0x03030303u;
          const uint32_t r = d - 9u * c0;
          const uint32_t c1s = (r * 10u) & 0x60606060u;
          acc.v[0][3 * h] = dp4a_us(c0, a[3 * h], acc.v[0][3 * h]);
          acc.v[0][3 * h + 1] = dp4a_us(c1s, a[3 * h + 1], acc.v[0][3 * h + 1]);
          acc.v[0][2] = dp4a_us(r, a[3 * h + 2], acc.v[0][2]);
          acc.v[0][5] = dp4a_us(c1s, a[3 * h + 2], acc.v[0][5]);
        }
        continue;
      }
      uint32_t code[6];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t d = h ? vhi : vlo;
        // d = v + 1 (the tile stores the biased value, so the divisions need no
        // bias add): (7 d) >> 6 = v / 9; r = v % 9 + 1;
        // (10 r) >> 5 = (v % 9) / 3; the third digit stays biased, c2 + 1 --
        // the records' chunk sums carry the matching term (write_group)
        // (multiply + shift, not multiply-high: IMAD.HI issues slower on B200 --
        // both divisions by mul.hi 16.4 us per cfg2 layer, both this way 15.6)
        const uint32_t c0 = ((d * 7u) >> 6) & 0x03030303u;
        const uint32_t r = d - 9u * c0;
        const uint32_t c1 = ((r * 10u) >> 5) & 0x03030303u;
        code[3 * h + 0] = c0;
        code[3 * h + 1] = c1;
        code[3 * h + 2] = r - 3u * c1;
      }
      if constexpr (MT == 1) {
        // one token: the 12 activation words of a word pair in three 16-byte loads
        if ((i & 1) == 0) {
          const uint4 *Q = reinterpret_cast<const uint4 *>(rec0 + 24 * i);
          tq[0] = Q[0];
          tq[1] = Q[1];
          tq[2] = Q[2];
        }
        const uint32_t a[6] = {(i & 1) ? tq[1].z : tq[0].x, (i & 1) ? tq[1].w : tq[0].y,
                               (i & 1) ? tq[2].x : tq[0].z, (i & 1) ? tq[2].y : tq[0].w,
                               (i & 1) ? tq[2].z : tq[1].x, (i & 1) ? tq[2].w : tq[1].y};
#pragma unroll
        for (int q = 0; q < 6; ++q) acc.v[0][q] = dp4a_us(code[q], a[q], acc.v[0][q]);
      } else {
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          if (m == 0 || m < M) {
            const uint2 *A = reinterpret_cast<const uint2 *>(rec0 + m * kTokStride + 24 * i);
            const uint2 a01 = A[0], a23 = A[1], a45 = A[2];
            const uint32_t a[6] = {a01.x, a01.y, a23.x, a23.y, a45.x, a45.y};
#pragma unroll
            for (int q = 0; q < 6; ++q) acc.v[m][q] = dp4a_us(code[q], a[q], acc.v[m][q]);
          }
        }
      }
    }
  }
  if constexpr (!kNoCsum)
#pragma unroll
  for (int m = 0; m < MT; ++m)
    if (m == 0 || m < M)
      acc.csum[m] += *reinterpret_cast<const int32_t *>(rec0 + m * kTokStride + F::kActWords * 4);
}

// Records-table mode: the activation sums of chunks [c0, c1) of the CTA's
// K-window for the tokens whose sums this lane's accumulator holds, from the
// per-token prefix table P[tok][c] (stride C + 1) built at the table fill --
// instead of one or two shared-memory loads and adds per chunk in the loop.
template <int FMT, int MT>
__device__ __forceinline__ void set_csum_from_prefix(Acc<FMT, MT> &acc, const int32_t *P,
                                                     int stride, int c0, int c1, int M) {
  const int t = threadIdx.x & 3;
#ifdef TB_I2S_MMA
  if constexpr (FMT == TB_I2S && kI2sMma<MT>) {
    using A = Acc<TB_I2S, MT>;
    if constexpr (A::kPlaneCols) {
      const int tok = t >> 1;
      acc.csum[0] = (tok == 0 || tok < M) ? P[tok * stride + c1] - P[tok * stride + c0] : 0;
    } else {
#pragma unroll
      for (int q = 0; q < A::kCs; ++q) {
        const int tok = 8 * (q >> 1) + 2 * t + (q & 1);
        acc.csum[q] = tok < M ? P[tok * stride + c1] - P[tok * stride + c0] : 0;
      }
    }
    return;
  }
#endif
#pragma unroll
  for (int m = 0; m < MT; ++m)
    acc.csum[m] = (m == 0 || m < M) ? P[m * stride + c1] - P[m * stride + c0] : 0;
}


}  // namespace tb
