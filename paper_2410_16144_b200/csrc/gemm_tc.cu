// Prefill ternary GEMM on the 5th-generation tensor cores (tcgen05.mma
// kind::i8, int32 accumulators in TMEM) -- BASELINE configs[3], M >= 128.
//
// The reference has no GEMM: a batch of M tokens is M independent calls of
// gemv_parallel (kernels.py:189-268), each token with its own absmax scale
// (core.py:116-134).  Here the M tokens' int8 codes form A [M][K] (K-major)
// and the packed ternary weights -- read from the same tiled layout the
// decode GEMV streams -- are unpacked to int8 {-1,0,1} into shared memory as
// B [N][K] (K-major); D[m][n] = sum_k A[m][k] * B[n][k] is exact in int32,
// so every accumulator equals the reference's for that token.
//
// Per CTA (persistent over (job, 128-row N tile) work items):
//   * all M <= 512 tokens stay on chip as up to 4 M=128 sub-tiles, each with
//     its own 128-column TMEM accumulator (512 columns), so a weight tile is
//     unpacked once and feeds 4 MMAs per K step;
//   * K advances 128 bytes per stage through a 2-stage shared-memory ring in
//     the UMMA canonical K-major SWIZZLE_128B layout (row r, 16-B chunk j at
//     r*128 + ((j ^ (r&7)) << 4), 1024-B aligned): A by cp.async (zero-filled
//     past M / lda), B unpacked in registers and stored swizzled;
//   * one thread issues tcgen05.mma (M=128, N=128, K=32) and tcgen05.commit
//     arrives on the stage's mbarrier, which the loaders wait on before
//     refilling that stage -- loads of stage k+1 overlap the MMAs of stage k;
//   * epilogue: tcgen05.ld 32x32b per warp (TMEM lanes 32*(warp%4)), then
//     acc * w_scale * a_scale[m] in float64 (core.py:99-101) to the outputs.
#include <algorithm>

#include "common.cuh"

namespace tb {

constexpr int kGemmBN = 128;      // weight rows per tile (MMA N)
constexpr int kGemmBK = 128;      // int8 K per stage = one 128-B swizzle atom
constexpr int kGemmSubM = 128;    // MMA M
constexpr int kGemmMaxMT = 4;     // M <= 512 tokens per launch
constexpr int kGemmThreads = 256;
constexpr int kGemmStages = 2;
constexpr int kGemmMaxJobs = 8;
constexpr int kSubTileBytes = kGemmSubM * kGemmBK;  // 16 KB
constexpr int kBTileBytes = kGemmBN * kGemmBK;      // 16 KB

struct GemmJob {
  const uint8_t *w;      // tiled layout (gemv.cu / tb_repack)
  const int8_t *act;     // [M][lda] int8, zero beyond cols
  const double *a_scale; // [M]
  double w_scale;
  int32_t *acc_out;      // [M][N] or null
  double *out64;         // [M][N] or null
  float *out32;          // [M][N] or null
  int N, C, lda;         // rows, 16-B chunks per row, activation row stride
  int tile0, ntiles;     // first work item, number of N tiles
};

struct GemmBatch {
  GemmJob jobs[kGemmMaxJobs];
  int njobs, total, M, MT;
};

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row groups 1024 B
// apart (SBO), LBO unused for swizzled K-major, version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) |
         ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// Instruction descriptor, kind::i8: D s32, A/B signed 8-bit, both K-major,
// N = 128 (>>3 at bit 17), M = 128 (>>4 at bit 24).
constexpr uint32_t kIdescI8 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kGemmBN >> 3) << 17) |
                              ((uint32_t)(kGemmSubM >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdescI8), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void cp_async16_zfill(uint32_t dst, const void *src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}

// 16 packed bytes of one row (64 weights) -> 64 int8 in {-1,0,1}, as four
// 16-byte words (word q = weights 16q..16q+15).
__device__ __forceinline__ uint32_t minus_one_bytes(uint32_t codes) {
  // per byte: code - 1 for codes in {0,1,2}, no borrow across bytes
  return ((codes | 0x80808080u) - 0x01010101u) ^ 0x80808080u;
}

template <int FMT>
__device__ __forceinline__ void unpack_chunk(const uint4 p, uint4 (&o)[4]) {
  const uint32_t w[4] = {p.x, p.y, p.z, p.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t r[4];
    if constexpr (FMT == TB_I2S) {
      // byte q of w[i]: weights 16i+4q+s at bits 2s (packing.py:200-206)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t t = (w[i] >> (8 * q)) & 0xFFu;
        const uint32_t u = t | (t << 6) | (t << 12) | (t << 18);  // bits 2s -> byte s
        r[q] = minus_one_bytes(u & 0x03030303u);
      }
    } else {
      // TL1 (packing.py:222-233): byte q = pairs (lo, hi) = weights 16i+4q..+3;
      // nibble n = 3a + b, a = w0 + 1, b = w1 + 1
      const uint32_t lo = w[i] & 0x0F0F0F0Fu, hi = (w[i] >> 4) & 0x0F0F0F0Fu;
      const uint32_t alo = __umulhi(lo, 11u << 27) & 0x03030303u;
      const uint32_t ahi = __umulhi(hi, 11u << 27) & 0x03030303u;
      const uint32_t blo = lo - 3u * alo, bhi = hi - 3u * ahi;
      // transpose: r[q] = (alo.q, blo.q, ahi.q, bhi.q)
      const uint32_t t0 = prmt(alo, blo, 0x5140u), t1 = prmt(alo, blo, 0x7362u);
      const uint32_t t2 = prmt(ahi, bhi, 0x5140u), t3 = prmt(ahi, bhi, 0x7362u);
      r[0] = minus_one_bytes(prmt(t0, t2, 0x5410u));
      r[1] = minus_one_bytes(prmt(t0, t2, 0x7632u));
      r[2] = minus_one_bytes(prmt(t1, t3, 0x5410u));
      r[3] = minus_one_bytes(prmt(t1, t3, 0x7632u));
    }
    o[i] = make_uint4(r[0], r[1], r[2], r[3]);
  }
}

template <int FMT>
__global__ void __launch_bounds__(kGemmThreads, 1) tgemm_kernel(const __grid_constant__ GemmBatch b) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t mbar[kGemmStages];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int MT = b.MT, M = b.M;
  const int stage_bytes = MT * kSubTileBytes + kBTileBytes;
  const uint32_t ncols = MT <= 1 ? 128u : (MT == 2 ? 256u : 512u);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_slot)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < kGemmStages; ++s) mbar_init(&mbar[s], 1);
    fence_mbar_init_cta();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  uint32_t g = 0;  // stages issued by this CTA (ring position and mbarrier phase)
  for (int item = blockIdx.x; item < b.total; item += gridDim.x) {
    int j = 0;
    while (j + 1 < b.njobs && b.jobs[j + 1].tile0 <= item) ++j;
    const GemmJob &J = b.jobs[j];
    const int n0 = (item - J.tile0) * kGemmBN;
    const int C = J.C;
    const int nk = (C + 1) / 2;  // 2 chunks (128 weights) per stage
    const int Npad = (J.N + kRowTile - 1) / kRowTile * kRowTile;

    for (int kb = 0; kb < nk; ++kb) {
      const int s = g & 1;
      const uint32_t use = g >> 1;
      if (use > 0) mbar_wait(&mbar[s], (use - 1) & 1);  // MMAs that read this stage are done
      uint8_t *sA = smem + s * stage_bytes;
      uint8_t *sB = sA + MT * kSubTileBytes;
      const uint32_t aA = smem_u32(sA);
      // A: MT*128 rows x 8 chunks of 16 B, zero-filled past M / lda
      const int na = MT * kGemmSubM * 8;
      for (int idx = tid; idx < na; idx += kGemmThreads) {
        const int r = idx >> 3, c16 = idx & 7;
        const int k = kb * kGemmBK + c16 * 16;
        const bool ok = r < M && k + 16 <= J.lda;
        const int8_t *src = ok ? J.act + (int64_t)r * J.lda + k : J.act;
        cp_async16_zfill(aA + (r >> 7) * kSubTileBytes + (r & 127) * 128 + ((c16 ^ (r & 7)) << 4),
                         src, ok);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      // B: 128 rows x 2 packed chunks -> int8, one (row, chunk) per thread
      {
        const int row = tid >> 1, cc = tid & 1;
        const int n = n0 + row, c = kb * 2 + cc;
        uint4 p = make_uint4(0, 0, 0, 0);
        const bool ok = n < Npad && c < C;
        if (ok)
          p = __ldg(reinterpret_cast<const uint4 *>(
              J.w + ((int64_t)(n >> 5) * C + c) * kTileChunkBytes + (n & 31) * 16));
        uint4 o[4];
        if (ok) {
          unpack_chunk<FMT>(p, o);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) o[q] = make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<uint4 *>(sB + row * 128 + (((cc * 4 + q) ^ (row & 7)) << 4)) = o[q];
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      // generic-proxy writes (st.shared, cp.async) -> visible to the tensor core
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        const uint32_t aB = smem_u32(sB);
        for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
          for (int k4 = 0; k4 < kGemmBK / 32; ++k4)
            mma_i8(tmem + mt * kGemmBN, umma_desc_sw128(aA + mt * kSubTileBytes + k4 * 32),
                   umma_desc_sw128(aB + k4 * 32), (kb > 0 || k4 > 0) ? 1u : 0u);
        }
        umma_commit(&mbar[s]);
      }
      ++g;
    }
    // epilogue: the last commit covers every MMA of this tile (issue order)
    mbar_wait(&mbar[(g - 1) & 1], ((g - 1) >> 1) & 1);
    tc_fence_after();
    {
      const int lg = warp & 3, ch = warp >> 2;  // TMEM lane group, column half
      for (int mt = 0; mt < MT; ++mt) {
        const int m = mt * kGemmSubM + lg * 32 + lane;
        const double as = m < M ? J.a_scale[m] : 0.0;
#pragma unroll 1
        for (int cb = 0; cb < 4; ++cb) {
          const int col = ch * 64 + cb * 16;
          uint32_t v[16];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
                "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
              : "r"(tmem + ((uint32_t)(lg * 32) << 16) + mt * kGemmBN + col));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (m < M) {
            const int nb = n0 + col;
            const int64_t o = (int64_t)m * J.N + nb;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              if (nb + e < J.N) {
                const int32_t a = (int32_t)v[e];
                if (J.acc_out) J.acc_out[o + e] = a;
                if (J.out64 || J.out32) {
                  const double y = static_cast<double>(a) * J.w_scale * as;  // core.py:99-101
                  if (J.out64) J.out64[o + e] = y;
                  if (J.out32) J.out32[o + e] = static_cast<float>(y);
                }
              }
            }
          }
        }
      }
    }
    tc_fence_before();
    __syncthreads();  // TMEM drained before the next tile's MMAs overwrite it
    tc_fence_after();
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
}

template <int FMT>
static int launch_gemm(GemmBatch &b, cudaStream_t s) {
  const int smem = kGemmStages * (b.MT * kSubTileBytes + kBTileBytes) + 1024;
  static int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    const int max_smem = kGemmStages * (kGemmMaxMT * kSubTileBytes + kBTileBytes) + 1024;
    if (cudaFuncSetAttribute(tgemm_kernel<FMT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             max_smem) != cudaSuccess)
      return TB_ERR_CUDA;
    configured_dev = dev;
  }
  const int grid = std::max(1, std::min(b.total, sm_count_cached()));
  tgemm_kernel<FMT><<<grid, kGemmThreads, smem, s>>>(b);
  TB_CHECK_LAUNCH();
  return TB_OK;
}

}  // namespace tb

using namespace tb;

extern "C" int tb_gemm_batch(int fmt, int64_t njobs, const tb_gemm_desc *descs, int64_t M,
                             void *stream) {
  if ((fmt != TB_I2S && fmt != TB_TL1) || njobs < 1 || njobs > kGemmMaxJobs || !descs || M < 1 ||
      M > kGemmMaxMT * kGemmSubM)
    return fmt == TB_TL2 ? TB_ERR_UNSUPPORTED : TB_ERR_ARGUMENT;
  GemmBatch b{};
  b.njobs = (int)njobs;
  b.M = (int)M;
  b.MT = (int)ceil_div(M, kGemmSubM);
  int tiles = 0;
  for (int64_t j = 0; j < njobs; ++j) {
    const tb_gemm_desc &d = descs[j];
    if (!d.tiled || !d.act || d.rows < 1 || d.cols < 1 || d.lda < 16 || (d.lda & 15) ||
        ((d.out64 || d.out32) && !d.a_scale) || (reinterpret_cast<uintptr_t>(d.act) & 15) ||
        (reinterpret_cast<uintptr_t>(d.tiled) & 15) || d.lda < d.cols)
      return TB_ERR_ARGUMENT;
    GemmJob &J = b.jobs[j];
    J.w = d.tiled;
    J.act = d.act;
    J.a_scale = d.a_scale;
    J.w_scale = d.w_scale;
    J.acc_out = d.acc_out;
    J.out64 = d.out64;
    J.out32 = d.out32;
    J.N = (int)d.rows;
    J.C = (int)ceil_div(ref_row_bytes(fmt, d.cols), kChunkBytes);
    J.lda = (int)d.lda;
    J.tile0 = tiles;
    J.ntiles = (int)ceil_div(d.rows, kGemmBN);
    tiles += J.ntiles;
  }
  b.total = tiles;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return fmt == TB_I2S ? launch_gemm<TB_I2S>(b, s) : launch_gemm<TB_TL1>(b, s);
}

extern "C" int tb_gemm_i8(int fmt, const uint8_t *tiled, int64_t rows, int64_t cols,
                          const int8_t *act, int64_t M, int64_t lda, const double *a_scale,
                          double w_scale, int32_t *acc_out, double *out64, float *out32,
                          void *stream) {
  if (M < 1) return TB_ERR_ARGUMENT;
  for (int64_t m0 = 0; m0 < M; m0 += kGemmMaxMT * kGemmSubM) {
    const int64_t mm = std::min<int64_t>(M - m0, kGemmMaxMT * kGemmSubM);
    tb_gemm_desc d{};
    d.tiled = tiled;
    d.rows = rows;
    d.cols = cols;
    d.act = act + m0 * lda;
    d.lda = lda;
    d.a_scale = a_scale ? a_scale + m0 : nullptr;
    d.w_scale = w_scale;
    d.acc_out = acc_out ? acc_out + m0 * rows : nullptr;
    d.out64 = out64 ? out64 + m0 * rows : nullptr;
    d.out32 = out32 ? out32 + m0 * rows : nullptr;
    const int st = tb_gemm_batch(fmt, 1, &d, mm, stream);
    if (st != TB_OK) return st;
  }
  return TB_OK;
}
