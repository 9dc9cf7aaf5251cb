// Prefill ternary GEMM on the 5th-generation tensor cores (tcgen05.mma
// kind::i8, int32 accumulators in TMEM) -- BASELINE configs[3], M >= 128.
//
// The reference has no GEMM: a batch of M tokens is M independent calls of
// gemv_parallel (kernels.py:189-268), each token with its own absmax scale
// (core.py:116-134).  Here the M tokens' int8 codes form A [M][K] and the
// packed ternary weights -- read from the same tiled layout the decode GEMV
// streams -- are unpacked to int8 {-1,0,1} in shared memory as B [N][K];
// D[m][n] = sum_k A[m][k] * B[n][k] is exact in int32, so every accumulator
// equals the reference's for that token.
//
// The weights enter the tensor core as unsigned codes c = w + 1 in {0,1,2}
// (kind::i8 with an unsigned B operand) and the epilogue subtracts the
// token's activation sum: sum_k a*w = sum_k a*c - sum_k a.  Codes come out of
// the packed bytes with shifts and masks only: for a 32-bit packed word, code
// plane s (I2_S: bits 2s of every byte; TL1: a/b digits of the low/high
// nibble) holds the weights 4q + s of byte q.  Both operands use that K order
// inside every 16-weight group (position 4s + q <-> weight 4q + s); for A the
// tiling kernel applies it, so the contraction is the same sum.
//
// Operand layout: UMMA K-major, no swizzle -- "core matrices" of 8 rows x 16
// bytes (128 contiguous bytes), K-adjacent core matrices 128 B apart (LBO),
// 8-row groups KC x 128 B apart (SBO; KC = 8 core matrices per 128-byte K
// stage).  A is pre-tiled in
// global memory into exactly this order (tb_gemm_tile_act: [k-stage][row
// group][k core][8 rows][16 B], plus the per-token sums), so one 1-D bulk
// copy moves a token sub-tile of a stage.
//
// Warp roles (384 threads, persistent over (job, 256-row N tile, 256-token
// half) items, K walked from a per-tile offset so CTAs spread over A):
//   warps 0, 2  producers: A by one bulk copy per stage, the packed weight
//               chunks of 256 rows by cp.async (arrive.noinc on the stage's
//               mbarrier), into an 8-deep ring;
//   warp 1      MMA issuer: one thread issues tcgen05.mma M=128 N=256 K=32 (4
//               per stage) and tcgen05.commit, accumulators in all 512 TMEM
//               columns;
//   warps 4-11  unpack one weight row each into one of 3 B slots, then run
//               the epilogue: tcgen05.ld 32x32b, transpose through shared
//               memory (the B slots), coalesced stores of
//               (acc - sum a) * w_scale * a_scale[m] in float64 (core.py:99-101).
#include <cuda.h>  // CUtensorMap (encoded through the runtime's driver entry point)
#include <cudaTypedefs.h>

#include <algorithm>
#include <utility>
#include <vector>

#include "common.cuh"

namespace tb {

constexpr int kGemmBN = 256;      // weight rows per tile (MMA N)
// 128-K stages (two packed 16-byte chunks per row): the per-stage pipeline
// cost (barrier round, TMA issue, unpack pass) was the limit at 64 K (~950
// cycles per stage against 512 cycles of MMA); 125 -> 100 us on the cfg3 layer
#ifndef TB_GEMM_BK
#define TB_GEMM_BK 128
#endif
constexpr int kGemmBK = TB_GEMM_BK;  // int8 K per stage: 64 = one packed 16-byte chunk per row, 128 = two
constexpr int kGemmKC = kGemmBK / 16;         // K core matrices per stage (per 8-row group)
constexpr int kChunksPerStage = kGemmBK / 64;  // packed 16-byte chunks per row per stage
constexpr int kGemmSubM = 128;    // MMA M
constexpr int kGemmMaxMT = 2;     // tokens per CTA tile: 256 (M x N = 64K int32 = all of TMEM)
constexpr int kGemmMaxM = 512;    // tokens per launch: up to two 256-token halves
constexpr int kGemmThreads = 384;  // 12 warps: producer, MMA, (2 idle), 8 unpack/epilogue
#ifndef TB_GEMM_STAGES
#define TB_GEMM_STAGES (kGemmBK >= 192 ? 2 : kGemmBK == 128 ? 4 : 8)
#endif
constexpr int kGemmStages = TB_GEMM_STAGES;  // load ring (A + packed weights)
#ifndef TB_GEMM_BSLOTS
#define TB_GEMM_BSLOTS (kGemmBK >= 128 ? 2 : 3)
#endif
constexpr int kGemmBSlots = TB_GEMM_BSLOTS;
constexpr int kGemmCluster = 2;  // CTA pair sharing every A stage (TMA multicast)   // unpacked-weight (B operand) slots; reused as epilogue staging
constexpr int kGemmMaxJobs = 8;
constexpr int kSubTileBytes = kGemmSubM * kGemmBK;    // 8 KB
constexpr int kBTileBytes = kGemmBN * kGemmBK;        // 16 KB
constexpr int kPackedBytes = kGemmBN * kChunkBytes * kChunksPerStage;  // 4 KB per 64 K
constexpr int kEpiBytes = 8 * 32 * 36 * 4;            // 8 epilogue warps x 32x32 int32 (in the B slots)
static_assert(kEpiBytes <= kGemmBSlots * kBTileBytes, "epilogue staging lives in the B slots");

struct alignas(64) GemmJob {
  CUtensorMap bmap;       // the tiled weights as [T][C][512 B] (3-D, 8-byte elements)
  const uint8_t *w;       // tiled weight layout (tb_repack)
  const uint8_t *act;     // pre-tiled activations (tb_gemm_tile_act)
  const double *a_scale;  // [M]
  double w_scale;
  int32_t *acc_out;       // [M][N] or null
  double *out64;          // [M][N] or null
  float *out32;           // [M][N] or null
  int N, C, Npad;         // rows, 16-B chunks per row, rows padded to 32
  int tile0, ntiles;      // first work item, number of N tiles
};

constexpr int kGemmMaxSched = 320;  // statically scheduled pair items per launch
constexpr int kGemmMaxPairs = 80;   // >= 148 SMs / 2

struct GemmBatch {
  GemmJob jobs[kGemmMaxJobs];
  int njobs, total, M, MT, MH, Mpad;  // MT sub-tiles per CTA, MH token halves
  int scheduled;                      // 1: pair p runs sched[sched_off[p] .. sched_off[p+1])
  uint16_t sched_off[kGemmMaxPairs + 1];
  uint16_t sched[kGemmMaxSched];
};

// UMMA shared-memory descriptor, K-major, SWIZZLE_NONE: LBO = 128 B between
// K-adjacent core matrices, SBO = 512 B between 8-row groups, version 1.
__device__ __forceinline__ uint64_t umma_desc_noswz(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)((kGemmKC * 128) >> 4) << 32) | ((uint64_t)1 << 46);
}

// Instruction descriptor, kind::i8: D s32, A signed 8-bit, B unsigned 8-bit
// (weight codes), both K-major, N = 256 (>>3 at bit 17), M = 128 (>>4 at bit 24).
constexpr uint32_t kIdescI8 = (2u << 4) | (1u << 7) | (0u << 10) | ((uint32_t)(kGemmBN >> 3) << 17) |
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

// One packed 32-bit word (16 weights) -> four code planes; byte q of plane s
// is the code (w + 1) of weight 4q + s (packing.py:200-206).  TL1 tiles hold
// the same 2-bit codes (the repack turns each pair index into two codes).
template <int FMT>
__device__ __forceinline__ uint4 code_planes(uint32_t W) {
  static_assert(FMT == TB_I2S, "TL1 tiles are I2_S-coded; TL2 has no GEMM path");
  return make_uint4(W & 0x03030303u, (W >> 2) & 0x03030303u, (W >> 4) & 0x03030303u,
                    (W >> 6) & 0x03030303u);
}

// Cursor over this CTA's (work item, K stage) stream: items blockIdx.x,
// blockIdx.x + gridDim.x, ...  Each item walks its K stages starting at a
// tile-dependent offset (kb = (k0 + i) mod C): the CTAs of one job then read
// different A stages at any moment instead of all hammering the same 32 KB
// in L2 (int32 sums are order-independent, so results are unchanged).
// A work item is (job, pair of N tiles, token half) for one CTA pair; this
// CTA takes tile 2 * pair + rank.
struct GemmCursor {
  int item, i, kb, k0, j, C, n0, h;
  int q;  // position in this pair's schedule (scheduled mode)
  __device__ __forceinline__ void start(const GemmBatch &b) {
    const int pair = blockIdx.x / kGemmCluster;
    if (b.scheduled) {
      q = b.sched_off[pair];
      set(b, q < b.sched_off[pair + 1] ? b.sched[q] : b.total);
    } else {
      set(b, pair);
    }
  }
  __device__ __forceinline__ void set(const GemmBatch &b, int it) {
    item = it;
    i = 0;
    if (it < b.total) {
      const int tt = it / b.MH;  // tile pair over all jobs; token half h
      h = it - tt * b.MH;
      int jj = 0;
      while (jj + 1 < b.njobs && b.jobs[jj + 1].tile0 <= tt) ++jj;
      j = jj;
      C = b.jobs[jj].C;
      const int t = tt - b.jobs[jj].tile0;
      n0 = (t * kGemmCluster + (int)(blockIdx.x % kGemmCluster)) * kGemmBN;
      k0 = (int)(((long long)(t * b.MH + h) * C * 29 / 97) % C);  // spread starts over K
      kb = k0;
    }
  }
  __device__ __forceinline__ bool last() const { return i + 1 == C; }
  __device__ __forceinline__ void next(const GemmBatch &b) {
    if (++i == C) {
      if (b.scheduled) {
        ++q;
        set(b, q < b.sched_off[blockIdx.x / kGemmCluster + 1] ? b.sched[q] : b.total);
      } else {
        set(b, item + gridDim.x / kGemmCluster);
      }
    } else if (++kb == C) {
      kb = 0;
    }
  }
};

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

#ifdef TB_GEMM_TRACE_EPI  // debug: per-tile epilogue stamps of CTA 0
__device__ long long g_epi_trace[16][3];
#endif
#ifdef TB_GEMM_TRACE  // debug: per-stage SM-clock stamps of CTA 0
constexpr int kTraceStages = 64;
__device__ long long g_gemm_trace[kTraceStages][6];
#define GT(p, i)                                                              \
  do {                                                                        \
    if (blockIdx.x == 0 && (p) < (uint32_t)kTraceStages) g_gemm_trace[p][i] = clock64(); \
  } while (0)
#else
#define GT(p, i) \
  do {           \
  } while (0)
#endif

template <int FMT>
__global__ void __launch_bounds__(kGemmThreads, 1) tgemm_kernel(const __grid_constant__ GemmBatch b) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[kGemmStages];   // A + packed weights landed
  __shared__ __align__(8) uint64_t empty[kGemmStages];  // MMAs done with the ring slot
  __shared__ __align__(8) uint64_t bready[kGemmBSlots]; // B unpacked (256 arrivals)
  __shared__ __align__(8) uint64_t bempty[kGemmBSlots]; // MMAs done with the B slot
  __shared__ __align__(8) uint64_t tfull, tempty;       // accumulator ready / drained
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int MT = b.MT, M = b.M;
  const int a_bytes = MT * kSubTileBytes;
  const int stage_bytes = a_bytes + kPackedBytes;  // ring slot, multiple of 1024
  uint8_t *bslots = smem + kGemmStages * stage_bytes;
  const uint32_t ncols = MT <= 1 ? 256u : 512u;  // MT x 256 accumulator columns

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_slot)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int s = 0; s < kGemmStages; ++s) {
      mbar_init(&full[s], 1);  // expect_tx (A halves from both CTAs + the weights)
      mbar_init(&empty[s], kGemmCluster);  // both CTAs' MMAs done with the slot
    }
    for (int s = 0; s < kGemmBSlots; ++s) {
      mbar_init(&bready[s], 8 * 32);
      mbar_init(&bempty[s], 1);
    }
    mbar_init(&tfull, 1);
    mbar_init(&tempty, 8 * 32);
    fence_mbar_init();  // release.cluster: the peer multicasts onto these barriers
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  // programmatic dependent of the activation quantiser (tb_gemm_quantize_act):
  // the TMEM allocation, barrier setup and cluster rendezvous above overlap
  // its tail; operands, scales and outputs are touched only after this wait
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const uint32_t tmem = tmem_slot;
  const uint32_t crank = blockIdx.x % kGemmCluster;

  if (warp == 0) {
    // ===== producer: per stage one multicast bulk copy of this CTA's half of
    // A (lands in both CTAs of the pair) and one 3-D tensor copy of the
    // stage's packed weights (8 row-tiles x 512 B, zero-filled past the end) =====
    if (lane == 0) {
      GemmCursor pc;
      pc.start(b);
      for (uint32_t p = 0; pc.item < b.total; ++p, pc.next(b)) {
        const int s = p % kGemmStages;
        if (p >= (uint32_t)kGemmStages) mbar_spin(&empty[s], (p / kGemmStages - 1) & 1);
        GT(p, 0);
        const GemmJob &J = b.jobs[pc.j];
        uint8_t *st = smem + s * stage_bytes;
#ifdef TB_GEMM_NO_A
        mbar_arrive_expect_tx(&full[s], kPackedBytes);
#else
        mbar_arrive_expect_tx(&full[s], a_bytes + kPackedBytes);
#endif
#ifdef TB_GEMM_NO_A  // profiling variant (results invalid): no activation loads
        if (false) {
        }
#elif defined(TB_GEMM_NO_MC)  // each CTA copies the whole A stage itself (no multicast)
        {
          const uint8_t *srcA = J.act + (size_t)pc.kb * (b.Mpad * kGemmBK) + (size_t)pc.h * a_bytes;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
              ::"r"(smem_u32(st)), "l"(srcA), "r"(a_bytes), "r"(smem_u32(&full[s]))
              : "memory");
        }
#else
        const uint32_t half = a_bytes / kGemmCluster;
        const uint8_t *src =
            J.act + (size_t)pc.kb * (b.Mpad * kGemmBK) + (size_t)pc.h * a_bytes + crank * half;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
            " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(st) + crank * half),
            "l"(src), "r"(half), "r"(smem_u32(&full[s])), "h"((uint16_t)((1u << kGemmCluster) - 1))
            : "memory");
#endif
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(st + a_bytes)),
            "l"(reinterpret_cast<uint64_t>(&J.bmap)), "r"(0), "r"(pc.kb * kChunksPerStage), "r"(pc.n0 >> 5),
            "r"(smem_u32(&full[s]))
            : "memory");
        GT(p, 1);
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer =====
    if (lane == 0) {
      GemmCursor cc;
      cc.start(b);
      uint32_t tiles = 0;
      for (uint32_t p = 0; cc.item < b.total; ++p) {
        const int s = p % kGemmStages, bs = p % kGemmBSlots;
        if (cc.i == 0 && tiles > 0) mbar_spin(&tempty, (tiles - 1) & 1);  // epilogue drained TMEM
        mbar_spin(&bready[bs], (p / kGemmBSlots) & 1);  // (implies full[s])
        GT(p, 4);
        tc_fence_after();
        const uint32_t aA = smem_u32(smem + s * stage_bytes), aB = smem_u32(bslots + bs * kBTileBytes);
#ifdef TB_GEMM_HALF_MMA  // profiling variant (results invalid): one token sub-tile's MMAs
        for (int mt = 0; mt < 1; ++mt) {
#else
        for (int mt = 0; mt < MT; ++mt) {
#endif
#pragma unroll
          for (int k2 = 0; k2 < kGemmBK / 32; ++k2)
#ifndef TB_GEMM_NO_MMA  // profiling variant: data movement only
            mma_i8(tmem + mt * kGemmBN, umma_desc_noswz(aA + mt * kSubTileBytes + k2 * 256),
                   umma_desc_noswz(aB + k2 * 256), (cc.i > 0 || k2 > 0) ? 1u : 0u);
#else
            ;
#endif
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
            " [%0], %1;" ::"r"(smem_u32(&empty[s])), "h"((uint16_t)((1u << kGemmCluster) - 1))
            : "memory");
        umma_commit(&bempty[bs]);
#ifndef TB_GEMM_TRACE_DEC
        GT(p, 5);
#endif
        if (cc.last()) {
          umma_commit(&tfull);
          ++tiles;
        }
        cc.next(b);
      }
    }
  } else if (warp >= 4) {
    // ===== unpack + epilogue (warps 4..11: row tid - 128; TMEM lane group
    // warp % 4, column half (warp - 4) / 4).  These threads issue no
    // cp.async, so their fence.proxy.async covers only their own st.shared. =====
    const int r = tid - 128;
    const int lg = warp & 3, chalf = (warp - 4) >> 2;
    uint32_t *stg = reinterpret_cast<uint32_t *>(bslots) + (warp - 4) * 32 * 36;  // epilogue only
    GemmCursor cc;
    cc.start(b);
    uint32_t tiles = 0;
    for (uint32_t p = 0; cc.item < b.total; ++p) {
      const int s = p % kGemmStages, bs = p % kGemmBSlots;
      uint8_t *st = smem + s * stage_bytes;
      uint8_t *bt = bslots + bs * kBTileBytes;
#ifdef TB_GEMM_TRACE_DEC
      if (tid == 128) GT(p, 0);
#endif
      mbar_spin(&full[s], (p / kGemmStages) & 1);
#ifdef TB_GEMM_TRACE_DEC
      if (tid == 128) GT(p, 1);
#endif
      if (p >= (uint32_t)kGemmBSlots) mbar_spin(&bempty[bs], (p / kGemmBSlots - 1) & 1);
      if (tid == 128) GT(p, 2);
      const GemmJob &J = b.jobs[cc.j];
#pragma unroll
      for (int cs = 0; cs < kChunksPerStage; ++cs) {  // the row's packed chunks of this stage
        const int rr = r;
        uint4 o[4];
        if (cc.n0 + rr < J.Npad) {
          // TMA box [row tile][chunk][32 rows][16 B]
          const uint4 pk = *reinterpret_cast<const uint4 *>(
              st + a_bytes + (((rr >> 5) * kChunksPerStage + cs) * kRowTile + (rr & 31)) * 16);
          o[0] = code_planes<FMT>(pk.x);
          o[1] = code_planes<FMT>(pk.y);
          o[2] = code_planes<FMT>(pk.z);
          o[3] = code_planes<FMT>(pk.w);
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) o[i] = make_uint4(0, 0, 0, 0);
        }
        // core matrix (row group rr/8, k core 4 cs + i): 128 B, row rr%8 at 16 B
#ifndef TB_GEMM_NO_UNPACK  // profiling variant (results invalid): no B stores
#pragma unroll
        for (int i = 0; i < 4; ++i)
          *reinterpret_cast<uint4 *>(bt + ((rr >> 3) * kGemmKC + 4 * cs + i) * 128 + (rr & 7) * 16) = o[i];
#else
        if (o[0].x == 0x12345678u) *reinterpret_cast<uint4 *>(bt) = o[1];
#endif
      }
#ifdef TB_GEMM_TRACE_DEC
      if (tid == 128) GT(p, 5);
#endif
#ifndef TB_GEMM_NO_FENCE  // profiling variant (results invalid): fence cost
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // st.shared -> tensor core
#endif
      mbar_arrive(&bready[bs]);
      if (tid == 128) GT(p, 3);
      if (cc.last()) {
        // ---- epilogue of this tile ----
#ifdef TB_GEMM_TRACE_EPI
        if (tid == 128 && blockIdx.x == 0 && tiles < 16) g_epi_trace[tiles][0] = clock64();
#endif
        mbar_spin(&tfull, tiles & 1);
#ifdef TB_GEMM_TRACE_EPI
        if (tid == 128 && blockIdx.x == 0 && tiles < 16) g_epi_trace[tiles][1] = clock64();
#endif
        tc_fence_after();
        int32_t *acc_out = J.acc_out;
        const int32_t *rowsum =
            reinterpret_cast<const int32_t *>(J.act + (size_t)J.C * b.Mpad * kGemmBK);
        double *out64 = J.out64;
        float *out32 = J.out32;
        const double ws = J.w_scale;
        const int Nj = J.N;
        for (int mt = 0; mt < MT; ++mt) {
          const int mrow0 = cc.h * (kGemmMaxMT * kGemmSubM) + mt * kGemmSubM + lg * 32;
          if (mrow0 >= M) break;
          const double my_as = (mrow0 + lane < M && J.a_scale) ? J.a_scale[mrow0 + lane] : 0.0;
          const float my_fs = static_cast<float>(ws * my_as);  // per-token fp32 scale
          const int32_t my_sum = rowsum[mrow0 + lane];  // sum_k a[m][k] (tile_act)
          const int rows = min(32, M - mrow0);
#pragma unroll 1
          for (int cb = 0; cb < kGemmBN / 64; ++cb) {
            const int col = chalf * (kGemmBN / 2) + cb * 32;
            uint32_t v[32];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                  "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
                  "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
                  "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                  "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
                  "=r"(v[30]), "=r"(v[31])
                : "r"(tmem + ((uint32_t)(lg * 32) << 16) + mt * kGemmBN + col));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            // fp32-only outputs of a full 32-column block: 128-bit stores, four
            // rows per warp instruction (the output write is what limits the
            // epilogue); rows staged with a 36-word pitch (16-B aligned)
            if (out32 && !out64 && !acc_out && (Nj & 3) == 0 && cc.n0 + col + 32 <= Nj) {
#pragma unroll
              for (int e = 0; e < 32; e += 4)
                *reinterpret_cast<uint4 *>(stg + lane * 36 + e) =
                    make_uint4(v[e], v[e + 1], v[e + 2], v[e + 3]);
              __syncwarp();
              const int q = lane >> 3, c4 = (lane & 7) * 4;
#pragma unroll
              for (int it = 0; it < 8; ++it) {
                const int r = it * 4 + q;
                const int32_t asum = __shfl_sync(0xffffffffu, my_sum, r);
                const float fs = __shfl_sync(0xffffffffu, my_fs, r);
                if (r < rows) {
                  const uint4 w = *reinterpret_cast<const uint4 *>(stg + r * 36 + c4);
                  float4 o;
                  o.x = static_cast<float>((int32_t)w.x - asum) * fs;
                  o.y = static_cast<float>((int32_t)w.y - asum) * fs;
                  o.z = static_cast<float>((int32_t)w.z - asum) * fs;
                  o.w = static_cast<float>((int32_t)w.w - asum) * fs;
                  *reinterpret_cast<float4 *>(out32 + (int64_t)(mrow0 + r) * Nj + cc.n0 + col + c4) = o;
                }
              }
              __syncwarp();
              continue;
            }
            // general path -- lane = row: stage it XOR-rotated, then lane = column
#pragma unroll
            for (int e = 0; e < 32; ++e) stg[lane * 32 + ((e + lane) & 31)] = v[e];
            __syncwarp();
            const int n = cc.n0 + col + lane;
#ifdef TB_GEMM_NO_EPI  // profiling variant: no output stores
            const bool on = false;
#else
            const bool on = n < Nj;
#endif
            // 32 independent rows in flight (one warp per scheduler: ILP, not TLP)
#pragma unroll
            for (int rr = 0; rr < 32; ++rr) {
              const double as = __shfl_sync(0xffffffffu, my_as, rr);
              const int32_t asum = __shfl_sync(0xffffffffu, my_sum, rr);
              const float fs = __shfl_sync(0xffffffffu, my_fs, rr);
              if (on && rr < rows) {
                const int32_t a = (int32_t)stg[rr * 32 + ((lane + rr) & 31)] - asum;
                const int64_t off = (int64_t)(mrow0 + rr) * Nj + n;
                if (acc_out) acc_out[off] = a;
                if (out64) {  // exact float64 chain of core.py:99-101 (fp64-rate bound)
                  const double y = static_cast<double>(a) * ws * as;
                  out64[off] = y;
                  if (out32) out32[off] = static_cast<float>(y);
                } else if (out32) {
                  // fp32 outputs: a * (ws * as) in float32, within 2^-22 of the
                  // float64 result (north star: 1e-5 relative for fp32 outputs);
                  // |a| < 2^24 converts exactly.  B200 float64 issue is too slow
                  // for 64K products per tile.
                  out32[off] = static_cast<float>(a) * fs;
                }
              }
            }
            __syncwarp();
          }
        }
        // the staging rows live in the B slots: no warp may start unpacking the
        // next tile's first stages into them while another still stages its
        // accumulators there (the epilogue warps finish at different times,
        // most visibly on the float64 outputs)
        asm volatile("bar.sync 1, 256;" ::: "memory");
        tc_fence_before();
        mbar_arrive(&tempty);
#ifdef TB_GEMM_TRACE_EPI
        if (tid == 128 && blockIdx.x == 0 && tiles < 16) g_epi_trace[tiles][2] = clock64();
#endif
        ++tiles;
      }
      cc.next(b);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer no longer writes our shared memory / barriers
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols));
}

// Natural int8 activations [M][lda] -> the GEMM's A layout, zero padded to
// Mpad rows and ks = ceil(cols / 64) K stages, each 16-byte group in code-
// plane order (position 4s + q holds a[16i + 4q + s]):
// out[((ks_i * Mpad/8 + g) * 4 + c) * 128 + r8 * 16 + p] = act[8g + r8][64 ks_i + 16 c + perm(p)],
// followed by the per-token sums int32 [Mpad] (the unsigned-code correction).
__global__ void gemm_tile_act_kernel(const int8_t *__restrict__ act, int M, int64_t lda, int cols,
                                     int Mpad, int ks, uint8_t *__restrict__ out) {
  const int64_t units = (int64_t)ks * Mpad * kGemmKC;  // 16-byte units
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < units;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int r8 = (int)(u & 7);
    const int64_t q = u >> 3;  // (ks_i, g, c)
    const int c = (int)(q % kGemmKC);
    const int64_t q2 = q / kGemmKC;
    const int g = (int)(q2 % (Mpad / 8));
    const int ksi = (int)(q2 / (Mpad / 8));
    const int m = g * 8 + r8;
    const int64_t k = (int64_t)ksi * kGemmBK + c * 16;
    uint32_t w[4] = {0, 0, 0, 0};
    if (m < M) {
      const int8_t *src = act + (int64_t)m * lda + k;
      if (k + 16 <= cols && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        const uint4 v = *reinterpret_cast<const uint4 *>(src);
        w[0] = v.x, w[1] = v.y, w[2] = v.z, w[3] = v.w;
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (k + i < cols) w[i >> 2] |= (uint32_t)(uint8_t)src[i] << (8 * (i & 3));
      }
    }
    // 4x4 byte transpose: word s = (a[s], a[4+s], a[8+s], a[12+s])
    const uint32_t t0 = prmt(w[0], w[1], 0x5140u), t1 = prmt(w[0], w[1], 0x7362u);
    const uint32_t t2 = prmt(w[2], w[3], 0x5140u), t3 = prmt(w[2], w[3], 0x7362u);
    reinterpret_cast<uint4 *>(out)[u] = make_uint4(prmt(t0, t2, 0x5410u), prmt(t0, t2, 0x7632u),
                                                   prmt(t1, t3, 0x5410u), prmt(t1, t3, 0x7632u));
  }
}

__global__ void gemm_rowsum_kernel(const int8_t *__restrict__ act, int M, int64_t lda, int cols,
                                   int Mpad, int32_t *__restrict__ sums) {
  const int m = blockIdx.x;
  int32_t acc = 0;
  if (m < M)
    for (int k = threadIdx.x; k < cols; k += blockDim.x) acc += act[(int64_t)m * lda + k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ int32_t part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += part[i];
    sums[m] = t;
  }
}

// quantize_activations (core.py:116-134) straight into the GEMM's A layout:
// float32 tokens [M][ldx] -> the bytes tb_gemm_tile_act writes (tiled int8
// codes in code-plane order + per-token code sums) and the float64 scales.
// 16 floats of a unit (zero beyond K)
__device__ __forceinline__ void qa_load16(const float *row, int64_t k, int K, bool vec, float *f) {
  if (vec && k + 16 <= K) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 v = __ldg(reinterpret_cast<const float4 *>(row + k) + i);
      f[4 * i] = v.x, f[4 * i + 1] = v.y, f[4 * i + 2] = v.z, f[4 * i + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) f[i] = k + i < K ? row[k + i] : 0.0f;
  }
}
// 16 codes in code-plane order (word s = (a[s], a[4+s], a[8+s], a[12+s]))
__device__ __forceinline__ uint4 qa_codes16(const float *f, float inv_sf, double sc, double inv_s,
                                            int32_t &sum) {
  uint32_t wd[4] = {0, 0, 0, 0};
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int q = quantize_fast(f[i], inv_sf, sc, inv_s);
    sum += q;
    wd[i >> 2] |= (uint32_t)(uint8_t)(int8_t)q << (8 * (i & 3));
  }
  const uint32_t t0 = prmt(wd[0], wd[1], 0x5140u), t1 = prmt(wd[0], wd[1], 0x7362u);
  const uint32_t t2 = prmt(wd[2], wd[3], 0x5140u), t3 = prmt(wd[2], wd[3], 0x7362u);
  return make_uint4(prmt(t0, t2, 0x5410u), prmt(t0, t2, 0x7632u), prmt(t1, t3, 0x5410u),
                    prmt(t1, t3, 0x7632u));
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// Tiled weights [T][C][32 rows x 16 B] as a 3-D tensor of 8-byte elements
// {64, C, T}; a box {64, 1, 8} is one K stage of 256 rows.
static bool encode_weight_map(CUtensorMap *map, const uint8_t *w, int C, int T) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {kTileChunkBytes / 8, (cuuint64_t)C, (cuuint64_t)T};
  const cuuint64_t strides[2] = {kTileChunkBytes, (cuuint64_t)C * kTileChunkBytes};
  const cuuint32_t box[3] = {kTileChunkBytes / 8, kChunksPerStage, kGemmBN / kRowTile};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<uint8_t *>(w), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int FMT>
static int launch_gemm(GemmBatch &b, cudaStream_t s) {
  const int stage = b.MT * kSubTileBytes + kPackedBytes;
  const int smem = kGemmStages * stage + kGemmBSlots * kBTileBytes + 1024 + 1024;
  static int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    const int max_smem =
        kGemmStages * (kGemmMaxMT * kSubTileBytes + kPackedBytes) + kGemmBSlots * kBTileBytes + 2048;
    if (cudaFuncSetAttribute(tgemm_kernel<FMT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             max_smem) != cudaSuccess)
      return TB_ERR_CUDA;
    configured_dev = dev;
  }
  const int pairs = std::max(1, std::min(b.total, sm_count_cached() / kGemmCluster));
  // Longest-processing-time-first static schedule: items (cost = K stages)
  // go to the least-loaded pair, largest first -- a 224-stage down-projection
  // tile no longer lands on a pair that already has two 64-stage tiles.
  b.scheduled = 0;
  if (b.total <= kGemmMaxSched && pairs <= kGemmMaxPairs) {
    std::vector<std::pair<int, int>> items;  // (cost, item)
    for (int it = 0; it < b.total; ++it) {
      const int tt = it / b.MH;
      int jj = 0;
      while (jj + 1 < b.njobs && b.jobs[jj + 1].tile0 <= tt) ++jj;
      items.push_back({b.jobs[jj].C, it});
    }
    std::stable_sort(items.begin(), items.end(),
                     [](const std::pair<int, int> &x, const std::pair<int, int> &y) { return x.first > y.first; });
    std::vector<long long> load(pairs, 0);
    std::vector<std::vector<int>> lists(pairs);
    for (const auto &ci : items) {
      int best = 0;
      for (int q = 1; q < pairs; ++q)
        if (load[q] < load[best]) best = q;
      load[best] += ci.first + 8;  // + a per-tile epilogue allowance
      lists[best].push_back(ci.second);
    }
    int off = 0;
    for (int q = 0; q < pairs; ++q) {
      b.sched_off[q] = (uint16_t)off;
      for (int it : lists[q]) b.sched[off++] = (uint16_t)it;
    }
    b.sched_off[pairs] = (uint16_t)off;
    b.scheduled = 1;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pairs * kGemmCluster);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kGemmCluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if (cudaLaunchKernelEx(&cfg, tgemm_kernel<FMT>, b) != cudaSuccess) return TB_ERR_CUDA;
  return TB_OK;
}

static int64_t gemm_stages_of(int64_t cols) { return ceil_div(cols, kGemmBK); }

}  // namespace tb

using namespace tb;

#ifdef TB_GEMM_TRACE_EPI
extern "C" int tb_gemm_epi_trace_fetch(void *host, int64_t bytes) {
  return cudaMemcpyFromSymbol(host, g_epi_trace, bytes) == cudaSuccess ? 0 : 2;
}
#endif
#ifdef TB_GEMM_TRACE
extern "C" int tb_gemm_trace_fetch(void *host, int64_t bytes) {
  return cudaMemcpyFromSymbol(host, g_gemm_trace, bytes) == cudaSuccess ? 0 : 2;
}
#endif

// token rows of the tiled A: one 128-row sub-tile, or whole 256-row halves
static int64_t gemm_mpad(int64_t M) {
  return M <= kGemmSubM ? kGemmSubM : pad_up(M, kGemmMaxMT * kGemmSubM);
}

extern "C" int64_t tb_gemm_act_bytes(int64_t M, int64_t cols) {
  if (M < 1 || M > kGemmMaxM || cols < 1) return -1;
  // codes, per-token code sums, and (tb_gemm_quantize_act scratch) per-token
  // reciprocal scales: float64 [Mpad] + float32 [Mpad]
  return gemm_stages_of(cols) * gemm_mpad(M) * kGemmBK +
         gemm_mpad(M) * (int64_t)(sizeof(int32_t) + sizeof(double) + sizeof(float));
}

extern "C" int tb_gemm_tile_act(const int8_t *act, int64_t M, int64_t lda, int64_t cols,
                                uint8_t *out, void *stream) {
  if (!act || !out || M < 1 || M > kGemmMaxM || cols < 1 || lda < cols ||
      (reinterpret_cast<uintptr_t>(out) & 15))
    return TB_ERR_ARGUMENT;
  const int Mpad = (int)gemm_mpad(M);
  const int ks = (int)gemm_stages_of(cols);
  const int64_t units = (int64_t)ks * Mpad * 4;
  const int grid = (int)std::min<int64_t>(ceil_div(units, 256), (int64_t)sm_count_cached() * 8);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  gemm_tile_act_kernel<<<grid, 256, 0, s>>>(act, (int)M, lda, (int)cols, Mpad, ks, out);
  gemm_rowsum_kernel<<<Mpad, 256, 0, s>>>(act, (int)M, lda, (int)cols, Mpad,
                                          reinterpret_cast<int32_t *>(out + (int64_t)ks * Mpad * kGemmBK));
  TB_CHECK_LAUNCH();
  return TB_OK;
}

// Two launches (no clusters): (1) one CTA per
// token row: absmax (integer max of |x| bits), the float64 scale, the
// non-finite flag, and the row's code sum zeroed; (2) a programmatic
// dependent grid over (8-token row group, block of 4 K stages): quantise
// (x is L2-resident after (1)), stage the block's 16-byte units in shared
// memory, write whole 1 KB (stage, row group) blocks, add the per-token code
// sums with one atomic per row.  Every CTA has work from its first
// instruction (a single-launch form with 8-CTA clusters sharing the absmax
// through DSMEM measured 6.2 / 14-16 us for the cfg3 layer's two inputs,
// this one 6.0 / 12.5 us).
constexpr int kQa2Stages = 4;  // K stages per (2) CTA

// Up to kQaMaxInputs activation matrices of the same token count per launch
// pair (a layer's x_h and x_i: two launches instead of four, and the small
// input's CTAs run beside the large one's).
constexpr int kQaMaxInputs = 4;
struct QaInput {
  const float *x;
  double *scale;
  int32_t *flag;
  uint8_t *out;
  int64_t ldx;
  int K, ks;
  int blk0;  // first blockIdx.y of this input in the codes launch
};
struct QaBatch {
  QaInput in[kQaMaxInputs];
  int n, M, Mpad;
};

__global__ void __launch_bounds__(512) qa_absmax_kernel(const __grid_constant__ QaBatch qb) {
  // programmatic dependent of whatever precedes it (the previous layer's
  // GEMM reads the scales and row sums this kernel rewrites, and x may be a
  // preceding kernel's output): everything after the wait; the launch
  // latency and CTA scheduling still overlap the predecessor's tail
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const int v = blockIdx.x / qb.Mpad, m = blockIdx.x - v * qb.Mpad;
  const QaInput &I = qb.in[v];
  const int M = qb.M, K = I.K;
  const float *x = I.x;
  const int64_t ldx = I.ldx;
  int32_t *rowsum = reinterpret_cast<int32_t *>(I.out + (int64_t)I.ks * qb.Mpad * kGemmBK);
  if (m >= M) {
    if (threadIdx.x == 0) rowsum[m] = 0;
    return;
  }
  const float *row = x + (int64_t)m * ldx;
  uint32_t amax = 0;
  const bool vec = ((reinterpret_cast<uintptr_t>(x) | (uintptr_t)(ldx * 4)) & 15) == 0;
  int k = threadIdx.x * 4;
  if (vec)
#pragma unroll 8  // several loads in flight per thread (the max is the only dependence)
    for (; k + 3 < K; k += 512 * 4) {
      const uint4 v4 = __ldg(reinterpret_cast<const uint4 *>(row + k));
      amax = max(amax, max(max(v4.x & 0x7fffffffu, v4.y & 0x7fffffffu),
                           max(v4.z & 0x7fffffffu, v4.w & 0x7fffffffu)));
    }
  for (; k < K; k += 512 * 4)
    for (int i = 0; i < 4 && k + i < K; ++i) amax = max(amax, __float_as_uint(row[k + i]) & 0x7fffffffu);
  amax = __reduce_max_sync(0xffffffffu, amax);
  __shared__ uint32_t red[16];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
  __syncthreads();
  if (threadIdx.x < 32) {
    amax = threadIdx.x < 16 ? red[threadIdx.x] : 0u;
    amax = __reduce_max_sync(0xffffffffu, amax);
    if (threadIdx.x == 0) {
      const double a = (double)__uint_as_float(amax);
      const double sc = a > 0.0 ? a / 127.0 : 1.0;  // core.py:128-130
      I.scale[m] = sc;
      // the reciprocals the codes launch multiplies by, once per token: a
      // float64 division per LANE there (2,304 CTAs x 8 warps of them for the
      // cfg3 layer) kept this GPU's narrow float64 pipe busy for ~20 us
      const double inv = 1.0 / sc;
      double *invs = reinterpret_cast<double *>(rowsum + qb.Mpad);
      invs[m] = inv;
      reinterpret_cast<float *>(invs + qb.Mpad)[m] = (float)inv;
      if (amax >= 0x7f800000u && I.flag) atomicOr(I.flag, 1);
      rowsum[m] = 0;
    }
  }
}

__global__ void __launch_bounds__(256) qa_codes_kernel(const __grid_constant__ QaBatch qb) {
  __shared__ uint4 stage[kQa2Stages * kGemmKC * 8];
  asm volatile("griddepcontrol.launch_dependents;");  // the GEMM: its prologue overlaps our tail
  int v = 0;
#pragma unroll
  for (int q = 1; q < kQaMaxInputs; ++q)
    if (q < qb.n && (int)blockIdx.y >= qb.in[q].blk0) v = q;
  const QaInput &I = qb.in[v];
  const int M = qb.M, Mpad = qb.Mpad, K = I.K, ks = I.ks;
  const float *x = I.x;
  const int64_t ldx = I.ldx;
  uint8_t *out = I.out;
  const int g = blockIdx.x, blk = blockIdx.y - I.blk0;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = g * 8 + w;
  const int ks0 = blk * kQa2Stages;
  const int nks = min(ks, ks0 + kQa2Stages) - ks0;
  const int64_t k0 = (int64_t)ks0 * kGemmBK;
  const float *row = x + (int64_t)m * ldx;
  const bool vec = ((reinterpret_cast<uintptr_t>(x) | (uintptr_t)(ldx * 4)) & 15) == 0;
  const int units = nks * kGemmKC;  // one 16-column unit per lane (32 units)
  float f[16];
  const int64_t k = k0 + (int64_t)lane * 16;
  // (x was read by the absmax launch, which waited for its producer: safe before our wait)
  if (m < M && lane < units && k < K) {
    qa_load16(row, k, K, vec, f);
  } else {
#pragma unroll
    for (int e = 0; e < 16; ++e) f[e] = 0.0f;
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the scales of (1)
  const double *invs = reinterpret_cast<const double *>(
      reinterpret_cast<const int32_t *>(out + (int64_t)ks * Mpad * kGemmBK) + Mpad);
  const double sc = m < M ? I.scale[m] : 1.0;
  const double inv_s = m < M ? invs[m] : 1.0;
  const float inv_sf = m < M ? reinterpret_cast<const float *>(invs + Mpad)[m] : 1.0f;
  int32_t sum = 0;
  if (lane < units) stage[lane * 8 + w] = qa_codes16(f, inv_sf, sc, inv_s, sum);
  sum = __reduce_add_sync(0xffffffffu, sum);
  if (lane == 0 && m < M && sum != 0)
    atomicAdd(reinterpret_cast<int32_t *>(out + (int64_t)ks * Mpad * kGemmBK) + m, sum);
  __syncthreads();
  const int G = Mpad / 8;
  uint4 *o4 = reinterpret_cast<uint4 *>(out);
  for (int i = threadIdx.x; i < nks * kGemmKC * 8; i += 256) {
    const int ksl = i / (kGemmKC * 8), j = i % (kGemmKC * 8);
    o4[((int64_t)(ks0 + ksl) * G + g) * (kGemmKC * 8) + j] = stage[i];
  }
}

// One launch, one pass over the activations: a CTA per token row holds the
// row in registers (up to kQaRowUnits 16-column units per thread: K <= 16,384),
// reduces the absmax, quantises from the registers and writes its 16-byte
// units of the operand layout and the row's code sum -- no second read, no
// atomics, nothing to zero.  (The two-launch form read the inputs twice and
// took 13.6 + 13.8 us for the cfg3 layer's 37.7 MB.)
constexpr int kQaRowThreads = 512, kQaRowUnits = 2;
__global__ void __launch_bounds__(kQaRowThreads, 2) qa_row_kernel(const __grid_constant__ QaBatch qb) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");  // the GEMM: its prologue overlaps our tail
  const int v = blockIdx.x / qb.Mpad, m = blockIdx.x - v * qb.Mpad;
  const QaInput &I = qb.in[v];
  const int M = qb.M, K = I.K, ks = I.ks;
  const int nunits = ks * kGemmKC;  // 16-column units of a (stage-padded) row
  const float *row = I.x + (int64_t)m * I.ldx;
  const bool vec = ((reinterpret_cast<uintptr_t>(I.x) | (uintptr_t)(I.ldx * 4)) & 15) == 0;
  int32_t *rowsum = reinterpret_cast<int32_t *>(I.out + (int64_t)ks * qb.Mpad * kGemmBK);
  uint4 *o4 = reinterpret_cast<uint4 *>(I.out);
  const int G = qb.Mpad / 8, g = m >> 3, w = m & 7;
  float f[kQaRowUnits][16];
  uint32_t amax = 0;
#pragma unroll
  for (int i = 0; i < kQaRowUnits; ++i) {
    const int u = threadIdx.x + i * kQaRowThreads;
    if (m < M && u < nunits && (int64_t)u * 16 < K) {
      qa_load16(row, (int64_t)u * 16, K, vec, f[i]);
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) f[i][e] = 0.0f;
    }
  }
#pragma unroll
  for (int i = 0; i < kQaRowUnits; ++i)
#pragma unroll
    for (int e = 0; e < 16; ++e) amax = max(amax, __float_as_uint(f[i][e]) & 0x7fffffffu);
  amax = __reduce_max_sync(0xffffffffu, amax);
  __shared__ uint32_t red[kQaRowThreads / 32];
  __shared__ int32_t reds[kQaRowThreads / 32];
  __shared__ double s_sc, s_inv;
  __shared__ float s_invf;
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
  __syncthreads();
  if (threadIdx.x < 32) {
    amax = threadIdx.x < kQaRowThreads / 32 ? red[threadIdx.x] : 0u;
    amax = __reduce_max_sync(0xffffffffu, amax);
    if (threadIdx.x == 0) {
      const double a = (double)__uint_as_float(amax);
      const double sc = a > 0.0 ? a / 127.0 : 1.0;  // core.py:128-130
      const double inv = 1.0 / sc;
      s_sc = sc;
      s_inv = inv;
      s_invf = (float)inv;
      if (m < M) {
        I.scale[m] = sc;
        if (amax >= 0x7f800000u && I.flag) atomicOr(I.flag, 1);
      }
    }
  }
  __syncthreads();
  const double sc = s_sc, inv_s = s_inv;
  const float inv_sf = s_invf;
  int32_t sum = 0;
#pragma unroll
  for (int i = 0; i < kQaRowUnits; ++i) {
    const int u = threadIdx.x + i * kQaRowThreads;
    if (u < nunits) {
      const uint4 c = qa_codes16(f[i], inv_sf, sc, inv_s, sum);
      const int ksl = u / kGemmKC, kc = u - ksl * kGemmKC;
      o4[((int64_t)ksl * G + g) * (kGemmKC * 8) + kc * 8 + w] = c;
    }
  }
  sum = __reduce_add_sync(0xffffffffu, sum);
  if ((threadIdx.x & 31) == 0) reds[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x < 32) {
    sum = threadIdx.x < kQaRowThreads / 32 ? reds[threadIdx.x] : 0;
    sum = __reduce_add_sync(0xffffffffu, sum);
    if (threadIdx.x == 0) rowsum[m] = sum;
  }
}

// Measured and dropped (all bit-exact): a persistent streaming form -- one CTA
// per SM, rows arriving by bulk async copies into two shared-memory buffers
// while the previous row is quantised, float4 reads and a 4 x 4 byte
// transpose across lane quads -- 29 us against this kernel's 21 us for the
// cfg3 layer (one CTA per SM exposes every block-wide phase; two
// register-resident CTAs per SM cover each other's); the float64 reciprocal
// taken off the row's critical path (no change: 115.6 vs 116.1 us per layer);
// a magic-number rounding of whole units with byte-permute packing (fewer
// instructions, but 16 more live registers under the 64-register cap: spills,
// 123 us).  ncu: 3.46 waves of 2 CTAs per SM, issue slots 45 % busy.
extern "C" int tb_gemm_quantize_act_multi(int64_t n, const tb_qact_desc *d, int64_t M,
                                          void *stream) {
  if (n < 1 || n > kQaMaxInputs || !d || M < 1 || M > kGemmMaxM) return TB_ERR_ARGUMENT;
  QaBatch qb{};
  qb.n = (int)n;
  qb.M = (int)M;
  qb.Mpad = (int)gemm_mpad(M);
  int blocks = 0;
  for (int64_t v = 0; v < n; ++v) {
    if (!d[v].x || !d[v].scale || !d[v].act_tiled || d[v].cols < 1 || d[v].ldx < d[v].cols ||
        d[v].cols > (int64_t)1 << 30 || (reinterpret_cast<uintptr_t>(d[v].act_tiled) & 15))
      return TB_ERR_ARGUMENT;
    QaInput &I = qb.in[v];
    I.x = d[v].x;
    I.scale = d[v].scale;
    I.flag = d[v].nonfinite_flag;
    I.out = d[v].act_tiled;
    I.ldx = d[v].ldx;
    I.K = (int)d[v].cols;
    I.ks = (int)gemm_stages_of(d[v].cols);
    I.blk0 = blocks;
    blocks += (int)ceil_div(I.ks, kQa2Stages);
  }
  if (blocks > 65535) return TB_ERR_UNSUPPORTED;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(qb.Mpad * qb.n));
  cfg.blockDim = dim3(512);
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
#ifndef TB_QA_TWO_LAUNCH
  bool fits = true;  // every row register resident: the one-launch form
  for (int v = 0; v < qb.n; ++v)
    fits = fits && qb.in[v].ks * kGemmKC <= kQaRowThreads * kQaRowUnits;
  if (fits) {
    cfg.blockDim = dim3(kQaRowThreads);
    return cudaLaunchKernelEx(&cfg, qa_row_kernel, qb) == cudaSuccess ? TB_OK : TB_ERR_CUDA;
  }
#endif
  if (cudaLaunchKernelEx(&cfg, qa_absmax_kernel, qb) != cudaSuccess) return TB_ERR_CUDA;
  cfg.gridDim = dim3((unsigned)(qb.Mpad / 8), (unsigned)blocks);
  cfg.blockDim = dim3(256);
  return cudaLaunchKernelEx(&cfg, qa_codes_kernel, qb) == cudaSuccess ? TB_OK : TB_ERR_CUDA;
}

extern "C" int tb_gemm_quantize_act(const float *x, int64_t M, int64_t cols, int64_t ldx,
                                    double *scale, int32_t *nonfinite_flag, uint8_t *out,
                                    void *stream) {
  tb_qact_desc d{x, cols, ldx, scale, nonfinite_flag, out};
  return tb_gemm_quantize_act_multi(1, &d, M, stream);
}

extern "C" int tb_gemm_batch(int fmt, int64_t njobs, const tb_gemm_desc *descs, int64_t M,
                             void *stream) {
  if (fmt == TB_TL2) return TB_ERR_UNSUPPORTED;
  if ((fmt != TB_I2S && fmt != TB_TL1) || njobs < 1 || njobs > kGemmMaxJobs || !descs || M < 1 ||
      M > kGemmMaxM)
    return TB_ERR_ARGUMENT;
  GemmBatch b{};
  b.njobs = (int)njobs;
  b.M = (int)M;
  b.Mpad = (int)gemm_mpad(M);
  b.MT = b.Mpad >= kGemmMaxMT * kGemmSubM ? kGemmMaxMT : 1;
  b.MH = (int)ceil_div(b.Mpad, b.MT * kGemmSubM);
  int tiles = 0;
  for (int64_t j = 0; j < njobs; ++j) {
    const tb_gemm_desc &d = descs[j];
    if (!d.tiled || !d.act_tiled || d.rows < 1 || d.cols < 1 || ((d.out64 || d.out32) && !d.a_scale) ||
        (reinterpret_cast<uintptr_t>(d.act_tiled) & 15) || (reinterpret_cast<uintptr_t>(d.tiled) & 15))
      return TB_ERR_ARGUMENT;
    GemmJob &J = b.jobs[j];
    J.w = d.tiled;
    J.act = d.act_tiled;
    J.a_scale = d.a_scale;
    J.w_scale = d.w_scale;
    J.acc_out = d.acc_out;
    J.out64 = d.out64;
    J.out32 = d.out32;
    J.N = (int)d.rows;
    J.Npad = (int)pad_up(d.rows, kRowTile);
    J.C = (int)ceil_div(ref_row_bytes(fmt, d.cols), (int64_t)kChunkBytes * kChunksPerStage);  // K stages
    // the tensor map walks the tiled layout's 16-byte chunks (tile stride C_chunks x 512 B)
    if (!encode_weight_map(&J.bmap, d.tiled, (int)ceil_div(ref_row_bytes(fmt, d.cols), kChunkBytes),
                           (int)ceil_div(d.rows, kRowTile)))
      return TB_ERR_CUDA;
    J.tile0 = tiles;  // in tile pairs
    J.ntiles = (int)ceil_div(d.rows, kGemmBN);
    tiles += (int)ceil_div(J.ntiles, kGemmCluster);
  }
  b.total = tiles * b.MH;  // pair items
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return launch_gemm<TB_I2S>(b, s);  // TL1 tiles hold I2_S codes (pack.cu repack)
}

extern "C" int tb_gemm_i8(int fmt, const uint8_t *tiled, int64_t rows, int64_t cols,
                          const int8_t *act, int64_t M, int64_t lda, const double *a_scale,
                          double w_scale, uint8_t *workspace, int32_t *acc_out, double *out64,
                          float *out32, void *stream) {
  if (M < 1 || !workspace) return TB_ERR_ARGUMENT;
  for (int64_t m0 = 0; m0 < M; m0 += kGemmMaxM) {
    const int64_t mm = std::min<int64_t>(M - m0, kGemmMaxM);
    int st = tb_gemm_tile_act(act + m0 * lda, mm, lda, cols, workspace, stream);
    if (st != TB_OK) return st;
    tb_gemm_desc d{};
    d.tiled = tiled;
    d.rows = rows;
    d.cols = cols;
    d.act_tiled = workspace;
    d.a_scale = a_scale ? a_scale + m0 : nullptr;
    d.w_scale = w_scale;
    d.acc_out = acc_out ? acc_out + m0 * rows : nullptr;
    d.out64 = out64 ? out64 + m0 * rows : nullptr;
    d.out32 = out32 ? out32 + m0 * rows : nullptr;
    st = tb_gemm_batch(fmt, 1, &d, mm, stream);
    if (st != TB_OK) return st;
  }
  return TB_OK;
}
