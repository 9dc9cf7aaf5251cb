// Decode GEMV (M <= 16) on the tiled I2_S / TL1 / TL2 layouts -- grouped.
//
// Replaces kernels.gemv_i2s / gemv_tl1 / gemv_tl2 / gemv_parallel
// (pkg/src/ternpack/kernels.py:86-157, 189-268) and the numba byte-table
// gathers (_fast.py:25-95).  The reference gathers one int32 table entry per
// packed byte; here the packed bytes are decoded in registers to 2-bit codes
// c = w + 1 in {0,1,2} (four per 32-bit word, one per byte lane) and
// contracted with dp4a against byte-transposed int8 activations (the
// "records" of gemv_records.cuh).  sum_k w_k a_k = sum_k c_k a_k - sum_k a_k,
// so per-chunk activation sums are subtracted once per chunk.  Integer results
// are exact, hence bit-identical to the reference's LUT/byte-table kernels.
//
// One launch serves a *group* of independent GEMVs ("jobs": e.g. the gate, up
// and down projections of a token, or every projection of a layer) so the
// weight stream never stops at a matrix boundary and the kernel's fixed
// costs (launch, first-byte latency, completion) are paid once per group.
//
// Data movement: persistent grid, one CTA per SM, every warp autonomous.  The
// jobs' (row tile, chunk) spaces are concatenated into one flat range -- each
// job's part a contiguous byte range of its tiled layout -- split evenly over
// all warps of the grid; each warp streams its range (weights, TL2 signs and
// the matching activation records) HBM/L2 -> SMEM through its own ring of
// cp.async.bulk stages, one mbarrier per stage: no CTA-wide synchronisation.
// lane = row of the 32-row tile, so activation reads are warp broadcasts and
// weight reads conflict-free 16-byte LDS.  A warp's partial sums for a row
// tile go to the job's self-cleaning int32 workspace with red.global.add; the
// warp that retires the tile's last chunk (acq_rel counter) applies the
// scales (core.py:99-101), writes the outputs and resets the workspace.
#include <algorithm>
#include <atomic>

#include "gemv_records.cuh"

namespace tb {

constexpr int kMaxInlineJobs = 20;  // a layer at M = 8: 6 projections x 2 K-windows of x_h + 6 K-windows of down
constexpr int kMaxSegs = 8;
constexpr int kMaxStepCluster = 4;  // fused step: CTAs sharing one quantisation
#ifndef TB_STEP_CLUSTER
#define TB_STEP_CLUSTER 2
#endif
constexpr int kStepCQ = TB_STEP_CLUSTER;

// Optional per-warp timeline (debug builds with -DTB_TIMELINE only).
#ifdef TB_TIMELINE
constexpr int kTimelineWarps = 148 * 32;
__device__ unsigned long long g_timeline[kTimelineWarps][5];
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
#ifdef TB_TL_CLOCK  // SM clock cycles (per-warp deltas only; SMs are not in sync)
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
#else
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
#endif
  return t;
}
#define TL_MARK(i)                                                    \
  do {                                                                \
    if (lane == 0 && gw < kTimelineWarps) g_timeline[gw][i] = globaltimer_ns(); \
  } while (0)
#else
#define TL_MARK(i) \
  do {             \
  } while (0)
#endif
// -DTB_TL_PROLOGUE: marks 1-3 time the fused prologue (weights issued, absmax
// reduced, records built) instead of the main loop
#ifdef TB_TL_PROLOGUE
#define TL_PMARK(i) TL_MARK(i)
#define TL_LMARK(i) \
  do {              \
  } while (0)
#else
#define TL_PMARK(i) \
  do {              \
  } while (0)
#define TL_LMARK(i) TL_MARK(i)
#endif

// FU: 0 = records path; 1 = fused step, small CTAs, several per SM; 3 = fused
// step, 8-warp CTAs, two per SM (record tables up to 56 KB: the ~100B stack's
// 43K-element inputs); 2 = fused step, 16 warps, one CTA per SM (larger tables
// or an isolated launch)
template <int FMT, int MT, int FU = 0>
struct Cfg {
  static constexpr bool kFused = FU >= 1 && FU <= 3;
  // FU = 4: the records path (M > 1 tokens, records built by a glue kernel)
  // with the CTA's records in ONE shared-memory table filled at entry instead
  // of staged per warp and ring stage: the ring carries weights only.
  static constexpr bool kTable = FU == 4;
#ifndef TB_MT1_WARPS
#define TB_MT1_WARPS 16
#endif
#ifndef TB_FUSED_WARPS
#define TB_FUSED_WARPS 5
#endif
#ifndef TB_FUSED_MINB
#define TB_FUSED_MINB 4
#endif
#ifndef TB_FUSED_RING
#define TB_FUSED_RING 3
#endif
  // fused step: small CTAs (I2_S / TL1: 5 warps with 3-stage rings, <= ~55 KB,
  // four per SM; TL2, whose decode needs more registers: 8 warps, two per SM)
  // -- the next steps' CTAs (programmatic dependent launch) quantise and
  // prefetch while this step's CTAs stream
#ifndef TB_TL2_WARPS
#define TB_TL2_WARPS 8
#endif
#ifndef TB_TL2_MINB
#define TB_TL2_MINB 2
#endif
#ifndef TB_TL2_RING
#define TB_TL2_RING 4
#endif
#ifndef TB_MED_WARPS
#define TB_MED_WARPS 8
#endif
#ifndef TB_MED_RING
#define TB_MED_RING 3
#endif
#ifndef TB_MED_RECTAB_KB
#define TB_MED_RECTAB_KB 56
#endif
  // records-table CTAs: 8 warps with 3-stage rings (48 KB) and a 60 KB table,
  // TWO per SM, so one CTA's table fill and tail (the previous layer's
  // finalize) overlap the other's weight stream -- with the pipelined layers
  // (tb_gemv_batch_launch_sync) the two are consecutive layers
#ifndef TB_TABLE_WARPS
#define TB_TABLE_WARPS 8
#endif
#ifndef TB_TABLE_MINB
#define TB_TABLE_MINB 2
#endif
#ifndef TB_TABLE_RING
#define TB_TABLE_RING 3
#endif
#ifndef TB_TABLE_KB
#define TB_TABLE_KB 60
#endif
  static constexpr int kWarps = FU == 1 ? (FMT == TB_TL2 ? TB_TL2_WARPS : TB_FUSED_WARPS)
                                : FU == 3 ? TB_MED_WARPS
                                : FU == 4 ? TB_TABLE_WARPS
                                          : (MT == 1 ? TB_MT1_WARPS : (MT <= 8 ? 16 : 8));
  static constexpr int kMinBlocks =
      FU == 1 ? (FMT == TB_TL2 ? TB_TL2_MINB : TB_FUSED_MINB) : FU == 3 ? 2 : FU == 4 ? TB_TABLE_MINB : 1;
#ifndef TB_MT1_RING
#define TB_MT1_RING (TB_MT1_WARPS > 16 ? 3 : 4)
#endif
  // M > 1: the deepest ring (<= 4 stages) that fits next to nothing else
  static constexpr int kStageBytesAll =
      kStageChunks * (kTileChunkBytes + Fmt<FMT>::kSignBytes + MT * Fmt<FMT>::kRecBytes);
  static constexpr int kFit = (225 * 1024) / (kWarps * kStageBytesAll);
  static constexpr int kRing = FU == 1 ? (FMT == TB_TL2 ? TB_TL2_RING : TB_FUSED_RING)
                               : FU == 3 ? TB_MED_RING
                               : FU == 4 ? TB_TABLE_RING
                               : (MT == 1 ? TB_MT1_RING : (kFit >= 4 ? 4 : (kFit >= 2 ? kFit : 2)));
  static constexpr int kThreads = 32 * kWarps;
  // register cap through the launch bounds (table mode: room for a glue CTA
  // beside two table CTAs -- 2 x 256 x 96 + 256 x 64 registers = the SM's 64K)
#ifndef TB_TABLE_BOUND_THREADS
#define TB_TABLE_BOUND_THREADS kThreads
#endif
  static constexpr int kBoundThreads = FU == 4 ? TB_TABLE_BOUND_THREADS : kThreads;
  // fused step: previous-step outputs finalised per thread at the wait point
  static constexpr int kFinPer = FU == 3 ? 3 : 2;
  // fused step: records live in a CTA-wide table after the ring, not per stage
  static constexpr int kStageBytes =
      kStageChunks * (kTileChunkBytes + Fmt<FMT>::kSignBytes + (kFused || kTable ? 0 : MT) * Fmt<FMT>::kRecBytes);
  static constexpr int kRingBytes = kWarps * kRing * kStageBytes;
#ifndef TB_SMALL_RECTAB_KB
#define TB_SMALL_RECTAB_KB 40
#endif
  static constexpr int kRecTabBytes =
      kTable ? TB_TABLE_KB * 1024
      : !kFused ? 0 : (FU == 3 ? TB_MED_RECTAB_KB : kMinBlocks >= 2 ? TB_SMALL_RECTAB_KB : 64) * 1024;  // records of all inputs
  static constexpr int kSmem = kRingBytes + kRecTabBytes;
  static_assert(kSmem <= 227 * 1024 - 512, "ring does not fit in shared memory");
};

struct GemvJob {
  const uint8_t *wmain;
  const uint8_t *wsign;
  const uint8_t *rec;  // [M][C][kRecBytes]
  const double *a_scale;
  double w_scale;
  int32_t *ws_acc;  // [16][Npad]
  int32_t *ws_cnt;  // [T]
  int32_t *acc_out;
  double *out64;
  float *out32;
  int N, Npad, C, M;
  int start;  // first flat chunk of this job
  int end;    // one past its last flat chunk (start + T * C)
  int src;    // fused step: index of the input vector this job contracts
  int c0;     // first record chunk of that input (a K-window job contracts
              // input columns [64 c0, ...) -- 96 c0 for TL2)
  int cin;    // records path: chunks per token row of the global records (>= c0 + C)
  int fin_m;  // tokens the finalize covers: M, or 0 for a job with no outputs
              // (a K-window whose sums land in a workspace another job finalises)
};

// Fused decode step (tgemv_kernel<FMT, 1, true>): the launch quantises its own
// float32 input vectors (every CTA, into shared memory), runs the grouped
// GEMV, and afterwards finalises the PREVIOUS step's batch -- whose grid has
// completed by then (griddepcontrol.wait) -- so a decode step is one launch.
constexpr int kMaxStepInputs = 4;
constexpr int kMaxNeedCtas = 160;  // per-CTA input masks (>= the 148 SMs of a B200)
constexpr int kMaxInlineFin = 8;   // previous-step jobs finalised from kernel parameters

// What the finalize needs of a job, carried in the next step's parameters so
// the tail of every CTA does no dependent descriptor loads.
struct FinJob {
  int32_t *ws_acc;
  int32_t *acc_out;
  double *out64;
  float *out32;
  const double *a_scale;
  double w_scale;
  int N, Npad, M;
};
struct StepInputs {
  const float *x[kMaxStepInputs];
  const int32_t *ready[kMaxStepInputs];  // optional: spin until != 0 before reading x
  double *scale[kMaxStepInputs];   // per-token scale out (read by the finalize)
  int32_t *flag[kMaxStepInputs];   // optional non-finite flag
  int K[kMaxStepInputs], C[kMaxStepInputs], off[kMaxStepInputs];  // off: record table offset
  int n;
  int x_after_wait;      // inputs produced by the preceding grid: read them after the wait
  int sticky_flags;      // store the non-finite flag only when set
  int self_fin;          // the launch finalises its own outputs (per-tile counters)
  int no_wait;           // ... and never waits for the preceding kernel (TB_STEP_INDEPENDENT)
  const GemvJob *prev;   // device job table finalised after this launch's own work
  int prev_njobs;
  int prev_inline;       // 1: prev jobs are in fin[] below
  FinJob fin[kMaxInlineFin];
  int32_t *tab_sync;     // table mode: the layer's sync block (see LayerSync), or null
  int tab_sync_want;     // ... and the glue's CTA count
  int16_t writer[kMaxStepInputs];  // CTA that publishes input v's scale / flag
  uint8_t need[kMaxNeedCtas];      // inputs (bit v) the CTA's jobs contract
};

struct GemvBatch {
  GemvJob jobs[kMaxInlineJobs];
  const GemvJob *table;  // device copy, used when njobs > kMaxInlineJobs
  int njobs;
  int total;  // flat chunks over all jobs
  // Warp ranges.  The flat chunk space is cut into segments (the fused step:
  // runs of jobs contracting the same input, so no CTA has to quantise two
  // inputs), each owning CTAs [seg_cta[s], seg_cta[s+1]) and chunks
  // [seg_chunk[s], seg_chunk[s+1]); segment warp w gets
  // unit * (base + (w < rem)) chunks (+ tail: its last warp).
  int unit;  // a ring stage, so stages rarely straddle a row tile
  int nseg;
  int seg_cta[kMaxSegs + 1], seg_chunk[kMaxSegs + 1];
  int seg_base[kMaxSegs], seg_rem[kMaxSegs], seg_tail[kMaxSegs];
  int defer_finalize;  // host: the caller finalises (e.g. in the next glue kernel)
  int max_entries;     // host: max over jobs of M * Npad (sizes the finalize grid)
  int fin_parts;       // device (glue): 8-CTA groups per job in the finalize rows
  StepInputs in;       // fused step only
};

// Job descriptor by value: inline jobs come from the (grid-constant) kernel
// parameters via indexed constant loads, larger groups from a global table.
__device__ __forceinline__ GemvJob job_at(const GemvBatch &b, int j) {
  if (b.table) return b.table[j];
  return b.jobs[j];
}

__device__ __forceinline__ int32_t ld_acquire_gpu(const int32_t *p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int atom_add_acq_rel(int *ptr, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(ptr), "r"(v)
               : "memory");
  return old;
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Publish a warp's partial sums of one row tile: fire-and-forget REDs into
// the job's int32 workspace (no fence, no completion counter -- measured at
// ~4.6 us per launch on B200 for a 43 MB group).  The grid boundary orders
// them before gemv_finalize_kernel, which applies the scales.
template <int FMT, int MT>
__device__ __forceinline__ void flush_tile(const GemvBatch &b, int j, int t,
                                           const Acc<FMT, MT> &acc, int M, int lane) {
#ifdef TB_NO_FLUSH  // profiling variant: drop the partial sums
  return;
#endif
  const GemvJob J = job_at(b, j);
#ifdef TB_I2S_MMA
  if constexpr (FMT == TB_I2S && kI2sMma<MT>) {  // tensor-core fragments: direct REDs
    acc.red_all(J.ws_acc, J.Npad, t * kRowTile, M);
    return;
  }
#endif
  const int row = t * kRowTile + lane;
#pragma unroll
  for (int m = 0; m < MT; ++m)
    if (m == 0 || m < M) red_add_s32(J.ws_acc + (int64_t)m * J.Npad + row, acc.total(m));
}

// After the GEMV grid: output = f64(acc) * w_scale * a_scale[m] (core.py:
// 99-101), optional int32 / f32 copies, and the workspace is zeroed again.
// Launched with programmatic dependent launch: griddepcontrol.wait blocks
// until the GEMV grid has completed and its memory operations are visible.
// Finalize job j with CTAs `part` of `nparts` (every thread of the CTA).
__device__ __forceinline__ void finalize_one(const GemvJob &J, int part, int nparts) {
  const int64_t total = (int64_t)J.fin_m * J.Npad;
  for (int64_t i = part * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)nparts * blockDim.x) {
    const int m = (int)(i / J.Npad), row = (int)(i - (int64_t)m * J.Npad);
    const int32_t v = atomicExch(J.ws_acc + i, 0);  // read and reset: one L2 operation
    if (row < J.N) {
      const int64_t o = (int64_t)m * J.N + row;
      if (J.acc_out) J.acc_out[o] = v;
      if (J.out64 || J.out32) {
        const double y = static_cast<double>(v) * J.w_scale * J.a_scale[m];
        if (J.out64) J.out64[o] = y;
        if (J.out32) J.out32[o] = static_cast<float>(y);
      }
    }
  }
}

// All inline previous-step jobs as ONE flat index space (a thread usually
// gets a single entry): every load is issued in the first round instead of one
// latency round per job.
__device__ __forceinline__ void finalize_fin_all(const FinJob *fin, int njobs, int part,
                                                 int nparts) {
  int64_t total = 0;
  for (int j = 0; j < njobs; ++j) total += (int64_t)fin[j].M * fin[j].Npad;
  for (int64_t i = part * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)nparts * blockDim.x) {
    int j = 0;
    int64_t k = i;
    while (k >= (int64_t)fin[j].M * fin[j].Npad) {
      k -= (int64_t)fin[j].M * fin[j].Npad;
      ++j;
    }
    const FinJob &J = fin[j];
    const int m = (int)(k / J.Npad), row = (int)(k - (int64_t)m * J.Npad);
    const int32_t v = atomicExch(J.ws_acc + k, 0);  // read and reset: one L2 operation
    if (row < J.N) {
      const int64_t o = (int64_t)m * J.N + row;
      if (J.acc_out) J.acc_out[o] = v;
      if (J.out64 || J.out32) {
        const double y = static_cast<double>(v) * J.w_scale * J.a_scale[m];
        if (J.out64) J.out64[o] = y;
        if (J.out32) J.out32[o] = static_cast<float>(y);
      }
    }
  }
}

// Flat entries first, first + stride, ... (the tail beyond one per thread).
__device__ __forceinline__ void finalize_fin_range(const FinJob *fin, int njobs, int64_t first,
                                                   int64_t stride) {
  int64_t total = 0;
  for (int j = 0; j < njobs; ++j) total += (int64_t)fin[j].M * fin[j].Npad;
  for (int64_t i = first; i < total; i += stride) {
    int j = 0;
    int64_t k = i;
    while (k >= (int64_t)fin[j].M * fin[j].Npad) {
      k -= (int64_t)fin[j].M * fin[j].Npad;
      ++j;
    }
    const FinJob &J = fin[j];
    const int m = (int)(k / J.Npad), row = (int)(k - (int64_t)m * J.Npad);
    const int32_t v = atomicExch(J.ws_acc + k, 0);  // read and reset: one L2 operation
    if (row < J.N) {
      const int64_t o = (int64_t)m * J.N + row;
      if (J.acc_out) J.acc_out[o] = v;
      const double y = static_cast<double>(v) * J.w_scale * J.a_scale[m];
      if (J.out64) J.out64[o] = y;
      if (J.out32) J.out32[o] = static_cast<float>(y);
    }
  }
}

__device__ __forceinline__ void finalize_job(const GemvBatch &b, int j, int part, int nparts) {
  finalize_one(job_at(b, j), part, nparts);
}

// grid (parts, njobs): every job finalised concurrently.
__global__ void gemv_finalize_kernel(const __grid_constant__ GemvBatch b) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  finalize_job(b, blockIdx.y, blockIdx.x, gridDim.x);
}

// ---------------------------------------------------------------------------
// "Glue" between two GEMV groups of a decode step, in ONE launch: finalize
// the previous group (scales -> outputs, workspace reset) and quantise the
// next group's input vectors into records.  Rows [0, q_tokens) of the grid
// are per-token 8-CTA clusters (quantize_token), the remaining rows finalise
// one job each.  Replaces 1 finalize + one quantise launch per input vector.
// ---------------------------------------------------------------------------
constexpr int kMaxGlueVecs = 4;

__device__ __forceinline__ int32_t ld_acquire_gpu_fwd(const int32_t *p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct QuantVec {
  const void *x;
  int8_t *qnat;
  double *scale;
  uint8_t *rec;
  int32_t *flag;
  int64_t K, ldx, ldq;
  int M, C, fmt, is_f64;
};

struct GlueParams {
  GemvBatch fin;  // fin.njobs == 0: nothing to finalise
  QuantVec q[kMaxGlueVecs];
  int nq, q_tokens;
  int early;      // quantise before griddepcontrol.wait (TB_GLUE_EARLY_QUANT)
  // pipelined layers (tb_step_glue_sync): this layer's sync block and the
  // previous layer's (null: the first layer of a pass waits for everything)
  int32_t *sync_self, *sync_prev;
  int publish_exit;  // a later glue consumes this glue's exit count
  int prev_exit_ctas;  // CTAs of the previous glue (what its exit count reaches)
  // pipelined layers: the previous layer's outputs, finalised by the
  // quantising CTAs themselves after their wait (jobs inline: no table loads)
  FinJob finl[kMaxInlineFin];
  int nfinl;
};

// Pipelined M > 1 layers.  Per layer, four counters in device memory:
//   [kSyRecs]  glue CTAs that have written their records
//   [kSySeen]  GEMV CTAs that have seen [kSyRecs] complete (the last resets both)
//   [kSyExit]  glue CTAs past their griddepcontrol.wait (the preceding GEMV --
//              and, through its tail wait, everything before it -- completed)
//   [kSyESeen] CTAs of the NEXT glue that have seen [kSyExit] complete (reset)
// Every wait is on a grid whose CTAs are all resident (it was launched
// before the waiter could start), so the spins cannot deadlock; they are
// bounded anyway (kSyncSpinLimit polls), and a timeout is counted in
// g_sync_timeouts (tb_sync_timeouts) instead of hanging the GPU.
constexpr int kSyRecs = 0, kSySeen = 1, kSyExit = 2, kSyESeen = 3;
constexpr int kSyncSpinLimit = 1 << 22;  // x ~100 ns: ~0.5 s
__device__ int g_sync_timeouts;

// thread 0 of the CTA waits for *cnt == want, the CTA is released by the
// barrier; the last of `consumers` CTAs to arrive resets the pair
__device__ __forceinline__ void sync_consume(int32_t *cnt, int32_t *seen, int want, int consumers) {
  if (threadIdx.x == 0) {
    int spins = 0;
    while (ld_acquire_gpu_fwd(cnt) != want) {
      __nanosleep(64);
      if (++spins > kSyncSpinLimit) {
        atomicAdd(&g_sync_timeouts, 1);
        break;
      }
    }
    if (atomicAdd(seen, 1) == consumers - 1) {
      atomicExch(cnt, 0);
      atomicExch(seen, 0);
    }
  }
  __syncthreads();
}
// the CTA's writes, then one count (release: the threadfence-reduction pattern)
__device__ __forceinline__ void sync_publish(int32_t *cnt) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(cnt, 1);
  }
}

template <int FMT>
__device__ __forceinline__ void glue_quant(const QuantVec &Q, int m) {
  if (Q.is_f64)
    quantize_token<FMT, double, 256>(static_cast<const double *>(Q.x), Q.K, Q.ldx, Q.qnat, Q.ldq,
                                     Q.scale, Q.C, Q.rec, Q.flag, m, blockIdx.x, gridDim.x);
  else
    quantize_token<FMT, float, 256>(static_cast<const float *>(Q.x), Q.K, Q.ldx, Q.qnat, Q.ldq,
                                    Q.scale, Q.C, Q.rec, Q.flag, m, blockIdx.x, gridDim.x);
}

// The glue's finalize: every job's M x Npad entries as ONE flat space in
// units of 4 (Npad is a multiple of 32, so a unit never straddles a job or a
// token row); int4 workspace loads, kGlueIlp units in flight per thread, and
// only as many CTAs as that needs (a few hundred, not one per 256 entries).
constexpr int kMaxGlueFin = 16;
constexpr int kGlueIlp = 4;
__device__ __forceinline__ void glue_finalize_units(const FinJob *fj, const int64_t *pre, int njobs,
                                                    int part, int nparts);
__device__ __forceinline__ void glue_finalize_flat(const GemvBatch &b, int part, int nparts) {
  __shared__ FinJob fj[kMaxGlueFin];
  __shared__ int64_t pre[kMaxGlueFin + 1];
  if ((int)threadIdx.x < b.njobs) {
    const GemvJob J = job_at(b, threadIdx.x);
    fj[threadIdx.x] = FinJob{J.ws_acc, J.acc_out, J.out64, J.out32, J.a_scale, J.w_scale,
                             J.N, J.Npad, J.fin_m};
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    pre[0] = 0;
    for (int j = 0; j < b.njobs; ++j) pre[j + 1] = pre[j] + (int64_t)fj[j].M * fj[j].Npad;
  }
  __syncthreads();
  glue_finalize_units(fj, pre, b.njobs, part, nparts);
}
// ... over jobs given inline in the kernel parameters (pipelined layers)
__device__ __forceinline__ void glue_finalize_inline(const FinJob *jobs, int njobs, int part,
                                                     int nparts) {
  __shared__ FinJob fj[kMaxInlineFin];
  __shared__ int64_t pre[kMaxInlineFin + 1];
  if ((int)threadIdx.x < njobs) fj[threadIdx.x] = jobs[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    pre[0] = 0;
    for (int j = 0; j < njobs; ++j) pre[j + 1] = pre[j] + (int64_t)fj[j].M * fj[j].Npad;
  }
  __syncthreads();
  glue_finalize_units(fj, pre, njobs, part, nparts);
}
__device__ __forceinline__ void glue_finalize_units(const FinJob *fj, const int64_t *pre, int njobs,
                                                    int part, int nparts) {
  struct { int njobs; } b{njobs};
  const int64_t units = pre[b.njobs] >> 2;
  const int64_t stride = (int64_t)nparts * blockDim.x;
  for (int64_t u0 = (int64_t)part * blockDim.x + threadIdx.x; u0 < units; u0 += stride * kGlueIlp) {
    int4 v[kGlueIlp];
    int jj[kGlueIlp];
    int64_t kk[kGlueIlp];
#pragma unroll
    for (int q = 0; q < kGlueIlp; ++q) {  // all loads first
      const int64_t u = u0 + q * stride;
      jj[q] = -1;
      if (u < units) {
        const int64_t e = u << 2;
        int j = 0;
        while (j + 1 < b.njobs && pre[j + 1] <= e) ++j;
        jj[q] = j;
        kk[q] = e - pre[j];
        // read and reset with atomics: a store after a load of the same
        // address waits for the load's data, serialising the ILP (measured:
        // the M = 8 finalize of a cfg4 layer 16 us -> ...)
        int32_t *ws = fj[j].ws_acc + kk[q];
        v[q] = make_int4(atomicExch(ws, 0), atomicExch(ws + 1, 0), atomicExch(ws + 2, 0),
                         atomicExch(ws + 3, 0));
      }
    }
#pragma unroll
    for (int q = 0; q < kGlueIlp; ++q) {
      if (jj[q] < 0) continue;
      const FinJob &J = fj[jj[q]];
      const int m = (int)(kk[q] / J.Npad), row0 = (int)(kk[q] - (int64_t)m * J.Npad);
      const double as = (J.out64 || J.out32) ? __ldcg(J.a_scale + m) : 0.0;
      const int32_t a[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int row = row0 + e;
        if (row < J.N) {
          const int64_t o = (int64_t)m * J.N + row;
          if (J.acc_out) J.acc_out[o] = a[e];
          const double y = static_cast<double>(a[e]) * J.w_scale * as;  // core.py:99-101
          if (J.out64) J.out64[o] = y;
          if (J.out32) J.out32[o] = static_cast<float>(y);
        }
      }
    }
  }
}

#ifndef TB_GLUE_MINB
#define TB_GLUE_MINB 3
#endif
__global__ void __launch_bounds__(256, TB_GLUE_MINB) glue_kernel(const __grid_constant__ GlueParams g) {
  // early: the quantisation (inputs that do not depend on the preceding
  // kernel, records that nothing in flight reads -- the caller's contract)
  // overlaps the preceding kernel; every CTA still waits for it before
  // exiting, so this grid's completion implies the predecessor's
  // pipelined layers (sync_self): the first layer of a pass (no sync_prev)
  // waits for everything before it; every other layer waits only for the
  // previous glue's EXIT count -- that glue exits after the GEMV two layers
  // back completed, so nothing in flight reads the record set (three in
  // rotation) or the scales this glue writes
  const bool piped = g.sync_self != nullptr;
  if (!g.early || (piped && !g.sync_prev)) asm volatile("griddepcontrol.wait;" ::: "memory");
  // the next GEMV group may launch now: its prologue prefetches weights (no
  // dependence on us) and then waits for this grid before reading records
  asm volatile("griddepcontrol.launch_dependents;");
  const int y = blockIdx.y;
  if (y < g.q_tokens) {
    if (piped && g.sync_prev)
      sync_consume(g.sync_prev + kSyExit, g.sync_prev + kSyESeen, g.prev_exit_ctas,
                   (int)gridDim.x * g.q_tokens);
    int v = 0, m = y;
    while (m >= g.q[v].M) {
      m -= g.q[v].M;
      ++v;
    }
    if (g.q[v].fmt == TB_TL2) glue_quant<TB_TL2>(g.q[v], m);
    else glue_quant<TB_I2S>(g.q[v], m);  // I2_S and TL1 share the record layout
    if (piped) sync_publish(g.sync_self + kSyRecs);  // the GEMV's table fill waits for this
    if (g.early) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (piped) {
      // the previous GEMV has completed: its outputs, finalised by these same
      // CTAs (already resident beside the streaming GEMV: no CTA sits waiting
      // in an SM slot the next layer's GEMV could use), then the exit count --
      // the glue that overwrites the scales read here waits for it
      if (g.nfinl > 0)
        glue_finalize_inline(g.finl, g.nfinl, y * gridDim.x + blockIdx.x,
                             g.q_tokens * gridDim.x);
      if (g.publish_exit) sync_publish(g.sync_self + kSyExit);
    }
    return;
  }
  if (g.early) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (g.fin.njobs <= kMaxGlueFin) {
    const int r = y - g.q_tokens;  // finalize rows: flat over every job's entries
    glue_finalize_flat(g.fin, r * gridDim.x + blockIdx.x, g.fin.fin_parts * gridDim.x);
  } else {
    const int r = y - g.q_tokens;  // (job, group) of 8 CTAs: one element per thread
    const int j = r / g.fin.fin_parts, part = r - j * g.fin.fin_parts;
    finalize_job(g.fin, j, part * gridDim.x + blockIdx.x, g.fin.fin_parts * gridDim.x);
  }
}

// Position of the warp's streaming cursor: job j, tile t, chunk c of the tile.
struct Cursor {
  int j, t, c;
};

__device__ __forceinline__ void cp_async16_cg(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16_ca(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Stage `cnt` chunks starting at cursor `cur` into `slot` with cp.async
// (every lane issues its own 16-byte copies: no TMA request-rate limit).
// Runs split at job boundaries (weights are contiguous within a job); the
// activation-record chunk index wraps at row-tile ends.
constexpr int kIssueWeights = 1, kIssueRecords = 2, kIssueAll = 3;

template <int FMT, int kWhat>
__device__ void issue_chunks(const GemvBatch &b, Cursor cur, int cnt, uint8_t *slot, int lane) {
  using F = Fmt<FMT>;
  uint8_t *sign_slot = slot + kStageChunks * kTileChunkBytes;
  uint8_t *act_slot = slot + kStageChunks * (kTileChunkBytes + F::kSignBytes);
#ifdef TB_NO_LOADS  // profiling variant: compute on stale shared memory only
  return;
#endif
  int done = 0;
  while (done < cnt) {
    GemvJob J = job_at(b, cur.j);
    const int C = J.C;
    const int left_in_job = J.end - (J.start + cur.t * C + cur.c);
    const int run = min(cnt - done, left_in_job);
    const int64_t g = (int64_t)cur.t * C + cur.c;  // chunk index in the job's tiled layout
    // weights: lane = row, 16 B per chunk (a coalesced 512 B per warp instruction)
    if (kWhat & kIssueWeights) {
      for (int r = 0; r < run; ++r)
        cp_async16_cg(slot + (done + r) * kTileChunkBytes + lane * 16,
                      J.wmain + (g + r) * kTileChunkBytes + lane * 16);
      if (FMT == TB_TL2 && lane < kTileSignBytes / 16)
        for (int r = 0; r < run; ++r)
          cp_async16_cg(sign_slot + (done + r) * kTileSignBytes + lane * 16,
                        J.wsign + (g + r) * kTileSignBytes + lane * 16);
    }
    // activation records of every token (chunk index wraps at row-tile ends)
    constexpr int RU = F::kRecBytes / 16;
    const int units = (kWhat & kIssueRecords) ? J.M * run * RU : 0;
    for (int u = lane; u < units; u += 32) {
      const int m = u / (run * RU);
      const int rem = u - m * run * RU;
      const int d = rem / RU, q = rem - d * RU;
      const int c = (cur.c + d) % C;
      cp_async16_ca(act_slot + (m * kStageChunks + done + d) * F::kRecBytes + q * 16,
                    J.rec + ((int64_t)m * J.cin + J.c0 + c) * F::kRecBytes + q * 16);
    }
    done += run;
    // advance the cursor
    cur.c += run;
    cur.t += cur.c / C;
    cur.c %= C;
    if (J.start + cur.t * C + cur.c >= J.end) {
      ++cur.j;
      cur.t = 0;
      cur.c = 0;
    }
  }
}

__device__ __forceinline__ void advance(const GemvBatch &b, Cursor &cur, int k) {
  GemvJob J = job_at(b, cur.j);
  cur.c += k;
  while (cur.c >= J.C) {
    cur.c -= J.C;
    ++cur.t;
    if (J.start + cur.t * J.C >= J.end) {
      ++cur.j;
      cur.t = 0;
      if (cur.j < b.njobs) J = job_at(b, cur.j);
    }
  }
}

// Issue cursor with the current job's pointers cached, so the common stage
// (4 chunks inside one row tile of one job) is 4 weight copies + 1 record copy
// per lane and no integer division.
struct IssueState {
  Cursor cur;
  const uint8_t *w;    // weights of chunk `cur` in the job's tiled layout
  const uint8_t *sgn;  // TL2 sign bits of chunk `cur`
  const uint8_t *rec;  // the job's record base
  int C, T, M, CI, C0;  // CI: record chunks per token row; C0: the window's first

  __device__ __forceinline__ void reset(const GemvBatch &b, Cursor c) {
    cur = c;
    const GemvJob J = job_at(b, c.j);
    C = J.C;
    M = J.M;
    CI = J.cin;
    T = (J.end - J.start) / J.C;
    const int64_t g = (int64_t)c.t * C + c.c;
    w = J.wmain + g * kTileChunkBytes;
    sgn = J.wsign + g * kTileSignBytes;
    rec = J.rec;
    C0 = J.c0;
  }

  template <int FMT, int kWhat = kIssueAll>
  __device__ __forceinline__ void issue(const GemvBatch &b, int cnt, uint8_t *slot, int lane) {
    using F = Fmt<FMT>;
    if (cnt == kStageChunks && cur.c + kStageChunks <= C) {
      uint8_t *sign_slot = slot + kStageChunks * kTileChunkBytes;
      uint8_t *act_slot = slot + kStageChunks * (kTileChunkBytes + F::kSignBytes);
#ifndef TB_NO_LOADS
      if (kWhat & kIssueWeights) {
#pragma unroll
        for (int r = 0; r < kStageChunks; ++r)
          cp_async16_cg(slot + r * kTileChunkBytes + lane * 16,
                        w + r * kTileChunkBytes + lane * 16);
        if (FMT == TB_TL2 && lane < kTileSignBytes / 16) {
#pragma unroll
          for (int r = 0; r < kStageChunks; ++r)
            cp_async16_cg(sign_slot + r * kTileSignBytes + lane * 16,
                          sgn + r * kTileSignBytes + lane * 16);
        }
      }
      if ((kWhat & kIssueRecords) && lane < kStageChunks * F::kRecBytes / 16)
        for (int m = 0; m < M; ++m)  // the stage's 4 records are contiguous
          cp_async16_ca(act_slot + m * kStageChunks * F::kRecBytes + lane * 16,
                        rec + ((int64_t)m * CI + C0 + cur.c) * F::kRecBytes + lane * 16);
#endif
      w += kStageChunks * kTileChunkBytes;
      sgn += kStageChunks * kTileSignBytes;
      cur.c += kStageChunks;
      if (cur.c == C) {
        cur.c = 0;
        if (++cur.t == T) {
          ++cur.j;
          cur.t = 0;
          if (cur.j < b.njobs) reset(b, cur);
        }
      }
      return;
    }
    issue_chunks<FMT, kWhat>(b, cur, cnt, slot, lane);  // general path: tile / job boundaries
    advance(b, cur, cnt);
    if (cur.j < b.njobs) reset(b, cur);
  }
};

template <int FMT, int MT, int FU, int CQ = 1>  // CQ: cluster size of the fused step
__global__ void __launch_bounds__(Cfg<FMT, MT, FU>::kBoundThreads, Cfg<FMT, MT, FU>::kMinBlocks)
    tgemv_kernel(const __grid_constant__ GemvBatch b) {
  using F = Fmt<FMT>;
  using CF = Cfg<FMT, MT, FU>;
  constexpr bool kFused = CF::kFused;
  constexpr bool kTable = CF::kTable;
  static_assert(!kFused || MT == 1, "the fused step is a one-token decode step");
  constexpr int kRing = CF::kRing;
  constexpr int kIssueMain = (kFused || kTable) ? kIssueWeights : kIssueAll;
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t *ring = smem + warp * kRing * CF::kStageBytes;
  uint8_t *rtab_base = smem + CF::kRingBytes;  // fused: record tables of the inputs

  const int gw = blockIdx.x * CF::kWarps + warp;
  TL_MARK(0);
  // let our programmatic dependent (finalize kernel / next step) launch early
  asm volatile("griddepcontrol.launch_dependents;");
  // Fused step: the input loads go out first -- they depend on nothing but the
  // CTA's input mask, while the warp-range and job lookups below are chains of
  // constant-bank loads that are cold at launch (~1.4 us measured before the
  // loads were issued when they came after them).
  // register groups of 16 inputs per thread (medium CTAs: 4, so a CTA pair holds a 32K input)
  constexpr int kMaxG = FU == 3 ? 4 : CQ >= 2 ? (CF::kThreads <= 128 ? 4 : CF::kThreads <= 192 ? 3 : 2) : (FMT == TB_TL2 ? (CF::kThreads >= 384 ? 2 : 3) : 4);
  RegQuant<FMT, CF::kThreads, kMaxG> rq;
  constexpr int cq = CQ;
  int crank = 0, need = 0;
  if constexpr (kFused) {
    need = blockIdx.x < kMaxNeedCtas ? b.in.need[blockIdx.x] : 0xF;
    crank = CQ > 1 ? (int)cluster_rank() : 0;
    if (cq > 1) cluster_arrive_relaxed();
    // inputs filled by a copy that signals completion (HostPipeline block
    // starts): an in-kernel wait instead of a graph edge, which would end the
    // programmatic-dependent-launch overlap with the previous step
#pragma unroll
    for (int v = 0; v < kMaxStepInputs; ++v)
      if (v < b.in.n && b.in.ready[v] && ((need >> v) & 1))
        while (ld_acquire_gpu(b.in.ready[v]) == 0) __nanosleep(200);
#ifndef TB_FUSED_NOLOAD  // profiling variants: TB_FUSED_NOLOAD / TB_FUSED_NOQ
    if (!b.in.x_after_wait) rq.load(b.in.x, b.in.K, b.in.C, b.in.n, need, crank, cq);
#else
    rq.G = 0;
#endif
  }
  int seg = 0;
#pragma unroll
  for (int q = 1; q < kMaxSegs; ++q)
    if (q < b.nseg && (int)blockIdx.x >= b.seg_cta[q]) seg = q;
  const int lw = gw - b.seg_cta[seg] * CF::kWarps;  // warp within the segment
  const int sbase = b.seg_base[seg], srem = b.seg_rem[seg];
  const int w0 = b.seg_chunk[seg] + b.unit * (lw * sbase + min(lw, srem));
  const int n = b.unit * (sbase + (lw < srem ? 1 : 0)) +
                (lw == (b.seg_cta[seg + 1] - b.seg_cta[seg]) * CF::kWarps - 1 ? b.seg_tail[seg] : 0);
  bool waited = false;
  int tab_C = 0, tab_M = 0;  // table mode: the segment's window (chunks) and tokens
  __shared__ double s_scale[kMaxStepInputs];
  int s_badm = 0;  // fused: non-finite inputs (bit v), identical in every thread
  if constexpr (!kFused && !kTable) {
    if (n <= 0) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      return;
    }
  }
  const int nst = (n + kStageChunks - 1) / kStageChunks;

  // locate the first chunk
  Cursor cur{0, 0, 0};
  IssueState is;  // issue cursor + cached job pointers (identical in every lane)
  if (n > 0) {
    if (b.table) {
      while (cur.j + 1 < b.njobs && job_at(b, cur.j + 1).start <= w0) ++cur.j;
    } else {  // inline jobs: independent constant loads, no dependent chain
#pragma unroll
      for (int j = 1; j < kMaxInlineJobs; ++j)
        if (j < b.njobs && b.jobs[j].start <= w0) cur.j = j;
    }
    GemvJob J = job_at(b, cur.j);
    const int local = w0 - J.start;
    cur.t = local / J.C;
    cur.c = local - cur.t * J.C;
    is.reset(b, cur);
  }
  // Prologue.  Weights never depend on the previous kernel, so the first
  // stages' weights are requested before griddepcontrol.wait (this kernel is
  // a programmatic dependent of whatever produced the activation records);
  // the records follow once the producer has completed.
  // record groups held in registers per thread (the rest take the looped path)
  if constexpr (kFused) {
    // (the input loads went out at entry; now the weight prefetch; the loaded
    // values are consumed after both.)  Thread-block cluster (launch
    // attribute): its Q CTAs quantise disjoint slices of the inputs (same
    // `need`) and share records through DSMEM.
#ifdef TB_TL_PM1_EARLY
    TL_PMARK(1);
#endif
#ifndef TB_PRE_STAGES
#define TB_PRE_STAGES kRing
#endif
    constexpr int kPre = TB_PRE_STAGES < kRing ? TB_PRE_STAGES : kRing;
#pragma unroll 1
    for (int k = 0; k < kPre; ++k) {
      if (k < nst) is.issue<FMT, kIssueWeights>(b, min(kStageChunks, n - k * kStageChunks),
                                                ring + k * CF::kStageBytes, lane);
      cp_async_commit();
    }
    if (b.in.x_after_wait) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      waited = true;
      rq.load(b.in.x, b.in.K, b.in.C, b.in.n, need, crank, cq);
    }
    // quantise every input vector into this CTA's record tables
    __shared__ float red[CF::kWarps * 4];
    __shared__ uint32_t cl_amax[kMaxStepCluster * 4];
    if (rq.fits()) {
#ifndef TB_FUSED_NOQ
#ifndef TB_TL_PM1_EARLY
      TL_PMARK(1);
#endif
#ifndef TB_FUSED_NORED
      s_badm = rq.reduce(b.in.n, s_scale, red, cl_amax, crank, cq);
#endif
      TL_PMARK(2);
#ifndef TB_FUSED_NOREC
      rq.records(b.in.off, rtab_base, cq);
#endif
      TL_PMARK(3);
#endif
      if (cq > 1) cluster_sync();  // every rank's records are in every table
    } else {
      if (cq > 1) {  // each rank quantises everything itself; keep the barrier count
        cluster_wait();
        cluster_sync();
        cluster_sync();
      }
      s_badm = 0;
      for (int v = 0; v < b.in.n; ++v) {  // large inputs: one loop per vector
        bool bad;
        const float amax = cta_absmax_f32<CF::kThreads>(b.in.x[v], b.in.K[v], bad, red);
        const double sc = amax > 0.f ? static_cast<double>(amax) / 127.0 : 1.0;  // core.py:128-130
        if (threadIdx.x == 0) s_scale[v] = sc;
        if (bad) s_badm |= 1 << v;
        cta_build_records<FMT, CF::kThreads>(b.in.x[v], b.in.K[v], b.in.C[v], sc,
                                             rtab_base + b.in.off[v]);
      }
    }
#pragma unroll 1
    for (int k = kPre; k < kRing; ++k) {  // the rest of the weight prologue
      if (k < nst) is.issue<FMT, kIssueWeights>(b, min(kStageChunks, n - k * kStageChunks),
                                                ring + k * CF::kStageBytes, lane);
      cp_async_commit();
    }
    __syncthreads();
  } else if constexpr (kTable) {
    // weights of the first ring stages first (no dependence on the glue),
    // then -- once the glue that built the records has completed -- the
    // CTA's records into the table: [C/4][M][4 chunks][record] (a ring
    // stage's token stride), the window [c0, c0 + C) of the segment's input
#pragma unroll 1
    for (int k = 0; k < kRing && k < nst; ++k)
      is.issue<FMT, kIssueWeights>(b, min(kStageChunks, n - k * kStageChunks),
                                   ring + k * CF::kStageBytes, lane);
    // pipelined layers: wait for the glue's records only (its CTAs count in
    // after writing them), not for its completion -- which would also wait
    // for the previous layer's GEMV; that wait moves to the tail, before the
    // previous layer is finalised
    if (b.in.tab_sync)
      sync_consume(b.in.tab_sync + kSyRecs, b.in.tab_sync + kSySeen, b.in.tab_sync_want,
                   (int)gridDim.x);
    else
      asm volatile("griddepcontrol.wait;" ::: "memory");
    {
      int sj = 0;
      const int sc = b.seg_chunk[seg];
      for (int j = 1; j < b.njobs; ++j)
        if (job_at(b, j).start <= sc) sj = j;
      const GemvJob J = job_at(b, sj);
      tab_C = J.C;
      tab_M = J.M;
      constexpr int RU = F::kRecBytes / 16;
      const int units = J.M * J.C * RU;
      for (int u = threadIdx.x; u < units; u += CF::kThreads) {
        const int m = u / (J.C * RU), rem = u - m * J.C * RU;
        const int c = rem / RU, q = rem - c * RU;
        cp_async16_cg(rtab_base + (((c >> 2) * J.M + m) * kStageChunks + (c & 3)) * F::kRecBytes + q * 16,
                      J.rec + ((int64_t)m * J.cin + J.c0 + c) * F::kRecBytes + q * 16);
      }
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    {
      // per-token prefix sums of the window's chunk activation sums (one warp
      // per token, a warp scan per 32 chunks): P[tok][c] = sum of chunks < c
      const int C = tab_C, M = tab_M;
      int32_t *P = reinterpret_cast<int32_t *>(rtab_base + tab_M * ((tab_C + 3) & ~3) * F::kRecBytes);
      for (int tok = warp; tok < M; tok += CF::kWarps) {
        int32_t carry = 0;
        if (lane == 0) P[tok * (C + 1)] = 0;
        for (int c0 = 0; c0 < C; c0 += 32) {
          const int c = c0 + lane;
          int32_t v = 0;
          if (c < C)
            v = *reinterpret_cast<const int32_t *>(
                rtab_base + (((c >> 2) * M + tok) * kStageChunks + (c & 3)) * F::kRecBytes +
                F::kActWords * 4);
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int32_t u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
          }
          if (c < C) P[tok * (C + 1) + c + 1] = carry + v;
          carry += __shfl_sync(0xffffffffu, v, 31);
        }
      }
    }
    __syncthreads();
#pragma unroll 1
    for (int k = 1; k < kRing; ++k) cp_async_commit();  // the ring's group arithmetic
  } else {
    IssueState wis = is;
#pragma unroll 1
    for (int k = 0; k < kRing && k < nst; ++k)
      wis.issue<FMT, kIssueWeights>(b, min(kStageChunks, n - k * kStageChunks),
                                    ring + k * CF::kStageBytes, lane);
    asm volatile("griddepcontrol.wait;" ::: "memory");
#pragma unroll 1
    for (int k = 0; k < kRing; ++k) {
      if (k < nst) is.issue<FMT, kIssueRecords>(b, min(kStageChunks, n - k * kStageChunks),
                                                ring + k * CF::kStageBytes, lane);
      cp_async_commit();  // group 0 also holds every prologue weight copy
    }
  }

  TL_LMARK(1);  // prologue done (fused: inputs quantised)
  // The fused step publishes partial sums only once the previous step's grid
  // has completed: it finalises (reads and zeroes) a workspace that a later
  // launch of the same batch would otherwise accumulate into.
  // The previous step's outputs: right after that wait each thread LOADS its
  // entry of the flat (job, row) space (one per thread when the grid covers
  // it) -- the loads complete while the warp keeps streaming -- and the
  // stores happen at the end, so no load latency sits in the CTA's tail.
  // Two entries per thread (a 148 x 160-thread grid covers 23,680 of the
  // cfg1 step's 32,768): both read-and-resets go out together at the wait.
  constexpr int kFinPer = CF::kFinPer;  // medium CTAs: 148 x 256 x 3 >= the 98,304 cfg4 rows
  int fin_j[kFinPer];
  int64_t fin_k[kFinPer];
  int32_t fin_v[kFinPer];
  double fin_as[kFinPer];
#pragma unroll
  for (int e = 0; e < kFinPer; ++e) fin_j[e] = -1, fin_k[e] = 0, fin_v[e] = 0, fin_as[e] = 0.0;
  auto fin_load = [&]() {
    if constexpr (kFused) {
      if (!b.in.prev_inline) return;
      const int64_t nthreads = (int64_t)gridDim.x * CF::kThreads;
#pragma unroll
      for (int e = 0; e < kFinPer; ++e) {
        int64_t k = (int64_t)gw * 32 + lane + e * nthreads;
        for (int j = 0; j < b.in.prev_njobs; ++j) {
          const FinJob &J = b.in.fin[j];
          const int64_t n = (int64_t)J.M * J.Npad;
          if (k < n) {
            fin_j[e] = j;
            fin_k[e] = k;
            fin_v[e] = atomicExch(J.ws_acc + k, 0);  // read and reset in one L2 operation
            const int m = (int)(k / J.Npad);
            fin_as[e] = J.a_scale ? __ldcg(J.a_scale + m) : 0.0;
            break;
          }
          k -= n;
        }
      }
    }
  };
  // Fused step: a finished tile's partial sums (one int32 per lane) are
  // stashed in registers instead of published, so the warp never stops its
  // weight stream at griddepcontrol.wait; the wait, the previous step's
  // finalize loads and the REDs all happen once the warp's range is done.
  // A range crossing more than kStash tiles waits at the overflow instead.
  constexpr int kStash = kFused ? 4 : 1;
  int ns = 0;
  int32_t st_v[kStash];
  int st_j[kStash], st_t[kStash];
  auto drain = [&]() {
#pragma unroll
    for (int s = 0; s < kStash; ++s)
      if (s < ns) {
#ifndef TB_NO_FLUSH
        red_add_s32(job_at(b, st_j[s]).ws_acc + st_t[s] * kRowTile + lane, st_v[s]);
#endif
      }
    ns = 0;
  };
  // Self-finalising launch (TB_STEP_SELF_FINALIZE, one launch at a time):
  // after publishing a tile's partial sums the warp adds the chunks it
  // contracted to the tile's counter (ws_cnt, behind a fence: the
  // threadfence-reduction pattern); the warp that completes the count (C
  // chunks) reads and resets the sums and writes the tile's outputs with this
  // launch's own scale -- the same expression as the finalize kernel.
  auto tile_done = [&](int j, int t, int cnt) {
    if constexpr (kFused) {
      const GemvJob J = job_at(b, j);
      __threadfence();
      __syncwarp();
      int last = 0;
      if (lane == 0) last = atomicAdd(J.ws_cnt + t, cnt) + cnt == J.C;
      if (!__shfl_sync(0xffffffffu, last, 0)) return;
      __threadfence();
      const int row = t * kRowTile + lane;
      const int32_t v = atomicExch(J.ws_acc + row, 0);
      if (lane == 0) atomicExch(J.ws_cnt + t, 0);
      if (row < J.N) {
        if (J.acc_out) J.acc_out[row] = v;
        const double y = static_cast<double>(v) * J.w_scale * s_scale[J.src];  // core.py:99-101
        if (J.out64) J.out64[row] = y;
        if (J.out32) J.out32[row] = static_cast<float>(y);
      }
    }
  };
  auto flush = [&](Acc<FMT, MT> &acc, int M, int cnt) {
    if constexpr (kTable) {  // the tile's activation sums: chunks [cur.c - cnt, cur.c) of the window
      const int32_t *P = reinterpret_cast<const int32_t *>(
          rtab_base + tab_M * ((tab_C + 3) & ~3) * F::kRecBytes);
      set_csum_from_prefix<FMT, MT>(acc, P, tab_C + 1, cur.c - cnt, cur.c, M);
    }
    if constexpr (kFused) {
      if (b.in.self_fin) {
        flush_tile<FMT, MT>(b, cur.j, cur.t, acc, M, lane);
        tile_done(cur.j, cur.t, cnt);
        return;
      }
      if (!waited) {
        if (ns < kStash) {
          const int32_t v = acc.total(0);
#pragma unroll
          for (int s = 0; s < kStash; ++s)
            if (s == ns) {
              st_v[s] = v;
              st_j[s] = cur.j;
              st_t[s] = cur.t;
            }
          ++ns;
          return;
        }
        asm volatile("griddepcontrol.wait;" ::: "memory");
        waited = true;
        fin_load();
        drain();
      }
    }
    flush_tile<FMT, MT>(b, cur.j, cur.t, acc, M, lane);
  };

  if (n > 0) {
    int C, M, T;  // shape of the current job
    const uint8_t *rtab = nullptr;  // fused: records of the current job's input
    auto load_shape = [&]() {
      const GemvJob J = job_at(b, cur.j);
      C = J.C;
      M = J.M;
      T = (J.end - J.start) / J.C;
      if constexpr (kFused) rtab = rtab_base + b.in.off[J.src] + J.c0 * F::kRecBytes;
      if constexpr (kTable) rtab = rtab_base;  // the segment's window
    };
    // table mode: chunk c's records (token stride = a ring stage's, kStageChunks records)
    auto tab_rec = [&](int c) -> const uint8_t * {
      return rtab + ((c >> 2) * M * kStageChunks + (c & 3)) * F::kRecBytes;
    };
    load_shape();
    Acc<FMT, MT> acc;
    acc.zero();
    int nch = 0;
    for (int k = 0; k < nst; ++k) {
      const int s = k % kRing;
      uint8_t *slot = ring + s * CF::kStageBytes;
      const uint8_t *slot_sign = slot + kStageChunks * kTileChunkBytes;
      const uint8_t *slot_act = slot + kStageChunks * (kTileChunkBytes + F::kSignBytes);
      const int nk = min(kStageChunks, n - k * kStageChunks);
      cp_async_wait<kRing - 1>();  // this lane's copies of stage k have landed
      __syncwarp();                 // ... and every other lane's
      if (k == 0) TL_LMARK(2);
      if (nk == kStageChunks && cur.c + kStageChunks <= C) {
        // fast path: four chunks of the current row tile, fully unrolled
        const uint8_t *act = kFused ? rtab + cur.c * F::kRecBytes : slot_act;
        if constexpr (kPairChunks<FMT, MT>) {
          // unshifted-plane tensor-core path: chunks contracted two at a time
#pragma unroll
          for (int j = 0; j < kStageChunks; j += 2) {
            const uint4 wa = load_wchunk<FMT, MT>(slot + j * kTileChunkBytes, lane);
            const uint4 wb = load_wchunk<FMT, MT>(slot + (j + 1) * kTileChunkBytes, lane);
            process_chunk_pair<MT, kTable>(wa, wb,
                                   kTable ? tab_rec(cur.c + j) : act + j * F::kRecBytes,
                                   kTable ? tab_rec(cur.c + j + 1) : act + (j + 1) * F::kRecBytes,
                                   M, acc);
          }
        } else
#pragma unroll
        for (int j = 0; j < kStageChunks; ++j) {
          const uint4 w4 = load_wchunk<FMT, MT>(slot + j * kTileChunkBytes, lane);
          uint32_t sg = 0;
          if (FMT == TB_TL2)
            sg = *reinterpret_cast<const uint32_t *>(slot_sign + j * kTileSignBytes + lane * 4);
          process_chunk<FMT, MT, kTable>(w4, sg, kTable ? tab_rec(cur.c + j) : act + j * F::kRecBytes, M,
                                 acc, j);
        }
        nch += kStageChunks;
        cur.c += kStageChunks;
      } else {
        for (int j = 0; j < nk; ++j) {
          if (cur.c == C) {  // next row tile (or next job)
            flush(acc, M, nch);
            nch = 0;
            acc.zero();
            cur.c = 0;
            if (++cur.t >= T) {
              ++cur.j;
              cur.t = 0;
              load_shape();
            }
          }
          const uint4 w4 = load_wchunk<FMT, MT>(slot + j * kTileChunkBytes, lane);
          uint32_t sg = 0;
          if (FMT == TB_TL2)
            sg = *reinterpret_cast<const uint32_t *>(slot_sign + j * kTileSignBytes + lane * 4);
          const uint8_t *act = kTable ? tab_rec(cur.c)
                               : kFused ? rtab + cur.c * F::kRecBytes : slot_act + j * F::kRecBytes;
          process_chunk<FMT, MT, kTable>(w4, sg, act, M, acc);
          ++nch;
          ++cur.c;
        }
      }
      if (cur.c == C && k + 1 < nst) {  // tile finished exactly at a stage boundary
        flush(acc, M, nch);
        nch = 0;
        acc.zero();
        cur.c = 0;
        if (++cur.t >= T) {
          ++cur.j;
          cur.t = 0;
          load_shape();
        }
      }
      __syncwarp();  // every lane is done reading the slot before it is refilled
      if (k + kRing < nst)
        is.issue<FMT, kIssueMain>(b, min(kStageChunks, n - (k + kRing) * kStageChunks), slot, lane);
      cp_async_commit();
    }
    TL_LMARK(3);
    if (nch > 0) flush(acc, M, nch);
  }
  TL_MARK(4);
  if constexpr (kTable) {
    // the previous batch's finalize (its grid completed before the glue this
    // launch waited on): every thread of the grid takes a strided share of
    // the flat (job, token, row) space, off the critical path of the next
    // launch's weight stream
    // (pipelined layers: the glue's completion -- it exits only after the
    // previous GEMV completed -- is awaited here; every launch of the chain
    // waits before it exits, so completion stays transitive)
    if (b.in.tab_sync) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (b.in.prev_inline) {
      // the jobs staged in shared memory (kernel-parameter loads with a
      // per-lane index serialise); 8 entries per thread per round, every
      // load issued before any use
      __shared__ FinJob s_fin[kMaxInlineFin];
      __shared__ int64_t s_pre[kMaxInlineFin + 1];
      if ((int)threadIdx.x < b.in.prev_njobs) s_fin[threadIdx.x] = b.in.fin[threadIdx.x];
      __syncthreads();
      if (threadIdx.x == 0) {
        s_pre[0] = 0;
        for (int j = 0; j < b.in.prev_njobs; ++j)
          s_pre[j + 1] = s_pre[j] + (int64_t)s_fin[j].M * s_fin[j].Npad;
      }
      __syncthreads();
      const int nj = b.in.prev_njobs;
      // warp-uniform runs of 32 entries (Npad is a multiple of 32: a run never
      // straddles a token row), lane = row: the job search and the token
      // index are uniform, 4 runs' loads in flight per warp
      const int64_t nruns = s_pre[nj] / 32;
      const int64_t nwarps = (int64_t)gridDim.x * CF::kWarps;
      for (int64_t r0 = gw; r0 < nruns; r0 += 4 * nwarps) {
        int32_t v[4];
        int jj[4], mm[4], rw[4];
        double as[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t r = r0 + u * nwarps;
          jj[u] = -1;
          if (r < nruns) {
            const int64_t e = r * 32;
            int j = 0;
            while (j + 1 < nj && s_pre[j + 1] <= e) ++j;
            const FinJob &J = s_fin[j];
            const int k = (int)(e - s_pre[j]);  // < 2^31: M * Npad of one job
            const int m = k / J.Npad;
            jj[u] = j;
            mm[u] = m;
            rw[u] = k - m * J.Npad + lane;
            int32_t *w = J.ws_acc + k + lane;
            v[u] = atomicExch(w, 0);  // read and reset (a plain store would wait for the load)
            as[u] = J.a_scale ? __ldcg(J.a_scale + m) : 0.0;
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (jj[u] < 0) continue;
          const FinJob &J = s_fin[jj[u]];
          if (rw[u] < J.N) {
            const int64_t o = (int64_t)mm[u] * J.N + rw[u];
            if (J.acc_out) J.acc_out[o] = v[u];
            const double y = static_cast<double>(v[u]) * J.w_scale * as[u];  // core.py:99-101
            if (J.out64) J.out64[o] = y;
            if (J.out32) J.out32[o] = static_cast<float>(y);
          }
        }
      }
    }
  }
  if constexpr (kFused) {
    if (!waited && !b.in.no_wait) {
#ifndef TB_NO_TAILWAIT  // profiling variant (results invalid): no chain serialisation
      asm volatile("griddepcontrol.wait;" ::: "memory");
      fin_load();
#endif
    }
    drain();
    // this step's scales (read by whoever finalises this batch), then the
    // previous step's outputs: its grid has completed, its sums are visible
    if (threadIdx.x < b.in.n && b.in.writer[threadIdx.x] == (int)blockIdx.x) {
      *b.in.scale[threadIdx.x] = s_scale[threadIdx.x];
      // plain store (this launch's verdict): the flag may live in mapped host memory
      const int bad = (s_badm >> threadIdx.x) & 1;
      if (b.in.flag[threadIdx.x] && (bad || !b.in.sticky_flags)) *b.in.flag[threadIdx.x] = bad;
    }
    if (b.in.prev_inline) {
#ifndef TB_NO_PREVFIN  // profiling variant: skip the previous step's finalize
#pragma unroll
      for (int e = 0; e < kFinPer; ++e) {
        if (fin_j[e] < 0) continue;  // the entries read (and reset) at the wait: stores only
        const FinJob &J = b.in.fin[fin_j[e]];
        const int m = (int)(fin_k[e] / J.Npad), row = (int)(fin_k[e] - (int64_t)m * J.Npad);
        if (row < J.N) {
          const int64_t o = (int64_t)m * J.N + row;
          if (J.acc_out) J.acc_out[o] = fin_v[e];
          const double y = static_cast<double>(fin_v[e]) * J.w_scale * fin_as[e];  // core.py:99-101
          if (J.out64) J.out64[o] = y;
          if (J.out32) J.out32[o] = static_cast<float>(y);
        }
      }
      // entries beyond kFinPer per thread of the grid (large previous steps)
      const int64_t nthreads = (int64_t)gridDim.x * CF::kThreads;
      int64_t total = 0;
      for (int j = 0; j < b.in.prev_njobs; ++j) total += (int64_t)b.in.fin[j].M * b.in.fin[j].Npad;
      if (total > kFinPer * nthreads) {
        finalize_fin_range(b.in.fin, b.in.prev_njobs, kFinPer * nthreads + (int64_t)gw * 32 + lane,
                           nthreads);
      }
#endif
    } else {
      for (int j = 0; j < b.in.prev_njobs; ++j) finalize_one(b.in.prev[j], blockIdx.x, gridDim.x);
    }
  }
}

// --------------------------------------------------------------------------
// host side
// --------------------------------------------------------------------------

// The finalize kernel is launched as a programmatic dependent of the GEMV, so
// its launch latency overlaps the GEMV (it waits in griddepcontrol.wait).
static int launch_finalize(const GemvBatch &b, cudaStream_t s) {
  const int threads = 256;
  // one element per thread: every job's accumulators are read concurrently
  const int parts = (int)std::max<int64_t>(1, ceil_div(b.max_entries, threads));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(parts, b.njobs);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, gemv_finalize_kernel, b) != cudaSuccess) return TB_ERR_CUDA;
  return TB_OK;
}

template <int FMT, int MT, int FU = 0>
static int launch_tgemv(GemvBatch &b, cudaStream_t s, int rec_tab_bytes = 0) {
  using CF = Cfg<FMT, MT, FU>;
  constexpr bool kFused = CF::kFused;
  if (kFused && rec_tab_bytes > CF::kRecTabBytes) return TB_ERR_UNSUPPORTED;
  static int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    if (cudaFuncSetAttribute(tgemv_kernel<FMT, MT, FU>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, CF::kSmem) != cudaSuccess)
      return TB_ERR_CUDA;
    if (kFused && cudaFuncSetAttribute(tgemv_kernel<FMT, MT, FU, kStepCQ>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       CF::kSmem) != cudaSuccess)
      return TB_ERR_CUDA;
    configured_dev = dev;
  }
  // spread over every SM (latency-bound sizes want the parallelism), one CTA
  // per SM, at least one chunk per warp
  // at least TB_MIN_WARP_CHUNKS chunks (16 KB) per warp: a small launch then
  // takes a fraction of the SMs, and consecutive launches of a chain run side
  // by side under programmatic dependent launch instead of each paying its
  // fixed costs on every SM (4 MB cfg0 GEMV: 3.7 -> 2.4 us per launch)
#ifndef TB_MIN_WARP_CHUNKS
#define TB_MIN_WARP_CHUNKS 32
#endif
  // independent launches (TB_STEP_INDEPENDENT) overlap many at a time: fewer,
  // fatter CTAs each (4096 x 4096: 25 CTAs, 1.01 us per launch against 1.31
  // at 50 and 1.98 at 100)
#ifndef TB_MIN_WARP_CHUNKS_IND
#define TB_MIN_WARP_CHUNKS_IND 64
#endif
  int64_t want = ceil_div(b.total, (int64_t)CF::kWarps *
                                       (kFused && b.in.no_wait ? TB_MIN_WARP_CHUNKS_IND
                                                               : TB_MIN_WARP_CHUNKS));
  if (kFused && b.in.prev_inline) {
    // ... but enough threads that the previous step's outputs are finalised
    // at kFinPer entries per thread, not in the serial tail loop
    int64_t prev = 0;
    for (int j = 0; j < b.in.prev_njobs; ++j) prev += (int64_t)b.in.fin[j].M * b.in.fin[j].Npad;
    want = std::max<int64_t>(want, ceil_div(prev, (int64_t)CF::kThreads * CF::kFinPer));
  }
  if (CF::kTable && b.table == nullptr) {  // at least one CTA per table segment
    int runs = 0;
    for (int j = 0; j < b.njobs; ++j)
      if (j == 0 || b.jobs[j].rec != b.jobs[j - 1].rec || b.jobs[j].c0 != b.jobs[j - 1].c0) ++runs;
    want = std::max<int64_t>(want, runs);
  }
  // (table mode: two CTAs per SM.  One per SM and launch -- the resident pair
  // then belongs to consecutive layers, one streaming while the other fills
  // or finalises -- moves data at the M = 1 rate (57.9 us per cfg4 layer with
  // the MMAs compiled out) but leaves a layer only 8 warps per SM to contract
  // with, and the ldmatrix -> LOP -> IMMA chains are latency bound: 106 us)
#ifndef TB_TABLE_GRID_MULT
#define TB_TABLE_GRID_MULT 2
#endif
  int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>((int64_t)sm_count_cached() * (CF::kTable ? TB_TABLE_GRID_MULT : 1), want));
  if (kFused && kStepCQ > 1 && grid > kStepCQ) grid -= grid % kStepCQ;  // whole CTA clusters
  const int nw = grid * CF::kWarps;
  // whole ring stages per warp: with C % 4 == 0 (I2_S / TL1 at K % 256 == 0)
  // no stage straddles a row tile, so the main loop stays on its fast path
  b.unit = b.total >= (int64_t)nw * kStageChunks ? kStageChunks : 1;
  // segments: one per run of same-input jobs (fused step), CTAs in
  // proportion to their chunks; otherwise one segment
  b.nseg = 1;
  b.seg_chunk[0] = 0;
  if (CF::kTable && (b.table != nullptr || rec_tab_bytes <= 0)) return TB_ERR_ARGUMENT;
  if ((kFused || CF::kTable) && b.table == nullptr) {
    // fused step: runs of jobs on the same input vector; table mode: runs of
    // jobs on the same records AND K-window (one table per CTA)
    int ns = 0, starts[kMaxInlineJobs + 1];
    for (int j = 0; j < b.njobs; ++j)
      if (j == 0 || b.jobs[j].src != b.jobs[j - 1].src ||
          (CF::kTable && (b.jobs[j].rec != b.jobs[j - 1].rec || b.jobs[j].c0 != b.jobs[j - 1].c0)))
        starts[ns++] = b.jobs[j].start;
    if (CF::kTable && (ns > kMaxSegs || ns > grid)) return TB_ERR_UNSUPPORTED;
    if (ns <= kMaxSegs && ns <= grid && ns > 1) {
      b.nseg = ns;
      for (int q = 0; q < ns; ++q) b.seg_chunk[q] = starts[q];
    }
  }
  b.seg_chunk[b.nseg] = b.total;
  // fused step: clusters of Q CTAs share the quantisation (segments in whole clusters)
  int Q = 1;
  if (kFused && kStepCQ > 1 && grid % kStepCQ == 0 && grid >= kStepCQ * b.nseg) Q = kStepCQ;
  {
    int assigned = 0;
    for (int q = 0; q < b.nseg; ++q) {
      const int64_t nq = b.seg_chunk[q + 1] - b.seg_chunk[q];
      int c = q + 1 == b.nseg ? grid - assigned
                              : Q * (int)std::llround((double)grid * nq / (double)b.total / Q);
      c = std::max(Q, std::min(c, grid - assigned - Q * (b.nseg - 1 - q)));
      b.seg_cta[q] = assigned;
      assigned += c;
      const int64_t sw = (int64_t)c * CF::kWarps;
      b.seg_base[q] = (int)((nq / b.unit) / sw);
      b.seg_rem[q] = (int)((nq / b.unit) % sw);
      b.seg_tail[q] = (int)(nq % b.unit);
    }
    b.seg_cta[b.nseg] = grid;
  }
  if (kFused) {
    // which inputs each CTA's chunk range touches (needs the jobs on the host)
    const int all = (1 << b.in.n) - 1;
    for (int v = 0; v < kMaxStepInputs; ++v) b.in.writer[v] = 0;
    if (b.table == nullptr && grid <= kMaxNeedCtas) {
      int seen = 0;
      for (int c = 0; c < grid; ++c) {
        int q = 0;
        while (q + 1 < b.nseg && c >= b.seg_cta[q + 1]) ++q;
        const int64_t w0 = (int64_t)(c - b.seg_cta[q]) * CF::kWarps, w1 = w0 + CF::kWarps;
        const int64_t lo = b.seg_chunk[q] + b.unit * (w0 * b.seg_base[q] + std::min<int64_t>(w0, b.seg_rem[q]));
        const int64_t hi = b.seg_chunk[q] + b.unit * (w1 * b.seg_base[q] + std::min<int64_t>(w1, b.seg_rem[q])) +
                           (c + 1 == b.seg_cta[q + 1] ? b.seg_tail[q] : 0);
        int m = 0;
        for (int j = 0; j < b.njobs; ++j)
          if (b.jobs[j].start < hi && b.jobs[j].end > lo) m |= 1 << b.jobs[j].src;
        b.in.need[c] = (uint8_t)m;
        for (int v = 0; v < b.in.n; ++v)
          if (((m >> v) & 1) && !((seen >> v) & 1)) b.in.writer[v] = (int16_t)c;
        seen |= m;
      }
      b.in.need[0] |= (uint8_t)(all & ~seen);  // unused inputs: CTA 0 still publishes a scale
      for (int c0 = 0; c0 < grid; c0 += Q) {  // one quantisation per cluster: the union
        int m = 0;
        for (int c = c0; c < c0 + Q; ++c) m |= b.in.need[c];
        for (int c = c0; c < c0 + Q; ++c) b.in.need[c] = (uint8_t)m;
      }
    } else {
      for (int c = 0; c < kMaxNeedCtas; ++c) b.in.need[c] = (uint8_t)all;
    }
  }
  // programmatic dependent launch: the prologue (job lookup, first weight
  // stages) overlaps the tail of the kernel that produced the records
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(CF::kThreads);
  cfg.dynamicSmemBytes = (kFused || CF::kTable) ? CF::kRingBytes + rec_tab_bytes : CF::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = Q;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = Q > 1 ? 2 : 1;
  if (cudaLaunchKernelEx(&cfg, Q > 1 ? tgemv_kernel<FMT, MT, FU, kStepCQ> : tgemv_kernel<FMT, MT, FU>,
                         b) != cudaSuccess)
    return TB_ERR_CUDA;
  return (kFused || b.defer_finalize) ? TB_OK : launch_finalize(b, s);
}

template <int FMT>
static int dispatch_m(GemvBatch &b, int maxM, cudaStream_t s) {
  if (maxM <= 1) return launch_tgemv<FMT, 1>(b, s);
  if (maxM <= 2) return launch_tgemv<FMT, 2>(b, s);
  if (maxM <= 4) return launch_tgemv<FMT, 4>(b, s);
  if (maxM <= 8) return launch_tgemv<FMT, 8>(b, s);
  return launch_tgemv<FMT, 16>(b, s);
}

static int rec_bytes_of(int fmt) {
  return fmt == TB_TL2 ? Fmt<TB_TL2>::kRecBytes : Fmt<TB_I2S>::kRecBytes;
}

static int64_t ws_counts_bytes(int64_t rows) {
  const int64_t T = ceil_div(rows, kRowTile);
  return pad_up((16 * T * kRowTile + T) * (int64_t)sizeof(int32_t), 256);
}

// Fill one job; returns TB_OK or an error.
static int make_job(int fmt, const uint8_t *tiled, const uint8_t *tiled_sign, int64_t rows,
                    int64_t cols, const uint8_t *rec, int64_t M, const double *a_scale,
                    double w_scale, void *workspace, int32_t *acc_out, double *out64,
                    float *out32, int64_t start, GemvJob &J, bool fused = false) {
  if (!tiled || (!rec && !fused) || !workspace || rows < 1 || cols < 1 || M < 1 || M > 16 ||
      (fmt == TB_TL2 && !tiled_sign) || ((out64 || out32) && !a_scale) ||
      (reinterpret_cast<uintptr_t>(rec) & 15) || (reinterpret_cast<uintptr_t>(tiled) & 15))
    return TB_ERR_ARGUMENT;
  const int64_t C = ceil_div(ref_row_bytes(fmt, cols), kChunkBytes);
  const int64_t T = ceil_div(rows, kRowTile);
  if (start + T * C >= ((int64_t)1 << 31)) return TB_ERR_UNSUPPORTED;
  J.wmain = tiled;
  J.wsign = tiled_sign;
  J.rec = rec;
  J.a_scale = a_scale;
  J.w_scale = w_scale;
  J.ws_acc = static_cast<int32_t *>(workspace);
  J.ws_cnt = J.ws_acc + 16 * T * kRowTile;
  J.acc_out = acc_out;
  J.out64 = out64;
  J.out32 = out32;
  J.N = (int)rows;
  J.Npad = (int)(T * kRowTile);
  J.C = (int)C;
  J.M = (int)M;
  J.start = (int)start;
  J.end = (int)(start + T * C);
  J.src = 0;
  J.c0 = 0;
  J.cin = (int)C;
  J.fin_m = (acc_out || out64 || out32) ? (int)M : 0;
  return TB_OK;
}

static int launch_batch(int fmt, GemvBatch &b, int maxM, cudaStream_t s) {
  if (fmt == TB_I2S) return dispatch_m<TB_I2S>(b, maxM, s);
  if (fmt == TB_TL1) return dispatch_m<TB_I2S>(b, maxM, s);  // same tiled codes (pack.cu)
  if (fmt == TB_TL2) return dispatch_m<TB_TL2>(b, maxM, s);
  return TB_ERR_ARGUMENT;
}

static int launch_step(int fmt, GemvBatch &b, int rec_tab_bytes, bool isolated, cudaStream_t s) {
  // small CTAs, several per SM (chained steps overlap) when the record tables
  // allow it; one 16-warp CTA per SM for big tables or an isolated launch
  const bool small = !isolated && rec_tab_bytes <= Cfg<TB_I2S, 1, 1>::kRecTabBytes;  // 40 KB
  const bool medium = !isolated && rec_tab_bytes <= Cfg<TB_I2S, 1, 3>::kRecTabBytes;  // 56 KB
  if (fmt == TB_I2S || fmt == TB_TL1)  // TL1 tiles hold I2_S codes
    return small    ? launch_tgemv<TB_I2S, 1, 1>(b, s, rec_tab_bytes)
           : medium ? launch_tgemv<TB_I2S, 1, 3>(b, s, rec_tab_bytes)
                    : launch_tgemv<TB_I2S, 1, 2>(b, s, rec_tab_bytes);
  if (fmt == TB_TL2)
    return small ? launch_tgemv<TB_TL2, 1, 1>(b, s, rec_tab_bytes)
                 : launch_tgemv<TB_TL2, 1, 2>(b, s, rec_tab_bytes);
  return TB_ERR_ARGUMENT;
}

}  // namespace tb

using namespace tb;

extern "C" int64_t tb_act_records_bytes(int fmt, int64_t M, int64_t cols) {
  if (M < 1 || cols < 1 || fmt < TB_I2S || fmt > TB_TL2) return -1;
  const int64_t C = ceil_div(ref_row_bytes(fmt, cols), kChunkBytes);
  return M * C * rec_bytes_of(fmt);
}

extern "C" int tb_prep_activations(int fmt, const int8_t *act, int64_t M, int64_t ld_act,
                                   int64_t act_len, int64_t cols, uint8_t *rec, void *stream) {
  if (!act || !rec || M < 1 || M > 16 || cols < 1 || act_len < 0 || act_len > ld_act ||
      fmt < TB_I2S || fmt > TB_TL2 || (reinterpret_cast<uintptr_t>(rec) & 15))
    return TB_ERR_ARGUMENT;
  const int64_t C = ceil_div(ref_row_bytes(fmt, cols), kChunkBytes);
  const int64_t n4 = M * C * 4;
  const int64_t cap = (int64_t)sm_count_cached() * 8;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cap, ceil_div(n4, 256)));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (fmt == TB_I2S)
    act_prep_kernel<TB_I2S><<<grid, 256, 0, s>>>(act, (int)M, ld_act, act_len, (int)C, rec);
  else if (fmt == TB_TL1)
    act_prep_kernel<TB_I2S><<<grid, 256, 0, s>>>(act, (int)M, ld_act, act_len, (int)C, rec);
  else
    act_prep_kernel<TB_TL2><<<grid, 256, 0, s>>>(act, (int)M, ld_act, act_len, (int)C, rec);
  TB_CHECK_LAUNCH();
  return TB_OK;
}

template <int FMT, typename T>
static cudaError_t launch_qrec(const T *x, int64_t M, int64_t K, int64_t ldx, int8_t *q,
                               int64_t ldq, double *scale, int C, uint8_t *rec, int32_t *flag,
                               cudaStream_t s) {
  // one 8-CTA cluster per token (portable cluster size), PDL-launched
  const int ncta = std::max(1, std::min(8, C));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ncta, (unsigned)M);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = ncta;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, quantize_records_kernel<FMT, T, 256>, x, K, ldx, q, ldq, scale,
                            C, rec, flag);
}

template <typename T>
static int qrec_impl(int fmt, const T *x, int64_t M, int64_t K, int64_t ldx, int8_t *q,
                     int64_t ldq, double *scale, uint8_t *rec, int32_t *flag, void *stream) {
  if (!x || !scale || !rec || M < 1 || K < 1 || ldx < K || (q && ldq < K) || fmt < TB_I2S ||
      fmt > TB_TL2 || (reinterpret_cast<uintptr_t>(rec) & 15))
    return TB_ERR_ARGUMENT;
  const int C = (int)ceil_div(ref_row_bytes(fmt, K), kChunkBytes);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (fmt == TB_I2S) e = launch_qrec<TB_I2S>(x, M, K, ldx, q, ldq, scale, C, rec, flag, s);
  else if (fmt == TB_TL1) e = launch_qrec<TB_I2S>(x, M, K, ldx, q, ldq, scale, C, rec, flag, s);
  else e = launch_qrec<TB_TL2>(x, M, K, ldx, q, ldq, scale, C, rec, flag, s);
  return e == cudaSuccess ? TB_OK : TB_ERR_CUDA;
}

extern "C" int tb_quantize_records_f32(int fmt, const float *x, int64_t M, int64_t K, int64_t ldx,
                                       int8_t *q, int64_t ldq, double *scale, uint8_t *rec,
                                       int32_t *flag, void *stream) {
  return qrec_impl(fmt, x, M, K, ldx, q, ldq, scale, rec, flag, stream);
}

extern "C" int tb_quantize_records_f64(int fmt, const double *x, int64_t M, int64_t K,
                                       int64_t ldx, int8_t *q, int64_t ldq, double *scale,
                                       uint8_t *rec, int32_t *flag, void *stream) {
  return qrec_impl(fmt, x, M, K, ldx, q, ldq, scale, rec, flag, stream);
}

extern "C" int64_t tb_gemv_workspace_bytes(int fmt, int64_t rows, int64_t cols) {
  if (rows < 1 || cols < 1 || fmt < TB_I2S || fmt > TB_TL2) return -1;
  return ws_counts_bytes(rows) + tb_act_records_bytes(fmt, 16, cols);
}

extern "C" int tb_gemv_records(int fmt, const uint8_t *tiled, const uint8_t *tiled_sign,
                               int64_t rows, int64_t cols, const uint8_t *rec, int64_t M,
                               const double *a_scale, double w_scale, void *workspace,
                               int32_t *acc_out, double *out64, float *out32, void *stream) {
  if (fmt < TB_I2S || fmt > TB_TL2) return TB_ERR_ARGUMENT;
  GemvBatch b{};
  int st = make_job(fmt, tiled, tiled_sign, rows, cols, rec, M, a_scale, w_scale, workspace,
                    acc_out, out64, out32, 0, b.jobs[0]);
  if (st != TB_OK) return st;
  b.njobs = 1;
  b.total = b.jobs[0].end;
  b.max_entries = b.jobs[0].M * b.jobs[0].Npad;
  return launch_batch(fmt, b, (int)M, static_cast<cudaStream_t>(stream));
}

extern "C" int64_t tb_gemv_job_bytes(void) { return (int64_t)sizeof(GemvJob); }

extern "C" int tb_gemv_batch_prepare(int fmt, int64_t njobs, const tb_gemv_desc *descs,
                                     void *table_host, int64_t *total_chunks, int32_t *max_m,
                                     int64_t *max_entries) {
  if (fmt < TB_I2S || fmt > TB_TL2 || njobs < 1 || !descs || !table_host || !total_chunks ||
      !max_m || !max_entries)
    return TB_ERR_ARGUMENT;
  GemvJob *host = static_cast<GemvJob *>(table_host);
  int64_t start = 0;
  int maxM = 1;
  int64_t maxE = 1;
  for (int64_t j = 0; j < njobs; ++j) {
    const tb_gemv_desc &d = descs[j];
    int st = make_job(fmt, d.tiled, d.tiled_sign, d.rows, d.cols, d.rec, d.M, d.a_scale,
                      d.w_scale, d.workspace, d.acc_out, d.out64, d.out32, start, host[j]);
    if (st != TB_OK) return st;
    start = host[j].end;
    maxM = std::max(maxM, (int)d.M);
    maxE = std::max(maxE, (int64_t)host[j].M * host[j].Npad);
  }
  *total_chunks = start;
  *max_m = maxM;
  *max_entries = maxE;
  return TB_OK;
}

extern "C" int tb_gemv_batch_launch(int fmt, const void *table_device, int64_t njobs,
                                    int64_t total_chunks, int32_t max_m, int64_t max_entries,
                                    int32_t finalize, void *stream) {
  if (fmt < TB_I2S || fmt > TB_TL2 || njobs < 1 || !table_device || total_chunks < 1 ||
      total_chunks >= ((int64_t)1 << 31) || max_m < 1 || max_m > 16 || max_entries < 1 ||
      max_entries >= ((int64_t)1 << 31))
    return TB_ERR_ARGUMENT;
  GemvBatch b{};
  b.table = static_cast<const GemvJob *>(table_device);
  b.njobs = (int)njobs;
  b.total = (int)total_chunks;
  b.defer_finalize = finalize ? 0 : 1;
  b.max_entries = (int)max_entries;
  return launch_batch(fmt, b, max_m, static_cast<cudaStream_t>(stream));
}

// As tb_gemv_batch_prepare, plus K-windows: job j contracts record columns
// [col0[j], col0[j] + descs[j].cols) of records built for rec_cols[j] columns
// (col0 a multiple of one record chunk; NULL arrays = whole records).
extern "C" int tb_gemv_batch_prepare_cols(int fmt, int64_t njobs, const tb_gemv_desc *descs,
                                          const int64_t *col0, const int64_t *rec_cols,
                                          void *table_host, int64_t *total_chunks,
                                          int32_t *max_m, int64_t *max_entries) {
  int st = tb_gemv_batch_prepare(fmt, njobs, descs, table_host, total_chunks, max_m, max_entries);
  if (st != TB_OK || (!col0 && !rec_cols)) return st;
  const int64_t chunk_w = fmt == TB_TL2 ? 96 : 64;
  GemvJob *host = static_cast<GemvJob *>(table_host);
  for (int64_t j = 0; j < njobs; ++j) {
    const int64_t c0 = col0 ? col0[j] : 0;
    const int64_t rc = rec_cols ? rec_cols[j] : descs[j].cols;
    if (c0 < 0 || c0 % chunk_w || c0 + descs[j].cols > rc) return TB_ERR_ARGUMENT;
    host[j].c0 = (int)(c0 / chunk_w);
    host[j].cin = (int)ceil_div(ref_row_bytes(fmt, rc), kChunkBytes);
  }
  return TB_OK;
}

static std::atomic<int64_t> g_table_launches{0};
extern "C" int64_t tb_gemv_table_launches(void) { return g_table_launches.load(); }

// As tb_gemv_batch_launch, with the host copy of a small job table (<= 10
// jobs): the jobs ride in the kernel parameters, and for 2 <= M tokens each
// CTA keeps its segment's records (one records buffer and K-window) in one
// shared-memory table instead of staging them per warp and ring stage.
static int batch_launch_inline(int fmt, const void *table_device, const void *table_host,
                               int64_t njobs, int64_t total_chunks, int32_t max_m,
                               int64_t max_entries, int32_t finalize,
                               const void *prev_table_host, int64_t prev_njobs,
                               int32_t *sync, int32_t glue_ctas, void *stream);
extern "C" int tb_gemv_batch_launch_inline(int fmt, const void *table_device,
                                           const void *table_host, int64_t njobs,
                                           int64_t total_chunks, int32_t max_m,
                                           int64_t max_entries, int32_t finalize,
                                           const void *prev_table_host, int64_t prev_njobs,
                                           void *stream) {
  return batch_launch_inline(fmt, table_device, table_host, njobs, total_chunks, max_m,
                             max_entries, finalize, prev_table_host, prev_njobs, nullptr, 0,
                             stream);
}

// The GEMV of a pipelined M > 1 layer: as tb_gemv_batch_launch_inline in
// records-table mode (anything else is TB_ERR_UNSUPPORTED: no silent
// fallback, the glue counts on its consumer), but the table fill waits for
// the glue's records through `sync` (the layer's block, glue_ctas from
// tb_step_glue_sync) instead of for the glue's completion, so the launch
// streams while the previous layer's GEMV is still draining; the previous
// batch is finalised in the tail, after griddepcontrol.wait.
extern "C" int tb_gemv_batch_launch_sync(int fmt, const void *table_device,
                                         const void *table_host, int64_t njobs,
                                         int64_t total_chunks, int32_t max_m,
                                         int64_t max_entries, const void *prev_table_host,
                                         int64_t prev_njobs, int32_t *sync, int32_t glue_ctas,
                                         void *stream) {
  if (!sync || glue_ctas < 1) return TB_ERR_ARGUMENT;
  return batch_launch_inline(fmt, table_device, table_host, njobs, total_chunks, max_m,
                             max_entries, 0, prev_table_host, prev_njobs, sync, glue_ctas, stream);
}

static int batch_launch_inline(int fmt, const void *table_device, const void *table_host,
                               int64_t njobs, int64_t total_chunks, int32_t max_m,
                               int64_t max_entries, int32_t finalize,
                               const void *prev_table_host, int64_t prev_njobs,
                               int32_t *sync, int32_t glue_ctas, void *stream) {
  if (!table_host || njobs > kMaxInlineJobs || max_m < 2) {
    if (prev_njobs > 0 || sync) return TB_ERR_UNSUPPORTED;  // the caller finalises the previous batch
    return tb_gemv_batch_launch(fmt, table_device, njobs, total_chunks, max_m, max_entries,
                                finalize, stream);
  }
  if (prev_njobs > kMaxInlineJobs) return TB_ERR_UNSUPPORTED;
  if (fmt < TB_I2S || fmt > TB_TL2 || njobs < 1 || !table_device || total_chunks < 1 ||
      total_chunks >= ((int64_t)1 << 31) || max_m > 16 || max_entries < 1 ||
      max_entries >= ((int64_t)1 << 31))
    return TB_ERR_ARGUMENT;
  GemvBatch b{};
  const GemvJob *h = static_cast<const GemvJob *>(table_host);
  int64_t tab = 0;
  for (int j = 0; j < njobs; ++j) {
    b.jobs[j] = h[j];
    // the segment's records + its per-token prefix sums of the chunk sums
    tab = std::max<int64_t>(tab, (int64_t)h[j].M * pad_up(h[j].C, kStageChunks) * rec_bytes_of(fmt) +
                                     pad_up((int64_t)h[j].M * (h[j].C + 1) * 4, 16));
  }
  b.table = nullptr;
  b.njobs = (int)njobs;
  b.total = (int)total_chunks;
  b.defer_finalize = finalize ? 0 : 1;
  b.max_entries = (int)max_entries;
  if (prev_njobs > 0) {  // finalise the previous batch in this launch's tail
    if (!prev_table_host) return TB_ERR_ARGUMENT;
    const GemvJob *ph = static_cast<const GemvJob *>(prev_table_host);
    int nf = 0;
    for (int j = 0; j < prev_njobs; ++j) {
      if (ph[j].fin_m == 0) continue;  // K-windows finalised through another job
      if (nf == kMaxInlineFin) return TB_ERR_UNSUPPORTED;
      FinJob &F = b.in.fin[nf++];
      F.ws_acc = ph[j].ws_acc;
      F.acc_out = ph[j].acc_out;
      F.out64 = ph[j].out64;
      F.out32 = ph[j].out32;
      F.a_scale = ph[j].a_scale;
      F.w_scale = ph[j].w_scale;
      F.N = ph[j].N;
      F.Npad = ph[j].Npad;
      F.M = ph[j].fin_m;
    }
    b.in.prev_njobs = nf;
    b.in.prev_inline = nf > 0 ? 1 : 0;
  }
  b.in.tab_sync = sync;
  b.in.tab_sync_want = glue_ctas;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int st = TB_ERR_UNSUPPORTED;
  if (tab <= Cfg<TB_I2S, 8, 4>::kRecTabBytes && max_m <= 8) {
    if (fmt == TB_I2S || fmt == TB_TL1)
      st = max_m <= 2 ? launch_tgemv<TB_I2S, 2, 4>(b, s, (int)tab)
           : max_m <= 4 ? launch_tgemv<TB_I2S, 4, 4>(b, s, (int)tab)
                        : launch_tgemv<TB_I2S, 8, 4>(b, s, (int)tab);
    if (st == TB_OK) g_table_launches.fetch_add(1, std::memory_order_relaxed);
    if (st == TB_OK || st == TB_ERR_CUDA) return st;
  }
  if (sync) return TB_ERR_UNSUPPORTED;
  // too large a table or too many segments: the records path, after a
  // separate finalize launch of the previous batch
  if (prev_njobs > 0) {
    GemvBatch pb{};
    const GemvJob *ph = static_cast<const GemvJob *>(prev_table_host);
    if (prev_njobs > kMaxInlineJobs) return TB_ERR_UNSUPPORTED;
    int64_t pe = 1;
    for (int j = 0; j < prev_njobs; ++j) {
      pb.jobs[j] = ph[j];
      pe = std::max<int64_t>(pe, (int64_t)ph[j].fin_m * ph[j].Npad);
    }
    pb.table = nullptr;
    pb.njobs = (int)prev_njobs;
    pb.max_entries = (int)pe;
    st = launch_finalize(pb, s);
    if (st != TB_OK) return st;
  }
  b.in = StepInputs{};
  b.table = static_cast<const GemvJob *>(table_device);
  return launch_batch(fmt, b, max_m, s);
}

extern "C" int tb_gemv_step_prepare_cols(int fmt, int64_t njobs, const tb_gemv_desc *descs,
                                         const int32_t *src, const int64_t *col0,
                                         int64_t ninputs, const int64_t *input_k,
                                         void *table_host, int64_t *total_chunks,
                                         int64_t *max_entries) {
  if (fmt < TB_I2S || fmt > TB_TL2 || njobs < 1 || !descs || !src || !input_k ||
      ninputs < 1 || ninputs > kMaxStepInputs || !table_host || !total_chunks || !max_entries)
    return TB_ERR_ARGUMENT;
  // one record chunk = 16 packed bytes = 64 I2_S / TL1 weights, 96 TL2 weights
  const int64_t chunk_w = fmt == TB_TL2 ? 96 : 64;
  GemvJob *host = static_cast<GemvJob *>(table_host);
  int64_t start = 0, maxE = 1;
  for (int64_t j = 0; j < njobs; ++j) {
    const tb_gemv_desc &d = descs[j];
    const int64_t c0 = col0 ? col0[j] : 0;
    if (src[j] < 0 || src[j] >= ninputs || d.M != 1 || c0 < 0 || c0 % chunk_w ||
        (col0 ? c0 + d.cols > input_k[src[j]] : d.cols != input_k[src[j]]))
      return TB_ERR_ARGUMENT;
    int st = make_job(fmt, d.tiled, d.tiled_sign, d.rows, d.cols, nullptr, 1, d.a_scale,
                      d.w_scale, d.workspace, d.acc_out, d.out64, d.out32, start, host[j], true);
    if (st != TB_OK) return st;
    host[j].src = src[j];
    host[j].c0 = (int)(c0 / chunk_w);
    start = host[j].end;
    maxE = std::max(maxE, (int64_t)host[j].Npad);
  }
  *total_chunks = start;
  *max_entries = maxE;
  return TB_OK;
}

extern "C" int tb_gemv_step_prepare(int fmt, int64_t njobs, const tb_gemv_desc *descs,
                                    const int32_t *src, int64_t ninputs, const int64_t *input_k,
                                    void *table_host, int64_t *total_chunks,
                                    int64_t *max_entries) {
  return tb_gemv_step_prepare_cols(fmt, njobs, descs, src, nullptr, ninputs, input_k, table_host,
                                   total_chunks, max_entries);
}

extern "C" int tb_gemv_step_launch(int fmt, const void *table_device, int64_t njobs,
                                   int64_t total_chunks, int64_t ninputs,
                                   const tb_step_input *inputs, int32_t x_after_wait,  /* TB_STEP_* flags */
                                   const void *prev_table_device, int64_t prev_njobs,
                                   const void *table_host, const void *prev_table_host,
                                   void *stream) {
  if (fmt < TB_I2S || fmt > TB_TL2 || njobs < 1 || !table_device || total_chunks < 1 ||
      total_chunks >= ((int64_t)1 << 31) || ninputs < 1 || ninputs > kMaxStepInputs ||
      !inputs || prev_njobs < 0 || (prev_njobs > 0 && !prev_table_device) ||
      (prev_njobs > 0 && prev_table_device == table_device))
    return TB_ERR_ARGUMENT;
  GemvBatch b{};
  b.table = static_cast<const GemvJob *>(table_device);
  b.njobs = (int)njobs;
  b.total = (int)total_chunks;
  const int rec = fmt == TB_TL2 ? Fmt<TB_TL2>::kRecBytes : Fmt<TB_I2S>::kRecBytes;
  int64_t off = 0;
  for (int64_t v = 0; v < ninputs; ++v) {
    const tb_step_input &in = inputs[v];
    if (!in.x || !in.scale || in.K < 1) return TB_ERR_ARGUMENT;
    const int64_t C = ceil_div(ref_row_bytes(fmt, in.K), kChunkBytes);
    b.in.x[v] = in.x;
    b.in.ready[v] = in.ready;
    b.in.scale[v] = in.scale;
    b.in.flag[v] = in.nonfinite_flag;
    b.in.K[v] = (int)in.K;
    b.in.C[v] = (int)C;
    b.in.off[v] = (int)off;
    off += C * rec;
  }
  if (off > 64 * 1024) return TB_ERR_UNSUPPORTED;  // (and <= the kernel's table, checked at launch)
  b.in.n = (int)ninputs;
  b.in.x_after_wait = (x_after_wait & TB_STEP_X_AFTER_WAIT) ? 1 : 0;
  b.in.sticky_flags = (x_after_wait & TB_STEP_STICKY_FLAGS) ? 1 : 0;
  b.in.self_fin = (x_after_wait & TB_STEP_SELF_FINALIZE) ? 1 : 0;
  b.in.no_wait = (x_after_wait & TB_STEP_INDEPENDENT) ? 1 : 0;
  if (b.in.no_wait && (!b.in.self_fin || b.in.x_after_wait)) return TB_ERR_ARGUMENT;
  if (b.in.self_fin) {
    // every job finalises its own workspace (no K-window sharing one), and
    // nothing of a previous launch is pending on this launch's grid
    if (!table_host || prev_njobs > 0) return TB_ERR_ARGUMENT;
    const GemvJob *h = static_cast<const GemvJob *>(table_host);
    for (int64_t j = 0; j < njobs; ++j)
      if (h[j].fin_m != 1) return TB_ERR_ARGUMENT;
  }
  const bool isolated = (x_after_wait & TB_STEP_ISOLATED) != 0;
  b.in.prev = static_cast<const GemvJob *>(prev_table_device);
  b.in.prev_njobs = (int)prev_njobs;
  b.in.prev_inline = 0;
  if (prev_table_host && prev_njobs > 0 && prev_njobs <= kMaxInlineFin) {
    const GemvJob *h = static_cast<const GemvJob *>(prev_table_host);
    for (int j = 0; j < prev_njobs; ++j) {
      FinJob &F = b.in.fin[j];
      F.ws_acc = h[j].ws_acc;
      F.acc_out = h[j].acc_out;
      F.out64 = h[j].out64;
      F.out32 = h[j].out32;
      F.a_scale = h[j].a_scale;
      F.w_scale = h[j].w_scale;
      F.N = h[j].N;
      F.Npad = h[j].Npad;
      F.M = h[j].fin_m;
    }
    b.in.prev_inline = 1;
  }
  if (table_host && njobs <= kMaxInlineJobs) {  // jobs inline in the kernel parameters
    const GemvJob *h = static_cast<const GemvJob *>(table_host);
    for (int j = 0; j < njobs; ++j) b.jobs[j] = h[j];
    b.table = nullptr;
  }
  return launch_step(fmt, b, (int)off, isolated, static_cast<cudaStream_t>(stream));
}

extern "C" int tb_gemv_batch_finalize(const void *table_device, int64_t njobs,
                                      int64_t max_entries, void *stream) {
  if (!table_device || njobs < 1 || njobs > 65535 || max_entries < 1 ||
      max_entries >= ((int64_t)1 << 31))
    return TB_ERR_ARGUMENT;
  GemvBatch b{};
  b.table = static_cast<const GemvJob *>(table_device);
  b.njobs = (int)njobs;
  b.max_entries = (int)max_entries;
  return launch_finalize(b, static_cast<cudaStream_t>(stream));
}

// Copy-in of a step's inputs from mapped pinned HOST memory with SM loads:
// one 16-byte load per thread, all in flight at once, so the copy costs about
// one PCIe round trip instead of a copy-engine launch (~10 us measured for a
// 72 KB H2D memcpy behind a busy stream).  The loads bypass the caches
// (ld.global.cv): the host rewrites the buffer between launches.  A
// programmatic-dependent step (TB_STEP_X_AFTER_WAIT) launches early and
// prefetches its weights meanwhile.
// Few, wide CTAs: an SM running one cannot host the dependent step's
// one-CTA-per-SM grid until it exits, so the copy occupies as few SMs as
// possible (kCopyPer loads in flight per thread).
constexpr int kCopyThreads = 1024, kCopyPer = 4;
__global__ void __launch_bounds__(kCopyThreads) copy_in_kernel(uint4 *__restrict__ dst,
                                                               const uint4 *src, int64_t n) {
  asm volatile("griddepcontrol.launch_dependents;");
#ifdef TB_TIMELINE  // the copy's entry / exit in the timeline's last row
  if (blockIdx.x == 0 && threadIdx.x == 0) g_timeline[kTimelineWarps - 1][0] = globaltimer_ns();
#endif
  const int64_t i0 = (int64_t)blockIdx.x * kCopyThreads * kCopyPer + threadIdx.x;
  uint4 v[kCopyPer];
#pragma unroll
  for (int u = 0; u < kCopyPer; ++u)
    if (i0 + u * kCopyThreads < n) v[u] = __ldcv(src + i0 + u * kCopyThreads);
#pragma unroll
  for (int u = 0; u < kCopyPer; ++u)
    if (i0 + u * kCopyThreads < n) dst[i0 + u * kCopyThreads] = v[u];
#ifdef TB_TIMELINE
  if (blockIdx.x == 0 && threadIdx.x == 0) g_timeline[kTimelineWarps - 1][1] = globaltimer_ns();
#endif
}

extern "C" int tb_copy_in(void *dst, const void *src_host, int64_t bytes, void *stream) {
  if (!dst || !src_host || bytes < 1 || (bytes & 15) ||
      (reinterpret_cast<uintptr_t>(dst) & 15) || (reinterpret_cast<uintptr_t>(src_host) & 15))
    return TB_ERR_ARGUMENT;
  const int64_t n = bytes / 16;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)ceil_div(n, (int64_t)kCopyThreads * kCopyPer));
  cfg.blockDim = dim3(kCopyThreads);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, copy_in_kernel, static_cast<uint4 *>(dst),
                         static_cast<const uint4 *>(src_host), n) != cudaSuccess)
    return TB_ERR_CUDA;
  return TB_OK;
}

extern "C" int tb_step_glue_ex(const void *fin_table_device, int64_t fin_njobs,
                               int64_t fin_max_entries, int64_t nq, const tb_quant_desc *q,
                               int32_t flags, void *stream);
extern "C" int tb_step_glue(const void *fin_table_device, int64_t fin_njobs,
                            int64_t fin_max_entries, int64_t nq, const tb_quant_desc *q,
                            void *stream) {
  return tb_step_glue_ex(fin_table_device, fin_njobs, fin_max_entries, nq, q, 0, stream);
}

static int glue_launch(const void *fin_table_device, int64_t fin_njobs,
                       int64_t fin_max_entries, int64_t nq, const tb_quant_desc *q,
                       int32_t flags, int32_t *sync_self, int32_t *sync_prev, int publish_exit,
                       int prev_exit_ctas, const FinJob *finl, int nfinl, void *stream);
extern "C" int tb_step_glue_ex(const void *fin_table_device, int64_t fin_njobs,
                               int64_t fin_max_entries, int64_t nq, const tb_quant_desc *q,
                               int32_t flags, void *stream) {
  return glue_launch(fin_table_device, fin_njobs, fin_max_entries, nq, q, flags, nullptr,
                     nullptr, 0, 0, nullptr, 0, stream);
}

// The glue of a pipelined M > 1 layer (see the sync counters above
// glue_kernel): quantises the layer's inputs and then -- the same CTAs, once
// the previous GEMV has completed -- finalises the PREVIOUS layer's batch
// (fin_table_host: its prepared host job table, or null).  sync_self = this
// layer's 4-int32 block, sync_prev = the previous layer's (null for the first
// layer of a pass, which then waits for the whole preceding chain),
// publish_exit != 0 when the next layer's glue will consume this one's exit
// count.  *glue_ctas = the CTA count the layer's GEMV launch (and the next
// glue, as prev_ctas) must be given.
extern "C" int tb_step_glue_sync(const void *fin_table_host, int64_t fin_njobs, int64_t nq,
                                 const tb_quant_desc *q, int32_t *sync_self,
                                 int32_t *sync_prev, int32_t prev_ctas, int32_t publish_exit,
                                 int32_t *glue_ctas, void *stream) {
  if (!sync_self || nq < 1 || !q || (sync_prev && prev_ctas < 1) || fin_njobs < 0 ||
      (fin_njobs > 0 && !fin_table_host))
    return TB_ERR_ARGUMENT;
  int64_t tokens = 0;
  for (int64_t v = 0; v < nq && v < kMaxGlueVecs; ++v) tokens += q[v].M;
  if (glue_ctas) *glue_ctas = (int32_t)(8 * tokens);
  FinJob fin[kMaxInlineFin];
  int nf = 0;
  const GemvJob *ph = static_cast<const GemvJob *>(fin_table_host);
  for (int64_t j = 0; j < fin_njobs; ++j) {
    if (ph[j].fin_m == 0) continue;  // K-windows finalised through another job
    if (nf == kMaxInlineFin) return TB_ERR_UNSUPPORTED;
    fin[nf++] = FinJob{ph[j].ws_acc, ph[j].acc_out, ph[j].out64, ph[j].out32, ph[j].a_scale,
                       ph[j].w_scale, ph[j].N, ph[j].Npad, ph[j].fin_m};
  }
  return glue_launch(nullptr, 0, 0, nq, q, TB_GLUE_EARLY_QUANT, sync_self, sync_prev,
                     publish_exit ? 1 : 0, prev_ctas, fin, nf, stream);
}

extern "C" int64_t tb_sync_timeouts(void) {
  int v = 0;
  if (cudaMemcpyFromSymbol(&v, g_sync_timeouts, sizeof(v)) != cudaSuccess) return -1;
  return v;
}

static int glue_launch(const void *fin_table_device, int64_t fin_njobs,
                       int64_t fin_max_entries, int64_t nq, const tb_quant_desc *q,
                       int32_t flags, int32_t *sync_self, int32_t *sync_prev, int publish_exit,
                       int prev_exit_ctas, const FinJob *finl, int nfinl, void *stream) {
  if (nq < 0 || nq > kMaxGlueVecs || (nq > 0 && !q) || fin_njobs < 0 ||
      (fin_njobs > 0 && (!fin_table_device || fin_max_entries < 1 ||
                         fin_max_entries >= ((int64_t)1 << 31))))
    return TB_ERR_ARGUMENT;
  GlueParams g{};
  g.fin.table = static_cast<const GemvJob *>(fin_table_device);
  g.fin.njobs = (int)fin_njobs;
  g.nq = (int)nq;
  g.early = (flags & 1) ? 1 : 0;
  g.sync_self = sync_self;
  g.sync_prev = sync_prev;
  g.publish_exit = publish_exit;
  g.prev_exit_ctas = prev_exit_ctas;
  g.nfinl = nfinl;
  for (int j = 0; j < nfinl; ++j) g.finl[j] = finl[j];
  int tokens = 0;
  for (int64_t v = 0; v < nq; ++v) {
    const tb_quant_desc &d = q[v];
    if (!d.x || !d.scale || !d.rec || d.M < 1 || d.K < 1 || d.ldx < d.K ||
        (d.q && d.ldq < d.K) || d.fmt < TB_I2S || d.fmt > TB_TL2 ||
        (reinterpret_cast<uintptr_t>(d.rec) & 15))
      return TB_ERR_ARGUMENT;
    QuantVec &Q = g.q[v];
    Q.x = d.x;
    Q.qnat = d.q;
    Q.scale = d.scale;
    Q.rec = d.rec;
    Q.flag = d.nonfinite_flag;
    Q.K = d.K;
    Q.ldx = d.ldx;
    Q.ldq = d.ldq;
    Q.M = (int)d.M;
    Q.C = (int)ceil_div(ref_row_bytes(d.fmt, d.K), kChunkBytes);
    Q.fmt = d.fmt;
    Q.is_f64 = d.x_is_f64 ? 1 : 0;
    tokens += Q.M;
  }
  g.q_tokens = tokens;
  // finalize rows: flat over all jobs (units of 4 entries, kGlueIlp units per
  // thread) when the table is small enough to stage; else 8-CTA groups per job
  int64_t fin_rows = 0;
  if (fin_njobs > kMaxGlueFin) {
    g.fin.fin_parts = fin_njobs > 0 ? (int)ceil_div(fin_max_entries, (int64_t)8 * 256) : 0;
    fin_rows = fin_njobs * g.fin.fin_parts;
  } else if (fin_njobs > 0) {
    // the caller passes the largest job's entries; bound the total by njobs x that
    const int64_t units = fin_njobs * fin_max_entries / 4;
    g.fin.fin_parts = (int)std::max<int64_t>(1, ceil_div(units, (int64_t)8 * 256 * kGlueIlp));
    fin_rows = g.fin.fin_parts;
  }
  const int64_t rows64 = tokens + fin_rows;
  if (rows64 > 65535) return TB_ERR_ARGUMENT;
  const int rows = (int)rows64;
  if (rows == 0) return TB_OK;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(8, rows);
  cfg.blockDim = dim3(256);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 8;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, glue_kernel, g) == cudaSuccess ? TB_OK : TB_ERR_CUDA;
}

extern "C" int tb_gemv(int fmt, const uint8_t *tiled, const uint8_t *tiled_sign, int64_t rows,
                       int64_t cols, const int8_t *act, int64_t M, int64_t ld_act,
                       int64_t act_len, const double *a_scale, double w_scale, void *workspace,
                       int32_t *acc_out, double *out64, float *out32, void *stream) {
  if (!tiled || !act || !workspace || rows < 1 || cols < 1 || M < 1 || M > 16 || ld_act < 1 ||
      act_len < 0 || act_len > ld_act || fmt < TB_I2S || fmt > TB_TL2)
    return TB_ERR_ARGUMENT;
  uint8_t *rec = static_cast<uint8_t *>(workspace) + ws_counts_bytes(rows);
  int st = tb_prep_activations(fmt, act, M, ld_act, act_len, cols, rec, stream);
  if (st != TB_OK) return st;
  return tb_gemv_records(fmt, tiled, tiled_sign, rows, cols, rec, M, a_scale, w_scale, workspace,
                         acc_out, out64, out32, stream);
}

#ifdef TB_TIMELINE
extern "C" int tb_timeline_fetch(void *host, int64_t bytes) {
  if (bytes > (int64_t)sizeof(g_timeline)) bytes = sizeof(g_timeline);
  return cudaMemcpyFromSymbol(host, g_timeline, bytes) == cudaSuccess ? TB_OK : TB_ERR_CUDA;
}
extern "C" int tb_timeline_clear(void) {
  void *p = nullptr;
  if (cudaGetSymbolAddress(&p, g_timeline) != cudaSuccess) return TB_ERR_CUDA;
  return cudaMemset(p, 0, sizeof(g_timeline)) == cudaSuccess ? TB_OK : TB_ERR_CUDA;
}
#endif
