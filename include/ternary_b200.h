/*
 * ternary_b200.h -- C ABI of the B200-native ternary BitLinear hot path.
 *
 * Drop-in boundary for the reference package ``ternpack`` (bitnet.cpp,
 * arXiv 2410.16144).  The reference's native boundary is its five numba
 * kernels (pkg/src/ternpack/_fast.py:25-147) plus the NumPy arithmetic of
 * core.py / packing.py / lut.py that surrounds them; each entry point below
 * names the reference interface it replaces.
 *
 * Conventions:
 *   - every buffer is a DEVICE pointer owned by the caller (plain pointers and
 *     sizes; no torch types), except where a name says `host`;
 *   - `stream` is a cudaStream_t passed as void*; nothing synchronises
 *     implicitly; kernels are reentrant and keep no global mutable state;
 *   - every function returns a tb_status (0 = OK); tb_strerror() maps it to
 *     text; data-dependent errors (invalid codes, non-finite input) are
 *     reported through caller-provided device int32 flags so the call stays
 *     asynchronous -- the Python mirror turns them into the reference's
 *     ValueError messages.
 *
 * Packed-weight layouts:
 *   reference layout   -- byte-identical to ternpack's PackedI2S.data,
 *                         PackedTL1.data, PackedTL2.index_data/sign_data
 *                         (packing.py:77-197): row-major, rows byte aligned;
 *   tiled layout       -- the GEMV layout: 32-row tiles, each row split into
 *                         16-byte chunks, stored [tile][chunk][row][16 B]
 *                         (TL2 sign bits alongside as [tile][chunk][row][4 B]);
 *                         it is a pure permutation of 16-byte granules of the
 *                         reference layout plus zero-weight padding.
 */
#ifndef TERNARY_B200_H
#define TERNARY_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum tb_status {
  TB_OK = 0,
  TB_ERR_ARGUMENT = 1,     /* bad size / null pointer / unsupported format    */
  TB_ERR_CUDA = 2,         /* a CUDA runtime call failed                      */
  TB_ERR_UNSUPPORTED = 3,  /* shape outside what this build handles           */
} tb_status;

typedef enum tb_format { TB_I2S = 1, TB_TL1 = 2, TB_TL2 = 3 } tb_format;

const char *tb_strerror(int status);
int tb_abi_version(void);            /* bumps on any signature change          */
int tb_device_sm_count(int device);  /* cached multiProcessorCount             */
int tb_stream_synchronize(void *stream); /* cudaStreamSynchronize (host paths that
                                            replay a graph on the caller's stream) */

/* ---------------------------------------------------------------- core.py */

/* quantize_activations (core.py:116-134), M tokens at once: x[M][ldx] (K valid
 * entries per row), q[M][ldq] int8 with zero padding up to ldq, scale[M] f64.
 * Bit-exact with the reference: float64 absmax, scale = amax/127 (1 when 0),
 * q = clip(trunc(x/scale + copysign(.5, x/scale)), -127, 127).
 * nonfinite_flag (device int32, may be NULL) is set to 1 on NaN/Inf input.   */
int tb_quantize_f32(const float *x, int64_t M, int64_t K, int64_t ldx,
                    int8_t *q, int64_t ldq, double *scale,
                    int32_t *nonfinite_flag, void *stream);
int tb_quantize_f64(const double *x, int64_t M, int64_t K, int64_t ldx,
                    int8_t *q, int64_t ldq, double *scale,
                    int32_t *nonfinite_flag, void *stream);

/* ternarize_weights (core.py:104-113), split in two so the scale is bit-exact
 * with NumPy's pairwise np.mean: the host enumerates the pairwise tree down to
 * `nsub` subtrees (offsets/lengths in device int64 arrays), the device sums
 * |w| over each subtree in NumPy's exact order, the host combines the partial
 * sums up the tree and divides by n; then tb_ternarize_apply writes
 * q = clip(rha(w / scale), -1, 1).                                          */
int tb_abs_pairwise_sums_f32(const float *w, const int64_t *sub_off,
                             const int64_t *sub_len, int64_t nsub,
                             double *sums, int32_t *nonfinite_flag, void *stream);
int tb_abs_pairwise_sums_f64(const double *w, const int64_t *sub_off,
                             const int64_t *sub_len, int64_t nsub,
                             double *sums, int32_t *nonfinite_flag, void *stream);
int tb_ternarize_apply_f32(const float *w, int64_t n, double scale, int8_t *q,
                           void *stream);
int tb_ternarize_apply_f64(const double *w, int64_t n, double scale, int8_t *q,
                           void *stream);

/* output = float64(acc) * w_scale * a_scale[m]  (core.py:99-101); either
 * output may be NULL.                                                      */
int tb_scale_outputs(const int32_t *acc, int64_t M, int64_t N, double w_scale,
                     const double *a_scale, double *out64, float *out32,
                     void *stream);

/* ------------------------------------------------------------ packing.py */

/* Reference-layout sizes (packing.py:42-53). */
int64_t tb_ref_row_bytes(int fmt, int64_t cols);       /* I2S/TL1/TL2 index */
int64_t tb_ref_sign_row_bytes(int64_t cols);           /* TL2 sign plane    */

/* encode_i2s / encode_tl1 / encode_tl2 (packing.py:200-262): int8 ternary
 * values [rows][cols] -> reference-layout bytes.  `sign` only for TL2.     */
int tb_encode(int fmt, const int8_t *values, int64_t rows, int64_t cols,
              uint8_t *out, uint8_t *sign, void *stream);
/* decode_* (packing.py:209-277).  bad_flag (device int32) is set to 1 on an
 * invalid code (I2S 0b11 / TL1 nibble > 8 / TL2 index > 13), 2 on a TL2
 * non-canonical zero.                                                       */
int tb_decode(int fmt, const uint8_t *data, const uint8_t *sign, int64_t rows,
              int64_t cols, int8_t *values, int32_t *bad_flag, void *stream);
/* validate() (packing.py:98-107, 135-141, 176-186): first_bad[0] = first row
 * with an invalid code, first_bad[1] = first row with a TL2 non-canonical
 * zero; both must be initialised to INT32_MAX by the caller.               */
int tb_validate(int fmt, const uint8_t *data, const uint8_t *sign, int64_t rows,
                int64_t cols, int32_t *first_bad, void *stream);

/* Tiled GEMV layout: sizes, repack from the reference layout, and inverse. */
int64_t tb_tiled_chunks(int fmt, int64_t cols);          /* 16-B chunks/row */
int64_t tb_tiled_bytes(int fmt, int64_t rows, int64_t cols);
int64_t tb_tiled_sign_bytes(int fmt, int64_t rows, int64_t cols);
int tb_repack(int fmt, const uint8_t *ref, const uint8_t *ref_sign, int64_t rows,
              int64_t cols, uint8_t *tiled, uint8_t *tiled_sign, void *stream);
int tb_unrepack(int fmt, const uint8_t *tiled, const uint8_t *tiled_sign,
                int64_t rows, int64_t cols, uint8_t *ref, uint8_t *ref_sign,
                void *stream);

/* ---------------------------------------------------------------- lut.py */

/* build_lut_tl1 / build_lut_tl2 (lut.py:72-84): act int8[len] zero-extended
 * to groups*2 (groups*3); entries int16 [groups][9] ([groups][14]).         */
int tb_build_lut(int fmt, const int8_t *act, int64_t len, int64_t groups,
                 int16_t *entries, void *stream);

/* ------------------------------------------------------------ kernels.py */

/* Decode GEMV / small-M GEMM on the tiled layout: replaces gemv_i2s /
 * gemv_tl1 / gemv_tl2 / gemv_parallel (kernels.py:86-157, 189-268) and the
 * numba byte-table gathers (_fast.py:25-95).  act int8 [M][ld_act] with
 * `act_len` valid entries per token (zero beyond), M <= 16.  Results are the
 * exact int32 dot products for every M; outputs (each may be NULL):
 *   acc_out[M][N] int32, out64[M][N] = f64(acc)*w_scale*a_scale[m],
 *   out32[M][N] = (float)out64.
 * The workspace (tb_gemv_workspace_bytes) must be zeroed once before first
 * use; every call leaves it zeroed again (self-cleaning), so one workspace
 * serves any number of back-to-back calls on ONE stream.                    */
int64_t tb_gemv_workspace_bytes(int fmt, int64_t rows, int64_t cols);

/* Activation "records": the decode GEMV's input form of M int8 activation
 * vectors -- per 16-byte weight chunk, the chunk's activations byte-
 * transposed to match the decoded code words plus their sum (80 B per chunk
 * for I2S/TL1, 112 B for TL2).  GEMVs that share an input (q/k/v, gate/up)
 * share one record buffer.  `rec` must be 16-byte aligned.                  */
int64_t tb_act_records_bytes(int fmt, int64_t M, int64_t cols);
int tb_prep_activations(int fmt, const int8_t *act, int64_t M, int64_t ld_act,
                        int64_t act_len, int64_t cols, uint8_t *rec, void *stream);
/* quantize_activations fused with record construction (core.py:116-134):
 * x[M][ldx] (K = cols valid) -> scale[M], records, and optionally the natural
 * int8 q[M][ldq] (bit-exact reference data; NULL to skip).                 */
int tb_quantize_records_f32(int fmt, const float *x, int64_t M, int64_t K,
                            int64_t ldx, int8_t *q, int64_t ldq, double *scale,
                            uint8_t *rec, int32_t *nonfinite_flag, void *stream);
int tb_quantize_records_f64(int fmt, const double *x, int64_t M, int64_t K,
                            int64_t ldx, int8_t *q, int64_t ldq, double *scale,
                            uint8_t *rec, int32_t *nonfinite_flag, void *stream);
/* The decode GEMV proper, on prepared records (one launch).                */
int tb_gemv_records(int fmt, const uint8_t *tiled, const uint8_t *tiled_sign,
                    int64_t rows, int64_t cols, const uint8_t *rec, int64_t M,
                    const double *a_scale, double w_scale, void *workspace,
                    int32_t *acc_out, double *out64, float *out32, void *stream);
/* Grouped decode GEMV: several independent GEMVs of one format in ONE launch
 * (the weight stream never stops at a matrix boundary).  prepare() fills a
 * caller-provided host buffer of njobs * tb_gemv_job_bytes() bytes; copy it
 * to device memory once, then launch() as often as needed (capturable: no
 * host sync, no allocation).                                                */
typedef struct tb_gemv_desc {
  const uint8_t *tiled;
  const uint8_t *tiled_sign;
  int64_t rows, cols;
  const uint8_t *rec; /* records of this GEMV's input (shared is fine)     */
  int64_t M;
  const double *a_scale;
  double w_scale;
  void *workspace; /* per GEMV, tb_gemv_workspace_bytes, zeroed once        */
  int32_t *acc_out;
  double *out64;
  float *out32;
} tb_gemv_desc;
int64_t tb_gemv_job_bytes(void);
/* Also reports max_entries = max over jobs of M * padded rows, which sizes
 * the finalize grid (one accumulator per thread).                          */
int tb_gemv_batch_prepare(int fmt, int64_t njobs, const tb_gemv_desc *descs,
                          void *table_host, int64_t *total_chunks, int32_t *max_m,
                          int64_t *max_entries);
/* finalize != 0: also launch the finalize pass (scales -> outputs, workspace
 * reset); 0: the caller finalises, e.g. inside the next tb_step_glue.       */
int tb_gemv_batch_launch(int fmt, const void *table_device, int64_t njobs,
                         int64_t total_chunks, int32_t max_m, int64_t max_entries,
                         int32_t finalize, void *stream);
/* As tb_gemv_batch_prepare, plus K-windows: job j contracts record columns
 * [col0[j], col0[j] + descs[j].cols) of a records buffer built for
 * rec_cols[j] columns (col0 a multiple of one record chunk: 64 weights, 96
 * for TL2; NULL arrays = whole records).  A job with acc_out, out64 and out32
 * all NULL is not finalised: its partial sums accumulate in its workspace,
 * which another job of the batch with the same workspace finalises (the
 * K-windows of one matrix).  Replaces nothing in the reference (its thread
 * pool splits rows only, kernels.py:181-186).                              */
int tb_gemv_batch_prepare_cols(int fmt, int64_t njobs, const tb_gemv_desc *descs,
                               const int64_t *col0, const int64_t *rec_cols, void *table_host,
                               int64_t *total_chunks, int32_t *max_m, int64_t *max_entries);
/* As tb_gemv_batch_launch, also given the host copy of a job table of <= 20
 * jobs: the jobs ride in the kernel parameters and, for 2 <= M <= 8 tokens
 * (I2_S / TL1), every CTA keeps its segment's records in one shared-memory
 * table (no per-warp record staging); larger tables fall back to the
 * records path.  prev_table_host / prev_njobs (optional): the host job table
 * of the batch launched before this one (completed before this launch's
 * inputs were produced); this launch finalises it in its tail (table mode
 * only: TB_ERR_UNSUPPORTED otherwise, and the caller finalises it).       */
/* Number of tb_gemv_batch_launch_inline calls that ran in records-table
 * mode (introspection for tests: the fallback is silent by design).       */
int64_t tb_gemv_table_launches(void);
int tb_gemv_batch_launch_inline(int fmt, const void *table_device, const void *table_host,
                                int64_t njobs, int64_t total_chunks, int32_t max_m,
                                int64_t max_entries, int32_t finalize,
                                const void *prev_table_host, int64_t prev_njobs, void *stream);

/* Decode-step glue in ONE launch: finalise a prepared GEMV batch (may be
 * empty: fin_njobs = 0) and quantise up to 4 activation matrices into
 * records (quantize_activations, core.py:116-134, one 8-CTA cluster per
 * token).  Both halves are independent, so a decode step is
 * glue(previous outputs, next inputs) + one grouped GEMV launch.            */
typedef struct tb_quant_desc {
  const void *x; /* [M][ldx] float32 or float64 (x_is_f64)                  */
  int32_t x_is_f64;
  int32_t fmt; /* record layout of the consuming GEMVs                     */
  int64_t M, K, ldx;
  int8_t *q; /* optional natural codes [M][ldq]                             */
  int64_t ldq;
  double *scale;
  uint8_t *rec;
  int32_t *nonfinite_flag;
} tb_quant_desc;
int tb_step_glue(const void *fin_table_device, int64_t fin_njobs,
                 int64_t fin_max_entries, int64_t nq, const tb_quant_desc *q,
                 void *stream);
/* As tb_step_glue; flags & TB_GLUE_EARLY_QUANT: the quantisation runs
 * before the programmatic-dependent-launch wait on the preceding kernel
 * (overlapping it), the finalize after it, and every CTA waits before
 * exiting.  The caller guarantees the inputs do not depend on the preceding
 * kernel and that no kernel still in flight reads the records or scales
 * being written (e.g. three record sets in rotation).                     */
#define TB_GLUE_EARLY_QUANT 1
int tb_step_glue_ex(const void *fin_table_device, int64_t fin_njobs, int64_t fin_max_entries,
                    int64_t nq, const tb_quant_desc *q, int32_t flags, void *stream);
/* Pipelined M > 1 decode layers (the reference token pass, bench.py:138-153,
 * for 2..8 tokens per step): layer l's grouped GEMV starts streaming as soon
 * as its activation records exist, while layer l-1's GEMV is still draining.
 * Each layer owns a block of 4 int32 counters in device memory, zero before
 * first use (the kernels reset them): tb_step_glue_sync quantises the layer's
 * inputs (quantize_activations, core.py:116-134; TB_GLUE_EARLY_QUANT rules,
 * three record sets in rotation) and counts its CTAs into sync_self, then --
 * the same CTAs, once the previous GEMV has completed -- finalises the previous
 * layer's batch (fin_table_host: its prepared host job table, or null); unless
 * sync_prev is null (first layer of a pass: it waits for the whole preceding
 * chain) it first waits for the previous layer's glue to have exited, which
 * that glue does only after the GEMV two layers back completed and was
 * finalised (prev_ctas = that call's *glue_ctas).
 * tb_gemv_batch_launch_sync is tb_gemv_batch_launch_inline in records-table
 * mode whose table fill waits for those counts (glue_ctas as returned by the
 * glue call) rather than for the glue's completion (prev_njobs = 0 when the
 * glue finalises; otherwise the previous batch is finalised in this launch's
 * tail, after griddepcontrol.wait).  Waits are bounded: a timeout
 * is counted (tb_sync_timeouts, -1 on a CUDA error) instead of hanging.     */
int tb_step_glue_sync(const void *fin_table_host, int64_t fin_njobs, int64_t nq,
                      const tb_quant_desc *q, int32_t *sync_self, int32_t *sync_prev,
                      int32_t prev_ctas, int32_t publish_exit, int32_t *glue_ctas,
                      void *stream);
int tb_gemv_batch_launch_sync(int fmt, const void *table_device, const void *table_host,
                              int64_t njobs, int64_t total_chunks, int32_t max_m,
                              int64_t max_entries, const void *prev_table_host,
                              int64_t prev_njobs, int32_t *sync, int32_t glue_ctas,
                              void *stream);
int64_t tb_sync_timeouts(void);
/* Fused one-token decode step in ONE launch (gemv.cu, tgemv_kernel<.,1,true>):
 * every CTA quantises the float32 input vectors itself (quantize_activations,
 * core.py:116-134, records kept in shared memory), streams the grouped GEMV
 * (jobs read input src[j]), and -- after its own work, once the preceding
 * grid has completed -- finalises the PREVIOUS step's batch (prev table; it
 * must not be this batch).  This step's outputs are finalised by the next
 * step launch or by tb_gemv_batch_finalize.  prepare(): descs[j].M == 1,
 * descs[j].cols == input_k[src[j]], descs[j].a_scale = the scale pointer
 * input src[j] will be given at launch.  x_after_wait != 0: the inputs are
 * produced by the preceding kernel (read after griddepcontrol.wait).
 * table_host / prev_table_host (optional): the prepared host tables -- small
 * batches then ride in the kernel parameters (each CTA quantises only the
 * inputs its jobs read; the previous step is finalised without descriptor
 * loads).                                                                    */
/* tb_gemv_step_launch `flags`: */
#define TB_STEP_X_AFTER_WAIT 1 /* inputs written by the preceding kernel          */
#define TB_STEP_ISOLATED 2     /* one launch at a time (no chained step to overlap):
                                  one 16-warp CTA per SM instead of four small ones */
#define TB_STEP_STICKY_FLAGS 4 /* non-finite flags are only ever SET (the caller
                                  clears them): one flag can cover many steps     */
#define TB_STEP_SELF_FINALIZE 8 /* the launch writes its OWN outputs: the warp
                                  that completes a row tile's partial sums (a
                                  per-tile chunk counter in the workspace)
                                  applies the scales -- no finalize launch and
                                  no next step needed (one-token latency path,
                                  HostStep).  Requires table_host, no prev
                                  table, every job finalising its own workspace,
                                  and no other launch in flight on the same
                                  workspaces.                                  */
#define TB_STEP_INDEPENDENT 16 /* with TB_STEP_SELF_FINALIZE: the launch never
                                  waits for the preceding kernel (no
                                  griddepcontrol.wait at all), so independent
                                  steps overlap freely instead of completing
                                  in launch order -- a stream of unrelated
                                  GEMVs (BASELINE configs[0]).  The caller
                                  guarantees that nothing the launch touches
                                  (inputs, workspaces, outputs, scales) is
                                  read or written by a kernel that can still
                                  be in flight -- e.g. reuse a step only after
                                  >= 16 other launches of this kind (a B200
                                  holds at most 4 of their CTAs per SM), or
                                  after a dependent (waiting) launch.          */
/* Copy `bytes` (a multiple of 16, 16-B aligned both sides) from mapped pinned
 * HOST memory to device memory with one kernel of 16-byte loads (no
 * copy-engine launch); a following TB_STEP_X_AFTER_WAIT step launch is its
 * programmatic dependent.  The one-token latency path's input copy
 * (HostStep); replaces the reference's host-side activation hand-off
 * (kernels.py:189, arrays passed to the numba kernel).                     */
int tb_copy_in(void *dst, const void *src_host, int64_t bytes, void *stream);
typedef struct tb_step_input {
  const float *x;          /* [K] float32 (device; 16-B alignment preferred)  */
  int64_t K;
  double *scale;           /* out: absmax / 127 (or 1) of this vector         */
  int32_t *nonfinite_flag; /* optional: 1 if this launch saw NaN / inf, else 0
                            (device or mapped pinned host memory)            */
  const int32_t *ready;    /* optional: the launch waits until *ready != 0
                            before reading x (e.g. set by the copy engine
                            after the host-to-device copy that fills x)     */
} tb_step_input;
int tb_gemv_step_prepare(int fmt, int64_t njobs, const tb_gemv_desc *descs,
                         const int32_t *src, int64_t ninputs, const int64_t *input_k,
                         void *table_host, int64_t *total_chunks,
                         int64_t *max_entries);
/* As tb_gemv_step_prepare, plus col0[j] (NULL = all 0): job j contracts input
 * columns [col0[j], col0[j] + descs[j].cols) of input src[j] -- a row-parallel
 * (K-sharded) projection whose per-token scale is that of the FULL input
 * vector (core.py:128: absmax over the whole token).  col0 must be a multiple
 * of one record chunk (64 weights for I2_S / TL1, 96 for TL2); a shard that
 * ends before the input does is zero-padded to whole chunks by tb_repack, so
 * the columns it does not own contribute exactly 0.  With col0 non-NULL
 * every job is such a window (col0[j] + cols <= K); with col0 NULL every
 * job must contract its whole input (cols == K).
 * Replaces nothing in the reference (its thread pool splits rows only,
 * kernels.py:181-186); it is the SURVEY §8(e) row-parallel shard.            */
int tb_gemv_step_prepare_cols(int fmt, int64_t njobs, const tb_gemv_desc *descs,
                              const int32_t *src, const int64_t *col0, int64_t ninputs,
                              const int64_t *input_k, void *table_host,
                              int64_t *total_chunks, int64_t *max_entries);
int tb_gemv_step_launch(int fmt, const void *table_device, int64_t njobs,
                        int64_t total_chunks, int64_t ninputs,
                        const tb_step_input *inputs, int32_t flags,
                        const void *prev_table_device, int64_t prev_njobs,
                        const void *table_host, const void *prev_table_host,
                        void *stream);
/* Finalise a batch's accumulators (scales -> outputs, workspace reset).    */
int tb_gemv_batch_finalize(const void *table_device, int64_t njobs,
                           int64_t max_entries, void *stream);
/* Convenience: tb_prep_activations into the workspace + tb_gemv_records.   */
int tb_gemv(int fmt, const uint8_t *tiled, const uint8_t *tiled_sign,
            int64_t rows, int64_t cols, const int8_t *act, int64_t M,
            int64_t ld_act, int64_t act_len, const double *a_scale,
            double w_scale, void *workspace, int32_t *acc_out, double *out64,
            float *out32, void *stream);

/* Prefill GEMM (BASELINE configs[3]) on the tcgen05 int8 tensor cores:
 * D[m][n] = sum_k act[m][k] * w[n][k], exact int32, for M tokens at once --
 * each row m equals the reference's gemv_parallel of token m (kernels.py:
 * 189-268; the reference has no GEMM, a batch is M GEMV calls).  Weights in
 * the tiled layout (tb_repack; I2_S or TL1).  Activations are first tiled
 * into the tensor-core operand order (tb_gemm_tile_act: int8 [M][lda], zero
 * beyond cols, M <= 512; out = tb_gemm_act_bytes(M, cols) bytes, 16-B
 * aligned); GEMMs over the same input share the tiled copy.
 * Outputs as tb_gemv, [M][rows] row-major per job, each may be NULL.
 * tb_gemm_batch: up to 8 GEMMs over the same M <= 512 in one launch (e.g. a
 * layer's projections).  tb_gemm_i8: one matrix, any M, natural int8 input,
 * `workspace` of tb_gemm_act_bytes(min(M, 512), cols) bytes.               */
int64_t tb_gemm_act_bytes(int64_t M, int64_t cols);
int tb_gemm_tile_act(const int8_t *act, int64_t M, int64_t lda, int64_t cols,
                     uint8_t *act_tiled, void *stream);
/* quantize_activations (core.py:116-134) of M <= 512 float32 tokens [M][ldx]
 * straight into the tensor-core operand (the bytes tb_gemm_tile_act writes
 * for the int8 codes, plus scale[M] float64) in one launch; nonfinite_flag
 * (may be NULL) is OR-ed with 1 if any input is NaN/inf (the caller raises
 * "activations must be finite").  TB_ERR_UNSUPPORTED for cols > 163840
 * (use tb_quantize_f32 + tb_gemm_tile_act).  Replaces, for a prefill batch,
 * the reference's per-token quantize_activations calls (bench.py:141-142).  */
int tb_gemm_quantize_act(const float *x, int64_t M, int64_t cols, int64_t ldx, double *scale,
                         int32_t *nonfinite_flag, uint8_t *act_tiled, void *stream);
/* The same for up to 4 activation matrices of one token count M in ONE
 * launch pair (a layer's hidden and intermediate inputs: the reference's
 * two quantize_activations calls per layer, bench.py:141-142).             */
typedef struct tb_qact_desc {
  const float *x;          /* [M][ldx] float32                               */
  int64_t cols, ldx;
  double *scale;           /* [M] per-token scales out                       */
  int32_t *nonfinite_flag; /* optional                                       */
  uint8_t *act_tiled;      /* tb_gemm_act_bytes(M, cols) bytes, 16-B aligned */
} tb_qact_desc;
int tb_gemm_quantize_act_multi(int64_t n, const tb_qact_desc *d, int64_t M, void *stream);
typedef struct tb_gemm_desc {
  const uint8_t *tiled;
  int64_t rows, cols;
  const uint8_t *act_tiled;
  const double *a_scale;
  double w_scale;
  int32_t *acc_out;
  double *out64;
  float *out32;
} tb_gemm_desc;
int tb_gemm_batch(int fmt, int64_t njobs, const tb_gemm_desc *descs, int64_t M,
                  void *stream);
int tb_gemm_i8(int fmt, const uint8_t *tiled, int64_t rows, int64_t cols,
               const int8_t *act, int64_t M, int64_t lda, const double *a_scale,
               double w_scale, uint8_t *workspace, int32_t *acc_out, double *out64,
               float *out32, void *stream);

/* LUT-driven TL1/TL2 GEMV for a caller-supplied LUT (gemv_tl1/gemv_tl2 with
 * an explicit LutTL1/LutTL2, kernels.py:109-157): lut int16 [groups][9|14];
 * every lookup reads the given entries, so corrupted tables behave exactly
 * as in the reference (runtime.py:191-196 fault injection).  acc_out must be
 * zero-initialised; a_scale is a single host scalar here.                 */
int tb_gemv_lut(int fmt, const uint8_t *tiled, const uint8_t *tiled_sign,
                int64_t rows, int64_t cols, const int16_t *lut, int64_t groups,
                int32_t *acc_out, void *stream);

/* gemv_ref_int32 (kernels.py:59-63) on unpacked int8 values [rows][cols];
 * gemv_f32_ref (kernels.py:66-72) on the dequantised fp32 matrix.          */
int tb_gemv_ref_int32(const int8_t *values, int64_t rows, int64_t cols,
                      const int8_t *act, int32_t *acc_out, void *stream);
int tb_gemv_f32_ref(const int8_t *values, int64_t rows, int64_t cols,
                    float w_scale, const float *x, float *out, void *stream);

/* ---- tensor parallel: row-parallel reduction over NVLink peer memory -----
 * (allreduce.cu; SURVEY §8(e).  The reference has no multi-device path; its
 * determinism contract -- any partition of the rows gives the same result,
 * SPEC.md:333 / kernels.py:181-186 -- is kept by summing the row-parallel
 * shards' int32 partial accumulators exactly before the scale of
 * core.py:99-101.)  A rank's partials of every layer live in one symmetric
 * buffer (tb_sym_alloc) that every peer maps (tb_ipc_*); flags are a
 * symmetric uint32[8] per rank, ctrl a rank-local zeroed uint32[4]
 * {epoch, done counter, watchdog mask, spare}: a peer whose signal does not
 * arrive within 4 s sets its bit in ctrl[2] and the launch carries on (its
 * results are invalid; the host checks ctrl[2] and falls back).
 * tb_rowpar_allreduce: one launch per layer, a programmatic dependent of the
 * step that finalised the partials; signals this rank's epoch to every peer,
 * waits for theirs, sums layer_off + [seg.off, seg.off + seg.n) over all
 * ranks and writes out32 = f32(f64(sum) * w_scale * *a_scale) (+ the int32
 * sums if acc_out).  ctas = 0: automatic.  Graph-capturable.
 * tb_rowpar_allreduce_emulated: all `world` ranks in ONE grid on one device
 * (tests): parts/flags/ctrl per rank, segs [world][nseg].                    */
typedef struct tb_rowpar_seg {
  int64_t off, n;
  double w_scale;
  const double *a_scale;
  float *out32;
  int32_t *acc_out;
} tb_rowpar_seg;
int tb_sym_alloc(int64_t bytes, void **ptr);  /* cudaMalloc + zero (IPC-able) */
int tb_sym_free(void *ptr);
int tb_ipc_handle_bytes(void);
int tb_ipc_get_handle(const void *ptr, void *handle_out);
int tb_ipc_open(const void *handle, void **ptr);
int tb_ipc_close(void *ptr);
int tb_rowpar_allreduce(int world, int rank, const int32_t *const *parts,
                        uint32_t *const *flags, uint32_t *ctrl, int64_t layer_off,
                        int64_t nseg, const tb_rowpar_seg *segs, int32_t ctas,
                        void *stream);
int tb_rowpar_allreduce_emulated(int world, const int32_t *const *parts,
                                 uint32_t *const *flags, uint32_t *const *ctrl,
                                 int64_t layer_off, int64_t nseg,
                                 const tb_rowpar_seg *segs, int32_t ctas, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* TERNARY_B200_H */
