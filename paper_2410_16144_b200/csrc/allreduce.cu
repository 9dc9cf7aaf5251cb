// Row-parallel reduction over NVLink peer memory.
//
// A tensor-parallel layer's row-parallel projections (o, down) leave int32
// PARTIAL accumulators on every rank (each rank contracted its K-slice).  The
// reference has no multi-device path; its determinism contract is that any
// partition of the work gives the same result (kernels.py:181-186),
// so the partials are summed as int32 -- exact and order independent -- and
// only then scaled: out = f64(sum) * w_scale * a_scale (core.py:99-101).
//
// One kernel does the whole exchange for a layer, one-shot, with no NCCL
// call: every rank's partials sit in a buffer that every peer has mapped
// (CUDA IPC over NVLink / NVSwitch).  Each CTA
//   1. waits (griddepcontrol.wait) for the grid that finalised this rank's
//      partials -- the launch is a programmatic dependent of that step, so
//      its launch latency hides under the step;
//   2. signals "my partials of this layer are complete" into every peer's
//      flag array (system-scope release store of a per-layer epoch);
//   3. waits until every peer has signalled the same epoch (acquire);
//   4. reads its slice of every rank's partials over NVLink, sums them as
//      int32 and writes the scaled fp32 outputs locally.
// The last CTA to finish advances the rank's epoch counter (device memory,
// so the launch is CUDA-graph replayable).  A rank can be at most one layer
// ahead of a peer (it waits for the peer's signal of each layer), and every
// layer has its own partial buffer, so no buffer is overwritten while a peer
// still reads it: the next write of layer l's partials comes a full token
// pass later, after the peer has signalled layer l + 1.
//
// Emulation (tests, one GPU): tb_rowpar_allreduce_emulated runs the kernel for
// all ranks as ONE grid (blockIdx.y = rank) over buffers in one process, so
// the ranks' waits are on CTAs of the same small, co-resident grid.
#include <cstring>

#include "common.cuh"

namespace tb {

constexpr int kArMaxRanks = 8;
constexpr int kArMaxSegs = 4;
constexpr int kArThreads = 256;
constexpr uint64_t kArTimeoutNs = 4000000000ull;  // peer-signal watchdog: 4 s

struct ArSeg {
  int64_t off, n;  // elements within the layer's partials
  double w_scale;
  const double *a_scale;
  float *out32;     // [n] (this rank)
  int32_t *acc_out; // optional [n]: the summed accumulators
};

struct ArParams {
  int world, rank, emulate, nseg;
  int64_t layer_off;                    // element offset of the layer in every part buffer
  const int32_t *part[kArMaxRanks];     // every rank's partial buffer (peer-mapped)
  uint32_t *flags[kArMaxRanks];         // every rank's flag array [kArMaxRanks] (peer-mapped)
  uint32_t *ctrl[kArMaxRanks];          // rank-local {epoch, done}; emulation: one per rank
  ArSeg seg[kArMaxRanks][kArMaxSegs];   // real ranks use seg[0][*]
};

__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u32(uint32_t *p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int4 ld_volatile_v4(const int32_t *p) {
  int4 v;
  asm volatile("ld.volatile.global.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ int32_t ld_volatile_s32(const int32_t *p) {
  int32_t v;
  asm volatile("ld.volatile.global.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ void ar_store(const ArSeg &S, int64_t i, int32_t s, double as) {
  const double y = static_cast<double>(s) * S.w_scale * as;  // core.py:99-101, left to right
  S.out32[i] = static_cast<float>(y);
  if (S.acc_out) S.acc_out[i] = s;
}

__global__ void __launch_bounds__(kArThreads) rowpar_allreduce_kernel(const __grid_constant__ ArParams P) {
  if (!P.emulate) asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int r = P.emulate ? (int)blockIdx.y : P.rank;
  const int si = P.emulate ? r : 0;
  uint32_t *ctrl = P.ctrl[si];
  __shared__ uint32_t s_epoch;
  if (threadIdx.x == 0) s_epoch = *reinterpret_cast<volatile uint32_t *>(ctrl) + 1u;
  __syncthreads();
  const uint32_t epoch = s_epoch;
  // every CTA signals (idempotent): no rank depends on one particular CTA
  // of a peer's grid being resident
  if (threadIdx.x < P.world) {
    __threadfence_system();
    st_release_sys_u32(P.flags[threadIdx.x] + r, epoch);
  }
  if (threadIdx.x < P.world) {
    // watchdog: a peer that never signals (a lost mapping, a rank that died)
    // must not hang the GPU -- after kArTimeoutNs the wait gives up, records
    // the peer in ctrl[2] (results of this launch are then invalid; the host
    // reads tb_rowpar_allreduce's ctrl[2] and falls back) and carries on
    const uint32_t *f = P.flags[r] + threadIdx.x;
    const uint64_t t0 = globaltimer_ns();
    // sticky: once a launch has timed out, later launches do not wait again
    const bool dead = *reinterpret_cast<volatile uint32_t *>(ctrl + 2) != 0u;
    while (!dead && (int32_t)(ld_acquire_sys_u32(f) - epoch) < 0) {
      __nanosleep(32);
      if (globaltimer_ns() - t0 > kArTimeoutNs) {
        atomicOr(ctrl + 2, 1u << threadIdx.x);
        break;
      }
    }
  }
  __syncthreads();

  // this CTA's slice of every segment, 4 elements per thread where aligned
  for (int q = 0; q < P.nseg; ++q) {
    const ArSeg &S = P.seg[si][q];
    const double as = *S.a_scale;
    const int64_t base = P.layer_off + S.off;
    const int64_t nvec = (base % 4 == 0) ? S.n / 4 : 0;
    for (int64_t v = blockIdx.x * (int64_t)kArThreads + threadIdx.x; v < nvec;
         v += (int64_t)gridDim.x * kArThreads) {
      int4 s = make_int4(0, 0, 0, 0);
#pragma unroll
      for (int p = 0; p < kArMaxRanks; ++p) {
        if (p < P.world) {
          const int4 x = ld_volatile_v4(P.part[p] + base + 4 * v);
          s.x += x.x;
          s.y += x.y;
          s.z += x.z;
          s.w += x.w;
        }
      }
      ar_store(S, 4 * v + 0, s.x, as);
      ar_store(S, 4 * v + 1, s.y, as);
      ar_store(S, 4 * v + 2, s.z, as);
      ar_store(S, 4 * v + 3, s.w, as);
    }
    for (int64_t i = 4 * nvec + blockIdx.x * (int64_t)kArThreads + threadIdx.x; i < S.n;
         i += (int64_t)gridDim.x * kArThreads) {
      int32_t s = 0;
      for (int p = 0; p < P.world; ++p) s += ld_volatile_s32(P.part[p] + base + i);
      ar_store(S, i, s, as);
    }
  }

  // the last CTA of this rank advances the epoch for the next launch
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ctrl + 1, 1u) == gridDim.x - 1) {
      ctrl[1] = 0;
      *reinterpret_cast<volatile uint32_t *>(ctrl) = epoch;
      __threadfence();
    }
  }
}

static int fill_params(ArParams &P, int world, const int32_t *const *parts,
                       uint32_t *const *flags, int64_t layer_off, int64_t nseg,
                       const tb_rowpar_seg *segs, int nseg_sets, int64_t &total) {
  if (world < 1 || world > kArMaxRanks || !parts || !flags || nseg < 1 || nseg > kArMaxSegs ||
      !segs || layer_off < 0)
    return TB_ERR_ARGUMENT;
  P.world = world;
  P.nseg = (int)nseg;
  P.layer_off = layer_off;
  for (int p = 0; p < world; ++p) {
    if (!parts[p] || !flags[p]) return TB_ERR_ARGUMENT;
    P.part[p] = parts[p];
    P.flags[p] = flags[p];
  }
  total = 0;
  for (int r = 0; r < nseg_sets; ++r) {
    int64_t t = 0;
    for (int q = 0; q < nseg; ++q) {
      const tb_rowpar_seg &s = segs[r * nseg + q];
      if (s.n < 1 || s.off < 0 || !s.a_scale || !s.out32) return TB_ERR_ARGUMENT;
      P.seg[r][q] = ArSeg{s.off, s.n, s.w_scale, s.a_scale, s.out32, s.acc_out};
      t += s.n;
    }
    total = t > total ? t : total;
  }
  return TB_OK;
}

}  // namespace tb

using namespace tb;

extern "C" int tb_sym_alloc(int64_t bytes, void **ptr) {
  if (bytes < 1 || !ptr) return TB_ERR_ARGUMENT;
  if (cudaMalloc(ptr, (size_t)bytes) != cudaSuccess) return TB_ERR_CUDA;
  if (cudaMemset(*ptr, 0, (size_t)bytes) != cudaSuccess) return TB_ERR_CUDA;
  return TB_OK;
}

extern "C" int tb_sym_free(void *ptr) {
  return cudaFree(ptr) == cudaSuccess ? TB_OK : TB_ERR_CUDA;
}

extern "C" int tb_ipc_handle_bytes(void) { return (int)sizeof(cudaIpcMemHandle_t); }

extern "C" int tb_ipc_get_handle(const void *ptr, void *handle_out) {
  if (!ptr || !handle_out) return TB_ERR_ARGUMENT;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, const_cast<void *>(ptr)) != cudaSuccess) return TB_ERR_CUDA;
  memcpy(handle_out, &h, sizeof(h));
  return TB_OK;
}

extern "C" int tb_ipc_open(const void *handle, void **ptr) {
  if (!handle || !ptr) return TB_ERR_ARGUMENT;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  if (cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
    return TB_ERR_CUDA;
  return TB_OK;
}

extern "C" int tb_ipc_close(void *ptr) {
  return cudaIpcCloseMemHandle(ptr) == cudaSuccess ? TB_OK : TB_ERR_CUDA;
}

extern "C" int tb_rowpar_allreduce(int world, int rank, const int32_t *const *parts,
                                   uint32_t *const *flags, uint32_t *ctrl, int64_t layer_off,
                                   int64_t nseg, const tb_rowpar_seg *segs, int32_t ctas,
                                   void *stream) {
  ArParams P{};
  int64_t total = 0;
  int st = fill_params(P, world, parts, flags, layer_off, nseg, segs, 1, total);
  if (st != TB_OK) return st;
  if (rank < 0 || rank >= world || !ctrl) return TB_ERR_ARGUMENT;
  P.rank = rank;
  P.emulate = 0;
  P.ctrl[0] = ctrl;
  const int want = (int)ceil_div(ceil_div(total, 4), kArThreads);
  const int grid = ctas > 0 ? ctas : (want < 1 ? 1 : (want > 64 ? 64 : want));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid, 1);
  cfg.blockDim = dim3(kArThreads);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, rowpar_allreduce_kernel, P) == cudaSuccess ? TB_OK
                                                                             : TB_ERR_CUDA;
}

extern "C" int tb_rowpar_allreduce_emulated(int world, const int32_t *const *parts,
                                            uint32_t *const *flags, uint32_t *const *ctrl,
                                            int64_t layer_off, int64_t nseg,
                                            const tb_rowpar_seg *segs, int32_t ctas,
                                            void *stream) {
  ArParams P{};
  int64_t total = 0;
  int st = fill_params(P, world, parts, flags, layer_off, nseg, segs, world, total);
  if (st != TB_OK) return st;
  if (!ctrl) return TB_ERR_ARGUMENT;
  for (int r = 0; r < world; ++r) {
    if (!ctrl[r]) return TB_ERR_ARGUMENT;
    P.ctrl[r] = ctrl[r];
  }
  P.rank = 0;
  P.emulate = 1;
  // every CTA of every emulated rank must be co-resident (they wait on each
  // other): a small grid, launched without programmatic overlap
  const int grid = ctas > 0 ? (ctas > 8 ? 8 : ctas) : 4;
  rowpar_allreduce_kernel<<<dim3(grid, world), kArThreads, 0, static_cast<cudaStream_t>(stream)>>>(P);
  return cudaGetLastError() == cudaSuccess ? TB_OK : TB_ERR_CUDA;
}
