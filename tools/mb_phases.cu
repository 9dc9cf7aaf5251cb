// Microbenchmark of the decode-GEMV's phases (launch, bulk copy, flush) on B200.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mb_phases.cu -o tools/mb_phases
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE, int FLUSH>
__global__ void phase_kernel(const uint8_t *__restrict__ src, int64_t bytes_per_warp, int *cnt, int *acc) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (MODE == 0) return;  // launch only
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 65536) + warp;
  uint8_t *buf = smem + (warp % 16) * 4096;
  int sum = 0;
  if (MODE == 1 || MODE == 2) {
    if (lane == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    for (int64_t off = 0; off < bytes_per_warp; off += 2048) {
      const uint32_t ph = (uint32_t)((off / 2048) & 1);
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(2048) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(buf)),
                     "l"(src + gw * bytes_per_warp + off), "r"(2048), "r"(smem_u32(bar)) : "memory");
      }
      uint32_t ok = 0;
      while (!ok) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(bar)), "r"(ph) : "memory");
      }
      sum += reinterpret_cast<const int *>(buf)[lane];
      __syncwarp();
    }
  } else if (MODE == 3) {  // plain LDG.128 streaming, 8 loads in flight per lane
    const int4 *p = reinterpret_cast<const int4 *>(src + gw * bytes_per_warp);
    const int64_t n = bytes_per_warp / 16;
    for (int64_t i = lane; i < n; i += 32 * 8) {
      int4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = (i + 32 * u < n) ? __ldg(p + i + 32 * u) : make_int4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < 8; ++u) sum += v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
  }
  if (MODE >= 2) {
    // distinct address per lane (as in the GEMV: lane = row)
    asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(acc + ((gw * 32 + lane) & 65535)), "r"(sum) : "memory");
    __syncwarp();
    if (FLUSH == 1 && lane == 0) {
      int old;
      asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(cnt + (gw & 1023)), "r"(1) : "memory");
      if (old == -5) acc[0] = 1;
    }
    if (FLUSH == 2 && lane == 0) {
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      int old = atomicAdd(cnt + (gw & 1023), 1);
      if (old == -5) acc[0] = 1;
    }
  } else if (sum == 0x7fffffff) {
    acc[0] = sum;
  }
}

template <int MODE, int FLUSH = 0>
float run(int grid, int threads, size_t smem, const uint8_t *src, int64_t bpw, int *cnt, int *acc, int iters) {
  CK(cudaFuncSetAttribute(phase_kernel<MODE, FLUSH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
  for (int i = 0; i < iters; ++i) phase_kernel<MODE, FLUSH><<<grid, threads, smem, s>>>(src, bpw, cnt, acc);
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, s));
  CK(cudaStreamSynchronize(s));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  CK(cudaGraphLaunch(ge, s));
  cudaEventRecord(b, s);
  CK(cudaStreamSynchronize(s));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / iters;
}

int main() {
  const size_t total = (size_t)1 << 30;
  uint8_t *src;
  int *cnt, *acc;
  CK(cudaMalloc(&src, total));
  CK(cudaMemset(src, 1, total));
  CK(cudaMalloc(&cnt, 4096));
  CK(cudaMalloc(&acc, 8192));
  const int iters = 40;
  for (int warps : {8, 16, 24}) {
    int threads = warps * 32;
    size_t smem = 65536 + 8 * 32 + 100 * 1024;
    printf("warps/CTA %d smem %zu KB\n", warps, smem / 1024);
    printf("  launch only            : %7.2f us\n", run<0, 0>(148, threads, smem, src, 0, cnt, acc, iters));
    for (int64_t mb : {4, 15, 60}) {
      int64_t bytes = mb << 20;
      int64_t bpw = ((bytes / (148 * warps)) / 2048 + 1) * 2048;
      float t1 = run<1>(148, threads, smem, src, bpw, cnt, acc, iters);
      float t2 = run<2, 0>(148, threads, smem, src, bpw, cnt, acc, iters);
      float t2a = run<2, 1>(148, threads, smem, src, bpw, cnt, acc, iters);
      float t2b = run<2, 2>(148, threads, smem, src, bpw, cnt, acc, iters);
      int64_t bpw16 = ((bytes / (148 * warps)) / 4096 + 1) * 4096;
      float t3 = run<3, 0>(148, threads, smem, src, bpw16, cnt, acc, iters);
      double b1 = (double)bpw * 148 * warps, b3 = (double)bpw16 * 148 * warps;
      printf("  %3lld MB: bulk %6.2f us %6.0f GB/s | +red %6.2f | +red+atom.acq_rel %6.2f | +red+fence+atom %6.2f | LDG x8+red %6.2f us %6.0f GB/s\n",
             (long long)mb, t1, b1 / t1 / 1e3, t2, t2a, t2b, t3, b3 / t3 / 1e3);
    }
  }
  return 0;
}
