// HBM streaming ceiling for a chain of decode-step-sized launches on B200.
// Every launch streams `bytes` (44 MB = the cfg1 step) from rotating buffers
// (> L2), per-warp contiguous ranges, no compute; launches are chained in a
// CUDA graph, optionally as programmatic dependents (PDL) so the next
// launch's prologue overlaps the previous launch's tail.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mb_stream2.cu -o tools/mb_stream2
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// MODE 1: cp.async.cg 16 B per lane, per-warp ring of R stages x SB bytes
// MODE 2: cp.async.bulk per warp (lane 0), ring of R stages x SB bytes
// WAIT: 0 none, 1 griddepcontrol.wait before the first consume, 2 at the end
template <int MODE, int R, int SB, int WAIT>
__global__ void stream_kernel(const uint8_t *__restrict__ src, int64_t bpw, int *out) {
  extern __shared__ __align__(128) uint8_t smem[];
  asm volatile("griddepcontrol.launch_dependents;");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * nw + warp;
  const uint8_t *base = src + gw * bpw;
  uint32_t sum = 0;
  uint8_t *ring = smem + warp * R * SB;
  const int nst = (int)(bpw / SB);
  if (MODE == 1) {
    constexpr int P = SB / 512;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (k < nst)
#pragma unroll
        for (int c = 0; c < P; ++c)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(ring + k * SB + c * 512 + lane * 16)),
                       "l"(base + (int64_t)k * SB + c * 512 + lane * 16) : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    if (WAIT == 1) asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int k = 0; k < nst; ++k) {
      asm volatile("cp.async.wait_group %0;" ::"n"(R - 1) : "memory");
      __syncwarp();
      const uint8_t *s = ring + (k % R) * SB;
#pragma unroll
      for (int c = 0; c < P; ++c) sum += reinterpret_cast<const uint4 *>(s + c * 512)[lane].x;
      __syncwarp();
      if (k + R < nst)
#pragma unroll
        for (int c = 0; c < P; ++c)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(ring + (k % R) * SB + c * 512 + lane * 16)),
                       "l"(base + (int64_t)(k + R) * SB + c * 512 + lane * 16) : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  } else {
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + nw * R * SB) + warp * R;
    if (lane == 0) {
      for (int k = 0; k < R; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar + k)), "r"(1));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (int k = 0; k < R && k < nst; ++k) {
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar + k)), "r"(SB) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(ring + k * SB)),
                     "l"(base + (int64_t)k * SB), "r"(SB), "r"(smem_u32(bar + k)) : "memory");
      }
    }
    if (WAIT == 1) asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncwarp();
    for (int k = 0; k < nst; ++k) {
      uint32_t ok = 0, ph = (k / R) & 1;
      while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(bar + k % R)), "r"(ph) : "memory");
      sum += reinterpret_cast<const uint32_t *>(ring + (k % R) * SB)[lane];
      __syncwarp();
      if (lane == 0 && k + R < nst) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar + k % R)), "r"(SB) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(ring + (k % R) * SB)),
                     "l"(base + (int64_t)(k + R) * SB), "r"(SB), "r"(smem_u32(bar + k % R)) : "memory");
      }
    }
  }
  if (WAIT == 2) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (sum == 0x12345678) out[0] = 1;
}

template <int MODE, int R, int SB, int WAIT>
void run(const char *name, uint8_t *buf, size_t nbuf, int64_t bytes, int warps, int ctas_per_sm, bool pdl) {
  auto k = stream_kernel<MODE, R, SB, WAIT>;
  const int grid = 148 * ctas_per_sm;
  const int64_t nw = (int64_t)grid * warps;
  int64_t bpw = (bytes / nw) / SB * SB;
  if (bpw < SB) bpw = SB;
  size_t smem = (size_t)warps * R * SB + warps * R * 8 + 128;
  if (smem > 227 * 1024) { printf("%-30s skip (smem %zu)\n", name, smem); return; }
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int *out;
  CK(cudaMalloc(&out, 4));
  const int nrot = (int)(nbuf / (bpw * nw));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  cudaGraph_t g;
  cudaGraphExec_t ge;
  const int iters = 40;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
  for (int i = 0; i < iters; ++i) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(warps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    const uint8_t *p = buf + (size_t)(i % nrot) * bpw * nw;
    CK(cudaLaunchKernelEx(&cfg, k, p, bpw, out));
  }
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, s));
  CK(cudaStreamSynchronize(s));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a, s);
    CK(cudaGraphLaunch(ge, s));
    cudaEventRecord(b, s);
    CK(cudaStreamSynchronize(s));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  double us = best * 1000.0 / iters;
  printf("%-30s %dx%2dw pdl%d %6.1f MB %7.2f us %7.0f GB/s\n", name, ctas_per_sm, warps, (int)pdl,
         bpw * nw / 1e6, us, bpw * nw / us / 1e3);
  fflush(stdout);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(s);
  cudaFree(out);
}

int main() {
  const size_t nbuf = (size_t)2 << 30;
  uint8_t *buf;
  CK(cudaMalloc(&buf, nbuf));
  CK(cudaMemset(buf, 3, nbuf));
  for (int64_t mb : {44, 256}) {
    int64_t bytes = mb * 1000000;
    printf("---- %lld MB per launch\n", (long long)mb);
    for (int pdl = 0; pdl < 2; ++pdl) {
      run<1, 4, 2048, 0>("cp.async 4x2KB", buf, nbuf, bytes, 16, 1, pdl);
      run<1, 4, 2048, 0>("cp.async 4x2KB", buf, nbuf, bytes, 8, 2, pdl);
      run<1, 6, 2048, 0>("cp.async 6x2KB", buf, nbuf, bytes, 8, 2, pdl);
      run<1, 4, 4096, 0>("cp.async 4x4KB", buf, nbuf, bytes, 8, 1, pdl);
      run<1, 3, 4096, 0>("cp.async 3x4KB", buf, nbuf, bytes, 8, 2, pdl);
      run<2, 4, 4096, 0>("bulk 4x4KB", buf, nbuf, bytes, 8, 1, pdl);
      run<2, 4, 4096, 0>("bulk 4x4KB", buf, nbuf, bytes, 4, 2, pdl);
      run<2, 6, 4096, 0>("bulk 6x4KB", buf, nbuf, bytes, 4, 2, pdl);
      run<2, 4, 8192, 0>("bulk 4x8KB", buf, nbuf, bytes, 4, 1, pdl);
      run<2, 3, 8192, 0>("bulk 3x8KB", buf, nbuf, bytes, 4, 2, pdl);
      run<2, 8, 4096, 0>("bulk 8x4KB", buf, nbuf, bytes, 4, 1, pdl);
      run<2, 6, 8192, 0>("bulk 6x8KB", buf, nbuf, bytes, 2, 2, pdl);
    }
    // dependency variants (PDL): wait before consuming / only at the end
    run<1, 4, 2048, 1>("cp.async 4x2KB wait-early", buf, nbuf, bytes, 8, 2, true);
    run<1, 4, 2048, 2>("cp.async 4x2KB wait-end", buf, nbuf, bytes, 8, 2, true);
    run<2, 4, 4096, 2>("bulk 4x4KB wait-end", buf, nbuf, bytes, 4, 2, true);
    run<2, 6, 8192, 2>("bulk 6x8KB wait-end", buf, nbuf, bytes, 2, 2, true);
  }
  return 0;
}
