// HBM streaming microbenchmark on B200: which load path reaches the roofline?
// Each variant streams `bytes` from rotating buffers (> L2) with 148 CTAs and
// per-warp contiguous ranges (the decode GEMV's access pattern), no compute.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mb_stream.cu -o tools/mb_stream
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// MODE 0: LDG.128, U loads in flight per lane
// MODE 1: cp.async.cg 16 B per lane into a per-warp ring of R stages x 2 KB
// MODE 2: cp.async.bulk per warp, ring of R stages x SB bytes (mbarrier)
template <int MODE, int U, int R, int SB>
__global__ void stream_kernel(const uint8_t *__restrict__ src, int64_t bpw, int *out) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * nw + warp;
  const uint8_t *base = src + gw * bpw;
  uint32_t sum = 0;
  if (MODE == 0) {
    const uint4 *p = reinterpret_cast<const uint4 *>(base);
    const int64_t n = bpw / 16;
    for (int64_t i = lane; i < n; i += 32 * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldg(p + i + 32 * u);
#pragma unroll
      for (int u = 0; u < U; ++u) sum += v[u].x ^ v[u].w;
    }
  } else if (MODE == 1) {
    uint8_t *ring = smem + warp * R * 2048;
    const int nst = (int)(bpw / 2048);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (k < nst)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(ring + k * 2048 + c * 512 + lane * 16)),
                       "l"(base + (int64_t)k * 2048 + c * 512 + lane * 16) : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int k = 0; k < nst; ++k) {
      asm volatile("cp.async.wait_group %0;" ::"n"(R - 1) : "memory");
      __syncwarp();
      const uint8_t *s = ring + (k % R) * 2048;
#pragma unroll
      for (int c = 0; c < 4; ++c) sum += reinterpret_cast<const uint4 *>(s + c * 512)[lane].x;
      __syncwarp();
      if (k + R < nst)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(ring + (k % R) * 2048 + c * 512 + lane * 16)),
                       "l"(base + (int64_t)(k + R) * 2048 + c * 512 + lane * 16) : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  } else {
    uint8_t *ring = smem + warp * R * SB;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + nw * R * SB) + warp * R;
    const int nst = (int)(bpw / SB);
    if (lane == 0) {
      for (int k = 0; k < R; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar + k)), "r"(1));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (int k = 0; k < R && k < nst; ++k) {
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar + k)), "r"(SB) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(ring + k * SB)),
                     "l"(base + (int64_t)k * SB), "r"(SB), "r"(smem_u32(bar + k)) : "memory");
      }
    }
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
  if (sum == 0x12345678) out[0] = 1;
}

template <int MODE, int U, int R, int SB>
void run(const char *name, uint8_t *buf, size_t nbuf, int64_t bytes, int warps) {
  auto k = stream_kernel<MODE, U, R, SB>;
  const int64_t nw = 148LL * warps;
  const int64_t gran = MODE == 2 ? SB : (MODE == 1 ? 2048 : 512 * U);
  int64_t bpw = (bytes / nw) / gran * gran;
  if (bpw < gran) bpw = gran;
  size_t smem = MODE == 0 ? 0 : (size_t)warps * R * (MODE == 1 ? 2048 : SB) + warps * R * 8 + 128;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int *out;
  CK(cudaMalloc(&out, 4));
  const int nrot = (int)(nbuf / (bpw * nw));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  cudaGraph_t g;
  cudaGraphExec_t ge;
  const int iters = 24;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
  for (int i = 0; i < iters; ++i)
    k<<<148, warps * 32, smem, s>>>(buf + (size_t)(i % nrot) * bpw * nw, bpw, out);
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
  double us = ms * 1000.0 / iters;
  fflush(stdout);
  printf("%-34s warps %2d  %6.1f MB  %7.2f us  %7.0f GB/s  (rot %d)\n", name, warps,
         bpw * nw / 1e6, us, bpw * nw / us / 1e3, nrot);
}

int main() {
  const size_t nbuf = (size_t)1 << 30;
  uint8_t *buf;
  CK(cudaMalloc(&buf, nbuf));
  CK(cudaMemset(buf, 3, nbuf));
  for (int64_t mb : {15, 44}) {
    int64_t bytes = mb << 20;
    printf("---- %lld MB per launch\n", (long long)mb);
    run<0, 4, 1, 1>("LDG.128 x4", buf, nbuf, bytes, 16);
    run<0, 8, 1, 1>("LDG.128 x8", buf, nbuf, bytes, 16);
    run<0, 8, 1, 1>("LDG.128 x8", buf, nbuf, bytes, 32);
    run<0, 16, 1, 1>("LDG.128 x16", buf, nbuf, bytes, 16);
    run<1, 1, 4, 1>("cp.async 4x2KB ring", buf, nbuf, bytes, 16);
    run<1, 1, 4, 1>("cp.async 4x2KB ring", buf, nbuf, bytes, 24);
    run<1, 1, 6, 1>("cp.async 6x2KB ring", buf, nbuf, bytes, 16);
    run<2, 1, 4, 2048>("bulk 4x2KB ring", buf, nbuf, bytes, 16);
    run<2, 1, 4, 4096>("bulk 4x4KB ring", buf, nbuf, bytes, 8);
    run<2, 1, 3, 8192>("bulk 3x8KB ring", buf, nbuf, bytes, 8);
    run<2, 1, 4, 8192>("bulk 4x8KB ring", buf, nbuf, bytes, 4);
    run<2, 1, 2, 16384>("bulk 2x16KB ring", buf, nbuf, bytes, 4);
  }
  return 0;
}
