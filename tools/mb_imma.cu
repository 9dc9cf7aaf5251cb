// Issue-rate microbenchmark on B200: legacy int8 mma.sync (m16n8k32 u8.s8)
// vs IDP.4A (dp4a) vs LOP3, per SM, with 8 independent accumulator chains.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mb_imma.cu -o tools/mb_imma
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(int iters, uint32_t seed, int *out) {
  uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  int c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) {
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      } else if (OP == 1) {
        asm volatile("dp4a.u32.s32 %0, %1, %2, %0;" : "+r"(c[j][0]) : "r"(a0 + j), "r"(b0));
      } else if (OP == 3) {
        asm volatile("mma.sync.aligned.m16n8k64.row.col.s32.u4.s4.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      } else {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                     : "r"(a0), "r"(a1), "r"(b0));
      }
    }
  }
  int s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 0x1234567) out[0] = s;
}

template <int OP>
void run(const char *name, int warps, int *out) {
  const int iters = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<OP><<<148, warps * 32>>>(iters, 1, out);
  cudaEventRecord(a);
  k<OP><<<148, warps * 32>>>(iters, 1, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double inst_per_sm = (double)warps * iters * 8;
  const double cycles = ms * 1e-3 * clk * 1e3;
  printf("%-22s warps/SM %2d: %8.3f ms  %.3f warp-instr/clk/SM (at %d MHz)\n", name, warps, ms,
         inst_per_sm / cycles, clk / 1000);
}

int main() {
  int *out;
  cudaMalloc(&out, 4);
  for (int w : {4, 8, 16, 32}) {
    run<0>("mma m16n8k32 u8.s8", w, out);
    run<2>("mma m16n8k16 u8.s8", w, out);
    run<1>("dp4a", w, out);
    run<3>("mma m16n8k64 u4.s4", w, out);
  }
  return 0;
}
