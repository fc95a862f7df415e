// Pipe-throughput microbenchmarks for the integer ops the butterflies use.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu && ./pipes
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;

template <int OP>
__global__ void k(u64 *out, long long iters, uint32_t s0) {
  uint32_t a[8], b[8];
  u64 w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = s0 + i * 77 + threadIdx.x; b[i] = s0 ^ (i * 12345); w[i] = a[i]; }
  for (long long it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) {  // IMAD.WIDE.U32 with 64-bit accumulate (dependent on itself)
        asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[i]) : "r"(a[i]), "r"(b[i]));
      } else if (OP == 1) {  // IMAD (32-bit mad.lo)
        asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(a[i]) : "r"(b[i]), "r"(a[(i + 1) & 7]));
      } else if (OP == 2) {  // IADD3
        asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(b[i]));
      } else if (OP == 3) {  // mul.hi.u32 (IMAD.HI)
        asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(b[i]));
      } else if (OP == 4) {  // 64-bit add (2 ALU ops)
        asm volatile("add.u64 %0, %0, %1;" : "+l"(w[i]) : "l"((u64)b[i]));
      } else if (OP == 5) {  // mix: 1 WIDE + 1 IMAD + 2 IADD3
        asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[i]) : "r"(a[i]), "r"(b[i]));
        asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(a[i]) : "r"(b[i]), "r"(a[(i + 1) & 7]));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(b[i]) : "r"(a[i]));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(b[i]) : "r"(s0));
      }
    }
  }
  u64 acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc ^= w[i] ^ a[i] ^ b[i];
  if (acc == 42) out[0] = acc;
}

template <int OP>
void run(const char *name, int ops_per_iter) {
  u64 *out;
  cudaMalloc(&out, 8);
  int blocks = 148 * 8, threads = 256;
  long long iters = 4096;
  k<OP><<<blocks, threads>>>(out, 16, 1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<OP><<<blocks, threads>>>(out, iters, 1);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double ops = (double)blocks * threads * iters * 8 * ops_per_iter;
  double per_sm_clk = ops / (ms * 1e-3) / 148 / (clk * 1e3);
  printf("%-28s %8.3f ms  %10.1f Gop/s  %6.2f lane-ops/clk/SM (at %d MHz max)\n", name, ms,
         ops / (ms * 1e-3) / 1e9, per_sm_clk, clk / 1000);
  cudaFree(out);
}

int main() {
  run<0>("IMAD.WIDE.U32 (mad.wide)", 1);
  run<1>("IMAD (mad.lo.u32)", 1);
  run<2>("IADD3 (add.u32)", 1);
  run<3>("IMAD.HI (mul.hi.u32)", 1);
  run<4>("64-bit add (add.u64)", 1);
  run<5>("mix WIDE+IMAD+2 IADD3", 4);
  return 0;
}
