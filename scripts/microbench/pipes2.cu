// Issue-rate microbenchmarks for the integer instructions of the butterflies
// (sm_100a).  Every chain feeds its own result back (no loop-invariant
// operands ptxas could hoist), 8 independent chains per thread, 8 warps per
// SMSP.  Reports warp-instructions per clock per SMSP.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes2 pipes2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;
#define CH 8
template <int OP>
__global__ void k(u64 *out, int iters, uint32_t s0) {
  uint32_t a[CH], b[CH];
  u64 w[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) { a[i] = s0 * (i + 3) + threadIdx.x; b[i] = s0 ^ (i * 2654435761u); w[i] = a[i] * 77ull + b[i]; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (OP == 0) {  // IMAD.WIDE.U32, 64-bit addend, operand from own result
        asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[i]) : "r"((uint32_t)(w[i] >> 32)), "r"(b[i]));
      } else if (OP == 1) {  // IMAD (mad.lo)
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b[i]), "r"(s0));
      } else if (OP == 2) {  // IMAD.HI
        asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b[i]), "r"(s0));
      } else if (OP == 3) {  // IADD3 (3-input, own result)
        asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(a[i]) : "r"(b[i]), "r"(a[(i + 1) % CH]));
      } else if (OP == 4) {  // LOP3 xor chain
        asm volatile("xor.b32 %0, %0, %1;\n\tshf.l.wrap.b32 %0, %0, %0, 7;" : "+r"(a[i]) : "r"(b[i]));
      } else if (OP == 5) {  // 1 WIDE + 2 IADD3-class ops
        asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[i]) : "r"((uint32_t)(w[i] >> 32)), "r"(b[i]));
        asm volatile("xor.b32 %0, %0, %1;\n\tshf.l.wrap.b32 %0, %0, %0, 7;" : "+r"(a[i]) : "r"(b[i]));
      } else if (OP == 6) {  // 1 IMAD + 1 ALU
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b[i]), "r"(s0));
        asm volatile("xor.b32 %0, %0, %1;" : "+r"(b[i]) : "r"(a[i]));
      }
    }
  }
  u64 acc = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) acc ^= w[i] ^ a[i] ^ b[i];
  if (acc == 42) out[0] = acc;
}
template <int OP>
void run(const char *name, double instr_per_chain_iter) {
  u64 *out;
  cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * 4, threads = 256;  // 32 warps/SM = 8 per SMSP
  int iters = 20000;
  k<OP><<<blocks, threads>>>(out, 100, 1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<OP><<<blocks, threads>>>(out, iters, 1);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double warp_instr = (double)blocks * threads / 32 * iters * CH * instr_per_chain_iter;
  double per_smsp_clk = warp_instr / (ms * 1e-3) / (sms * 4) / (clk * 1e3);
  printf("%-34s %8.3f ms  %6.3f warp-instr/clk/SMSP (clock %d MHz)\n", name, ms, per_smsp_clk, clk / 1000);
  cudaFree(out);
}
int main() {
  run<0>("IMAD.WIDE.U32", 1);
  run<1>("IMAD (mad.lo)", 1);
  run<2>("IMAD.HI (mad.hi)", 1);
  run<3>("IADD3 x2", 2);
  run<4>("LOP3+SHF", 2);
  run<5>("WIDE + LOP3 + SHF", 3);
  run<6>("IMAD + LOP3", 2);
  return 0;
}
