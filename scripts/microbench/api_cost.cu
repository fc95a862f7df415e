// Host cost of ONE nttmul_ntt_ct call with an idle device queue (median of
// 500 calls, each timed alone and followed by a synchronize), on the legacy
// default stream and on a non-blocking stream.  Link against the built
// library; run with and without NTTB_NO_GRAPH=1.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I include api_cost.cu \
//     -L paper_2209_01290_b200 -lnttmul_b200 -Xlinker -rpath=$PWD/paper_2209_01290_b200
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "nttmul_b200.h"

int main() {
  const uint64_t q = 1152921504606830593ULL;  // 2^60 - 2^14 + 1 (any odd q works here)
  cudaStream_t nb;
  cudaStreamCreateWithFlags(&nb, cudaStreamNonBlocking);
  for (int log_n : {13, 16}) {
    const size_t n = size_t(1) << log_n;
    uint64_t *a, *tw;
    cudaMalloc(&a, n * 8);
    cudaMalloc(&tw, n * 16);
    cudaMemset(a, 0, n * 8);
    cudaMemset(tw, 0, n * 16);
    for (int which = 0; which < 2; ++which) {
      cudaStream_t st = which ? nb : nullptr;
      std::vector<double> t;
      for (int i = 0; i < 520; ++i) {  // (back-to-back variant below)
        auto t0 = std::chrono::steady_clock::now();
        int s = nttmul_ntt_ct(a, tw, q, 0, 0, 0, 0, 0, log_n, 1, st);
        auto t1 = std::chrono::steady_clock::now();
        cudaStreamSynchronize(st);
        if (s) { std::printf("err %d %s\n", s, nttmul_last_error()); return 1; }
        if (i >= 20) t.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
      }
      std::sort(t.begin(), t.end());
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, st);
      auto b0 = std::chrono::steady_clock::now();
      for (int i = 0; i < 200; ++i) nttmul_ntt_ct(a, tw, q, 0, 0, 0, 0, 0, log_n, 1, st);
      auto b1 = std::chrono::steady_clock::now();
      cudaEventRecord(e1, st);
      cudaStreamSynchronize(st);
      float dev_ms = 0;
      cudaEventElapsedTime(&dev_ms, e0, e1);
      const double b2b = std::chrono::duration<double, std::micro>(b1 - b0).count() / 200;
      std::printf("{\"log_n\": %d, \"stream\": \"%s\", \"median_us\": %.2f, \"p10_us\": %.2f, "
                  "\"back_to_back_us\": %.2f, \"back_to_back_device_us\": %.2f}\n",
                  log_n, which ? "nonblocking" : "legacy", t[t.size() / 2], t[t.size() / 10], b2b,
                  dev_ms * 1e3 / 200);
    }
    cudaFree(a);
    cudaFree(tw);
  }
  return 0;
}
