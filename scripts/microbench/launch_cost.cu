// Host issue cost per call (us) of: a plain <<<>>> launch, cudaLaunchKernelEx
// with the programmatic-stream-serialization attribute, three PDL launches,
// and cudaGraphLaunch of a captured 1- and 3-kernel graph (with PDL edges).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 launch_cost.cu -o /tmp/lc
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(int *p) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (p && threadIdx.x == 0) p[blockIdx.x] += 1;
}

static void pdl(cudaStream_t st, int *p) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(64);
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, p);
}

template <class F>
static double per_call(F f, cudaStream_t st, int reps = 2000) {
  for (int i = 0; i < 50; ++i) f();
  cudaStreamSynchronize(st);
  double best = 1e30;
  for (int r = 0; r < 5; ++r) {
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) f();
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(st);
    double us = std::chrono::duration<double, std::micro>(t1 - t0).count() / reps;
    if (us < best) best = us;
  }
  return best;
}

int main() {
  cudaStream_t st, cap;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
  int *p;
  cudaMalloc(&p, 4096);
  cudaMemset(p, 0, 4096);
  cudaGraphExec_t g1, g3;
  for (int n : {1, 3}) {
    cudaGraph_t g;
    cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < n; ++i) pdl(cap, p);
    cudaError_t e = cudaStreamEndCapture(cap, &g);
    if (e != cudaSuccess) std::printf("capture: %s\n", cudaGetErrorString(e));
    cudaGraphInstantiate(n == 1 ? &g1 : &g3, g, 0);
  }
  std::printf("{\"plain_us\": %.2f, ", per_call([&] { k<<<64, 128, 0, st>>>(p); }, st));
  std::printf("\"pdl_ex_us\": %.2f, ", per_call([&] { pdl(st, p); }, st));
  std::printf("\"pdl_x3_us\": %.2f, ", per_call([&] { pdl(st, p); pdl(st, p); pdl(st, p); }, st));
  std::printf("\"graph1_us\": %.2f, ", per_call([&] { cudaGraphLaunch(g1, st); }, st));
  std::printf("\"graph3_us\": %.2f, ", per_call([&] { cudaGraphLaunch(g3, st); }, st));
  int d;
  std::printf("\"getdevice_us\": %.3f, ", per_call([&] { cudaGetDevice(&d); }, st, 100000));
  std::printf("\"getlasterror_us\": %.3f}\n", per_call([&] { cudaGetLastError(); }, st, 100000));
  std::printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
