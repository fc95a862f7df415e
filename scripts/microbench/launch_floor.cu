// Device time per call (us) of near-empty launches replayed from a CUDA
// graph of 20 calls: one plain 64-CTA kernel, one cooperative kernel with a
// grid barrier (cooperative_groups), and three PDL-chained kernels - the
// floor under a single small transform's schedule.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 launch_floor.cu -o /tmp/lf
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_plain(unsigned long long *p) {
  if (threadIdx.x == 0) p[blockIdx.x] += 1;
}
__global__ void k_grid(unsigned long long *p) {
  if (threadIdx.x == 0) p[blockIdx.x] += 1;
  cooperative_groups::this_grid().sync();
  if (threadIdx.x == 0) p[blockIdx.x ^ 1] += 1;
}
// monotonic arrival counter: CTA barrier of launch k completes at
// (k + 1) * gridDim.x arrivals
__global__ void k_custom(unsigned long long *p, unsigned *ctr) {
  if (threadIdx.x == 0) p[blockIdx.x] += 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned old;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
    const unsigned target = (old / gridDim.x + 1) * gridDim.x;
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while (static_cast<int>(v - target) < 0);
  }
  __syncthreads();
  if (threadIdx.x == 0) p[blockIdx.x ^ 1] += 1;
}
__global__ void k_coop_nosync(unsigned long long *p) {
  if (threadIdx.x == 0) p[blockIdx.x] += 1;
}
__global__ void k_pdl(unsigned long long *p) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) p[blockIdx.x] += 1;
}

template <class F>
static double graph_us(F issue, cudaStream_t st) {
  cudaGraph_t g;
  cudaGraphExec_t x;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < 20; ++i) issue();
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&x, g, 0);
  for (int i = 0; i < 3; ++i) cudaGraphLaunch(x, st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  for (int i = 0; i < 10; ++i) cudaGraphLaunch(x, st);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e3 / 200;
}

// per call, `calls` separate submissions (no graph batching): the device
// timeline when the host submits one call at a time
template <class F>
static double stream_us(F issue, cudaStream_t st, int calls = 50) {
  for (int i = 0; i < 5; ++i) issue();
  cudaStreamSynchronize(st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  for (int i = 0; i < calls; ++i) issue();
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e3 / calls;
}

template <class F>
static cudaGraphExec_t one_graph(F issue, cudaStream_t st) {
  cudaGraph_t g;
  cudaGraphExec_t x;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  issue();
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&x, g, 0);
  return x;
}

int main() {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  unsigned long long *p;
  cudaMalloc(&p, 1 << 16);  // [0, 4096) data, then the counter
  cudaMemset(p, 0, 1 << 16);
  for (int blocks : {64, 128}) {
    const double plain = graph_us([&] { k_plain<<<blocks, 128, 0, st>>>(p); }, st);
    const double grid = graph_us([&] {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(blocks);
      cfg.blockDim = dim3(128);
      cfg.stream = st;
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeCooperative;
      a[0].val.cooperative = 1;
      cfg.attrs = a;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k_grid, p);
    }, st);
    const double pdl3 = graph_us([&] {
      for (int i = 0; i < 3; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(blocks);
        cfg.blockDim = dim3(128);
        cfg.stream = st;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        a[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = a;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k_pdl, p);
      }
    }, st);
    auto coop = [&](auto kern, auto... args) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(blocks);
      cfg.blockDim = dim3(128);
      cfg.stream = st;
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeCooperative;
      a[0].val.cooperative = 1;
      cfg.attrs = a;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, kern, args...);
    };
    unsigned *ctr = reinterpret_cast<unsigned *>(p + 4096);
    const double coop0 = graph_us([&] { coop(k_coop_nosync, p); }, st);
    const double cust = graph_us([&] { k_custom<<<blocks, 128, 0, st>>>(p, ctr); }, st);
    const double cust_coop = graph_us([&] { coop(k_custom, p, ctr); }, st);
    std::printf("{\"blocks\": %d, \"plain_us\": %.2f, \"coop_gridsync_us\": %.2f, \"pdl_x3_us\": %.2f, "
                "\"coop_nosync_us\": %.2f, \"custom_barrier_us\": %.2f, \"custom_barrier_coop_us\": %.2f}\n",
                blocks, plain, grid, pdl3, coop0, cust, cust_coop);
  }
  {
    auto coop1 = [&] {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(128);
      cfg.blockDim = dim3(256);
      cfg.stream = st;
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeCooperative;
      a[0].val.cooperative = 1;
      cfg.attrs = a;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k_grid, p);
    };
    auto plain1 = [&] { k_plain<<<128, 256, 0, st>>>(p); };
    cudaGraphExec_t gc = one_graph(coop1, st), gp = one_graph(plain1, st);
    std::printf("{\"separate_calls\": 50, \"plain_direct_us\": %.2f, \"plain_graph_us\": %.2f, "
                "\"coop_sync_direct_us\": %.2f, \"coop_sync_graph_us\": %.2f}\n",
                stream_us(plain1, st), stream_us([&] { cudaGraphLaunch(gp, st); }, st),
                stream_us(coop1, st), stream_us([&] { cudaGraphLaunch(gc, st); }, st));
  }
  std::printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
