// capi.cu - extern "C" entry points (include/nttmul_b200.h) and launchers.
//
// Every function validates sizes, alignment and device-pointer-ness, launches
// on the caller's stream and returns a status code; it never aborts and never
// synchronizes (except where documented).  Reference interfaces replaced are
// cited per function in the header.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <map>
#include <mutex>
#include <utility>

#include "nttmul_b200.h"
#include "ntt_kernels.cuh"
#include "cluster_kernels.cuh"
#include "grid_kernels.cuh"
#include "verify_kernels.cuh"
#include "crt_kernels.cuh"

using namespace nttb;

namespace {

thread_local char g_err[256] = "";

int fail(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_status(const char *what) {
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return NTTMUL_OK;
  return fail(NTTMUL_ELAUNCH, "%s: %s", what, cudaGetErrorString(e));
}

typedef unsigned __int128 u128;

inline u64 mulmod_host(u64 a, u64 b, u64 q) {
  return static_cast<u64>((static_cast<u128>(a) * b) % q);
}
inline u64 shoup_host(u64 w, u64 q) {
  return static_cast<u64>((static_cast<u128>(w) << 64) / q);
}
inline int bitlen(u64 x) { return x ? 64 - __builtin_clzll(x) : 0; }

int check_dev(const void *p, size_t align, const char *name) {
  if (!p) return fail(NTTMUL_EPTR, "%s is NULL", name);
  if (reinterpret_cast<uintptr_t>(p) % align)
    return fail(NTTMUL_EALIGN, "%s not %zu-byte aligned", name, align);
  // cudaPointerGetAttributes costs ~1 us of host time per call: remember
  // the last few device pointers this thread validated (device addresses
  // never turn into host addresses under UVA; a freed one passed again is
  // the caller's use-after-free, which the reference does not check either)
  thread_local const void *seen[16] = {};
  thread_local int next = 0;
  for (const void *s : seen)
    if (s == p) return NTTMUL_OK;
  cudaPointerAttributes at;
  const cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(NTTMUL_EPTR, "%s: %s", name, cudaGetErrorString(e));
  }
  if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged)
    return fail(NTTMUL_EPTR, "%s is not device memory", name);
  seen[next] = p;
  next = (next + 1) % 16;
  return NTTMUL_OK;
}

#define CHECK(x)                    \
  do {                              \
    const int _s = (x);             \
    if (_s != NTTMUL_OK) return _s; \
  } while (0)

inline cudaStream_t S(void *s) { return static_cast<cudaStream_t>(s); }

inline unsigned grid_for(long long n, int threads, long long cap = 148LL * 64) {
  long long g = (n + threads - 1) / threads;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g < 1 ? 1 : g);
}

// ---- dynamic shared memory opt-in (once per kernel and device) ------------
// cudaFuncSetAttribute costs host time on every call; remember the largest
// size already granted per (kernel, device).
template <class K>
int smem_optin(K kernel, size_t bytes) {
  if (bytes <= 48 * 1024) return NTTMUL_OK;
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, size_t> granted;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_pair(reinterpret_cast<const void *>(kernel), dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = granted.find(key);
  if (it != granted.end() && it->second >= bytes) return NTTMUL_OK;
  const cudaError_t e = cudaFuncSetAttribute(
      kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (e != cudaSuccess)
    return fail(NTTMUL_ECUDA, "smem opt-in %zu B: %s", bytes, cudaGetErrorString(e));
  granted[key] = bytes;
  return NTTMUL_OK;
}

// The largest shared-memory carveout for kernels whose residency is set by
// their shared memory (the CRT kernels: 26 KB per 128-thread block).  Left
// to the driver, the carveout - and with it the blocks per SM - varied from
// run to run (crt_decompose 0.031 .. 0.088 ms per polynomial).
template <class K>
int prefer_smem(K kernel) {
  static std::atomic<unsigned long long> done{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ULL << (dev & 63);
  if (done.load() & bit) return NTTMUL_OK;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared) != cudaSuccess)
    return cuda_status("shared memory carveout");
  done.fetch_or(bit);
  return NTTMUL_OK;
}

// ---- launch with programmatic dependent launch ------------------------------
// The column / row kernels of a transform are launched with programmatic
// stream serialization: each may be scheduled while its predecessor's last
// wave still runs and waits (griddepcontrol.wait) for its results, so the
// launch gaps between the three launches of a product disappear
// (ntt_kernels.cuh pdl_wait).  NTTB_NO_PDL=1 (environment) launches plainly.
template <class K, class Arg>
int launch_pdl(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t st, const Arg &arg) {
  static const bool off = std::getenv("NTTB_NO_PDL") != nullptr;
  if (grid.x == 0) return NTTMUL_OK;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = off ? 0 : 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, arg);
  if (e != cudaSuccess) return fail(NTTMUL_ELAUNCH, "launch: %s", cudaGetErrorString(e));
  return NTTMUL_OK;
}

// ---- row kernel dispatch ---------------------------------------------------
#ifndef NTTB_ROW_PF
// L2 prefetch of the rows one resident wave ahead: measured slower since the
// launches overlap (PDL): row kernel 0.5213 -> 0.5168 ms without it, cfg2
// +1.2 % (r2 A/B, 2 runs each); off
#define NTTB_ROW_PF 0
#endif
template <int LOG_R, int FWD, bool MID, int INV, int MODE, int LB>
int launch_row_t(const RowParams &P, long long rows, cudaStream_t st) {
  constexpr int NP = MID ? 2 : 1;
  const size_t smem = NP * RowGeom<LOG_R>::PADN * sizeof(u64);
  auto k = row_kernel<LOG_R, FWD, MID, INV, MODE, LB>;
  CHECK(smem_optin(k, smem));
  static long long slots = 0;  // resident CTAs per device for this instantiation
  if (!slots) {
    int dev = 0, sms = 148, nb = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, RowGeom<LOG_R>::T, smem) !=
            cudaSuccess || nb < 1) {
      cudaGetLastError();
      nb = 1;
    }
    slots = static_cast<long long>(nb) * sms;
    if (std::getenv("NTTB_DEBUG_OCC"))
      std::fprintf(stderr, "row_kernel<%d,%d,%d,%d,%d,%d>: %d CTAs/SM, smem %zu\n", LOG_R, FWD,
                   int(MID), INV, MODE, LB, nb, smem);
  }
  RowParams Q = P;
  Q.nrows = rows;
  Q.pf_dist = NTTB_ROW_PF ? slots : 0;
  CHECK(launch_pdl(k, dim3(static_cast<unsigned>(rows)), dim3(RowGeom<LOG_R>::T), smem, st, Q));
  return cuda_status("row_kernel");
}

template <int FWD, bool MID, int INV, int MODE, int LB>
int launch_row_m(int log_r, const RowParams &P, long long rows, cudaStream_t st) {
  switch (log_r) {
    case 10: return launch_row_t<10, FWD, MID, INV, MODE, LB>(P, rows, st);
    case 11: return launch_row_t<11, FWD, MID, INV, MODE, LB>(P, rows, st);
    case 12: return launch_row_t<12, FWD, MID, INV, MODE, LB>(P, rows, st);
    case 13: return launch_row_t<13, FWD, MID, INV, MODE, LB>(P, rows, st);
  }
  return fail(NTTMUL_EINVAL, "row size 2^%d unsupported", log_r);
}

// ---- fused row kernel ---------------------------------------------------------
template <int MODE, int LB>
int launch_row_fused(int log_r, const RowParams &P, long long rows, cudaStream_t st) {
  return launch_row_m<FWD_TRUNC, true, INV_SKIP, MODE, LB>(log_r, P, rows, st);
}

// ---- column kernel dispatch -------------------------------------------------
template <bool INV, int LB, int LOG_R>
int launch_col_r(int log_n1, const ColParams &P, cudaStream_t st) {
  const long long total = P.nsrc * (P.npolys << LOG_R);  // columns
#define NTTB_COL(LN)                                                                 \
  CHECK(launch_pdl(col_kernel<LN, INV, LB, LOG_R>,                                     \
                   dim3(static_cast<unsigned>(total / ColGeom<INV, LN, LOG_R>::SPAN)), \
                   dim3(COL_THREADS), 0, st, P))
  switch (log_n1) {
    case 1: NTTB_COL(1); break;
    case 2: NTTB_COL(2); break;
    case 3: NTTB_COL(3); break;
    case 4: NTTB_COL(4); break;
    case 5: NTTB_COL(5); break;
    default: return fail(NTTMUL_EINVAL, "column count 2^%d unsupported", log_n1);
  }
#undef NTTB_COL
  return cuda_status("col_kernel");
}

template <bool INV, int LB>
int launch_col(int log_n1, int log_r, const ColParams &P, cudaStream_t st) {
  switch (log_r) {
    case 10: return launch_col_r<INV, LB, 10>(log_n1, P, st);
    case 11: return launch_col_r<INV, LB, 11>(log_n1, P, st);
    case 12: return launch_col_r<INV, LB, 12>(log_n1, P, st);
    case 13: return launch_col_r<INV, LB, 13>(log_n1, P, st);
  }
  return fail(NTTMUL_EINVAL, "row length 2^%d unsupported", log_r);
}

// ---- strided column passes (latency schedule) --------------------------------
template <bool INV, int LB>
int launch_pass(int r, const PassParams &P, cudaStream_t st) {
  const long long units = P.npolys << (P.log_n - r);
  const dim3 grid(static_cast<unsigned>((units + PASS_THREADS - 1) / PASS_THREADS));
  switch (r) {
    case 1: CHECK(launch_pdl(pass_kernel<1, INV, LB>, grid, dim3(PASS_THREADS), 0, st, P)); break;
    case 2: CHECK(launch_pdl(pass_kernel<2, INV, LB>, grid, dim3(PASS_THREADS), 0, st, P)); break;
    case 3: CHECK(launch_pdl(pass_kernel<3, INV, LB>, grid, dim3(PASS_THREADS), 0, st, P)); break;
    default: return fail(NTTMUL_EINVAL, "pass of %d stages", r);
  }
  return cuda_status("pass_kernel");
}

// The column stages [0, c) of the latency schedule as passes of <= 3 stages
// (balanced: 4 -> 2 + 2, 5 -> 3 + 2, 6 -> 3 + 3, 7 -> 3 + 2 + 2).
inline int pass_plan(int c, int *r) {
  const int np = (c + 2) / 3;
  for (int i = 0; i < np; ++i) r[i] = c / np + (i < c % np ? 1 : 0);
  return np;
}

// Row length of the latency schedule: 2^10 words, 2^11 at n = 2^17
// (latency sweep over 2^10 .. 2^13 rows, profiles/r2/latency_rows_r2.jsonl:
// 2^17 ntt 13.1 -> 11.3 us, intt 12.2 -> 11.6 us; longer rows lose at every
// smaller size).
inline int lat_log_r(int log_n) { return log_n >= 17 ? 11 : 10; }

// ---- radix split of n > 4096 into N1 columns x N2 = 2^log_r row length ----
// Default 2^12 rows; nttmul_set_split picks 2^10 .. 2^13 per size (cfg5
// sweep).  Index = log_n; 0 = default.
int g_split[NTTMUL_MAX_LOG_N + 1] = {0};

// Default split (cfg5 sweep r2, profiles/r2/cfg5_sweep_r2.jsonl): the fused
// product keeps 4096-word rows at every size (its row kernel carries the
// Karatsuba middle); the standalone transforms use 1024-word rows up to
// n = 2^15 (more, smaller CTAs: -35 % single-transform latency at 2^13 /
// 2^14, -3..-8 % per transform batched), 2048-word rows for a single 2^16
// transform (latency) and 4096-word rows for batched 2^16 and for 2^17.
inline int row_log(int log_n, bool xform = false, long long npolys = 0) {
  if (log_n <= COL_LOG_R) return log_n;
  const int r = g_split[log_n];
  if (r) return r;
  if (!xform) return COL_LOG_R;
  if (log_n <= 15) return 10;
  if (log_n == 16) return npolys <= 4 ? 11 : COL_LOG_R;
  return COL_LOG_R;
}

// ---- small kernel -----------------------------------------------------------
template <int LB>
int launch_small(const SmallParams &P, int mode, long long npolys, cudaStream_t st) {
  const int n = 1 << P.log_n;
  const int threads = n / 2 < 32 ? 32 : (n / 2 > 256 ? 256 : n / 2);
  const size_t smem = (P.mid ? 2 : 1) * static_cast<size_t>(n) * sizeof(u64);
  switch (mode) {
    case 0: CHECK(smem_optin(small_kernel<0, LB>, smem));
      small_kernel<0, LB><<<static_cast<unsigned>(npolys), threads, smem, st>>>(P); break;
    case 1: CHECK(smem_optin(small_kernel<1, LB>, smem));
      small_kernel<1, LB><<<static_cast<unsigned>(npolys), threads, smem, st>>>(P); break;
    default: CHECK(smem_optin(small_kernel<2, LB>, smem));
      small_kernel<2, LB><<<static_cast<unsigned>(npolys), threads, smem, st>>>(P); break;
  }
  return cuda_status("small_kernel");
}

// ---- cluster kernel (one thread-block cluster per polynomial) ------------
// Schedule per transform size for n = 2^13 .. 2^16: the three-launch
// column / row / column pipeline through HBM or the single cluster launch
// (cluster_kernels.cuh).  Index = log_n; NTTMUL_SCHED_* values.
int g_sched_fused[NTTMUL_MAX_LOG_N + 1] = {0};
int g_sched_xform[NTTMUL_MAX_LOG_N + 1] = {0};

template <int LOG_N1, int KIND, int MODE, int LB>
int launch_cluster_t(const ClusterParams &P, long long npolys, cudaStream_t st) {
  using C = ClusterGeom<LOG_N1>;
  constexpr int NP = KIND == CL_FUSED ? 2 : 1;
  constexpr size_t smem =
      (KIND == CL_INV ? C::G::PADN : (NP * C::G::PADN + C::N2)) * sizeof(u64);
  auto k = cluster_kernel<LOG_N1, KIND, MODE, LB>;
  CHECK(smem_optin(k, smem));
  static std::atomic<unsigned long long> ready{0};  // cluster-size opt-in done, per device
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ULL << (dev & 63);
  if (C::N1 > 8 && !(ready.load() & bit)) {
    if (cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
        cudaSuccess)
      return cuda_status("cluster size 16 opt-in");
    ready.fetch_or(bit);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(npolys << LOG_N1));
  cfg.blockDim = dim3(C::T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C::N1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static bool told = false;
  if (!told && std::getenv("NTTB_DEBUG_OCC")) {
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, k, &cfg) != cudaSuccess) cudaGetLastError();
    std::fprintf(stderr, "cluster_kernel<%d,%d,%d,%d>: %d active clusters of %d CTAs, smem %zu\n",
                 LOG_N1, KIND, MODE, LB, nc, C::N1, smem);
    told = true;
  }
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k, P);
  if (e != cudaSuccess) return fail(NTTMUL_ELAUNCH, "cluster_kernel: %s", cudaGetErrorString(e));
  return cuda_status("cluster_kernel");
}

template <int KIND, int MODE, int LB>
int launch_cluster(int log_n1, const ClusterParams &P, long long npolys, cudaStream_t st) {
  if (npolys == 0) return NTTMUL_OK;
  switch (log_n1) {
    case 1: return launch_cluster_t<1, KIND, MODE, LB>(P, npolys, st);
    case 2: return launch_cluster_t<2, KIND, MODE, LB>(P, npolys, st);
    case 3: return launch_cluster_t<3, KIND, MODE, LB>(P, npolys, st);
    case 4: return launch_cluster_t<4, KIND, MODE, LB>(P, npolys, st);
  }
  return fail(NTTMUL_EINVAL, "cluster schedule: 2^%d rows unsupported", log_n1);
}

// Default schedule (NTTMUL_SCHED_AUTO) per size, from the round-2
// measurements (profiles/r2/NOTES.md).
// Latency schedule of the standalone transforms before the grid kernel:
// strided passes + rows of 2^10 (2^11 at 2^17), three or four PDL-chained
// launches (latency_sweep r2, profiles/r2/latency_r2.jsonl: 2^16 ntt 9.9 ->
// 7.9 us over the column / row kernels).  Superseded by the one-launch grid
// schedule for single transforms; kept as NTTMUL_SCHED_PASSES.
inline bool use_passes(int log_n, long long /*npolys*/, bool /*inverse*/) {
  if (log_n <= COL_LOG_R || g_split[log_n]) return false;
  return g_sched_xform[log_n] == NTTMUL_SCHED_PASSES;
}

inline bool use_cluster(const int *table, int log_n, long long npolys) {
  if (log_n <= COL_LOG_R || log_n > COL_LOG_R + 4) return false;
  if (g_split[log_n] && g_split[log_n] != COL_LOG_R) return false;  // rows of 4096 only
  const int s = table[log_n];
  if (s == NTTMUL_SCHED_THREE) return false;
  if (s == NTTMUL_SCHED_CLUSTER) return true;
  // auto (schedule_sweep / cfg5 sweep r2, profiles/r2/NOTES.md): the
  // cluster launch wins only for the fused product at n = 2^13 with up to
  // ~1k limb-products (-3 %); the three launches win for larger batches and
  // sizes (their column passes overlap the row kernel of the other stream
  // half; a cluster CTA waits on its own HBM phases), and the 1024-word
  // split beats the cluster for single transforms.
  return table == g_sched_fused && log_n == COL_LOG_R + 1 && npolys <= 1024;
}

// ---- grid kernel (one cooperative launch per transform) -------------------
// Rows of 2^B words, 2^A = n / 2^B CTAs per polynomial, 2^LOG_E elements
// per thread and pass (grid_kernels.cuh).  Geometry per size from the grid
// sweep (scripts/grid_sweep.py, profiles/r2/grid_sweep_r2.jsonl): one
// element pair per thread (LOG_E = 1) up to 2^16, pairs of pairs at 2^17.
// The grid barrier slot table of the current device (the launch picks its
// slot from %gridid); nullptr = cooperative launch + cooperative_groups
// grid sync, selected by NTTB_GRID_COOP=1.
int grid_barrier_slot(unsigned **slots) {
  static const bool coop = std::getenv("NTTB_GRID_COOP") != nullptr;
  *slots = nullptr;
  if (coop) return NTTMUL_OK;
  thread_local unsigned *base[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cuda_status("device");
  if (!base[dev]) {
    void *p = nullptr;
    if (cudaGetSymbolAddress(&p, g_grid_barriers) != cudaSuccess)
      return cuda_status("grid barrier slots");
    base[dev] = static_cast<unsigned *>(p);
  }
  *slots = base[dev];
  return NTTMUL_OK;
}

// A grid launch that would not fit co-resident: an error when the schedule
// was forced (NTTMUL_SCHED_GRID), else NTTB_DECLINED and the caller falls
// back to the multi-launch schedule.
constexpr int NTTB_DECLINED = -1;

template <int A, int B, int LOG_E, bool INV, int KIND, int LB>
int launch_grid_t(GridParams P, long long npolys, bool forced, cudaStream_t st) {
  using G = GridGeom<A, B, LOG_E>;
  const size_t smem = grid_smem_bytes<A, B, LOG_E>();
  auto k = grid_kernel<A, B, LOG_E, INV, KIND, LB>;
  CHECK(smem_optin(k, smem));
  // every CTA of the launch must be resident at once (grid barrier)
  static std::atomic<int> cap{0};
  if (!cap.load()) {
    int per_sm = 0, sms = 0, dev = 0;
    cudaGetDevice(&dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, G::T, smem) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      return cuda_status("grid occupancy");
    cap.store(per_sm * sms);
  }
  const long long blocks = npolys << A;
  if (blocks > cap.load()) {
    if (!forced) return NTTB_DECLINED;
    return fail(NTTMUL_EINVAL, "grid schedule: %lld CTAs exceed the %d co-resident", blocks,
                cap.load());
  }
  CHECK(grid_barrier_slot(&P.barrier));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(blocks));
  cfg.blockDim = dim3(G::T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = P.barrier ? 0 : 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k, P);
  if (e != cudaSuccess) return fail(NTTMUL_ELAUNCH, "grid_kernel: %s", cudaGetErrorString(e));
  return cuda_status("grid_kernel");
}

// log_n -> instantiation.  Built with -DNTTB_GRID_SWEEP, the forward
// (< 2^60 moduli) and inverse kernels of every (A, LOG_E) of the sweep are
// instantiated too and NTTB_GRID_A / NTTB_GRID_E select one.
template <bool INV, int KIND, int LB>
int launch_grid(int log_n, const GridParams &P, long long npolys, bool forced, cudaStream_t st) {
#ifdef NTTB_GRID_SWEEP
  if constexpr ((!INV && LB == 16 && KIND == FWD_FULL) || (INV && LB == 8 && KIND == INV_FULL)) {
    static const int A = std::getenv("NTTB_GRID_A") ? std::atoi(std::getenv("NTTB_GRID_A")) : 0;
    static const int E = std::getenv("NTTB_GRID_E") ? std::atoi(std::getenv("NTTB_GRID_E")) : 0;
#define NTTB_G(LN, AV, EV)                \
  if (log_n == LN && A == AV && E == EV) \
    return launch_grid_t<AV, LN - AV, EV, INV, KIND, LB>(P, npolys, forced, st);
#define NTTB_GE(LN, AV) NTTB_G(LN, AV, 1) NTTB_G(LN, AV, 2) NTTB_G(LN, AV, 3)
    NTTB_GE(13, 5) NTTB_GE(13, 6)
    NTTB_GE(14, 6) NTTB_GE(14, 7)
    NTTB_GE(15, 6) NTTB_GE(15, 7)
    NTTB_GE(16, 7) NTTB_GE(16, 8)
    NTTB_GE(17, 7) NTTB_GE(17, 8)
#undef NTTB_GE
#undef NTTB_G
  }
#endif
  switch (log_n) {
    case 13: return launch_grid_t<5, 8, 1, INV, KIND, LB>(P, npolys, forced, st);
    case 14: return launch_grid_t<7, 7, 1, INV, KIND, LB>(P, npolys, forced, st);
    case 15: return launch_grid_t<7, 8, 1, INV, KIND, LB>(P, npolys, forced, st);
    case 16: return launch_grid_t<7, 9, 1, INV, KIND, LB>(P, npolys, forced, st);
    case 17: return launch_grid_t<7, 10, 2, INV, KIND, LB>(P, npolys, forced, st);
  }
  return fail(NTTMUL_EINVAL, "grid schedule: n = 2^%d unsupported", log_n);
}

// Fused product in one launch (grid_fused_kernel): rows as for the
// standalone grid schedule, one element pair per thread.  Returns
// NTTB_DECLINED when the launch would not fit co-resident and the schedule
// was not forced.

template <int A, int B, int MODE, int LB>
int launch_grid_fused_t(GridFusedParams P, long long npolys, bool forced, cudaStream_t st) {
  using G = GridGeom<A, B, 1>;
  const size_t smem = grid_fused_smem_bytes<A, B>();
  auto k = grid_fused_kernel<A, B, MODE, LB>;
  CHECK(smem_optin(k, smem));
  static std::atomic<int> cap{0};
  if (!cap.load()) {
    int per_sm = 0, sms = 0, dev = 0;
    cudaGetDevice(&dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, G::T, smem) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      return cuda_status("grid occupancy");
    cap.store(per_sm * sms);
  }
  const long long blocks = npolys << A;
  if (blocks > cap.load()) {
    if (!forced) return NTTB_DECLINED;
    return fail(NTTMUL_EINVAL, "grid schedule: %lld CTAs exceed the %d co-resident", blocks,
                cap.load());
  }
  CHECK(grid_barrier_slot(&P.barrier));
  if (!P.barrier) return fail(NTTMUL_EINVAL, "fused grid schedule needs a barrier slot");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(blocks));
  cfg.blockDim = dim3(G::T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k, P);
  if (e != cudaSuccess)
    return fail(NTTMUL_ELAUNCH, "grid_fused_kernel: %s", cudaGetErrorString(e));
  return cuda_status("grid_fused_kernel");
}

template <int MODE, int LB>
int launch_grid_fused(int log_n, const GridFusedParams &P, long long npolys, bool forced,
                      cudaStream_t st) {
  switch (log_n) {
    case 13: return launch_grid_fused_t<5, 8, MODE, LB>(P, npolys, forced, st);
    case 14: return launch_grid_fused_t<7, 7, MODE, LB>(P, npolys, forced, st);
    case 15: return launch_grid_fused_t<7, 8, MODE, LB>(P, npolys, forced, st);
    case 16: return launch_grid_fused_t<7, 9, MODE, LB>(P, npolys, forced, st);
    case 17: return launch_grid_fused_t<7, 10, MODE, LB>(P, npolys, forced, st);
  }
  return fail(NTTMUL_EINVAL, "grid schedule: n = 2^%d unsupported", log_n);
}

// fused product: 0 = no, 1 = auto (may decline), 2 = forced
// Auto limits per size (limb-products per call), from the grid sweeps
// (profiles/r2/grid_fused_r2.jsonl, grid_fused_big_r2.jsonl): one launch vs
// three, 2^13 x 32 products 34.6 -> 18.4 us, 2^14 x 8 26.8 -> 18.9 us (x 16
// even), 2^15 x 8 35.9 -> 22.7 us, 2^16 x 4 36.9 -> 19.2 us; above the
// co-resident CTA count the launcher declines (three launches).
inline int grid_fused_auto_max(int log_n) {
  switch (log_n) {
    case 13: return 32;
    case 14: return 8;
    case 15: return 8;
    case 16: return 4;
    default: return 2;
  }
}

// fused product: 0 = no, 1 = auto (may decline), 2 = forced
inline int use_grid_fused(int log_n, long long npolys) {
  if (log_n <= COL_LOG_R || log_n > 17 || g_split[log_n]) return 0;
  const int s = g_sched_fused[log_n];
  if (s == NTTMUL_SCHED_GRID) return 2;
  return s == NTTMUL_SCHED_AUTO && npolys <= grid_fused_auto_max(log_n) ? 1 : 0;
}

// Auto limits for the standalone transforms (grid_default_r2 /
// grid_batch_r2 / grid_big_r2.jsonl: one 2^16 ntt 8.1-9.3 -> 5.2 us; two
// 2^16 11.0 -> 6.8 us, four 11.6 -> 9.0 us; 2^13 x 8 5.8 -> 4.7 us, 2^15 x 8
// 12.6 -> 11.3 us; 2^14 x 4 even, x 8 7.9 -> 12.2 us); larger batches keep
// the column / row kernels.  Every auto geometry holds its batch x 2^A CTAs
// co-resident.
inline int grid_auto_max(int log_n) {
  switch (log_n) {
    case 13: return 8;
    case 15: return 8;
    default: return 4;
  }
}

// 0 = no, 1 = auto (may decline), 2 = forced
inline int use_grid(int log_n, long long npolys) {
  if (log_n <= COL_LOG_R || log_n > 17 || g_split[log_n]) return 0;
  const int s = g_sched_xform[log_n];
  if (s == NTTMUL_SCHED_GRID) return 2;
  return s == NTTMUL_SCHED_AUTO && npolys <= grid_auto_max(log_n) ? 1 : 0;
}

constexpr int SMALL_MAX_LOG = 9;  // n <= 2^9 -> small kernel

// ---- composite transforms -----------------------------------------------------
template <int LB>
int run_forward(u64 *a, const TwSet &tw, const LimbSet &ls, int log_n,
                long long npolys, bool truncate, cudaStream_t st) {
  if (npolys == 0) return NTTMUL_OK;
  if (log_n <= SMALL_MAX_LOG) {
    SmallParams P{a, a, nullptr, tw, ls, log_n, truncate ? FWD_TRUNC : FWD_FULL, 0,
                  INV_NONE, FIN_PLAIN};
    return launch_small<LB>(P, NTTMUL_RED_ONE_SUB, npolys, st);
  }
  const int log_r = row_log(log_n, true, npolys);
  const int log_n1 = log_n - log_r;
  if constexpr (LB == 16) {  // (instantiated for the < 2^60 moduli only)
    if (use_cluster(g_sched_xform, log_n, npolys)) {
      ClusterParams P{a, a, nullptr, tw, ls, truncate ? FWD_TRUNC : FWD_FULL, INV_NONE,
                      FIN_PLAIN};
      return launch_cluster<CL_FWD, 2, LB>(log_n - COL_LOG_R, P, npolys, st);
    }
  }
  if (const int g = use_grid(log_n, npolys)) {
    GridParams P{a, tw, ls, FIN_PLAIN, nullptr};
    const int s = truncate ? launch_grid<false, FWD_TRUNC, LB>(log_n, P, npolys, g == 2, st)
                           : launch_grid<false, FWD_FULL, LB>(log_n, P, npolys, g == 2, st);
    if (s != NTTB_DECLINED) return s;
  }
  if (use_passes(log_n, npolys, false)) {
    const int LAT_LOG_R = lat_log_r(log_n);
    const int c = log_n - LAT_LOG_R;
    int r[4];
    const int np = pass_plan(c, r);
    for (int i = 0, s0 = 0; i < np; s0 += r[i], ++i) {
      PassParams Q{a, tw, ls, log_n, s0, npolys, FIN_LAZY};
      CHECK((launch_pass<false, LB>(r[i], Q, st)));
    }
    RowParams R{a, a, nullptr, tw, ls, c, FIN_PLAIN, 0};
    return truncate ? launch_row_m<FWD_TRUNC, false, INV_NONE, 2, LB>(LAT_LOG_R, R, npolys << c, st)
                    : launch_row_m<FWD_FULL, false, INV_NONE, 2, LB>(LAT_LOG_R, R, npolys << c, st);
  }
  if (log_n1 > 0) {
    ColParams C{a, nullptr, a, nullptr, 1, npolys, tw, ls, FIN_LAZY};
    CHECK((launch_col<false, LB>(log_n1, log_r, C, st)));
  }
  RowParams R{a, a, nullptr, tw, ls, log_n1, FIN_PLAIN, 0};
  const long long rows = npolys << log_n1;
  return truncate ? launch_row_m<FWD_TRUNC, false, INV_NONE, 2, LB>(log_r, R, rows, st)
                  : launch_row_m<FWD_FULL, false, INV_NONE, 2, LB>(log_r, R, rows, st);
}

template <int LB>
int run_inverse(u64 *a, const TwSet &tw, const LimbSet &ls, int log_n,
                long long npolys, bool skip, int fin, cudaStream_t st) {
  if (npolys == 0) return NTTMUL_OK;
  if (log_n <= SMALL_MAX_LOG) {
    SmallParams P{a, a, nullptr, tw, ls, log_n, FWD_NONE, 0, skip ? INV_SKIP : INV_FULL,
                  fin};
    return launch_small<LB>(P, NTTMUL_RED_ONE_SUB, npolys, st);
  }
  const int log_r = row_log(log_n, true, npolys);
  const int log_n1 = log_n - log_r;
  if constexpr (LB == 8) {  // (the inverse of every modulus < 2^61)
    if (use_cluster(g_sched_xform, log_n, npolys)) {
      ClusterParams P{a, a, nullptr, tw, ls, FWD_NONE, skip ? INV_SKIP : INV_FULL, fin};
      return launch_cluster<CL_INV, 2, LB>(log_n - COL_LOG_R, P, npolys, st);
    }
  }
  if (const int g = use_grid(log_n, npolys)) {
    GridParams P{a, tw, ls, fin, nullptr};
    const int s = skip ? launch_grid<true, INV_SKIP, LB>(log_n, P, npolys, g == 2, st)
                       : launch_grid<true, INV_FULL, LB>(log_n, P, npolys, g == 2, st);
    if (s != NTTB_DECLINED) return s;
  }
  if (use_passes(log_n, npolys, true)) {
    const int LAT_LOG_R = lat_log_r(log_n);
    const int c = log_n - LAT_LOG_R;
    RowParams R{a, a, nullptr, tw, ls, c, fin, 0};
    CHECK((skip ? launch_row_m<FWD_NONE, false, INV_SKIP, 2, LB>(LAT_LOG_R, R, npolys << c, st)
                : launch_row_m<FWD_NONE, false, INV_FULL, 2, LB>(LAT_LOG_R, R, npolys << c, st)));
    int r[4];
    const int np = pass_plan(c, r);
    int s0 = c;
    for (int i = np - 1; i >= 0; --i) {
      s0 -= r[i];
      PassParams Q{a, tw, ls, log_n, s0, npolys, s0 == 0 ? fin : FIN_LAZY};
      CHECK((launch_pass<true, LB>(r[i], Q, st)));
    }
    return NTTMUL_OK;
  }
  RowParams R{a, a, nullptr, tw, ls, log_n1, fin, 0};
  const long long rows = npolys << log_n1;
  CHECK((skip ? launch_row_m<FWD_NONE, false, INV_SKIP, 2, LB>(log_r, R, rows, st)
              : launch_row_m<FWD_NONE, false, INV_FULL, 2, LB>(log_r, R, rows, st)));
  if (log_n1 > 0) {
    ColParams C{a, nullptr, a, nullptr, 1, npolys, tw, ls, fin};
    CHECK((launch_col<true, LB>(log_n1, log_r, C, st)));
  }
  return NTTMUL_OK;
}

// The fused product for n > 4096 is COL -> ROW -> COL^-1; the intermediates
// round-trip HBM (a' -> c, b' -> ws).  phases: bit 0 = forward column pass,
// bit 1 = row kernel, bit 2 = inverse column pass (n > 4096 only; smaller n
// always runs as one row kernel).  (Measured and removed in round 1: an
// L2-resident chunked pipeline with discard.global.L2 scratch, a persistent
// row kernel, a bulk-copy column pipeline and a cooperative group-persistent
// kernel - all slower, profiles/r1/NOTES.md.)
template <int MODE, int LB>
int run_polymul_m(u64 *c, const u64 *a, const u64 *b, u64 *ws, const TwSet &tw,
                  LimbSet ls, int log_n, long long npolys, int phases,
                  cudaStream_t st) {
  if (npolys == 0) return NTTMUL_OK;
  if (log_n <= SMALL_MAX_LOG) {
    if (!(phases & 2)) return NTTMUL_OK;
    SmallParams P{c, a, b, tw, ls, log_n, FWD_TRUNC, 1, INV_SKIP, FIN_SCALED_SKIP};
    return launch_small<LB>(P, MODE, npolys, st);
  }
  const int log_r = row_log(log_n);
  const int log_n1 = log_n - log_r;
  if (log_n1 == 0) {
    if (!(phases & 2)) return NTTMUL_OK;
    RowParams R{c, a, b, tw, ls, 0, FIN_SCALED_SKIP, 0};
    return launch_row_fused<MODE, LB>(log_r, R, npolys, st);
  }
  if (phases == 7) {
    if (const int g = use_grid_fused(log_n, npolys)) {
      GridFusedParams P{c, a, b, ws, tw, ls, nullptr};
      const int s = launch_grid_fused<MODE, LB>(log_n, P, npolys, g == 2, st);
      if (s != NTTB_DECLINED) return s;
    }
  }
  if constexpr (MODE == NTTMUL_RED_ONE_SUB && LB >= 16) {  // the proposed / dhem
    // constants with every modulus < 2^60 (the BASELINE bases)
    if (phases == 7 && use_cluster(g_sched_fused, log_n, npolys)) {
      ClusterParams P{c, a, b, tw, ls, FWD_TRUNC, INV_SKIP, FIN_SCALED_SKIP};
      return launch_cluster<CL_FUSED, MODE, LB>(log_n - COL_LOG_R, P, npolys, st);
    }
  }
  if (phases & 1) {
    ColParams C{a, b, c, ws, 2, npolys, tw, ls, FIN_LAZY};
    CHECK((launch_col<false, LB>(log_n1, log_r, C, st)));
  }
  if (phases & 2) {
    RowParams R{c, c, ws, tw, ls, log_n1, FIN_SCALED_SKIP, 1};
    CHECK((launch_row_fused<MODE, LB>(log_r, R, npolys << log_n1, st)));
  }
  if (phases & 4) {
    ColParams C{c, nullptr, c, nullptr, 1, npolys, tw, ls, FIN_SCALED_SKIP};
    CHECK((launch_col<true, LB>(log_n1, log_r, C, st)));
  }
  return NTTMUL_OK;
}

// lb: lazy bound selected from the moduli (16: all < 2^60, 8: all < 2^61,
// 4: up to 62 bits)
int run_polymul_one(int mode, int lb, u64 *c, const u64 *a, const u64 *b, u64 *ws,
                    const TwSet &tw, const LimbSet &ls, int log_n, long long npolys,
                    int phases, cudaStream_t st);

// Two-stream split of a large fused batch (n > 4096, full product): the two
// halves run on internal streams, so the HBM-bound column launches of one
// half overlap the integer-bound row launch of the other (sweep: +2.7 % on
// cfg3, scripts/stream_overlap.py; more parts or a staggered start measured
// slower, sweep_r41 / sweep_r53).  Fork / join with events on the caller's
// stream, so callers still see one ordered operation.  Streams and events
// are per host thread and device (thread_local), so concurrent callers never
// share a fork/join event.
constexpr int SPLIT_PARTS = 2;

struct SideStreams {
  cudaStream_t s[SPLIT_PARTS] = {};
  cudaEvent_t fork = nullptr, join[SPLIT_PARTS] = {};
};

int side_streams(SideStreams **out) {
  thread_local SideStreams sides[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cuda_status("device");
  SideStreams &sd = sides[dev];
  if (!sd.s[0]) {
    if (cudaEventCreateWithFlags(&sd.fork, cudaEventDisableTiming) != cudaSuccess)
      return cuda_status("split streams");
    for (int k = 0; k < SPLIT_PARTS; ++k)
      if (cudaStreamCreateWithFlags(&sd.s[k], cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&sd.join[k], cudaEventDisableTiming) != cudaSuccess)
        return cuda_status("split streams");
  }
  *out = &sd;
  return NTTMUL_OK;
}

int run_polymul(int mode, int lb, u64 *c, const u64 *a, const u64 *b, u64 *ws,
                const TwSet &tw, const LimbSet &ls, int log_n, long long npolys,
                int phases, cudaStream_t st) {
  const bool split = phases == 7 && log_n > COL_LOG_R && npolys >= 64 * SPLIT_PARTS &&
                     !(mode == NTTMUL_RED_ONE_SUB && lb >= 16 &&
                       use_cluster(g_sched_fused, log_n, npolys));
  if (!split)
    return run_polymul_one(mode, lb, c, a, b, ws, tw, ls, log_n, npolys, phases, st);
  SideStreams *sd = nullptr;
  CHECK(side_streams(&sd));
  if (cudaEventRecord(sd->fork, st) != cudaSuccess) return cuda_status("split fork");
  const long long n = 1LL << log_n;
  long long off = 0;
  for (int p = 0; p < SPLIT_PARTS; ++p) {
    const long long cnt = (npolys - off) / (SPLIT_PARTS - p);
    LimbSet lk = ls;
    lk.base = static_cast<int>((ls.base + off) % (ls.num > 0 ? ls.num : 1));
    if (cudaStreamWaitEvent(sd->s[p], sd->fork) != cudaSuccess) return cuda_status("split wait");
    CHECK(run_polymul_one(mode, lb, c + off * n, a + off * n, b + off * n, ws + off * n, tw, lk,
                          log_n, cnt, phases, sd->s[p]));
    if (cudaEventRecord(sd->join[p], sd->s[p]) != cudaSuccess ||
        cudaStreamWaitEvent(st, sd->join[p]) != cudaSuccess)
      return cuda_status("split join");
    off += cnt;
  }
  return NTTMUL_OK;
}

int run_polymul_one(int mode, int lb, u64 *c, const u64 *a, const u64 *b, u64 *ws,
                    const TwSet &tw, const LimbSet &ls, int log_n, long long npolys,
                    int phases, cudaStream_t st) {
#define NTTB_PM(M, LBV) run_polymul_m<M, LBV>(c, a, b, ws, tw, ls, log_n, npolys, phases, st)
  if (lb == 32) return NTTB_PM(2, 32);
  if (lb == 16) {
    switch (mode) {
      case 0: return NTTB_PM(0, 16);
      case 1: return NTTB_PM(1, 16);
      default: return NTTB_PM(2, 16);
    }
  }
  if (lb == 8) {
    switch (mode) {
      case 0: return NTTB_PM(0, 8);
      case 1: return NTTB_PM(1, 8);
      default: return NTTB_PM(2, 8);
    }
  }
  switch (mode) {
    case 0: return NTTB_PM(0, 4);
    case 1: return NTTB_PM(1, 4);
    default: return NTTB_PM(2, 4);
  }
#undef NTTB_PM
}

inline int lazy_bound(u64 q) { return q < (1ULL << 60) ? 16 : (q < (1ULL << 61) ? 8 : 4); }

int check_log_n(int log_n, int min_log) {
  if (log_n < min_log || log_n > NTTMUL_MAX_LOG_N)
    return fail(NTTMUL_EINVAL, "log_n=%d outside [%d, %d]", log_n, min_log,
                NTTMUL_MAX_LOG_N);
  return NTTMUL_OK;
}

// one-prime limb from the reference's (q, mode, mu, s_in, s_out); the scale
// constants use w1_inv when given (inverse transforms)
int single_limb(Limb *L, u64 q, int mode, u64 mu, int s_in, int s_out,
                int log_n, u64 w1_inv) {
  // the scale constants cost ~2 log_n 128-bit remainders on the host: keep
  // the last few limbs per thread (a plan's transforms repeat the same one)
  struct Entry {
    u64 q, mu, w1;
    int mode, s_in, s_out, log_n;
    Limb limb;
  };
  constexpr int NE = 8;
  thread_local Entry cache[NE];
  thread_local int used = 0, next = 0;
  for (int i = 0; i < used; ++i) {
    const Entry &e = cache[i];
    if (e.q == q && e.mu == mu && e.w1 == w1_inv && e.mode == mode && e.s_in == s_in &&
        e.s_out == s_out && e.log_n == log_n) {
      *L = e.limb;
      return NTTMUL_OK;
    }
  }
  CHECK(nttmul_limb_prepare(L, q, mode, mu, s_in, s_out, log_n, w1_inv));
  cache[next] = Entry{q, mu, w1_inv, mode, s_in, s_out, log_n, *L};
  next = (next + 1) % NE;
  if (used < NE) ++used;
  return NTTMUL_OK;
}

// ---- launch-graph cache -----------------------------------------------------
// A short call (a single transform or product of n >= 2^13: two to four
// launches) costs ~2.3 us of host time per cudaLaunchKernelEx on the B200
// hosts (scripts/microbench/launch_cost.cu) - more than its device time.  A
// call that repeats with identical arguments (pointers, sizes, constants,
// schedule knobs) is captured into a CUDA graph on its second occurrence
// and replayed from then on with one cudaGraphLaunch (~2 us for three
// kernels, programmatic edges kept).  Per host thread; the first occurrence
// of a key launches directly, so every kernel attribute is already set when
// the capture runs.  Skipped for work of more than GRAPH_MAX_WORDS words
// (device-bound), while the caller's stream is itself being captured, and
// under NTTB_NO_GRAPH=1.
constexpr long long GRAPH_MAX_WORDS = 1LL << 21;
std::atomic<unsigned> g_config_epoch{0};  // bumped by set_split / set_schedule

struct GraphEntry {
  u64 key[16];
  int nkey = 0;
  int dev = -1;
  unsigned epoch = 0;
  int seen = 0;  // 1 = launched directly once, 2 = graph (or -1: not capturable)
  cudaGraphExec_t exec = nullptr;
};

template <class F>
int run_graphed(const u64 *key, int nkey, long long words, cudaStream_t st, F &&issue) {
  static const bool off = std::getenv("NTTB_NO_GRAPH") != nullptr;
  if (off || words > GRAPH_MAX_WORDS) return issue(st);
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
    cudaGetLastError();
    return issue(st);
  }
  if (cs != cudaStreamCaptureStatusNone) return issue(st);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cuda_status("device");
  constexpr int NE = 16;
  thread_local GraphEntry table[NE];
  thread_local int next = 0;
  thread_local cudaStream_t cap[64] = {};
  const unsigned epoch = g_config_epoch.load(std::memory_order_relaxed);
  GraphEntry *hit = nullptr;
  for (GraphEntry &e : table)
    if (e.nkey == nkey && e.dev == dev && e.epoch == epoch &&
        std::memcmp(e.key, key, nkey * sizeof(u64)) == 0) {
      hit = &e;
      break;
    }
  if (!hit) {  // first occurrence: remember the key, launch directly
    GraphEntry &e = table[next];
    next = (next + 1) % NE;
    if (e.exec) cudaGraphExecDestroy(e.exec);  // (in-flight launches complete)
    e.exec = nullptr;
    std::memcpy(e.key, key, nkey * sizeof(u64));
    e.nkey = nkey;
    e.dev = dev;
    e.epoch = epoch;
    e.seen = 1;
    return issue(st);
  }
  if (hit->seen < 0) return issue(st);
  if (!hit->exec) {  // second occurrence: capture on a private stream
    if (dev < 0 || dev >= 64) return issue(st);
    if (!cap[dev] && cudaStreamCreateWithFlags(&cap[dev], cudaStreamNonBlocking) != cudaSuccess)
      return cuda_status("graph capture stream");
    if (cudaStreamBeginCapture(cap[dev], cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      cudaGetLastError();
      hit->seen = -1;
      return issue(st);
    }
    const int s = issue(cap[dev]);
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(cap[dev], &g);
    cudaGraphExec_t x = nullptr;
    const bool ok = s == NTTMUL_OK && e == cudaSuccess && g &&
                    cudaGraphInstantiate(&x, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    if (!ok) {
      if (std::getenv("NTTB_DEBUG_GRAPH")) std::fprintf(stderr, "graph capture failed: %d %s\n", s, cudaGetErrorString(e));
      cudaGetLastError();
      hit->seen = -1;
      return issue(st);
    }
    hit->exec = x;
    hit->seen = 2;
    if (std::getenv("NTTB_DEBUG_GRAPH")) std::fprintf(stderr, "graph captured (key %llu)\n", (unsigned long long)key[0]);
  }
  if (cudaGraphLaunch(hit->exec, st) != cudaSuccess) return cuda_status("graph launch");
  return NTTMUL_OK;
}

TwSet one_table(const u64 *pairs) {
  const ulonglong2 *t = reinterpret_cast<const ulonglong2 *>(pairs);
  return TwSet{t, t, 0};
}

}  // namespace

// =============================================================================
extern "C" {

int nttmul_abi_version(void) { return 1; }

const char *nttmul_last_error(void) { return g_err; }

int nttmul_limb_prepare(nttmul_limb_t *out, uint64_t q, int mode, uint64_t mu,
                        int s_in, int s_out, int log_n, uint64_t w1_inv) {
  if (!out) return fail(NTTMUL_EINVAL, "limb output is NULL");
  if (q < 3 || !(q & 1)) return fail(NTTMUL_EINVAL, "modulus %llu must be odd and >= 3",
                                     static_cast<unsigned long long>(q));
  const int m = bitlen(q);
  if (m > 62) return fail(NTTMUL_EINVAL, "modulus has %d bits; at most 62 supported", m);
  if (log_n < 1 || log_n > NTTMUL_MAX_LOG_N) return fail(NTTMUL_EINVAL, "log_n=%d", log_n);
  std::memset(out, 0, sizeof(*out));
  out->q = q;
  out->mode = static_cast<uint32_t>(mode);
  out->log_n = static_cast<uint32_t>(log_n);
  if (mode == NTTMUL_RED_BUILTIN) {
    out->mu_sh = 0;
    out->s_in = 0;
    out->s_hi = 0;
  } else if (mode == NTTMUL_RED_TWO_SUB || mode == NTTMUL_RED_ONE_SUB) {
    if (s_in < 0 || s_in > 63 || s_out < 1 || s_out > 127)
      return fail(NTTMUL_EINVAL, "shifts s_in=%d s_out=%d out of range", s_in, s_out);
    if (s_out <= 64) {
      const int sh = 64 - s_out;
      if (sh && (mu >> (64 - sh))) return fail(NTTMUL_EINVAL, "mu too wide for s_out=%d", s_out);
      out->mu_sh = mu << sh;
      out->s_hi = 0;
    } else {
      out->mu_sh = mu;
      out->s_hi = static_cast<uint32_t>(s_out - 64);
    }
    out->s_in = static_cast<uint32_t>(s_in);
  } else {
    return fail(NTTMUL_EINVAL, "unknown reduction mode %d", mode);
  }
  // 2^-k mod q = ((q+1)/2)^k
  const u64 half = (q + 1) >> 1;
  u64 f_full = 1, f_skip = 1;
  for (int i = 0; i < log_n; ++i) f_full = mulmod_host(f_full, half, q);
  for (int i = 0; i < log_n - 1; ++i) f_skip = mulmod_host(f_skip, half, q);
  const u64 w1 = w1_inv % q;
  const u64 g_full = mulmod_host(w1, f_full, q), g_skip = mulmod_host(w1, f_skip, q);
  const u64 full[4] = {f_full, shoup_host(f_full, q), g_full, shoup_host(g_full, q)};
  const u64 skip[4] = {f_skip, shoup_host(f_skip, q), g_skip, shoup_host(g_skip, q)};
  std::memcpy(out->sc_full, full, sizeof(full));
  std::memcpy(out->sc_skip, skip, sizeof(skip));
  return NTTMUL_OK;
}

int nttmul_twiddle_tables(uint64_t *tw_fwd, uint64_t *tw_inv, uint64_t *fwd_pairs,
                          uint64_t *inv_pairs, uint64_t q, uint64_t psi,
                          uint64_t psi_inv, int log_n, void *stream) {
  CHECK(check_log_n(log_n, 1));
  if (psi >= q || psi_inv >= q) return fail(NTTMUL_EINVAL, "psi not reduced");
  if (tw_fwd) CHECK(check_dev(tw_fwd, 8, "tw_fwd"));
  if (tw_inv) CHECK(check_dev(tw_inv, 8, "tw_inv"));
  if (fwd_pairs) CHECK(check_dev(fwd_pairs, 16, "fwd_pairs"));
  if (inv_pairs) CHECK(check_dev(inv_pairs, 16, "inv_pairs"));
  const int m = bitlen(q);
  Limb L;
  CHECK(nttmul_limb_prepare(&L, q, NTTMUL_RED_ONE_SUB,
                            static_cast<u64>((static_cast<u128>(1) << (2 * m + 1)) / q),
                            m - 2, m + 3, log_n, 1));
  const long long n = 1LL << log_n;
  twiddle_kernel<<<grid_for(n, 256, 1LL << 30), 256, 0, S(stream)>>>(
      tw_fwd, tw_inv, reinterpret_cast<ulonglong2 *>(fwd_pairs),
      reinterpret_cast<ulonglong2 *>(inv_pairs), psi, psi_inv, log_n, L);
  return cuda_status("twiddle_kernel");
}

int nttmul_shoup_pairs(uint64_t *pairs, const uint64_t *tw, uint64_t q, int64_t n,
                       void *stream) {
  if (n < 0) return fail(NTTMUL_EINVAL, "n < 0");
  if (n == 0) return NTTMUL_OK;
  if (q < 3 || bitlen(q) > 62) return fail(NTTMUL_EINVAL, "bad modulus");
  CHECK(check_dev(pairs, 16, "pairs"));
  CHECK(check_dev(tw, 8, "tw"));
  shoup_pairs_kernel<<<grid_for(n, 256, 1LL << 30), 256, 0, S(stream)>>>(
      reinterpret_cast<ulonglong2 *>(pairs), tw, q, n);
  return cuda_status("shoup_pairs_kernel");
}

int nttmul_check_twiddles(const uint64_t *tw_fwd, const uint64_t *tw_inv, uint64_t q,
                          int64_t n, uint64_t *bad_out, void *stream) {
  if (n < 1) return fail(NTTMUL_EINVAL, "n < 1");
  CHECK(check_dev(tw_fwd, 8, "tw_fwd"));
  CHECK(check_dev(tw_inv, 8, "tw_inv"));
  CHECK(check_dev(bad_out, 8, "bad_out"));
  Limb L;
  std::memset(&L, 0, sizeof(L));
  L.q = q;
  if (cudaMemsetAsync(bad_out, 0, 8, S(stream)) != cudaSuccess)
    return cuda_status("memset");
  check_twiddles_kernel<<<grid_for(n, 256, 1LL << 30), 256, 0, S(stream)>>>(
      tw_fwd, tw_inv, n, reinterpret_cast<unsigned long long *>(bad_out), L);
  return cuda_status("check_twiddles_kernel");
}

int nttmul_ntt_ct(uint64_t *a, const uint64_t *tw_pairs, uint64_t q, int mode,
                  uint64_t mu, int s_in, int s_out, int truncate, int log_n,
                  int64_t batch, void *stream) {
  CHECK(check_log_n(log_n, 1));
  if (batch < 0) return fail(NTTMUL_EINVAL, "batch < 0");
  if (batch == 0) return NTTMUL_OK;
  CHECK(check_dev(a, 8, "a"));
  CHECK(check_dev(tw_pairs, 16, "tw_pairs"));
  LimbSet ls;
  ls.table = nullptr;
  ls.num = 1;
  ls.base = 0;
  CHECK(single_limb(&ls.single, q, mode, mu, s_in, s_out, log_n, 1));
  const TwSet tw = one_table(tw_pairs);
  const bool tr = truncate != 0;
  auto issue = [&](cudaStream_t st) {
    switch (lazy_bound(q)) {
      case 16: return run_forward<16>(a, tw, ls, log_n, batch, tr, st);
      case 8: return run_forward<8>(a, tw, ls, log_n, batch, tr, st);
      default: return run_forward<4>(a, tw, ls, log_n, batch, tr, st);
    }
  };
  if (log_n <= SMALL_MAX_LOG) return issue(S(stream));  // one launch
  const u64 key[] = {1, reinterpret_cast<u64>(a), reinterpret_cast<u64>(tw_pairs), q,
                     static_cast<u64>(mode), mu, static_cast<u64>(s_in),
                     static_cast<u64>(s_out), static_cast<u64>(tr), static_cast<u64>(log_n),
                     static_cast<u64>(batch)};
  return run_graphed(key, sizeof(key) / sizeof(u64), batch << log_n, S(stream), issue);
}

int nttmul_intt_gs(uint64_t *a, const uint64_t *tw_pairs, uint64_t q, uint64_t half_q,
                   int mode, uint64_t mu, int s_in, int s_out, int scaled,
                   int skip_first, int log_n, int64_t batch, uint64_t w1_inv,
                   void *stream) {
  CHECK(check_log_n(log_n, 1));
  if (batch < 0) return fail(NTTMUL_EINVAL, "batch < 0");
  if (half_q != (q + 1) / 2) return fail(NTTMUL_EINVAL, "half_q != (q+1)/2");
  if (batch == 0) return NTTMUL_OK;
  CHECK(check_dev(a, 8, "a"));
  CHECK(check_dev(tw_pairs, 16, "tw_pairs"));
  LimbSet ls;
  ls.table = nullptr;
  ls.num = 1;
  ls.base = 0;
  CHECK(single_limb(&ls.single, q, mode, mu, s_in, s_out, log_n, w1_inv));
  const int fin = scaled ? (skip_first ? FIN_SCALED_SKIP : FIN_SCALED_FULL) : FIN_PLAIN;
  const TwSet tw = one_table(tw_pairs);
  const bool skip = skip_first != 0;
  // the inverse uses the same [0, 4q) range for LB 8 and 16
  auto issue = [&](cudaStream_t st) {
    return lazy_bound(q) >= 8 ? run_inverse<8>(a, tw, ls, log_n, batch, skip, fin, st)
                              : run_inverse<4>(a, tw, ls, log_n, batch, skip, fin, st);
  };
  if (log_n <= SMALL_MAX_LOG) return issue(S(stream));  // one launch
  const u64 key[] = {2, reinterpret_cast<u64>(a), reinterpret_cast<u64>(tw_pairs), q,
                     static_cast<u64>(mode), mu, static_cast<u64>(s_in),
                     static_cast<u64>(s_out), static_cast<u64>(fin), static_cast<u64>(skip),
                     static_cast<u64>(log_n), static_cast<u64>(batch), w1_inv};
  return run_graphed(key, sizeof(key) / sizeof(u64), batch << log_n, S(stream), issue);
}

int nttmul_fused_middle(const uint64_t *ah, const uint64_t *bh, uint64_t *ch,
                        const uint64_t *tw_pairs, uint64_t q, int mode, uint64_t mu,
                        int s_in, int s_out, int log_n, int64_t batch, void *stream) {
  CHECK(check_log_n(log_n, 2));
  if (batch < 0) return fail(NTTMUL_EINVAL, "batch < 0");
  if (batch == 0) return NTTMUL_OK;
  CHECK(check_dev(ah, 8, "ah"));
  CHECK(check_dev(bh, 8, "bh"));
  CHECK(check_dev(ch, 8, "ch"));
  CHECK(check_dev(tw_pairs, 16, "tw_pairs"));
  Limb L;
  CHECK(single_limb(&L, q, mode, mu, s_in, s_out, log_n, 1));
  const long long npairs = batch << (log_n - 1);
  const ulonglong2 *tw = reinterpret_cast<const ulonglong2 *>(tw_pairs);
  const unsigned g = grid_for(npairs, 256);
  switch (mode) {
    case 0: fused_middle_kernel<0><<<g, 256, 0, S(stream)>>>(ah, bh, ch, tw, log_n, npairs, L); break;
    case 1: fused_middle_kernel<1><<<g, 256, 0, S(stream)>>>(ah, bh, ch, tw, log_n, npairs, L); break;
    default: fused_middle_kernel<2><<<g, 256, 0, S(stream)>>>(ah, bh, ch, tw, log_n, npairs, L); break;
  }
  return cuda_status("fused_middle_kernel");
}

int nttmul_hadamard(const uint64_t *a, const uint64_t *b, uint64_t *out, int64_t n,
                    uint64_t q, int mode, uint64_t mu, int s_in, int s_out,
                    void *stream) {
  if (n < 0) return fail(NTTMUL_EINVAL, "n < 0");
  if (n == 0) return NTTMUL_OK;
  CHECK(check_dev(a, 8, "a"));
  CHECK(check_dev(b, 8, "b"));
  CHECK(check_dev(out, 8, "out"));
  Limb L;
  CHECK(single_limb(&L, q, mode, mu, s_in, s_out, 1, 1));
  const unsigned g = grid_for(n, 256);
  switch (mode) {
    case 0: hadamard_kernel<0><<<g, 256, 0, S(stream)>>>(a, b, out, n, L); break;
    case 1: hadamard_kernel<1><<<g, 256, 0, S(stream)>>>(a, b, out, n, L); break;
    default: hadamard_kernel<2><<<g, 256, 0, S(stream)>>>(a, b, out, n, L); break;
  }
  return cuda_status("hadamard_kernel");
}

int nttmul_scale(uint64_t *a, uint64_t factor, int64_t n, uint64_t q, int mode,
                 uint64_t mu, int s_in, int s_out, void *stream) {
  if (n < 0) return fail(NTTMUL_EINVAL, "n < 0");
  if (n == 0) return NTTMUL_OK;
  CHECK(check_dev(a, 8, "a"));
  Limb L;
  CHECK(single_limb(&L, q, mode, mu, s_in, s_out, 1, 1));
  const unsigned g = grid_for(n, 256);
  switch (mode) {
    case 0: scale_kernel<0><<<g, 256, 0, S(stream)>>>(a, factor, n, L); break;
    case 1: scale_kernel<1><<<g, 256, 0, S(stream)>>>(a, factor, n, L); break;
    default: scale_kernel<2><<<g, 256, 0, S(stream)>>>(a, factor, n, L); break;
  }
  return cuda_status("scale_kernel");
}

int nttmul_mulmod_loop(const uint64_t *a, const uint64_t *b, int64_t n, uint64_t q,
                       int mode, uint64_t mu, int s_in, int s_out, uint64_t passes,
                       uint64_t *sink_out, void *stream) {
  if (n < 0) return fail(NTTMUL_EINVAL, "n < 0");
  CHECK(check_dev(sink_out, 8, "sink_out"));
  if (cudaMemsetAsync(sink_out, 0, 8, S(stream)) != cudaSuccess)
    return cuda_status("memset");
  if (n == 0 || passes == 0) return NTTMUL_OK;
  CHECK(check_dev(a, 8, "a"));
  CHECK(check_dev(b, 8, "b"));
  Limb L;
  CHECK(single_limb(&L, q, mode, mu, s_in, s_out, 1, 1));
  const unsigned g = grid_for(n, 256);
  switch (mode) {
    case 0: mulmod_loop_kernel<0><<<g, 256, 0, S(stream)>>>(a, b, n, passes, sink_out, L); break;
    case 1: mulmod_loop_kernel<1><<<g, 256, 0, S(stream)>>>(a, b, n, passes, sink_out, L); break;
    default: mulmod_loop_kernel<2><<<g, 256, 0, S(stream)>>>(a, b, n, passes, sink_out, L); break;
  }
  return cuda_status("mulmod_loop_kernel");
}

int nttmul_polymul_fused_rns_phases(uint64_t *c, const uint64_t *a, const uint64_t *b,
                                    const nttmul_limb_t *limbs, const uint64_t *fwd_pairs,
                                    const uint64_t *inv_pairs, int log_n, int num_limbs,
                                    int64_t batch, int mode, uint64_t *workspace,
                                    int phases, void *stream) {
  CHECK(check_log_n(log_n, 2));
  if (num_limbs < 1) return fail(NTTMUL_EINVAL, "num_limbs < 1");
  if (batch < 0) return fail(NTTMUL_EINVAL, "batch < 0");
  if (batch == 0) return NTTMUL_OK;
  CHECK(check_dev(c, 8, "c"));
  CHECK(check_dev(a, 8, "a"));
  CHECK(check_dev(b, 8, "b"));
  CHECK(check_dev(limbs, 8, "limbs"));
  CHECK(check_dev(fwd_pairs, 16, "fwd_pairs"));
  CHECK(check_dev(inv_pairs, 16, "inv_pairs"));
  if (log_n > COL_LOG_R) {
    CHECK(check_dev(workspace, 8, "workspace"));
    if (workspace == a || workspace == c)
      return fail(NTTMUL_EINVAL, "workspace may not alias a or c");
  }
  if (c == b && log_n > COL_LOG_R)
    return fail(NTTMUL_EINVAL, "c may not alias b");
  const int lb = (mode & NTTMUL_MODE_NARROW60) ? 16 : ((mode & NTTMUL_MODE_NARROW) ? 8 : 4);
  const bool wide35 = (mode & NTTMUL_MODE_WIDE35) != 0;
  // NTTMUL_MODE_PM (shift-shaped moduli) is accepted and ignored: its
  // schedule measured slower and was removed (pm_r36)
  mode &= ~(NTTMUL_MODE_NARROW | NTTMUL_MODE_NARROW60 | NTTMUL_MODE_WIDE35 | NTTMUL_MODE_PM);
  if (mode < 0 || mode > 2) return fail(NTTMUL_EINVAL, "unknown reduction mode %d", mode);
  // lazy bound "32": the [0, 16q) ranges with multiply-based reductions
  // (every modulus in [2^34, 2^60)), for the proposed-shape constants
  int lbx = lb;
  if (mode == NTTMUL_RED_ONE_SUB && lb == 16 && wide35) lbx = 32;
  LimbSet ls;
  ls.table = limbs;
  ls.num = num_limbs;
  ls.base = 0;
  std::memset(&ls.single, 0, sizeof(ls.single));
  const long long stride = 1LL << log_n;
  TwSet tw{reinterpret_cast<const ulonglong2 *>(fwd_pairs),
           reinterpret_cast<const ulonglong2 *>(inv_pairs), stride};
  const long long npolys = batch * num_limbs;
  auto issue = [&](cudaStream_t st) {
    return run_polymul(mode, lbx, c, a, b, workspace, tw, ls, log_n, npolys, phases, st);
  };
  if (log_n <= COL_LOG_R) return issue(S(stream));  // one launch
  const u64 key[] = {3, reinterpret_cast<u64>(c), reinterpret_cast<u64>(a),
                     reinterpret_cast<u64>(b), reinterpret_cast<u64>(limbs),
                     reinterpret_cast<u64>(fwd_pairs), reinterpret_cast<u64>(inv_pairs),
                     reinterpret_cast<u64>(workspace), static_cast<u64>(log_n),
                     static_cast<u64>(num_limbs), static_cast<u64>(batch),
                     static_cast<u64>(mode), static_cast<u64>(lbx), static_cast<u64>(phases)};
  return run_graphed(key, sizeof(key) / sizeof(u64), npolys << log_n, S(stream), issue);
}

int nttmul_set_split(int log_n, int log_r) {
  if (log_n <= COL_LOG_R || log_n > NTTMUL_MAX_LOG_N ||
      (log_r != 0 && (log_r < 10 || log_r > 13 || log_n - log_r < 1 || log_n - log_r > 5)))
    return fail(NTTMUL_EINVAL, "set_split(%d, %d)", log_n, log_r);
  g_split[log_n] = log_r;
  g_config_epoch.fetch_add(1);
  return NTTMUL_OK;
}

int nttmul_set_schedule(int which, int log_n, int schedule) {
  if (which < 0 || which > 1 || log_n < COL_LOG_R + 1 || log_n > NTTMUL_MAX_LOG_N ||
      schedule < NTTMUL_SCHED_AUTO || schedule > NTTMUL_SCHED_GRID ||
      (schedule == NTTMUL_SCHED_PASSES && which == 0) ||
      (schedule == NTTMUL_SCHED_CLUSTER && log_n > COL_LOG_R + 4))
    return fail(NTTMUL_EINVAL, "set_schedule(%d, %d, %d)", which, log_n, schedule);
  (which == 0 ? g_sched_fused : g_sched_xform)[log_n] = schedule;
  g_config_epoch.fetch_add(1);
  return NTTMUL_OK;
}

int nttmul_polymul_fused_rns(uint64_t *c, const uint64_t *a, const uint64_t *b,
                             const nttmul_limb_t *limbs, const uint64_t *fwd_pairs,
                             const uint64_t *inv_pairs, int log_n, int num_limbs,
                             int64_t batch, int mode, uint64_t *workspace,
                             void *stream) {
  return nttmul_polymul_fused_rns_phases(c, a, b, limbs, fwd_pairs, inv_pairs, log_n,
                                         num_limbs, batch, mode, workspace, 7, stream);
}

// Host-buffer product: chunks of `chunk_cts` ciphertexts flow through NBUF
// device buffer sets; H2D (own stream), the fused kernels (caller's stream)
// and D2H (own stream) of different chunks overlap, so the call is bound by
// the slower PCIe direction instead of the sum of copies and compute.
int nttmul_polymul_fused_rns_host(uint64_t *c_host, const uint64_t *a_host,
                                  const uint64_t *b_host, const nttmul_limb_t *limbs,
                                  const uint64_t *fwd_pairs, const uint64_t *inv_pairs,
                                  int log_n, int num_limbs, int64_t batch, int mode,
                                  uint64_t *dev_buf, int64_t chunk_cts, void *stream) {
  constexpr int NBUF = NTTMUL_HOST_NBUF;
  CHECK(check_log_n(log_n, 2));
  if (num_limbs < 1) return fail(NTTMUL_EINVAL, "num_limbs < 1");
  if (batch < 0 || chunk_cts < 1) return fail(NTTMUL_EINVAL, "batch < 0 or chunk_cts < 1");
  if (batch == 0) return NTTMUL_OK;
  if (!c_host || !a_host || !b_host) return fail(NTTMUL_EPTR, "host buffer is NULL");
  CHECK(check_dev(dev_buf, 16, "dev_buf"));
  struct Pipe {
    cudaStream_t s_in, s_out;
    cudaEvent_t ev_start, ev_in[NBUF], ev_done[NBUF], ev_out[NBUF];
  };
  thread_local Pipe pipes[64];  // copy streams / events per host thread and device
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return cuda_status("device");
  Pipe &pp = pipes[dev];
  cudaStream_t &s_in = pp.s_in, &s_out = pp.s_out;
  cudaEvent_t &ev_start = pp.ev_start, *ev_in = pp.ev_in, *ev_done = pp.ev_done,
              *ev_out = pp.ev_out;
  if (!s_in) {
    if (cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming) != cudaSuccess)
      return cuda_status("host pipeline streams");
    for (int i = 0; i < NBUF; ++i)
      if (cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&ev_done[i], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&ev_out[i], cudaEventDisableTiming) != cudaSuccess)
        return cuda_status("host pipeline events");
  }
  const cudaStream_t sc = S(stream);
  const long long per_ct = static_cast<long long>(num_limbs) << log_n;  // words
  const long long set_words = 4 * chunk_cts * per_ct;                    // a, b, c, ws
  // copies of chunk i start only after everything queued on the caller's
  // stream before this call (the caller's timing events bracket the call)
  if (cudaEventRecord(ev_start, sc) != cudaSuccess || cudaStreamWaitEvent(s_in, ev_start) != cudaSuccess)
    return cuda_status("host pipeline start");
  const long long nchunks = (batch + chunk_cts - 1) / chunk_cts;
  for (long long i = 0; i < nchunks; ++i) {
    const int s = static_cast<int>(i % NBUF);
    const long long cts = (i + 1) * chunk_cts > batch ? batch - i * chunk_cts : chunk_cts;
    const size_t bytes = static_cast<size_t>(cts * per_ct) * sizeof(u64);
    const long long off = i * chunk_cts * per_ct;
    u64 *da = dev_buf + s * set_words, *db = da + chunk_cts * per_ct;
    u64 *dc = db + chunk_cts * per_ct, *dw = dc + chunk_cts * per_ct;
    if (i >= NBUF && cudaStreamWaitEvent(s_in, ev_done[s]) != cudaSuccess)  // a, b consumed
      return cuda_status("host pipeline wait");
    if (cudaMemcpyAsync(da, a_host + off, bytes, cudaMemcpyHostToDevice, s_in) != cudaSuccess ||
        cudaMemcpyAsync(db, b_host + off, bytes, cudaMemcpyHostToDevice, s_in) != cudaSuccess ||
        cudaEventRecord(ev_in[s], s_in) != cudaSuccess || cudaStreamWaitEvent(sc, ev_in[s]) != cudaSuccess)
      return cuda_status("host pipeline H2D");
    if (i >= NBUF && cudaStreamWaitEvent(sc, ev_out[s]) != cudaSuccess)  // c drained
      return cuda_status("host pipeline wait");
    CHECK(nttmul_polymul_fused_rns(dc, da, db, limbs, fwd_pairs, inv_pairs, log_n, num_limbs,
                                   cts, mode, dw, stream));
    if (cudaEventRecord(ev_done[s], sc) != cudaSuccess || cudaStreamWaitEvent(s_out, ev_done[s]) != cudaSuccess ||
        cudaMemcpyAsync(c_host + off, dc, bytes, cudaMemcpyDeviceToHost, s_out) != cudaSuccess ||
        cudaEventRecord(ev_out[s], s_out) != cudaSuccess)
      return cuda_status("host pipeline D2H");
  }
  // the caller's stream completes when the last result has landed in c_host
  const int last = static_cast<int>((nchunks - 1) % NBUF);
  if (cudaStreamWaitEvent(sc, ev_out[last]) != cudaSuccess) return cuda_status("host pipeline end");
  return NTTMUL_OK;
}

int nttmul_negacyclic_naive(uint64_t *out, const uint64_t *a, const uint64_t *b, uint64_t q,
                            int64_t n, int64_t batch, void *stream) {
  if (n < 1 || n > (1 << 20) || batch < 0) return fail(NTTMUL_EINVAL, "n=%lld batch=%lld",
                                                       static_cast<long long>(n),
                                                       static_cast<long long>(batch));
  if (q < 2) return fail(NTTMUL_EINVAL, "modulus %llu", static_cast<unsigned long long>(q));
  if (batch == 0) return NTTMUL_OK;
  CHECK(check_dev(out, 8, "out"));
  CHECK(check_dev(a, 8, "a"));
  CHECK(check_dev(b, 8, "b"));
  if (out == a || out == b) return fail(NTTMUL_EINVAL, "out may not alias a or b");
  const int bpp = static_cast<int>((n + NAIVE_THREADS - 1) / NAIVE_THREADS);
  naive_kernel<<<static_cast<unsigned>(batch * bpp), NAIVE_THREADS, 0, S(stream)>>>(
      out, a, b, q, static_cast<int>(n), bpp);
  return cuda_status("naive_kernel");
}

int nttmul_sweep_random(int bits, uint64_t nsamples, uint64_t seed, uint64_t *tallies,
                        uint64_t *result, void *stream) {
  if (bits < 2 || bits > 63) return fail(NTTMUL_EINVAL, "bits=%d outside [2, 63]", bits);
  CHECK(check_dev(tallies, 8, "tallies"));
  CHECK(check_dev(result, 8, "result"));
  if (cudaMemsetAsync(tallies, 0, 12 * 8, S(stream)) != cudaSuccess ||
      cudaMemsetAsync(result, 0, 8, S(stream)) != cudaSuccess ||
      cudaMemsetAsync(result + 1, 0xff, 8, S(stream)) != cudaSuccess)
    return cuda_status("sweep init");
  if (nsamples == 0) return NTTMUL_OK;
  sweep_random_kernel<<<grid_for(static_cast<long long>(nsamples), 256, 148LL * 16), 256, 0,
                        S(stream)>>>(bits, nsamples, seed,
                                     reinterpret_cast<unsigned long long *>(tallies),
                                     reinterpret_cast<unsigned long long *>(result));
  return cuda_status("sweep_random_kernel");
}

int nttmul_sweep_exhaustive(uint64_t q_lo, uint64_t q_hi, uint64_t *tallies, uint64_t *result,
                            void *stream) {
  if (q_hi >= (1u << 16)) return fail(NTTMUL_EINVAL, "q_hi=%llu must be < 2^16",
                                      static_cast<unsigned long long>(q_hi));
  CHECK(check_dev(tallies, 8, "tallies"));
  CHECK(check_dev(result, 8, "result"));
  if (cudaMemsetAsync(tallies, 0, 12 * 8, S(stream)) != cudaSuccess ||
      cudaMemsetAsync(result, 0, 8, S(stream)) != cudaSuccess ||
      cudaMemsetAsync(result + 1, 0xff, 8, S(stream)) != cudaSuccess)
    return cuda_status("sweep init");
  const u64 q0 = q_lo | 1;
  if (q0 < 3 && q_hi >= q0) return fail(NTTMUL_EINVAL, "q_lo must be >= 2");
  if (q_hi < q0) return NTTMUL_OK;
  const unsigned nq = static_cast<unsigned>((q_hi - q0) / 2 + 1);
  const u64 xmax = q_hi * q_hi;
  const unsigned gx = grid_for(static_cast<long long>(xmax), 256, 64);
  sweep_exhaustive_kernel<<<dim3(gx, nq), 256, 0, S(stream)>>>(
      q_lo, reinterpret_cast<unsigned long long *>(tallies),
      reinterpret_cast<unsigned long long *>(result));
  return cuda_status("sweep_exhaustive_kernel");
}

int nttmul_gather(uint64_t *out, const uint64_t *in, const int64_t *idx, int64_t n,
                  int64_t batch, void *stream) {
  if (n < 1 || batch < 0) return fail(NTTMUL_EINVAL, "n=%lld batch=%lld",
                                      static_cast<long long>(n), static_cast<long long>(batch));
  if (batch == 0) return NTTMUL_OK;
  CHECK(check_dev(out, 8, "out"));
  CHECK(check_dev(in, 8, "in"));
  CHECK(check_dev(idx, 8, "idx"));
  if (out == in) return fail(NTTMUL_EINVAL, "out may not alias in");
  const long long total = n * batch;
  gather_kernel<<<grid_for(total, 256), 256, 0, S(stream)>>>(
      out, in, reinterpret_cast<const long long *>(idx), n, total);
  return cuda_status("gather_kernel");
}

int nttmul_crt_decompose(uint64_t *res, const uint64_t *words, const uint64_t *primes,
                         const uint64_t *word_pairs, int num_limbs, int num_words,
                         int64_t batch, int64_t n, void *stream) {
  if (num_limbs < 1 || num_words < 1 || num_words > 64 || batch < 0 || n < 1)
    return fail(NTTMUL_EINVAL, "crt_decompose: L=%d W=%d", num_limbs, num_words);
  if (batch == 0) return NTTMUL_OK;
  CHECK(check_dev(res, 8, "res"));
  CHECK(check_dev(words, 8, "words"));
  CHECK(check_dev(primes, 8, "primes"));
  CHECK(check_dev(word_pairs, 16, "word_pairs"));
  const long long total = batch * n;
  const auto *pw = reinterpret_cast<const ulonglong2 *>(word_pairs);
  const unsigned grid = grid_for(total, CRT_THREADS);
  const size_t smem = (static_cast<size_t>(CRT_THREADS) * crt_stride(num_words) +
                       static_cast<size_t>(num_limbs) * num_words) * sizeof(u64) +
                      num_limbs * sizeof(CrtLimbConsts);
  if (smem > 200 * 1024) return fail(NTTMUL_EINVAL, "crt_decompose: L=%d W=%d too large",
                                     num_limbs, num_words);
  CHECK(smem_optin(crt_decompose_kernel, smem));
  CHECK(prefer_smem(crt_decompose_kernel));
  crt_decompose_kernel<<<grid, CRT_THREADS, smem, S(stream)>>>(res, words, primes, pw, num_limbs,
                                                               num_words, n, total);
  return cuda_status("crt_decompose_kernel");
}

int nttmul_crt_reconstruct(uint64_t *words, const uint64_t *res, const uint64_t *primes,
                           const uint64_t *inv_pairs, const uint64_t *m_words,
                           const uint64_t *q_words, const double *q_recip, int num_limbs,
                           int num_words, int64_t batch, int64_t n, void *stream) {
  if (num_limbs < 1 || num_limbs > 128 || num_words < 1 || num_words > 64 || batch < 0 || n < 1)
    return fail(NTTMUL_EINVAL, "crt_reconstruct: L=%d W=%d", num_limbs, num_words);
  if (batch == 0) return NTTMUL_OK;
  CHECK(check_dev(words, 8, "words"));
  CHECK(check_dev(res, 8, "res"));
  CHECK(check_dev(primes, 8, "primes"));
  CHECK(check_dev(inv_pairs, 16, "inv_pairs"));
  CHECK(check_dev(m_words, 8, "m_words"));
  CHECK(check_dev(q_words, 8, "q_words"));
  CHECK(check_dev(q_recip, 8, "q_recip"));
  const long long total = batch * n;
  const auto *iv = reinterpret_cast<const ulonglong2 *>(inv_pairs);
  const unsigned grid = grid_for(total, CRT_THREADS);
  const size_t smem =
      static_cast<size_t>(CRT_THREADS) * (crt_stride(num_words) + num_limbs) * sizeof(u64);
  CHECK(smem_optin(crt_reconstruct_kernel, smem));
  CHECK(prefer_smem(crt_reconstruct_kernel));
  crt_reconstruct_kernel<<<grid, CRT_THREADS, smem, S(stream)>>>(
      words, res, primes, iv, m_words, q_words, q_recip, num_limbs, num_words, n, total);
  return cuda_status("crt_reconstruct_kernel");
}

int nttmul_modmul_roof(const nttmul_limb_t *limb_host, int kind, int blocks, int threads,
                       int64_t iters, uint64_t *sink_out, double *modmuls_out,
                       void *stream) {
  if (!limb_host || blocks < 1 || threads < 32 || threads > 256 || iters < 1)
    return fail(NTTMUL_EINVAL, "bad microbenchmark geometry");
  CHECK(check_dev(sink_out, 8, "sink_out"));
  constexpr int CH = 8;
  const Limb L = *limb_host;
  const u64 w = (L.q >> 1) | 1, wp = shoup_host(w, L.q);
  if (kind == 1) {
    modmul_roof_kernel<1, 2, CH><<<blocks, threads, 0, S(stream)>>>(iters, sink_out, L, w, wp);
  } else if (kind == 2 || kind == 3) {
    if (L.q >= (1ULL << 61)) return fail(NTTMUL_EINVAL, "butterfly roof needs q < 2^61");
    if (kind == 2)
      modmul_roof_kernel<2, 2, CH><<<blocks, threads, 0, S(stream)>>>(iters, sink_out, L, w, wp);
    else
      modmul_roof_kernel<3, 2, CH><<<blocks, threads, 0, S(stream)>>>(iters, sink_out, L, w, wp);
    if (modmuls_out) *modmuls_out = static_cast<double>(blocks) * threads * iters * (CH / 2);
    return cuda_status("modmul_roof_kernel");
  } else {
    switch (L.mode) {
      case 0: modmul_roof_kernel<0, 0, CH><<<blocks, threads, 0, S(stream)>>>(iters, sink_out, L, w, wp); break;
      case 1: modmul_roof_kernel<0, 1, CH><<<blocks, threads, 0, S(stream)>>>(iters, sink_out, L, w, wp); break;
      default: modmul_roof_kernel<0, 2, CH><<<blocks, threads, 0, S(stream)>>>(iters, sink_out, L, w, wp); break;
    }
  }
  if (modmuls_out) *modmuls_out = static_cast<double>(blocks) * threads * iters * CH;
  return cuda_status("modmul_roof_kernel");
}

}  // extern "C"
