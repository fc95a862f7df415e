// cluster_kernels.cuh - one thread-block CLUSTER per limb-product: the whole
// n = N1 x 4096 transform stays on chip (distributed shared memory).
//
// The three-launch schedule (ntt_kernels.cuh: COL -> ROW -> COL^-1) sends
// every intermediate through HBM: a', b' written and re-read, c' written
// and re-read - 72n bytes per limb-product against the 24n algorithmic ones,
// and for small N1 (n = 2^13, 2^14: one or two column stages) the column
// launches cost more time than their share of the arithmetic.  Here the
// cluster's N1 CTAs (cluster rank r owns row r of a and b, 64 KB of shared
// memory, exactly the row kernel's layout) do, in ONE launch:
//   A. rank r loads column slab r (4096/N1 columns x N1 rows) of a and b from
//      HBM (coalesced row segments), runs the log2(N1) column stages in
//      registers, stages the results in shared memory grouped by destination
//      row, and the bulk-copy engine moves each row segment into the shared
//      memory of the CTA that owns the row (cp.async.bulk shared::cluster,
//      completion counted on the owner's mbarrier - no cluster barrier);
//   B. cluster barrier; every CTA runs the fused row pass of the row kernel
//      on its own row, entirely in shared memory (row stages of a and b,
//      Karatsuba middle, inverse row stages) - c' stays in shared memory;
//   C. cluster barrier; rank r gathers column slab r of c' from the N1 CTAs
//      (ld.shared::cluster), runs the inverse column stages with the folded
//      scale, and writes c to HBM.
// HBM sees 24n bytes per product (read a, b; write c); the element traffic
// between CTAs (16n bytes scattered, 8n gathered) runs over the SM-to-SM
// network.  This is the paper's on-chip "LOM" schedule
// with a cluster in place of one large block.  The same cluster transforms
// one polynomial for the standalone ntt_ct / intt_gs (phases A + B, or
// B + C).  The butterflies, twiddles and reduction schedule are those of the
// column and row kernels, so every output is bit-identical to them and to
// the reference (_kernels.pyx:52-177).
#pragma once
#include "ntt_kernels.cuh"

namespace nttb {

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `local` (a shared-memory pointer of this CTA)
// in the CTA of cluster rank `rank`
__device__ __forceinline__ unsigned dsmem_addr(const void *local, unsigned rank) {
  unsigned r;
  asm("mapa.shared::cluster.u32 %0, %1, %2;"
      : "=r"(r)
      : "r"(static_cast<unsigned>(__cvta_generic_to_shared(local))), "r"(rank));
  return r;
}
// Bulk copy of `bytes` (multiple of 16) from this CTA's shared memory to the
// shared::cluster address `dst`, completing `bytes` of transaction count on
// the (possibly remote) mbarrier at shared::cluster address `mbar`.  (Plain
// st.shared::cluster stores were measured against: any of them in the kernel
// makes ptxas spill ~270 B per thread in the row phase.)
__device__ __forceinline__ void bulk_to_cluster(unsigned dst, const void *src, unsigned bytes,
                                                unsigned mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, "
      "[%3];" ::"r"(dst),
      "r"(static_cast<unsigned>(__cvta_generic_to_shared(src))), "r"(bytes), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(u64 *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(bar))),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ u64 dsmem_ld(unsigned addr) {
  u64 v;
  asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
  return v;
}

enum ClusterKind {
  CL_FUSED = 0,  // c = a * b (truncated forwards, Karatsuba middle, scaled skip-first inverse)
  CL_FWD = 1,    // forward transform of in0 -> out (full or truncated)
  CL_INV = 2     // inverse transform of in0 -> out (full or skip-first; fin)
};

struct ClusterParams {
  u64 *out;
  const u64 *in0;
  const u64 *in1;
  TwSet tw;
  LimbSet limbs;
  int fwd;  // FwdKind (CL_FWD)
  int inv;  // InvKind (CL_INV)
  int fin;  // FinalMode of the global last inverse stage (CL_FUSED, CL_INV)
};

template <int LOG_N1>
struct ClusterGeom {
  static constexpr int N1 = 1 << LOG_N1;     // rows = CTAs per cluster
  static constexpr int N2 = 1 << COL_LOG_R;  // row length
  static constexpr int SW = N2 / N1;         // columns per slab (per CTA)
  using G = RowGeom<COL_LOG_R>;
  static constexpr int T = G::T;             // 512 threads
  static_assert(LOG_N1 >= 1 && LOG_N1 <= 4, "cluster of 2..16 CTAs");
};

// Phase A: column stages of slab r of the NP polynomials; the results are
// staged by destination row (segment e = row e's columns [r SW, (r+1) SW),
// in the row buffer's swizzled order - the swizzle permutes words inside
// 16-word groups, so a segment maps onto itself) and bulk-copied into buffer
// p of the row owners.  Every load of a thread (16 words: NP * SW / T
// columns of N1 rows) is issued before the first butterfly.  `stage` holds
// the slab of one polynomial (N2 words), refilled once the copies of the
// previous one have read it.
template <int LOG_N1, int NP, int LB>
__device__ __forceinline__ void cluster_columns_fwd(u64 *sm, u64 *stage, const ulonglong2 *stw,
                                                    const u64 *g0, const u64 *g1, unsigned r,
                                                    u64 *mbar, const Mod &M) {
  using C = ClusterGeom<LOG_N1>;
  using G = typename C::G;
  constexpr int TPP = C::SW >= C::T ? C::SW / C::T : 1;  // columns per thread per polynomial
  const int c0 = static_cast<int>(r) * C::SW;
  const bool active = C::SW >= C::T || threadIdx.x < C::SW;
  // all NP polynomials' loads up front when they fit 16 words per thread
  // (n <= 2^15), else polynomial by polynomial
  constexpr bool ALL = NP * TPP * C::N1 <= 16;
  u64 x[NP][TPP][1][C::N1];
  auto load = [&](int p) {
    if (active) {
#pragma unroll
      for (int k = 0; k < TPP; ++k)
#pragma unroll
        for (int e = 0; e < C::N1; ++e)
          x[p][k][0][e] = (p == 0 ? g0 : g1)[c0 + threadIdx.x + k * C::T + e * C::N2];
    }
  };
  if (ALL) {
#pragma unroll
    for (int p = 0; p < NP; ++p) load(p);
  }
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    if (!ALL) load(p);
    if (p > 0) __syncthreads();  // the previous polynomial's copies have read `stage`
    if (active) {
#pragma unroll
      for (int k = 0; k < TPP; ++k) {
        const int col = c0 + threadIdx.x + k * C::T;
        col_fwd_stages<LB, LOG_N1>(x[p][k], stw, M);
        const int so = G::idx(col) - c0;  // position inside the segment
#pragma unroll
        for (int e = 0; e < C::N1; ++e) stage[e * C::SW + so] = x[p][k][0][e];
      }
    }
    fence_proxy_async();  // the generic-proxy writes above -> the bulk copies
    if (p == 0) cluster_wait();  // every owner's arrival barrier is initialised
    __syncthreads();
    if (threadIdx.x < C::N1) {
      const unsigned e = threadIdx.x;
      bulk_to_cluster(dsmem_addr(sm + p * G::PADN + c0, e), stage + e * C::SW,
                      C::SW * sizeof(u64), dsmem_addr(mbar, e));
      bulk_commit();
      bulk_wait_read();  // the staging buffer may be refilled
    }
  }
}

// Phase C: inverse column stages of slab r of the rows' buffer 0 -> HBM
// (all of a thread's shared::cluster loads issued first).
template <int LOG_N1, int LB>
__device__ __forceinline__ void cluster_columns_inv(const u64 *sm, const ulonglong2 *stw,
                                                    u64 *gout, unsigned r, const Limb &L,
                                                    const Mod &M, int fin) {
  using C = ClusterGeom<LOG_N1>;
  using G = typename C::G;
  constexpr int TPP = C::SW >= C::T ? C::SW / C::T : 1;
  if (C::SW < C::T && threadIdx.x >= C::SW) return;  // (n = 2^16: half the threads)
  const int c0 = static_cast<int>(r) * C::SW;
  u64 x[TPP][1][C::N1];
#pragma unroll
  for (int k = 0; k < TPP; ++k) {
    const u64 *src = sm + G::idx(c0 + threadIdx.x + k * C::T);
#pragma unroll
    for (int e = 0; e < C::N1; ++e) x[k][0][e] = dsmem_ld(dsmem_addr(src, e));
  }
#pragma unroll
  for (int k = 0; k < TPP; ++k) {
    const int col = c0 + threadIdx.x + k * C::T;
    col_inv_stages<LB, LOG_N1>(x[k], stw, L, M, fin);
#pragma unroll
    for (int e = 0; e < C::N1; ++e) gout[col + e * C::N2] = x[k][0][e];
  }
}

template <int LOG_N1, int KIND, int MODE, int LB>
__global__ void __launch_bounds__(RowGeom<COL_LOG_R>::T, NTTB_ROW_MINB_FUSED)
    cluster_kernel(const ClusterParams P) {
  using C = ClusterGeom<LOG_N1>;
  using G = typename C::G;
  constexpr int LOG_R = COL_LOG_R;
  extern __shared__ u64 sm[];  // [row of a | row of b (CL_FUSED)] [staging: N2 words]
  __shared__ ulonglong2 stw[2][C::N1];  // column-stage twiddles tw[1 .. N1): fwd, inv
  __shared__ u64 mbar;                  // the rows' arrival (phase A)
  const unsigned r = cluster_rank();
  const long long poly = blockIdx.x >> LOG_N1;
  int limb;
  const Limb &L = *limb_ptr(P.limbs, poly, limb);
  const Mod M = mod_for<LB>(L.q);
  const ulonglong2 *twf = P.tw.fwd + limb * P.tw.stride;
  const ulonglong2 *twi = P.tw.inv + limb * P.tw.stride;
  const u64 rowbase = C::N1 + r;
  const long long pbase = poly << (LOG_N1 + LOG_R);  // first word of the polynomial
  const long long off = pbase + (static_cast<long long>(r) << LOG_R);  // this CTA's row

  constexpr int NP = KIND == CL_FUSED ? 2 : 1;
  // every CTA initialises its arrival barrier (expecting its NP rows) and
  // announces that it runs: the others send it rows only after waiting on
  // this cluster phase
  if (KIND != CL_INV && threadIdx.x == 0) {
    sbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_arrive_expect(&mbar, NP * C::N2 * sizeof(u64));
  }
  cluster_arrive_relaxed();
  if (threadIdx.x < 2 * C::N1) {
    const int w = threadIdx.x >= C::N1;
    stw[w][threadIdx.x - w * C::N1] = (w ? twi : twf)[threadIdx.x - w * C::N1];
  }
  __syncthreads();

  if constexpr (KIND == CL_FUSED || KIND == CL_FWD) {
    // ---- A: column stages, bulk-copied to the row owners ----
    u64 *stage = sm + NP * G::PADN;
    cluster_columns_fwd<LOG_N1, NP, LB>(sm, stage, stw[0], P.in0 + pbase,
                                        NP > 1 ? P.in1 + pbase : nullptr, r, &mbar, M);
    sbar_wait(&mbar, 0);  // this CTA's rows have arrived
    // ---- B: the row stages in shared memory ----
    if constexpr (KIND == CL_FUSED) {
      head_fwd_all<LB, LOG_R, 2, 0, false>(sm, nullptr, nullptr, rowbase, twf, M);
      tail_pass<LB, LOG_R, 2, FWD_TRUNC, true, INV_SKIP, MODE>(sm, rowbase, twf, twi, L, M);
      row_sync<LOG_R, G::S0(G::NPASS - 1)>();
      head_inv_all<LB, LOG_R, G::NPASS - 1, false>(sm, nullptr, rowbase, twi, L, M, FIN_LAZY);
    } else {
      head_fwd_all<LB, LOG_R, 1, 0, false>(sm, nullptr, nullptr, rowbase, twf, M);
      if (P.fwd == FWD_TRUNC)
        tail_pass<LB, LOG_R, 1, FWD_TRUNC, false, INV_NONE, MODE>(sm, rowbase, twf, twi, L, M);
      else
        tail_pass<LB, LOG_R, 1, FWD_FULL, false, INV_NONE, MODE>(sm, rowbase, twf, twi, L, M);
      __syncthreads();
#pragma unroll 4
      for (int i = threadIdx.x; i < G::N2; i += G::T) P.out[off + i] = sm[G::idx(i)];
      return;  // no other CTA reads this one's shared memory any more
    }
  } else {
    // ---- B (inverse): the row's inverse stages, from HBM into shared memory ----
#pragma unroll 4
    for (int i = threadIdx.x; i < G::N2; i += G::T) sm[G::idx(i)] = P.in0[off + i];
    __syncthreads();
    if (P.inv == INV_SKIP)
      tail_pass<LB, LOG_R, 1, FWD_NONE, false, INV_SKIP, MODE>(sm, rowbase, twf, twi, L, M);
    else
      tail_pass<LB, LOG_R, 1, FWD_NONE, false, INV_FULL, MODE>(sm, rowbase, twf, twi, L, M);
    row_sync<LOG_R, G::S0(G::NPASS - 1)>();
    head_inv_all<LB, LOG_R, G::NPASS - 1, false>(sm, nullptr, rowbase, twi, L, M, FIN_LAZY);
    cluster_wait();  // the start-up phase
  }
  // ---- C: inverse column stages, gathered from the row owners -> HBM ----
  cluster_arrive();
  cluster_wait();
  cluster_columns_inv<LOG_N1, LB>(sm, stw[1], P.out + pbase, r, L, M, P.fin);
  __syncwarp();
  // no CTA may exit while another still reads its shared memory
  cluster_arrive();
  cluster_wait();
}

}  // namespace nttb
