// grid_kernels.cuh - one-launch latency schedule of a standalone transform.
//
// A single forward / inverse transform of n = 2^13 .. 2^17 words is a few
// microseconds of chained launches: the latency schedule of capi.cu
// (strided column passes + 1024-word rows) takes three launches for 2^16,
// each paying a kernel boundary and an L2 round trip.  Here the transform
// is ONE launch of 2^A co-resident CTAs per polynomial, n = 2^A rows x 2^B
// words:
//   column phase  CTA c owns columns [c W, c W + W), W = 2^(B-A): all 2^A
//                 rows of them (W-word coalesced segments), and runs the A
//                 column stages (half-size k >= 2^B) in register passes
//                 through shared memory;
//   grid barrier  (slot_barrier below, or cooperative_groups' grid sync);
//   row phase     CTA c owns row c and runs the B row stages.
// The inverse runs the phases mirrored.  A single transform is a latency
// chain per warp (ncu r2: ~5.6 stall cycles per issued instruction, one or
// two warps per SM), so threads own only 2^LOG_E elements per pass: 2^16
// words run as 512 short warps of 4 elements instead of 256 long ones of 8.
// Butterflies, twiddles, lazy ranges and the final canonicalisation are the
// radix.cuh units of every other schedule, so outputs are bit-identical to
// them and to the reference's merged transforms (_kernels.pyx:52-129).
#pragma once
#include <cooperative_groups.h>

#include "ntt_kernels.cuh"

namespace nttb {

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem) : "memory");
}

struct GridParams {
  u64 *a;
  TwSet tw;
  LimbSet limbs;
  int fin;             // inverse: FinalMode of the global last stage
  unsigned *barrier;   // the grid barrier slot table (nullptr: cooperative launch)
};

// Grid barrier of a plain (non-cooperative) launch whose CTAs are all
// co-resident (the host checks the grid against the occupancy): one
// counter word per launch, the slot chosen by the launch itself from its
// %gridid - the context's temporal launch number, distinct for every launch
// including each replay of a captured graph - modulo GRID_SLOTS.  Two grid
// launches share a word only if one still runs 2^18 kernel launches after
// the other started.  The arrivals add up to exactly 2^31 (CTA 0 adds
// 2^31 - (n - 1), the others 1), so the barrier is complete when bit 31
// flips and the low bits return to their previous value (0): the word is
// valid for its next user without a reset - the flip-bit scheme of
// cooperative_groups' grid sync, minus the cooperative launch, which costs
// ~2 us more per call when replayed from a graph
// (scripts/microbench/launch_floor.cu).
constexpr int GRID_SLOTS = 1 << 18;
__device__ unsigned g_grid_barriers[GRID_SLOTS];

__device__ __forceinline__ unsigned *launch_slot(unsigned *slots) {
  unsigned long long id;
  asm volatile("mov.u64 %0, %%gridid;" : "=l"(id));
  return slots + (id & (GRID_SLOTS - 1));
}

__device__ __forceinline__ void slot_barrier(unsigned *bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned nb = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
    // release / acquire at gpu scope: cumulative over the CTA's writes,
    // which the CTA barriers order before / after thread 0's operations
    unsigned old, v;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;"
                 : "=r"(old) : "l"(bar), "r"(nb) : "memory");
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (((old ^ v) & 0x80000000u) == 0);
  }
  __syncthreads();
}

// 2^B-word rows, 2^A per polynomial, 2^LOG_E elements per thread and pass
// (passes of <= LOG_E stages).
template <int A, int B, int LOG_E>
struct GridGeom {
  static constexpr int T = 1 << (B - LOG_E);  // threads per CTA
  static constexpr int W = 1 << (B - A);      // columns per CTA in the column phase
  static constexpr int PADN = (1 << B) + (1 << B) / 16;
  __device__ __forceinline__ static int idx(int o) { return o + (o >> 4); }
  // K stages as passes of <= LOG_E stages (balanced)
  template <int K>
  struct Plan {
    static constexpr int NPASS = (K + LOG_E - 1) / LOG_E;
    __host__ __device__ static constexpr int R(int i) {
      return K / NPASS + (i < K % NPASS ? 1 : 0);
    }
    __host__ __device__ static constexpr int S0(int i) { return i == 0 ? 0 : S0(i - 1) + R(i - 1); }
  };
};

// Barrier between two passes (first stages S0a, S0b; Ra, Rb stages) of a
// 2^B-element grid transform.  A pass of R == LOG_E stages gives each
// thread one unit; when its groups span at most the 2^(5+LOG_E) elements of
// a warp (B - S0 <= 5 + LOG_E), warp w's units cover exactly elements
// [w 2^(5+LOG_E), (w+1) 2^(5+LOG_E)).  If both passes are like that, every
// warp reads only what it wrote itself: a warp barrier suffices.
template <int B, int LOG_E, int S0a, int Ra, int S0b, int Rb>
__device__ __forceinline__ void pass_sync() {
  constexpr bool WA = Ra == LOG_E && B - S0a <= 5 + LOG_E;
  constexpr bool WB = Rb == LOG_E && B - S0b <= 5 + LOG_E;
  if constexpr (WA && WB)
    __syncwarp();
  else
    __syncthreads();
}

// Shared-memory bytes of a grid kernel: the row (padded), its twiddles and
// the column twiddles.
template <int A, int B, int LOG_E>
constexpr size_t grid_smem_bytes() {
  return GridGeom<A, B, LOG_E>::PADN * sizeof(u64) +
         ((size_t(1) << B) + (size_t(1) << A)) * sizeof(ulonglong2);
}

// One pass of R stages starting at stage S0 of a 2^B-element transform
// spread over the CTA: units of 2^R elements spaced 2^LK apart (the
// radix.cuh unit), UNITS / T per thread.  Element o lives at GridGeom::idx(o)
// in shared memory or, for FROM_G / TO_G, at gaddr(o) in global memory
// (read from gin, written to gout).
// Forward passes stop after TS stages (truncated transforms); inverse
// passes run stages TS-1 .. 0, the last with inv_stage0 when STAGE0 (global
// stage 0, FinalMode fin).  CANON: canonicalise the forward output.
template <int LB, int A, int B, int LOG_E, int S0, int R, bool INV, bool FROM_G, bool TO_G, int TS,
          bool STAGE0, bool CANON, class GA>
__device__ __forceinline__ void grid_pass(u64 *__restrict__ sm, const u64 *gin, u64 *gout, GA gaddr,
                                          const ulonglong2 *__restrict__ tw, const Limb &L,
                                          const Mod &M, int fin) {
  using G = GridGeom<A, B, LOG_E>;
  constexpr int LK = B - S0 - R;
  constexpr int UNITS = 1 << (B - R);
  static_assert(UNITS % G::T == 0, "grid pass: every thread owns the same number of units");
#pragma unroll
  for (int w = 0; w < UNITS / G::T; ++w) {
    const int u = threadIdx.x + w * G::T;
    const int grp = u >> LK;
    const int o0 = (grp << (B - S0)) + (u & ((1 << LK) - 1));
    u64 x[1][1 << R];
#pragma unroll
    for (int e = 0; e < (1 << R); ++e) {
      const int o = o0 + (e << LK);
      x[0][e] = FROM_G ? gin[gaddr(o)] : sm[G::idx(o)];
    }
    const u64 B0 = (1ULL << S0) + static_cast<u64>(grp);
    if constexpr (!INV) {
      fwd_radix<LB, R, TS, 1>(x, B0, tw, M);  // starts with a reducing stage
      if constexpr (CANON) {
#pragma unroll
        for (int e = 0; e < (1 << R); ++e) x[0][e] = canon_fwd<LB>(x[0][e], M);
      }
    } else if constexpr (STAGE0) {
      inv_radix<LB, R, TS, 1, 1>(x, B0, tw, M);
      inv_stage0<LB, R, 1>(x, B0, tw, L, M, fin);
    } else {
      inv_radix<LB, R, TS, 0, 1>(x, B0, tw, M);
    }
#pragma unroll
    for (int e = 0; e < (1 << R); ++e) {
      const int o = o0 + (e << LK);
      if (TO_G)
        gout[gaddr(o)] = x[0][e];
      else
        sm[G::idx(o)] = x[0][e];
    }
  }
}

// Column phase: the A column stages of this CTA's W columns.  Element
// o = row * W + col stands for word (row << B) + c0 + col of the
// polynomial; in that numbering the column stages are exactly stages
// 0 .. A-1 of a 2^B-element transform (group of stage s = row >> (A - s),
// twiddle tw[2^s + group] of the global table), and consecutive units
// step over the columns first, so warps touch contiguous W-word segments.
template <int LB, int A, int B, int LOG_E, bool INV, int I, bool GIN = true>
__device__ __forceinline__ void grid_cols(u64 *sm, const u64 *gin, u64 *gout, int c0,
                                          const ulonglong2 *tw, const Limb &L, const Mod &M,
                                          int fin) {
  using P = typename GridGeom<A, B, LOG_E>::template Plan<A>;
  constexpr int NP = P::NPASS;
  if constexpr (I >= 0 && I < NP) {
    constexpr int S0 = P::S0(I), R = P::R(I);
    auto gaddr = [c0](int o) {
      return (static_cast<long long>(o >> (B - A)) << B) + c0 + (o & ((1 << (B - A)) - 1));
    };
    if constexpr (!INV) {
      grid_pass<LB, A, B, LOG_E, S0, R, false, GIN && I == 0, I == NP - 1, R, false, false>(
          sm, gin, gout, gaddr, tw, L, M, fin);
      if constexpr (I + 1 < NP) pass_sync<B, LOG_E, S0, R, P::S0(I + 1), P::R(I + 1)>();
      grid_cols<LB, A, B, LOG_E, false, I + 1, GIN>(sm, gin, gout, c0, tw, L, M, fin);
    } else {
      grid_pass<LB, A, B, LOG_E, S0, R, true, GIN && I == NP - 1, I == 0, R, I == 0, false>(
          sm, gin, gout, gaddr, tw, L, M, fin);
      if constexpr (I > 0) pass_sync<B, LOG_E, S0, R, P::S0(I - 1), P::R(I - 1)>();
      grid_cols<LB, A, B, LOG_E, true, I - 1, GIN>(sm, gin, gout, c0, tw, L, M, fin);
    }
  }
}

// Row phase: the B row stages of one row (twiddles staged at stw, base 1:
// row-local stage s, group g -> stw[2^s + g]).  Forward passes run upward
// from row-local stage 0 (the first reads global, the last canonicalises
// and writes global); inverse passes run downward (the first reads global,
// the last writes global, lazy).
template <int LB, int A, int B, int LOG_E, bool INV, int KIND, int I, bool GIN = true>
__device__ __forceinline__ void grid_row(u64 *sm, u64 *row, const ulonglong2 *stw, const Limb &L,
                                         const Mod &M) {
  using P = typename GridGeom<A, B, LOG_E>::template Plan<B>;
  constexpr int NP = P::NPASS;
  if constexpr (I >= 0 && I < NP) {
    constexpr int S0 = P::S0(I), R = P::R(I);
    constexpr bool TOP = S0 + R == B;  // the pass holding row-local stage B-1
    auto gaddr = [](int o) { return static_cast<long long>(o); };
    if constexpr (!INV) {
      constexpr int TS = (TOP && KIND == FWD_TRUNC) ? R - 1 : R;
      grid_pass<LB, A, B, LOG_E, S0, R, false, GIN && I == 0, I == NP - 1, TS, false,
                I == NP - 1>(sm, row, row, gaddr, stw, L, M, FIN_LAZY);
      if constexpr (I + 1 < NP) pass_sync<B, LOG_E, S0, R, P::S0(I + 1), P::R(I + 1)>();
      grid_row<LB, A, B, LOG_E, false, KIND, I + 1, GIN>(sm, row, stw, L, M);
    } else {
      constexpr int TS = (TOP && KIND == INV_SKIP) ? R - 1 : R;
      grid_pass<LB, A, B, LOG_E, S0, R, true, GIN && I == NP - 1, I == 0, TS, false, false>(
          sm, row, row, gaddr, stw, L, M, FIN_LAZY);
      if constexpr (I > 0) pass_sync<B, LOG_E, S0, R, P::S0(I - 1), P::R(I - 1)>();
      grid_row<LB, A, B, LOG_E, true, KIND, I - 1, GIN>(sm, row, stw, L, M);
    }
  }
}

// KIND: FwdKind (INV false) or InvKind (INV true)
template <int A, int B, int LOG_E, bool INV, int KIND, int LB>
__global__ void __launch_bounds__(GridGeom<A, B, LOG_E>::T) grid_kernel(const GridParams P) {
  using G = GridGeom<A, B, LOG_E>;
  static_assert(A >= 1 && B >= A, "grid geometry: at least one column per CTA");
  extern __shared__ u64 sm[];
  const long long poly = blockIdx.x >> A;
  const int r = static_cast<int>(blockIdx.x & ((1u << A) - 1));
  int limb;
  const Limb &L = *limb_ptr(P.limbs, poly, limb);
  const Mod M = mod_for<LB>(L.q);
  const ulonglong2 *tw = (INV ? P.tw.inv : P.tw.fwd) + limb * P.tw.stride;
  u64 *a = P.a + (poly << (A + B));
  const u64 rowbase = (1ULL << A) + r;
  u64 *row = a + (static_cast<long long>(r) << B);
  // Everything the first phase needs is staged into shared memory by one
  // batch of cp.async at kernel start - the column twiddles tw[1 .. 2^A)
  // at ctw[i], the row's twiddles tw[(rowbase << s) + g] (row-local stage
  // s) at stw[(1 << s) + g], and the first phase's data (forward: the CTA's
  // column block; inverse: its row) - so the first phase waits one memory
  // latency instead of one L2 round trip per pass, and every later pass
  // reads twiddles from shared memory (the row passes index stw with base 1).
  ulonglong2 *stw = reinterpret_cast<ulonglong2 *>(sm + G::PADN);
  ulonglong2 *ctw = stw + (1 << B);
  for (int i = threadIdx.x; i < (1 << B); i += G::T) {
    if (i == 0) continue;
    const int s = 31 - __clz(i);
    cp_async16(stw + i, tw + ((rowbase << s) + (i - (1 << s))));
  }
  for (int i = threadIdx.x + 1; i < (1 << A); i += G::T) cp_async16(ctw + i, tw + i);
  if constexpr (!INV) {
#pragma unroll
    for (int w = 0; w < (1 << B) / G::T; ++w) {  // column block: o = row * W + col
      const int o = threadIdx.x + w * G::T;
      cp_async8(sm + G::idx(o), a + (static_cast<long long>(o >> (B - A)) << B) + r * G::W +
                                    (o & (G::W - 1)));
    }
  } else {
#pragma unroll
    for (int w = 0; w < (1 << B) / G::T; ++w) {
      const int o = threadIdx.x + w * G::T;
      cp_async8(sm + G::idx(o), row + o);
    }
  }
  cp_async_commit();
  auto grid_sync = [&] {
    if (P.barrier)
      slot_barrier(launch_slot(P.barrier));
    else
      cooperative_groups::this_grid().sync();
  };
  constexpr int NPC = G::template Plan<A>::NPASS;
  constexpr int NPR = G::template Plan<B>::NPASS;
  cp_async_wait<0>();
  __syncthreads();
  if constexpr (!INV) {
    grid_cols<LB, A, B, LOG_E, false, 0, false>(sm, a, a, r * G::W, ctw, L, M, FIN_LAZY);
    grid_sync();
    grid_row<LB, A, B, LOG_E, false, KIND, 0>(sm, row, stw, L, M);
  } else {
    grid_row<LB, A, B, LOG_E, true, KIND, NPR - 1, false>(sm, row, stw, L, M);
    grid_sync();
    grid_cols<LB, A, B, LOG_E, true, NPC - 1>(sm, a, a, r * G::W, ctw, L, M, P.fin);
  }
}


// ---------------------------------------------------------------------------
// Fused product in one launch (polymul_fused of up to a few limb-products):
// column phase of a -> c and b -> ws (the A truncated-transform column
// stages), grid barrier, row phase (row stages 0 .. B-2 of a and b, the
// Karatsuba middle on consecutive pairs, inverse row stages B-2 .. 0),
// grid barrier, inverse column phase of c with the 2^-(log n - 1) scale.
// The stages, the middle (fused_pair / fused_pair_lazy per reduction MODE)
// and the lazy ranges are those of the row kernel's fused tail, so results
// are bit-identical to the three-launch schedule (reference
// polymul_fused / _kernels.pyx fused_middle, paper Alg. 8).

struct GridFusedParams {
  u64 *c;
  const u64 *a;
  const u64 *b;
  u64 *ws;
  TwSet tw;
  LimbSet limbs;
  unsigned *barrier;  // the grid barrier slot table
};

template <int A, int B>
constexpr size_t grid_fused_smem_bytes() {
  return 2 * GridGeom<A, B, 1>::PADN * sizeof(u64) +
         2 * ((size_t(1) << B) + (size_t(1) << A)) * sizeof(ulonglong2);
}

// forward row stages [I, N) of a and b (one stage per pass; the first
// reads the rows from global memory)
template <int LB, int A, int B, int I, int N>
__device__ __forceinline__ void grid_fused_fwd(u64 *sa, u64 *sb, const u64 *ga, const u64 *gb,
                                               const ulonglong2 *stw, const Limb &L,
                                               const Mod &M) {
  if constexpr (I < N) {
    auto gaddr = [](int o) { return static_cast<long long>(o); };
    grid_pass<LB, A, B, 1, I, 1, false, I == 0, false, 1, false, false>(sa, ga, nullptr, gaddr,
                                                                        stw, L, M, FIN_LAZY);
    grid_pass<LB, A, B, 1, I, 1, false, I == 0, false, 1, false, false>(sb, gb, nullptr, gaddr,
                                                                        stw, L, M, FIN_LAZY);
    pass_sync<B, 1, I, 1, I + 1, 1>();  // (after the last: the middle, stage B-1 pairs)
    grid_fused_fwd<LB, A, B, I + 1, N>(sa, sb, ga, gb, stw, L, M);
  }
}

// inverse row stages I .. 0 of c (the last writes the row to global, lazy)
template <int LB, int A, int B, int I>
__device__ __forceinline__ void grid_fused_inv(u64 *sc, u64 *gc, const ulonglong2 *stw,
                                               const Limb &L, const Mod &M) {
  if constexpr (I >= 0) {
    auto gaddr = [](int o) { return static_cast<long long>(o); };
    grid_pass<LB, A, B, 1, I, 1, true, false, I == 0, 1, false, false>(sc, nullptr, gc, gaddr,
                                                                      stw, L, M, FIN_LAZY);
    if constexpr (I > 0) pass_sync<B, 1, I, 1, I - 1, 1>();
    grid_fused_inv<LB, A, B, I - 1>(sc, gc, stw, L, M);
  }
}

// (register budget for 1024 resident threads per SM: 64 per thread, so
// up to 4 limb-products of 2^16 / 2 of 2^17 fit co-resident in one launch)
template <int A, int B>
constexpr int grid_fused_minb() {
  return GridGeom<A, B, 1>::T >= 1024 ? 1 : 1024 / GridGeom<A, B, 1>::T;
}

template <int A, int B, int MODE, int LB>
__global__ void __launch_bounds__(GridGeom<A, B, 1>::T, (grid_fused_minb<A, B>()))
    grid_fused_kernel(const GridFusedParams P) {
  using G = GridGeom<A, B, 1>;
  static_assert(A >= 1 && B >= A && B >= 2, "fused grid geometry");
  // lazy Barrett middle (proposed / dhem constants, all moduli < 2^60), as
  // in the row kernel's fused tail
  constexpr bool LAZY_MID = NTTB_LAZY_MID && MODE == NTTMUL_RED_ONE_SUB && LB >= 16;
  constexpr bool FAST = LAZY_MID && LB >= 32;
  extern __shared__ u64 sm[];
  u64 *sa = sm;
  u64 *sb = sm + G::PADN;
  ulonglong2 *stf = reinterpret_cast<ulonglong2 *>(sm + 2 * G::PADN);
  ulonglong2 *sti = stf + (1 << B);
  ulonglong2 *ctf = sti + (1 << B);  // column twiddles tw[1 .. 2^A)
  ulonglong2 *cti = ctf + (1 << A);
  const long long poly = blockIdx.x >> A;
  const int r = static_cast<int>(blockIdx.x & ((1u << A) - 1));
  int limb;
  const Limb &L = *limb_ptr(P.limbs, poly, limb);
  const Mod M = mod_for<LB>(L.q);
  const ulonglong2 *twf = P.tw.fwd + limb * P.tw.stride;
  const ulonglong2 *twi = P.tw.inv + limb * P.tw.stride;
  const long long off = poly << (A + B);
  const long long roff = off + (static_cast<long long>(r) << B);
  const u64 rowbase = (1ULL << A) + r;
  // one batch of cp.async (as in grid_kernel): the row's forward / inverse
  // twiddles, the column twiddles, and the CTA's column blocks of a and b
  for (int i = threadIdx.x; i < (1 << B); i += G::T) {
    if (i == 0) continue;
    const int s = 31 - __clz(i);
    const u64 j = (rowbase << s) + (i - (1 << s));
    cp_async16(stf + i, twf + j);
    cp_async16(sti + i, twi + j);
  }
  for (int i = threadIdx.x + 1; i < (1 << A); i += G::T) {
    cp_async16(ctf + i, twf + i);
    cp_async16(cti + i, twi + i);
  }
#pragma unroll
  for (int w = 0; w < (1 << B) / G::T; ++w) {  // column blocks: o = row * W + col
    const int o = threadIdx.x + w * G::T;
    const long long go = off + (static_cast<long long>(o >> (B - A)) << B) + r * G::W +
                         (o & (G::W - 1));
    cp_async8(sa + G::idx(o), P.a + go);
    cp_async8(sb + G::idx(o), P.b + go);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  // column phase: a -> c, b -> ws
  grid_cols<LB, A, B, 1, false, 0, false>(sa, P.a + off, P.c + off, r * G::W, ctf, L, M,
                                          FIN_LAZY);
  grid_cols<LB, A, B, 1, false, 0, false>(sb, P.b + off, P.ws + off, r * G::W, ctf, L, M,
                                          FIN_LAZY);
  slot_barrier(launch_slot(P.barrier));
  // row phase
  grid_fused_fwd<LB, A, B, 0, B - 1>(sa, sb, P.c + roff, P.ws + roff, stf, L, M);
  {
    const int q = threadIdx.x;  // pair (2q, 2q + 1); T = 2^(B-1) pairs
    const u64 a0 = sa[G::idx(2 * q)], a1 = sa[G::idx(2 * q + 1)];
    const u64 b0 = sb[G::idx(2 * q)], b1 = sb[G::idx(2 * q + 1)];
    // twiddle of the row-local stage B-2 group of the pair; sign of the z
    // term = parity of the global pair index = parity of q
    const ulonglong2 w = stf[(1 << (B - 2)) + (q >> 1)];
    u64 c0, c1;
    if constexpr (LAZY_MID)
      fused_pair_lazy<FAST>(to2q_any<LB>(a0, M), to2q_any<LB>(a1, M), to2q_any<LB>(b0, M),
                            to2q_any<LB>(b1, M), w.x, w.y, (q & 1) != 0, L, M, c0, c1);
    else
      fused_pair<MODE>(canon_fwd<LB>(a0, M), canon_fwd<LB>(a1, M), canon_fwd<LB>(b0, M),
                       canon_fwd<LB>(b1, M), w.x, w.y, (q & 1) != 0, L, M, c0, c1);
    sa[G::idx(2 * q)] = c0;
    sa[G::idx(2 * q + 1)] = c1;
  }
  pass_sync<B, 1, B - 1, 1, B - 2, 1>();  // middle -> first inverse pass
  grid_fused_inv<LB, A, B, B - 2>(sa, P.c + roff, sti, L, M);
  slot_barrier(launch_slot(P.barrier));
  grid_cols<LB, A, B, 1, true, G::template Plan<A>::NPASS - 1>(sa, P.c + off, P.c + off,
                                                                 r * G::W, cti, L, M,
                                                                 FIN_SCALED_SKIP);
}

}  // namespace nttb
