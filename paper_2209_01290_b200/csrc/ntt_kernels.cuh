// ntt_kernels.cuh - the sm_100a kernels of the polymul hot path.
//
// Data layout in HBM: polynomials are uint64[n], back to back ([batch, n] or
// [batch, limbs, n]); twiddles are {w, w'} pairs, one [n] table per prime.
//
// Large transforms (n = 2^13 .. 2^17) use a stage-grouped 2D split
// n = N1 x N2 with N2 = 4096 (one "row"): the merged-CT stages with half-size
// k >= N2 act independently on each column j mod N2 and need only the N1-1
// twiddles tw[1..N1), so the COLUMN kernel gives each thread one column in
// registers (coalesced across threads); the remaining stages stay inside a
// contiguous row, which the ROW kernel keeps in shared memory and registers
// (two 4-stage register passes + one 16-consecutive-element tail).  The
// inverse is the mirror (row kernel first, then column kernel).  The fused
// polymul is COL(a,b) -> ROW(fwd a,b + Karatsuba middle + inverse) -> COL^-1.
// Output order and values are exactly the reference's merged transforms
// (reference _kernels.pyx:52-129): only the schedule of the same butterflies
// changes.  Transforms with n <= 2^12 need no column kernel; n < 2^10 uses the
// simple one-CTA-per-polynomial kernel.
#pragma once
#include <cuda_runtime.h>

#include "radix.cuh"

namespace nttb {

struct TwSet {
  const ulonglong2 *fwd;  // table of limb 0
  const ulonglong2 *inv;
  long long stride;       // entries between consecutive limbs (0: one prime)
};

struct LimbSet {
  const Limb *table;  // device [num] or nullptr -> use `single`
  Limb single;
  int num;
  int base;           // polynomial index offset of this launch (chunking)
};

// pointer form: fields are read where used instead of living in registers
// for the whole kernel (the table entry stays in L1; the single-prime
// struct lives in kernel-parameter space)
__device__ __forceinline__ const Limb *limb_ptr(const LimbSet &S, long long poly, int &limb) {
  if (S.table) {
    // 32-bit remainder (a 64-bit one is a long emulated sequence); poly
    // indices of one launch stay far below 2^32 (each is >= 4 KiB of HBM)
    limb = static_cast<int>((static_cast<unsigned>(poly) + static_cast<unsigned>(S.base)) %
                            static_cast<unsigned>(S.num));
    return S.table + limb;
  }
  limb = 0;
  return &S.single;
}

__device__ __forceinline__ Limb get_limb(const LimbSet &S, long long poly,
                                         int &limb) {
  if (S.table) {
    limb = static_cast<int>((poly + S.base) % S.num);
    return S.table[limb];
  }
  limb = 0;
  return S.single;
}

// L2 eviction-priority hints for the global streams of the pipeline:
// inputs read for the last time are loaded evict-first, intermediates that
// the next launch reads again (a', b' -> row kernel, c' -> inverse columns)
// are stored evict-last, the final product evict-first.  NTTB_L2_HINTS=0
// turns them into plain accesses.
#ifndef NTTB_L2_HINTS
#define NTTB_L2_HINTS 0  // measured +-0 % on the step, inverse columns slower (sweep_r33)
#endif
enum L2Hint { L2_NORMAL = 0, L2_FIRST = 1, L2_LAST = 2 };

template <int H>
__device__ __forceinline__ u64 l2_policy() {
  u64 pol = 0;
  if (H == L2_FIRST)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else if (H == L2_LAST)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

template <int H>
__device__ __forceinline__ u64 ldg_hint(const u64 *p) {
  if (!NTTB_L2_HINTS || H == L2_NORMAL) return *p;
  u64 v;
  asm volatile("ld.global.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(l2_policy<H>()));
  return v;
}

template <int H>
__device__ __forceinline__ void stg_hint(u64 *p, u64 v) {
  if (!NTTB_L2_HINTS || H == L2_NORMAL) {
    *p = v;
    return;
  }
  asm volatile("st.global.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(l2_policy<H>())
               : "memory");
}

// Drop a consumed scratch line from L2 without writing it back to HBM
// (sm_80+ discard.global.L2): intermediates of the fused pipeline live and
// die in L2.  `line` must be 128-byte aligned and fully consumed.
__device__ __forceinline__ void discard_line(const void *line) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(line) : "memory");
}

#ifdef NTTB_PHASE_TIMING
// debug builds only: per-CTA clock64 stamps at row-kernel phase boundaries
__device__ unsigned long long g_phase[1 << 16][8];
#define NTTB_STAMP(i)                                                            \
  do {                                                                           \
    if (threadIdx.x == 0 && blockIdx.x < (1u << 16)) g_phase[blockIdx.x][i] = clock64(); \
  } while (0)
#else
#define NTTB_STAMP(i) \
  do {                \
  } while (0)
#endif


// resident CTAs per SM the row kernels are compiled for (register budget)
#ifndef NTTB_ROW_MINB_FUSED
#define NTTB_ROW_MINB_FUSED 2
#endif
#ifndef NTTB_ROW_MINB
#define NTTB_ROW_MINB 2
#endif

enum FwdKind { FWD_NONE = 0, FWD_FULL = 1, FWD_TRUNC = 2 };
enum InvKind { INV_NONE = 0, INV_FULL = 1, INV_SKIP = 2 };

// ---------------------------------------------------------------------------
// ROW kernel
//
// One CTA owns one contiguous row of N2 = 2^LOG_R coefficients (of a and b
// when fused).  Each thread owns E = 2^LOG_E elements per pass.  The row's
// HEAD = LOG_R - LOG_E leading stages run as register passes of <= LOG_E
// stages over strided units (shared memory between passes); the last LOG_E
// stages (the "tail") run on E consecutive elements, with the Karatsuba
// middle in between when fused.  Inverse = mirror.

#ifndef NTTB_ROW_LOG_E
#define NTTB_ROW_LOG_E 3
#endif
#ifndef NTTB_PREFETCH_B
#define NTTB_PREFETCH_B 1
#endif
#ifndef NTTB_LAZY_MID
#define NTTB_LAZY_MID 1
#endif
#ifndef NTTB_FAST_RED
#define NTTB_FAST_RED 1
#endif
// issue a unit's twiddle loads before its data loads (hides their L2
// latency; measured -2.7 % row-kernel time, sweep_r18)
#ifndef NTTB_B_OWN_COPIES
#define NTTB_B_OWN_COPIES 1
#endif
#ifndef NTTB_FWD_P_UNROLL
#define NTTB_FWD_P_UNROLL 0
#endif
#ifndef NTTB_TW_PREFETCH
#define NTTB_TW_PREFETCH 1
#endif

template <int LOG_R, int LOG_E = NTTB_ROW_LOG_E>
struct RowGeom {
  static constexpr int N2 = 1 << LOG_R;
  static constexpr int E = 1 << LOG_E;
  static constexpr int T = N2 / E;                 // threads per CTA
  // shared-memory layout of a row: 4096-element rows with 8-element units use
  // an XOR swizzle (conflict-free for every pass, no padding); other shapes
  // pad one word per 16
  static constexpr bool SWZ = (LOG_R == 12 && LOG_E == 3);
  static constexpr int PADN = SWZ ? N2 : N2 + N2 / 16;
  __device__ __forceinline__ static int idx(int o) {
    if (SWZ) {
      const int row = o >> 4;
      return o ^ ((row & 7) | ((row & 4) << 1));
    }
    return o + (o >> 4);
  }
  static constexpr int HEAD = LOG_R - LOG_E;       // stages before the tail
  static constexpr int NPASS = (HEAD + LOG_E - 1) / LOG_E;
  // stages of head pass i (balanced) and its first stage
  __host__ __device__ static constexpr int R(int i) { return HEAD / NPASS + (i < HEAD % NPASS ? 1 : 0); }
  __host__ __device__ static constexpr int S0(int i) { return i == 0 ? 0 : S0(i - 1) + R(i - 1); }
  static_assert(NPASS >= 1 && NPASS <= 4, "row geometry");
};

// Swizzled index of element o0 + (e << LK) of a pass unit (o0 = the unit's
// first element), with the XOR swizzle hoisted out of the element loop: for
// strides of >= 8 rows (LK >= 7) the mask is the same for every element, so
// the addresses are idx(o0) + immediate; for the 4-row stride of the middle
// pass (LK = 6, unit start in rows 0-3 of an 8-row group) the mask flips by
// f(4) = 12 on odd elements.  Other shapes use RowGeom::idx directly.
#ifndef NTTB_SWZ_HOIST
#define NTTB_SWZ_HOIST 2  // 1: the 8- and 4-row strides only; 2: also the 2-word stride and the tail
#endif
// For the 2-word stride of the last head pass (LK = 3, unit start in
// words 0-7 of a 64-word block) element e sits in row 4g + e/2 at column
// bit 3 = e & 1, so idx = (idx(o0) ^ (8 (e & 1) ^ e / 2)) + 16 (e / 2).
// LK = 0 (the tail's 8 consecutive words, o0 = 8 t): idx = idx(o0) ^ e.
template <int LOG_R, int LK>
struct UnitIdx {
  using G = RowGeom<LOG_R>;
  static constexpr bool HOIST =
      NTTB_SWZ_HOIST && G::SWZ && (LK >= 6 || (NTTB_SWZ_HOIST > 1 && (LK == 3 || LK == 0)));
  int b0, b1;
  __device__ __forceinline__ explicit UnitIdx(int o0) {
    if constexpr (HOIST) {
      b0 = G::idx(o0);
      b1 = LK == 6 ? (b0 ^ 12) : b0;
    } else {
      b0 = o0;
      b1 = o0;
    }
  }
  __device__ __forceinline__ int operator()(int e) const {
    if constexpr (HOIST && LK >= 6) return ((e & 1) ? b1 : b0) + (e << LK);
    if constexpr (HOIST && LK == 3) return (b0 ^ ((8 * (e & 1)) ^ (e >> 1))) + 16 * (e >> 1);
    if constexpr (HOIST && LK == 0) return b0 ^ e;
    return G::idx(b0 + (e << LK));
  }
};

struct RowParams {
  u64 *out;
  const u64 *in0;
  const u64 *in1;
  TwSet tw;
  LimbSet limbs;
  int log_n1;  // rows per polynomial = 2^log_n1
  int fin;     // FinalMode of the global last inverse stage (if in this kernel)
  int discard_in;  // inputs are pipeline scratch: discard their L2 lines once read
  long long nrows;    // rows in this launch
  long long pf_dist;  // > 0: prefetch the input rows of row + pf_dist into L2
};

// bulk prefetch of [p, p + bytes) into L2 (no register or smem cost)
__device__ __forceinline__ void prefetch_l2(const void *p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// forward head pass: R stages starting at row-local stage S0.  The NP
// polynomials are processed one after the other (the second pass over the
// same twiddles hits L1), so only E data words per thread are live.
template <int LB, int LOG_R, int S0, int R, int NP, bool FROM_GLOBAL>
__device__ __forceinline__ void head_fwd(u64 *__restrict__ sm,
                                         const u64 *__restrict__ g0,
                                         const u64 *__restrict__ g1,
                                         u64 rowbase,
                                         const ulonglong2 *__restrict__ tw,
                                         const Mod &M) {
  using G = RowGeom<LOG_R>;
  constexpr int U = G::E >> R;         // units per thread
  constexpr int LK = LOG_R - S0 - R;   // log2(k_last)
#if NTTB_FWD_P_UNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
  for (int p = 0; p < NP; ++p) {  // not unrolled: one polynomial's state live
    const u64 *__restrict__ g = p == 0 ? g0 : g1;
    u64 *__restrict__ s = sm + p * G::PADN;
#pragma unroll
    for (int w = 0; w < U; ++w) {
      const int u = threadIdx.x + w * G::T;
      const int grp = u >> LK;
      const int o0 = (grp << (LOG_R - S0)) + (u & ((1 << LK) - 1));
#if NTTB_TW_PREFETCH
      TwBuf<0, R> twb;
      tw_prefetch(twb, tw, (rowbase << S0) + grp);
#endif
      const UnitIdx<LOG_R, LK> ix(o0);
      u64 x[1][1 << R];
#pragma unroll
      for (int e = 0; e < (1 << R); ++e) {
        const int o = o0 + (e << LK);
        x[0][e] = FROM_GLOBAL ? ldg_hint<L2_FIRST>(g + o) : s[ix(e)];
      }
#if NTTB_TW_PREFETCH
      fwd_radix_pf<LB, R, R, 1, S0 & 1>(x, twb, M);
#else
      fwd_radix<LB, R, R, 1, S0 & 1>(x, (rowbase << S0) + grp, tw, M);
#endif
#pragma unroll
      for (int e = 0; e < (1 << R); ++e) s[ix(e)] = x[0][e];
    }
  }
}

// inverse head pass (mirror of head_fwd); TO_GLOBAL only for S0 == 0
template <int LB, int LOG_R, int S0, int R, bool TO_GLOBAL>
__device__ __forceinline__ void head_inv(u64 *__restrict__ sm,
                                         u64 *__restrict__ gout, u64 rowbase,
                                         const ulonglong2 *__restrict__ tw,
                                         const Limb &L, const Mod &M, int fin) {
  using G = RowGeom<LOG_R>;
  constexpr int U = G::E >> R;
  constexpr int LK = LOG_R - S0 - R;
#pragma unroll
  for (int w = 0; w < U; ++w) {
    const int u = threadIdx.x + w * G::T;
    const int g = u >> LK;
    const int o0 = (g << (LOG_R - S0)) + (u & ((1 << LK) - 1));
    const u64 B0 = (rowbase << S0) + g;
#if NTTB_TW_PREFETCH
    TwBuf<0, R> twb;
    tw_prefetch(twb, tw, B0);
#endif
    u64 x[1][1 << R];
    const UnitIdx<LOG_R, LK> ix(o0);
#pragma unroll
    for (int e = 0; e < (1 << R); ++e) x[0][e] = sm[ix(e)];
    if (TO_GLOBAL) {
#if NTTB_TW_PREFETCH
      inv_radix_pf<LB, R, R, 1, 1>(x, twb, M);
#else
      inv_radix<LB, R, R, 1, 1>(x, B0, tw, M);
#endif
      inv_stage0<LB, R, 1>(x, B0, tw, L, M, fin);
#pragma unroll
      for (int e = 0; e < (1 << R); ++e) stg_hint<L2_LAST>(gout + o0 + (e << LK), x[0][e]);
    } else {
#if NTTB_TW_PREFETCH
      inv_radix_pf<LB, R, R, 0, 1>(x, twb, M);
#else
      inv_radix<LB, R, R, 0, 1>(x, B0, tw, M);
#endif
#pragma unroll
      for (int e = 0; e < (1 << R); ++e) sm[ix(e)] = x[0][e];
    }
  }
}

// Pull the twiddle pairs the thread's unit of head pass I will read into L1
// before the barrier that precedes the pass (no registers: prefetch.L1), so
// the loads issued after the barrier hit L1 instead of waiting on L2.  Stage
// t of the unit reads the 2^t consecutive pairs starting at (B0 << t).
#ifndef NTTB_TW_L1PF
#define NTTB_TW_L1PF 0  // measured +-0 (row 0.5289 ms both ways, r50): twiddle latency is not the limiter
#endif
__device__ __forceinline__ void prefetch_l1(const void *p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
template <int R>
__device__ __forceinline__ void tw_prefetch_l1(const ulonglong2 *tw, u64 B0) {
#pragma unroll
  for (int t = 0; t < R; ++t) {
    prefetch_l1(tw + (B0 << t));
    if (t >= 3) prefetch_l1(tw + (B0 << t) + (1 << t) - 1);  // > 128 B range
  }
}
template <int LOG_R, int I>
__device__ __forceinline__ void pass_tw_l1(const ulonglong2 *tw, u64 rowbase) {
  using G = RowGeom<LOG_R>;
  if constexpr (NTTB_TW_L1PF && I < G::NPASS && (G::E >> G::R(I)) == 1) {
    constexpr int LK = LOG_R - G::S0(I) - G::R(I);
    const u64 B0 = (rowbase << G::S0(I)) + (threadIdx.x >> LK);
    tw_prefetch_l1<G::R(I)>(tw, B0);
  }
}

// Barrier between two row passes.  A pass with first stage S0 transforms
// independent blocks of 2^(LOG_R - S0) elements; when every pass gives each
// thread one unit (R == LOG_E), the threads that own a block are the
// 2^(LOG_R - S0 - LOG_E) consecutive threads tid / that-many, in the passes
// on both sides of the barrier (pass blocks nest, and the tail's 8-element
// units sit inside the last pass's blocks).  So only those threads need to
// meet: a warp-level sync for blocks of <= 32 threads, a named barrier for
// blocks of 64..T/2 threads, the CTA barrier only for whole-row blocks.
#ifndef NTTB_LOCAL_SYNC
#define NTTB_LOCAL_SYNC 1
#endif
template <int LOG_R, int S0_BLOCK>
__device__ __forceinline__ void row_sync() {
  using G = RowGeom<LOG_R>;
  constexpr bool ONE_UNIT = G::HEAD % G::NPASS == 0 && G::HEAD / G::NPASS == NTTB_ROW_LOG_E;
  constexpr int THREADS = 1 << (LOG_R - S0_BLOCK - NTTB_ROW_LOG_E);
  if constexpr (!NTTB_LOCAL_SYNC || !ONE_UNIT || THREADS >= G::T) {
    __syncthreads();
  } else if constexpr (THREADS <= 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + static_cast<int>(threadIdx.x) / THREADS),
                 "n"(THREADS)
                 : "memory");
  }
}

// all forward head passes, pass i = 0 .. NPASS-1 (pass 0 reads global)
template <int LB, int LOG_R, int NP, int I = 0>
__device__ __forceinline__ void head_fwd_all(u64 *sm, const u64 *g0, const u64 *g1,
                                             u64 rowbase, const ulonglong2 *tw,
                                             const Mod &M) {
  using G = RowGeom<LOG_R>;
  if constexpr (I < G::NPASS) {
    head_fwd<LB, LOG_R, G::S0(I), G::R(I), NP, I == 0>(sm, g0, g1, rowbase, tw, M);
    pass_tw_l1<LOG_R, I + 1>(tw, rowbase);
    if constexpr (NTTB_TW_L1PF && I + 1 == G::NPASS && G::HEAD > 0) {
      // the tail's forward stage twiddles (its inverse ones come from the
      // other table, prefetched by the caller's tail)
      tw_prefetch_l1<(LOG_R - G::HEAD) - 1>(tw, (rowbase << G::HEAD) + threadIdx.x);
    }
    row_sync<LOG_R, G::S0(I)>();
    if (I == 0) NTTB_STAMP(1);
    head_fwd_all<LB, LOG_R, NP, I + 1>(sm, g0, g1, rowbase, tw, M);
  }
}

// all inverse head passes, pass i = NPASS-1 .. 0 (pass 0 writes global)
template <int LB, int LOG_R, int I>
__device__ __forceinline__ void head_inv_all(u64 *sm, u64 *gout, u64 rowbase,
                                             const ulonglong2 *tw, const Limb &L,
                                             const Mod &M, int fin) {
  using G = RowGeom<LOG_R>;
  if constexpr (I > 0) {
    head_inv<LB, LOG_R, G::S0(I), G::R(I), false>(sm, nullptr, rowbase, tw, L, M,
                                                  FIN_LAZY);
    pass_tw_l1<LOG_R, I - 1>(tw, rowbase);
    row_sync<LOG_R, G::S0(I - 1)>();
    head_inv_all<LB, LOG_R, I - 1>(sm, gout, rowbase, tw, L, M, fin);
  } else {
    head_inv<LB, LOG_R, 0, G::R(0), true>(sm, gout, rowbase, tw, L, M, fin);
  }
}

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
#if NTTB_L2_HINTS
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem),
               "l"(l2_policy<L2_FIRST>())
               : "memory");
#else
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
#endif
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// issue the async copy of one row (N2 words) into padded smem
template <int LOG_R>
__device__ __forceinline__ void row_prefetch(u64 *__restrict__ dst, const u64 *__restrict__ src) {
  using G = RowGeom<LOG_R>;
  if constexpr (G::SWZ && NTTB_SWZ_HOIST) {  // stride T = 512 words = 32 rows: same mask
    const int b = G::idx(threadIdx.x);
#pragma unroll
    for (int k = 0; k < G::N2 / G::T; ++k)
      cp_async8(dst + b + k * G::T, src + threadIdx.x + k * G::T);
  } else {
#pragma unroll
    for (int i = threadIdx.x; i < G::N2; i += G::T) cp_async8(dst + G::idx(i), src + i);
  }
}

// all forward head passes of ONE polynomial already in smem `s`
template <int LB, int LOG_R, int I = 0>
__device__ __forceinline__ void head_fwd_all_smem(u64 *s, u64 rowbase, const ulonglong2 *tw,
                                                  const Mod &M) {
  using G = RowGeom<LOG_R>;
  if constexpr (I < G::NPASS) {
    head_fwd<LB, LOG_R, G::S0(I), G::R(I), 1, false>(s, nullptr, nullptr, rowbase, tw, M);
    __syncthreads();
    head_fwd_all_smem<LB, LOG_R, I + 1>(s, rowbase, tw, M);
  }
}

// tail pass: E consecutive elements per thread (the last LOG_E row-local
// stages), optionally with the fused middle in between.
template <int LB, int LOG_R, int NP, int FWD, bool MID, int INV, int MODE>
__device__ __forceinline__ void tail_pass(u64 *__restrict__ sm, u64 rowbase,
                                          const ulonglong2 *__restrict__ twf,
                                          const ulonglong2 *__restrict__ twi,
                                          const Limb &L, const Mod &M) {
  using G = RowGeom<LOG_R>;
  constexpr int E = G::E;
  constexpr int LE = G::HEAD == 0 ? 0 : LOG_R - G::HEAD;  // = LOG_E
  // lazy Barrett middle (proposed/dhem constants, all moduli < 2^60)
  constexpr bool LAZY_MID = NTTB_LAZY_MID && MODE == NTTMUL_RED_ONE_SUB && LB >= 16;
  // multiply-based partial reductions around the middle (LB = 32)
  constexpr bool FAST = LAZY_MID && LB >= 32;
  const int o0 = threadIdx.x * E;
  const u64 B0 = (rowbase << G::HEAD) + threadIdx.x;
#if NTTB_TW_PREFETCH
  TwBuf<0, LE - 1> twb;
  if constexpr (MID) tw_prefetch(twb, twf, B0);
#endif
  const UnitIdx<LOG_R, 0> ix(o0);
  u64 xa[1][E];
#pragma unroll
  for (int e = 0; e < E; ++e) xa[0][e] = sm[ix(e)];
  if constexpr (MID) {
    // a's last truncated stages first, parked (canonical) in its own smem
    // slots; then b's, kept in registers and overwritten by c pair by pair.
#if NTTB_TW_PREFETCH
    fwd_radix_pf<LB, LE, LE - 1, 1, G::HEAD & 1>(xa, twb, M);
#else
    fwd_radix<LB, LE, LE - 1, 1, G::HEAD & 1>(xa, B0, twf, M);
#endif
#pragma unroll
    for (int e = 0; e < E; ++e)
      sm[ix(e)] =
          LAZY_MID ? to2q_any<LB>(xa[0][e], M) : canon_fwd<LB>(xa[0][e], M);
#pragma unroll
    for (int e = 0; e < E; ++e) xa[0][e] = sm[G::PADN + ix(e)];
#if NTTB_TW_PREFETCH
    fwd_radix_pf<LB, LE, LE - 1, 1, G::HEAD & 1>(xa, twb, M);
    tw_prefetch(twb, twi, B0);  // inverse twiddles of the same groups
#else
    fwd_radix<LB, LE, LE - 1, 1, G::HEAD & 1>(xa, B0, twf, M);
#endif
    // pair p = (2p, 2p+1); twiddle tw[n/4 + i/2] == tw[(B0 << (LE-2)) + p/2]
    // (the k = 2 stage's group twiddle); sign of the z term = parity of the
    // global pair index = parity of p.
#pragma unroll
    for (int p = 0; p < E / 2; p += 2) {
      const ulonglong2 w = ldtw(twf, (B0 << (LE - 2)) + (p >> 1));
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i0 = 2 * (p + h);
        if constexpr (LAZY_MID)
          fused_pair_lazy<FAST, lb_pm<LB>()>(sm[ix(i0)], sm[ix(i0 + 1)],
                                to2q_any<LB>(xa[0][i0], M), to2q_any<LB>(xa[0][i0 + 1], M), w.x,
                                w.y, h != 0, L, M, xa[0][i0], xa[0][i0 + 1]);
        else
          fused_pair<MODE>(sm[ix(i0)], sm[ix(i0 + 1)],
                           canon_fwd<LB>(xa[0][i0], M), canon_fwd<LB>(xa[0][i0 + 1], M),
                           w.x, w.y, h != 0, L, M, xa[0][i0], xa[0][i0 + 1]);
      }
    }
#if NTTB_TW_PREFETCH
    inv_radix_pf<LB, LE, LE - 1, 0, 1>(xa, twb, M);
#else
    inv_radix<LB, LE, LE - 1, 0, 1>(xa, B0, twi, M);
#endif
#pragma unroll
    for (int e = 0; e < E; ++e) sm[ix(e)] = xa[0][e];
  } else {
    static_assert(NP == 1, "unfused row passes transform one polynomial");
    if (FWD == FWD_FULL) fwd_radix<LB, LE, LE, 1, G::HEAD & 1>(xa, B0, twf, M);
    if (FWD == FWD_TRUNC) fwd_radix<LB, LE, LE - 1, 1, G::HEAD & 1>(xa, B0, twf, M);
    if (INV == INV_FULL) inv_radix<LB, LE, LE, 0, 1>(xa, B0, twi, M);
    if (INV == INV_SKIP) inv_radix<LB, LE, LE - 1, 0, 1>(xa, B0, twi, M);
    if (INV == INV_NONE) {
#pragma unroll
      for (int e = 0; e < E; ++e) xa[0][e] = canon_fwd<LB>(xa[0][e], M);
    }
#pragma unroll
    for (int e = 0; e < E; ++e) sm[ix(e)] = xa[0][e];
  }
}

// fused tail with a and b in separate smem buffers (persistent kernel);
// c is written over a.
template <int LB, int LOG_R, int MODE>
__device__ __forceinline__ void tail_pass_split(u64 *__restrict__ sa, u64 *__restrict__ sb,
                                                u64 rowbase,
                                                const ulonglong2 *__restrict__ twf,
                                                const ulonglong2 *__restrict__ twi,
                                                const Limb &L, const Mod &M) {
  using G = RowGeom<LOG_R>;
  constexpr int E = G::E;
  constexpr int LE = LOG_R - G::HEAD;
  const int o0 = threadIdx.x * E;
  const u64 B0 = (rowbase << G::HEAD) + threadIdx.x;
  u64 xa[1][E];
#pragma unroll
  for (int e = 0; e < E; ++e) xa[0][e] = sa[G::idx(o0 + e)];
  fwd_radix<LB, LE, LE - 1, 1, G::HEAD & 1>(xa, B0, twf, M);
#pragma unroll
  for (int e = 0; e < E; ++e) sa[G::idx(o0 + e)] = canon_fwd<LB>(xa[0][e], M);
#pragma unroll
  for (int e = 0; e < E; ++e) xa[0][e] = sb[G::idx(o0 + e)];
  fwd_radix<LB, LE, LE - 1, 1, G::HEAD & 1>(xa, B0, twf, M);
#pragma unroll
  for (int p = 0; p < E / 2; p += 2) {
    const ulonglong2 w = ldtw(twf, (B0 << (LE - 2)) + (p >> 1));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i0 = 2 * (p + h);
      fused_pair<MODE>(sa[G::idx(o0 + i0)], sa[G::idx(o0 + i0 + 1)], canon_fwd<LB>(xa[0][i0], M),
                       canon_fwd<LB>(xa[0][i0 + 1], M), w.x, w.y, h != 0, L, M, xa[0][i0],
                       xa[0][i0 + 1]);
    }
  }
  inv_radix<LB, LE, LE - 1, 0, 1>(xa, B0, twi, M);
#pragma unroll
  for (int e = 0; e < E; ++e) sa[G::idx(o0 + e)] = xa[0][e];
}

// Split CTA barrier (mbarrier): every thread arrives as soon as its writes
// are done and waits only where it needs the other threads' data, so the
// work placed between arrive and wait hides the barrier.
#ifndef NTTB_SPLIT_BAR
#define NTTB_SPLIT_BAR 1
#endif
__device__ __forceinline__ void sbar_init(u64 *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(bar))),
               "r"(count)
               : "memory");
}
__device__ __forceinline__ void sbar_arrive(u64 *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(bar)))
               : "memory");
}
__device__ __forceinline__ void sbar_wait(u64 *bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "SBAR_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra SBAR_WAIT_%=;\n\t}" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(bar))),
      "r"(parity)
      : "memory");
}

template <int LOG_R, int FWD, bool MID, int INV, int MODE, int LB>
__global__ void __launch_bounds__(RowGeom<LOG_R>::T,
                                  MID ? NTTB_ROW_MINB_FUSED : NTTB_ROW_MINB)
    row_kernel(const RowParams P) {
  using G = RowGeom<LOG_R>;
  constexpr int NP = MID ? 2 : 1;
  extern __shared__ u64 sm[];
  const long long row = blockIdx.x;
  const long long poly = row >> P.log_n1;
  const int r = static_cast<int>(row & ((1LL << P.log_n1) - 1));
  int limb;
  const Limb &L = *limb_ptr(P.limbs, poly, limb);
  const Mod M = mod_for<LB>(L.q);
  const ulonglong2 *twf = P.tw.fwd + limb * P.tw.stride;
  const ulonglong2 *twi = P.tw.inv + limb * P.tw.stride;
  const u64 rowbase = (1ULL << P.log_n1) + r;  // (N1 + r): group index base
  const long long off = row * G::N2;
  NTTB_STAMP(0);
  // Rows are dispatched in order, so the CTA that takes row + pf_dist (one
  // resident wave later) starts about when this one ends: pull its inputs
  // into L2 now so its first pass does not wait on HBM latency.
  if (FWD != FWD_NONE && P.pf_dist > 0 && threadIdx.x == 0 && row + P.pf_dist < P.nrows) {
    const long long nx = (row + P.pf_dist) * G::N2;
    prefetch_l2(P.in0 + nx, G::N2 * sizeof(u64));
    if (NP > 1) prefetch_l2(P.in1 + nx, G::N2 * sizeof(u64));
  }

  constexpr bool SPLIT = NTTB_SPLIT_BAR && NTTB_B_OWN_COPIES && G::R(0) == NTTB_ROW_LOG_E &&
                        G::NPASS >= 2;
  __shared__ u64 sbar[2];  // SPLIT: a's / b's first pass written
  if (MID && NTTB_PREFETCH_B && SPLIT) {
    // b's row streams into its smem slot (cp.async, each thread exactly the
    // words its own first-pass unit reads) while a's first pass loads and
    // transforms a.  The CTA-wide dependency pass 0 -> pass 1 is split per
    // polynomial: arrive after a's pass 0, b's pass 0, wait(a), a's pass 1,
    // wait(b), b's pass 1 - the waits are mostly satisfied by then.
    if (threadIdx.x == 0) {
      sbar_init(&sbar[0], G::T);
      sbar_init(&sbar[1], G::T);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    row_prefetch<LOG_R>(sm + G::PADN, P.in1 + off);
    cp_async_commit();
    __syncthreads();  // barrier init visible (all threads are at the start)
    head_fwd<LB, LOG_R, 0, G::R(0), 1, true>(sm, P.in0 + off, nullptr, rowbase, twf, M);
    sbar_arrive(&sbar[0]);
    cp_async_wait<0>();
    head_fwd<LB, LOG_R, 0, G::R(0), 1, false>(sm + G::PADN, nullptr, nullptr, rowbase, twf, M);
    sbar_arrive(&sbar[1]);
    sbar_wait(&sbar[0], 0);
    head_fwd<LB, LOG_R, G::S0(1), G::R(1), 1, false>(sm, nullptr, nullptr, rowbase, twf, M);
    sbar_wait(&sbar[1], 0);
    head_fwd<LB, LOG_R, G::S0(1), G::R(1), 1, false>(sm + G::PADN, nullptr, nullptr, rowbase,
                                                     twf, M);
    row_sync<LOG_R, G::S0(1)>();
    head_fwd_all<LB, LOG_R, NP, 2>(sm, nullptr, nullptr, rowbase, twf, M);
    if (P.discard_in) {
      constexpr int LINES = G::N2 * 8 / 128;
      for (int i = threadIdx.x; i < NP * LINES; i += G::T)
        discard_line((i < LINES ? P.in0 : P.in1) + off + (i % LINES) * 16);
    }
  } else if (MID && NTTB_PREFETCH_B) {
    // b's row streams into its smem slot (cp.async) while a's first pass
    // loads and transforms a; then b's first pass runs from smem.
    row_prefetch<LOG_R>(sm + G::PADN, P.in1 + off);
    cp_async_commit();
    head_fwd<LB, LOG_R, 0, G::R(0), 1, true>(sm, P.in0 + off, nullptr, rowbase, twf, M);
    NTTB_STAMP(5);
    cp_async_wait<0>();
    // Thread t copied exactly the words t + 512 k that its pass-0 unit of b
    // reads (row_prefetch and head_fwd<S0 = 0> share the mapping), so its
    // own wait_group makes them visible: no CTA barrier before b's pass 0.
    if (!(NTTB_B_OWN_COPIES && G::R(0) == NTTB_ROW_LOG_E))
      __syncthreads();
    NTTB_STAMP(1);
    head_fwd<LB, LOG_R, 0, G::R(0), 1, false>(sm + G::PADN, nullptr, nullptr, rowbase, twf, M);
    pass_tw_l1<LOG_R, 1>(twf, rowbase);
    __syncthreads();
    NTTB_STAMP(6);
    head_fwd_all<LB, LOG_R, NP, 1>(sm, nullptr, nullptr, rowbase, twf, M);
    if (P.discard_in) {
      constexpr int LINES = G::N2 * 8 / 128;
      for (int i = threadIdx.x; i < NP * LINES; i += G::T)
        discard_line((i < LINES ? P.in0 : P.in1) + off + (i % LINES) * 16);
    }
  } else if (FWD != FWD_NONE) {
    head_fwd_all<LB, LOG_R, NP>(sm, P.in0 + off, NP > 1 ? P.in1 + off : nullptr, rowbase,
                                twf, M);
    if (P.discard_in) {  // every element of the input rows is now in smem
      constexpr int LINES = G::N2 * 8 / 128;
      for (int i = threadIdx.x; i < NP * LINES; i += G::T) {
        const u64 *src = (i < LINES ? P.in0 : P.in1) + off;
        discard_line(src + (i % LINES) * 16);
      }
    }
  } else {
#pragma unroll 4
    for (int i = threadIdx.x; i < G::N2; i += G::T) sm[G::idx(i)] = P.in0[off + i];
    __syncthreads();
  }
  NTTB_STAMP(2);
  tail_pass<LB, LOG_R, NP, FWD, MID, INV, MODE>(sm, rowbase, twf, twi, L, M);
  if (INV != INV_NONE || MID) pass_tw_l1<LOG_R, G::NPASS - 1>(twi, rowbase);
  if (INV != INV_NONE || MID)
    row_sync<LOG_R, G::S0(G::NPASS - 1)>();  // the inverse passes read back this tail
  else
    __syncthreads();  // the plain store below reads the whole row
  NTTB_STAMP(3);
  if (INV != INV_NONE || MID) {
    head_inv_all<LB, LOG_R, G::NPASS - 1>(sm, P.out + off, rowbase, twi, L, M,
                                          P.log_n1 == 0 ? P.fin : FIN_LAZY);
    NTTB_STAMP(4);
#ifdef NTTB_PHASE_TIMING
    __syncthreads();  // the CTA's last warp
    NTTB_STAMP(7);
#endif
  } else {
#pragma unroll 4
    for (int i = threadIdx.x; i < G::N2; i += G::T) P.out[off + i] = sm[G::idx(i)];
  }
}

// ---------------------------------------------------------------------------
// PERSISTENT fused row kernel with a software-pipelined input stream.
//
// One CTA per resident slot walks rows gridDim.x apart.  The next row's
// inputs are copied (cp.async) into the SAME two buffers as soon as each
// becomes free, so no extra shared memory is needed: b's buffer is free once
// the tail has consumed b (its copy is issued before the last inverse pass),
// a's buffer once the last inverse pass has read it (its copy is issued at
// the end of the row).  The next row then starts with b's first pass (data
// already landed) while a's copy completes.  In the one-row-per-CTA kernel
// both CTAs of an SM start together and wait on HBM together; here that
// latency hides behind the previous row's last pass.

// inverse head passes I .. 1, each followed by its barrier (the one after
// pass 1 is the whole-row barrier before pass 0)
template <int LB, int LOG_R, int I>
__device__ __forceinline__ void head_inv_to1(u64 *sm, u64 rowbase, const ulonglong2 *tw,
                                             const Limb &L, const Mod &M) {
  using G = RowGeom<LOG_R>;
  if constexpr (I > 0) {
    head_inv<LB, LOG_R, G::S0(I), G::R(I), false>(sm, nullptr, rowbase, tw, L, M, FIN_LAZY);
    row_sync<LOG_R, G::S0(I - 1)>();
    head_inv_to1<LB, LOG_R, I - 1>(sm, rowbase, tw, L, M);
  }
}

template <int LOG_R, int MODE, int LB>
__global__ void __launch_bounds__(RowGeom<LOG_R>::T, NTTB_ROW_MINB_FUSED)
    row_fused_persistent(const RowParams P, long long nrows) {
  using G = RowGeom<LOG_R>;
  extern __shared__ u64 sm[];
  u64 *const sa = sm, *const sb = sm + G::PADN;
  long long row = blockIdx.x;
  if (row < nrows) {
    row_prefetch<LOG_R>(sb, P.in1 + row * G::N2);
    cp_async_commit();
    row_prefetch<LOG_R>(sa, P.in0 + row * G::N2);
    cp_async_commit();
  }
  for (; row < nrows; row += gridDim.x) {
    const long long poly = row >> P.log_n1;
    const int r = static_cast<int>(row & ((1LL << P.log_n1) - 1));
    int limb;
    const Limb &L = *limb_ptr(P.limbs, poly, limb);
    const Mod M = mod_for<LB>(L.q);
    const ulonglong2 *twf = P.tw.fwd + limb * P.tw.stride;
    const ulonglong2 *twi = P.tw.inv + limb * P.tw.stride;
    const u64 rowbase = (1ULL << P.log_n1) + r;
    const long long off = row * G::N2;
    const long long next = row + gridDim.x;
    NTTB_STAMP(0);
    cp_async_wait<1>();  // b(row) has landed; a(row) may still be in flight
    __syncthreads();
    head_fwd<LB, LOG_R, 0, G::R(0), 1, false>(sb, nullptr, nullptr, rowbase, twf, M);
    cp_async_wait<0>();  // a(row)
    __syncthreads();
    head_fwd<LB, LOG_R, 0, G::R(0), 1, false>(sa, nullptr, nullptr, rowbase, twf, M);
    __syncthreads();
    NTTB_STAMP(1);
    head_fwd_all<LB, LOG_R, 2, 1>(sm, nullptr, nullptr, rowbase, twf, M);
    NTTB_STAMP(2);
    tail_pass<LB, LOG_R, 2, FWD_TRUNC, true, INV_SKIP, MODE>(sm, rowbase, twf, twi, L, M);
    row_sync<LOG_R, G::S0(G::NPASS - 1)>();
    NTTB_STAMP(3);
    head_inv_to1<LB, LOG_R, G::NPASS - 1>(sm, rowbase, twi, L, M);
    // whole-row barrier passed: b is dead, refill its buffer with b(next)
    if (next < nrows) row_prefetch<LOG_R>(sb, P.in1 + next * G::N2);
    cp_async_commit();
    head_inv<LB, LOG_R, 0, G::R(0), true>(sa, P.out + off, rowbase, twi, L, M,
                                          P.log_n1 == 0 ? P.fin : FIN_LAZY);
    __syncthreads();  // every thread has read a's buffer
    if (next < nrows) row_prefetch<LOG_R>(sa, P.in0 + next * G::N2);
    cp_async_commit();
    NTTB_STAMP(4);
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// COLUMN kernels (N2 = 4096 columns per polynomial, N1 = 2^LOG_N1 rows)

#ifndef NTTB_COL_LOG_R
#define NTTB_COL_LOG_R 12
#endif
#ifndef NTTB_COL_VEC
#define NTTB_COL_VEC 1
#endif
#ifndef NTTB_COL_SMEM_TW
#define NTTB_COL_SMEM_TW 1
#endif
#ifndef NTTB_COL_MINB
#define NTTB_COL_MINB 4  // forward columns at 4 CTAs/SM (64 regs) since the loads go out first: col fwd 0.145 -> 0.123 ms (sweep_r60)
#endif
#ifndef NTTB_COL_INV_LOADS_FIRST
#define NTTB_COL_INV_LOADS_FIRST 1  // with 4 CTAs/SM: col inv 0.0803 -> 0.0763 ms (sweep_r62)
#endif
#ifndef NTTB_COL_MINB_INV
#define NTTB_COL_MINB_INV 4
#endif
constexpr int COL_LOG_R = NTTB_COL_LOG_R;  // row length used for n > 2^COL_LOG_R
constexpr int COL_THREADS = 256;
constexpr int COL_VEC = NTTB_COL_VEC;      // adjacent columns per thread (1 or 2)
static_assert(COL_VEC == 1 || COL_VEC == 2, "column vector width");

struct ColParams {
  const u64 *src0;
  const u64 *src1;
  u64 *dst0;
  u64 *dst1;
  int nsrc;  // 1 or 2 source/destination pairs
  long long npolys;
  TwSet tw;
  LimbSet limbs;
  int fin;  // inverse: FinalMode of the last stage (global m == 1)
  int discard_src;  // sources are pipeline scratch: discard after reading
};

// Each thread owns COL_VEC adjacent columns (one 8*COL_VEC-byte vector per
// row, coalesced across the warp) and runs all LOG_N1 column stages on them
// in registers; the stages' twiddles tw[1 .. N1) are uniform across the grid.
// Per-direction geometry (measured, sweep_r26): the forward pass (two
// sources, 4 stages) runs one column per thread with up to 128 registers;
// the inverse pass (one source + folded scale) one column per thread at 4
// CTAs per SM (64 registers).
template <bool INV, int LOG_N1 = 4>
struct ColGeom {
  static constexpr int V = NTTB_COL_VEC;
  // 32-word columns (n = 2^17) need the register budget of 2 CTAs/SM
  static constexpr int MINB = LOG_N1 >= 5 ? 2 : (INV ? NTTB_COL_MINB_INV : NTTB_COL_MINB);
};

template <int LOG_N1, bool INV, int LB>
__global__ void __launch_bounds__(COL_THREADS, (ColGeom<INV, LOG_N1>::MINB)) col_kernel(const ColParams P) {
  constexpr int N1 = 1 << LOG_N1;
  constexpr int V = ColGeom<INV>::V;
  const long long vecs = (P.npolys << COL_LOG_R) / V;  // column vectors per source
  // a CTA's COL_THREADS * V columns lie in one polynomial of one source
  // (4096 columns per polynomial), so source, polynomial and limb are
  // CTA-uniform: derive them from blockIdx only
  const long long cta0 = blockIdx.x * static_cast<long long>(COL_THREADS);
  if (cta0 >= vecs * P.nsrc) return;
  const int which = cta0 >= vecs ? 1 : 0;
  const long long rem = (cta0 - (which ? vecs : 0)) * V + threadIdx.x * V;  // first column
  const long long poly = ((cta0 - (which ? vecs : 0)) * V) >> COL_LOG_R;
  const long long base =
      (poly << (COL_LOG_R + LOG_N1)) + (rem & ((1 << COL_LOG_R) - 1));
  int limb;
  const Limb &L = *limb_ptr(P.limbs, poly, limb);
  const Mod M = mod_for_stages<LB>(L.q);
  const u64 *__restrict__ src = (which ? P.src1 : P.src0) + base;
  u64 *__restrict__ dst = (which ? P.dst1 : P.dst0) + base;
#if NTTB_COL_SMEM_TW
  // The N1 - 1 column twiddles are the same for the whole CTA (its 256
  // columns lie in one polynomial): stage them in shared memory so the
  // butterflies read them just in time (LDS broadcast) instead of the
  // compiler hoisting 2 x (N1 - 1) global loads into registers.  The
  // column loads go out first and the staging barrier overlaps their HBM
  // latency (forward -4 %, then 4 CTAs/SM -15 %; inverse at 4 CTAs/SM -5 %).
  __shared__ ulonglong2 stw[N1];
  auto stage_tw = [&] {
    const ulonglong2 *tg = (INV ? P.tw.inv : P.tw.fwd) + limb * P.tw.stride;
    if (threadIdx.x < N1) stw[threadIdx.x] = tg[threadIdx.x];
    __syncthreads();
  };
  if (INV && !NTTB_COL_INV_LOADS_FIRST) stage_tw();
#endif
  u64 x[V][N1];
#pragma unroll
  for (int e = 0; e < N1; ++e) {
    const long long o = static_cast<long long>(e) << COL_LOG_R;
    if (V == 2) {
      const ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(src + o);
      x[0][e] = v.x;
      x[V - 1][e] = v.y;
    } else {
      x[0][e] = ldg_hint<L2_FIRST>(src + o);
    }
  }
#if NTTB_COL_SMEM_TW
  if (!INV || NTTB_COL_INV_LOADS_FIRST) stage_tw();
#endif
#if NTTB_COL_SMEM_TW
  const ulonglong2 *twc = stw;
#else
  const ulonglong2 *twc = (INV ? P.tw.inv : P.tw.fwd) + limb * P.tw.stride;
#endif
  if constexpr (LOG_N1 == 5 && V == 1) {
    // 32-row columns (n = 2^17): the stage whose pairs straddle the two
    // 16-element halves runs on the whole column, the other four stages as
    // two radix-16 units (B0 = 2 + h) - the single 5-stage unit is not
    // register-promoted by the compiler (its 32-word array went to local
    // memory).  Same butterflies, twiddles and reduction parity.
    if (!INV) {
      const ulonglong2 w = ldtw(twc, 1);
#pragma unroll
      for (int e = 0; e < 16; ++e) ct_bfly<LB, true>(x[0][e], x[0][e + 16], w.x, w.y, M);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      u64 y[1][16];
#pragma unroll
      for (int e = 0; e < 16; ++e) y[0][e] = x[0][16 * h + e];
      if (!INV)
        fwd_radix<LB, 4, 4, 1, 1>(y, 2 + h, twc, M);
      else
        inv_radix<LB, 4, 4, 0, 1>(y, 2 + h, twc, M);
#pragma unroll
      for (int e = 0; e < 16; ++e) x[0][16 * h + e] = y[0][e];
    }
    if (INV) inv_stage0<LB, LOG_N1, V>(x, 1, twc, L, M, P.fin);
  } else if (!INV) {
    fwd_radix<LB, LOG_N1, LOG_N1, V>(x, 1, twc, M);
  } else {
    const ulonglong2 *twi = twc;
    inv_radix<LB, LOG_N1, LOG_N1, 1, V>(x, 1, twi, M);
    inv_stage0<LB, LOG_N1, V>(x, 1, twi, L, M, P.fin);
  }
  if (P.discard_src && (threadIdx.x & (16 / V - 1)) == 0) {
    // these 16/V lanes consumed whole 128-byte lines (16 columns x N1 rows)
#pragma unroll
    for (int e = 0; e < N1; ++e) discard_line(src + (static_cast<long long>(e) << COL_LOG_R));
  }
#pragma unroll
  for (int e = 0; e < N1; ++e) {
    const long long o = static_cast<long long>(e) << COL_LOG_R;
    if (V == 2) {
      *reinterpret_cast<ulonglong2 *>(dst + o) = make_ulonglong2(x[0][e], x[V - 1][e]);
    } else {
      if (INV)
        stg_hint<L2_FIRST>(dst + o, x[0][e]);  // the product: not read again here
      else
        stg_hint<L2_LAST>(dst + o, x[0][e]);   // a', b': the row kernel reads them next
    }
  }
}

// ---------------------------------------------------------------------------
// PIPELINED COLUMN kernel (default for n > 4096).
//
// The plain column kernel above is latency-bound: each thread's 2 x N1
// strided loads must land before any arithmetic, and 128 registers per
// thread cap residency at 16 warps per SM.  Here a persistent CTA streams
// column TILES (N1 rows x TC columns, rows contiguous TC*8-byte segments)
// through a STAGES-deep shared-memory ring with the bulk-copy engine
// (cp.async.bulk global->shared, completion counted on an mbarrier), so
// the next tiles are in flight while the current one is transformed; results
// go back through the same buffer with bulk shared->global stores.  One
// thread owns one column (N1 values in registers); a warp reads 32
// consecutive words of a row - conflict-free.

namespace bulk {
__device__ __forceinline__ unsigned saddr(const void *p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(u64 *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u64 *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(u64 *bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(saddr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void load(void *dst, const void *src, unsigned bytes, u64 *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar))
      : "memory");
}
__device__ __forceinline__ void store(void *dst, const void *src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(saddr(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
}  // namespace bulk

#ifndef NTTB_COLPIPE_TC
#define NTTB_COLPIPE_TC 256
#endif
#ifndef NTTB_COLPIPE_STAGES
#define NTTB_COLPIPE_STAGES 2
#endif
template <int LOG_N1>
struct ColPipeGeom {
  static constexpr int N1 = 1 << LOG_N1;
  static constexpr int TC = LOG_N1 >= 5 ? 128 : NTTB_COLPIPE_TC;  // columns per tile = threads
  static constexpr int STAGES = NTTB_COLPIPE_STAGES;
  static constexpr int TILE_WORDS = N1 * TC;
  static constexpr int TILES_PER_POLY = (1 << COL_LOG_R) / TC;
  static constexpr size_t SMEM = STAGES * TILE_WORDS * sizeof(u64) + 64;  // + barriers
};

template <int LOG_N1, bool INV, int LB>
__global__ void __launch_bounds__(ColPipeGeom<LOG_N1>::TC)
    col_pipe_kernel(const ColParams P) {
  using G = ColPipeGeom<LOG_N1>;
  constexpr int N1 = G::N1, TC = G::TC, S = G::STAGES;
  constexpr unsigned ROW_BYTES = TC * sizeof(u64);
  extern __shared__ __align__(128) u64 csm[];
  u64 *bars = csm + S * G::TILE_WORDS;
  const long long per_src = P.npolys * G::TILES_PER_POLY;
  const long long ntiles = per_src * P.nsrc;
  // tile -> (source, polynomial, first column)
  auto where = [&](long long t, int &which, long long &poly, int &col0) {
    which = t >= per_src ? 1 : 0;
    const long long r = t - (which ? per_src : 0);
    poly = r / G::TILES_PER_POLY;
    col0 = static_cast<int>(r % G::TILES_PER_POLY) * TC;
  };
  auto issue_load = [&](long long t, int s) {
    int which, col0;
    long long poly;
    where(t, which, poly, col0);
    const u64 *src = (which ? P.src1 : P.src0) + (poly << (COL_LOG_R + LOG_N1)) + col0;
    bulk::mbar_expect_tx(bars + s, N1 * ROW_BYTES);
#pragma unroll 1
    for (int e = 0; e < N1; ++e)
      bulk::load(csm + s * G::TILE_WORDS + e * TC, src + (static_cast<long long>(e) << COL_LOG_R),
                 ROW_BYTES, bars + s);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) bulk::mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = 0; s < S; ++s) {
      const long long t = blockIdx.x + static_cast<long long>(s) * gridDim.x;
      if (t < ntiles) issue_load(t, s);
    }
  int it = 0;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int s = it % S;
    int which, col0;
    long long poly;
    where(t, which, poly, col0);
    int limb;
    const Limb &L = *limb_ptr(P.limbs, poly, limb);
    const Mod M = mod_for_stages<LB>(L.q);
    u64 *buf = csm + s * G::TILE_WORDS;
    bulk::mbar_wait(bars + s, (it / S) & 1);
    u64 x[1][N1];
#pragma unroll
    for (int e = 0; e < N1; ++e) x[0][e] = buf[e * TC + threadIdx.x];
    if (!INV) {
      fwd_radix<LB, LOG_N1, LOG_N1, 1>(x, 1, P.tw.fwd + limb * P.tw.stride, M);
    } else {
      const ulonglong2 *twi = P.tw.inv + limb * P.tw.stride;
      inv_radix<LB, LOG_N1, LOG_N1, 1, 1>(x, 1, twi, M);
      inv_stage0<LB, LOG_N1, 1>(x, 1, twi, L, M, P.fin);
    }
#pragma unroll
    for (int e = 0; e < N1; ++e) buf[e * TC + threadIdx.x] = x[0][e];
    bulk::fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      u64 *dst = (which ? P.dst1 : P.dst0) + (poly << (COL_LOG_R + LOG_N1)) + col0;
#pragma unroll 1
      for (int e = 0; e < N1; ++e)
        bulk::store(dst + (static_cast<long long>(e) << COL_LOG_R), buf + e * TC, ROW_BYTES);
      bulk::commit();
      // refill the buffer stored one iteration ago (its reads are done once
      // at most the group just committed is still reading)
      if (it >= 1) {
        const int sp = (it - 1) % S;
        const long long tn = t - gridDim.x + static_cast<long long>(S) * gridDim.x;
        if (tn < ntiles) {
          bulk::wait_read<1>();
          issue_load(tn, sp);
        }
      }
    }
  }
  // the last tile's buffer is never refilled; drain outstanding stores
  if (threadIdx.x == 0) bulk::wait_all();
}

// ---------------------------------------------------------------------------
// GROUP-PERSISTENT FUSED kernel (the fused product for n = N1 x 4096).
//
// The three-launch pipeline (COL -> ROW -> COL^-1) sends every intermediate
// through HBM (72 n bytes per limb-product instead of 24 n) and runs the two
// column launches latency-bound.  Here one cooperative launch keeps all of
// it on chip: the resident CTAs form groups of N1; a group owns one
// limb-product at a time and walks it through three phases separated by a
// group barrier (release/acquire on a global counter):
//   1. CTA i transforms column slab i (4096/N1 columns x N1 rows of a and b,
//      read from HBM) and writes a', b' to the group's scratch;
//   2. CTA i runs the fused row pass on row i (row stages of a, b, the
//      Karatsuba middle and the inverse row stages) from scratch, c' over a';
//   3. CTA i runs the inverse column stages (with the folded scale) on slab
//      i of c' and writes c to HBM.
// Scratch (triple-buffered per group, 3 MiB per group for n = 2^16) stays in
// L2, and every scratch line is discarded once consumed, so HBM sees only a,
// b (read) and c (written).  Different groups drift out of phase, so the
// memory-bound column phases of one group overlap the integer-bound row
// phases of the group sharing its SMs.

struct GroupParams {
  u64 *out;
  const u64 *a;
  const u64 *b;
  u64 *scratch;            // groups x 3 buffers x {a', b'} x n words
  unsigned *counters;      // two per group, zero at launch
  TwSet tw;
  LimbSet limbs;
  long long npolys;
  int groups;
};

// split group barrier: arrive (release) after a phase, wait (acquire) later,
// so independent work can run in between
__device__ __forceinline__ void group_arrive(unsigned *ctr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
  }
}
__device__ __forceinline__ void group_wait(unsigned *ctr, unsigned target) {
  if (threadIdx.x == 0) {
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while (v < target);
    __threadfence();  // also invalidates this SM's L1 (scratch written elsewhere)
  }
  __syncthreads();
}

// scratch buffers of product number `it` of a group: {a' (then c'), b'}
__device__ __forceinline__ u64 *group_buf(const GroupParams &P, int g, int it, long long n) {
  return P.scratch + (static_cast<long long>(g) * 3 + it % 3) * 2 * n;
}

// phase 1: forward column stages of slab i of a and b -> a', b'
template <int LOG_N1, int LB>
__device__ __noinline__ void group_phase1(const GroupParams &P, long long p, int i, u64 *sa) {
  constexpr int N1 = 1 << LOG_N1, N2 = 1 << COL_LOG_R, SW = N2 / N1;
  constexpr long long N = static_cast<long long>(N1) * N2;
  int limb;
  const Limb &L = *limb_ptr(P.limbs, p, limb);
  const Mod M = mod_for_stages<LB>(L.q);
  const ulonglong2 *twf = P.tw.fwd + limb * P.tw.stride;
#pragma unroll 1
  for (int j = threadIdx.x; j < 2 * SW; j += blockDim.x) {
    const int which = j >= SW;
    const int col = i * SW + (j - (which ? SW : 0));
    const u64 *src = (which ? P.b : P.a) + p * N + col;
    u64 *dst = sa + (which ? N : 0) + col;
    u64 x[1][N1];
#pragma unroll
    for (int e = 0; e < N1; ++e) x[0][e] = src[static_cast<long long>(e) * N2];
    fwd_radix<LB, LOG_N1, LOG_N1, 1>(x, 1, twf, M);
#pragma unroll
    for (int e = 0; e < N1; ++e) dst[static_cast<long long>(e) * N2] = x[0][e];
  }
}

// phase 2: the fused row pass on row i of (a', b'); c' over a'
template <int LOG_N1, int MODE, int LB>
__device__ __noinline__ void group_phase2(const GroupParams &P, long long p, int i, u64 *sa,
                                          u64 *sm) {
  using G = RowGeom<COL_LOG_R>;
  constexpr int N1 = 1 << LOG_N1, N2 = G::N2;
  constexpr long long N = static_cast<long long>(N1) * N2;
  int limb;
  const Limb &L = *limb_ptr(P.limbs, p, limb);
  const Mod M = mod_for<LB>(L.q);
  const ulonglong2 *twf = P.tw.fwd + limb * P.tw.stride;
  const ulonglong2 *twi = P.tw.inv + limb * P.tw.stride;
  const u64 rowbase = static_cast<u64>(N1) + i;
  const long long off = static_cast<long long>(i) * N2;
  const u64 *sb = sa + N;
  row_prefetch<COL_LOG_R>(sm + G::PADN, sb + off);
  cp_async_commit();
  head_fwd<LB, COL_LOG_R, 0, G::R(0), 1, true>(sm, sa + off, nullptr, rowbase, twf, M);
  cp_async_wait<0>();
  __syncthreads();
  head_fwd<LB, COL_LOG_R, 0, G::R(0), 1, false>(sm + G::PADN, nullptr, nullptr, rowbase, twf, M);
  __syncthreads();
  head_fwd_all<LB, COL_LOG_R, 2, 1>(sm, nullptr, nullptr, rowbase, twf, M);
  // b' is consumed: drop its lines from L2 without a write-back
  constexpr int LINES = N2 * 8 / 128;
  for (int l = threadIdx.x; l < LINES; l += blockDim.x) discard_line(sb + off + l * 16);
  tail_pass<LB, COL_LOG_R, 2, FWD_TRUNC, true, INV_SKIP, MODE>(sm, rowbase, twf, twi, L, M);
  row_sync<COL_LOG_R, G::S0(G::NPASS - 1)>();
  head_inv_all<LB, COL_LOG_R, G::NPASS - 1>(sm, sa + off, rowbase, twi, L, M, FIN_LAZY);
}

// phase 3: inverse column stages (+ folded scale) of slab i of c' -> c
template <int LOG_N1, int LB>
__device__ __noinline__ void group_phase3(const GroupParams &P, long long p, int i, u64 *sa) {
  constexpr int N1 = 1 << LOG_N1, N2 = 1 << COL_LOG_R, SW = N2 / N1;
  constexpr long long N = static_cast<long long>(N1) * N2;
  int limb;
  const Limb &L = *limb_ptr(P.limbs, p, limb);
  const Mod M = mod_for_stages<LB>(L.q);
  const ulonglong2 *twi = P.tw.inv + limb * P.tw.stride;
#pragma unroll 1
  for (int j = threadIdx.x; j < SW; j += blockDim.x) {
    const int col = i * SW + j;
    const u64 *src = sa + col;
    u64 x[1][N1];
#pragma unroll
    for (int e = 0; e < N1; ++e) x[0][e] = src[static_cast<long long>(e) * N2];
    inv_radix<LB, LOG_N1, LOG_N1, 1, 1>(x, 1, twi, M);
    inv_stage0<LB, LOG_N1, 1>(x, 1, twi, L, M, FIN_SCALED_SKIP);
    // every lane's loads have returned (their values were consumed): the
    // 16 consecutive columns of a 128-byte line per row can be dropped
    if ((j & 15) == 0)
#pragma unroll
      for (int e = 0; e < N1; ++e) discard_line(src + static_cast<long long>(e) * N2);
    u64 *dst = P.out + p * N + col;
#pragma unroll
    for (int e = 0; e < N1; ++e) dst[static_cast<long long>(e) * N2] = x[0][e];
  }
}

// Schedule per CTA (k = the group's k-th product), with split barriers so
// independent work fills the waits:
//   P1(0) arrive1 | for k: wait1(k) P2(k) arrive2 [P1(k+1) arrive1] wait2(k) P3(k)
// Scratch is triple-buffered: a slow CTA may still read buffer k-1 in P3(k-1)
// while a fast one writes buffer k+1 in P1(k+1).
template <int LOG_N1, int MODE, int LB>
__global__ void __launch_bounds__(RowGeom<COL_LOG_R>::T, NTTB_ROW_MINB_FUSED)
    group_fused_kernel(const GroupParams P) {
  constexpr int N1 = 1 << LOG_N1;
  constexpr long long N = static_cast<long long>(N1) << COL_LOG_R;
  extern __shared__ u64 sm[];
  const int g = blockIdx.x / N1, i = blockIdx.x % N1;
  if (g >= P.groups) return;
  unsigned *ctr1 = P.counters + 2 * g, *ctr2 = ctr1 + 1;
  unsigned t1 = 0, t2 = 0;
  if (g < P.npolys) {
    group_phase1<LOG_N1, LB>(P, g, i, group_buf(P, g, 0, N));
    group_arrive(ctr1);
    t1 += N1;
  }
  int k = 0;
#ifdef NTTB_PHASE_TIMING
#define GSTAMP(j) \
  if (k == 4 && threadIdx.x == 0 && blockIdx.x < (1u << 16)) g_phase[blockIdx.x][j] = clock64();
#else
#define GSTAMP(j)
#endif
  for (long long p = g; p < P.npolys; p += P.groups, ++k) {
    u64 *sa = group_buf(P, g, k, N);
    GSTAMP(0);
    group_wait(ctr1, t1);
    GSTAMP(1);
    group_phase2<LOG_N1, MODE, LB>(P, p, i, sa, sm);
    group_arrive(ctr2);
    GSTAMP(2);
    t2 += N1;
    if (p + P.groups < P.npolys) {
      group_phase1<LOG_N1, LB>(P, p + P.groups, i, group_buf(P, g, k + 1, N));
      group_arrive(ctr1);
      t1 += N1;
    }
    GSTAMP(3);
    group_wait(ctr2, t2);
    GSTAMP(4);
    group_phase3<LOG_N1, LB>(P, p, i, sa);
    GSTAMP(5);
  }
#undef GSTAMP
}

// ---------------------------------------------------------------------------
// SMALL kernel: n <= 2^12, one CTA per polynomial (per pair when fused);
// stage loop over shared memory.  Used for n < 2^10 (the reference's unit
// test sizes); also a schedule-independent cross-check of the row kernel.

struct SmallParams {
  u64 *out;
  const u64 *in0;
  const u64 *in1;
  TwSet tw;
  LimbSet limbs;
  int log_n;
  int fwd;  // FwdKind
  int mid;  // fused middle (requires two inputs)
  int inv;  // InvKind
  int fin;  // FinalMode for the m == 1 inverse stage
};

template <int MODE, int LB>
__global__ void __launch_bounds__(256) small_kernel(const SmallParams P) {
  extern __shared__ u64 sm[];
  const int n = 1 << P.log_n;
  const int np = P.mid ? 2 : 1;
  const long long poly = blockIdx.x;
  int limb;
  const Limb L = get_limb(P.limbs, poly, limb);
  const Mod M = mod_for<LB>(L.q);
  const ulonglong2 *twf = P.tw.fwd + limb * P.tw.stride;
  const ulonglong2 *twi = P.tw.inv + limb * P.tw.stride;
  const long long off = poly * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    sm[i] = P.in0[off + i];
    if (np > 1) sm[n + i] = P.in1[off + i];
  }
  __syncthreads();
  if (P.fwd != FWD_NONE) {
    const int limit = (P.fwd == FWD_TRUNC) ? n / 2 : n;
    for (int m = 1, k = n / 2, stage = 0; m < limit; m <<= 1, k >>= 1, ++stage) {
      for (int b = threadIdx.x; b < n / 2; b += blockDim.x) {
        const int i = b / k, j = 2 * i * k + (b % k);
        const ulonglong2 w = ldtw(twf, m + i);
        for (int p = 0; p < np; ++p)
          if (LB < 16 || (stage & 1) == 0)
            ct_bfly<LB, true>(sm[p * n + j], sm[p * n + j + k], w.x, w.y, M);
          else
            ct_bfly<LB, false>(sm[p * n + j], sm[p * n + j + k], w.x, w.y, M);
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < np * n; i += blockDim.x) sm[i] = canon_fwd<LB>(sm[i], M);
    __syncthreads();
  }
  if (P.mid) {
    for (int i = threadIdx.x; i < n / 2; i += blockDim.x) {
      const ulonglong2 w = ldtw(twf, n / 4 + i / 2);
      u64 c0, c1;
      fused_pair<MODE>(sm[2 * i], sm[2 * i + 1], sm[n + 2 * i], sm[n + 2 * i + 1],
                       w.x, w.y, (i & 1) != 0, L, M, c0, c1);
      sm[2 * i] = c0;
      sm[2 * i + 1] = c1;
    }
    __syncthreads();
  }
  if (P.inv != INV_NONE) {
    const int m0 = (P.inv == INV_SKIP) ? n / 4 : n / 2;
    const int k0 = (P.inv == INV_SKIP) ? 2 : 1;
    for (int m = m0, k = k0; m >= 1; m >>= 1, k <<= 1) {
      for (int b = threadIdx.x; b < n / 2; b += blockDim.x) {
        const int i = b / k, j = 2 * i * k + (b % k);
        if (m == 1 && P.fin >= FIN_SCALED_FULL) {
          const u64 *sc = (P.fin == FIN_SCALED_FULL) ? L.sc_full : L.sc_skip;
          const u64 s[4] = {sc[0], sc[1], sc[2], sc[3]};
          gs_bfly_last_scaled<LB>(sm[j], sm[j + k], s, M);
        } else {
          const ulonglong2 w = ldtw(twi, m + i);
          gs_bfly<LB>(sm[j], sm[j + k], w.x, w.y, M);
        }
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = canon_inv<LB>(sm[i], M);
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) P.out[off + i] = sm[i];
}

// ---------------------------------------------------------------------------
// elementwise kernels (reference _kernels.pyx hadamard / scale / fused_middle
// / mulmod_loop)

template <int MODE>
__global__ void __launch_bounds__(256)
    hadamard_kernel(const u64 *__restrict__ a, const u64 *__restrict__ b,
                    u64 *__restrict__ out, long long n, const Limb L) {
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * 256)
    out[i] = mulred<MODE>(a[i], b[i], L);
}

template <int MODE>
__global__ void __launch_bounds__(256)
    scale_kernel(u64 *__restrict__ a, u64 factor, long long n, const Limb L) {
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * 256)
    a[i] = mulred<MODE>(a[i], factor, L);
}

template <int MODE>
__global__ void __launch_bounds__(256)
    fused_middle_kernel(const u64 *__restrict__ ah, const u64 *__restrict__ bh,
                        u64 *__restrict__ ch, const ulonglong2 *__restrict__ tw,
                        int log_n, long long npairs, const Limb L) {
  const int half = 1 << (log_n - 1);
  for (long long g = blockIdx.x * 256LL + threadIdx.x; g < npairs;
       g += static_cast<long long>(gridDim.x) * 256) {
    const long long i = g & (half - 1);
    const ulonglong2 w = ldtw(tw, (1LL << (log_n - 2)) + (i >> 1));
    u64 c0, c1;
    fused_pair<MODE>(ah[2 * g], ah[2 * g + 1], bh[2 * g], bh[2 * g + 1], w.x, w.y,
                     (i & 1) != 0, L, make_mod(L.q), c0, c1);
    ch[2 * g] = c0;
    ch[2 * g + 1] = c1;
  }
}

template <int MODE>
__global__ void __launch_bounds__(256)
    mulmod_loop_kernel(const u64 *__restrict__ a, const u64 *__restrict__ b,
                       long long n, u64 passes, u64 *sink, const Limb L) {
  u64 acc = 0;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * 256) {
    const u64 r = mulred<MODE>(a[i], b[i], L);
    if (passes & 1) acc ^= r;  // x ^ x == 0: an even pass count cancels
  }
  for (int o = 16; o > 0; o >>= 1) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicXor(reinterpret_cast<unsigned long long *>(sink), static_cast<unsigned long long>(acc));
}

// ---------------------------------------------------------------------------
// plan construction (reference params.py:153-181) and validation (:184-207)

__device__ __forceinline__ u64 powmod(u64 base, u64 e, const Limb &L) {
  u64 r = 1 % L.q;
  while (e) {
    if (e & 1) r = mulred<NTTMUL_RED_ONE_SUB>(r, base, L);
    base = mulred<NTTMUL_RED_ONE_SUB>(base, base, L);
    e >>= 1;
  }
  return r;
}

__device__ __forceinline__ u64 shoup_companion(u64 w, u64 q) {
  return static_cast<u64>((static_cast<unsigned __int128>(w) << 64) / q);
}

// L must carry the proposed-variant Barrett constants.
__global__ void __launch_bounds__(256)
    twiddle_kernel(u64 *tw_fwd, u64 *tw_inv, ulonglong2 *fwd_pairs,
                   ulonglong2 *inv_pairs, u64 psi, u64 psi_inv, int log_n,
                   const Limb L) {
  const long long i = blockIdx.x * 256LL + threadIdx.x;
  if (i >= (1LL << log_n)) return;
  const u64 br = __brevll(static_cast<u64>(i)) >> (64 - log_n);
  const u64 f = powmod(psi, br, L);
  const u64 v = powmod(psi_inv, br, L);
  if (tw_fwd) tw_fwd[i] = f;
  if (tw_inv) tw_inv[i] = v;
  if (fwd_pairs) fwd_pairs[i] = make_ulonglong2(f, shoup_companion(f, L.q));
  if (inv_pairs) inv_pairs[i] = make_ulonglong2(v, shoup_companion(v, L.q));
}

__global__ void __launch_bounds__(256)
    shoup_pairs_kernel(ulonglong2 *pairs, const u64 *tw, u64 q, long long n) {
  const long long i = blockIdx.x * 256LL + threadIdx.x;
  if (i < n) pairs[i] = make_ulonglong2(tw[i], shoup_companion(tw[i], q));
}

__global__ void __launch_bounds__(256)
    check_twiddles_kernel(const u64 *f, const u64 *v, long long n,
                          unsigned long long *bad, const Limb L) {
  const long long i = blockIdx.x * 256LL + threadIdx.x;
  if (i >= n) return;
  int b = 0;
  if (f[i] >= L.q || v[i] >= L.q ||
      mulred<NTTMUL_RED_BUILTIN>(f[i], v[i], L) != 1)
    b = 1;
  if (i == 0 && (f[0] != 1 || v[0] != 1)) b += 1;
  if (b) atomicAdd(bad, static_cast<unsigned long long>(b));
}

// ---------------------------------------------------------------------------
// register-resident modmul microbenchmark (int-pipe roof)

template <int KIND, int MODE, int CHAINS>
__global__ void __launch_bounds__(256)
    modmul_roof_kernel(long long iters, u64 *sink, const Limb L, u64 w,
                       u64 wp) {
  u64 x[CHAINS];
  const Mod M = (KIND >= 4 && L.q >= (1ULL << 34)) ? make_mod_fast(L.q) : make_mod(L.q);
  const u64 seed = (blockIdx.x * 256ULL + threadIdx.x) * 0x9E3779B97F4A7C15ULL;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = (seed + c * 0x632BE59BD9B4E019ULL) % L.q;
  for (long long it = 0; it < iters; ++it) {
    if (KIND == 2) {  // Harvey forward butterflies, [0, 8q) lazy bound
#pragma unroll
      for (int c = 0; c < CHAINS / 2; ++c) ct_bfly<8>(x[c], x[c + CHAINS / 2], w, wp, M);
    } else if (KIND == 3) {  // inverse butterflies, [0, 4q)
#pragma unroll
      for (int c = 0; c < CHAINS / 2; ++c) gs_bfly<8>(x[c], x[c + CHAINS / 2], w, wp, M);
    } else if (KIND == 4) {  // forward butterflies, LB = 32 pattern (reduce, plain, plain)
#pragma unroll
      for (int c = 0; c < CHAINS / 2; ++c) {
        ct_bfly<32, true>(x[c], x[c + CHAINS / 2], w, wp, M);
        ct_bfly<32, false>(x[c], x[c + CHAINS / 2], w, wp, M);
        ct_bfly<32, false>(x[c], x[c + CHAINS / 2], w, wp, M);
      }
    } else if (KIND == 6) {  // forward butterflies, shift-shaped moduli (LB = 33: reduce, plain)
#pragma unroll
      for (int c = 0; c < CHAINS / 2; ++c) {
        ct_bfly<33, true>(x[c], x[c + CHAINS / 2], w, wp, M);
        ct_bfly<33, false>(x[c], x[c + CHAINS / 2], w, wp, M);
      }
    } else if (KIND == 7) {  // inverse butterflies, shift-shaped moduli
#pragma unroll
      for (int c = 0; c < CHAINS / 2; ++c) {
        gs_bfly<33, true>(x[c], x[c + CHAINS / 2], w, wp, M);
        gs_bfly<33, false>(x[c], x[c + CHAINS / 2], w, wp, M);
      }
    } else if (KIND == 5) {  // inverse butterflies, LB = 32 pattern (reduce, plain)
#pragma unroll
      for (int c = 0; c < CHAINS / 2; ++c) {
        gs_bfly<32, true>(x[c], x[c + CHAINS / 2], w, wp, M);
        gs_bfly<32, false>(x[c], x[c + CHAINS / 2], w, wp, M);
      }
    } else {
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) {
        if (KIND == 0)
          x[c] = mulred<MODE>(x[c], x[(c + 1) % CHAINS], L);
        else
          x[c] = shoup(x[c], w, wp, M);
      }
    }
  }
  u64 acc = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc ^= x[c];
  if (acc == 0x123456789ULL) atomicXor(reinterpret_cast<unsigned long long *>(sink), static_cast<unsigned long long>(acc));  // keep the work alive
}

}  // namespace nttb
