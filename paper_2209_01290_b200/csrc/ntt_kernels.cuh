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
#ifndef NTTB_LAZY_MID
#define NTTB_LAZY_MID 1
#endif
#ifndef NTTB_ROW_TAIL_G
#define NTTB_ROW_TAIL_G 1  // standalone rows: tail reads / writes global directly
#endif

#ifndef NTTB_ROW_LOG_E12
#define NTTB_ROW_LOG_E12 NTTB_ROW_LOG_E  // elements per thread of the 4096-word rows
#endif
constexpr int row_log_e(int log_r) { return log_r == 12 ? NTTB_ROW_LOG_E12 : NTTB_ROW_LOG_E; }

template <int LOG_R, int LOG_E = row_log_e(LOG_R)>
struct RowGeom {
  static constexpr int LE = LOG_E;
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
  int discard_in;  // inputs are pipeline scratch: drop their L2 lines once read
  long long nrows;    // rows in this launch
  long long pf_dist;  // > 0: prefetch the input rows of row + pf_dist into L2
};

// Drop a consumed scratch line from L2 without writing it back to HBM
// (discard.global.L2).  `line` must be 128-byte aligned and fully consumed.
__device__ __forceinline__ void discard_line(const void *line) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(line) : "memory");
}

// Programmatic dependent launch (the column / row / column launches of one
// transform): a kernel signals at its start that its dependents may be
// scheduled (their CTAs then take the SM slots its last wave leaves free)
// and waits for its predecessor's results before touching global data.
// Without the launch attribute both are no-ops / return at once.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

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
#pragma unroll 1
  for (int p = 0; p < NP; ++p) {  // not unrolled: one polynomial's state live
    const u64 *__restrict__ g = p == 0 ? g0 : g1;
    u64 *__restrict__ s = sm + p * G::PADN;
#pragma unroll
    for (int w = 0; w < U; ++w) {
      const int u = threadIdx.x + w * G::T;
      const int grp = u >> LK;
      const int o0 = (grp << (LOG_R - S0)) + (u & ((1 << LK) - 1));
      TwBuf<0, R> twb;
      tw_prefetch(twb, tw, (rowbase << S0) + grp);
      const UnitIdx<LOG_R, LK> ix(o0);
      u64 x[1][1 << R];
#pragma unroll
      for (int e = 0; e < (1 << R); ++e) {
        const int o = o0 + (e << LK);
        x[0][e] = FROM_GLOBAL ? g[o] : s[ix(e)];
      }
      fwd_radix_pf<LB, R, R, 1, S0 & 1>(x, twb, M);
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
    TwBuf<0, R> twb;
    tw_prefetch(twb, tw, B0);
    u64 x[1][1 << R];
    const UnitIdx<LOG_R, LK> ix(o0);
#pragma unroll
    for (int e = 0; e < (1 << R); ++e) x[0][e] = sm[ix(e)];
    if (TO_GLOBAL) {
      inv_radix_pf<LB, R, R, 1, 1>(x, twb, M);
      inv_stage0<LB, R, 1>(x, B0, tw, L, M, fin);
#pragma unroll
      for (int e = 0; e < (1 << R); ++e) *(gout + o0 + (e << LK)) = x[0][e];
    } else {
      inv_radix_pf<LB, R, R, 0, 1>(x, twb, M);
#pragma unroll
      for (int e = 0; e < (1 << R); ++e) sm[ix(e)] = x[0][e];
    }
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
  constexpr bool ONE_UNIT = G::HEAD % G::NPASS == 0 && G::HEAD / G::NPASS == G::LE;
  constexpr int THREADS = 1 << (LOG_R - S0_BLOCK - G::LE);
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

// all forward head passes, pass i = 0 .. NPASS-1 (pass 0 reads global when
// G0, else every pass works in shared memory)
template <int LB, int LOG_R, int NP, int I = 0, bool G0 = true>
__device__ __forceinline__ void head_fwd_all(u64 *sm, const u64 *g0, const u64 *g1,
                                             u64 rowbase, const ulonglong2 *tw,
                                             const Mod &M) {
  using G = RowGeom<LOG_R>;
  if constexpr (I < G::NPASS) {
    head_fwd<LB, LOG_R, G::S0(I), G::R(I), NP, G0 && I == 0>(sm, g0, g1, rowbase, tw, M);
    row_sync<LOG_R, G::S0(I)>();
    head_fwd_all<LB, LOG_R, NP, I + 1, G0>(sm, g0, g1, rowbase, tw, M);
  }
}

// all inverse head passes, pass i = NPASS-1 .. 0 (pass 0 writes global when
// TO_GLOBAL, else back to shared memory with more inverse stages to follow)
template <int LB, int LOG_R, int I, bool TO_GLOBAL = true>
__device__ __forceinline__ void head_inv_all(u64 *sm, u64 *gout, u64 rowbase,
                                             const ulonglong2 *tw, const Limb &L,
                                             const Mod &M, int fin) {
  using G = RowGeom<LOG_R>;
  if constexpr (I > 0) {
    head_inv<LB, LOG_R, G::S0(I), G::R(I), false>(sm, nullptr, rowbase, tw, L, M,
                                                  FIN_LAZY);
    row_sync<LOG_R, G::S0(I - 1)>();
    head_inv_all<LB, LOG_R, I - 1, TO_GLOBAL>(sm, gout, rowbase, tw, L, M, fin);
  } else {
    head_inv<LB, LOG_R, 0, G::R(0), TO_GLOBAL>(sm, gout, rowbase, tw, L, M, fin);
  }
}

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
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
  TwBuf<0, LE - 1> twb;
  if constexpr (MID) tw_prefetch(twb, twf, B0);
  const UnitIdx<LOG_R, 0> ix(o0);
  u64 xa[1][E];
#pragma unroll
  for (int e = 0; e < E; ++e) xa[0][e] = sm[ix(e)];
  if constexpr (MID) {
    // a's last truncated stages first, parked (canonical) in its own smem
    // slots; then b's, kept in registers and overwritten by c pair by pair.
    fwd_radix_pf<LB, LE, LE - 1, 1, G::HEAD & 1>(xa, twb, M);
#pragma unroll
    for (int e = 0; e < E; ++e)
      sm[ix(e)] =
          LAZY_MID ? to2q_any<LB>(xa[0][e], M) : canon_fwd<LB>(xa[0][e], M);
#pragma unroll
    for (int e = 0; e < E; ++e) xa[0][e] = sm[G::PADN + ix(e)];
    fwd_radix_pf<LB, LE, LE - 1, 1, G::HEAD & 1>(xa, twb, M);
    tw_prefetch(twb, twi, B0);  // inverse twiddles of the same groups
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
          fused_pair_lazy<FAST>(sm[ix(i0)], sm[ix(i0 + 1)],
                                to2q_any<LB>(xa[0][i0], M), to2q_any<LB>(xa[0][i0 + 1], M), w.x,
                                w.y, h != 0, L, M, xa[0][i0], xa[0][i0 + 1]);
        else
          fused_pair<MODE>(sm[ix(i0)], sm[ix(i0 + 1)],
                           canon_fwd<LB>(xa[0][i0], M), canon_fwd<LB>(xa[0][i0 + 1], M),
                           w.x, w.y, h != 0, L, M, xa[0][i0], xa[0][i0 + 1]);
      }
    }
    inv_radix_pf<LB, LE, LE - 1, 0, 1>(xa, twb, M);
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

// Tail pass of a standalone (unfused) row reading its E consecutive words
// straight from global memory (inverse rows: no staging copy + barrier in
// front) or writing them straight back (forward rows: no barrier + copy
// loop behind).  16-byte accesses when the row is 16-byte aligned.
template <int LB, int LOG_R, int FWD, int INV, bool G_IN, bool G_OUT>
__device__ __forceinline__ void tail_plain_g(u64 *__restrict__ sm, const u64 *gin, u64 *gout,
                                             u64 rowbase, const ulonglong2 *__restrict__ twf,
                                             const ulonglong2 *__restrict__ twi, const Mod &M) {
  using G = RowGeom<LOG_R>;
  constexpr int E = G::E;
  constexpr int LE = G::HEAD == 0 ? 0 : LOG_R - G::HEAD;
  const int o0 = threadIdx.x * E;
  const u64 B0 = (rowbase << G::HEAD) + threadIdx.x;
  const UnitIdx<LOG_R, 0> ix(o0);
  u64 xa[1][E];
  if constexpr (G_IN) {
    if ((reinterpret_cast<uintptr_t>(gin) & 15) == 0) {
      const ulonglong2 *v = reinterpret_cast<const ulonglong2 *>(gin + o0);
#pragma unroll
      for (int e = 0; e < E / 2; ++e) {
        const ulonglong2 t = v[e];
        xa[0][2 * e] = t.x;
        xa[0][2 * e + 1] = t.y;
      }
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) xa[0][e] = gin[o0 + e];
    }
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) xa[0][e] = sm[ix(e)];
  }
  if (FWD == FWD_FULL) fwd_radix<LB, LE, LE, 1, G::HEAD & 1>(xa, B0, twf, M);
  if (FWD == FWD_TRUNC) fwd_radix<LB, LE, LE - 1, 1, G::HEAD & 1>(xa, B0, twf, M);
  if (INV == INV_FULL) inv_radix<LB, LE, LE, 0, 1>(xa, B0, twi, M);
  if (INV == INV_SKIP) inv_radix<LB, LE, LE - 1, 0, 1>(xa, B0, twi, M);
  if (INV == INV_NONE) {
#pragma unroll
    for (int e = 0; e < E; ++e) xa[0][e] = canon_fwd<LB>(xa[0][e], M);
  }
  if constexpr (G_OUT) {
    if ((reinterpret_cast<uintptr_t>(gout) & 15) == 0) {
      ulonglong2 *v = reinterpret_cast<ulonglong2 *>(gout + o0);
#pragma unroll
      for (int e = 0; e < E / 2; ++e) v[e] = make_ulonglong2(xa[0][2 * e], xa[0][2 * e + 1]);
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) gout[o0 + e] = xa[0][e];
    }
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) sm[ix(e)] = xa[0][e];
  }
}

// Split CTA barrier (mbarrier): every thread arrives as soon as its writes
// are done and waits only where it needs the other threads' data, so the
// work placed between arrive and wait hides the barrier.
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

// resident CTAs per SM of a row kernel (512-thread rows: 2; the 1024-thread
// rows of the 8192-word split: 1)
template <int LOG_R, bool MID>
constexpr int row_minb() {
  return RowGeom<LOG_R>::T >= 1024 ? 1 : (MID ? NTTB_ROW_MINB_FUSED : NTTB_ROW_MINB);
}

template <int LOG_R, int FWD, bool MID, int INV, int MODE, int LB>
__global__ void __launch_bounds__(RowGeom<LOG_R>::T, (row_minb<LOG_R, MID>()))
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
  pdl_launch_dependents();
  pdl_wait();
  // Rows are dispatched in order, so the CTA that takes row + pf_dist (one
  // resident wave later) starts about when this one ends: pull its inputs
  // into L2 now so its first pass does not wait on HBM latency.
  if (FWD != FWD_NONE && P.pf_dist > 0 && threadIdx.x == 0 && row + P.pf_dist < P.nrows) {
    const long long nx = (row + P.pf_dist) * G::N2;
    prefetch_l2(P.in0 + nx, G::N2 * sizeof(u64));
    if (NP > 1) prefetch_l2(P.in1 + nx, G::N2 * sizeof(u64));
  }

  __shared__ u64 sbar[2];  // a's / b's first pass written
  if constexpr (MID) {
    static_assert(G::R(0) == G::LE && G::NPASS >= 2, "fused row geometry");
    // b's row streams into its smem slot (cp.async, each thread exactly the
    // words its own first-pass unit reads) while a's first pass loads and
    // transforms a.  The CTA-wide dependency pass 0 -> pass 1 is split per
    // polynomial (mbarrier): arrive after a's pass 0, b's pass 0, wait(a),
    // a's pass 1, wait(b), b's pass 1 - the waits are mostly satisfied by
    // then (row 0.529 -> 0.519 ms, r55).
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
      // the input rows are pipeline scratch (a' in c, b' in the workspace)
      // and now live only in shared memory: drop their L2 lines without a
      // write-back.  (This loop also changes ptxas's schedule of the tail:
      // without it the kernel spills 40 instead of 24 bytes and runs 1.6 %
      // slower, r2 A/B.)
      constexpr int LINES = G::N2 * 8 / 128;
      for (int i = threadIdx.x; i < NP * LINES; i += G::T)
        discard_line((i < LINES ? P.in0 : P.in1) + off + (i % LINES) * 16);
    }
  } else if constexpr (FWD != FWD_NONE && INV == INV_NONE && NTTB_ROW_TAIL_G) {
    // standalone forward row: the tail writes the row straight to global
    head_fwd_all<LB, LOG_R, NP>(sm, P.in0 + off, nullptr, rowbase, twf, M);
    tail_plain_g<LB, LOG_R, FWD, INV, false, true>(sm, nullptr, P.out + off, rowbase, twf, twi,
                                                   M);
    return;
  } else if constexpr (FWD == FWD_NONE && INV != INV_NONE && NTTB_ROW_TAIL_G) {
    // standalone inverse row: the tail reads the row straight from global
    tail_plain_g<LB, LOG_R, FWD, INV, true, false>(sm, P.in0 + off, nullptr, rowbase, twf, twi,
                                                   M);
    row_sync<LOG_R, G::S0(G::NPASS - 1)>();
    head_inv_all<LB, LOG_R, G::NPASS - 1>(sm, P.out + off, rowbase, twi, L, M,
                                          P.log_n1 == 0 ? P.fin : FIN_LAZY);
    return;
  } else if (FWD != FWD_NONE) {
    head_fwd_all<LB, LOG_R, NP>(sm, P.in0 + off, nullptr, rowbase, twf, M);
  } else {
#pragma unroll 4
    for (int i = threadIdx.x; i < G::N2; i += G::T) sm[G::idx(i)] = P.in0[off + i];
    __syncthreads();
  }
  tail_pass<LB, LOG_R, NP, FWD, MID, INV, MODE>(sm, rowbase, twf, twi, L, M);
  if (INV != INV_NONE || MID)
    row_sync<LOG_R, G::S0(G::NPASS - 1)>();  // the inverse passes read back this tail
  else
    __syncthreads();  // the plain store below reads the whole row
  if (INV != INV_NONE || MID) {
    head_inv_all<LB, LOG_R, G::NPASS - 1>(sm, P.out + off, rowbase, twi, L, M,
                                          P.log_n1 == 0 ? P.fin : FIN_LAZY);
  } else {
#pragma unroll 4
    for (int i = threadIdx.x; i < G::N2; i += G::T) P.out[off + i] = sm[G::idx(i)];
  }
}

// ---------------------------------------------------------------------------
// COLUMN kernels (N2 = 4096 columns per polynomial, N1 = 2^LOG_N1 rows)

#ifndef NTTB_COL_MINB
#define NTTB_COL_MINB 4  // forward columns at 4 CTAs/SM (64 regs) since the loads go out first: col fwd 0.145 -> 0.123 ms (sweep_r60)
#endif
#ifndef NTTB_COL_MINB_INV
#define NTTB_COL_MINB_INV 4  // with the loads first: col inv 0.0803 -> 0.0763 ms (sweep_r62)
#endif
constexpr int COL_LOG_R = 12;  // row length used for n > 2^12
constexpr int COL_THREADS = 256;

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
};

// The LOG_N1 column stages of one column held in registers (merged-CT
// stages with half-size k >= N2: group index B0 = 1 at the first stage, so
// they read only tw[1 .. N1)).
template <int LB, int LOG_N1>
__device__ __forceinline__ void col_fwd_stages(u64 (&x)[1][1 << LOG_N1],
                                               const ulonglong2 *twc, const Mod &M) {
  if constexpr (LOG_N1 == 5) {
    // 32-row columns (n = 2^17): the stage whose pairs straddle the two
    // 16-element halves runs on the whole column, the other four stages as
    // two radix-16 units (B0 = 2 + h) - the single 5-stage unit is not
    // register-promoted by the compiler (its 32-word array went to local
    // memory).  Same butterflies, twiddles and reduction parity.
    const ulonglong2 w = ldtw(twc, 1);
#pragma unroll
    for (int e = 0; e < 16; ++e) ct_bfly<LB, true>(x[0][e], x[0][e + 16], w.x, w.y, M);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      u64 y[1][16];
#pragma unroll
      for (int e = 0; e < 16; ++e) y[0][e] = x[0][16 * h + e];
      fwd_radix<LB, 4, 4, 1, 1>(y, 2 + h, twc, M);
#pragma unroll
      for (int e = 0; e < 16; ++e) x[0][16 * h + e] = y[0][e];
    }
  } else {
    fwd_radix<LB, LOG_N1, LOG_N1, 1>(x, 1, twc, M);
  }
}

// Mirror: the inverse column stages, the last one (global m = 1) with the
// final treatment `fin` (scale folded in, canonical output).
template <int LB, int LOG_N1>
__device__ __forceinline__ void col_inv_stages(u64 (&x)[1][1 << LOG_N1], const ulonglong2 *twc,
                                               const Limb &L, const Mod &M, int fin) {
  if constexpr (LOG_N1 == 5) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      u64 y[1][16];
#pragma unroll
      for (int e = 0; e < 16; ++e) y[0][e] = x[0][16 * h + e];
      inv_radix<LB, 4, 4, 0, 1>(y, 2 + h, twc, M);
#pragma unroll
      for (int e = 0; e < 16; ++e) x[0][16 * h + e] = y[0][e];
    }
  } else {
    inv_radix<LB, LOG_N1, LOG_N1, 1, 1>(x, 1, twc, M);
  }
  inv_stage0<LB, LOG_N1, 1>(x, 1, twc, L, M, fin);
}

// Each thread owns COLS columns (one 8-byte word per row each, coalesced
// across the warp; the CTA's columns are first + t + k 256) and runs all
// LOG_N1 column stages on them in registers; the stages' twiddles tw[1 ..
// N1) are uniform across the CTA.  Short columns (N1 <= 8) take several per
// thread so that 16 loads per thread are in flight.
// LOG_R: the row length 2^LOG_R of the split (= the number of columns of a
// polynomial); COL_LOG_R = 12 unless nttmul_set_split chose another.
template <bool INV, int LOG_N1, int LOG_R = COL_LOG_R>
struct ColGeom {
  // 32-word columns (n = 2^17) need the register budget of 2 CTAs/SM
  static constexpr int MINB = LOG_N1 >= 5 ? 2 : (INV ? NTTB_COL_MINB_INV : NTTB_COL_MINB);
  static constexpr int WANT = LOG_N1 >= 4 ? 1 : (16 >> LOG_N1);
  static constexpr int COLS = COL_THREADS * WANT <= (1 << LOG_R) ? WANT : (1 << LOG_R) / COL_THREADS;
  static constexpr int SPAN = COL_THREADS * COLS;  // columns per CTA
};

template <int LOG_N1, bool INV, int LB, int LOG_R = COL_LOG_R>
__global__ void __launch_bounds__(COL_THREADS, (ColGeom<INV, LOG_N1>::MINB)) col_kernel(const ColParams P) {
  constexpr int N1 = 1 << LOG_N1;
  using CG = ColGeom<INV, LOG_N1, LOG_R>;
  constexpr int COLS = CG::COLS;
  const long long cols = P.npolys << LOG_R;  // columns per source
  // a CTA's SPAN columns lie in one polynomial of one source (4096 columns
  // per polynomial), so source, polynomial and limb are CTA-uniform: derive
  // them from blockIdx only
  const long long cta0 = blockIdx.x * static_cast<long long>(CG::SPAN);
  if (cta0 >= cols * P.nsrc) return;
  const int which = cta0 >= cols ? 1 : 0;
  const long long first = cta0 - (which ? cols : 0);
  const long long poly = first >> LOG_R;
  const long long base = (poly << (LOG_R + LOG_N1)) + ((first + threadIdx.x) & ((1 << LOG_R) - 1));
  int limb;
  const Limb &L = *limb_ptr(P.limbs, poly, limb);
  const Mod M = mod_for_stages<LB>(L.q);
  const u64 *__restrict__ src = (which ? P.src1 : P.src0) + base;
  u64 *__restrict__ dst = (which ? P.dst1 : P.dst0) + base;
  pdl_launch_dependents();
  pdl_wait();
  // The column loads go out first; the N1 - 1 twiddles (the same for the
  // whole CTA) are staged in shared memory behind them, so the butterflies
  // read them just in time (LDS broadcast) instead of the compiler hoisting
  // 2 x (N1 - 1) global loads into registers, and the staging barrier
  // overlaps the HBM latency (forward -4 %, then 4 CTAs/SM -15 %; inverse
  // at 4 CTAs/SM -5 %).
  u64 x[COLS][1][N1];
#pragma unroll
  for (int k = 0; k < COLS; ++k)
#pragma unroll
    for (int e = 0; e < N1; ++e)
      x[k][0][e] = src[(static_cast<long long>(e) << LOG_R) + k * COL_THREADS];
  __shared__ ulonglong2 stw[N1];
  const ulonglong2 *tg = (INV ? P.tw.inv : P.tw.fwd) + limb * P.tw.stride;
  if (threadIdx.x < N1) stw[threadIdx.x] = tg[threadIdx.x];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < COLS; ++k) {
    if (!INV)
      col_fwd_stages<LB, LOG_N1>(x[k], stw, M);
    else
      col_inv_stages<LB, LOG_N1>(x[k], stw, L, M, P.fin);
#pragma unroll
    for (int e = 0; e < N1; ++e)
      dst[(static_cast<long long>(e) << LOG_R) + k * COL_THREADS] = x[k][0][e];
  }
}

// ---------------------------------------------------------------------------
// STRIDED PASS kernel: R consecutive column stages [S0, S0 + R) of one
// transform over global memory, one 2^R-element unit per thread (elements
// k_last = n >> (S0 + R) apart, consecutive threads on consecutive j, so
// every load and store is coalesced).  The latency schedule of a single
// large transform chains a few of these (3 stages each) before a row
// kernel of 1024-word rows: more, shorter CTAs than one column kernel whose
// threads each carry a whole 16- or 32-deep column.

struct PassParams {
  u64 *a;
  TwSet tw;
  LimbSet limbs;
  int log_n;
  int s0;
  long long npolys;
  int fin;  // inverse pass with s0 == 0: FinalMode of the global last stage
};

constexpr int PASS_THREADS = 128;

template <int R, bool INV, int LB>
__global__ void __launch_bounds__(PASS_THREADS) pass_kernel(const PassParams P) {
  pdl_launch_dependents();
  pdl_wait();
  const int log_u = P.log_n - R;              // units per polynomial = 2^log_u
  const int log_k = P.log_n - P.s0 - R;       // log2(k_last)
  const long long uid = blockIdx.x * static_cast<long long>(PASS_THREADS) + threadIdx.x;
  if (uid >= (P.npolys << log_u)) return;
  const long long poly = uid >> log_u;
  const long long u = uid & ((1LL << log_u) - 1);
  const long long grp = u >> log_k;
  const long long j = u & ((1LL << log_k) - 1);
  int limb;
  const Limb &L = *limb_ptr(P.limbs, poly, limb);
  const Mod M = mod_for_stages<LB>(L.q);
  const ulonglong2 *tw = (INV ? P.tw.inv : P.tw.fwd) + limb * P.tw.stride;
  u64 *base = P.a + (poly << P.log_n) + (grp << (log_k + R)) + j;
  u64 x[1][1 << R];
#pragma unroll
  for (int e = 0; e < (1 << R); ++e) x[0][e] = base[static_cast<long long>(e) << log_k];
  const u64 B0 = (1ULL << P.s0) + static_cast<u64>(grp);
  if (!INV) {
    fwd_radix<LB, R, R, 1>(x, B0, tw, M);  // starts with a reducing stage
  } else if (P.s0 == 0) {
    inv_radix<LB, R, R, 1, 1>(x, B0, tw, M);
    inv_stage0<LB, R, 1>(x, B0, tw, L, M, P.fin);
  } else {
    inv_radix<LB, R, R, 0, 1>(x, B0, tw, M);
  }
#pragma unroll
  for (int e = 0; e < (1 << R); ++e) base[static_cast<long long>(e) << log_k] = x[0][e];
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
  const Mod M = make_mod(L.q);
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
