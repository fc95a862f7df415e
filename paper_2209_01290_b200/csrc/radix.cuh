// radix.cuh - register-resident multi-stage butterflies.
//
// The merged CT forward NTT (reference _kernels.pyx:52-85, paper Alg. 5) at
// stage "m groups, half-size k" pairs (j, j+k) inside group i = j / 2k with
// twiddle tw[m + i].  A thread that owns 2^R elements spaced k_last apart
// (one "unit") can run R consecutive stages in registers: at unit-local stage
// t the unit splits into 2^t groups and group gi uses tw[(B0 << t) + gi],
// where B0 is the twiddle index of the unit's group at its first stage.
// The GS inverse (reference _kernels.pyx:88-129, Alg. 6) is the exact mirror
// with the inverse table.  Everything below is fully unrolled: element and
// twiddle indices are compile-time, so the arrays live in registers.
#pragma once
#include "modarith.cuh"

namespace nttb {

// Twiddle pair load.  NTTB_TW_LDG selects the read-only (.nc) path; the
// default plain load keeps the compiler from hoisting every pass's twiddles
// above the CTA barriers (which multiplies register pressure).
__device__ __forceinline__ ulonglong2 ldtw(const ulonglong2 *__restrict__ tw,
                                           u64 idx) {
#ifdef NTTB_TW_LDG
  return __ldg(tw + idx);
#else
  return tw[idx];
#endif
}

// Forward stages t in [0, TSTOP) of a radix-2^R unit, NP polynomials sharing
// the twiddles.  Values stay in the forward lazy range of LB.
// PAR: parity of the kernel-local index of stage t = 0 (LB = 16 reduces on
// even kernel-local stages, so every kernel starts with a reducing stage).
template <int LB, int R, int TSTOP, int NP, int PAR = 0>
__device__ __forceinline__ void fwd_radix(u64 (&x)[NP][1 << R], u64 B0,
                                          const ulonglong2 *__restrict__ tw,
                                          const Mod &M) {
#pragma unroll
  for (int t = 0; t < TSTOP; ++t) {
    const int half = 1 << (R - 1 - t);
#pragma unroll
    for (int gi = 0; gi < (1 << t); ++gi) {
      const ulonglong2 w = ldtw(tw, (B0 << t) + gi);
#pragma unroll
      for (int e = 0; e < half; ++e) {
        const int i0 = gi * 2 * half + e;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          if (((PAR + t) & 1) == 0)
            ct_bfly<LB, true>(x[p][i0], x[p][i0 + half], w.x, w.y, M);
          else
            ct_bfly<LB, false>(x[p][i0], x[p][i0 + half], w.x, w.y, M);
        }
      }
    }
  }
}

// Inverse stages t = TSTART-1 down to TEND (inverse lazy range of LB).
template <int LB, int R, int TSTART, int TEND, int NP>
__device__ __forceinline__ void inv_radix(u64 (&x)[NP][1 << R], u64 B0,
                                          const ulonglong2 *__restrict__ tw,
                                          const Mod &M) {
#pragma unroll
  for (int t = TSTART - 1; t >= TEND; --t) {
    const int half = 1 << (R - 1 - t);
#pragma unroll
    for (int gi = 0; gi < (1 << t); ++gi) {
      const ulonglong2 w = ldtw(tw, (B0 << t) + gi);
#pragma unroll
      for (int e = 0; e < half; ++e) {
        const int i0 = gi * 2 * half + e;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          if (((TSTART - 1 - t) & 1) == 0)  // each call starts with a reducing stage
            gs_bfly<LB, true>(x[p][i0], x[p][i0 + half], w.x, w.y, M);
          else
            gs_bfly<LB, false>(x[p][i0], x[p][i0 + half], w.x, w.y, M);
        }
      }
    }
  }
}

// Twiddle prefetch: the (B0 << t) + gi pairs of stages [T0, T1) of a unit,
// packed stage by stage (stage t at offset (1 << t) - (1 << T0)).  Issuing
// them before the unit's data loads overlaps their L2 latency.
template <int T0, int T1>
struct TwBuf {
  static constexpr int N = (1 << T1) - (1 << T0);
  ulonglong2 w[N > 0 ? N : 1];
};

template <int T0, int T1>
__device__ __forceinline__ void tw_prefetch(TwBuf<T0, T1> &b, const ulonglong2 *__restrict__ tw,
                                            u64 B0) {
#pragma unroll
  for (int t = T0; t < T1; ++t)
#pragma unroll
    for (int gi = 0; gi < (1 << t); ++gi) b.w[(1 << t) - (1 << T0) + gi] = ldtw(tw, (B0 << t) + gi);
}

// fwd_radix over stages [0, TSTOP) with prefetched twiddles
template <int LB, int R, int TSTOP, int NP, int PAR = 0>
__device__ __forceinline__ void fwd_radix_pf(u64 (&x)[NP][1 << R], const TwBuf<0, TSTOP> &b,
                                             const Mod &M) {
#pragma unroll
  for (int t = 0; t < TSTOP; ++t) {
    const int half = 1 << (R - 1 - t);
#pragma unroll
    for (int gi = 0; gi < (1 << t); ++gi) {
      const ulonglong2 w = b.w[(1 << t) - 1 + gi];
#pragma unroll
      for (int e = 0; e < half; ++e) {
        const int i0 = gi * 2 * half + e;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          if (((PAR + t) & 1) == 0)
            ct_bfly<LB, true>(x[p][i0], x[p][i0 + half], w.x, w.y, M);
          else
            ct_bfly<LB, false>(x[p][i0], x[p][i0 + half], w.x, w.y, M);
        }
      }
    }
  }
}

// inv_radix over stages TSTART-1 .. TEND with prefetched twiddles of [0, TS)
template <int LB, int R, int TSTART, int TEND, int NP, int TS>
__device__ __forceinline__ void inv_radix_pf(u64 (&x)[NP][1 << R], const TwBuf<0, TS> &b,
                                             const Mod &M) {
#pragma unroll
  for (int t = TSTART - 1; t >= TEND; --t) {
    const int half = 1 << (R - 1 - t);
#pragma unroll
    for (int gi = 0; gi < (1 << t); ++gi) {
      const ulonglong2 w = b.w[(1 << t) - 1 + gi];
#pragma unroll
      for (int e = 0; e < half; ++e) {
        const int i0 = gi * 2 * half + e;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          if (((TSTART - 1 - t) & 1) == 0)
            gs_bfly<LB, true>(x[p][i0], x[p][i0 + half], w.x, w.y, M);
          else
            gs_bfly<LB, false>(x[p][i0], x[p][i0 + half], w.x, w.y, M);
        }
      }
    }
  }
}

// Final-mode of the last inverse stage that a kernel runs.
enum FinalMode {
  FIN_LAZY = 0,         // more inverse stages follow in another pass/kernel
  FIN_PLAIN = 1,        // global last stage, unscaled, canonical output
  FIN_SCALED_FULL = 2,  // global last stage, x 2^-log_n (intt_gs scaled)
  FIN_SCALED_SKIP = 3   // global last stage, x 2^-(log_n-1) (skip_first)
};

// Stage t = 0 of an inverse unit (one group, twiddle tw[B0]) with the final
// treatment.  The scaled modes are only legal when B0 == 1 (global m == 1).
template <int LB, int R, int NP>
__device__ __forceinline__ void inv_stage0(u64 (&x)[NP][1 << R], u64 B0,
                                           const ulonglong2 *__restrict__ tw,
                                           const Limb &L, const Mod &M, int fin) {
  constexpr int half = 1 << (R - 1);
  if (fin >= FIN_SCALED_FULL) {
    u64 sc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      sc[i] = (fin == FIN_SCALED_FULL) ? L.sc_full[i] : L.sc_skip[i];
#pragma unroll
    for (int e = 0; e < half; ++e)
#pragma unroll
      for (int p = 0; p < NP; ++p) gs_bfly_last_scaled<LB>(x[p][e], x[p][e + half], sc, M);
  } else {
    const ulonglong2 w = ldtw(tw, B0);
    if (fin == FIN_PLAIN) {
#pragma unroll
      for (int e = 0; e < half; ++e)
#pragma unroll
        for (int p = 0; p < NP; ++p)
          gs_bfly_last_plain<LB>(x[p][e], x[p][e + half], w.x, w.y, M);
    } else {
#pragma unroll
      for (int e = 0; e < half; ++e)
#pragma unroll
        for (int p = 0; p < NP; ++p) gs_bfly<LB>(x[p][e], x[p][e + half], w.x, w.y, M);
    }
  }
}

}  // namespace nttb
