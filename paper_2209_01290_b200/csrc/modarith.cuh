// modarith.cuh - 64-bit-word modular arithmetic for sm_100a.
//
// Device restatement of the reference's reduction layer:
//   * Barrett variants (paper Algs. 2-4; reference modarith.py:136-149 and
//     _kernels.pyx:25-35 `_red`) for data x data products.  The quotient
//     estimate ((x >> s_in) * mu) >> s_out is ONE __umul64hi against a
//     pre-shifted mu (nttmul_limb_t.mu_sh, s_hi), so no 128-bit shifts or
//     runtime mode branches remain in the hot loop (mode is a template arg).
//   * Shoup multiplication for products by a fixed twiddle (a Barrett
//     reduction whose quotient constant floor(w * 2^64 / q) is precomputed per
//     twiddle), used with Harvey's lazy butterflies: forward values live in
//     [0, 4q), inverse values in [0, 2q); canonical [0, q) only at API edges.
//     Valid for q < 2^62 (the reference's m <= 62 admissibility bound,
//     modarith.py:57-60), which keeps 4q < 2^64.
// All results that leave a kernel are canonical, so they are bit-identical to
// the reference regardless of which internal reduction produced them.
#pragma once
#include <cstdint>

#include "nttmul_b200.h"

namespace nttb {

typedef uint64_t u64;
typedef nttmul_limb_t Limb;

// x >= m ? x - m : x, for x < m + 2^63 (sign test on the wrapped difference:
// IADD3 + IADD3.X + 2 SEL, no 64-bit compare).
__device__ __forceinline__ u64 csub(u64 x, u64 m) {
  const u64 t = x - m;
  return (static_cast<long long>(t) < 0) ? x : t;
}

// Shoup: x * w mod q in [0, 2q) for any 64-bit x, w < q, wp = floor(w 2^64/q).
__device__ __forceinline__ u64 shoup_lazy(u64 x, u64 w, u64 wp, u64 q) {
  const u64 qh = __umul64hi(x, wp);
  return x * w - qh * q;
}

__device__ __forceinline__ u64 shoup(u64 x, u64 w, u64 wp, u64 q) {
  return csub(shoup_lazy(x, w, wp, q), q);
}

// Barrett data x data product, a, b canonical.  MODE: NTTMUL_RED_*.
template <int MODE>
__device__ __forceinline__ u64 mulred(u64 a, u64 b, const Limb &L) {
  const u64 lo = a * b;
  const u64 hi = __umul64hi(a, b);
  if (MODE == NTTMUL_RED_BUILTIN) {
    const unsigned __int128 x = (static_cast<unsigned __int128>(hi) << 64) | lo;
    return static_cast<u64>(x % L.q);
  }
  // c = x >> s_in, valid for s_in in [0, 63]
  const u64 c = (lo >> L.s_in) | ((hi << 1) << (63 - L.s_in));
  const u64 quot = __umul64hi(c, L.mu_sh) >> L.s_hi;
  u64 r = lo - quot * L.q;  // exact: true remainder + (<=2) q < 2^64
  r = csub(r, L.q);
  if (MODE == NTTMUL_RED_TWO_SUB) r = csub(r, L.q);
  return r;
}

// ---- butterflies ----------------------------------------------------------

// Merged CT forward butterfly (reference _kernels.pyx:66-80), Harvey lazy:
// X, Y in [0, 4q) -> X + wY, X - wY in [0, 4q).
__device__ __forceinline__ void ct_bfly(u64 &X, u64 &Y, u64 w, u64 wp, u64 q,
                                        u64 q2) {
  const u64 x = csub(X, q2);
  const u64 t = shoup_lazy(Y, w, wp, q);
  X = x + t;
  Y = x - t + q2;
}

// Merged GS inverse butterfly (reference _kernels.pyx:102-118, unscaled),
// Harvey lazy: X, Y in [0, 2q) -> X + Y, w (X - Y) in [0, 2q).
__device__ __forceinline__ void gs_bfly(u64 &X, u64 &Y, u64 w, u64 wp, u64 q,
                                        u64 q2) {
  const u64 s = csub(X + Y, q2);
  const u64 d = X - Y + q2;
  X = s;
  Y = shoup_lazy(d, w, wp, q);
}

// Last GS stage (m = 1) with the scale folded in: canonical outputs.
// sc = {f, f', tw_inv[1] f, (tw_inv[1] f)'}.  Replaces the reference's
// per-stage halving (Zhang scaling, _kernels.pyx:115-117); the canonical
// results are identical.
__device__ __forceinline__ void gs_bfly_last_scaled(u64 &X, u64 &Y,
                                                    const u64 (&sc)[4], u64 q,
                                                    u64 q2) {
  const u64 s = X + Y;
  const u64 d = X - Y + q2;
  X = shoup(s, sc[0], sc[1], q);
  Y = shoup(d, sc[2], sc[3], q);
}

// Last GS stage without scaling: canonical outputs.
__device__ __forceinline__ void gs_bfly_last_plain(u64 &X, u64 &Y, u64 w,
                                                   u64 wp, u64 q, u64 q2) {
  gs_bfly(X, Y, w, wp, q, q2);
  X = csub(X, q);
  Y = csub(Y, q);
}

// [0, 4q) -> [0, q)
__device__ __forceinline__ u64 canon4(u64 x, u64 q, u64 q2) {
  return csub(csub(x, q2), q);
}

// Karatsuba-fused middle pair (paper Alg. 8 lines 3-14, reference
// _kernels.pyx:142-173): inputs canonical, outputs canonical.  The twiddle
// product z = v * tw[n/4 + i/2] uses the Shoup pair; the three data products
// use the Barrett variant MODE.
template <int MODE>
__device__ __forceinline__ void fused_pair(u64 a0, u64 a1, u64 b0, u64 b1,
                                           u64 w, u64 wp, bool odd,
                                           const Limb &L, u64 &c0, u64 &c1) {
  const u64 q = L.q;
  const u64 u = mulred<MODE>(a0, b0, L);
  const u64 v = mulred<MODE>(a1, b1, L);
  const u64 s1 = csub(a0 + a1, q);
  const u64 s2 = csub(b0 + b1, q);
  const u64 ww = mulred<MODE>(s1, s2, L);
  const u64 y = csub(ww + q - u, q);
  c1 = csub(y + q - v, q);
  const u64 z = shoup(v, w, wp, q);
  c0 = odd ? csub(u + q - z, q) : csub(u + z, q);
}

}  // namespace nttb
