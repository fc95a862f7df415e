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
//     twiddle), with an approximate three-partial-product quotient, used in
//     lazy butterflies (see LB below); canonical [0, q) only at API edges.
// All results that leave a kernel are canonical, so they are bit-identical to
// the reference regardless of which internal reduction produced them.
#pragma once
#include <cstdint>

#include "nttmul_b200.h"

namespace nttb {

typedef uint64_t u64;
typedef nttmul_limb_t Limb;



// x >= m ? x - m : x, sign-test form (valid for x < m + 2^63): IADD3 +
// IADD3.X + ISETP + 2 SEL.  (A carry-chain form - the borrow of the 64-bit
// subtraction selecting the result - raised spills in the row kernel.)
__device__ __forceinline__ u64 csub(u64 x, u64 m) {
  const u64 t = x - m;
  return (static_cast<long long>(t) < 0) ? x : t;
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

// ---- explicit 32-bit multiply building blocks ----------------------------
// On sm_100 every integer multiply (IMAD, IMAD.WIDE) issues to the single
// "fmaheavy" pipe, which is the roof of this whole path.  These wrappers pin
// the exact SASS (IMAD.WIDE.U32 / IMAD) so ptxas cannot expand a 64-bit
// product into carry-fixup chains.

__device__ __forceinline__ uint32_t lo32(u64 x) { return static_cast<uint32_t>(x); }
__device__ __forceinline__ uint32_t hi32(u64 x) { return static_cast<uint32_t>(x >> 32); }

__device__ __forceinline__ u64 mulw(uint32_t a, uint32_t b) {
  u64 d;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(d) : "r"(a), "r"(b));
  return d;
}

__device__ __forceinline__ u64 madw(uint32_t a, uint32_t b, u64 c) {
  u64 d;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}

// 32-bit multiply-add and {lo, hi} packing in PTX.  Written as C++
// (`(u64)h << 32 | lo` with h = sum of products) the composition is
// re-associated by the compiler into a 64-bit add whose low half adds zero
// (a wasted IADD3 + IMAD.X per product); the explicit forms keep it to the
// 32-bit IMAD chain.
__device__ __forceinline__ uint32_t madlo(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

__device__ __forceinline__ u64 pack(uint32_t lo, uint32_t hi) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}

// Per-prime constants the butterflies need.
struct Mod {
  u64 q, q2, q4, q8;
  uint32_t nql, nqh;  // halves of 2^64 - q
  uint32_t fr, fs;    // LB >= 32 only: multiply-based reduction constants (reduce2q)
};

__device__ __forceinline__ Mod make_mod(u64 q) {
  Mod m;
  m.q = q;
  m.q2 = 2 * q;
  m.q4 = 4 * q;
  m.q8 = 8 * q;
  const u64 nq = 0 - q;
  m.nql = lo32(nq);
  m.nqh = hi32(nq);
  m.fr = 0;
  m.fs = 0;
  return m;
}

// Multiply-based partial reduction of any x < 2^64 to [0, 2q) for moduli of
// 35..62 bits: k = floor(hi32(x) r / 2^(32+s)) with r = floor(2^(64+s)/q) - 1
// < 2^32 (s = bits(q) - 33) undershoots floor(x/q) by at most 1 (the dropped
// low word contributes < 2^(33-bits) and r's truncation < 2^-26), so
// x - k q lies in [0, 2q).  One IMAD.HI + one IMAD.WIDE + IMAD + a 64-bit
// subtract, instead of a chain of conditional subtractions.  The constants
// come from a double division (rd < 2^32; the -1 absorbs its rounding).
__device__ __forceinline__ Mod make_mod_fast(u64 q) {
  Mod m = make_mod(q);
  const int bits = 64 - __clzll(static_cast<long long>(q));
  m.fs = static_cast<uint32_t>(bits - 33);
  const double rd = ldexp(1.0, 64 + static_cast<int>(m.fs)) / static_cast<double>(q);
  m.fr = static_cast<uint32_t>(rd) - 1;
  return m;
}

// LB = 32: the LB = 16 lazy ranges for moduli of 35..60 bits, where the
// fused middle's partial reductions are multiply-based (reduce2q).  (Using
// them for the transform stages' corrections too measured slower: the
// IMAD.HI / IMAD.WIDE quotient lands on the already busier multiply pipe,
// row 0.574 vs 0.551 ms, sweep_r35.)
template <int LB>
__device__ __forceinline__ Mod mod_for(u64 q) {
  return LB >= 32 ? make_mod_fast(q) : make_mod(q);
}
// Constants for kernels that run transform stages only (no fused middle):
// no multiply-based reduction constants, so no double division.
template <int LB>
__device__ __forceinline__ Mod mod_for_stages(u64 q) {
  return make_mod(q);
}

__device__ __forceinline__ u64 reduce2q(u64 x, const Mod &M) {
  uint32_t k;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(k) : "r"(hi32(x)), "r"(M.fr));
  k >>= M.fs;
  const uint32_t kh = k * hi32(M.q);
  return x - (mulw(k, lo32(M.q)) + (static_cast<u64>(kh) << 32));
}

// floor(x * y / 2^64) - e, e in {0, 1}: the high word from three of the
// four 32x32 partial products (x_lo * y_lo, < 2^64, is dropped).  The
// middle column x_hi y_lo + x_lo y_hi is summed exactly as
// (x_hi y_lo + lo32(x_lo y_hi)) + hi32(x_lo y_hi) 2^32.
// 3 IMAD.WIDE.U32 + one 64-bit add.
__device__ __forceinline__ u64 mulhi_approx(u64 x, u64 y) {
  const uint32_t xl = lo32(x), xh = hi32(x);
  const u64 b = mulw(xl, hi32(y));
  const u64 c = madw(xh, lo32(y), lo32(b));  // <= (2^32-1)^2 + 2^32-1 < 2^64
  return madw(xh, hi32(y), hi32(b)) + hi32(c);
}

// x * y mod 2^64 + a as 32-bit pieces: 1 IMAD.WIDE.U32 + 2 IMAD
__device__ __forceinline__ u64 mullo_add(uint32_t xl, uint32_t xh, uint32_t yl, uint32_t yh,
                                         u64 a) {
  const u64 t = madw(xl, yl, a);
  uint32_t h = hi32(t);
  h = madlo(xl, yh, h);
  h = madlo(xh, yl, h);
  return pack(lo32(t), h);
}

// Shoup product x * w mod q in [0, 4q) for any x < 2^64 (w < q,
// wp = floor(w 2^64 / q)).  The quotient uses three of the four partial
// products of x * wp (the x_lo * wp_lo term and the low halves of the cross
// terms are dropped): it undershoots floor(x wp / 2^64) by at most 2, so the
// remainder lands in [0, 4q) instead of [0, 2q).  The remainder is formed as
// x*w + qh*(2^64 - q) mod 2^64 so every step is a multiply-accumulate:
// 5 IMAD.WIDE.U32 + 4 IMAD + one 64-bit add.  (Measured faster than the
// mulhi_approx chain below inside the butterflies: ptxas schedules the two
// independent cross products better.)
__device__ __forceinline__ u64 shoup4(u64 x, u64 w, u64 wp, const Mod &M) {
  const uint32_t xl = lo32(x), xh = hi32(x);
  const u64 b = mulw(xl, hi32(wp));
  const u64 c = mulw(xh, lo32(wp));
  const u64 qh = madw(xh, hi32(wp), static_cast<u64>(hi32(b)) + hi32(c));
  const uint32_t ql = lo32(qh), qhh = hi32(qh);
  const u64 a = madw(ql, M.nql, mulw(xl, lo32(w)));
  uint32_t h = hi32(a);
  h = madlo(xl, hi32(w), h);
  h = madlo(xh, lo32(w), h);
  h = madlo(ql, M.nqh, h);
  h = madlo(qhh, M.nql, h);
  return pack(lo32(a), h);
}

// Lazy Barrett data x data product for the paper's proposed-shape constants
// (mode NTTMUL_RED_ONE_SUB: proposed or dhem, modulus m <= 60 bits): a * b < 4 q^2
// (e.g. a, b < 2q).  T = a b exactly (4 IMAD.WIDE.U32 in a carry-free
// chain); c = T >> s_in (< 2^64); quot = hi64(c mu_sh) - e (mulhi_approx)
// undershoots floor(T / q) by at most 4 (Barrett's own <= 1 for canonical
// inputs, < 2 more from c < 2^(m+4), 1 from the approximate high word), so
// r = T - quot q lies in [0, 5q).  8 IMAD.WIDE.U32 + 2 IMAD in total.
__device__ __forceinline__ u64 mulred_lazy(u64 a, u64 b, const Limb &L, const Mod &M) {
  const uint32_t al = lo32(a), ah = hi32(a), bl = lo32(b), bh = hi32(b);
  const u64 p0 = mulw(al, bl);
  const u64 p1 = madw(al, bh, hi32(p0));
  const u64 p2 = madw(ah, bl, lo32(p1));
  const u64 tlo = pack(lo32(p0), lo32(p2));
  const u64 thi = madw(ah, bh, hi32(p1)) + hi32(p2);
  const u64 c = (tlo >> L.s_in) | ((thi << 1) << (63 - L.s_in));
  const u64 quot = mulhi_approx(c, L.mu_sh) >> L.s_hi;
  return mullo_add(lo32(quot), hi32(quot), M.nql, M.nqh, tlo);
}

// ---- butterflies ----------------------------------------------------------
//
// LB selects the lazy bound.  LB = 8 (every modulus < 2^61): forward values
// live in [0, 8q), inverse values in [0, 4q) and the [0, 4q) Shoup result
// needs no correction.  LB = 4 (moduli up to the reference's 62-bit limit,
// modarith.py:57-60): Harvey's classic [0, 4q) / [0, 2q) with one extra
// correction of the Shoup result.  Canonical [0, q) only at API edges, so
// outputs are bit-identical to the reference either way.

// Merged CT forward butterfly (reference _kernels.pyx:66-80).
// LB = 16 (moduli < 2^60) alternates reducing (RED) and non-reducing stages:
// a RED stage takes X < 16q to [0, 8q) and emits < 12q, the next stage
// skips the correction and emits < 16q - half the forward corrections.

template <int LB, bool RED = true>
__device__ __forceinline__ void ct_bfly(u64 &X, u64 &Y, u64 w, u64 wp, const Mod &M) {
  if (LB >= 16) {
    const u64 x = RED ? csub(X, M.q8) : X;
    const u64 t = shoup4(Y, w, wp, M);
    X = x + t;
    Y = x - t + M.q4;
  } else if (LB == 8) {
    const u64 x = csub(X, M.q4);
    const u64 t = shoup4(Y, w, wp, M);
    X = x + t;
    Y = x - t + M.q4;
  } else {
    const u64 x = csub(X, M.q2);
    const u64 t = csub(shoup4(Y, w, wp, M), M.q2);
    X = x + t;
    Y = x - t + M.q2;
  }
}

// Merged GS inverse butterfly (reference _kernels.pyx:102-118, unscaled).
template <int LB, bool RED = true>
__device__ __forceinline__ void gs_bfly(u64 &X, u64 &Y, u64 w, u64 wp, const Mod &M) {
  if (LB >= 8) {
    const u64 s = csub(X + Y, M.q4);
    const u64 d = X - Y + M.q4;
    X = s;
    Y = shoup4(d, w, wp, M);
  } else {
    const u64 s = csub(X + Y, M.q2);
    const u64 d = X - Y + M.q2;
    X = s;
    Y = csub(shoup4(d, w, wp, M), M.q2);
  }
}

// forward-range value -> [0, q)
template <int LB>
__device__ __forceinline__ u64 canon_fwd(u64 x, const Mod &M) {
  if (LB >= 16) x = csub(x, M.q8);
  if (LB >= 8) x = csub(x, M.q4);
  return csub(csub(x, M.q2), M.q);
}

// inverse-range value -> [0, q)
template <int LB>
__device__ __forceinline__ u64 canon_inv(u64 x, const Mod &M) {
  if (LB >= 8) x = csub(x, M.q2);
  return csub(x, M.q);
}

// exact canonical product by a fixed multiplier
__device__ __forceinline__ u64 shoup(u64 x, u64 w, u64 wp, const Mod &M) {
  return csub(csub(shoup4(x, w, wp, M), M.q2), M.q);
}

// Last GS stage (m = 1) with the scale folded in: canonical outputs.
// sc = {f, f', tw_inv[1] f, (tw_inv[1] f)'}.  Replaces the reference's
// per-stage halving (Zhang scaling, _kernels.pyx:115-117); the canonical
// results are identical.
template <int LB>
__device__ __forceinline__ void gs_bfly_last_scaled(u64 &X, u64 &Y, const u64 (&sc)[4],
                                                    const Mod &M) {
  const u64 s = X + Y;
  const u64 d = X - Y + (LB >= 8 ? M.q4 : M.q2);
  X = shoup(s, sc[0], sc[1], M);
  Y = shoup(d, sc[2], sc[3], M);
}

// Last GS stage without scaling: canonical outputs.
template <int LB>
__device__ __forceinline__ void gs_bfly_last_plain(u64 &X, u64 &Y, u64 w, u64 wp,
                                                   const Mod &M) {
  gs_bfly<LB>(X, Y, w, wp, M);
  X = canon_inv<LB>(X, M);
  Y = canon_inv<LB>(Y, M);
}

// Karatsuba-fused middle pair (paper Alg. 8 lines 3-14, reference
// _kernels.pyx:142-173): inputs canonical, outputs canonical.  The twiddle
// product z = v * tw[n/4 + i/2] uses the Shoup pair; the three data products
// use the Barrett variant MODE.
template <int MODE>
__device__ __forceinline__ void fused_pair(u64 a0, u64 a1, u64 b0, u64 b1,
                                           u64 w, u64 wp, bool odd,
                                           const Limb &L, const Mod &M, u64 &c0,
                                           u64 &c1) {
  const u64 q = L.q;
  const u64 u = mulred<MODE>(a0, b0, L);
  const u64 v = mulred<MODE>(a1, b1, L);
  const u64 s1 = csub(a0 + a1, q);
  const u64 s2 = csub(b0 + b1, q);
  const u64 ww = mulred<MODE>(s1, s2, L);
  const u64 y = csub(ww + q - u, q);
  c1 = csub(y + q - v, q);
  const u64 z = shoup(v, w, wp, M);
  c0 = odd ? csub(u + q - z, q) : csub(u + z, q);
}

// forward-range value (LB >= 16) -> [0, 2q): multiply-based for LB = 32,
// three conditional subtractions for LB = 16
template <int LB>
__device__ __forceinline__ u64 to2q_any(u64 x, const Mod &M) {
  return LB >= 32 ? reduce2q(x, M) : csub(csub(csub(x, M.q8), M.q4), M.q2);
}

// Lazy Karatsuba-fused middle pair for the LB = 16 path (all q < 2^60,
// proposed-shape Barrett constants): inputs in [0, 2q), outputs c0, c1 in
// [0, 4q) (the inverse lazy range, so the inverse stages take them as is).
// Same algebra as fused_pair / reference _kernels.pyx:142-173; canonical
// results after the inverse transform are identical.
template <bool FAST>
__device__ __forceinline__ void fused_pair_lazy(u64 a0, u64 a1, u64 b0, u64 b1, u64 w, u64 wp,
                                                bool odd, const Limb &L, const Mod &M,
                                                u64 &c0, u64 &c1) {
  const u64 u = mulred_lazy(a0, b0, L, M);     // [0, 5q)
  const u64 v = mulred_lazy(a1, b1, L, M);     // [0, 5q)
  const u64 s1 = csub(a0 + a1, M.q2);              // [0, 2q)
  const u64 s2 = csub(b0 + b1, M.q2);
  const u64 ww = mulred_lazy(s1, s2, L, M);    // [0, 5q)
  const u64 y = ww + M.q8 + M.q2 - u - v;          // (0, 15q)
  const u64 z = shoup4(v, w, wp, M);           // [0, 4q)
  const u64 x = odd ? u + M.q4 - z : u + z;        // [0, 9q)
  if (FAST) {  // -> [0, 2q)
    c1 = reduce2q(y, M);
    c0 = reduce2q(x, M);
  } else {  // -> [0, 4q)
    c1 = csub(csub(y, M.q8), M.q4);
    c0 = csub(csub(x, M.q8), M.q4);
  }
}

}  // namespace nttb
