// crt_kernels.cuh - RNS decomposition and CRT reconstruction on sm_100a
// (the steps either side of the polymul path: reference rns.py:82-108).
//
// Big integers are little-endian 64-bit words: a polynomial of n
// coefficients below Q = prod q_i is uint64[n, W], W = ceil(bits(Q) / 64);
// residues use the polymul layout [B, L, n].
//
// decompose:   c mod q_i = sum_w c_w (2^(64 w) mod q_i)  (mod q_i) - one Shoup
//              product per word against precomputed constants.
// reconstruct: c = sum_i y_i (Q / q_i) - k Q with y_i = r_i (Q/q_i)^-1 mod q_i
//              and k = floor(sum_i y_i / q_i) (the multiword sum is < L Q);
//              k comes from a double-precision sum and is corrected by one
//              conditional add / subtract of Q, so the result is exact.
// Both are exactly the reference's values (canonical residues; the unique
// representative in [0, Q)).
#pragma once
#include <cuda_runtime.h>

#include "modarith.cuh"

namespace nttb {

// ---- decompose: one thread per coefficient, all limbs ----------------------
template <int WMAX>
__global__ void __launch_bounds__(256)
    crt_decompose_kernel(u64 *__restrict__ res, const u64 *__restrict__ words,
                         const u64 *__restrict__ qs, const ulonglong2 *__restrict__ pw,
                         int L, int W, long long n, long long total) {
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long b = t / n, j = t - b * n;
    u64 c[WMAX];
#pragma unroll
    for (int w = 0; w < WMAX; ++w) c[w] = w < W ? words[t * W + w] : 0;
    for (int i = 0; i < L; ++i) {
      const u64 q = qs[i];
      const Mod M = make_mod(q);
      u64 acc = 0;
#pragma unroll
      for (int w = 0; w < WMAX; ++w) {
        if (w < W) {
          const ulonglong2 p = pw[i * W + w];
          const u64 r = csub(csub(shoup4(c[w], p.x, p.y, M), M.q2), q);  // [0, q)
          acc = csub(acc + r, q);
        }
      }
      res[(b * L + i) * n + j] = acc;
    }
  }
}

// ---- reconstruct: one thread per coefficient -------------------------------
template <int WMAX>
__global__ void __launch_bounds__(128)
    crt_reconstruct_kernel(u64 *__restrict__ words, const u64 *__restrict__ res,
                           const u64 *__restrict__ qs, const ulonglong2 *__restrict__ inv,
                           const u64 *__restrict__ mw, const u64 *__restrict__ bigq,
                           const double *__restrict__ qrecip, int L, int W, long long n,
                           long long total) {
  typedef unsigned __int128 u128;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long b = t / n, j = t - b * n;
    u64 acc[WMAX + 1];
#pragma unroll
    for (int w = 0; w <= WMAX; ++w) acc[w] = 0;
    double frac = 0.0;
    for (int i = 0; i < L; ++i) {
      const u64 q = qs[i];
      const Mod M = make_mod(q);
      const ulonglong2 iv = inv[i];
      const u64 y = shoup(res[(b * L + i) * n + j], iv.x, iv.y, M);  // canonical
      frac += static_cast<double>(y) * qrecip[i];
      u64 carry = 0;
#pragma unroll
      for (int w = 0; w < WMAX; ++w) {
        if (w < W) {
          const u128 s = static_cast<u128>(y) * mw[i * W + w] + acc[w] + carry;
          acc[w] = static_cast<u64>(s);
          carry = static_cast<u64>(s >> 64);
        }
      }
#pragma unroll
      for (int w = 0; w < WMAX; ++w)
        if (w == W) acc[w] += carry;  // top word (sum < L Q < 2^(64 W + 64))
      if (W == WMAX) acc[WMAX] += carry;
    }
    // acc -= k Q with k = floor(frac), then one correction either way
    const u64 k = static_cast<u64>(floor(frac));
    u64 borrow = 0, kc = 0;
#pragma unroll
    for (int w = 0; w <= WMAX; ++w) {
      if (w <= W) {
        const u128 kq = static_cast<u128>(k) * (w < W ? bigq[w] : 0) + kc;
        kc = static_cast<u64>(kq >> 64);
        const u64 sub = static_cast<u64>(kq);
        const u64 a = acc[w];
        const u64 d = a - sub - borrow;
        borrow = (a < sub) || (a - sub < borrow) ? 1 : 0;
        acc[w] = d;
      }
    }
    // top word (index W): ~0 after an over-subtraction (k one too large),
    // 1 or 0 otherwise (k exact or one too small)
    u64 top = 0;
#pragma unroll
    for (int w = 0; w <= WMAX; ++w)
      if (w == W) top = acc[w];
    if (top == ~0ULL) {  // negative: add Q back
      u64 c = 0;
#pragma unroll
      for (int w = 0; w < WMAX; ++w) {
        if (w < W) {
          const u128 s = static_cast<u128>(acc[w]) + bigq[w] + c;
          acc[w] = static_cast<u64>(s);
          c = static_cast<u64>(s >> 64);
        }
      }
    } else {  // subtract Q once more if acc >= Q
      int ge = top != 0 ? 2 : 1;  // compare from the top word down
#pragma unroll
      for (int w = WMAX - 1; w >= 0; --w) {
        if (w < W && ge == 1) {
          if (acc[w] > bigq[w]) ge = 2;
          else if (acc[w] < bigq[w]) ge = 0;
        }
      }
      if (ge) {
        u64 br = 0;
#pragma unroll
        for (int w = 0; w < WMAX; ++w) {
          if (w < W) {
            const u64 a = acc[w], s = bigq[w];
            acc[w] = a - s - br;
            br = (a < s) || (a - s < br) ? 1 : 0;
          }
        }
      }
    }
#pragma unroll
    for (int w = 0; w < WMAX; ++w)
      if (w < W) words[t * W + w] = acc[w];
  }
}

}  // namespace nttb
