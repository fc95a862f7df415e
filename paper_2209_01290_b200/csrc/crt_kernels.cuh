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

// A block's coefficients are CRT_THREADS consecutive rows of W words: they
// move between HBM and shared memory with coalesced accesses, and each thread
// reads / writes its own row from shared memory with an odd word stride
// (conflict-free 8-byte accesses).
constexpr int CRT_THREADS = 128;
constexpr int CRT_ILP = 7;  // limbs per decompose pass (cfg3: 21 = 3 x 7)
__host__ __device__ constexpr int crt_stride(int W) { return W | 1; }

// ---- decompose: one thread per coefficient, all limbs ----------------------
// c mod q = (sum_w c_w R_w) mod q with R_w = 2^(64 w) mod q: the W products
// c_w R_w (< 2^124) are summed EXACTLY in a 128-bit accumulator with a carry
// word (PTX mad.lo.cc / madc.hi.cc, one 64x64 multiply-add per word, no
// reduction inside the loop), and the sum top 2^128 + hi 2^64 + lo is
// reduced once: shoup(lo, 1) + shoup(hi, 2^64 mod q) + top (2^128 mod q),
// canonicalised.  CRT_ILP limbs run side by side (independent carry
// chains).  The thread's words stay in its shared-memory row, the R table
// and the per-limb constants in shared memory (broadcast reads).
struct CrtLimbConsts {
  u64 q, f1;        // q, floor(2^64 / q)  (Shoup pair of the constant 1)
  u64 t1, t1p;      // 2^64 mod q and its Shoup companion
  u64 t2;           // 2^128 mod q
};

__device__ __forceinline__ void mac128(u64 &lo, u64 &hi, u64 &top, u64 a, u64 b) {
  asm("mad.lo.cc.u64 %0, %3, %4, %0;\n\t"
      "madc.hi.cc.u64 %1, %3, %4, %1;\n\t"
      "addc.u64 %2, %2, 0;"
      : "+l"(lo), "+l"(hi), "+l"(top)
      : "l"(a), "l"(b));
}

__global__ void __launch_bounds__(CRT_THREADS)
    crt_decompose_kernel(u64 *__restrict__ res, const u64 *__restrict__ words,
                         const u64 *__restrict__ qs, const ulonglong2 *__restrict__ pw,
                         int L, int W, long long n, long long total) {
  extern __shared__ u64 cw[];
  const int S = crt_stride(W);
  u64 *R = cw + CRT_THREADS * S;                                  // [L][W]
  CrtLimbConsts *K = reinterpret_cast<CrtLimbConsts *>(R + L * W);  // [L]
  for (int k = threadIdx.x; k < L * W; k += CRT_THREADS) R[k] = pw[k].x;
  // the constants are entries of the word table: pw[i][w] = {2^(64 w) mod q,
  // its Shoup companion}; hi (top) can be non-zero only when W >= 2 (3)
  for (int i = threadIdx.x; i < L; i += CRT_THREADS) {
    CrtLimbConsts c;
    c.q = qs[i];
    c.f1 = pw[i * W].y;
    c.t1 = W >= 2 ? pw[i * W + 1].x : 0;
    c.t1p = W >= 2 ? pw[i * W + 1].y : 0;
    c.t2 = W >= 3 ? pw[i * W + 2].x : 0;
    K[i] = c;
  }
  for (long long t0 = blockIdx.x * static_cast<long long>(CRT_THREADS); t0 < total;
       t0 += static_cast<long long>(gridDim.x) * CRT_THREADS) {
    const int rows = total - t0 < CRT_THREADS ? static_cast<int>(total - t0) : CRT_THREADS;
    __syncthreads();
    for (int k = threadIdx.x; k < rows * W; k += CRT_THREADS)
      cw[(k / W) * S + k % W] = words[t0 * W + k];
    __syncthreads();
    if (threadIdx.x >= rows) continue;
    const long long t = t0 + threadIdx.x;
    const long long b = t / n, j = t - b * n;
    const u64 *row = cw + threadIdx.x * S;
    for (int i0 = 0; i0 < L; i0 += CRT_ILP) {
      u64 lo[CRT_ILP], hi[CRT_ILP], top[CRT_ILP];
      int li[CRT_ILP];
#pragma unroll
      for (int u = 0; u < CRT_ILP; ++u) {
        li[u] = i0 + u < L ? i0 + u : i0;
        lo[u] = hi[u] = top[u] = 0;
      }
#pragma unroll 4
      for (int w = 0; w < W; ++w) {
        const u64 c = row[w];
#pragma unroll
        for (int u = 0; u < CRT_ILP; ++u) mac128(lo[u], hi[u], top[u], c, R[li[u] * W + w]);
      }
#pragma unroll
      for (int u = 0; u < CRT_ILP; ++u) {
        const CrtLimbConsts &c = K[li[u]];
        const Mod M = make_mod(c.q);
        // each part canonical first (q may have 62 bits); top <= 1: the sum
        // is below 2^128.4
        const u64 r0 = csub(csub(shoup4(lo[u], 1, c.f1, M), M.q2), M.q);
        const u64 r1 = csub(csub(shoup4(hi[u], c.t1, c.t1p, M), M.q2), M.q);
        u64 r = csub(r0 + r1, M.q);
        r = csub(r + (top[u] ? c.t2 : 0), M.q);
        if (i0 + u < L) res[(b * L + i0 + u) * n + j] = r;
      }
    }
  }
}

// ---- reconstruct: one thread per coefficient -------------------------------
// sum_i y_i M_i is formed column by column (word w from the low halves of
// y_i M_i[w] plus the high halves of column w-1 and the carry), straight
// into the thread's shared-memory row; then k Q is subtracted and one
// correction applied on that row.  y_i live in shared memory too.
__global__ void __launch_bounds__(CRT_THREADS)
    crt_reconstruct_kernel(u64 *__restrict__ words, const u64 *__restrict__ res,
                           const u64 *__restrict__ qs, const ulonglong2 *__restrict__ inv,
                           const u64 *__restrict__ mw, const u64 *__restrict__ bigq,
                           const double *__restrict__ qrecip, int L, int W, long long n,
                           long long total) {
  typedef unsigned __int128 u128;
  extern __shared__ u64 cw[];
  const int S = crt_stride(W);
  u64 *ys = cw + CRT_THREADS * S;  // [L][CRT_THREADS]
  for (long long t0 = blockIdx.x * static_cast<long long>(CRT_THREADS); t0 < total;
       t0 += static_cast<long long>(gridDim.x) * CRT_THREADS) {
    const int rows = total - t0 < CRT_THREADS ? static_cast<int>(total - t0) : CRT_THREADS;
    __syncthreads();  // the previous tile's rows have been stored
    if (threadIdx.x < rows) {
      const long long t = t0 + threadIdx.x;
      const long long b = t / n, j = t - b * n;
      double frac = 0.0;
      for (int i = 0; i < L; ++i) {
        const u64 q = qs[i];
        const Mod M = make_mod(q);
        const ulonglong2 iv = inv[i];
        const u64 y = shoup(res[(b * L + i) * n + j], iv.x, iv.y, M);  // canonical
        ys[i * CRT_THREADS + threadIdx.x] = y;
        frac += static_cast<double>(y) * qrecip[i];
      }
      const u64 k = static_cast<u64>(floor(frac));  // exact or off by one
      u64 *row = cw + threadIdx.x * S;
      // column sums: word w = lo(col), carry = hi(col); the top word (< L)
      // is kept in `top`
      u128 carry = 0, hsum = 0;
      for (int w = 0; w < W; ++w) {
        u128 col = carry + hsum;
        u128 hnext = 0;
        for (int i = 0; i < L; ++i) {
          const u128 p = static_cast<u128>(ys[i * CRT_THREADS + threadIdx.x]) * mw[i * W + w];
          col += static_cast<u64>(p);
          hnext += static_cast<u64>(p >> 64);
        }
        row[w] = static_cast<u64>(col);
        carry = col >> 64;
        hsum = hnext;
      }
      u64 top = static_cast<u64>(carry + hsum);
      // row -= k Q
      u64 borrow = 0, kc = 0;
      for (int w = 0; w < W; ++w) {
        const u128 kq = static_cast<u128>(k) * bigq[w] + kc;
        kc = static_cast<u64>(kq >> 64);
        const u64 sub = static_cast<u64>(kq), a = row[w];
        row[w] = a - sub - borrow;
        borrow = (a < sub) || (a - sub < borrow) ? 1 : 0;
      }
      top = top - kc - borrow;
      if (top == ~0ULL) {  // k was one too large: add Q back
        u64 c = 0;
        for (int w = 0; w < W; ++w) {
          const u128 s2 = static_cast<u128>(row[w]) + bigq[w] + c;
          row[w] = static_cast<u64>(s2);
          c = static_cast<u64>(s2 >> 64);
        }
      } else {  // k exact or one too small: subtract Q once if row >= Q
        bool ge = top != 0;
        if (!ge) {
          ge = true;  // equal counts as >=
          for (int w = W - 1; w >= 0; --w) {
            if (row[w] != bigq[w]) {
              ge = row[w] > bigq[w];
              break;
            }
          }
        }
        if (ge) {
          u64 br = 0;
          for (int w = 0; w < W; ++w) {
            const u64 a = row[w], s2 = bigq[w];
            row[w] = a - s2 - br;
            br = (a < s2) || (a - s2 < br) ? 1 : 0;
          }
        }
      }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < rows * W; k += CRT_THREADS)
      words[t0 * W + k] = cw[(k / W) * S + k % W];
  }
}

}  // namespace nttb
