// verify_kernels.cuh - the reference's verification kernels on sm_100a:
// the O(n^2) schoolbook oracle and the bulk Barrett-variant sweeps
// (reference _kernels.pyx:200-356), plus the index gather that maps the
// merged-CT spectrum onto the four-step "vendor" order (nttcore.py:489-497).
//
// Integer results are exact restatements: the schoolbook uses division
// (u128 % q) exactly like the reference; the sweeps replay the reference's
// truncating u128 arithmetic (_red_counted, _kernels.pyx:38-50) and its
// splitmix64 stream (_kernels.pyx:231-238), so tallies and first-mismatch
// reports are identical.
#pragma once
#include <cuda_runtime.h>

#include "modarith.cuh"

namespace nttb {

typedef unsigned __int128 u128;

// ---- schoolbook negacyclic product (reference _kernels.pyx:200-223) -------
// One thread per output coefficient k of one polynomial:
//   c_k = sum_{i<=k} a_i b_{k-i} - sum_{i>k} a_i b_{k-i+n}  (mod q).
// b is staged in shared memory in tiles; every product is reduced by
// division, the accumulator by one conditional subtraction per step, as in
// the reference (canonical result, so the order of additions is immaterial).
constexpr int NAIVE_THREADS = 256;
constexpr int NAIVE_TILE = 1024;

__global__ void __launch_bounds__(NAIVE_THREADS)
    naive_kernel(u64 *__restrict__ out, const u64 *__restrict__ a, const u64 *__restrict__ b,
                 u64 q, int n, int blocks_per_poly) {
  __shared__ u64 sa[NAIVE_TILE];
  const long long poly = blockIdx.x / blocks_per_poly;
  const int k = (blockIdx.x % blocks_per_poly) * NAIVE_THREADS + threadIdx.x;
  const u64 *pa = a + poly * n, *pb = b + poly * n;
  u64 acc = 0;
  for (int t0 = 0; t0 < n; t0 += NAIVE_TILE) {
    const int cnt = n - t0 < NAIVE_TILE ? n - t0 : NAIVE_TILE;
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += NAIVE_THREADS) sa[i] = pa[t0 + i];
    __syncthreads();
    if (k < n) {
      for (int ii = 0; ii < cnt; ++ii) {
        const int i = t0 + ii;
        const int j = k - i;
        const u64 p = static_cast<u64>((static_cast<u128>(sa[ii]) * pb[j >= 0 ? j : j + n]) % q);
        if (j >= 0) {
          acc += p;
          if (acc >= q) acc -= q;
        } else {
          acc = acc + q - p;
          if (acc >= q) acc -= q;
        }
      }
    }
  }
  if (k < n) out[poly * n + k] = acc;
}

// ---- Barrett variant sweeps (reference _kernels.pyx:226-356) --------------

__device__ __forceinline__ void variant_params(u64 q, int vi, u64 &mu, int &s_in, int &s_out) {
  const int m = 64 - __clzll(static_cast<long long>(q));
  if (vi == 0) {  // classical
    mu = static_cast<u64>((static_cast<u128>(1) << (2 * m)) / q);
    s_in = m - 1;
    s_out = m + 1;
  } else if (vi == 1) {  // dhem
    mu = static_cast<u64>((static_cast<u128>(1) << (2 * m + 3)) / q);
    s_in = m - 2;
    s_out = m + 5;
  } else {  // proposed
    mu = static_cast<u64>((static_cast<u128>(1) << (2 * m + 1)) / q);
    s_in = m - 2;
    s_out = m + 3;
  }
}

// the reference's truncating estimate + subtraction loop, with its count
__device__ __forceinline__ u64 red_counted(u128 x, u64 q, u64 mu, int s_in, int s_out,
                                           int &nsubs) {
  const u64 c = static_cast<u64>(x >> s_in);
  const u64 quot = static_cast<u64>((static_cast<u128>(c) * mu) >> s_out);
  u64 rem = static_cast<u64>(x - static_cast<u128>(quot) * q);
  int k = 0;
  while (rem >= q) {
    rem -= q;
    ++k;
  }
  nsubs = k;
  return rem;
}

// splitmix64 output for the stream state AFTER `draws` increments
__device__ __forceinline__ u64 splitmix_at(u64 seed, u64 draws) {
  u64 z = seed + draws * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// block-level reduction of the 12 tallies + mismatch count into global
// accumulators; first = min over a totally ordered mismatch key
struct SweepAcc {
  unsigned long long t[12];
  unsigned long long mism;
};

__device__ __forceinline__ void sweep_flush(SweepAcc &acc, unsigned long long *g_tallies,
                                            unsigned long long *g_res) {
#pragma unroll
  for (int i = 0; i < 13; ++i) {
    unsigned long long v = i < 12 ? acc.t[i] : acc.mism;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(i < 12 ? g_tallies + i : g_res, v);
  }
}

// g_res[0] = mismatches, g_res[1] = min key of a mismatch (init ~0)
__global__ void sweep_random_kernel(int bits, u64 nsamples, u64 seed,
                                    unsigned long long *g_tallies, unsigned long long *g_res) {
  SweepAcc acc = {};
  const u64 lo = 1ULL << (bits - 1), span = 1ULL << (bits - 1);
  const bool with_dhem = bits <= 60;
  unsigned long long first = ~0ULL;
  for (u64 s = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; s < nsamples;
       s += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u64 q = (lo + splitmix_at(seed, 3 * s + 1) % span) | 1;
    const u64 aa = splitmix_at(seed, 3 * s + 2) % q;
    const u64 bb = splitmix_at(seed, 3 * s + 3) % q;
    const u128 x = static_cast<u128>(aa) * bb;
    const u64 want = static_cast<u64>(x % q);
    for (int vi = 0; vi < 3; ++vi) {
      if (vi == 1 && !with_dhem) continue;
      u64 mu;
      int s_in, s_out, ns;
      variant_params(q, vi, mu, s_in, s_out);
      const u64 got = red_counted(x, q, mu, s_in, s_out, ns);
      acc.t[vi * 4 + (ns < 3 ? ns : 3)] += 1;
      if (got != want) {
        acc.mism += 1;
        const unsigned long long key = 3ULL * s + vi;
        if (key < first) first = key;
      }
    }
  }
  sweep_flush(acc, g_tallies, g_res);
  if (first != ~0ULL) atomicMin(g_res + 1, first);
}

// all odd q in [q_lo, q_hi] (q_hi < 2^16) x all x in [0, q^2): grid.y walks
// the moduli, the threads of grid.x the x range
__global__ void sweep_exhaustive_kernel(u64 q_lo, unsigned long long *g_tallies,
                                        unsigned long long *g_res) {
  const u64 qi = blockIdx.y;
  const u64 q = (q_lo | 1) + 2 * qi;
  u64 mu[3];
  int s_in[3], s_out[3];
  for (int vi = 0; vi < 3; ++vi) variant_params(q, vi, mu[vi], s_in[vi], s_out[vi]);
  SweepAcc acc = {};
  unsigned long long first = ~0ULL;
  const u64 xmax = q * q;
  for (u64 x = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; x < xmax;
       x += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u64 want = x % q;
    for (int vi = 0; vi < 3; ++vi) {
      int ns;
      const u64 got = red_counted(x, q, mu[vi], s_in[vi], s_out[vi], ns);
      acc.t[vi * 4 + (ns < 3 ? ns : 3)] += 1;
      if (got != want) {
        acc.mism += 1;
        const unsigned long long key = (qi << 34) | (x << 2) | static_cast<u64>(vi);
        if (key < first) first = key;
      }
    }
  }
  sweep_flush(acc, g_tallies, g_res);
  if (first != ~0ULL) atomicMin(g_res + 1, first);
}

// ---- index gather: out[b, v] = in[b, idx[v]] ------------------------------
__global__ void gather_kernel(u64 *__restrict__ out, const u64 *__restrict__ in,
                              const long long *__restrict__ idx, long long n, long long total) {
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long b = t / n, v = t - b * n;
    out[t] = in[b * n + idx[v]];
  }
}

}  // namespace nttb
