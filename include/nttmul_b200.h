/*
 * nttmul_b200.h - C ABI of the B200 (sm_100a) negacyclic polymul hot path.
 *
 * This is the drop-in boundary for the reference package `nttmul`'s kernel
 * surface (what `nttmul.backend.kernels()` returns, reference
 * pkg/src/nttmul/backend.py:51-53, implemented by pkg/src/nttmul/_kernels.pyx).
 * Every entry point takes plain device pointers and sizes - no torch types -
 * and returns an int status (NTTMUL_OK == 0); nothing aborts.
 *
 * Conventions shared by all entry points
 *   - coefficient vectors are uint64 residues, C-contiguous, n = 2^log_n per
 *     polynomial; `batch` polynomials are laid out back to back ([batch, n]).
 *     Batched RNS entry points use [batch, num_limbs, n].
 *   - twiddle tables are passed in the PAIR layout produced by
 *     nttmul_twiddle_tables / nttmul_shoup_pairs: entry i is {w_i, w'_i} with
 *     w_i = the reference table value tw[i] (psi^{+-bit_reverse(i)},
 *     reference pkg/src/nttmul/params.py:157-167) and
 *     w'_i = floor(w_i * 2^64 / q) (its Shoup companion).  16-byte aligned.
 *   - (q, mode, mu, s_in, s_out) are the reduction parameters returned by the
 *     reference Modulus.reduction_params (pkg/src/nttmul/modarith.py:68-83);
 *     mode 0 = builtin (division), 1 = two-subtraction Barrett (classical),
 *     2 = one-subtraction Barrett (dhem / proposed, paper Alg. 3/4).
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *     asynchronous with respect to the host, like any kernel launch.
 *   - operation counts (reference `counts` argument) are closed-form and are
 *     filled by the host shim, not by these functions.
 */
#ifndef NTTMUL_B200_H
#define NTTMUL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define NTTMUL_OK 0
#define NTTMUL_EINVAL 1   /* bad sizes / log_n / reduction parameters      */
#define NTTMUL_EALIGN 2   /* pointer not 8-byte (data) / 16-byte (twiddle) */
#define NTTMUL_EPTR 3     /* pointer is not device-accessible memory       */
#define NTTMUL_ELAUNCH 4  /* kernel launch failed                          */
#define NTTMUL_ECUDA 5    /* other CUDA runtime error                      */

/* reduction modes (reference _kernels.pyx:20-22 RED_BUILTIN/TWO_SUB/ONE_SUB) */
#define NTTMUL_RED_BUILTIN 0
#define NTTMUL_RED_TWO_SUB 1
#define NTTMUL_RED_ONE_SUB 2

/* OR-ed into the `mode` of the batched RNS entry points when EVERY limb's
 * modulus is below 2^61: enables the [0, 8q) lazy-reduction bound (fewer
 * corrections).  Without it the [0, 4q) bound valid up to 62-bit moduli is
 * used; setting it with a 62-bit modulus gives wrong results. */
#define NTTMUL_MODE_NARROW 0x100
/* OR-ed in (with or without NTTMUL_MODE_NARROW) when EVERY modulus is below
 * 2^60: the forward transform then corrects only every other stage
 * ([0, 16q) range).  Setting it with a larger modulus gives wrong results. */
#define NTTMUL_MODE_NARROW60 0x200
/* OR-ed in (with NTTMUL_MODE_NARROW60) when EVERY modulus has at least 35
 * bits: the fused product's middle then uses multiply-based partial
 * reductions instead of conditional-subtraction chains. */
#define NTTMUL_MODE_WIDE35 0x400
/* Accepted and ignored (ABI 1 compatibility): the shift-shaped-modulus
 * schedule it selected measured slower and was removed. */
#define NTTMUL_MODE_PM 0x800

/* largest supported transform: n = 2^17 (BASELINE cfg4) */
#define NTTMUL_MAX_LOG_N 17

/*
 * Per-prime constant block.  One per RNS limb; the batched entry
 * points read a device array of these.  Filled by nttmul_limb_prepare from
 * the reference's reduction parameters; device code never divides.
 */
typedef struct nttmul_limb {
  uint64_t q;        /* odd modulus, bit length m <= 62                       */
  uint64_t mu_sh;    /* Barrett mu pre-shifted: quot = umulhi(c, mu_sh) >> s_hi */
  /* Scale folded into the last GS stage (m = 1).  The reference halves every
   * executed stage (_kernels.pyx:115-117): a full scaled inverse multiplies by
   * 2^-log_n, the skip_first one (log_n - 1 stages) by 2^-(log_n - 1).
   * sc_full = {f, Shoup(f), tw_inv[1]*f, Shoup(.)} with f = 2^-log_n;
   * sc_skip likewise with f = 2^-(log_n-1).                                  */
  uint64_t sc_full[4];
  uint64_t sc_skip[4];
  uint32_t s_in;     /* Barrett input shift (m-1 classical, m-2 dhem/proposed) */
  uint32_t s_hi;     /* extra right shift after umulhi (s_out - 64, or 0)     */
  uint32_t mode;     /* NTTMUL_RED_*                                          */
  uint32_t log_n;
} nttmul_limb_t;     /* 96 bytes */

/* ---- library information ------------------------------------------------ */

/* ABI version of this header (bumped on signature changes). */
int nttmul_abi_version(void);
/* Human-readable description of the last non-zero status on this thread. */
const char *nttmul_last_error(void);

/* ---- host-side constant preparation -------------------------------------- */

/*
 * Fill `out` for modulus q and the reference reduction parameters.
 * `w1_inv` is tw_inv[1] (= psi^-(n/2), the twiddle of the last GS stage); it
 * and the scale factor are folded into that stage (north star: "N^-1
 * scaling folded into the final INTT stage").  Host-only; no CUDA calls.
 * Replaces: Modulus.reduction_params + NttPlan.n_inv (modarith.py:68-83,
 * params.py:175).
 */
int nttmul_limb_prepare(nttmul_limb_t *out, uint64_t q, int mode, uint64_t mu,
                        int s_in, int s_out, int log_n, uint64_t w1_inv);

/* ---- twiddle tables (reference params.py:153-181 _plan_from_root) -------- */

/*
 * Generate on the device, for one prime:
 *   tw_fwd[i] = psi^bit_reverse(i), tw_inv[i] = psi^-bit_reverse(i)   (plain)
 *   fwd_pairs[i] = {tw_fwd[i], Shoup(tw_fwd[i])}, inv_pairs likewise.
 * Any of the four output pointers may be NULL.  i < 2^log_n.
 */
int nttmul_twiddle_tables(uint64_t *tw_fwd, uint64_t *tw_inv,
                          uint64_t *fwd_pairs, uint64_t *inv_pairs,
                          uint64_t q, uint64_t psi, uint64_t psi_inv,
                          int log_n, void *stream);

/* pairs[i] = {tw[i], floor(tw[i] * 2^64 / q)} for i < n (tw canonical). */
int nttmul_shoup_pairs(uint64_t *pairs, const uint64_t *tw, uint64_t q,
                       int64_t n, void *stream);

/*
 * Count i < n with tw_fwd[i]*tw_inv[i] mod q != 1, plus 1 if either table's
 * entry 0 is not 1 (reference validate_plan, params.py:203-207).  The count is
 * written to *bad_out (device pointer to one uint64).
 */
int nttmul_check_twiddles(const uint64_t *tw_fwd, const uint64_t *tw_inv,
                          uint64_t q, int64_t n, uint64_t *bad_out,
                          void *stream);

/* ---- the reference kernel surface (_kernels.pyx), batched over one prime -- */

/*
 * Merged CT forward NTT, in place, normal -> bit-reversed order.
 * truncate != 0 omits the final stage.  Replaces _kernels.pyx:52-85 ntt_ct.
 */
int nttmul_ntt_ct(uint64_t *a, const uint64_t *tw_pairs, uint64_t q, int mode,
                  uint64_t mu, int s_in, int s_out, int truncate, int log_n,
                  int64_t batch, void *stream);

/*
 * Merged GS inverse NTT, in place, bit-reversed -> normal order.  scaled != 0
 * yields the true inverse (the reference halves every output; here n^-1 is
 * folded into the last stage - identical canonical results).  skip_first
 * starts at m = n/4 (the fused-middle layout).  half_q is accepted for
 * signature parity and checked to equal (q+1)/2.  w1_inv must be
 * tw_inv[1] of the table (the twiddle the reference reads at m = 1, i = 0,
 * _kernels.pyx:100); it lets the scale fold into that stage's product.
 * Replaces _kernels.pyx:88-129 intt_gs.
 */
int nttmul_intt_gs(uint64_t *a, const uint64_t *tw_pairs, uint64_t q,
                   uint64_t half_q, int mode, uint64_t mu, int s_in, int s_out,
                   int scaled, int skip_first, int log_n, int64_t batch,
                   uint64_t w1_inv, void *stream);

/*
 * Karatsuba fused middle loop (paper Alg. 8 lines 3-14) on truncated
 * spectra; ch may alias neither ah nor bh.  Replaces _kernels.pyx:132-177.
 */
int nttmul_fused_middle(const uint64_t *ah, const uint64_t *bh, uint64_t *ch,
                        const uint64_t *tw_pairs, uint64_t q, int mode,
                        uint64_t mu, int s_in, int s_out, int log_n,
                        int64_t batch, void *stream);

/* out[i] = a[i]*b[i] mod q, i < n.  Replaces _kernels.pyx:180-188. */
int nttmul_hadamard(const uint64_t *a, const uint64_t *b, uint64_t *out,
                    int64_t n, uint64_t q, int mode, uint64_t mu, int s_in,
                    int s_out, void *stream);

/* a[i] = a[i]*factor mod q, in place.  Replaces _kernels.pyx:191-199. */
int nttmul_scale(uint64_t *a, uint64_t factor, int64_t n, uint64_t q,
                 int mode, uint64_t mu, int s_in, int s_out, void *stream);

/*
 * XOR over `passes` passes of (a[i]*b[i] mod q), written to *sink_out (device
 * pointer to one uint64).  Replaces _kernels.pyx:359-371 mulmod_loop.
 */
int nttmul_mulmod_loop(const uint64_t *a, const uint64_t *b, int64_t n,
                       uint64_t q, int mode, uint64_t mu, int s_in, int s_out,
                       uint64_t passes, uint64_t *sink_out, void *stream);

/* ---- fused polymul (reference polymul.py:147-172 polymul_fused) ---------- */

/*
 * c = a * b mod (x^n + 1, q_l) for every (ciphertext, limb) pair of a
 * [batch, num_limbs, n] layout.  limbs: device array [num_limbs];
 * fwd_pairs / inv_pairs: device [num_limbs, n] pair tables (only the first
 * n/2 entries of each are read - the halved FusedPlan footprint,
 * polymul.py:36-55).  mode: the reduction mode every limb was prepared
 * with (one variant per basis, reference RnsBasis.build variant argument),
 * optionally OR NTTMUL_MODE_NARROW.
 * workspace: device scratch of batch*num_limbs*n uint64, needed when
 * log_n > 12 (may alias b when b may be destroyed; never a or c).  c may
 * alias a.
 * Replaces the per-limb loop rns.py:116-119 around polymul_fused.
 */
int nttmul_polymul_fused_rns(uint64_t *c, const uint64_t *a, const uint64_t *b,
                             const nttmul_limb_t *limbs,
                             const uint64_t *fwd_pairs,
                             const uint64_t *inv_pairs, int log_n,
                             int num_limbs, int64_t batch, int mode,
                             uint64_t *workspace, void *stream);

/*
 * Same as nttmul_polymul_fused_rns, running only the selected launches:
 * bit 0 = forward column pass (a, b), bit 1 = fused row kernel, bit 2 =
 * inverse column pass.  phases = 7 is the full product.  For timing each
 * kernel of the pipeline separately with events between the calls.
 */
int nttmul_polymul_fused_rns_phases(uint64_t *c, const uint64_t *a,
                                    const uint64_t *b,
                                    const nttmul_limb_t *limbs,
                                    const uint64_t *fwd_pairs,
                                    const uint64_t *inv_pairs, int log_n,
                                    int num_limbs, int64_t batch, int mode,
                                    uint64_t *workspace, int phases,
                                    void *stream);

/*
 * Same product over HOST buffers (c_host, a_host, b_host: [batch, num_limbs,
 * 2^log_n] uint64, pinned for full overlap).  This is the call the reference's
 * own entry point corresponds to (polymul_rns over numpy arrays,
 * rns.py:111-120, with polymul_batch's ciphertext loop polymul.py:175-207):
 * host arrays in, host array out.  The batch is streamed in chunks of
 * `chunk_cts` ciphertexts through NTTMUL_HOST_NBUF device buffer sets in
 * `dev_buf` (>= NTTMUL_HOST_NBUF * 4 * chunk_cts * num_limbs * 2^log_n words,
 * 16-byte aligned); host->device copies, the fused kernels and device->host
 * copies of different chunks overlap on three streams.  Work is ordered after
 * everything already queued on `stream`, and `stream` completes when c_host
 * holds the full result.
 */
#define NTTMUL_HOST_NBUF 3
int nttmul_polymul_fused_rns_host(uint64_t *c_host, const uint64_t *a_host,
                                  const uint64_t *b_host,
                                  const nttmul_limb_t *limbs,
                                  const uint64_t *fwd_pairs,
                                  const uint64_t *inv_pairs, int log_n,
                                  int num_limbs, int64_t batch, int mode,
                                  uint64_t *dev_buf, int64_t chunk_cts,
                                  void *stream);

/*
 * Schedule of the transforms of n = 2^13 .. 2^17 (process-wide, per size; the
 * cluster schedule covers 2^13 .. 2^16):
 * which = 0 selects the fused product (nttmul_polymul_fused_rns*), 1 the
 * standalone ntt_ct / intt_gs.  NTTMUL_SCHED_THREE runs the column / row /
 * column launches through HBM; NTTMUL_SCHED_CLUSTER one launch of one
 * thread-block cluster per polynomial (the rows in distributed shared
 * memory, 24n HBM bytes per product); NTTMUL_SCHED_AUTO (default) picks the
 * measured-faster one.  All give identical results.
 */
/*
 * Radix split of the transforms of n = 2^13 .. 2^17 into N1 = n / 2^log_r
 * columns x 2^log_r-word rows (process-wide, per size; three-launch
 * schedule): log_r in 10 .. 13 with 1 <= log2(N1) <= 5, or 0 for the default
 * 2^12 (the cluster schedule always uses 2^12).  All splits give identical
 * results; they trade column stages (HBM round trips) against row stages
 * (the 2^13 rows run 1024-thread CTAs at one per SM).  BASELINE cfg5 sweep.
 */
int nttmul_set_split(int log_n, int log_r);

#define NTTMUL_SCHED_AUTO 0
#define NTTMUL_SCHED_THREE 1
#define NTTMUL_SCHED_CLUSTER 2
/* standalone transforms only: the column stages as strided passes of <= 3
 * stages (more, shorter CTAs) before rows of 1024 words - the latency
 * schedule of a single large transform */
#define NTTMUL_SCHED_PASSES 3
/* ONE launch of 2^A co-resident CTAs per polynomial (column stages, grid
 * barrier, row stages; the fused product: forward columns, barrier, rows
 * with the Karatsuba middle, barrier, inverse columns) - the latency
 * schedule of up to a few transforms / limb-products of 2^13 .. 2^17 words
 * (default for <= 4 per call); a forced launch larger than the co-resident
 * CTA count fails with NTTMUL_EINVAL */
#define NTTMUL_SCHED_GRID 4
int nttmul_set_schedule(int which, int log_n, int schedule);

/* ---- RNS decomposition / CRT reconstruction (rns.py:82-108) ------------- */

/*
 * Big-integer coefficients (little-endian uint64 words, words[b, j, 0..W))
 * -> residues res[b, i, j] = c mod q_i for b < batch, j < n, i < L.
 * word_pairs[i, w] = {2^(64 w) mod q_i, Shoup companion} (uint64[L, W, 2]).
 * Replaces decompose (rns.py:82-91).  W <= 64 words, q_i < 2^62.
 */
int nttmul_crt_decompose(uint64_t *res, const uint64_t *words,
                         const uint64_t *primes, const uint64_t *word_pairs,
                         int num_limbs, int num_words, int64_t batch,
                         int64_t n, void *stream);

/*
 * Residues res[b, i, j] (canonical) -> the unique words[b, j, 0..W) in
 * [0, Q), Q = prod q_i.  inv_pairs[i] = {(Q/q_i)^-1 mod q_i, companion},
 * m_words[i, w] = words of Q/q_i, q_words[w] = words of Q, q_recip[i] =
 * 1.0 / q_i.  Replaces reconstruct (rns.py:94-108).
 */
int nttmul_crt_reconstruct(uint64_t *words, const uint64_t *res,
                           const uint64_t *primes, const uint64_t *inv_pairs,
                           const uint64_t *m_words, const uint64_t *q_words,
                           const double *q_recip, int num_limbs, int num_words,
                           int64_t batch, int64_t n, void *stream);

/* ---- verification kernels ---------------------------------------------- */

/*
 * Schoolbook negacyclic product out = a * b mod (x^n + 1, q) of `batch`
 * independent [n] polynomials (device pointers), every product reduced by
 * division.  Replaces negacyclic_naive (_kernels.pyx:200-223), the O(n^2)
 * oracle.  out may not alias a or b; q >= 2 (operands need not be reduced).
 */
int nttmul_negacyclic_naive(uint64_t *out, const uint64_t *a, const uint64_t *b,
                            uint64_t q, int64_t n, int64_t batch, void *stream);

/*
 * Barrett-variant sweeps against division (sweep_random / sweep_exhaustive,
 * _kernels.pyx:226-356).  Device outputs: tallies uint64[3][4] (classical,
 * dhem, proposed x 0/1/2/3+ correctional subtractions; overwritten) and
 * result uint64[2] = {mismatches, first-mismatch key (~0 when none)}.
 * sweep_random: key = 3 * sample + variant; the sample's (q, a, b) are the
 * reference's splitmix64 draws 3*sample+1 .. 3*sample+3.  bits in [2, 63];
 * the dhem variant is skipped for bits > 60 like the reference.
 * sweep_exhaustive: all odd q in [q_lo, q_hi] (q_hi < 2^16), all x < q^2;
 * key = (q index << 34) | (x << 2) | variant.
 */
int nttmul_sweep_random(int bits, uint64_t nsamples, uint64_t seed,
                        uint64_t *tallies, uint64_t *result, void *stream);
int nttmul_sweep_exhaustive(uint64_t q_lo, uint64_t q_hi, uint64_t *tallies,
                            uint64_t *result, void *stream);

/*
 * out[b, v] = in[b, idx[v]] for b < batch, v < n (device pointers; idx is
 * int64[n] with entries in [0, n)).  Maps the merged-CT spectrum onto the
 * four-step transform's vendor order (ntt_2d / ntt_2d_permutation,
 * nttcore.py:405-497) and back.  out may not alias in.
 */
int nttmul_gather(uint64_t *out, const uint64_t *in, const int64_t *idx,
                  int64_t n, int64_t batch, void *stream);

/* ---- measurement --------------------------------------------------------- */

/*
 * Register-resident modmul throughput microbenchmark (the int-pipe roof):
 * every thread runs `iters` iterations of `chains` independent dependent
 * modmul chains.  kind 0 = Barrett data*data (mode from limb), 1 = Shoup
 * (fixed multiplicand), 2 = lazy forward CT butterfly, 3 = lazy inverse GS
 * butterfly (kinds 2/3 count one modmul per butterfly; need q < 2^61).
 * Writes an XOR sink to *sink_out so the
 * work cannot be elided.  Returns the number of modmuls issued in *modmuls_out (host).
 */
int nttmul_modmul_roof(const nttmul_limb_t *limb_host, int kind, int blocks,
                       int threads, int64_t iters, uint64_t *sink_out,
                       double *modmuls_out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* NTTMUL_B200_H */
