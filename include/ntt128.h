/*
 * ntt128.h -- C ABI of the B200-native 128-bit modular NTT and modular BLAS
 * library (libntt128.so), a from-scratch sm_100a implementation of the hot path
 * of arxiv 2509.12494 ("Towards Closing the Performance Gap for Cryptographic
 * Kernels Between CPUs and Specialized Hardware").
 *
 * Citations are PAPER.md / SPEC.md lines under the paper's text (§ / Eq. given).
 *
 * ---------------------------------------------------------------------------
 * Data layout (all entry points).  A residue x in Z_q (0 <= x < q < 2^128) is
 * 16 bytes: two little-endian uint64 limbs [lo, hi], x = hi * 2^64 + lo -- the
 * double-word [x0, x1] of Eq. def_dw stored low limb first,
 * i.e. the memory image of unsigned __int128.  A polynomial of length N is N
 * consecutive residues in natural coefficient order; a batch is B consecutive
 * polynomials, [B][N][2] uint64.  Device pointers must be 16-byte aligned.
 *
 * Ownership.  Every data pointer is caller-owned device memory; the library
 * never retains it after the call returns.  A plan owns its device tables
 * (allocated on `device` at create, freed by destroy).  Host pointers (q, root,
 * scalars) are read during the call only.
 *
 * Asynchrony.  Calls validate arguments synchronously, then enqueue kernels on
 * `stream` and return.  A kernel fault surfaces at the caller's next sync.
 * NTT128_ERR_CUDA is returned when a launch or allocation fails at enqueue.
 *
 * Preconditions.  Inputs are residues (< q): "a,b,c in Z_q".
 * They are not checked unless NTT128_FLAG_CHECK_INPUT is set on the plan (or
 * passed to a vec128 call); unreduced input gives unspecified output.
 *
 * Aliasing.  In place (out == in, z == x or z == y) is allowed everywhere except
 * where a function says otherwise (the four-step pass C and natural-layout calls
 * refuse it with NTT128_ERR_INVALID_ARG).  Partial overlap is undefined.
 *
 * Errors.  No exception crosses the ABI.  Every function returns a status;
 * on error nothing is enqueued and outputs are untouched.
 * ------------------------------------------------------------------------- */
#ifndef NTT128_H
#define NTT128_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *ntt128_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
    NTT128_OK = 0,
    NTT128_ERR_INVALID_ARG = 1,  /* null pointer, log2n out of [1, 26], batch == 0, n_moduli not 1 or batch, unknown flag bits */
    NTT128_ERR_MODULUS = 2,      /* q even or q < 3 */
    NTT128_ERR_NOT_PRIME = 3,    /* q fails the plan's Miller-Rabin test */
    NTT128_ERR_NO_ROOT = 4,      /* N does not divide q-1 (cyclic) / 2N does not divide q-1 (negacyclic) */
    NTT128_ERR_BAD_ROOT = 5,     /* root does not have exact order N (cyclic) / 2N (negacyclic), or root >= q */
    NTT128_ERR_ALIGNMENT = 6,    /* a device pointer is not 16-byte aligned */
    NTT128_ERR_INPUT_RANGE = 7,  /* only with NTT128_FLAG_CHECK_INPUT: some input coefficient >= q */
    NTT128_ERR_OOM = 8,          /* device allocation failed */
    NTT128_ERR_CUDA = 9,         /* a CUDA call failed at enqueue */
    NTT128_ERR_UNSUPPORTED = 10  /* valid request this build does not implement */
} ntt128_status;

/* plan flags */
#define NTT128_CYCLIC 0u            /* root = omega of exact order N; y_k = sum_j x_j omega^{jk} (Eq. ntt) */
#define NTT128_NEGACYCLIC 1u        /* root = psi of exact order 2N; y_k = sum_j x_j psi^{j(2k+1)}, the evaluation at psi^{2k+1} */
#define NTT128_FLAG_CHECK_INPUT 0x100u /* validate inputs < q on every call (synchronises the stream) */
/* Chained calls (DESIGN.md §6 "Chained calls"): consecutive transforms of this plan on one
 * stream overlap polynomial by polynomial -- the first pass of a call starts on polynomial p
 * once the previous call's last pass has finished p, instead of waiting for the previous
 * call's whole grid (the passes inside one call already overlap this way).  The library
 * applies it only when the previous library call on the stream was this plan's own transform
 * (forward, inverse, polymul, bitrev) and each buffer of the new call is either one of the
 * previous call's buffers (same base pointer) or disjoint from all of them; otherwise the
 * call waits for the whole previous grid.  Contract: between two such calls the caller
 * enqueues on that stream no kernel launched with programmatic stream serialization (PDL)
 * that touches their buffers, other than this library's own calls (plain kernels, copies
 * and memsets are ordered as usual).  Results are identical with or without the flag. */
#define NTT128_FLAG_CHAIN 0x200u

/* opaque; its tables are immutable after create; safe to share across streams and threads
 * (per-stream pass-overlap counters and scratch are cached inside, at most 8 streams: a
 * further stream evicts the least recently used entry once its last use has completed) */
typedef struct ntt128_plan_s *ntt128_plan_t;

/* Create a plan for `batch` transforms of length N = 2^log2n (1 <= log2n <= 26).
 *   q_host:    [n_moduli][2] uint64 {lo, hi}: odd primes 3 <= q < 2^128 (any width;
 *              deliberately beyond the paper's 124-bit Barrett limit, PAPER.md:208,
 *              because the BASELINE configs use 128-bit q -- DESIGN.md reading c1)
 *   root_host: [n_moduli][2]: omega (cyclic) or psi (negacyclic) per modulus; the
 *              root is a plan input (reading c8)
 *   n_moduli:  1 (all polynomials share q) or batch (polynomial b uses modulus b, the
 *              RNS case of BASELINE cfg 3)
 *   flags:     NTT128_CYCLIC or NTT128_NEGACYCLIC, optionally | NTT128_FLAG_CHECK_INPUT
 *              and / or | NTT128_FLAG_CHAIN
 *   device:    CUDA device ordinal that owns the plan tables
 * Validates primality (Miller-Rabin), divisibility and the root's exact order, then
 * builds per-modulus Montgomery constants and twiddle tables on the device
 * (untimed plan work; "twiddles are precomputed per stage"). */
ntt128_status ntt128_plan_create(ntt128_plan_t *out, uint32_t log2n, uint32_t batch, const uint64_t *q_host,
                                 const uint64_t *root_host, uint32_t n_moduli, uint32_t flags, int device);

/* Forward transform of the whole batch, natural order in and out (
 * DESIGN.md reading c6).  d_in/d_out: [batch][N][2] uint64 device arrays. */
ntt128_status ntt128_forward(const ntt128_plan_t plan, const uint64_t *d_in, uint64_t *d_out, ntt128_stream_t stream);

/* Inverse: x_j = N^{-1} sum_k y_k omega^{-jk} (cyclic, reading c7) or
 * x_j = N^{-1} psi^{-j} sum_k y_k omega^{-jk} (negacyclic).  inverse(forward(x)) == x. */
ntt128_status ntt128_inverse(const ntt128_plan_t plan, const uint64_t *d_in, uint64_t *d_out, ntt128_stream_t stream);

/* Polynomial product through the transform: d_c = a * b mod (X^N + 1) for negacyclic
 * plans, mod (X^N - 1) for cyclic plans (NTT, point-wise product,
 * inverse NTT).  d_a, d_b, d_c: [batch][N][2]; d_c may alias d_a or d_b.
 * Uses 2 x batch x N x 16 bytes of scratch per stream (an in-place multi-pass forward /
 * inverse: batch x N x 16), allocated by the plan on the first such call on that stream
 * and kept in the plan's per-stream cache. */
ntt128_status ntt128_polymul(const ntt128_plan_t plan, const uint64_t *d_a, const uint64_t *d_b, uint64_t *d_c,
                             ntt128_stream_t stream);

/* Negacyclic transforms with the spectrum in bit-reversed order (SURVEY.md §8(f) f1,
 * DESIGN.md §6): forward_bitrev writes Y[i] = y_{brev_n(i)} = a(psi^{2 brev_n(i) + 1}), the
 * natural-order negacyclic spectrum y (ntt128_forward) permuted by n-bit bit reversal;
 * inverse_bitrev(forward_bitrev(a)) == a.  Computed without any permutation or twist
 * multiply: Cooley-Tukey stages from the top index bit down with psi-merged twiddles
 * psi^{brev_n(2^(n-1-b) + i)}, Gentleman-Sande stages back (the negacyclic NTT of
 * PAPER.md:266-277 in the order point-wise products do not care about).  In place
 * (d_out == d_in) is allowed.  Negacyclic plans with log2n >= 10 only; otherwise
 * NTT128_ERR_UNSUPPORTED.  ntt128_polymul uses this path when it is available. */
ntt128_status ntt128_forward_bitrev(const ntt128_plan_t plan, const uint64_t *d_in, uint64_t *d_out,
                                    ntt128_stream_t stream);
ntt128_status ntt128_inverse_bitrev(const ntt128_plan_t plan, const uint64_t *d_in, uint64_t *d_out,
                                    ntt128_stream_t stream);

/* Plan properties (host-side queries). */
ntt128_status ntt128_plan_info(const ntt128_plan_t plan, uint32_t *log2n, uint32_t *batch, uint32_t *n_moduli,
                               uint32_t *flags, uint32_t *num_passes);

/* Arithmetic class of the plan's plain forward / inverse calls (host-side query):
 * *cls = NTT128_CLASS_MONTGOMERY (0): Montgomery products (36 word products per butterfly),
 * lazy per modulus size; NTT128_CLASS_PSEUDO_MERSENNE (1): every modulus is 2^b - c with
 * c 2^(128-b) < 2^32 (the largest NTT-friendly primes below a power of two)
 * and the plan is cyclic with >= 2 passes -- products fold 2^128 = c 2^(128-b) (mod q 2^(128-b)),
 * 21 word products per butterfly.  Results are the same canonical residues
 * either way ("bitwise-identical"); the class only changes the cost. */
#define NTT128_CLASS_MONTGOMERY 0u
#define NTT128_CLASS_PSEUDO_MERSENNE 1u
ntt128_status ntt128_plan_arith_class(const ntt128_plan_t plan, uint32_t *cls);

void ntt128_plan_destroy(ntt128_plan_t plan);

/* ---------------------------------------------------------------------------
 * Modular BLAS over one modulus q (§2.3; BLAS as "looping over
 * ... modular arithmetic").  n elements (any n >= 0; n == 0 is a
 * no-op returning OK; reading c14).  q: host {lo, hi}, odd, 3 <= q < 2^128
 * (primality not required).  flags: 0 or NTT128_FLAG_CHECK_INPUT.
 *   vec128_add : z = x + y mod q   (Eq. saddmod)
 *   vec128_sub : z = x - y mod q   (Eq. ssubmod)
 *   vec128_mul : z = x * y mod q   (point-wise product, "a special case of gemv")
 *   vec128_axpy: y = a * x + y mod q, in place on y; a: host scalar {lo, hi} < q
 * ------------------------------------------------------------------------- */
ntt128_status vec128_add(uint64_t *d_z, const uint64_t *d_x, const uint64_t *d_y, size_t n, const uint64_t *q,
                         uint32_t flags, ntt128_stream_t stream);
ntt128_status vec128_sub(uint64_t *d_z, const uint64_t *d_x, const uint64_t *d_y, size_t n, const uint64_t *q,
                         uint32_t flags, ntt128_stream_t stream);
ntt128_status vec128_mul(uint64_t *d_z, const uint64_t *d_x, const uint64_t *d_y, size_t n, const uint64_t *q,
                         uint32_t flags, ntt128_stream_t stream);
ntt128_status vec128_axpy(uint64_t *d_y, const uint64_t *a, const uint64_t *d_x, size_t n, const uint64_t *q,
                          uint32_t flags, ntt128_stream_t stream);

/* ---------------------------------------------------------------------------
 * Distributed four-step NTT of one huge polynomial (BASELINE cfg 5, N = 2^26; SURVEY.md
 * §8(a) row a13, §8(e)).  N = n1 n2, j = j1 + n1 j2, k = k2 + n2 k1, w = omega; since
 * jk = j1 k2 + n2 j1 k1 + n1 j2 k2 (mod N), Eq. ntt is exactly
 *   pass A:  z[j1][k2] = sum_{j2} x[j1 + n1 j2] w^{n1 j2 k2}               (n2-point NTTs)
 *   pass C:  y[k2 + n2 k1] = sum_{j1} (w^{j1 k2} z[j1][k2]) w^{n2 j1 k1}    (n1-point NTTs)
 * with the twiddle w^{j1 k2} applied by pass C as it loads z (one product per element).
 * G = world ranks (a power of two, G <= 8, dividing n1 and n2), one process per GPU; the
 * caller moves the blocks between ranks with an all-to-all of equal splits (NCCL over
 * NVLink), e.g. torch.distributed.all_to_all_single.  Layouts (R1 = n1/G, R2 = n2/G, rank g):
 *   "columns" X_g[R1][n2]: X_g[r][j2] = x[(g R1 + r) + n1 j2]       (forward input / inverse output)
 *   "rows"    Y_g[R2][n1]: Y_g[r][k1] = y[(g R2 + r) + n2 k1]       (forward output / inverse input)
 *   send [G][R1][R2] (forward): send[h][r][c] = z[g R1 + r][h R2 + c], block h goes to rank h;
 *   recv [G][R1][R2]: recv[g'][r][c] = z[g' R1 + r][g R2 + c] (block g' came from rank g').
 * Inverse: pass A = Z[k2][j1] = sum_{k1} y[k2 + n2 k1] w^{-n2 j1 k1} (rows), send / recv
 * [G][R2][R1] by the destination of j1; pass C = x[j1 + n1 j2] = sum_{k2} (N^{-1} w^{-j1 k2}
 * Z[k2][j1]) w^{-n1 j2 k2} (the whole N^{-1} rides on pass C's twiddle factor).  A four-step object holds one working buffer of
 * N/G residues: use it on one stream at a time.
 * ------------------------------------------------------------------------- */
typedef struct ntt128_fourstep_s *ntt128_fourstep_t;

/* log2n1, log2n2 >= 1, log2n1 + log2n2 <= 26; q, omega: host {lo, hi}, omega of exact order
 * N = 2^(log2n1 + log2n2); world G a power of two <= 8 with 2 G <= n1 and 2 G <= n2 when
 * G > 1 (exchange blocks at least 2 residues wide); 0 <= rank < world.
 * Builds the sub-plans and the rank's twiddle-factor tables ([R2][n1] forward, [R1][n2]
 * inverse: 2 N/G residues) on `device`. */
ntt128_status ntt128_fourstep_create(ntt128_fourstep_t *out, uint32_t log2n1, uint32_t log2n2, const uint64_t *q,
                                     const uint64_t *omega, uint32_t rank, uint32_t world, int device);
/* forward, before the exchange: X_g (columns) -> send [G][R1][R2] (pass A; its last pass
 * stores straight into the blocks) */
ntt128_status ntt128_fourstep_forward_a(const ntt128_fourstep_t fs, const uint64_t *d_cols, uint64_t *d_send,
                                        ntt128_stream_t stream);
/* forward, after the exchange: recv [G][R1][R2] -> Y_g (rows); d_recv != d_rows */
ntt128_status ntt128_fourstep_forward_c(const ntt128_fourstep_t fs, const uint64_t *d_recv, uint64_t *d_rows,
                                        ntt128_stream_t stream);
/* inverse, before the exchange: Y_g (rows) -> send [G][R2][R1] */
ntt128_status ntt128_fourstep_inverse_a(const ntt128_fourstep_t fs, const uint64_t *d_rows, uint64_t *d_send,
                                        ntt128_stream_t stream);
/* inverse, after the exchange: recv [G][R2][R1] -> X_g (columns); d_recv != d_cols */
ntt128_status ntt128_fourstep_inverse_c(const ntt128_fourstep_t fs, const uint64_t *d_recv, uint64_t *d_cols,
                                        ntt128_stream_t stream);
/* Fused exchange: pass A whose LAST transform pass stores each output
 * straight into its destination rank's receive buffer (peer memory over NVLink/NVSwitch)
 * at the offset the all-to-all would have used -- the layout ntt128_fourstep_*_c expects.
 * No send buffer and no collective.  peers: host array of `world` device pointers,
 * peers[h] = rank h's [G][R1][R2] (forward) / [G][R2][R1] (inverse) receive buffer mapped
 * into this process (e.g. torch symmetric memory; peers[rank] is the local one).  The
 * caller orders the writes: a barrier across ranks before the call (every peer is done
 * reading its receive buffer) and after it (every block has landed) before pass C.
 * Every pointer is validated before anything is enqueued. */
ntt128_status ntt128_fourstep_forward_a_peers(const ntt128_fourstep_t fs, const uint64_t *d_cols,
                                              const uint64_t *const *peers, ntt128_stream_t stream);
ntt128_status ntt128_fourstep_inverse_a_peers(const ntt128_fourstep_t fs, const uint64_t *d_rows,
                                              const uint64_t *const *peers, ntt128_stream_t stream);
/* Natural block layout ("rank g holds a contiguous N/G slice", a mode
 * costing one more exchange at each end).  Rank g holds x[g N/G + i] and, after the
 * forward, y[g N/G + i], i < N/G.  A direction is: pack -> exchange -> *_a_nat ->
 * exchange -> *_c_nat -> exchange -> unpack, every exchange an all-to-all of equal
 * blocks (block h -> rank h).  Same arithmetic as the transposed layouts above; pack and
 * unpack are data movement only (one HBM read + write of the slice each).
 *   forward_pack:   x slice [R2][G][R1] (j2 = g R2 + a, j1 = h R1 + r) -> send [G][R2][R1]
 *   forward_a_nat:  recv [G][R2][R1] (= [n2][R1], X_g[r][j2] = recv[j2 R1 + r]) -> send [G][R1][R2]
 *   forward_c_nat:  recv [G][R1][R2] (as forward_c) -> send [G][R2][R1], block h = k1 in [h R1, (h+1) R1)
 *   forward_unpack: recv [G][R2][R1] (= [n2][R1]) -> y slice [R1][n2] (k1 = g R1 + b)
 *   inverse_pack:   y slice [R1][G][R2] -> send [G][R1][R2]
 *   inverse_a_nat:  recv [G][R1][R2] (= [n1][R2], Y_g[r][k1] = recv[k1 R2 + r]) -> send [G][R2][R1]
 *   inverse_c_nat:  recv [G][R2][R1] (as inverse_c) -> send [G][R1][R2], block h = j2 in [h R2, (h+1) R2)
 *   inverse_unpack: recv [G][R1][R2] (= [n1][R2]) -> x slice [R2][n1]
 * Input and output must not alias (NTT128_ERR_INVALID_ARG); 16-byte aligned device
 * buffers of N/G residues each; the *_nat passes use the object's working buffer. */
ntt128_status ntt128_fourstep_forward_pack(const ntt128_fourstep_t fs, const uint64_t *d_nat, uint64_t *d_send,
                                           ntt128_stream_t stream);
ntt128_status ntt128_fourstep_forward_a_nat(const ntt128_fourstep_t fs, const uint64_t *d_recv, uint64_t *d_send,
                                            ntt128_stream_t stream);
ntt128_status ntt128_fourstep_forward_c_nat(const ntt128_fourstep_t fs, const uint64_t *d_recv, uint64_t *d_send,
                                            ntt128_stream_t stream);
ntt128_status ntt128_fourstep_forward_unpack(const ntt128_fourstep_t fs, const uint64_t *d_recv, uint64_t *d_nat,
                                             ntt128_stream_t stream);
ntt128_status ntt128_fourstep_inverse_pack(const ntt128_fourstep_t fs, const uint64_t *d_nat, uint64_t *d_send,
                                           ntt128_stream_t stream);
ntt128_status ntt128_fourstep_inverse_a_nat(const ntt128_fourstep_t fs, const uint64_t *d_recv, uint64_t *d_send,
                                            ntt128_stream_t stream);
ntt128_status ntt128_fourstep_inverse_c_nat(const ntt128_fourstep_t fs, const uint64_t *d_recv, uint64_t *d_send,
                                            ntt128_stream_t stream);
ntt128_status ntt128_fourstep_inverse_unpack(const ntt128_fourstep_t fs, const uint64_t *d_recv, uint64_t *d_nat,
                                             ntt128_stream_t stream);
void ntt128_fourstep_destroy(ntt128_fourstep_t fs);

/* ---------------------------------------------------------------------------
 * Wider moduli (the paper's generalisation to larger bit widths,
 * PAPER.md:807-808).  Residues of any odd prime q < 2^256 as four little-endian uint64
 * limbs (32 bytes); arrays [batch][N][4] uint64, 16-byte aligned.  Cyclic NTT of Eq. ntt,
 * natural order in and out, inverse with N^{-1}; same ownership / asynchrony / error
 * conventions as the 128-bit plans above.  log2n in [1, 24]; flags must be 0.
 *   q_host, root_host: [n_moduli][4] uint64 (root of exact order N); n_moduli 1 or batch.
 * Plan creation validates primality (Miller-Rabin, 20 bases), N | q - 1 and the root's
 * order on the host (milliseconds per modulus).  A plan whose moduli are all < 2^192 (and
 * vec256_mul with such a q) computes with 6-word arithmetic; the layout is unchanged
 * (the top limb of every residue is zero).
 * ------------------------------------------------------------------------- */
typedef struct ntt256_plan_s *ntt256_plan_t;
ntt128_status ntt256_plan_create(ntt256_plan_t *out, uint32_t log2n, uint32_t batch, const uint64_t *q_host,
                                 const uint64_t *root_host, uint32_t n_moduli, uint32_t flags, int device);
ntt128_status ntt256_forward(const ntt256_plan_t plan, const uint64_t *d_in, uint64_t *d_out, ntt128_stream_t stream);
ntt128_status ntt256_inverse(const ntt256_plan_t plan, const uint64_t *d_in, uint64_t *d_out, ntt128_stream_t stream);
void ntt256_plan_destroy(ntt256_plan_t plan);
/* z = x * y mod q element-wise over 256-bit residues (n elements; q: 4 host limbs) */
ntt128_status vec256_mul(uint64_t *d_z, const uint64_t *d_x, const uint64_t *d_y, size_t n, const uint64_t *q,
                         ntt128_stream_t stream);

/* Human-readable name of a status code (static storage). */
const char *ntt128_status_string(ntt128_status s);

/* Number of library kernels launched by this process so far (all entry points; a
 * host-side counter used by the bench to report gpu_launches). */
uint64_t ntt128_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* NTT128_H */
