/*
 * oracle128.c -- plain, slow, obviously-correct CPU oracle for the 128-bit
 * modular NTT and modular BLAS of arxiv 2509.12494.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code
 * with the CUDA path (paper_2509_12494_b200/csrc, include/): no headers, helpers
 * or tables in common.
 *
 * Arithmetic is on unsigned __int128 (the paper's "natively supported
 * double-word representation ... used for benchmarking", §3.1).
 * Every result is the canonical representative in [0, q); parity with the GPU is
 * bit-exact.
 *
 * Each function cites the passage it follows.  Readings of the paper that are
 * not literal are listed in DESIGN.md §3 ("readings").
 *
 * Array layout: element i of a residue vector is two uint64 [lo, hi] at
 * p[2i], p[2i+1] (the memory image of unsigned __int128, little endian).
 *
 * Pins (see tests/test_oracle_*.py): Python big-int arithmetic, Fermat's little
 * theorem, sympy primality, SPEC/PAPER worked examples under tests/golden/,
 * O(N^2) brute force DFTs in pure Python, closed forms.  No function here is
 * "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

static inline u128 ld(const uint64_t *p) { return ((u128)p[1] << 64) | p[0]; }
static inline void st(uint64_t *p, u128 v) { p[0] = (uint64_t)v; p[1] = (uint64_t)(v >> 64); }

/* ---------------------------------------------------------------------------
 * Double-word product, Eq. muls (§2.2), omega0 = 64:
 *   c = (a0 b0) 2^128 + (a0 b1 + a1 b0) 2^64 + a1 b1
 * with a = [a0, a1] = a0 2^64 + a1.  Returned as the 256-bit pair (hi, lo).
 * ------------------------------------------------------------------------- */
static void mul_full(u128 a, u128 b, u128 *hi, u128 *lo) {
    uint64_t a0 = (uint64_t)(a >> 64), a1 = (uint64_t)a;
    uint64_t b0 = (uint64_t)(b >> 64), b1 = (uint64_t)b;
    u128 p00 = (u128)a0 * b0;          /* weight 2^128 */
    u128 p01 = (u128)a0 * b1;          /* weight 2^64  */
    u128 p10 = (u128)a1 * b0;          /* weight 2^64  */
    u128 p11 = (u128)a1 * b1;          /* weight 1     */
    /* middle = p01 + p10 may need 129 bits */
    u128 mid = p01 + p10;
    u128 mid_carry = (mid < p01) ? 1 : 0;            /* bit 128 of the middle sum */
    u128 l = p11 + (mid << 64);
    u128 c = (l < p11) ? 1 : 0;                      /* carry out of the low half */
    u128 h = p00 + (mid >> 64) + (mid_carry << 64) + c;
    *hi = h;
    *lo = l;
}

/* ---------------------------------------------------------------------------
 * Remainder of a 256-bit value by q: restoring binary long division, the literal
 * definition x mod q.  r is kept as 129 bits
 * (u128 plus a carry flag) so that any q < 2^128 works.
 * ------------------------------------------------------------------------- */
static u128 rem_u256(u128 hi, u128 lo, u128 q) {
    u128 r = 0;
    int start = 255;
    if (hi < q) { r = hi; start = 127; }   /* the first 128 steps would just rebuild hi */
    for (int i = start; i >= 0; i--) {
        unsigned bit = (unsigned)((i >= 128 ? (hi >> (i - 128)) : (lo >> i)) & 1);
        unsigned top = (unsigned)(r >> 127);          /* bit shifted out of 128 */
        r = (r << 1) | bit;
        if (top || r >= q) r -= q;                   /* wraps correctly when top = 1 */
    }
    return r;
}

/* Eq. saddmod: c = a + b - q if a + b >= q else a + b.
 * The sum is formed with an explicit 129th bit (carry) so q up to 2^128-1 works
 * (reading c3 in DESIGN.md: Table 1 / Listing 1 carry logic is not transcribed). */
static u128 addmod(u128 a, u128 b, u128 q) {
    u128 s = a + b;
    int carry = s < a;
    if (carry || s >= q) s -= q;
    return s;
}

/* Eq. ssubmod: c = a - b + q if a < b else a - b. */
static u128 submod(u128 a, u128 b, u128 q) {
    return (a >= b) ? a - b : a - b + q;
}

/* Eq. 1 third line: c = a b mod q, as the exact remainder of
 * the double-word product (Eq. muls).  Barrett (Eq. barrett) computes the same
 * unique value faster; the oracle uses the definition. */
static u128 mulmod(u128 a, u128 b, u128 q) {
    u128 hi, lo;
    mul_full(a, b, &hi, &lo);
    return rem_u256(hi, lo, q);
}

static u128 powmod(u128 a, u128 e, u128 q) {
    u128 r = 1 % q, b = a % q;
    while (e) {
        if (e & 1) r = mulmod(r, b, q);
        b = mulmod(b, b, q);
        e >>= 1;
    }
    return r;
}

/* inverse of a in Z_q for prime q: a^(q-2) (Fermat) */
static u128 invmod(u128 a, u128 q) { return powmod(a, q - 2, q); }

/* Miller-Rabin with the first 40 prime bases (probable prime; pinned against
 * sympy's BPSW in tests/test_oracle_primes.py). */
static int is_prime(u128 n) {
    static const unsigned bases[40] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59, 61, 67, 71,
                                       73, 79, 83, 89, 97, 101, 103, 107, 109, 113, 127, 131, 137, 139, 149, 151, 157, 163, 167, 173};
    if (n < 2) return 0;
    for (int i = 0; i < 40; i++) {
        if (n == bases[i]) return 1;
        if (n % bases[i] == 0) return 0;
    }
    u128 d = n - 1;
    int s = 0;
    while ((d & 1) == 0) { d >>= 1; s++; }
    for (int i = 0; i < 40; i++) {
        u128 x = powmod(bases[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int comp = 1;
        for (int r = 1; r < s; r++) {
            x = mulmod(x, x, n);
            if (x == n - 1) { comp = 0; break; }
        }
        if (comp) return 0;
    }
    return 1;
}

/* ===========================================================================
 * Exported scalar entry points (pointer args: [lo, hi] pairs)
 * ======================================================================== */
void o_mul_full(const uint64_t *a, const uint64_t *b, uint64_t *out4) {
    u128 hi, lo;
    mul_full(ld(a), ld(b), &hi, &lo);
    st(out4, lo);
    st(out4 + 2, hi);
}
void o_rem_u256(const uint64_t *x4, const uint64_t *q, uint64_t *r) { st(r, rem_u256(ld(x4 + 2), ld(x4), ld(q))); }
void o_addmod(const uint64_t *a, const uint64_t *b, const uint64_t *q, uint64_t *r) { st(r, addmod(ld(a), ld(b), ld(q))); }
void o_submod(const uint64_t *a, const uint64_t *b, const uint64_t *q, uint64_t *r) { st(r, submod(ld(a), ld(b), ld(q))); }
void o_mulmod(const uint64_t *a, const uint64_t *b, const uint64_t *q, uint64_t *r) { st(r, mulmod(ld(a), ld(b), ld(q))); }
void o_powmod(const uint64_t *a, const uint64_t *e, const uint64_t *q, uint64_t *r) { st(r, powmod(ld(a), ld(e), ld(q))); }
void o_invmod(const uint64_t *a, const uint64_t *q, uint64_t *r) { st(r, invmod(ld(a), ld(q))); }
int o_is_prime(const uint64_t *n) { return is_prime(ld(n)); }

/* Largest prime p < 2^bits with p = 1 mod m, skipping the first `skip` such
 * primes (descending scan over p = k m + 1; SURVEY.md §8(c) readings c10, c11).
 * Returns 0 on success. */
int o_find_prime(int bits, const uint64_t *m_, int skip, uint64_t *out) {
    u128 m = ld(m_);
    u128 top = (bits == 128) ? ~(u128)0 : (((u128)1 << bits) - 1); /* largest value < 2^bits */
    u128 k = (top - 1) / m;                                         /* k m + 1 <= top */
    u128 lower = (bits <= 1) ? 0 : ((u128)1 << (bits - 1));
    for (; k > 0; k--) {
        u128 p = k * m + 1;
        if (p < lower) return 1;
        if (is_prime(p)) {
            if (skip == 0) { st(out, p); return 0; }
            skip--;
        }
    }
    return 1;
}

/* ===========================================================================
 * Modular BLAS (§2.3; "looping over scalar ...
 * modular arithmetic").  Per element: Eq. saddmod / ssubmod / Eq. 1 product;
 * axpy y = a x + y, in place on y (reading c13).
 * ======================================================================== */
void o_vadd(uint64_t *z, const uint64_t *x, const uint64_t *y, int64_t n, const uint64_t *q_) {
    u128 q = ld(q_);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) st(z + 2 * i, addmod(ld(x + 2 * i), ld(y + 2 * i), q));
}
void o_vsub(uint64_t *z, const uint64_t *x, const uint64_t *y, int64_t n, const uint64_t *q_) {
    u128 q = ld(q_);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) st(z + 2 * i, submod(ld(x + 2 * i), ld(y + 2 * i), q));
}
void o_vmul(uint64_t *z, const uint64_t *x, const uint64_t *y, int64_t n, const uint64_t *q_) {
    u128 q = ld(q_);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) st(z + 2 * i, mulmod(ld(x + 2 * i), ld(y + 2 * i), q));
}
void o_axpy(uint64_t *y, const uint64_t *a_, const uint64_t *x, int64_t n, const uint64_t *q_) {
    u128 q = ld(q_), a = ld(a_);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) st(y + 2 * i, addmod(mulmod(a, ld(x + 2 * i), q), ld(y + 2 * i), q));
}

/* ===========================================================================
 * NTT, Eq. ntt (§2.3): y_k = sum_{j<n} x_j w^{jk} mod q.
 * ======================================================================== */

/* O(n^2) definition, running power w^k then (w^k)^j. */
static void dft_one(uint64_t *y, const uint64_t *x, int64_t n, u128 w, u128 q) {
    u128 wk = 1 % q;
    for (int64_t k = 0; k < n; k++) {
        u128 acc = 0, p = 1 % q;
        for (int64_t j = 0; j < n; j++) {
            acc = addmod(acc, mulmod(ld(x + 2 * j), p, q), q);
            p = mulmod(p, wk, q);
        }
        st(y + 2 * k, acc);
        wk = mulmod(wk, w, q);
    }
}

/* Textbook iterative radix-2 Cooley-Tukey (bit-reverse copy, then log n stages
 * of n/2 butterflies, each "one modular addition, one modular subtraction, and
 * one modular multiplication", §3.2).  Natural order in and out. */
static void ntt_one(uint64_t *y, const uint64_t *x, int64_t n, u128 w, u128 q) {
    int logn = 0;
    while (((int64_t)1 << logn) < n) logn++;
    u128 *a = (u128 *)malloc(sizeof(u128) * (size_t)n);
    for (int64_t i = 0; i < n; i++) {
        int64_t r = 0;
        for (int b = 0; b < logn; b++) r |= ((i >> b) & 1) << (logn - 1 - b);
        a[r] = ld(x + 2 * i);
    }
    for (int64_t len = 2; len <= n; len <<= 1) {
        u128 wl = powmod(w, (u128)(n / len), q);          /* primitive len-th root */
        for (int64_t s = 0; s < n; s += len) {
            u128 t = 1 % q;
            for (int64_t j = 0; j < len / 2; j++) {
                u128 u = a[s + j];
                u128 v = mulmod(a[s + j + len / 2], t, q);
                a[s + j] = addmod(u, v, q);
                a[s + j + len / 2] = submod(u, v, q);
                t = mulmod(t, wl, q);
            }
        }
    }
    for (int64_t i = 0; i < n; i++) st(y + 2 * i, a[i]);
    free(a);
}

/* Batched forward transforms: polynomial b uses modulus qs[b % nq], root ws[b % nq].
 * kind 0 = O(n^2) definition, 1 = radix-2 (threads over polynomials only). */
void o_ntt_batch(uint64_t *y, const uint64_t *x, int64_t batch, int64_t n, const uint64_t *ws,
                 const uint64_t *qs, int64_t nq, int kind) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < batch; b++) {
        int64_t m = b % nq;
        if (kind == 0) dft_one(y + 2 * n * b, x + 2 * n * b, n, ld(ws + 2 * m), ld(qs + 2 * m));
        else ntt_one(y + 2 * n * b, x + 2 * n * b, n, ld(ws + 2 * m), ld(qs + 2 * m));
    }
}

/* Inverse (reading c7): x = n^{-1} * DFT_{w^{-1}}(y). */
void o_intt_batch(uint64_t *x, const uint64_t *y, int64_t batch, int64_t n, const uint64_t *ws,
                  const uint64_t *qs, int64_t nq, int kind) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < batch; b++) {
        int64_t m = b % nq;
        u128 q = ld(qs + 2 * m), w = ld(ws + 2 * m);
        u128 winv = invmod(w, q), ninv = invmod((u128)n % q, q);
        uint64_t *o = x + 2 * n * b;
        if (kind == 0) dft_one(o, y + 2 * n * b, n, winv, q);
        else ntt_one(o, y + 2 * n * b, n, winv, q);
        for (int64_t i = 0; i < n; i++) st(o + 2 * i, mulmod(ld(o + 2 * i), ninv, q));
    }
}

/* One transform, large n: radix-2 with each stage's butterflies split over
 * threads (same algorithm as ntt_one; the twiddle of butterfly j in a block of
 * length len is wl^j, computed by powmod so that blocks are independent). */
void o_ntt_large(uint64_t *y, const uint64_t *x, int64_t n, const uint64_t *w_, const uint64_t *q_, int inverse) {
    u128 q = ld(q_), w = ld(w_);
    if (inverse) w = invmod(w, q);
    int logn = 0;
    while (((int64_t)1 << logn) < n) logn++;
    u128 *a = (u128 *)malloc(sizeof(u128) * (size_t)n);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        int64_t r = 0;
        for (int b = 0; b < logn; b++) r |= ((i >> b) & 1) << (logn - 1 - b);
        a[r] = ld(x + 2 * i);
    }
    for (int64_t len = 2; len <= n; len <<= 1) {
        u128 wl = powmod(w, (u128)(n / len), q);
        int64_t half = len / 2;
        /* butterfly index t in [0, n/2): block s = t / half, offset j = t % half */
#pragma omp parallel
        {
            int64_t prev_j = -1;
            u128 tw = 0;
#pragma omp for schedule(static)
            for (int64_t t = 0; t < n / 2; t++) {
                int64_t s = (t / half) * len, j = t % half;
                if (prev_j >= 0 && j == prev_j + 1) tw = mulmod(tw, wl, q);
                else tw = powmod(wl, (u128)j, q);
                prev_j = j;
                u128 u = a[s + j];
                u128 v = mulmod(a[s + j + half], tw, q);
                a[s + j] = addmod(u, v, q);
                a[s + j + half] = submod(u, v, q);
            }
        }
    }
    u128 ninv = inverse ? invmod((u128)n % q, q) : 1;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) st(y + 2 * i, inverse ? mulmod(a[i], ninv, q) : a[i]);
    free(a);
}

/* Single output y_k of Eq. ntt by direct O(n) evaluation, sum_j x_j (w^k)^j,
 * split over threads with per-chunk starting power (w^k)^start.  Independent of
 * the radix-2 structure; used to sample outputs at huge n. */
void o_ntt_eval(const uint64_t *x, int64_t n, const uint64_t *w_, const uint64_t *q_, int64_t k, uint64_t *out) {
    u128 q = ld(q_), w = ld(w_);
    u128 wk = powmod(w, (u128)k, q);
    u128 total = 0;
#pragma omp parallel
    {
        u128 acc = 0;
#pragma omp for schedule(static)
        for (int64_t c = 0; c < 256; c++) {
            int64_t lo = n * c / 256, hi = n * (c + 1) / 256;
            u128 p = powmod(wk, (u128)lo, q);
            for (int64_t j = lo; j < hi; j++) {
                acc = addmod(acc, mulmod(ld(x + 2 * j), p, q), q);
                p = mulmod(p, wk, q);
            }
        }
#pragma omp critical
        total = addmod(total, acc, q);
    }
    st(out, total);
}

/* ===========================================================================
 * Polynomial products (PAPER.md:266-271 schoolbook product; cyclic and
 * negacyclic reductions, SPEC.md:517-534 and reading c9 in DESIGN.md).
 * ======================================================================== */

/* full schoolbook product, 2n-1 coefficients: c_j = sum_i a_i b_{j-i} mod q */
void o_poly_mul_schoolbook(uint64_t *c, const uint64_t *a, const uint64_t *b, int64_t n, const uint64_t *q_) {
    u128 q = ld(q_);
    for (int64_t j = 0; j < 2 * n - 1; j++) {
        u128 acc = 0;
        for (int64_t i = 0; i < n; i++) {
            int64_t k = j - i;
            if (k < 0 || k >= n) continue;
            acc = addmod(acc, mulmod(ld(a + 2 * i), ld(b + 2 * k), q), q);
        }
        st(c + 2 * j, acc);
    }
}

/* c = a b mod (X^n - 1) (sign = +1) or mod (X^n + 1) (sign = -1), O(n^2):
 * the coefficient of X^{i+j} goes to index (i+j) mod n, negated when i+j >= n
 * for the negacyclic ring. */
void o_conv(uint64_t *c, const uint64_t *a, const uint64_t *b, int64_t n, const uint64_t *q_, int negacyclic) {
    u128 q = ld(q_);
    u128 *acc = (u128 *)calloc((size_t)n, sizeof(u128));
    for (int64_t i = 0; i < n; i++) {
        u128 ai = ld(a + 2 * i);
        for (int64_t j = 0; j < n; j++) {
            u128 p = mulmod(ai, ld(b + 2 * j), q);
            int64_t k = i + j;
            if (k >= n) {
                k -= n;
                acc[k] = negacyclic ? submod(acc[k], p, q) : addmod(acc[k], p, q);
            } else {
                acc[k] = addmod(acc[k], p, q);
            }
        }
    }
    for (int64_t k = 0; k < n; k++) st(c + 2 * k, acc[k]);
    free(acc);
}

/* Negacyclic transform by definition (reading c9): y_k = sum_j x_j psi^{j(2k+1)},
 * i.e. the evaluation of x(X) at psi^{2k+1}, psi of order 2n.  O(n^2). */
void o_negacyclic_dft(uint64_t *y, const uint64_t *x, int64_t n, const uint64_t *psi_, const uint64_t *q_) {
    u128 q = ld(q_), psi = ld(psi_);
    u128 psi2 = mulmod(psi, psi, q);
    u128 z = psi;                                       /* psi^{2k+1} for k = 0 */
    for (int64_t k = 0; k < n; k++) {
        u128 acc = 0, p = 1 % q;
        for (int64_t j = 0; j < n; j++) {
            acc = addmod(acc, mulmod(ld(x + 2 * j), p, q), q);
            p = mulmod(p, z, q);
        }
        st(y + 2 * k, acc);
        z = mulmod(z, psi2, q);
    }
}

/* Negacyclic forward/inverse via twist + cyclic NTT (reading c9):
 *   forward: y = NTT_w(x_j psi^j),  w = psi^2
 *   inverse: x_j = psi^{-j} * INTT_w(y)_j
 * batched, polynomial b uses qs/psis[b % nq]; threads over polynomials. */
void o_negacyclic_batch(uint64_t *out, const uint64_t *in, int64_t batch, int64_t n, const uint64_t *psis,
                        const uint64_t *qs, int64_t nq, int inverse) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < batch; b++) {
        int64_t m = b % nq;
        u128 q = ld(qs + 2 * m), psi = ld(psis + 2 * m);
        u128 w = mulmod(psi, psi, q);
        const uint64_t *src = in + 2 * n * b;
        uint64_t *dst = out + 2 * n * b;
        uint64_t *tmp = (uint64_t *)malloc(sizeof(uint64_t) * 2 * (size_t)n);
        if (!inverse) {
            u128 p = 1 % q;
            for (int64_t j = 0; j < n; j++) { st(tmp + 2 * j, mulmod(ld(src + 2 * j), p, q)); p = mulmod(p, psi, q); }
            ntt_one(dst, tmp, n, w, q);
        } else {
            u128 winv = invmod(w, q), ninv = invmod((u128)n % q, q), psiinv = invmod(psi, q);
            ntt_one(tmp, src, n, winv, q);
            u128 p = ninv;
            for (int64_t j = 0; j < n; j++) { st(dst + 2 * j, mulmod(ld(tmp + 2 * j), p, q)); p = mulmod(p, psiinv, q); }
        }
        free(tmp);
    }
}

/* Negacyclic product via transforms: c = INTT(NTT(a) . NTT(b)), batched. */
void o_negacyclic_polymul_batch(uint64_t *c, const uint64_t *a, const uint64_t *b, int64_t batch, int64_t n,
                                const uint64_t *psis, const uint64_t *qs, int64_t nq) {
    size_t sz = sizeof(uint64_t) * 2 * (size_t)n * (size_t)batch;
    uint64_t *fa = (uint64_t *)malloc(sz), *fb = (uint64_t *)malloc(sz);
    o_negacyclic_batch(fa, a, batch, n, psis, qs, nq, 0);
    o_negacyclic_batch(fb, b, batch, n, psis, qs, nq, 0);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < batch * n; i++) {
        int64_t m = (i / n) % nq;
        st(fa + 2 * i, mulmod(ld(fa + 2 * i), ld(fb + 2 * i), ld(qs + 2 * m)));
    }
    o_negacyclic_batch(c, fa, batch, n, psis, qs, nq, 1);
    free(fa);
    free(fb);
}

int o_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
