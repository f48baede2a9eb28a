/*
 * oracle256.c -- plain, slow, obviously-correct CPU oracle for the wider-modulus NTT
 * ("wider multi-word moduli (192/256-bit) by recursive
 * decomposition", the paper's stated generalisation, "Generalizing to
 * larger bit-widths").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's oracle
 * legs may load this library.  It shares no code with the CUDA path
 * (paper_2509_12494_b200/csrc, include/) nor with oracle128.c.
 *
 * A residue is 256 bits as four uint64 limbs, little endian (x = sum x[i] 2^(64 i)),
 * 0 <= x < q for any odd modulus q < 2^256.  Definitions written out:
 *   - the product: schoolbook over 64-bit limbs (Eq. muls generalised to four words,
 *     PAPER.md:244-249), each limb product formed with unsigned __int128;
 *   - the remainder: restoring binary long division of the 512-bit product (the
 *     literal definition of x mod q);
 *   - Eq. saddmod / ssubmod with an explicit 257th bit;
 *   - the NTT by definition (Eq. ntt) for small N and the textbook
 *     iterative radix-2 Cooley-Tukey for larger N; the inverse with N^{-1}.
 * Pins: tests/test_oracle256.py (Python integers, Fermat, DFT by definition in pure
 * Python, closed forms, round trips).  No function here is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;
typedef struct { uint64_t w[4]; } u256;

static u256 ld4(const uint64_t *p) { u256 r; memcpy(r.w, p, 32); return r; }
static void st4(uint64_t *p, u256 v) { memcpy(p, v.w, 32); }

static int cmp4(u256 a, u256 b) {
    for (int i = 3; i >= 0; i--) {
        if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
    }
    return 0;
}
/* a + b with carry out */
static u256 add4(u256 a, u256 b, unsigned *carry) {
    u256 r;
    unsigned c = 0;
    for (int i = 0; i < 4; i++) {
        u128 s = (u128)a.w[i] + b.w[i] + c;
        r.w[i] = (uint64_t)s;
        c = (unsigned)(s >> 64);
    }
    *carry = c;
    return r;
}
/* a - b with borrow out */
static u256 sub4(u256 a, u256 b, unsigned *borrow) {
    u256 r;
    unsigned bw = 0;
    for (int i = 0; i < 4; i++) {
        u128 d = (u128)a.w[i] - b.w[i] - bw;
        r.w[i] = (uint64_t)d;
        bw = (unsigned)((d >> 64) & 1);
    }
    *borrow = bw;
    return r;
}

/* Eq. saddmod: s = a + b as a 257-bit value; subtract q when s >= q */
static u256 addmod4(u256 a, u256 b, u256 q) {
    unsigned c, bw;
    u256 s = add4(a, b, &c);
    u256 d = sub4(s, q, &bw);
    return (c || !bw) ? d : s;   /* s >= q  <=>  carry out, or no borrow from s - q */
}
/* Eq. ssubmod: a - b, plus q when it borrowed */
static u256 submod4(u256 a, u256 b, u256 q) {
    unsigned bw, c;
    u256 d = sub4(a, b, &bw);
    return bw ? add4(d, q, &c) : d;
}

/* the 512-bit schoolbook product p[0..7] = a b */
static void mul_full4(u256 a, u256 b, uint64_t p[8]) {
    memset(p, 0, 64);
    for (int i = 0; i < 4; i++) {
        uint64_t carry = 0;
        for (int j = 0; j < 4; j++) {
            u128 t = (u128)a.w[i] * b.w[j] + p[i + j] + carry;
            p[i + j] = (uint64_t)t;
            carry = (uint64_t)(t >> 64);
        }
        p[i + 4] = carry;
    }
}
/* x mod q by restoring long division over the bits of x[0..nw-1] (the definition) */
static u256 rem_words(const uint64_t *x, int nw, u256 q) {
    u256 r = {{0, 0, 0, 0}};
    for (int i = nw * 64 - 1; i >= 0; i--) {
        unsigned top = (unsigned)(r.w[3] >> 63);                 /* bit 256 after the shift */
        for (int k = 3; k > 0; k--) r.w[k] = (r.w[k] << 1) | (r.w[k - 1] >> 63);
        r.w[0] = (r.w[0] << 1) | ((x[i / 64] >> (i % 64)) & 1);
        if (top || cmp4(r, q) >= 0) {
            unsigned bw;
            r = sub4(r, q, &bw);                                  /* wraps correctly when top */
        }
    }
    return r;
}
static u256 mulmod4(u256 a, u256 b, u256 q) {
    uint64_t p[8];
    mul_full4(a, b, p);
    return rem_words(p, 8, q);
}
static u256 powmod4(u256 a, u256 e, u256 q) {
    u256 r = {{1, 0, 0, 0}};
    r = rem_words(r.w, 4, q);
    for (int i = 255; i >= 0; i--) {
        r = mulmod4(r, r, q);
        if ((e.w[i / 64] >> (i % 64)) & 1) r = mulmod4(r, a, q);
    }
    return r;
}
static u256 invmod4(u256 a, u256 q) {   /* q prime: a^(q-2) (Fermat) */
    u256 two = {{2, 0, 0, 0}};
    unsigned bw;
    return powmod4(a, sub4(q, two, &bw), q);
}
static u256 from_u64(uint64_t v) { u256 r = {{v, 0, 0, 0}}; return r; }

/* ---------------------------------------------------------------- exported scalars */
void o4_mul_full(const uint64_t *a, const uint64_t *b, uint64_t *out8) { mul_full4(ld4(a), ld4(b), out8); }
void o4_addmod(const uint64_t *a, const uint64_t *b, const uint64_t *q, uint64_t *r) { st4(r, addmod4(ld4(a), ld4(b), ld4(q))); }
void o4_submod(const uint64_t *a, const uint64_t *b, const uint64_t *q, uint64_t *r) { st4(r, submod4(ld4(a), ld4(b), ld4(q))); }
void o4_mulmod(const uint64_t *a, const uint64_t *b, const uint64_t *q, uint64_t *r) { st4(r, mulmod4(ld4(a), ld4(b), ld4(q))); }
void o4_powmod(const uint64_t *a, const uint64_t *e, const uint64_t *q, uint64_t *r) { st4(r, powmod4(ld4(a), ld4(e), ld4(q))); }

/* ---------------------------------------------------------------- vectors */
void o4_vmul(uint64_t *z, const uint64_t *x, const uint64_t *y, int64_t n, const uint64_t *q_) {
    u256 q = ld4(q_);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) st4(z + 4 * i, mulmod4(ld4(x + 4 * i), ld4(y + 4 * i), q));
}

/* ---------------------------------------------------------------- NTT
 * Eq. ntt: y_k = sum_j x_j w^{jk} mod q, natural order in and out. */
static void dft_one(uint64_t *y, const uint64_t *x, int64_t n, u256 w, u256 q) {
    u256 wk = rem_words(from_u64(1).w, 4, q);           /* w^k */
    for (int64_t k = 0; k < n; k++) {
        u256 acc = {{0, 0, 0, 0}}, p = rem_words(from_u64(1).w, 4, q);   /* p = w^{jk} */
        for (int64_t j = 0; j < n; j++) {
            acc = addmod4(acc, mulmod4(ld4(x + 4 * j), p, q), q);
            p = mulmod4(p, wk, q);
        }
        st4(y + 4 * k, acc);
        wk = mulmod4(wk, w, q);
    }
}
/* textbook iterative radix-2 Cooley-Tukey: bit-reversed copy, then log2 n stages */
static void ntt_one(uint64_t *y, const uint64_t *x, int64_t n, u256 w, u256 q) {
    int lg = 0;
    while (((int64_t)1 << lg) < n) lg++;
    for (int64_t i = 0; i < n; i++) {
        int64_t r = 0;
        for (int b = 0; b < lg; b++) r |= ((i >> b) & 1) << (lg - 1 - b);
        memcpy(y + 4 * r, x + 4 * i, 32);
    }
    for (int64_t len = 2; len <= n; len <<= 1) {
        /* wl = w^(n / len), a primitive len-th root */
        u256 e = from_u64((uint64_t)(n / len));
        u256 wl = powmod4(w, e, q);
        for (int64_t s = 0; s < n; s += len) {
            u256 t = rem_words(from_u64(1).w, 4, q);
            for (int64_t j = 0; j < len / 2; j++) {
                u256 u = ld4(y + 4 * (s + j));
                u256 v = mulmod4(ld4(y + 4 * (s + j + len / 2)), t, q);
                st4(y + 4 * (s + j), addmod4(u, v, q));
                st4(y + 4 * (s + j + len / 2), submod4(u, v, q));
                t = mulmod4(t, wl, q);
            }
        }
    }
}
/* batch of transforms, polynomial b with modulus qs[b % nq] and root ws[b % nq]; inverse:
 * x = N^{-1} DFT_{w^{-1}}(y).  small != 0 selects the O(N^2) definition. */
void o4_ntt_batch(uint64_t *out, const uint64_t *in, int64_t batch, int64_t n, const uint64_t *ws,
                  const uint64_t *qs, int64_t nq, int inverse, int small) {
#pragma omp parallel for schedule(dynamic)
    for (int64_t b = 0; b < batch; b++) {
        u256 q = ld4(qs + 4 * (b % nq)), w = ld4(ws + 4 * (b % nq));
        if (inverse) w = invmod4(w, q);
        uint64_t *y = out + 4 * n * b;
        const uint64_t *x = in + 4 * n * b;
        if (small) dft_one(y, x, n, w, q);
        else ntt_one(y, x, n, w, q);
        if (inverse) {
            u256 ninv = invmod4(rem_words(from_u64((uint64_t)n).w, 4, q), q);
            for (int64_t i = 0; i < n; i++) st4(y + 4 * i, mulmod4(ld4(y + 4 * i), ninv, q));
        }
    }
}

/* ---------------------------------------------------------------- primes (plan inputs)
 * Miller-Rabin with the first 40 primes as bases (n odd, n > 200), the same test the
 * 128-bit oracle pins against sympy's BPSW. */
static int is_prime4(u256 n) {
    static const uint64_t bases[40] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59, 61, 67, 71,
                                       73, 79, 83, 89, 97, 101, 103, 107, 109, 113, 127, 131, 137, 139, 149, 151, 157, 163, 167, 173};
    if ((n.w[0] & 1) == 0) return 0;
    for (int i = 0; i < 40; i++) {   /* trial division by the bases: remainder of n mod p */
        u256 r = rem_words(n.w, 4, from_u64(bases[i]));
        if (r.w[0] == 0) return cmp4(n, from_u64(bases[i])) == 0;
    }
    unsigned bw;
    u256 nm1 = sub4(n, from_u64(1), &bw);
    u256 d = nm1;
    int s = 0;
    while ((d.w[0] & 1) == 0) {
        for (int k = 0; k < 3; k++) d.w[k] = (d.w[k] >> 1) | (d.w[k + 1] << 63);
        d.w[3] >>= 1;
        s++;
    }
    for (int i = 0; i < 40; i++) {
        u256 x = powmod4(from_u64(bases[i]), d, n);
        if (cmp4(x, from_u64(1)) == 0 || cmp4(x, nm1) == 0) continue;
        int ok = 0;
        for (int r = 1; r < s && !ok; r++) {
            x = mulmod4(x, x, n);
            if (cmp4(x, nm1) == 0) ok = 1;
        }
        if (!ok) return 0;
    }
    return 1;
}
int o4_is_prime(const uint64_t *n) { return is_prime4(ld4(n)); }
/* the (skip)-th largest prime q < 2^bits with q = 1 mod m (m a power of two < 2^64):
 * descending scan over q = k m + 1 */
int o4_find_prime(int bits, uint64_t m, int skip, uint64_t *out) {
    u256 top = {{0, 0, 0, 0}};                 /* 2^bits - m + 1: the largest k m + 1 < 2^bits */
    if (bits < 256) top.w[bits / 64] = (uint64_t)1 << (bits % 64);
    unsigned bw, c;
    u256 q = sub4(top, from_u64(m), &bw);       /* wraps for bits = 256: 2^256 - m */
    q = add4(q, from_u64(1), &c);
    for (long it = 0; it < 10000000; it++) {
        if (is_prime4(q)) {
            if (skip == 0) { st4(out, q); return 1; }
            skip--;
        }
        q = sub4(q, from_u64(m), &bw);
    }
    return 0;
}

int o4_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
