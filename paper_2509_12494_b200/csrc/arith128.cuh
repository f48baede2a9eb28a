// arith128.cuh -- 128-bit modular arithmetic for sm_100a, on four 32-bit words.
//
// The paper builds 128-bit "double-word" arithmetic from 64-bit machine words and
// carry chains (Eq. def_dw / Eq. muls) and proposes MQX, an ISA
// extension with a widening multiply, add-with-carry and sub-with-borrow
// (§4).  On sm_100a every SIMT lane already has those at
// omega0 = 32 bits: ptxas fuses a `mad.lo.cc.u32` / `madc.hi.cc.u32` pair into one
// IMAD.WIDE.U32 with carry-in/carry-out predicates, and `add.cc`/`addc` become
// IADD3 with carry predicates.  The code below is written in that PTX so the
// SASS is the MQX-style sequence natively.
//
// Residues are canonical (< q) at every interface; q is any odd modulus < 2^128
// (reading c1: the paper's 124-bit Barrett limit, does not
// apply).  Sums and Montgomery remainders that exceed 2^128 keep their 129th bit
// in an extra word (SURVEY.md §0 finding 2: lazy reduction is impossible here).
//
// mulmod is Montgomery (R = 2^128, word-serial CIOS, even/odd split): the paper's Barrett
// (Eq. barrett) computes the same unique residue; Montgomery
// needs no 129-bit quotient estimate and costs 32 IMAD.WIDE + 4 IMAD.
#pragma once
#include <cstdint>

namespace ntt128 {

struct U128 {
    uint32_t w[4];  // little endian: value = w[0] + w[1] 2^32 + w[2] 2^64 + w[3] 2^96
};

// Per-modulus constants (device copy of the plan's host computation).
struct ModC {
    uint32_t q[4];
    uint32_t qinv0;     // -q^{-1} mod 2^32
    uint32_t pad[3];
    uint32_t one_m[4];  // R mod q            (Montgomery form of 1)
    uint32_t r2[4];     // R^2 mod q          (to-Montgomery factor)
    uint32_t ninv_m[4]; // N^{-1} R mod q     (Montgomery form of N^{-1})
    uint32_t ninv_rm[4];// N^{-1} R^2 mod q   (Montgomery form of N^{-1} R: undoes a point-wise R^{-1})
};

__device__ __forceinline__ U128 u128_from(uint4 v) { return U128{{v.x, v.y, v.z, v.w}}; }
__device__ __forceinline__ uint4 u128_to(const U128& a) { return make_uint4(a.w[0], a.w[1], a.w[2], a.w[3]); }

// c = a + b mod q (Eq. saddmod): 129-bit sum, 129-bit compare
// against q via a borrow chain, branch-free select.
__device__ __forceinline__ U128 add_mod(const U128& a, const U128& b, const uint32_t q[4]) {
    uint32_t s0, s1, s2, s3, s4, d0, d1, d2, d3, bw;
    asm("add.cc.u32  %0, %5, %9;\n\t"
        "addc.cc.u32 %1, %6, %10;\n\t"
        "addc.cc.u32 %2, %7, %11;\n\t"
        "addc.cc.u32 %3, %8, %12;\n\t"
        "addc.u32    %4, 0, 0;"
        : "=r"(s0), "=r"(s1), "=r"(s2), "=r"(s3), "=r"(s4)
        : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]), "r"(b.w[3]));
    asm("sub.cc.u32  %0, %5, %10;\n\t"
        "subc.cc.u32 %1, %6, %11;\n\t"
        "subc.cc.u32 %2, %7, %12;\n\t"
        "subc.cc.u32 %3, %8, %13;\n\t"
        "subc.u32    %4, %9, 0;"
        : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(d3), "=r"(bw)
        : "r"(s0), "r"(s1), "r"(s2), "r"(s3), "r"(s4), "r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]));
    // bw == 0 (no borrow): s >= q, take d; bw == 0xffffffff: take s
    U128 r;
    r.w[0] = (s0 & bw) | (d0 & ~bw);
    r.w[1] = (s1 & bw) | (d1 & ~bw);
    r.w[2] = (s2 & bw) | (d2 & ~bw);
    r.w[3] = (s3 & bw) | (d3 & ~bw);
    return r;
}

// c = a - b mod q (Eq. ssubmod): borrow chain, then + (q & mask).
__device__ __forceinline__ U128 sub_mod(const U128& a, const U128& b, const uint32_t q[4]) {
    uint32_t d0, d1, d2, d3, bw;
    asm("sub.cc.u32  %0, %5, %9;\n\t"
        "subc.cc.u32 %1, %6, %10;\n\t"
        "subc.cc.u32 %2, %7, %11;\n\t"
        "subc.cc.u32 %3, %8, %12;\n\t"
        "subc.u32    %4, 0, 0;"
        : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(d3), "=r"(bw)
        : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]), "r"(b.w[3]));
    U128 r;
    asm("add.cc.u32  %0, %4, %8;\n\t"
        "addc.cc.u32 %1, %5, %9;\n\t"
        "addc.cc.u32 %2, %6, %10;\n\t"
        "addc.u32    %3, %7, %11;"
        : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3])
        : "r"(d0), "r"(d1), "r"(d2), "r"(d3), "r"(q[0] & bw), "r"(q[1] & bw), "r"(q[2] & bw), "r"(q[3] & bw));
    return r;
}

// Montgomery product core, even/odd alternating CIOS (R = 2^128, 32-bit digits b_i of b).
// Preconditions: b < q and either a < 2^128 (any odd q < 2^128) or, for the lazy
// callers, a < 4q with q < 2^126 / a < 2q with q < 2^127.  Output: T = a b R^-1 + {0, q},
// T < 2q, as five words t[0..4] (t[4] <= 1; t[4] == 0 when 2q <= 2^128).
//
// The running value is held as 2^32 T_i = X + 2^32 Y with two multiword accumulators
// whose 64-bit partial products are all register-pair aligned: X collects the
// a_even b_i = (a0 + a2 2^64) b_i and m (q0 + q2 2^64) products, Y the odd ones
// (a1 + a3 2^64) b_i and m (q1 + q3 2^64).  After a digit X_0 = 0 and the division by
// 2^32 is a change of roles instead of a 5-word add: the next X is Y with X_1 added to
// its word 0 (the carry of that add has weight 2^32 and enters the next Y chain as
// its carry-in), the next Y is X / 2^64 (words X_2, X_3, X_4 used as the addends of
// the next a_odd b_i products, so the shift costs nothing).  Per digit: 8 IMAD.WIDE,
// 1 IMAD (m = X_0 q'), 4 carry ops; one 5-word add at the end.  Every dropped carry
// is proven absent in tools/model/mont_eo_model.c (which asserts it on 10^6 cases
// including q = 2^128 - 1 and a = 2^128 - 1).
template <bool TOP>
__device__ __forceinline__ void mont_core(const U128& a, const U128& b, const uint32_t q[4], uint32_t qinv0,
                                          uint32_t t[5]) {
    uint32_t x0, x1, x2, x3, x4, y0, y1, y2, y3, y4, m;
    // digit 0: X = a_even b0, Y = a_odd b0 (fresh 64-bit products, no carries)
    asm("{\n\t.reg .u64 p;\n\t"
        "mul.wide.u32 p, %8, %12;\n\tmov.b64 {%0, %1}, p;\n\t"
        "mul.wide.u32 p, %10, %12;\n\tmov.b64 {%2, %3}, p;\n\t"
        "mul.wide.u32 p, %9, %12;\n\tmov.b64 {%4, %5}, p;\n\t"
        "mul.wide.u32 p, %11, %12;\n\tmov.b64 {%6, %7}, p;\n\t}"
        : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3), "=r"(y0), "=r"(y1), "=r"(y2), "=r"(y3)
        : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(b.w[0]));
    m = x0 * qinv0;
    asm("mad.lo.cc.u32  %0, %5, %6, %0;\n\t"
        "madc.hi.cc.u32 %1, %5, %6, %1;\n\t"
        "madc.lo.cc.u32 %2, %5, %7, %2;\n\t"
        "madc.hi.cc.u32 %3, %5, %7, %3;\n\t"
        "addc.u32       %4, 0, 0;"
        : "+r"(x0), "+r"(x1), "+r"(x2), "+r"(x3), "=r"(x4)
        : "r"(m), "r"(q[0]), "r"(q[2]));
    asm("mad.lo.cc.u32  %0, %5, %6, %0;\n\t"
        "madc.hi.cc.u32 %1, %5, %6, %1;\n\t"
        "madc.lo.cc.u32 %2, %5, %7, %2;\n\t"
        "madc.hi.cc.u32 %3, %5, %7, %3;\n\t"
        "addc.u32       %4, 0, 0;"
        : "+r"(y0), "+r"(y1), "+r"(y2), "+r"(y3), "=r"(y4)
        : "r"(m), "r"(q[1]), "r"(q[3]));
#pragma unroll
    for (int i = 1; i < 4; i++) {
        uint32_t n0, n1, n2, n3, n4;
        // X' = Y + X_1 (+ a_even b_i below); Y' = X / 2^64 + carry + a_odd b_i (no carry out)
        asm("add.cc.u32     %0, %0, %9;\n\t"
            "madc.lo.cc.u32 %5, %12, %13, %10;\n\t"
            "madc.hi.cc.u32 %6, %12, %13, %11;\n\t"
            "madc.lo.cc.u32 %7, %14, %13, %15;\n\t"
            "madc.hi.u32    %8, %14, %13, 0;\n\t"
            "mad.lo.cc.u32  %0, %16, %13, %0;\n\t"
            "madc.hi.cc.u32 %1, %16, %13, %1;\n\t"
            "madc.lo.cc.u32 %2, %17, %13, %2;\n\t"
            "madc.hi.cc.u32 %3, %17, %13, %3;\n\t"
            "addc.u32       %4, %4, 0;"
            : "+r"(y0), "+r"(y1), "+r"(y2), "+r"(y3), "+r"(y4), "=&r"(n0), "=&r"(n1), "=&r"(n2), "=&r"(n3)
            : "r"(x1), "r"(x2), "r"(x3), "r"(a.w[1]), "r"(b.w[i]), "r"(a.w[3]), "r"(x4), "r"(a.w[0]), "r"(a.w[2]));
        m = y0 * qinv0;
        asm("mad.lo.cc.u32  %0, %5, %6, %0;\n\t"
            "madc.hi.cc.u32 %1, %5, %6, %1;\n\t"
            "madc.lo.cc.u32 %2, %5, %7, %2;\n\t"
            "madc.hi.cc.u32 %3, %5, %7, %3;\n\t"
            "addc.u32       %4, %4, 0;"
            : "+r"(y0), "+r"(y1), "+r"(y2), "+r"(y3), "+r"(y4)
            : "r"(m), "r"(q[0]), "r"(q[2]));
        asm("mad.lo.cc.u32  %0, %5, %6, %0;\n\t"
            "madc.hi.cc.u32 %1, %5, %6, %1;\n\t"
            "madc.lo.cc.u32 %2, %5, %7, %2;\n\t"
            "madc.hi.cc.u32 %3, %5, %7, %3;\n\t"
            "addc.u32       %4, 0, 0;"
            : "+r"(n0), "+r"(n1), "+r"(n2), "+r"(n3), "=r"(n4)
            : "r"(m), "r"(q[1]), "r"(q[3]));
        // roles: X <- X' (held in y), Y <- Y' (held in n)
        x0 = y0; x1 = y1; x2 = y2; x3 = y3; x4 = y4;
        y0 = n0; y1 = n1; y2 = n2; y3 = n3; y4 = n4;
    }
    // T = Y + X / 2^32 (X_0 == 0)
    if (TOP) {
        asm("add.cc.u32  %0, %5, %10;\n\t"
            "addc.cc.u32 %1, %6, %11;\n\t"
            "addc.cc.u32 %2, %7, %12;\n\t"
            "addc.cc.u32 %3, %8, %13;\n\t"
            "addc.u32    %4, %9, 0;"
            : "=r"(t[0]), "=r"(t[1]), "=r"(t[2]), "=r"(t[3]), "=r"(t[4])
            : "r"(y0), "r"(y1), "r"(y2), "r"(y3), "r"(y4), "r"(x1), "r"(x2), "r"(x3), "r"(x4));
    } else {   // T < 2q <= 2^128: word 4 is zero
        asm("add.cc.u32  %0, %4, %8;\n\t"
            "addc.cc.u32 %1, %5, %9;\n\t"
            "addc.cc.u32 %2, %6, %10;\n\t"
            "addc.u32    %3, %7, %11;"
            : "=r"(t[0]), "=r"(t[1]), "=r"(t[2]), "=r"(t[3])
            : "r"(y0), "r"(y1), "r"(y2), "r"(y3), "r"(x1), "r"(x2), "r"(x3), "r"(x4));
        t[4] = 0;
    }
}

// Montgomery product a * b * 2^-128 mod q, canonical result.  Preconditions: b < q,
// a < 2^128, q odd.  32 IMAD.WIDE + 4 IMAD per call (the 36 algorithmic products of
// §8(d)); T < 2q keeps its bit 128 in t[4]; one conditional subtraction.
__device__ __forceinline__ U128 mont_mul(const U128& a, const U128& b, const uint32_t q[4], uint32_t qinv0) {
    uint32_t t[5];
    mont_core<true>(a, b, q, qinv0, t);
    uint32_t d0, d1, d2, d3, bw;
    asm("sub.cc.u32  %0, %5, %10;\n\t"
        "subc.cc.u32 %1, %6, %11;\n\t"
        "subc.cc.u32 %2, %7, %12;\n\t"
        "subc.cc.u32 %3, %8, %13;\n\t"
        "subc.u32    %4, %9, 0;"
        : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(d3), "=r"(bw)
        : "r"(t[0]), "r"(t[1]), "r"(t[2]), "r"(t[3]), "r"(t[4]), "r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]));
    U128 r;
    r.w[0] = (t[0] & bw) | (d0 & ~bw);
    r.w[1] = (t[1] & bw) | (d1 & ~bw);
    r.w[2] = (t[2] & bw) | (d2 & ~bw);
    r.w[3] = (t[3] & bw) | (d3 & ~bw);
    return r;
}

// ---------------------------------------------------------------------------------------
// Lazy reduction, by modulus class:
//   q < 2^126 ("lazy"): butterfly values in [0, 4q) (4q < 2^128), Harvey butterflies;
//   2^126 <= q < 2^127 ("half"): values in [0, 2q) (2q < 2^128), add/sub modulo 2q;
//   q >= 2^127: canonical values (mont_mul, add_mod, sub_mod).
// mont_mul_lazy: b < q and a < 4q (q < 2^126) or a < 2q (q < 2^127) -> T = a b R^-1 + {0, q}
// in [0, 2q) (T < q (1 + a / R) < 2q); no final subtraction, no fifth word.
__device__ __forceinline__ U128 mont_mul_lazy(const U128& a, const U128& b, const uint32_t q[4], uint32_t qinv0) {
    uint32_t t[5];
    mont_core<false>(a, b, q, qinv0, t);
    return U128{{t[0], t[1], t[2], t[3]}};
}

// x - m if x >= m else x (x < 2^128, m < 2^128): one borrow chain and a select.  With
// m = 2q it maps [0, 4q) to [0, 2q); with m = q, [0, 2q) to [0, q).
__device__ __forceinline__ U128 reduce_2q(const U128& x, const uint32_t q2[4]) {
    uint32_t d0, d1, d2, d3, bw;
    asm("sub.cc.u32  %0, %5, %9;\n\t"
        "subc.cc.u32 %1, %6, %10;\n\t"
        "subc.cc.u32 %2, %7, %11;\n\t"
        "subc.cc.u32 %3, %8, %12;\n\t"
        "subc.u32    %4, 0, 0;"
        : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(d3), "=r"(bw)
        : "r"(x.w[0]), "r"(x.w[1]), "r"(x.w[2]), "r"(x.w[3]), "r"(q2[0]), "r"(q2[1]), "r"(q2[2]), "r"(q2[3]));
    U128 r;
    r.w[0] = (x.w[0] & bw) | (d0 & ~bw);
    r.w[1] = (x.w[1] & bw) | (d1 & ~bw);
    r.w[2] = (x.w[2] & bw) | (d2 & ~bw);
    r.w[3] = (x.w[3] & bw) | (d3 & ~bw);
    return r;
}

// u + t (no reduction; caller guarantees u + t < 2^128)
__device__ __forceinline__ U128 add_nored(const U128& u, const U128& t) {
    U128 s;
    asm("add.cc.u32  %0, %4, %8;\n\t"
        "addc.cc.u32 %1, %5, %9;\n\t"
        "addc.cc.u32 %2, %6, %10;\n\t"
        "addc.u32    %3, %7, %11;"
        : "=r"(s.w[0]), "=r"(s.w[1]), "=r"(s.w[2]), "=r"(s.w[3])
        : "r"(u.w[0]), "r"(u.w[1]), "r"(u.w[2]), "r"(u.w[3]), "r"(t.w[0]), "r"(t.w[1]), "r"(t.w[2]), "r"(t.w[3]));
    return s;
}
// u - t + c (no reduction; caller guarantees 0 <= u - t + c < 2^128)
__device__ __forceinline__ U128 sub_add_nored(const U128& u, const U128& t, const uint32_t c[4]) {
    U128 s;
    asm("sub.cc.u32  %0, %4, %8;\n\t"
        "subc.cc.u32 %1, %5, %9;\n\t"
        "subc.cc.u32 %2, %6, %10;\n\t"
        "subc.u32    %3, %7, %11;\n\t"
        "add.cc.u32  %0, %0, %12;\n\t"
        "addc.cc.u32 %1, %1, %13;\n\t"
        "addc.cc.u32 %2, %2, %14;\n\t"
        "addc.u32    %3, %3, %15;"
        : "=&r"(s.w[0]), "=&r"(s.w[1]), "=&r"(s.w[2]), "=&r"(s.w[3])
        : "r"(u.w[0]), "r"(u.w[1]), "r"(u.w[2]), "r"(u.w[3]), "r"(t.w[0]), "r"(t.w[1]), "r"(t.w[2]), "r"(t.w[3]),
          "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]));
    return s;
}

// u 2^-s mod q, 1 <= s <= 31 (the inverse transform's N^-1 = 2^-n on the last stage's u
// branch, DESIGN.md §5 "N^-1 by one short digit"): a single s-bit Montgomery digit,
// m = u_0 (-q^-1) mod 2^s, so u + m q = 0 mod 2^s, and T = (u + m q) / 2^s = u 2^-s (mod q)
// with T < q + u / 2^s.  4 low + 4 high 32x32 products and 4 funnel shifts instead of a
// 36-product Montgomery multiplication by N^-1 R.  t[4] is T's bit 128 (T < 2^129).
__device__ __forceinline__ void shr_core(const U128& u, uint32_t s, const uint32_t q[4], uint32_t qinv0, uint32_t t[5]) {
    const uint32_t m = (u.w[0] * qinv0) & ((1u << s) - 1u);
    uint32_t x0, x1, x2, x3, x4;
    asm("mad.lo.cc.u32  %0, %5, %6, %10;\n\t"
        "madc.lo.cc.u32 %1, %5, %7, %11;\n\t"
        "madc.lo.cc.u32 %2, %5, %8, %12;\n\t"
        "madc.lo.cc.u32 %3, %5, %9, %13;\n\t"
        "addc.u32       %4, 0, 0;\n\t"
        "mad.hi.cc.u32  %1, %5, %6, %1;\n\t"
        "madc.hi.cc.u32 %2, %5, %7, %2;\n\t"
        "madc.hi.cc.u32 %3, %5, %8, %3;\n\t"
        "madc.hi.u32    %4, %5, %9, %4;"
        : "=&r"(x0), "=&r"(x1), "=&r"(x2), "=&r"(x3), "=&r"(x4)
        : "r"(m), "r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]), "r"(u.w[0]), "r"(u.w[1]), "r"(u.w[2]), "r"(u.w[3]));
    t[0] = __funnelshift_r(x0, x1, s);
    t[1] = __funnelshift_r(x1, x2, s);
    t[2] = __funnelshift_r(x2, x3, s);
    t[3] = __funnelshift_r(x3, x4, s);
    t[4] = x4 >> s;
}
// canonical u 2^-s mod q for u < q (T < q + q / 2^s < 2q: one conditional subtraction)
__device__ __forceinline__ U128 shr_mod(const U128& u, uint32_t s, const uint32_t q[4], uint32_t qinv0) {
    uint32_t t[5];
    shr_core(u, s, q, qinv0, t);
    uint32_t d0, d1, d2, d3, bw;
    asm("sub.cc.u32  %0, %5, %10;\n\t"
        "subc.cc.u32 %1, %6, %11;\n\t"
        "subc.cc.u32 %2, %7, %12;\n\t"
        "subc.cc.u32 %3, %8, %13;\n\t"
        "subc.u32    %4, %9, 0;"
        : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(d3), "=r"(bw)
        : "r"(t[0]), "r"(t[1]), "r"(t[2]), "r"(t[3]), "r"(t[4]), "r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]));
    U128 r;
    r.w[0] = (t[0] & bw) | (d0 & ~bw);
    r.w[1] = (t[1] & bw) | (d1 & ~bw);
    r.w[2] = (t[2] & bw) | (d2 & ~bw);
    r.w[3] = (t[3] & bw) | (d3 & ~bw);
    return r;
}
// lazy u 2^-s mod q in [0, 2q): u < 4q with q < 2^126 and s >= 2, or u < 2q with q < 2^127
// (T < q + u / 2^s <= 2q < 2^128: no fifth word)
__device__ __forceinline__ U128 shr_mod_lazy(const U128& u, uint32_t s, const uint32_t q[4], uint32_t qinv0) {
    uint32_t t[5];
    shr_core(u, s, q, qinv0, t);
    return U128{{t[0], t[1], t[2], t[3]}};
}

// a < q check (for NTT128_FLAG_CHECK_INPUT): borrow out of a - q
__device__ __forceinline__ bool lt_q(const U128& a, const uint32_t q[4]) {
    uint32_t bw;
    asm("{\n\t.reg .u32 d0, d1, d2, d3;\n\t"
        "sub.cc.u32  d0, %1, %5;\n\t"
        "subc.cc.u32 d1, %2, %6;\n\t"
        "subc.cc.u32 d2, %3, %7;\n\t"
        "subc.cc.u32 d3, %4, %8;\n\t"
        "subc.u32    %0, 0, 0;\n\t}"
        : "=r"(bw)
        : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]));
    return bw != 0;
}

}  // namespace ntt128
