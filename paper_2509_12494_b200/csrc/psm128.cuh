// psm128.cuh -- arithmetic for pseudo-Mersenne moduli q = 2^b - c (124 <= b <= 128 here, any
// b with c 2^(128-b) < 2^32), the "PSM" class of the plain cyclic multi-pass NTT kernels.
//
// The largest NTT-friendly primes below a power of two (the paper's workloads: "128-bit
// primes") have this shape.  With s = 128 - b and
// Q = q 2^s = 2^128 - C, C = c 2^s < 2^32, arithmetic modulo Q is arithmetic modulo q
// (q | Q), and 2^128 = C (mod Q): a 256-bit product H 2^128 + L folds to H C + L
// (4 word products), and its fifth word folds once more with the quotient estimate l4 + 1
// (1 product) straight to the residue modulo Q.  A butterfly's product costs 16 + 4 + 1 = 21
// word products instead of Montgomery's 36 (DESIGN.md §5 "Pseudo-Mersenne class"); twiddles
// are stored as plain residues.
//
// Representation between stages: ANY 128-bit value congruent to the residue modulo q
// (not canonical, not even < Q); psm_canon maps it to [0, q) in the last pass's store.
// psm_mul returns t < Q, so the butterfly's u + t and u - t fold their carry / borrow once
// (psm_add1 / psm_sub1); the twiddle-1 butterflies add and subtract two arbitrary
// representatives and fold twice (psm_add / psm_sub).  C = 2^32 - 1 is excluded by the host.
// The word-level algorithm (every carry, every bound) is modelled and checked against
// Python integers in tools/model/psm_model.py (CPU test tests/test_psm_model.py).
#pragma once
#include <cstdint>

#include "arith128.cuh"

namespace ntt128 {

// s = 128 - bitlen(q); C = 2^128 - q 2^s (eligibility, checked by the host: words 1..3 of
// q 2^s are all ones, so C = -(q_0 2^s) mod 2^32, C >= 1).
__device__ __forceinline__ uint32_t psm_shift(const uint32_t q[4]) { return (uint32_t)__clz((int)q[3]); }
__device__ __forceinline__ uint32_t psm_C(const uint32_t q[4], uint32_t s) { return 0u - (q[0] << s); }

// a + b (mod Q), a, b < 2^128: the carry folds as + C; a second carry (both operands within
// C of 2^128) leaves a value < C, and + C again cannot overflow.
__device__ __forceinline__ U128 psm_add(const U128& a, const U128& b, uint32_t C) {
    uint32_t s0, s1, s2, s3, k;
    asm("add.cc.u32  %0, %5, %9;\n\t"
        "addc.cc.u32 %1, %6, %10;\n\t"
        "addc.cc.u32 %2, %7, %11;\n\t"
        "addc.cc.u32 %3, %8, %12;\n\t"
        "addc.u32    %4, 0, 0;"
        : "=r"(s0), "=r"(s1), "=r"(s2), "=r"(s3), "=r"(k)
        : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]), "r"(b.w[3]));
    const uint32_t f = (0u - k) & C;
    asm("add.cc.u32  %0, %0, %5;\n\t"
        "addc.cc.u32 %1, %1, 0;\n\t"
        "addc.cc.u32 %2, %2, 0;\n\t"
        "addc.cc.u32 %3, %3, 0;\n\t"
        "addc.u32    %4, 0, 0;"
        : "+r"(s0), "+r"(s1), "+r"(s2), "+r"(s3), "=r"(k)
        : "r"(f));
    const uint32_t f2 = (0u - k) & C;   // k == 1: the value is < C < 2^32 (words 1..3 are zero)
    asm("add.cc.u32  %0, %0, %2;\n\t"
        "addc.u32    %1, %1, 0;"
        : "+r"(s0), "+r"(s1)
        : "r"(f2));
    return U128{{s0, s1, s2, s3}};
}

// a - b (mod Q): the borrow folds as - C (-2^128 = -C); a second borrow leaves a value
// >= 2^128 - C, and - C again cannot borrow (2^128 - 2C > 0) and touches words 0..1 only
// when words 2..3 are all ones -- the chain still runs over four words for the first fold.
__device__ __forceinline__ U128 psm_sub(const U128& a, const U128& b, uint32_t C) {
    uint32_t d0, d1, d2, d3, bw;
    asm("sub.cc.u32  %0, %5, %9;\n\t"
        "subc.cc.u32 %1, %6, %10;\n\t"
        "subc.cc.u32 %2, %7, %11;\n\t"
        "subc.cc.u32 %3, %8, %12;\n\t"
        "subc.u32    %4, 0, 0;"
        : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(d3), "=r"(bw)
        : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]), "r"(b.w[3]));
    const uint32_t f = bw & C;
    asm("sub.cc.u32  %0, %0, %5;\n\t"
        "subc.cc.u32 %1, %1, 0;\n\t"
        "subc.cc.u32 %2, %2, 0;\n\t"
        "subc.cc.u32 %3, %3, 0;\n\t"
        "subc.u32    %4, 0, 0;"
        : "+r"(d0), "+r"(d1), "+r"(d2), "+r"(d3), "=r"(bw)
        : "r"(f));
    const uint32_t f2 = bw & C;         // second borrow: the value is >= 2^128 - C (words 1..3 all ones)
    asm("sub.cc.u32  %0, %0, %2;\n\t"
        "subc.u32    %1, %1, 0;"
        : "+r"(d0), "+r"(d1)
        : "r"(f2));
    return U128{{d0, d1, d2, d3}};
}

// a + t and a - t (mod Q) for any a < 2^128 and t < Q = 2^128 - C (psm_mul's results): one fold
// suffices.  a + t - 2^128 + C <= (2^128 - 1) + (Q - 1) - 2^128 + C = 2^128 - 2: no second carry;
// a - t + 2^128 - C >= 2^128 - (Q - 1) - C = 1: no second borrow.
__device__ __forceinline__ U128 psm_add1(const U128& a, const U128& t, uint32_t C) {
    uint32_t s0, s1, s2, s3, k;
    asm("add.cc.u32  %0, %5, %9;\n\t"
        "addc.cc.u32 %1, %6, %10;\n\t"
        "addc.cc.u32 %2, %7, %11;\n\t"
        "addc.cc.u32 %3, %8, %12;\n\t"
        "addc.u32    %4, 0, 0;"
        : "=r"(s0), "=r"(s1), "=r"(s2), "=r"(s3), "=r"(k)
        : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(t.w[0]), "r"(t.w[1]), "r"(t.w[2]), "r"(t.w[3]));
    const uint32_t f = k ? C : 0u;
    asm("add.cc.u32  %0, %0, %4;\n\t"
        "addc.cc.u32 %1, %1, 0;\n\t"
        "addc.cc.u32 %2, %2, 0;\n\t"
        "addc.u32    %3, %3, 0;"
        : "+r"(s0), "+r"(s1), "+r"(s2), "+r"(s3)
        : "r"(f));
    return U128{{s0, s1, s2, s3}};
}
__device__ __forceinline__ U128 psm_sub1(const U128& a, const U128& t, uint32_t C) {
    uint32_t d0, d1, d2, d3, bw;
    asm("sub.cc.u32  %0, %5, %9;\n\t"
        "subc.cc.u32 %1, %6, %10;\n\t"
        "subc.cc.u32 %2, %7, %11;\n\t"
        "subc.cc.u32 %3, %8, %12;\n\t"
        "subc.u32    %4, 0, 0;"
        : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(d3), "=r"(bw)
        : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(t.w[0]), "r"(t.w[1]), "r"(t.w[2]), "r"(t.w[3]));
    const uint32_t f = bw ? C : 0u;
    asm("sub.cc.u32  %0, %0, %4;\n\t"
        "subc.cc.u32 %1, %1, 0;\n\t"
        "subc.cc.u32 %2, %2, 0;\n\t"
        "subc.u32    %3, %3, 0;"
        : "+r"(d0), "+r"(d1), "+r"(d2), "+r"(d3)
        : "r"(f));
    return U128{{d0, d1, d2, d3}};
}

// a * b (mod Q) for a < 2^128, b < q (a twiddle): the result is < Q.  The 4 x 4 schoolbook
// product is accumulated in two register-pair-aligned halves (every 64-bit partial product lands on an aligned pair, so
// each is one IMAD.WIDE with carry in / out): E collects a_i b_j with i + j even (words
// 0..7), O those with i + j odd (words 1..8 of the product, o[0] at word 1; the top word o7
// only ever holds carries).  P = E + 2^32 O, then the folds described in the header.
__device__ __forceinline__ U128 psm_mul(const U128& a, const U128& b, uint32_t C) {
    uint32_t e0, e1, e2, e3, e4, e5, e6, e7;
    uint32_t o0, o1, o2, o3, o4, o5, o6;
    // E: (a0 b0 | a0 b2 | a1 b3 | a3 b3) fresh, then + (a1 b1 | a2 b2) and + (a2 b0 | a3 b1) at pairs 2, 4
    asm("{\n\t.reg .u64 p;\n\t"
        "mul.wide.u32 p, %8, %12;\n\tmov.b64 {%0, %1}, p;\n\t"
        "mul.wide.u32 p, %8, %14;\n\tmov.b64 {%2, %3}, p;\n\t"
        "mul.wide.u32 p, %9, %15;\n\tmov.b64 {%4, %5}, p;\n\t"
        "mul.wide.u32 p, %11, %15;\n\tmov.b64 {%6, %7}, p;\n\t"
        "mad.lo.cc.u32  %2, %9, %13, %2;\n\t"
        "madc.hi.cc.u32 %3, %9, %13, %3;\n\t"
        "madc.lo.cc.u32 %4, %10, %14, %4;\n\t"
        "madc.hi.cc.u32 %5, %10, %14, %5;\n\t"
        "addc.cc.u32    %6, %6, 0;\n\t"
        "addc.u32       %7, %7, 0;\n\t"
        "mad.lo.cc.u32  %2, %10, %12, %2;\n\t"
        "madc.hi.cc.u32 %3, %10, %12, %3;\n\t"
        "madc.lo.cc.u32 %4, %11, %13, %4;\n\t"
        "madc.hi.cc.u32 %5, %11, %13, %5;\n\t"
        "addc.cc.u32    %6, %6, 0;\n\t"
        "addc.u32       %7, %7, 0;\n\t}"
        : "=&r"(e0), "=&r"(e1), "=&r"(e2), "=&r"(e3), "=&r"(e4), "=&r"(e5), "=&r"(e6), "=&r"(e7)
        : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]), "r"(b.w[3]));
    // O (word 1 based): (a0 b1 | a0 b3 | a2 b3) fresh at pairs 0, 2, 4; + (a1 b0 | a1 b2 | a3 b2);
    // + (a2 b1) and + (a3 b0) at pair 2 with the carry run through pair 4 and o6
    asm("{\n\t.reg .u64 p;\n\t"
        "mul.wide.u32 p, %7, %12;\n\tmov.b64 {%0, %1}, p;\n\t"
        "mul.wide.u32 p, %7, %14;\n\tmov.b64 {%2, %3}, p;\n\t"
        "mul.wide.u32 p, %9, %14;\n\tmov.b64 {%4, %5}, p;\n\t"
        "mad.lo.cc.u32  %0, %8, %11, %0;\n\t"
        "madc.hi.cc.u32 %1, %8, %11, %1;\n\t"
        "madc.lo.cc.u32 %2, %8, %13, %2;\n\t"
        "madc.hi.cc.u32 %3, %8, %13, %3;\n\t"
        "madc.lo.cc.u32 %4, %10, %13, %4;\n\t"
        "madc.hi.cc.u32 %5, %10, %13, %5;\n\t"
        "addc.u32       %6, 0, 0;\n\t"
        "mad.lo.cc.u32  %2, %9, %12, %2;\n\t"
        "madc.hi.cc.u32 %3, %9, %12, %3;\n\t"
        "addc.cc.u32    %4, %4, 0;\n\t"
        "addc.cc.u32    %5, %5, 0;\n\t"
        "addc.u32       %6, %6, 0;\n\t"
        "mad.lo.cc.u32  %2, %10, %11, %2;\n\t"
        "madc.hi.cc.u32 %3, %10, %11, %3;\n\t"
        "addc.cc.u32    %4, %4, 0;\n\t"
        "addc.cc.u32    %5, %5, 0;\n\t"
        "addc.u32       %6, %6, 0;\n\t}"
        : "=&r"(o0), "=&r"(o1), "=&r"(o2), "=&r"(o3), "=&r"(o4), "=&r"(o5), "=&r"(o6)
        : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]), "r"(b.w[3]));
    // P = E + 2^32 O (P < 2^256: no carry out of word 7)
    asm("add.cc.u32  %0, %0, %7;\n\t"
        "addc.cc.u32 %1, %1, %8;\n\t"
        "addc.cc.u32 %2, %2, %9;\n\t"
        "addc.cc.u32 %3, %3, %10;\n\t"
        "addc.cc.u32 %4, %4, %11;\n\t"
        "addc.cc.u32 %5, %5, %12;\n\t"
        "addc.u32    %6, %6, %13;"
        : "+r"(e1), "+r"(e2), "+r"(e3), "+r"(e4), "+r"(e5), "+r"(e6), "+r"(e7)
        : "r"(o0), "r"(o1), "r"(o2), "r"(o3), "r"(o4), "r"(o5), "r"(o6));
    // first fold: L + H C with H = (e4..e7): even words of H onto pairs 0, 2; odd ones onto words 1..4.
    // L + H C < 2^128 + (2^128 - 2)(2^32 - 1) < 2^160: the fifth word l4 holds it all.
    uint32_t l4;
    asm("mad.lo.cc.u32  %0, %5, %9, %0;\n\t"
        "madc.hi.cc.u32 %1, %5, %9, %1;\n\t"
        "madc.lo.cc.u32 %2, %7, %9, %2;\n\t"
        "madc.hi.cc.u32 %3, %7, %9, %3;\n\t"
        "addc.u32       %4, 0, 0;\n\t"
        "mad.lo.cc.u32  %1, %6, %9, %1;\n\t"
        "madc.hi.cc.u32 %2, %6, %9, %2;\n\t"
        "madc.lo.cc.u32 %3, %8, %9, %3;\n\t"
        "madc.hi.u32    %4, %8, %9, %4;"
        : "+r"(e0), "+r"(e1), "+r"(e2), "+r"(e3), "=&r"(l4)
        : "r"(e4), "r"(e5), "r"(e6), "r"(e7), "r"(C));
    // second fold with the quotient estimate l4 + 1: y = L' + l4 C < 2^128 + 2^64 is the value modulo
    // Q up to one subtraction of Q = 2^128 - C, and y >= Q exactly when z = y + C = L' + (l4 + 1) C
    // carries out of 128 bits.  Carry: z - 2^128 = y - Q is the result; no carry: undo the + C.
    // Either way the result is < Q, which lets the butterfly's add / sub fold only once.
    // (l4 <= C: H <= q - 1 because b < q, so H C + L < 2^128 (C + 1); the host excludes C = 2^32 - 1.)
    uint32_t k;
    const uint32_t m = l4 + 1u;
    asm("mad.lo.cc.u32  %0, %5, %6, %0;\n\t"
        "madc.hi.cc.u32 %1, %5, %6, %1;\n\t"
        "addc.cc.u32    %2, %2, 0;\n\t"
        "addc.cc.u32    %3, %3, 0;\n\t"
        "addc.u32       %4, 0, 0;"
        : "+r"(e0), "+r"(e1), "+r"(e2), "+r"(e3), "=r"(k)
        : "r"(m), "r"(C));
    const uint32_t f = k ? 0u : C;   // no carry: subtract the C again (cannot borrow: y >= 0)
    asm("sub.cc.u32  %0, %0, %4;\n\t"
        "subc.cc.u32 %1, %1, 0;\n\t"
        "subc.cc.u32 %2, %2, 0;\n\t"
        "subc.u32    %3, %3, 0;"
        : "+r"(e0), "+r"(e1), "+r"(e2), "+r"(e3)
        : "r"(f));
    return U128{{e0, e1, e2, e3}};
}

// Any 128-bit representative -> the canonical residue in [0, q), q = 2^b - c, s = 128 - b,
// c = C >> s: v = vh 2^b + vl with vh < 2^s, so v = vl + vh c (mod q) < 2^b + 2^32, and one
// conditional subtraction of q finishes (vl + vh c - q < c + 2^32 < q).  s = 0: vh = 0.
__device__ __forceinline__ U128 psm_canon(const U128& v, const uint32_t q[4], uint32_t s, uint32_t C) {
    const uint32_t vh = __funnelshift_l(v.w[3], 0u, s);      // v.w[3] >> (32 - s), 0 when s == 0
    const uint32_t top = v.w[3] & (0xffffffffu >> s);
    const uint32_t add = vh * (C >> s);
    U128 r;
    asm("add.cc.u32  %0, %4, %8;\n\t"
        "addc.cc.u32 %1, %5, 0;\n\t"
        "addc.cc.u32 %2, %6, 0;\n\t"
        "addc.u32    %3, %7, 0;"
        : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3])
        : "r"(v.w[0]), "r"(v.w[1]), "r"(v.w[2]), "r"(top), "r"(add));
    return reduce_2q(r, q);
}

}  // namespace ntt128
