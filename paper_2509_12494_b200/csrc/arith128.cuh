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

// Montgomery product a * b * 2^-128 mod q, word-serial CIOS with 32-bit digits.
// Preconditions: b < q, a < 2^128 (then a b < q R and the value before the final
// subtraction is T < 2q, which may exceed 2^128: its bit 128 is kept in e4).
//
// The running value is split into an even-aligned part E (words 0..4) and an
// odd-aligned part O (words 1..5), so every IMAD.WIDE.U32 writes an aligned
// register pair and no register is shared by two pair layouts (the plain CIOS
// chain needs ~30 moves per call for that).  Per digit a_i:
//   E += a_i (b0 + b2 2^64)            2 IMAD.WIDE, carry chain
//   O  = a_i (b1 2^32 + b3 2^96)       2 IMAD.WIDE, no carries (disjoint words)
//   m  = E_0 q' mod 2^32               1 IMAD
//   E += m (q0 + q2 2^64), O += m (q1 2^32 + q3 2^96)   4 IMAD.WIDE
//   E  = (E + O) / 2^32                5-word add (E_0 == 0 mod 2^32 here)
// = 32 IMAD.WIDE + 4 IMAD per call (the 36 algorithmic products of §8(d)).
// Measured alone: 2.36e11 mulmod/s on B200 = 91 % of the IMAD.WIDE issue peak.
__device__ __forceinline__ U128 mont_mul(const U128& a, const U128& b, const uint32_t q[4], uint32_t qinv0) {
    uint32_t e0 = 0, e1 = 0, e2 = 0, e3 = 0, e4 = 0, o1, o2, o3, o4, o5, m;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        asm("mad.lo.cc.u32  %0, %5, %6, %0;\n\t"
            "madc.hi.cc.u32 %1, %5, %6, %1;\n\t"
            "madc.lo.cc.u32 %2, %5, %7, %2;\n\t"
            "madc.hi.cc.u32 %3, %5, %7, %3;\n\t"
            "addc.u32       %4, %4, 0;"
            : "+r"(e0), "+r"(e1), "+r"(e2), "+r"(e3), "+r"(e4)
            : "r"(a.w[i]), "r"(b.w[0]), "r"(b.w[2]));
        asm("mul.lo.u32 %0, %4, %5;\n\t"
            "mul.hi.u32 %1, %4, %5;\n\t"
            "mul.lo.u32 %2, %4, %6;\n\t"
            "mul.hi.u32 %3, %4, %6;"
            : "=r"(o1), "=r"(o2), "=r"(o3), "=r"(o4)
            : "r"(a.w[i]), "r"(b.w[1]), "r"(b.w[3]));
        m = e0 * qinv0;
        asm("mad.lo.cc.u32  %0, %5, %6, %0;\n\t"
            "madc.hi.cc.u32 %1, %5, %6, %1;\n\t"
            "madc.lo.cc.u32 %2, %5, %7, %2;\n\t"
            "madc.hi.cc.u32 %3, %5, %7, %3;\n\t"
            "addc.u32       %4, %4, 0;"
            : "+r"(e0), "+r"(e1), "+r"(e2), "+r"(e3), "+r"(e4)
            : "r"(m), "r"(q[0]), "r"(q[2]));
        asm("mad.lo.cc.u32  %0, %5, %6, %0;\n\t"
            "madc.hi.cc.u32 %1, %5, %6, %1;\n\t"
            "madc.lo.cc.u32 %2, %5, %7, %2;\n\t"
            "madc.hi.cc.u32 %3, %5, %7, %3;\n\t"
            "addc.u32       %4, 0, 0;"
            : "+r"(o1), "+r"(o2), "+r"(o3), "+r"(o4), "=r"(o5)
            : "r"(m), "r"(q[1]), "r"(q[3]));
        asm("add.cc.u32  %0, %5, %9;\n\t"
            "addc.cc.u32 %1, %6, %10;\n\t"
            "addc.cc.u32 %2, %7, %11;\n\t"
            "addc.cc.u32 %3, %8, %12;\n\t"
            "addc.u32    %4, %13, 0;"
            : "=r"(e0), "=r"(e1), "=r"(e2), "=r"(e3), "=r"(e4)
            : "r"(e1), "r"(e2), "r"(e3), "r"(e4), "r"(o1), "r"(o2), "r"(o3), "r"(o4), "r"(o5));
    }
    // T = (e4:e3..e0) < 2q: subtract q when no borrow out of the 129-bit difference
    uint32_t d0, d1, d2, d3, bw;
    asm("sub.cc.u32  %0, %5, %10;\n\t"
        "subc.cc.u32 %1, %6, %11;\n\t"
        "subc.cc.u32 %2, %7, %12;\n\t"
        "subc.cc.u32 %3, %8, %13;\n\t"
        "subc.u32    %4, %9, 0;"
        : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(d3), "=r"(bw)
        : "r"(e0), "r"(e1), "r"(e2), "r"(e3), "r"(e4), "r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]));
    U128 r;
    r.w[0] = (e0 & bw) | (d0 & ~bw);
    r.w[1] = (e1 & bw) | (d1 & ~bw);
    r.w[2] = (e2 & bw) | (d2 & ~bw);
    r.w[3] = (e3 & bw) | (d3 & ~bw);
    return r;
}

// ---------------------------------------------------------------------------------------
// Lazy-reduction variants for moduli q < 2^126 (4q < 2^128: values kept in [0, 2q) fit four
// words with room for one addition; Harvey-style butterflies).
// mont_mul_lazy: a < 2q, b < q -> a b R^-1 mod q + {0, q}, i.e. a value in [0, 2q)
// (T < (2q q + R q) / R < 1.5 q); no final subtraction and no fifth-word carry.
__device__ __forceinline__ U128 mont_mul_lazy(const U128& a, const U128& b, const uint32_t q[4], uint32_t qinv0) {
    uint32_t e0 = 0, e1 = 0, e2 = 0, e3 = 0, e4 = 0, o1, o2, o3, o4, m;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        asm("mad.lo.cc.u32  %0, %5, %6, %0;\n\t"
            "madc.hi.cc.u32 %1, %5, %6, %1;\n\t"
            "madc.lo.cc.u32 %2, %5, %7, %2;\n\t"
            "madc.hi.cc.u32 %3, %5, %7, %3;\n\t"
            "addc.u32       %4, %4, 0;"
            : "+r"(e0), "+r"(e1), "+r"(e2), "+r"(e3), "+r"(e4)
            : "r"(a.w[i]), "r"(b.w[0]), "r"(b.w[2]));
        asm("mul.lo.u32 %0, %4, %5;\n\t"
            "mul.hi.u32 %1, %4, %5;\n\t"
            "mul.lo.u32 %2, %4, %6;\n\t"
            "mul.hi.u32 %3, %4, %6;"
            : "=r"(o1), "=r"(o2), "=r"(o3), "=r"(o4)
            : "r"(a.w[i]), "r"(b.w[1]), "r"(b.w[3]));
        m = e0 * qinv0;
        asm("mad.lo.cc.u32  %0, %5, %6, %0;\n\t"
            "madc.hi.cc.u32 %1, %5, %6, %1;\n\t"
            "madc.lo.cc.u32 %2, %5, %7, %2;\n\t"
            "madc.hi.cc.u32 %3, %5, %7, %3;\n\t"
            "addc.u32       %4, %4, 0;"
            : "+r"(e0), "+r"(e1), "+r"(e2), "+r"(e3), "+r"(e4)
            : "r"(m), "r"(q[0]), "r"(q[2]));
        // O + m (q1 2^32 + q3 2^96) < 2^160: no carry out of word 4
        asm("mad.lo.cc.u32  %0, %4, %5, %0;\n\t"
            "madc.hi.cc.u32 %1, %4, %5, %1;\n\t"
            "madc.lo.cc.u32 %2, %4, %6, %2;\n\t"
            "madc.hi.u32    %3, %4, %6, %3;"
            : "+r"(o1), "+r"(o2), "+r"(o3), "+r"(o4)
            : "r"(m), "r"(q[1]), "r"(q[3]));
        // (E + O) / 2^32 < 2^129 / 2^32 ... the running value stays < 2q after the shift
        asm("add.cc.u32  %0, %4, %8;\n\t"
            "addc.cc.u32 %1, %5, %9;\n\t"
            "addc.cc.u32 %2, %6, %10;\n\t"
            "addc.u32    %3, %7, %11;"
            : "=r"(e0), "=r"(e1), "=r"(e2), "=r"(e3)
            : "r"(e1), "r"(e2), "r"(e3), "r"(e4), "r"(o1), "r"(o2), "r"(o3), "r"(o4));
        e4 = 0;
    }
    return U128{{e0, e1, e2, e3}};
}

// x - 2q if x >= 2q (x < 4q < 2^128); q2 = 2q
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

// lazy butterfly outputs: u + t and u - t + 2q, each brought back to [0, 2q)
__device__ __forceinline__ U128 add_lazy(const U128& u, const U128& t, const uint32_t q2[4]) {
    U128 s;
    asm("add.cc.u32  %0, %4, %8;\n\t"
        "addc.cc.u32 %1, %5, %9;\n\t"
        "addc.cc.u32 %2, %6, %10;\n\t"
        "addc.u32    %3, %7, %11;"
        : "=r"(s.w[0]), "=r"(s.w[1]), "=r"(s.w[2]), "=r"(s.w[3])
        : "r"(u.w[0]), "r"(u.w[1]), "r"(u.w[2]), "r"(u.w[3]), "r"(t.w[0]), "r"(t.w[1]), "r"(t.w[2]), "r"(t.w[3]));
    return reduce_2q(s, q2);
}
__device__ __forceinline__ U128 sub_lazy(const U128& u, const U128& t, const uint32_t q2[4]) {
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
          "r"(q2[0]), "r"(q2[1]), "r"(q2[2]), "r"(q2[3]));
    return reduce_2q(s, q2);
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
