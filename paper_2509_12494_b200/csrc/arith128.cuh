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
// mulmod is Montgomery (R = 2^128, word-serial CIOS): the paper's Barrett
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
// Preconditions: b < q, a < 2^128 (then a b < q R and the result before the final
// subtraction is < 2q, which may exceed 2^128: it is kept in t4).  Result < q.
// Per call: 32 IMAD.WIDE.U32 (16 of a_i*b_j, 16 of m_i*q_j) + 4 IMAD (m_i).
__device__ __forceinline__ U128 mont_mul(const U128& a, const U128& b, const uint32_t q[4], uint32_t qinv0) {
    uint32_t t0 = 0, t1 = 0, t2 = 0, t3 = 0, t4 = 0, t5, m;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        // (t5:t4..t0) += a_i * b   (even-word products, then odd-word products)
        asm("mad.lo.cc.u32  %0, %6, %7, %0;\n\t"
            "madc.hi.cc.u32 %1, %6, %7, %1;\n\t"
            "madc.lo.cc.u32 %2, %6, %9, %2;\n\t"
            "madc.hi.cc.u32 %3, %6, %9, %3;\n\t"
            "addc.u32       %4, %4, 0;\n\t"
            "mad.lo.cc.u32  %1, %6, %8, %1;\n\t"
            "madc.hi.cc.u32 %2, %6, %8, %2;\n\t"
            "madc.lo.cc.u32 %3, %6, %10, %3;\n\t"
            "madc.hi.cc.u32 %4, %6, %10, %4;\n\t"
            "addc.u32       %5, 0, 0;"
            : "+r"(t0), "+r"(t1), "+r"(t2), "+r"(t3), "+r"(t4), "=r"(t5)
            : "r"(a.w[i]), "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]), "r"(b.w[3]));
        m = t0 * qinv0;
        // (t5..t0) += m * q; afterwards t0 == 0 and the value is shifted down a word
        asm("mad.lo.cc.u32  %0, %6, %7, %0;\n\t"
            "madc.hi.cc.u32 %1, %6, %7, %1;\n\t"
            "madc.lo.cc.u32 %2, %6, %9, %2;\n\t"
            "madc.hi.cc.u32 %3, %6, %9, %3;\n\t"
            "addc.cc.u32    %4, %4, 0;\n\t"
            "addc.u32       %5, %5, 0;\n\t"
            "mad.lo.cc.u32  %1, %6, %8, %1;\n\t"
            "madc.hi.cc.u32 %2, %6, %8, %2;\n\t"
            "madc.lo.cc.u32 %3, %6, %10, %3;\n\t"
            "madc.hi.cc.u32 %4, %6, %10, %4;\n\t"
            "addc.u32       %5, %5, 0;"
            : "+r"(t0), "+r"(t1), "+r"(t2), "+r"(t3), "+r"(t4), "+r"(t5)
            : "r"(m), "r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]));
        t0 = t1; t1 = t2; t2 = t3; t3 = t4; t4 = t5;
    }
    // (t4:t3..t0) < 2q: subtract q when no borrow out of the 129-bit difference
    uint32_t d0, d1, d2, d3, bw;
    asm("sub.cc.u32  %0, %5, %10;\n\t"
        "subc.cc.u32 %1, %6, %11;\n\t"
        "subc.cc.u32 %2, %7, %12;\n\t"
        "subc.cc.u32 %3, %8, %13;\n\t"
        "subc.u32    %4, %9, 0;"
        : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(d3), "=r"(bw)
        : "r"(t0), "r"(t1), "r"(t2), "r"(t3), "r"(t4), "r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]));
    U128 r;
    r.w[0] = (t0 & bw) | (d0 & ~bw);
    r.w[1] = (t1 & bw) | (d1 & ~bw);
    r.w[2] = (t2 & bw) | (d2 & ~bw);
    r.w[3] = (t3 & bw) | (d3 & ~bw);
    return r;
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
