// arith_variants.cuh -- arithmetic variants measured and NOT adopted (the
// mulmod-variant study): the merge-every-digit CIOS and Shoup products by a constant.
// Micro-benchmark use only; the product library does not include this file.
#pragma once
#include "../../paper_2509_12494_b200/csrc/arith128.cuh"

namespace ntt128 {

// Previous formulation (one accumulator pair merged every digit), kept for the
// microbenchmark comparison in tools/micro/bfly_rate.cu.
__device__ __forceinline__ U128 mont_mul_v1(const U128& a, const U128& b, const uint32_t q[4], uint32_t qinv0) {
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

// ---- Shoup product by a plan constant, lazy class (q < 2^126; DESIGN.md §5 "Shoup").
// w < q plain (not Montgomery form), wp = floor(w 2^128 / q) precomputed.  The quotient
// estimate qh = floor(v wp / 2^128) is computed from the 13 word products at positions >= 2
// only (the 3 dropped ones sum to < 2^99 < 2^128, so qh is short by at most 1); then
// r = v w - qh q = lo128(v w) + lo128(qh (2^128 - q)) lies in [0, 3q) (Shoup's [0, 2q) plus
// at most one q) for any v < 2^128, and one conditional subtraction of 2q gives [0, 2q).
// 25 IMAD.WIDE + 8 IMAD against 32 + 4 for mont_mul_lazy (8.7 % more products/s measured,
// tools/micro/shoup_rate.cu).
// words 4..7 of the sum of the 13 partial products a_i b_j with i + j >= 2
__device__ __forceinline__ void mulhi128_trunc(uint32_t h[4], const uint32_t a[4], const uint32_t b[4]) {
    asm("{\n\t.reg .u32 t2, t3;\n\t"
        // row a0: b2 -> (2,3), b3 -> (3,4)
        "mul.lo.u32 t2, %4, %10;\n\t mul.hi.u32 t3, %4, %10;\n\t"
        "mad.lo.cc.u32 t3, %4, %11, t3;\n\t madc.hi.u32 %0, %4, %11, 0;\n\t"
        // row a1: b1 -> (2,3), b3 -> (4,5); then b2 -> (3,4)
        "mad.lo.cc.u32 t2, %5, %9, t2;\n\t madc.hi.cc.u32 t3, %5, %9, t3;\n\t madc.lo.cc.u32 %0, %5, %11, %0;\n\t"
        "madc.hi.cc.u32 %1, %5, %11, 0;\n\t addc.u32 %2, 0, 0;\n\t"
        "mad.lo.cc.u32 t3, %5, %10, t3;\n\t madc.hi.cc.u32 %0, %5, %10, %0;\n\t addc.cc.u32 %1, %1, 0;\n\t addc.u32 %2, %2, 0;\n\t"
        // row a2: b0 -> (2,3), b2 -> (4,5); b1 -> (3,4), b3 -> (5,6)
        "mad.lo.cc.u32 t2, %6, %8, t2;\n\t madc.hi.cc.u32 t3, %6, %8, t3;\n\t madc.lo.cc.u32 %0, %6, %10, %0;\n\t"
        "madc.hi.cc.u32 %1, %6, %10, %1;\n\t addc.cc.u32 %2, %2, 0;\n\t addc.u32 %3, 0, 0;\n\t"
        "mad.lo.cc.u32 t3, %6, %9, t3;\n\t madc.hi.cc.u32 %0, %6, %9, %0;\n\t madc.lo.cc.u32 %1, %6, %11, %1;\n\t"
        "madc.hi.cc.u32 %2, %6, %11, %2;\n\t addc.u32 %3, %3, 0;\n\t"
        // row a3: b0 -> (3,4), b2 -> (5,6); b1 -> (4,5), b3 -> (6,7)
        "mad.lo.cc.u32 t3, %7, %8, t3;\n\t madc.hi.cc.u32 %0, %7, %8, %0;\n\t madc.lo.cc.u32 %1, %7, %10, %1;\n\t"
        "madc.hi.cc.u32 %2, %7, %10, %2;\n\t addc.u32 %3, %3, 0;\n\t"
        "mad.lo.cc.u32 %0, %7, %9, %0;\n\t madc.hi.cc.u32 %1, %7, %9, %1;\n\t madc.lo.cc.u32 %2, %7, %11, %2;\n\t"
        "madc.hi.u32 %3, %7, %11, %3;\n\t}"
        : "=&r"(h[0]), "=&r"(h[1]), "=&r"(h[2]), "=&r"(h[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]));
}
// low 128 bits of a b + c d (12 IMAD.WIDE + 8 IMAD)
__device__ __forceinline__ void mullo128_sum(uint32_t r[4], const uint32_t a[4], const uint32_t b[4], const uint32_t c[4],
                                             const uint32_t d[4]) {
    asm("mul.lo.u32 %0, %4, %8;\n\t mul.hi.u32 %1, %4, %8;\n\t mul.lo.u32 %2, %4, %10;\n\t mul.hi.u32 %3, %4, %10;\n\t"
        "mad.lo.cc.u32 %1, %4, %9, %1;\n\t madc.hi.cc.u32 %2, %4, %9, %2;\n\t madc.lo.u32 %3, %4, %11, %3;\n\t"
        "mad.lo.cc.u32 %1, %5, %8, %1;\n\t madc.hi.cc.u32 %2, %5, %8, %2;\n\t madc.lo.u32 %3, %5, %10, %3;\n\t"
        "mad.lo.cc.u32 %2, %5, %9, %2;\n\t madc.hi.u32 %3, %5, %9, %3;\n\t"
        "mad.lo.cc.u32 %2, %6, %8, %2;\n\t madc.hi.u32 %3, %6, %8, %3;\n\t"
        "mad.lo.u32 %3, %6, %9, %3;\n\t mad.lo.u32 %3, %7, %8, %3;\n\t"
        "mad.lo.cc.u32 %0, %12, %16, %0;\n\t madc.hi.cc.u32 %1, %12, %16, %1;\n\t madc.lo.cc.u32 %2, %12, %18, %2;\n\t"
        "madc.hi.u32 %3, %12, %18, %3;\n\t"
        "mad.lo.cc.u32 %1, %12, %17, %1;\n\t madc.hi.cc.u32 %2, %12, %17, %2;\n\t madc.lo.u32 %3, %12, %19, %3;\n\t"
        "mad.lo.cc.u32 %1, %13, %16, %1;\n\t madc.hi.cc.u32 %2, %13, %16, %2;\n\t madc.lo.u32 %3, %13, %18, %3;\n\t"
        "mad.lo.cc.u32 %2, %13, %17, %2;\n\t madc.hi.u32 %3, %13, %17, %3;\n\t"
        "mad.lo.cc.u32 %2, %14, %16, %2;\n\t madc.hi.u32 %3, %14, %16, %3;\n\t"
        "mad.lo.u32 %3, %14, %17, %3;\n\t mad.lo.u32 %3, %15, %16, %3;"
        : "=&r"(r[0]), "=&r"(r[1]), "=&r"(r[2]), "=&r"(r[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]),
          "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(d[0]), "r"(d[1]), "r"(d[2]), "r"(d[3]));
}
// v w mod q in [0, 2q): v < 2^128, w < q < 2^126, wp = floor(w 2^128 / q), qn = 2^128 - q, q2 = 2q
__device__ __forceinline__ U128 shoup_mul_lazy(const U128& v, const U128& w, const U128& wp, const uint32_t qn[4],
                                               const uint32_t q2[4]) {
    uint32_t h[4], r[4];
    mulhi128_trunc(h, v.w, wp.w);
    mullo128_sum(r, v.w, w.w, h, qn);
    return reduce_2q(U128{{r[0], r[1], r[2], r[3]}}, q2);
}

}  // namespace ntt128
