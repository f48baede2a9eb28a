// barrett128.cuh -- general 128-bit modular product a * b mod q by Barrett reduction
// (Eq. barrett; HAC Algorithm 14.42 with base 2^32, k = 4 words),
// for q in (2^127, 2^128): mu = floor(2^256 / q) = 2^128 + mu' with mu' < 2^128.
//
//   P  = a b                         (16 word products, 256 bits)
//   q1 = floor(P / 2^96)             (5 words)
//   q2 = q1 mu = q1 mu' + q1 2^128   (q1 mu' truncated: products at word positions < 3
//                                     dropped -> q3 below exact or one short)
//   q3 = floor(q2 / 2^160)           (Q - q3 <= 3 for Q = floor(P / q))
//   r  = (P - q3 q) mod 2^160 in [0, 4q), then up to three subtractions of q.
// = 16 + 14 + 13 word products (40 wide + 3 low) against 64 wide + 8 low for the two
// Montgomery products (x y R^-1, then * R^2) it replaces in vec128_mul.
//
// Written as portable host/device C++ on 64-bit limbs of 32-bit words, so the same code
// is exercised on the CPU by tests/test_barrett_host.py (against Python integers) and
// compiled for sm_100a (nvcc emits IMAD.WIDE.U32 for the 32x32->64 products).
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define B128_HD __host__ __device__ __forceinline__
#else
#define B128_HD inline
#endif

namespace ntt128 {

struct BarrettC {
    uint32_t q[4];
    uint32_t mu[4];   // mu' = floor(2^256 / q) - 2^128
};

// r = a * b mod q (a, b < q, 2^127 < q < 2^128); all arrays little-endian 32-bit words.
B128_HD void barrett_mul(const uint32_t a[4], const uint32_t b[4], const BarrettC& c, uint32_t r[4]) {
    // ---- P = a b: product scanning, one 64-bit partial product at a time into a 96-bit column sum
    uint32_t P[8];
    {
        uint64_t lo = 0;      // running column sum, low 64 bits
        uint32_t hi = 0;      // bits 64..95
#pragma unroll
        for (int k = 0; k < 7; k++) {
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const int j = k - i;
                if (j < 0 || j > 3) continue;
                const uint64_t p = (uint64_t)a[i] * b[j];
                lo += p;
                hi += lo < p;
            }
            P[k] = (uint32_t)lo;
            lo = (lo >> 32) | ((uint64_t)hi << 32);
            hi = 0;
        }
        P[7] = (uint32_t)lo;
    }
    // ---- q3 = floor((q1 mu' [positions >= 3] + q1 2^128) / 2^160), q1 = P[3..7]
    uint32_t q3[4];
    {
        const uint32_t* q1 = P + 3;
        uint64_t lo = 0;
        uint32_t hi = 0;
        // columns 3 and 4 (word positions of q1 mu'): only their carry into column 5 matters
#pragma unroll
        for (int k = 3; k < 9; k++) {
#pragma unroll
            for (int i = 0; i < 5; i++) {
                const int j = k - i;
                if (j < 0 || j > 3) continue;
                const uint64_t p = (uint64_t)q1[i] * c.mu[j];
                lo += p;
                hi += lo < p;
            }
            if (k >= 4) {   // + q1 2^128: q1[k - 4] at column k
                const uint64_t p = q1[k - 4];
                lo += p;
                hi += lo < p;
            }
            if (k >= 5) q3[k - 5] = (uint32_t)lo;
            lo = (lo >> 32) | ((uint64_t)hi << 32);
            hi = 0;
        }
        // column 9 (above q3[3]) is zero: q3 <= Q = floor(P / q) < q < 2^128
    }
    // ---- r = (P - q3 q) mod 2^160
    uint32_t R[5];
    {
        uint64_t lo = 0;
        uint32_t hi = 0;
        uint32_t t[5];
#pragma unroll
        for (int k = 0; k < 5; k++) {
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const int j = k - i;
                if (j < 0 || j > 3) continue;
                const uint64_t p = (uint64_t)q3[i] * c.q[j];
                lo += p;
                hi += lo < p;
            }
            t[k] = (uint32_t)lo;
            lo = (lo >> 32) | ((uint64_t)hi << 32);
            hi = 0;
        }
        uint64_t borrow = 0;
#pragma unroll
        for (int k = 0; k < 5; k++) {
            const uint64_t d = (uint64_t)P[k] - t[k] - borrow;
            R[k] = (uint32_t)d;
            borrow = (d >> 32) & 1;
        }
    }
    // ---- up to three conditional subtractions of q (r < 4q < 2^130)
#pragma unroll
    for (int it = 0; it < 3; it++) {
        uint32_t d[5];
        uint64_t borrow = 0;
#pragma unroll
        for (int k = 0; k < 5; k++) {
            const uint64_t qk = k < 4 ? c.q[k] : 0;
            const uint64_t x = (uint64_t)R[k] - qk - borrow;
            d[k] = (uint32_t)x;
            borrow = (x >> 32) & 1;
        }
        const uint32_t keep = 0u - (uint32_t)borrow;   // all ones: R < q, keep R
#pragma unroll
        for (int k = 0; k < 5; k++) R[k] = (R[k] & keep) | (d[k] & ~keep);
    }
    r[0] = R[0];
    r[1] = R[1];
    r[2] = R[2];
    r[3] = R[3];
}

#if defined(__CUDACC__)
// The same algorithm on the device with explicit carry chains (PTX mad.lo.cc / madc.hi.cc
// pairs fuse into IMAD.WIDE.U32 with carry predicates; every 64-bit partial product sits
// at a register-pair-aligned position of an even- or odd-position accumulator, as in
// arith128.cuh's mont_core).  Bit-identical to barrett_mul (same q3, same corrections).
__device__ __forceinline__ void barrett_mul_dev(const uint32_t a[4], const uint32_t b[4], const BarrettC& c,
                                                uint32_t r[4]) {
    // ---- P = a b: E = even-position products (words 0..7), O = odd ones, O stored one word down
    uint32_t e0, e1, e2, e3, e4, e5, e6, e7, o0, o1, o2, o3, o4, o5, o6;
    asm("mul.lo.u32     %0, %15, %19;\n\t"
        "mul.hi.u32     %1, %15, %19;\n\t"
        "mul.lo.u32     %2, %15, %21;\n\t"
        "mul.hi.u32     %3, %15, %21;\n\t"
        "mad.lo.cc.u32  %2, %16, %20, %2;\n\t"
        "madc.hi.cc.u32 %3, %16, %20, %3;\n\t"
        "madc.lo.cc.u32 %4, %16, %22, 0;\n\t"
        "madc.hi.u32    %5, %16, %22, 0;\n\t"
        "mad.lo.cc.u32  %2, %17, %19, %2;\n\t"
        "madc.hi.cc.u32 %3, %17, %19, %3;\n\t"
        "madc.lo.cc.u32 %4, %17, %21, %4;\n\t"
        "madc.hi.cc.u32 %5, %17, %21, %5;\n\t"
        "addc.u32       %6, 0, 0;\n\t"
        "mad.lo.cc.u32  %4, %18, %20, %4;\n\t"
        "madc.hi.cc.u32 %5, %18, %20, %5;\n\t"
        "madc.lo.cc.u32 %6, %18, %22, %6;\n\t"
        "madc.hi.u32    %7, %18, %22, 0;\n\t"
        // O: word k of O is position k + 1
        "mul.lo.u32     %8, %15, %20;\n\t"
        "mul.hi.u32     %9, %15, %20;\n\t"
        "mul.lo.u32     %10, %15, %22;\n\t"
        "mul.hi.u32     %11, %15, %22;\n\t"
        "mad.lo.cc.u32  %8, %16, %19, %8;\n\t"
        "madc.hi.cc.u32 %9, %16, %19, %9;\n\t"
        "madc.lo.cc.u32 %10, %16, %21, %10;\n\t"
        "madc.hi.cc.u32 %11, %16, %21, %11;\n\t"
        "addc.u32       %12, 0, 0;\n\t"
        "mad.lo.cc.u32  %10, %17, %20, %10;\n\t"
        "madc.hi.cc.u32 %11, %17, %20, %11;\n\t"
        "madc.lo.cc.u32 %12, %17, %22, %12;\n\t"
        "madc.hi.u32    %13, %17, %22, 0;\n\t"
        "mad.lo.cc.u32  %10, %18, %19, %10;\n\t"
        "madc.hi.cc.u32 %11, %18, %19, %11;\n\t"
        "madc.lo.cc.u32 %12, %18, %21, %12;\n\t"
        "madc.hi.cc.u32 %13, %18, %21, %13;\n\t"
        "addc.u32       %14, 0, 0;"
        : "=&r"(e0), "=&r"(e1), "=&r"(e2), "=&r"(e3), "=&r"(e4), "=&r"(e5), "=&r"(e6), "=&r"(e7),
          "=&r"(o0), "=&r"(o1), "=&r"(o2), "=&r"(o3), "=&r"(o4), "=&r"(o5), "=&r"(o6)
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]));
    uint32_t P[8];
    P[0] = e0;
    asm("add.cc.u32  %0, %7, %14;\n\t"
        "addc.cc.u32 %1, %8, %15;\n\t"
        "addc.cc.u32 %2, %9, %16;\n\t"
        "addc.cc.u32 %3, %10, %17;\n\t"
        "addc.cc.u32 %4, %11, %18;\n\t"
        "addc.cc.u32 %5, %12, %19;\n\t"
        "addc.u32    %6, %13, %20;"
        : "=r"(P[1]), "=r"(P[2]), "=r"(P[3]), "=r"(P[4]), "=r"(P[5]), "=r"(P[6]), "=r"(P[7])
        : "r"(e1), "r"(e2), "r"(e3), "r"(e4), "r"(e5), "r"(e6), "r"(e7),
          "r"(o0), "r"(o1), "r"(o2), "r"(o3), "r"(o4), "r"(o5), "r"(o6));
    // ---- q3 = words 5..8 of (q1 mu' at positions >= 3) + q1 2^128, q1 = P[3..7]
    // F: even positions 4, 6 (words 4..9); G: odd positions 3, 5, 7 (words 3..8)
    uint32_t f4, f5, f6, f7, f8, g3, g4, g5, g6, g7, g8;
    asm("mul.lo.u32     %0, %12, %19;\n\t"          // (1,3) @4
        "mul.hi.u32     %1, %12, %19;\n\t"
        "mul.lo.u32     %2, %14, %19;\n\t"          // (3,3) @6
        "mul.hi.u32     %3, %14, %19;\n\t"
        "mad.lo.cc.u32  %0, %13, %18, %0;\n\t"      // (2,2) @4
        "madc.hi.cc.u32 %1, %13, %18, %1;\n\t"
        "madc.lo.cc.u32 %2, %15, %18, %2;\n\t"      // (4,2) @6
        "madc.hi.cc.u32 %3, %15, %18, %3;\n\t"
        "addc.u32       %4, 0, 0;\n\t"
        "mad.lo.cc.u32  %0, %14, %17, %0;\n\t"      // (3,1) @4
        "madc.hi.cc.u32 %1, %14, %17, %1;\n\t"
        "addc.cc.u32    %2, %2, 0;\n\t"
        "addc.cc.u32    %3, %3, 0;\n\t"
        "addc.u32       %4, %4, 0;\n\t"
        "mad.lo.cc.u32  %0, %15, %16, %0;\n\t"      // (4,0) @4
        "madc.hi.cc.u32 %1, %15, %16, %1;\n\t"
        "addc.cc.u32    %2, %2, 0;\n\t"
        "addc.cc.u32    %3, %3, 0;\n\t"
        "addc.u32       %4, %4, 0;\n\t"
        // + q1 2^128: q1[i] at word 4 + i
        "add.cc.u32     %0, %0, %11;\n\t"
        "addc.cc.u32    %1, %1, %12;\n\t"
        "addc.cc.u32    %2, %2, %13;\n\t"
        "addc.cc.u32    %3, %3, %14;\n\t"
        "addc.u32       %4, %4, %15;"
        : "=&r"(f4), "=&r"(f5), "=&r"(f6), "=&r"(f7), "=&r"(f8)
        : "r"(0), "r"(0), "r"(0), "r"(0), "r"(0), "r"(0),
          "r"(P[3]), "r"(P[4]), "r"(P[5]), "r"(P[6]), "r"(P[7]),
          "r"(c.mu[0]), "r"(c.mu[1]), "r"(c.mu[2]), "r"(c.mu[3]));
    asm("mul.lo.u32     %0, %6, %14;\n\t"           // (0,3) @3
        "mul.hi.u32     %1, %6, %14;\n\t"
        "mul.lo.u32     %2, %8, %14;\n\t"           // (2,3) @5
        "mul.hi.u32     %3, %8, %14;\n\t"
        "mul.lo.u32     %4, %10, %14;\n\t"          // (4,3) @7
        "mul.hi.u32     %5, %10, %14;\n\t"
        "mad.lo.cc.u32  %0, %7, %13, %0;\n\t"       // (1,2) @3
        "madc.hi.cc.u32 %1, %7, %13, %1;\n\t"
        "madc.lo.cc.u32 %2, %9, %13, %2;\n\t"       // (3,2) @5
        "madc.hi.cc.u32 %3, %9, %13, %3;\n\t"
        "addc.cc.u32    %4, %4, 0;\n\t"
        "addc.u32       %5, %5, 0;\n\t"
        "mad.lo.cc.u32  %0, %8, %12, %0;\n\t"       // (2,1) @3
        "madc.hi.cc.u32 %1, %8, %12, %1;\n\t"
        "madc.lo.cc.u32 %2, %10, %12, %2;\n\t"      // (4,1) @5
        "madc.hi.cc.u32 %3, %10, %12, %3;\n\t"
        "addc.cc.u32    %4, %4, 0;\n\t"
        "addc.u32       %5, %5, 0;\n\t"
        "mad.lo.cc.u32  %0, %9, %11, %0;\n\t"       // (3,0) @3
        "madc.hi.cc.u32 %1, %9, %11, %1;\n\t"
        "addc.cc.u32    %2, %2, 0;\n\t"
        "addc.cc.u32    %3, %3, 0;\n\t"
        "addc.cc.u32    %4, %4, 0;\n\t"
        "addc.u32       %5, %5, 0;"
        : "=&r"(g3), "=&r"(g4), "=&r"(g5), "=&r"(g6), "=&r"(g7), "=&r"(g8)
        : "r"(P[3]), "r"(P[4]), "r"(P[5]), "r"(P[6]), "r"(P[7]),
          "r"(c.mu[0]), "r"(c.mu[1]), "r"(c.mu[2]), "r"(c.mu[3]));
    uint32_t s0, s1, s2, s3;   // q3 = (F + G) words 5..8 (word 3 is g3 alone; carry from word 4)
    asm("{\n\t.reg .u32 t4;\n\t"
        "add.cc.u32  t4, %4, %9;\n\t"
        "addc.cc.u32 %0, %5, %10;\n\t"
        "addc.cc.u32 %1, %6, %11;\n\t"
        "addc.cc.u32 %2, %7, %12;\n\t"
        "addc.u32    %3, %8, %13;\n\t}"
        : "=r"(s0), "=r"(s1), "=r"(s2), "=r"(s3)
        : "r"(f4), "r"(f5), "r"(f6), "r"(f7), "r"(f8), "r"(g4), "r"(g5), "r"(g6), "r"(g7), "r"(g8));
    // ---- t = q3 q mod 2^160: U = even positions (0, 2, 4), V = odd (1, 3) -> R = P - U - V
    uint32_t u0, u1, u2, u3, u4, v1, v2, v3, v4;
    asm("mul.lo.u32     %0, %9, %13;\n\t"           // (0,0) @0
        "mul.hi.u32     %1, %9, %13;\n\t"
        "mul.lo.u32     %2, %9, %15;\n\t"           // (0,2) @2
        "mul.hi.u32     %3, %9, %15;\n\t"
        "mad.lo.cc.u32  %2, %10, %14, %2;\n\t"      // (1,1) @2
        "madc.hi.cc.u32 %3, %10, %14, %3;\n\t"
        "madc.lo.u32    %4, %10, %16, 0;\n\t"       // (1,3) @4, low word only
        "mad.lo.cc.u32  %2, %11, %13, %2;\n\t"      // (2,0) @2
        "madc.hi.cc.u32 %3, %11, %13, %3;\n\t"
        "madc.lo.u32    %4, %11, %15, %4;\n\t"      // (2,2) @4
        "mad.lo.u32     %4, %12, %14, %4;\n\t"      // (3,1) @4
        "mul.lo.u32     %5, %9, %14;\n\t"           // (0,1) @1
        "mul.hi.u32     %6, %9, %14;\n\t"
        "mul.lo.u32     %7, %9, %16;\n\t"           // (0,3) @3
        "mul.hi.u32     %8, %9, %16;\n\t"
        "mad.lo.cc.u32  %5, %10, %13, %5;\n\t"      // (1,0) @1
        "madc.hi.cc.u32 %6, %10, %13, %6;\n\t"
        "madc.lo.cc.u32 %7, %10, %15, %7;\n\t"      // (1,2) @3
        "madc.hi.u32    %8, %10, %15, %8;\n\t"
        "mad.lo.cc.u32  %7, %11, %14, %7;\n\t"      // (2,1) @3
        "madc.hi.u32    %8, %11, %14, %8;\n\t"
        "mad.lo.cc.u32  %7, %12, %13, %7;\n\t"      // (3,0) @3
        "madc.hi.u32    %8, %12, %13, %8;"
        : "=&r"(u0), "=&r"(u1), "=&r"(u2), "=&r"(u3), "=&r"(u4), "=&r"(v1), "=&r"(v2), "=&r"(v3), "=&r"(v4)
        : "r"(s0), "r"(s1), "r"(s2), "r"(s3), "r"(c.q[0]), "r"(c.q[1]), "r"(c.q[2]), "r"(c.q[3]));
    uint32_t R0, R1, R2, R3, R4;
    asm("{\n\t.reg .u32 w1, w2, w3, w4;\n\t"
        "add.cc.u32  w1, %6, %10;\n\t"              // t = U + V (mod 2^160), t0 = u0
        "addc.cc.u32 w2, %7, %11;\n\t"
        "addc.cc.u32 w3, %8, %12;\n\t"
        "addc.u32    w4, %9, %13;\n\t"
        "sub.cc.u32  %0, %14, %5;\n\t"              // R = P - t (mod 2^160)
        "subc.cc.u32 %1, %15, w1;\n\t"
        "subc.cc.u32 %2, %16, w2;\n\t"
        "subc.cc.u32 %3, %17, w3;\n\t"
        "subc.u32    %4, %18, w4;\n\t}"
        : "=r"(R0), "=r"(R1), "=r"(R2), "=r"(R3), "=r"(R4)
        : "r"(u0), "r"(u1), "r"(u2), "r"(u3), "r"(u4), "r"(v1), "r"(v2), "r"(v3), "r"(v4),
          "r"(P[0]), "r"(P[1]), "r"(P[2]), "r"(P[3]), "r"(P[4]));
    // ---- R in [0, 4q): three conditional subtractions of q
#pragma unroll
    for (int it = 0; it < 3; it++) {
        uint32_t d0, d1, d2, d3, d4, bw;
        asm("sub.cc.u32  %0, %6, %11;\n\t"
            "subc.cc.u32 %1, %7, %12;\n\t"
            "subc.cc.u32 %2, %8, %13;\n\t"
            "subc.cc.u32 %3, %9, %14;\n\t"
            "subc.cc.u32 %4, %10, 0;\n\t"
            "subc.u32    %5, 0, 0;"
            : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(d3), "=r"(d4), "=r"(bw)
            : "r"(R0), "r"(R1), "r"(R2), "r"(R3), "r"(R4), "r"(c.q[0]), "r"(c.q[1]), "r"(c.q[2]), "r"(c.q[3]));
        R0 = (R0 & bw) | (d0 & ~bw);
        R1 = (R1 & bw) | (d1 & ~bw);
        R2 = (R2 & bw) | (d2 & ~bw);
        R3 = (R3 & bw) | (d3 & ~bw);
        if (it < 2) R4 = (R4 & bw) | (d4 & ~bw);
    }
    r[0] = R0;
    r[1] = R1;
    r[2] = R2;
    r[3] = R3;
}
#endif

}  // namespace ntt128
