// Bit-level model of the even/odd-alternating Montgomery product used by
// arith128.cuh (mont_mul_eo / mont_mul_eo_lazy) and of the lazy butterflies.
// Every 32-bit word operation is emulated with explicit carries, and every
// place where the PTX drops a carry (a chain that ends without .cc, a word
// assumed not to overflow) is asserted.  Results are checked against
// unsigned __int128 / 256-bit reference arithmetic.
//
//   gcc -O2 -o /tmp/mont_eo_model tools/model/mont_eo_model.c && /tmp/mont_eo_model
//
// This is a development model of the kernel arithmetic (not the oracle, not
// product code).
#include <assert.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

typedef unsigned __int128 u128;
typedef uint32_t u32;
typedef uint64_t u64;

static u64 rng_state = 0x1234567;
static u64 sm64(void) {
    u64 z = (rng_state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static u128 r128(void) { return ((u128)sm64() << 64) | sm64(); }

// ---- 32-bit word primitives with a carry flag (PTX semantics)
static u32 CF;
static u32 add_cc(u32 a, u32 b) { u64 s = (u64)a + b; CF = (u32)(s >> 32); return (u32)s; }
static u32 addc_cc(u32 a, u32 b) { u64 s = (u64)a + b + CF; CF = (u32)(s >> 32); return (u32)s; }
static u32 addc(u32 a, u32 b) { u64 s = (u64)a + b + CF; assert((s >> 32) == 0); return (u32)s; }  // carry must not be lost
static u32 sub_cc(u32 a, u32 b) { u64 d = (u64)a - b; CF = (u32)(d >> 63); return (u32)d; }     // CF = borrow
static u32 subc_cc(u32 a, u32 b) { u64 d = (u64)a - b - CF; CF = (u32)(d >> 63); return (u32)d; }
static u32 subc(u32 a, u32 b) { u64 d = (u64)a - b - CF; return (u32)d; }
// IMAD.WIDE-style pair ops: (lo, hi) += x*y (+CF on lo), carry out in CF
static void mad_pair(u32* lo, u32* hi, u32 x, u32 y, int carry_in) {
    u64 p = (u64)x * y;
    u64 s = (u64)*lo + (u32)p + (carry_in ? CF : 0);
    *lo = (u32)s;
    u64 t = (u64)*hi + (u32)(p >> 32) + (s >> 32);
    *hi = (u32)t;
    CF = (u32)(t >> 32);
}

static void words(u128 v, u32 w[4]) { for (int i = 0; i < 4; i++) w[i] = (u32)(v >> (32 * i)); }
static u128 val4(const u32 w[4]) { u128 v = 0; for (int i = 3; i >= 0; i--) v = (v << 32) | w[i]; return v; }

// reference: a * b * 2^-128 mod q (q odd), via 256-bit long division on u128 halves
static u128 mulmod_ref(u128 a, u128 b, u128 q) {
    // schoolbook 256-bit product then restoring remainder
    u64 a0 = (u64)a, a1 = (u64)(a >> 64), b0 = (u64)b, b1 = (u64)(b >> 64);
    u128 p00 = (u128)a0 * b0, p01 = (u128)a0 * b1, p10 = (u128)a1 * b0, p11 = (u128)a1 * b1;
    u128 mid = (p00 >> 64) + (u64)p01 + (u64)p10;
    u128 lo = (mid << 64) | (u64)p00;
    u128 hi = p11 + (p01 >> 64) + (p10 >> 64) + (mid >> 64);
    u128 r = 0;
    for (int i = 255; i >= 0; i--) {
        u32 top = (u32)(r >> 127);
        u32 bit = i >= 128 ? (u32)(hi >> (i - 128)) & 1 : (u32)(lo >> i) & 1;
        r = (r << 1) | bit;
        if (top || r >= q) r -= q;
    }
    return r;
}
static u128 powmod(u128 b, u128 e, u128 q) {
    u128 r = 1 % q;
    while (e) { if (e & 1) r = mulmod_ref(r, b, q); b = mulmod_ref(b, b, q); e >>= 1; }
    return r;
}
// R^-1 mod q via R^(q-2)... q prime not guaranteed in the random tests: use extended approach:
// montgomery result check: T * R == a * b (mod q), R mod q = 2^128 mod q
static u128 rmod(u128 q) { return (u128)(-(u128)q) % q; }  // 2^128 mod q

// ---- the algorithm (mirrors arith128.cuh mont_mul_eo): returns T (5 words) before the final subtraction
static void mont_eo_core(const u32 a[4], const u32 b[4], const u32 q[4], u32 qinv0, u32 T[5]) {
    u32 X[5], Y[5], m;
    // digit 0
    { u64 p = (u64)a[0] * b[0]; X[0] = (u32)p; X[1] = (u32)(p >> 32); p = (u64)a[2] * b[0]; X[2] = (u32)p; X[3] = (u32)(p >> 32); }
    { u64 p = (u64)a[1] * b[0]; Y[0] = (u32)p; Y[1] = (u32)(p >> 32); p = (u64)a[3] * b[0]; Y[2] = (u32)p; Y[3] = (u32)(p >> 32); }
    m = X[0] * qinv0;
    mad_pair(&X[0], &X[1], m, q[0], 0); mad_pair(&X[2], &X[3], m, q[2], 1); X[4] = addc(0, 0);
    mad_pair(&Y[0], &Y[1], m, q[1], 0); mad_pair(&Y[2], &Y[3], m, q[3], 1); Y[4] = addc(0, 0);
    assert(X[0] == 0);
    for (int i = 1; i < 4; i++) {
        u32 Xn[5], Yn[5];
        // X' := Y with Y0 += X1 (carry -> Y' word 0, weight 2^32)
        Xn[0] = add_cc(Y[0], X[1]); Xn[1] = Y[1]; Xn[2] = Y[2]; Xn[3] = Y[3];
        // Y' = (X2, X3) + a1 b + CF ; (X4, 0) + a3 b + CF  -- no carry out (asserted)
        Yn[0] = X[2]; Yn[1] = X[3];
        mad_pair(&Yn[0], &Yn[1], a[1], b[i], 1);
        Yn[2] = X[4]; Yn[3] = 0;
        mad_pair(&Yn[2], &Yn[3], a[3], b[i], 1);
        assert(CF == 0);
        // X' += a_even b_i, carry -> X'4 = Y4 + CF
        mad_pair(&Xn[0], &Xn[1], a[0], b[i], 0); mad_pair(&Xn[2], &Xn[3], a[2], b[i], 1); Xn[4] = addc(Y[4], 0);
        m = Xn[0] * qinv0;
        mad_pair(&Xn[0], &Xn[1], m, q[0], 0); mad_pair(&Xn[2], &Xn[3], m, q[2], 1); Xn[4] = addc(Xn[4], 0);
        mad_pair(&Yn[0], &Yn[1], m, q[1], 0); mad_pair(&Yn[2], &Yn[3], m, q[3], 1); Yn[4] = addc(0, 0);
        assert(Xn[0] == 0);
        for (int k = 0; k < 5; k++) { X[k] = Xn[k]; Y[k] = Yn[k]; }
    }
    // T = Y + X / 2^32
    T[0] = add_cc(Y[0], X[1]); T[1] = addc_cc(Y[1], X[2]); T[2] = addc_cc(Y[2], X[3]); T[3] = addc_cc(Y[3], X[4]);
    T[4] = addc(Y[4], 0);
}

static int nbits(u128 v) { int n = 0; while (v) { n++; v >>= 1; } return n; }

static void check_one(u128 q, u128 a, u128 b, int lazy) {
    u32 qw[4], aw[4], bw[4], T[5];
    words(q, qw); words(a, aw); words(b, bw);
    u32 inv = 1; for (int i = 0; i < 5; i++) inv *= 2 - qw[0] * inv;
    u32 qinv0 = (u32)(-inv);
    mont_eo_core(aw, bw, qw, qinv0, T);
    u128 t = val4(T);
    // T (129 bits) must be < 2q, congruent to a b R^-1
    u128 expect = mulmod_ref(mulmod_ref(a % q, b, q), 1, q);  // a b mod q
    // check T * R == a b (mod q): (t + T4 2^128) * R mod q
    u128 R = rmod(q);
    u128 tt = t % q;
    if (T[4]) tt = (tt + R) % q;          // + 2^128
    assert(T[4] <= 1);
    u128 lhs = mulmod_ref(tt, R, q);
    assert(lhs == expect);
    // T < 2q
    if (T[4]) { assert(q > ((u128)1 << 127)); assert(t < (u128)(2 * q)); }  // 2q wraps: t + 2^128 < 2q <=> t < 2q - 2^128
    else if (q <= ((u128)1 << 127)) assert(t < 2 * q);
    if (lazy) {
        assert(T[4] == 0);
        assert(t < 2 * q);
    }
}

int main(int argc, char** argv) {
    long n = argc > 1 ? atol(argv[1]) : 200000;
    u128 qs[16];
    int nq = 0;
    qs[nq++] = ~(u128)0 - 55295 + 1;                                 // cfg1 prime 2^128 - 55295
    qs[nq++] = ~(u128)0 - 2013265919 + 1;                            // cfg5
    qs[nq++] = ~(u128)0;                                             // 2^128 - 1 (odd, worst case bound)
    qs[nq++] = ((u128)0x804671da650e225bull << 64) | 0x9b75f6b15a9a0001ull;  // random 128-bit
    qs[nq++] = ((u128)1 << 127) + 1;                                 // just above 2^127
    qs[nq++] = ((u128)1 << 127) - 1;                                 // 127-bit
    qs[nq++] = ((u128)0x7fffffffffffffffull << 64) | 0xffffffffff860001ull;  // cfg3 q1 (127-bit)
    qs[nq++] = ((u128)0x3fffffffffffffffull << 64) | 0xfffffffffffc0001ull;  // cfg3 q2 (126-bit)
    qs[nq++] = ((u128)1 << 126) - 1;
    qs[nq++] = ((u128)0x0fffffffffffffffull << 64) | 0xfffffffffa60001ull;   // 124-bit
    qs[nq++] = 97;
    qs[nq++] = 65537;
    long checked = 0;
    for (int k = 0; k < nq; k++) {
        u128 q = qs[k];
        int lazy = nbits(q) <= 126;   // q < 2^126
        u128 amax = lazy ? 4 * q : ~(u128)0;   // lazy inputs a < 4q; full inputs a < 2^128
        u128 edges[] = {0, 1, 2, q - 1, q - 2, q / 2, q / 2 + 1, 0xffffffffull, 0x100000000ull, ~(u128)0 >> 64,
                        (u128)1 << 64, ((u128)1 << 96) - 1, ((u128)1 << 127) - 1, (u128)1 << 127, ~(u128)0, amax - 1,
                        amax - 2, 2 * q - 1, 3 * q - 1};
        int ne = sizeof(edges) / sizeof(edges[0]);
        for (int i = 0; i < ne; i++)
            for (int j = 0; j < ne; j++) {
                u128 a = edges[i], b = edges[j];
                if (lazy && a >= amax) continue;
                if (b >= q) continue;
                check_one(q, a, b, lazy); checked++;
            }
        for (long t = 0; t < n; t++) {
            u128 a = r128(), b = r128() % q;
            if (lazy) a %= amax;
            if (t & 1) a = amax - 1 - (a % 1000);  // near the top of the input range
            check_one(q, a, b, lazy); checked++;
        }
    }
    printf("mont_eo model: %ld products checked, all carries accounted for\n", checked);
    return 0;
}
