// host128.h -- host-side 128-bit modular arithmetic for plan construction and
// argument validation (primality, root order, Montgomery constants).
//
// Product code: independent of oracle/ (Montgomery multiplication with two 64-bit
// digits here; the oracle uses shift-subtract remainders).  Runs only at plan
// create / call validation, never per element.
#pragma once
#include <cstdint>

namespace ntt128h {

typedef unsigned __int128 u128;

static inline u128 make(uint64_t lo, uint64_t hi) { return ((u128)hi << 64) | lo; }

struct Mont {
    u128 q;     // odd modulus
    u128 qp;    // -q^{-1} mod 2^128
    u128 r1;    // 2^128 mod q
    u128 r2;    // 2^256 mod q

    explicit Mont(u128 q_) : q(q_) {
        u128 inv = 1;  // Newton iteration: inv = q^{-1} mod 2^(2^k)
        for (int i = 0; i < 7; i++) inv *= (u128)2 - q * inv;
        qp = (u128)0 - inv;
        r1 = ((u128)0 - q) % q;  // (2^128 - q) mod q == 2^128 mod q
        r2 = r1;
        for (int i = 0; i < 128; i++) r2 = add(r2, r2);
    }
    u128 add(u128 a, u128 b) const {
        u128 s = a + b;
        bool c = s < a;
        return (c || s >= q) ? s - q : s;
    }
    u128 sub(u128 a, u128 b) const { return a >= b ? a - b : a - b + q; }

    // a * b * 2^-128 mod q, two 64-bit digits (a, b < q)
    u128 mul(u128 a, u128 b) const {
        uint64_t b0 = (uint64_t)b, b1 = (uint64_t)(b >> 64);
        uint64_t q0 = (uint64_t)q, q1 = (uint64_t)(q >> 64);
        uint64_t qp0 = (uint64_t)qp;
        // t = (t2:t1:t0), 192 bits + carry word
        uint64_t t0 = 0, t1 = 0, t2 = 0, t3 = 0;
        for (int i = 0; i < 2; i++) {
            uint64_t ai = (uint64_t)(a >> (64 * i));
            u128 p = (u128)ai * b0 + t0;
            t0 = (uint64_t)p;
            p = (u128)ai * b1 + t1 + (uint64_t)(p >> 64);
            t1 = (uint64_t)p;
            u128 s = (u128)t2 + (uint64_t)(p >> 64);
            t2 = (uint64_t)s;
            t3 = (uint64_t)(s >> 64);
            uint64_t m = t0 * qp0;
            p = (u128)m * q0 + t0;
            p = (u128)m * q1 + t1 + (uint64_t)(p >> 64);
            t0 = (uint64_t)p;
            s = (u128)t2 + (uint64_t)(p >> 64);
            t1 = (uint64_t)s;
            t2 = t3 + (uint64_t)(s >> 64);
        }
        u128 t = make(t0, t1);  // value = t2 * 2^128 + t, < 2q
        if (t2 || t >= q) t -= q;
        return t;
    }
    u128 to_m(u128 a) const { return mul(a % q, r2); }
    u128 from_m(u128 a) const { return mul(a, 1); }
    u128 mulmod(u128 a, u128 b) const { return from_m(mul(to_m(a), to_m(b))); }
    u128 pow(u128 a, u128 e) const {
        u128 r = r1 % q, x = to_m(a);
        while (e) {
            if (e & 1) r = mul(r, x);
            x = mul(x, x);
            e >>= 1;
        }
        return from_m(r);
    }
    u128 inv(u128 a) const { return pow(a, q - 2); }
};

// Miller-Rabin with 24 fixed prime bases (probable prime for 128-bit inputs).
static inline bool is_probable_prime(u128 n) {
    static const uint32_t bases[24] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59, 61, 67, 71, 73, 79, 83, 89};
    if (n < 2) return false;
    for (uint32_t b : bases) {
        if (n == b) return true;
        if (n % b == 0) return false;
    }
    Mont M(n);
    u128 d = n - 1;
    int s = 0;
    while (!(d & 1)) { d >>= 1; s++; }
    for (uint32_t b : bases) {
        u128 x = M.pow(b, d);
        if (x == 1 || x == n - 1) continue;
        bool composite = true;
        for (int r = 1; r < s; r++) {
            x = M.mulmod(x, x);
            if (x == n - 1) { composite = false; break; }
        }
        if (composite) return false;
    }
    return true;
}

}  // namespace ntt128h
