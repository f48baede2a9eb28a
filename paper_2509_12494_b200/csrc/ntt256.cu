// ntt256.cu -- wider-modulus NTT: the radix-2 NTT of Eq. ntt
// and the point-wise product over any odd prime q < 2^256, residues as
// four 64-bit limbs (32 bytes), arithmetic on eight 32-bit words (arith256_gen.cuh:
// Montgomery R = 2^256, 128 + 8 word products per product).  The paper's stated
// generalisation to larger bit widths (e.g. zero-knowledge proofs).
//
// Same pass structure as the 128-bit path (ntt128.cu): decimation in time
// from bit-reversed input, the bit reversal folded into the first pass's gather, passes of
// at most 8 stages on groups of 2^B elements, twiddles per pass in consumption order
// (Montgomery form), stage-0 butterflies without a multiply, N^-1 folded into the
// inverse's last stage.  One group per CTA, radix-4 register rounds (4 elements x 8 words
// per thread), a 32-byte residue kept as two 16-byte planes in shared memory so every
// 8-lane phase touches distinct banks (slot l + l/8, as in the 128-bit kernels).  Values
// canonical, except in plans whose moduli are all < R/4 (the lazy class, template LZ: [0, 4q)
// between stages, Harvey butterflies, canonicalised in the last pass's store).
// Word count W (template parameter): plans and vec256_mul whose moduli are all < 2^192 run
// the 6-word arithmetic (Montgomery R = 2^192, 72 + 6 word products per product instead of
// 128 + 8); storage stays 32 bytes per residue with the top limb zero.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/ntt128.h"
#include "arith256_gen.cuh"
#include "ntt128_internal.h"

void ntt128_count_launch(uint64_t k);

namespace {

using namespace ntt256;

// ----------------------------------------------------------------------------- host 256-bit helpers
// Plain schoolbook / shift-and-add arithmetic for plan-time constants only.
struct H256 {
    uint64_t w[4];
};
inline H256 h_from(uint64_t v) { return H256{{v, 0, 0, 0}}; }
inline int h_cmp(const H256& a, const H256& b) {
    for (int i = 3; i >= 0; i--)
        if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
    return 0;
}
inline bool h_is_zero(const H256& a) { return !(a.w[0] | a.w[1] | a.w[2] | a.w[3]); }
inline H256 h_sub(const H256& a, const H256& b) {
    H256 r;
    unsigned __int128 bw = 0;
    for (int i = 0; i < 4; i++) {
        unsigned __int128 d = (unsigned __int128)a.w[i] - b.w[i] - (uint64_t)bw;
        r.w[i] = (uint64_t)d;
        bw = (d >> 64) & 1;
    }
    return r;
}
// (a + b) mod q for a, b < q (the sum may carry out of 256 bits)
inline H256 h_addmod(const H256& a, const H256& b, const H256& q) {
    H256 s;
    unsigned __int128 c = 0;
    for (int i = 0; i < 4; i++) {
        unsigned __int128 t = (unsigned __int128)a.w[i] + b.w[i] + (uint64_t)c;
        s.w[i] = (uint64_t)t;
        c = t >> 64;
    }
    if (c || h_cmp(s, q) >= 0) s = h_sub(s, q);
    return s;
}
inline H256 h_mulmod(const H256& a, const H256& b, const H256& q) {   // double and add over b's bits
    H256 r = h_from(0);
    for (int i = 255; i >= 0; i--) {
        r = h_addmod(r, r, q);
        if ((b.w[i / 64] >> (i % 64)) & 1) r = h_addmod(r, a, q);
    }
    return r;
}
inline H256 h_powmod(const H256& a, const H256& e, const H256& q) {
    H256 r = h_from(1);
    for (int i = 255; i >= 0; i--) {
        r = h_mulmod(r, r, q);
        if ((e.w[i / 64] >> (i % 64)) & 1) r = h_mulmod(r, a, q);
    }
    return r;
}
inline H256 h_add_nc(const H256& a, const H256& b) {   // a + b < 2^256
    H256 r;
    unsigned __int128 c = 0;
    for (int i = 0; i < 4; i++) {
        const unsigned __int128 t = (unsigned __int128)a.w[i] + b.w[i] + (uint64_t)c;
        r.w[i] = (uint64_t)t;
        c = t >> 64;
    }
    return r;
}
inline H256 h_shr1(const H256& a) {
    H256 r;
    for (int i = 0; i < 3; i++) r.w[i] = (a.w[i] >> 1) | (a.w[i + 1] << 63);
    r.w[3] = a.w[3] >> 1;
    return r;
}
bool h_is_probable_prime(const H256& n) {
    static const uint64_t bases[20] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59, 61, 67, 71};
    if (!(n.w[0] & 1)) return false;
    if (h_cmp(n, h_from(72)) < 0) {
        for (uint64_t b : bases) if (n.w[0] == b && !n.w[1] && !n.w[2] && !n.w[3]) return true;
        return false;
    }
    const H256 nm1 = h_sub(n, h_from(1));
    H256 d = nm1;
    int s = 0;
    while (!(d.w[0] & 1)) { d = h_shr1(d); s++; }
    for (uint64_t b : bases) {
        H256 x = h_powmod(h_from(b), d, n);
        if (h_cmp(x, h_from(1)) == 0 || h_cmp(x, nm1) == 0) continue;
        bool ok = false;
        for (int r = 1; r < s && !ok; r++) {
            x = h_mulmod(x, x, n);
            ok = h_cmp(x, nm1) == 0;
        }
        if (!ok) return false;
    }
    return true;
}
inline void h_words(const H256& v, uint32_t w[8]) {
    for (int i = 0; i < 8; i++) w[i] = (uint32_t)(v.w[i / 2] >> (32 * (i % 2)));
}
inline uint4 h_lo4(const H256& v) { return make_uint4((uint32_t)v.w[0], (uint32_t)(v.w[0] >> 32), (uint32_t)v.w[1], (uint32_t)(v.w[1] >> 32)); }
inline uint4 h_hi4(const H256& v) { return make_uint4((uint32_t)v.w[2], (uint32_t)(v.w[2] >> 32), (uint32_t)v.w[3], (uint32_t)(v.w[3] >> 32)); }

// ----------------------------------------------------------------------------- device helpers
#ifndef NTT256_SHIFT_SCALE
#define NTT256_SHIFT_SCALE 1   // 0: the inverse's N^-1 on u by a Montgomery product (A/B)
#endif
struct ModC256 {
    uint32_t q[8];
    uint32_t qinv0;
    uint32_t one_m[8];    // R mod q
    uint32_t r2[8];       // R^2 mod q
    uint32_t ninv_m[8];   // N^-1 R mod q
    uint32_t q2[8];       // 2q (lazy class only: q < R / 4)
};

struct E256 {
    uint32_t w[8];
};
// W = 6: words 6 and 7 are zero by construction (known to the compiler: no registers spent)
template <int W>
__device__ __forceinline__ E256 e_from(uint4 lo, uint4 hi) {
    return E256{{lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, W == 8 ? hi.z : 0u, W == 8 ? hi.w : 0u}};
}
__device__ __forceinline__ uint4 e_lo(const E256& e) { return make_uint4(e.w[0], e.w[1], e.w[2], e.w[3]); }
__device__ __forceinline__ uint4 e_hi(const E256& e) { return make_uint4(e.w[4], e.w[5], e.w[6], e.w[7]); }
template <int W>
__device__ __forceinline__ E256 e_ld(const uint4* p) { return e_from<W>(p[0], p[1]); }   // 32-byte element at p
__device__ __forceinline__ void e_st(uint4* p, const E256& e) { p[0] = e_lo(e); p[1] = e_hi(e); }
template <int W>
__device__ __forceinline__ E256 mmul(const E256& a, const E256& b, const ModC256& M) {
    E256 r;
    if (W == 8) {
        mont_mul256(a.w, b.w, M.q, M.qinv0, r.w);
    } else {
        mont_mul192(a.w, b.w, M.q, M.qinv0, r.w);
        r.w[6] = r.w[7] = 0;
    }
    return r;
}
template <int W>
__device__ __forceinline__ void addm(const E256& a, const E256& b, const ModC256& M, E256& r) {
    if (W == 8) {
        add_mod256(a.w, b.w, M.q, r.w);
    } else {
        add_mod192(a.w, b.w, M.q, r.w);
        r.w[6] = r.w[7] = 0;
    }
}
template <int W>
__device__ __forceinline__ void subm(const E256& a, const E256& b, const ModC256& M, E256& r) {
    if (W == 8) {
        sub_mod256(a.w, b.w, M.q, r.w);
    } else {
        sub_mod192(a.w, b.w, M.q, r.w);
        r.w[6] = r.w[7] = 0;
    }
}
// Lazy class (every modulus < R / 4 = 2^(32 W - 2)): values in [0, 4q) between stages and
// Harvey butterflies, as the 128-bit LAZY class; bounds checked by
// tools/model/mont_eo_model_w.py (check_lazy).
template <int W>
__device__ __forceinline__ E256 mmul_lazy(const E256& a, const E256& b, const ModC256& M) {
    E256 r;
    if (W == 8) {
        mont_mul256_lazy(a.w, b.w, M.q, M.qinv0, r.w);
    } else {
        mont_mul192_lazy(a.w, b.w, M.q, M.qinv0, r.w);
        r.w[6] = r.w[7] = 0;
    }
    return r;
}
template <int W>
__device__ __forceinline__ void add_nr(const E256& a, const E256& b, E256& r) {
    if (W == 8) {
        add_nored256(a.w, b.w, r.w);
    } else {
        add_nored192(a.w, b.w, r.w);
        r.w[6] = r.w[7] = 0;
    }
}
template <int W>
__device__ __forceinline__ void sub_add_nr(const E256& a, const E256& b, const uint32_t c[8], E256& r) {
    if (W == 8) {
        sub_add_nored256(a.w, b.w, c, r.w);
    } else {
        sub_add_nored192(a.w, b.w, c, r.w);
        r.w[6] = r.w[7] = 0;
    }
}
template <int W>
__device__ __forceinline__ E256 red_c(const E256& a, const uint32_t c[8]) {
    E256 r;
    if (W == 8) {
        reduce_c256(a.w, c, r.w);
    } else {
        reduce_c192(a.w, c, r.w);
        r.w[6] = r.w[7] = 0;
    }
    return r;
}
__device__ __forceinline__ uint32_t brev_n(uint32_t x, int bits) { return bits == 0 ? 0u : (__brev(x) >> (32 - bits)); }
// u 2^-s mod q (1 <= s <= 31, u < q): one s-bit Montgomery digit, as shr_mod in arith128.cuh --
// m = u_0 (-q^-1) mod 2^s, T = (u + m q) / 2^s < q + u / 2^s < 2q, one conditional subtraction
// (T may reach bit 256: ninth word).  The inverse's last stage: u N^-1 = u 2^-n.
template <int W>
__device__ __forceinline__ E256 shr256(const E256& u, uint32_t s, const ModC256& M) {
    const uint32_t m = (u.w[0] * M.qinv0) & ((1u << s) - 1u);
    uint32_t x[W + 1];
    uint64_t c = 0;
#pragma unroll
    for (int i = 0; i < W; i++) {
        const uint64_t t = (uint64_t)m * M.q[i] + u.w[i] + c;   // < 2^64
        x[i] = (uint32_t)t;
        c = t >> 32;
    }
    x[W] = (uint32_t)c;
    uint32_t t[W + 1];
#pragma unroll
    for (int i = 0; i < W; i++) t[i] = __funnelshift_r(x[i], x[i + 1], s);
    t[W] = x[W] >> s;
    uint32_t d[W];
    int64_t bw = 0;
#pragma unroll
    for (int i = 0; i < W; i++) {
        const int64_t v = (int64_t)t[i] - (int64_t)M.q[i] + bw;
        d[i] = (uint32_t)v;
        bw = v >> 32;                                            // 0 or -1
    }
    const bool ge = ((int64_t)t[W] + bw) >= 0;                   // T >= q
    E256 r;
#pragma unroll
    for (int i = 0; i < 8; i++) r.w[i] = i < W ? (ge ? d[i] : t[i]) : 0u;
    return r;
}

// out[m][i] = scale_m base_m^i (Montgomery form), i < count: product over the set bits of i
template <int W>
__global__ void k_pow256(uint4* out, uint64_t stride, uint64_t count, const uint4* pow2, int K, const uint4* scale,
                         const ModC256* mods) {
    const int m = blockIdx.y;
    const ModC256 M = mods[m];
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x) {
        E256 r = e_ld<W>(scale + 2 * m);
        uint64_t e = i;
        int k = 0;
        while (e) {
            if (e & 1) r = mmul<W>(r, e_ld<W>(pow2 + 2 * ((size_t)m * K + k)), M);
            e >>= 1;
            k++;
        }
        e_st(out + 2 * (m * stride + i), r);
    }
}
// per-pass twiddles in consumption order (the 128-bit k_gather_pass_tw formula)
__global__ void k_gather256(uint4* out, uint64_t out_stride, const uint4* T, const uint4* T_last, uint64_t tw_stride,
                            uint32_t n, uint32_t lo, uint32_t b) {
    const int m = blockIdx.y;
    const uint32_t K = (1u << b) - 1;
    const uint64_t count = ((uint64_t)1 << lo) * K;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t L = e / K;
        const uint32_t k = (uint32_t)(e - L * K);
        const int sl = 31 - __clz(k + 1);
        const uint64_t jj = k + 1 - (1u << sl);
        const uint32_t s = lo + sl;
        const uint64_t j = (jj << lo) | L;
        const uint4* src = (T_last && s == n - 1) ? T_last + 2 * (m * tw_stride + j) : T + 2 * (m * tw_stride + (j << (n - 1 - s)));
        out[2 * (m * out_stride + e)] = src[0];
        out[2 * (m * out_stride + e) + 1] = src[1];
    }
}

struct Pass256Args {
    ModC256 mc0;              // nq == 1: the modulus as a kernel parameter (uniform registers in the rounds)
    const uint4* src;
    uint4* dst;
    const uint4* pt;          // [nq][pt_stride] 32-byte twiddles
    const ModC256* mods;
    uint64_t pt_stride;
    uint64_t total_groups;
    uint32_t n, lo, nq;
};

__device__ __forceinline__ int slot256(int l) { return l + (l >> 3); }

// threads per group (E = 4 residues each) and groups per CTA (at least 64 threads)
template <int B>
struct Shape256 {
    static constexpr int G = 1 << B;
    static constexpr int RB = B >= 2 ? 2 : B;
    static constexpr int E = 1 << RB;
    static constexpr int T = G / E;
    static constexpr int C = T >= 64 ? 1 : 64 / T;
    static constexpr int GP = G + G / 8 + 1;
};

#ifndef NTT256_MINB6
#define NTT256_MINB6 1        // resident CTAs per SM the 6-word pass kernels are register-budgeted for
#endif
#ifndef NTT256_MINB8
#define NTT256_MINB8 1
#endif
template <int B, bool FIRST, bool SCALE_LAST, int W, bool LZ>
__global__ void __launch_bounds__(Shape256<B>::C * Shape256<B>::T, W == 6 ? NTT256_MINB6 : NTT256_MINB8)
k_ntt256_pass(const __grid_constant__ Pass256Args a) {
    using S = Shape256<B>;
    constexpr int G = S::G, RB = S::RB, E = S::E, T = S::T, C = S::C, GP = S::GP;
    constexpr int ROUNDS = (B + RB - 1) / RB;
    __shared__ uint4 lo_p[C * GP], hi_p[C * GP];   // the two 16-byte planes of each residue
    __shared__ uint4 tw_lo[C * G], tw_hi[C * G];

    const uint32_t n = a.n, lo = a.lo, gbits = n - B;
    const uint64_t N = 1ull << n;
    const int c = threadIdx.x / T, t = threadIdx.x % T;
    const uint64_t gg_raw = (uint64_t)blockIdx.x * C + c;
    const bool live = gg_raw < a.total_groups;
    const uint64_t gg = live ? gg_raw : a.total_groups - 1;
    const uint64_t poly = gg >> gbits, g = gg & ((1ull << gbits) - 1);
    const uint32_t m = a.nq == 1 ? 0 : (uint32_t)poly;
    uint4* glo = lo_p + c * GP;
    uint4* ghi = hi_p + c * GP;
    uint4* twl = tw_lo + c * G;
    uint4* twh = tw_hi + c * G;
    // twiddles of this group's set (L = g mod 2^lo; a first pass has one set)
    {
        const uint64_t L = FIRST ? 0 : (g & ((1ull << lo) - 1));
        const uint4* src = a.pt + 2 * (m * a.pt_stride + L * (G - 1));
        for (int e = t; e < G - 1; e += T) { twl[e] = src[2 * e]; twh[e] = src[2 * e + 1]; }
    }
    // rows t + i T of the group
    uint64_t gbase, gstride;
    if (FIRST) {
        gbase = ((uint64_t)t << gbits) | g;
        gstride = (uint64_t)T << gbits;
    } else {
        const uint64_t H = g >> lo, L = g & ((1ull << lo) - 1);
        gbase = (H << (lo + B)) | ((uint64_t)t << lo) | L;
        gstride = (uint64_t)T << lo;
    }
    const uint4* srcp = a.src + 2 * (poly * N + gbase);
#pragma unroll
    for (int i = 0; i < E; i++) {
        const int r = t + i * T;
        const int l = FIRST ? (int)brev_n((uint32_t)r, B) : r;
        const uint4* p = srcp + 2 * i * gstride;
        glo[slot256(l)] = p[0];
        ghi[slot256(l)] = p[1];
    }
    __syncthreads();
    // the rounds, instantiated once per source of the modulus: a kernel parameter (nq == 1:
    // uniform registers, UR operands in the products) or the device table (lanes may differ)
    auto rounds = [&](const ModC256& M) {
    #pragma unroll 1
        for (int rd = 0; rd < ROUNDS; rd++) {
            const int slo = rd * RB;
            const int w = (slo + RB <= B) ? slo : B - RB;
            const int tlo = t & ((1 << w) - 1);
            const int l0 = ((t >> w) << (w + RB)) | tlo;
            E256 x[E];
    #pragma unroll
            for (int k = 0; k < E; k++) {
                const int s = slot256(l0 | (k << w));
                x[k] = e_from<W>(glo[s], ghi[s]);
            }
    #pragma unroll
            for (int bit = 0; bit < RB; bit++) {
                const int sl = w + bit;
                if (sl < slo) continue;
                const bool last = SCALE_LAST && lo + sl == n - 1;
                const bool trivial = FIRST && sl == 0 && !last;
    #pragma unroll
                for (int kk = 0; kk < E / 2; kk++) {
                    const int k0 = ((kk >> bit) << (bit + 1)) | (kk & ((1 << bit) - 1));
                    const int k1 = k0 | (1 << bit);
                    E256 v = x[k1], u = x[k0];
                    if (LZ) {                // Harvey: u' in [0, 2q), t in [0, 2q); u' + t, u' - t + 2q
                        E256 t = v, us = u;  // stage 0 of a first pass: canonical inputs, twiddle 1
                        if (!trivial) {
                            const int ti = (1 << sl) - 1 + tlo + ((kk & ((1 << bit) - 1)) << w);
                            t = mmul_lazy<W>(v, e_from<W>(twl[ti], twh[ti]), M);
                            if (last) us = (NTT256_SHIFT_SCALE && n >= 1) ? shr256<W>(u, n, M)
                                                                        : mmul<W>(u, E256{{M.ninv_m[0], M.ninv_m[1], M.ninv_m[2], M.ninv_m[3], M.ninv_m[4],
                                                                                           M.ninv_m[5], M.ninv_m[6], M.ninv_m[7]}}, M);
                            else us = red_c<W>(u, M.q2);
                        }
                        add_nr<W>(us, t, x[k0]);
                        sub_add_nr<W>(us, t, M.q2, x[k1]);
                        continue;
                    }
                    if (!trivial) {
                        const int ti = (1 << sl) - 1 + tlo + ((kk & ((1 << bit) - 1)) << w);
                        v = mmul<W>(v, e_from<W>(twl[ti], twh[ti]), M);
                        if (last) u = (NTT256_SHIFT_SCALE && n >= 1) ? shr256<W>(u, n, M)
                                                                   : mmul<W>(u, E256{{M.ninv_m[0], M.ninv_m[1], M.ninv_m[2], M.ninv_m[3], M.ninv_m[4],
                                                                                      M.ninv_m[5], M.ninv_m[6], M.ninv_m[7]}}, M);
                    }
                    addm<W>(u, v, M, x[k0]);
                    subm<W>(u, v, M, x[k1]);
                }
            }
    #pragma unroll
            for (int k = 0; k < E; k++) {
                const int s = slot256(l0 | (k << w));
                glo[s] = e_lo(x[k]);
                ghi[s] = e_hi(x[k]);
            }
            __syncthreads();
        }
    };
    if (a.nq == 1) rounds(a.mc0);
    else rounds(a.mods[m]);
    if (LZ && lo + B == n) {   // the transform's last pass: [0, 4q) -> canonical [0, q) before the store
        const ModC256& M = a.nq == 1 ? a.mc0 : a.mods[m];
#pragma unroll
        for (int i = 0; i < E; i++) {
            const int s = slot256(t + i * T);
            const E256 v = red_c<W>(red_c<W>(e_from<W>(glo[s], ghi[s]), M.q2), M.q);
            glo[s] = e_lo(v);
            ghi[s] = e_hi(v);
        }
        __syncthreads();
    }
    if (!live) return;
    // store: the first pass writes the group as contiguous rows (natural order within it)
    if (FIRST) {
        uint4* dstp = a.dst + 2 * (poly * N + ((uint64_t)brev_n((uint32_t)g, gbits) << B));
#pragma unroll
        for (int i = 0; i < E; i++) {
            const int l = t + i * T;
            dstp[2 * l] = glo[slot256(l)];
            dstp[2 * l + 1] = ghi[slot256(l)];
        }
    } else {
        uint4* dstp = a.dst + 2 * (poly * N + gbase);
#pragma unroll
        for (int i = 0; i < E; i++) {
            const int l = t + i * T;
            uint4* p = dstp + 2 * i * gstride;
            p[0] = glo[slot256(l)];
            p[1] = ghi[slot256(l)];
        }
    }
}

// z = x y mod q: two Montgomery products (x y R^-1, then * R^2)
template <int W>
__global__ void k_vmul256(uint4* z, const uint4* x, const uint4* y, uint64_t n, const ModC256 M) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const E256 t = mmul<W>(e_ld<W>(x + 2 * i), e_ld<W>(y + 2 * i), M);
        e_st(z + 2 * i, mmul<W>(t, E256{{M.r2[0], M.r2[1], M.r2[2], M.r2[3], M.r2[4], M.r2[5], M.r2[6], M.r2[7]}}, M));
    }
}

typedef void (*Pass256Fn)(const Pass256Args);
template <bool FIRST, bool SL, int W, bool LZ>
Pass256Fn pass256_fn_w(int B) {
    switch (B) {
        case 1: return k_ntt256_pass<1, FIRST, SL, W, LZ>;
        case 2: return k_ntt256_pass<2, FIRST, SL, W, LZ>;
        case 3: return k_ntt256_pass<3, FIRST, SL, W, LZ>;
        case 4: return k_ntt256_pass<4, FIRST, SL, W, LZ>;
        case 5: return k_ntt256_pass<5, FIRST, SL, W, LZ>;
        case 6: return k_ntt256_pass<6, FIRST, SL, W, LZ>;
        case 7: return k_ntt256_pass<7, FIRST, SL, W, LZ>;
        default: return k_ntt256_pass<8, FIRST, SL, W, LZ>;
    }
}
template <bool FIRST, bool SL>
Pass256Fn pass256_fn(int B, int W, bool lz) {
    if (W == 6) return lz ? pass256_fn_w<FIRST, SL, 6, true>(B) : pass256_fn_w<FIRST, SL, 6, false>(B);
    return lz ? pass256_fn_w<FIRST, SL, 8, true>(B) : pass256_fn_w<FIRST, SL, 8, false>(B);
}

std::vector<int> pass_bits256(int n) {
    std::vector<int> b;
    const int np = (n + 7) / 8;
    for (int i = 0; i < np; i++) b.push_back(n / np + (i < n % np ? 1 : 0));
    return b;
}

// words of the Montgomery radix R = 2^(32 W): 6 when q < 2^192, else 8
inline int words_for(const H256& q) { return q.w[3] == 0 ? 6 : 8; }   // 64-bit limbs: q < 2^192
// lazy class of a W-word plan: q < R / 4 = 2^(32 W - 2) (4q fits the W words)
#ifndef NTT256_LAZY
#define NTT256_LAZY 1         // 0: every plan canonical (A/B experiment build)
#endif
inline bool lazy_ok(const H256& q, int W) { return NTT256_LAZY && (q.w[W / 2 - 1] >> 62) == 0; }

ModC256 make_modc(const H256& q, uint64_t N, int W) {
    ModC256 c;
    memset(&c, 0, sizeof(c));
    h_words(q, c.q);
    uint32_t inv = 1;
    for (int i = 0; i < 5; i++) inv *= 2 - c.q[0] * inv;
    c.qinv0 = 0u - inv;
    H256 r = h_from(1);                     // R mod q = 2^(32 W) mod q, R^2 mod q: repeated doubling
    for (int i = 0; i < 32 * W; i++) r = h_addmod(r, r, q);
    H256 r2 = r;
    for (int i = 0; i < 32 * W; i++) r2 = h_addmod(r2, r2, q);
    h_words(r, c.one_m);
    h_words(r2, c.r2);
    if (!(q.w[3] >> 63)) h_words(h_add_nc(q, q), c.q2);   // 2q < 2^256
    if (N > 1) {
        const H256 ninv = h_powmod(h_from(N), h_sub(q, h_from(2)), q);
        h_words(h_mulmod(ninv, r, q), c.ninv_m);
    }
    return c;
}

}  // namespace

struct ntt256_plan_s {
    uint32_t log2n, batch, nq;
    int words;                          // 6 (every modulus < 2^192) or 8
    bool lazy;                          // every modulus < 2^(32 words - 2): lazy class (values in [0, 4q))
    int device;
    uint64_t N;
    std::vector<int> bits;
    ModC256* d_mods = nullptr;
    ModC256 mc0;                        // host copy of modulus 0 (nq == 1 launches carry it as a parameter)
    std::vector<uint4*> d_fwd, d_inv;   // per pass [nq][stride] 32-byte twiddles
    std::vector<uint64_t> stride;
};

static void plan256_free(ntt256_plan_s* p) {
    if (!p) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(p->device);
    cudaFree(p->d_mods);
    for (auto* t : p->d_fwd) cudaFree(t);
    for (auto* t : p->d_inv) cudaFree(t);
    cudaSetDevice(prev);
    delete p;
}

// table[m][i] = scale_m base_m^i, i < count (Montgomery form), on the device
static cudaError_t gen256(uint4* out, uint64_t stride, uint64_t count, const std::vector<H256>& qs,
                          const std::vector<H256>& base, const std::vector<H256>& scale, const ModC256* d_mods, int W) {
    const int nq = (int)qs.size(), K = 32;
    std::vector<uint4> pow2((size_t)nq * K * 2), sc((size_t)nq * 2);
    for (int m = 0; m < nq; m++) {
        H256 r = h_from(1);
        for (int i = 0; i < 32 * W; i++) r = h_addmod(r, r, qs[m]);   // R mod q
        H256 b = base[m];                                              // base^(2^k), normal form
        for (int k = 0; k < K; k++) {
            const H256 bm = h_mulmod(b, r, qs[m]);                     // Montgomery form
            pow2[2 * ((size_t)m * K + k)] = h_lo4(bm);
            pow2[2 * ((size_t)m * K + k) + 1] = h_hi4(bm);
            b = h_mulmod(b, b, qs[m]);
        }
        const H256 s = h_mulmod(scale[m], r, qs[m]);
        sc[2 * m] = h_lo4(s);
        sc[2 * m + 1] = h_hi4(s);
    }
    uint4 *d_pow2 = nullptr, *d_sc = nullptr;
    cudaError_t e = cudaMalloc(&d_pow2, pow2.size() * sizeof(uint4));
    if (e == cudaSuccess) e = cudaMalloc(&d_sc, sc.size() * sizeof(uint4));
    if (e == cudaSuccess) e = cudaMemcpy(d_pow2, pow2.data(), pow2.size() * sizeof(uint4), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d_sc, sc.data(), sc.size() * sizeof(uint4), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        unsigned gx = (unsigned)((count + 255) / 256);
        if (gx > 4096) gx = 4096;
        if (gx == 0) gx = 1;
        if (W == 6) k_pow256<6><<<dim3(gx, nq), 256>>>(out, stride, count, d_pow2, K, d_sc, d_mods);
        else k_pow256<8><<<dim3(gx, nq), 256>>>(out, stride, count, d_pow2, K, d_sc, d_mods);
        ntt128_count_launch(1);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
    }
    cudaFree(d_pow2);
    cudaFree(d_sc);
    return e;
}

static H256 h_load(const uint64_t* p) { return H256{{p[0], p[1], p[2], p[3]}}; }

extern "C" ntt128_status ntt256_plan_create(ntt256_plan_t* out, uint32_t log2n, uint32_t batch, const uint64_t* q_host,
                                            const uint64_t* root_host, uint32_t n_moduli, uint32_t flags, int device) {
    if (!out || !q_host || !root_host) return NTT128_ERR_INVALID_ARG;
    *out = nullptr;
    if (log2n < 1 || log2n > 24 || batch == 0 || flags != 0) return NTT128_ERR_INVALID_ARG;
    if (n_moduli != 1 && n_moduli != batch) return NTT128_ERR_INVALID_ARG;
    const uint64_t N = 1ull << log2n;
    std::vector<H256> qs, omega, omega_inv, ones, ninv;
    for (uint32_t m = 0; m < n_moduli; m++) {
        const H256 q = h_load(q_host + 4 * m), w = h_load(root_host + 4 * m);
        if (!(q.w[0] & 1) || h_cmp(q, h_from(3)) < 0) return NTT128_ERR_MODULUS;
        if (!h_is_probable_prime(q)) return NTT128_ERR_NOT_PRIME;
        // N | q - 1
        const H256 qm1 = h_sub(q, h_from(1));
        if (qm1.w[0] & (N - 1)) return NTT128_ERR_NO_ROOT;
        if (h_cmp(w, q) >= 0) return NTT128_ERR_BAD_ROOT;
        if (h_cmp(h_powmod(w, h_from(N / 2), q), qm1) != 0) return NTT128_ERR_BAD_ROOT;   // exact order N
        qs.push_back(q);
        omega.push_back(w);
        omega_inv.push_back(h_powmod(w, h_sub(q, h_from(2)), q));
        ones.push_back(h_from(1));
        ninv.push_back(h_powmod(h_from(N), h_sub(q, h_from(2)), q));
    }
    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) return NTT128_ERR_INVALID_ARG;
    ntt256_plan_s* p = new (std::nothrow) ntt256_plan_s();
    if (!p) { cudaSetDevice(prev); return NTT128_ERR_OOM; }
    p->log2n = log2n;
    p->batch = batch;
    p->nq = n_moduli;
    p->device = device;
    p->N = N;
    p->bits = pass_bits256((int)log2n);
    p->words = 6;
    for (auto& q : qs)
        if (words_for(q) == 8) p->words = 8;
    const int W = p->words;
    p->lazy = true;
    for (auto& q : qs)
        if (!lazy_ok(q, W)) p->lazy = false;
    ntt128_status st = NTT128_OK;
    std::vector<ModC256> mc;
    for (auto& q : qs) mc.push_back(make_modc(q, N, W));
    p->mc0 = mc[0];
    if (cudaMalloc(&p->d_mods, n_moduli * sizeof(ModC256)) != cudaSuccess) st = NTT128_ERR_OOM;
    else if (cudaMemcpy(p->d_mods, mc.data(), n_moduli * sizeof(ModC256), cudaMemcpyHostToDevice) != cudaSuccess)
        st = NTT128_ERR_CUDA;
    const uint64_t half = N / 2 > 0 ? N / 2 : 1;
    uint4 *tf = nullptr, *ti = nullptr, *tl = nullptr;
    if (st == NTT128_OK && (cudaMalloc(&tf, 32 * half * n_moduli) != cudaSuccess ||
                            cudaMalloc(&ti, 32 * half * n_moduli) != cudaSuccess ||
                            cudaMalloc(&tl, 32 * half * n_moduli) != cudaSuccess))
        st = NTT128_ERR_OOM;
    if (st == NTT128_OK && (gen256(tf, half, half, qs, omega, ones, p->d_mods, W) != cudaSuccess ||
                            gen256(ti, half, half, qs, omega_inv, ones, p->d_mods, W) != cudaSuccess ||
                            gen256(tl, half, half, qs, omega_inv, ninv, p->d_mods, W) != cudaSuccess))
        st = NTT128_ERR_CUDA;
    int lo = 0;
    for (size_t i = 0; i < p->bits.size() && st == NTT128_OK; i++) {
        const int b = p->bits[i];
        const uint64_t stride = ((uint64_t)1 << lo) * (((uint64_t)1 << b) - 1);
        p->stride.push_back(stride);
        uint4 *f = nullptr, *v = nullptr;
        if (cudaMalloc(&f, 32 * stride * n_moduli) != cudaSuccess || cudaMalloc(&v, 32 * stride * n_moduli) != cudaSuccess)
            st = NTT128_ERR_OOM;
        p->d_fwd.push_back(f);
        p->d_inv.push_back(v);
        if (st != NTT128_OK) break;
        unsigned gx = (unsigned)((stride + 255) / 256);
        if (gx > 4096) gx = 4096;
        const bool last = i + 1 == p->bits.size();
        k_gather256<<<dim3(gx, n_moduli), 256>>>(f, stride, tf, nullptr, half, log2n, lo, b);
        k_gather256<<<dim3(gx, n_moduli), 256>>>(v, stride, ti, last ? tl : nullptr, half, log2n, lo, b);
        ntt128_count_launch(2);
        if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) st = NTT128_ERR_CUDA;
        lo += b;
    }
    cudaFree(tf);
    cudaFree(ti);
    cudaFree(tl);
    cudaSetDevice(prev);
    if (st != NTT128_OK) {
        plan256_free(p);
        return st;
    }
    *out = p;
    return NTT128_OK;
}

extern "C" void ntt256_plan_destroy(ntt256_plan_t p) { plan256_free(p); }

static ntt128_status run256(ntt256_plan_s* p, const uint4* src, uint4* dst, cudaStream_t st, bool inverse) {
    const int n = (int)p->log2n;
    const size_t np = p->bits.size();
    int lo = 0;
    for (size_t i = 0; i < np; i++) {
        const int B = p->bits[i];
        const bool first = i == 0, sl = inverse && i + 1 == np;
        const bool lz = p->lazy;
        Pass256Fn fn = first ? (sl ? pass256_fn<true, true>(B, p->words, lz) : pass256_fn<true, false>(B, p->words, lz))
                             : (sl ? pass256_fn<false, true>(B, p->words, lz) : pass256_fn<false, false>(B, p->words, lz));
        Pass256Args a;
        memset(&a, 0, sizeof(a));
        a.src = first ? src : dst;
        a.dst = dst;
        a.pt = inverse ? p->d_inv[i] : p->d_fwd[i];
        a.mods = p->d_mods;
        a.mc0 = p->mc0;
        a.pt_stride = p->stride[i];
        a.total_groups = (uint64_t)p->batch << (n - B);
        a.n = (uint32_t)n;
        a.lo = (uint32_t)lo;
        a.nq = p->nq;
        const int T = (1 << B) >= 4 ? (1 << B) / 4 : 1;
        const int C = T >= 64 ? 1 : 64 / T;
        fn<<<(unsigned)((a.total_groups + C - 1) / C), C * T, 0, st>>>(a);
        ntt128_count_launch(1);
        if (cudaGetLastError() != cudaSuccess) return NTT128_ERR_CUDA;
        lo += B;
    }
    return NTT128_OK;
}

static ntt128_status transform256(const ntt256_plan_t p, const uint64_t* d_in, uint64_t* d_out, ntt128_stream_t s,
                                  bool inverse) {
    if (!p || !d_in || !d_out) return NTT128_ERR_INVALID_ARG;
    if (((uintptr_t)d_in | (uintptr_t)d_out) & 15u) return NTT128_ERR_ALIGNMENT;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(p->device);
    ntt128_status r;
    if (d_in == d_out) {      // the first pass gathers bit-reversed columns: not in place
        const size_t bytes = (size_t)p->N * p->batch * 32;
        uint4* tmp = nullptr;
        if (cudaMallocAsync(&tmp, bytes, (cudaStream_t)s) != cudaSuccess) { cudaSetDevice(prev); return NTT128_ERR_OOM; }
        cudaMemcpyAsync(tmp, d_in, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)s);
        r = run256(p, tmp, (uint4*)d_out, (cudaStream_t)s, inverse);
        cudaFreeAsync(tmp, (cudaStream_t)s);
    } else {
        r = run256(p, (const uint4*)d_in, (uint4*)d_out, (cudaStream_t)s, inverse);
    }
    cudaSetDevice(prev);
    return r;
}
extern "C" ntt128_status ntt256_forward(const ntt256_plan_t p, const uint64_t* d_in, uint64_t* d_out, ntt128_stream_t s) {
    uint64_t g0, g1;
    ntt128_stream_gen((cudaStream_t)s, &g0, &g1);   // NTT128_FLAG_CHAIN: other library work on the stream
    return transform256(p, d_in, d_out, s, false);
}
extern "C" ntt128_status ntt256_inverse(const ntt256_plan_t p, const uint64_t* d_in, uint64_t* d_out, ntt128_stream_t s) {
    uint64_t g0, g1;
    ntt128_stream_gen((cudaStream_t)s, &g0, &g1);
    return transform256(p, d_in, d_out, s, true);
}

extern "C" ntt128_status vec256_mul(uint64_t* d_z, const uint64_t* d_x, const uint64_t* d_y, size_t n, const uint64_t* q_,
                                    ntt128_stream_t s) {
    if (!q_) return NTT128_ERR_INVALID_ARG;
    const H256 q = h_load(q_);
    if (!(q.w[0] & 1) || h_cmp(q, h_from(3)) < 0) return NTT128_ERR_MODULUS;
    if (n == 0) return NTT128_OK;
    if (!d_z || !d_x || !d_y) return NTT128_ERR_INVALID_ARG;
    if (((uintptr_t)d_z | (uintptr_t)d_x | (uintptr_t)d_y) & 15u) return NTT128_ERR_ALIGNMENT;
    uint64_t g0, g1;
    ntt128_stream_gen((cudaStream_t)s, &g0, &g1);
    const int W = words_for(q);
    const ModC256 M = make_modc(q, 1, W);
    unsigned g = (unsigned)((n + 255) / 256);
    if (g > 148 * 8) g = 148 * 8;
    if (W == 6) k_vmul256<6><<<g, 256, 0, (cudaStream_t)s>>>((uint4*)d_z, (const uint4*)d_x, (const uint4*)d_y, n, M);
    else k_vmul256<8><<<g, 256, 0, (cudaStream_t)s>>>((uint4*)d_z, (const uint4*)d_x, (const uint4*)d_y, n, M);
    ntt128_count_launch(1);
    return cudaGetLastError() == cudaSuccess ? NTT128_OK : NTT128_ERR_CUDA;
}
