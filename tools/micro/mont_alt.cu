// Register-only butterfly rate of mont_core formulations (radix-4 rounds, modulus in uniform
// registers as in the pass kernels):
//   V0: arith128.cuh's mont_core (the last a_odd b_i product of a digit as madc.lo/madc.hi
//       with the 64-bit addend {X_4, 0} -> IMAD + IMAD.HI + a zeroed register half);
//   VA: that product as mul.wide (IMAD.WIDE, RZ addend) and X_4 + carry added by two addc.
// Results are checked equal.  Build: tools/micro/build.sh mont_alt
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "arith128.cuh"
using namespace ntt128;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <bool TOP>
__device__ __forceinline__ void mont_core_a(const U128& a, const U128& b, const uint32_t q[4], uint32_t qinv0, uint32_t t[5]) {
    uint32_t x0, x1, x2, x3, x4, y0, y1, y2, y3, y4, m;
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
        asm("{\n\t.reg .u64 p;\n\t.reg .u32 pl, ph;\n\t"
            "mul.wide.u32   p, %14, %13;\n\t"
            "mov.b64        {pl, ph}, p;\n\t"
            "add.cc.u32     %0, %0, %9;\n\t"
            "madc.lo.cc.u32 %5, %12, %13, %10;\n\t"
            "madc.hi.cc.u32 %6, %12, %13, %11;\n\t"
            "addc.cc.u32    %7, pl, %15;\n\t"
            "addc.u32       %8, ph, 0;\n\t"
            "mad.lo.cc.u32  %0, %16, %13, %0;\n\t"
            "madc.hi.cc.u32 %1, %16, %13, %1;\n\t"
            "madc.lo.cc.u32 %2, %17, %13, %2;\n\t"
            "madc.hi.cc.u32 %3, %17, %13, %3;\n\t"
            "addc.u32       %4, %4, 0;\n\t}"
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
        x0 = y0; x1 = y1; x2 = y2; x3 = y3; x4 = y4;
        y0 = n0; y1 = n1; y2 = n2; y3 = n3; y4 = n4;
    }
    if (TOP) {
        asm("add.cc.u32  %0, %5, %10;\n\t"
            "addc.cc.u32 %1, %6, %11;\n\t"
            "addc.cc.u32 %2, %7, %12;\n\t"
            "addc.cc.u32 %3, %8, %13;\n\t"
            "addc.u32    %4, %9, 0;"
            : "=r"(t[0]), "=r"(t[1]), "=r"(t[2]), "=r"(t[3]), "=r"(t[4])
            : "r"(y0), "r"(y1), "r"(y2), "r"(y3), "r"(y4), "r"(x1), "r"(x2), "r"(x3), "r"(x4));
    } else {
        asm("add.cc.u32  %0, %4, %8;\n\t"
            "addc.cc.u32 %1, %5, %9;\n\t"
            "addc.cc.u32 %2, %6, %10;\n\t"
            "addc.u32    %3, %7, %11;"
            : "=r"(t[0]), "=r"(t[1]), "=r"(t[2]), "=r"(t[3])
            : "r"(y0), "r"(y1), "r"(y2), "r"(y3), "r"(x1), "r"(x2), "r"(x3), "r"(x4));
        t[4] = 0;
    }
}
template <int V> __device__ __forceinline__ U128 mlazy(const U128& a, const U128& b, const uint32_t q[4], uint32_t qi) {
    uint32_t t[5];
    if (V == 0) mont_core<false>(a, b, q, qi, t); else mont_core_a<false>(a, b, q, qi, t);
    return U128{{t[0], t[1], t[2], t[3]}};
}
template <int V> __device__ __forceinline__ U128 mfull(const U128& a, const U128& b, const uint32_t q[4], uint32_t qi) {
    uint32_t t[5];
    if (V == 0) mont_core<true>(a, b, q, qi, t); else mont_core_a<true>(a, b, q, qi, t);
    uint32_t d0, d1, d2, d3, bw;
    asm("sub.cc.u32  %0, %5, %10;\n\tsubc.cc.u32 %1, %6, %11;\n\tsubc.cc.u32 %2, %7, %12;\n\tsubc.cc.u32 %3, %8, %13;\n\tsubc.u32    %4, %9, 0;"
        : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(d3), "=r"(bw)
        : "r"(t[0]), "r"(t[1]), "r"(t[2]), "r"(t[3]), "r"(t[4]), "r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]));
    return U128{{(t[0] & bw) | (d0 & ~bw), (t[1] & bw) | (d1 & ~bw), (t[2] & bw) | (d2 & ~bw), (t[3] & bw) | (d3 & ~bw)}};
}

struct QC { uint32_t q[4], q2[4], qinv0; };
template <int V, int CLS>
__global__ void __launch_bounds__(256, 4) k(uint4* io, const uint4* tw, const __grid_constant__ QC c, int iters) {
    U128 x[4], w[2];
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
    for (int k = 0; k < 4; k++) x[k] = u128_from(io[tid * 4 + k]);
    w[0] = u128_from(tw[0]); w[1] = u128_from(tw[1]);
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int bit = 0; bit < 2; bit++) {
#pragma unroll
            for (int kk = 0; kk < 2; kk++) {
                const int k0 = ((kk >> bit) << (bit + 1)) | (kk & ((1 << bit) - 1));
                const int k1 = k0 | (1 << bit);
                const U128 u = x[k0];
                if (CLS == 3) {
                    const U128 us = reduce_2q(u, c.q2);
                    const U128 v = mlazy<V>(x[k1], w[(kk + bit) & 1], c.q, c.qinv0);
                    x[k0] = add_nored(us, v); x[k1] = sub_add_nored(us, v, c.q2);
                } else {
                    const U128 v = mfull<V>(x[k1], w[(kk + bit) & 1], c.q, c.qinv0);
                    x[k0] = add_mod(u, v, c.q); x[k1] = sub_mod(u, v, c.q);
                }
            }
        }
    }
#pragma unroll
    for (int k = 0; k < 4; k++) io[tid * 4 + k] = u128_to(x[k]);
}

int main() {
    cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0)); const int sms = p.multiProcessorCount;
    const int threads = 256, blocks = sms * 4, iters = 512;
    const size_t n = (size_t)threads * blocks * 4;
    std::vector<uint4> h(n); for (size_t i = 0; i < n; i++) h[i] = make_uint4(i * 2654435761u, i, 77, 0x0fffffff);
    uint4 *d, *dtw;
    CK(cudaMalloc(&d, n * 16)); CK(cudaMalloc(&dtw, 32));
    uint4 tw[2] = {make_uint4(0x12345, 0x6789, 0xabcdef, 0x0fffffff), make_uint4(0x54321, 0x9876, 0xfedcba, 0x0ffffff0)};
    CK(cudaMemcpy(dtw, tw, 32, cudaMemcpyHostToDevice));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int cls : {0, 3}) {
        unsigned __int128 q = cls == 0 ? (~(unsigned __int128)0 - 8257535 + 1) : (((unsigned __int128)1 << 125) - 262143);
        unsigned __int128 inv = 1; for (int i = 0; i < 7; i++) inv *= 2 - q * inv;
        QC c = {}; for (int i = 0; i < 4; i++) { c.q[i] = (uint32_t)(q >> (32 * i)); c.q2[i] = (uint32_t)((2 * q) >> (32 * i)); }
        c.qinv0 = (uint32_t)(-inv);
        unsigned long long hs[2];
        for (int v = 0; v < 2; v++) {
            CK(cudaMemcpy(d, h.data(), n * 16, cudaMemcpyHostToDevice));
            auto launch = [&]() {
                if (cls == 0) { if (v == 0) k<0, 0><<<blocks, threads>>>(d, dtw, c, iters); else k<1, 0><<<blocks, threads>>>(d, dtw, c, iters); }
                else { if (v == 0) k<0, 3><<<blocks, threads>>>(d, dtw, c, iters); else k<1, 3><<<blocks, threads>>>(d, dtw, c, iters); }
            };
            launch(); CK(cudaDeviceSynchronize());
            std::vector<uint4> r(n); CK(cudaMemcpy(r.data(), d, n * 16, cudaMemcpyDeviceToHost));
            unsigned long long x = 0; for (size_t i = 0; i < n; i++) x = x * 1000003ull + r[i].x + 7ull * r[i].w; hs[v] = x;
            float best = 1e30f;
            for (int r2 = 0; r2 < 3; r2++) { cudaEventRecord(e0); launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms); }
            const double bf = (double)threads * blocks * iters * 4;
            printf("{\"class\":\"%s\",\"variant\":\"%s\",\"bfly_per_clk_sm_at1965\":%.4f}\n", cls == 0 ? "FULL" : "LAZY", v == 0 ? "V0" : "VA", bf / (best * 1e-3) / (sms * 1.965e9));
        }
        printf("{\"class\":\"%s\",\"results_equal\":%d}\n", cls == 0 ? "FULL" : "LAZY", hs[0] == hs[1]);
    }
    return 0;
}
