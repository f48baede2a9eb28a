// Register-only radix-2 butterfly throughput (no memory traffic): the compute
// ceiling of the NTT pass kernel's arithmetic.  Variants of add/sub mod q:
//   V0: product arith128.cuh (select by LOP3 masks)
//   V1: 3-input IADD3 chain + predicated correction
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "arith_variants.cuh"
using namespace ntt128;
#ifndef EPT
#define EPT 8
#endif
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

// a + b mod q: d = a + b - q in one 3-input chain; if it borrowed (d < 0), add q back
__device__ __forceinline__ U128 add_mod_p(const U128& a, const U128& b, const uint32_t q[4]) {
    U128 r;
    asm("{\n\t.reg .u32 t;\n\t.reg .pred p;\n\t"
        "add.cc.u32  %0, %4, %8;\n\t"
        "addc.cc.u32 %1, %5, %9;\n\t"
        "addc.cc.u32 %2, %6, %10;\n\t"
        "addc.cc.u32 %3, %7, %11;\n\t"
        "addc.u32    t, 0, 0;\n\t"
        "sub.cc.u32  %0, %0, %12;\n\t"
        "subc.cc.u32 %1, %1, %13;\n\t"
        "subc.cc.u32 %2, %2, %14;\n\t"
        "subc.cc.u32 %3, %3, %15;\n\t"
        "subc.u32    t, t, 0;\n\t"
        "setp.ne.u32 p, t, 0;\n\t"
        "@p add.cc.u32  %0, %0, %12;\n\t"
        "@p addc.cc.u32 %1, %1, %13;\n\t"
        "@p addc.cc.u32 %2, %2, %14;\n\t"
        "@p addc.u32    %3, %3, %15;\n\t}"
        : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3])
        : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]), "r"(b.w[3]),
          "r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]));
    return r;
}
// a - b mod q: borrow chain; if borrowed add q
__device__ __forceinline__ U128 sub_mod_p(const U128& a, const U128& b, const uint32_t q[4]) {
    U128 r;
    asm("{\n\t.reg .u32 t;\n\t.reg .pred p;\n\t"
        "sub.cc.u32  %0, %4, %8;\n\t"
        "subc.cc.u32 %1, %5, %9;\n\t"
        "subc.cc.u32 %2, %6, %10;\n\t"
        "subc.cc.u32 %3, %7, %11;\n\t"
        "subc.u32    t, 0, 0;\n\t"
        "setp.ne.u32 p, t, 0;\n\t"
        "@p add.cc.u32  %0, %0, %12;\n\t"
        "@p addc.cc.u32 %1, %1, %13;\n\t"
        "@p addc.cc.u32 %2, %2, %14;\n\t"
        "@p addc.u32    %3, %3, %15;\n\t}"
        : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3])
        : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]), "r"(b.w[3]),
          "r"(q[0]), "r"(q[1]), "r"(q[2]), "r"(q[3]));
    return r;
}

template <int V, int E>
__global__ void __launch_bounds__(256) k_bfly(uint4* io, const uint4* tw, const ModC* mods, int iters, int* bad) {
    const ModC M = mods[V == 2 ? (threadIdx.x >> 10) : 0];
    const uint32_t q[4] = {M.q[0], M.q[1], M.q[2], M.q[3]};
    U128 x[E], w[E / 2];
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
    for (int k = 0; k < E; k++) x[k] = u128_from(io[tid * E + k]);
#pragma unroll
    for (int k = 0; k < E / 2; k++) w[k] = u128_from(tw[k]);
    constexpr int RB = E == 2 ? 1 : (E == 4 ? 2 : 3);   // stages per register round
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int bit = 0; bit < RB; bit++) {
#pragma unroll
            for (int kk = 0; kk < E / 2; kk++) {
                const int k0 = ((kk >> bit) << (bit + 1)) | (kk & ((1 << bit) - 1));
                const int k1 = k0 | (1 << bit);
                const U128 u = x[k0];
                const uint32_t q2[4] = {M.r2[0], M.r2[1], M.r2[2], M.r2[3]};   // r2 slot holds 2q here
                if (V == 3) {          // Harvey (q < 2^126), values in [0, 4q)
                    const U128 us = reduce_2q(u, q2);
                    const U128 v = mont_mul_lazy(x[k1], w[(kk + bit) % (E / 2)], q, M.qinv0);
                    x[k0] = add_nored(us, v); x[k1] = sub_add_nored(us, v, q2);
                    continue;
                }
                if (V == 5) {          // half-lazy (q < 2^127), values in [0, 2q)
                    const U128 v = mont_mul_lazy(x[k1], w[(kk + bit) % (E / 2)], q, M.qinv0);
                    x[k0] = add_mod(u, v, q2); x[k1] = sub_mod(u, v, q2);
                    continue;
                }
                const U128 v = V == 4 ? mont_mul_v1(x[k1], w[(kk + bit) % (E / 2)], q, M.qinv0)
                                      : mont_mul(x[k1], w[(kk + bit) % (E / 2)], q, M.qinv0);
                if (V != 1) { x[k0] = add_mod(u, v, q); x[k1] = sub_mod(u, v, q); }
                else { x[k0] = add_mod_p(u, v, q); x[k1] = sub_mod_p(u, v, q); }
            }
        }
    }
#pragma unroll
    for (int k = 0; k < E; k++) io[tid * E + k] = u128_to(x[k]);
}

int main() {
    cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0)); int sms = p.multiProcessorCount;
    unsigned __int128 q = ~(unsigned __int128)0 - 8257535 + 1;  // cfg2 prime
    unsigned __int128 inv = 1; for (int i = 0; i < 7; i++) inv *= 2 - q * inv;
    ModC mc = {}; for (int i = 0; i < 4; i++) mc.q[i] = (uint32_t)(q >> (32 * i)); mc.qinv0 = (uint32_t)(-inv);
    constexpr int E = EPT;
    const int threads = 256, iters = 256;
    ModC* dm; uint4* dtw; int* dbad; CK(cudaMalloc(&dm, sizeof(ModC))); CK(cudaMemcpy(dm, &mc, sizeof(ModC), cudaMemcpyHostToDevice));
    std::vector<uint4> tw(E / 2); for (int k = 0; k < E / 2; k++) tw[k] = make_uint4(0x12345 + k, 0x6789 * k, 0xabcdef, 0x0fffffff);
    CK(cudaMalloc(&dtw, 16 * E)); CK(cudaMemcpy(dtw, tw.data(), 16 * E / 2, cudaMemcpyHostToDevice)); CK(cudaMalloc(&dbad, 4));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    {   // lazy variant on a 125-bit prime (q = 2^125 - 2^18... any odd q < 2^126 for timing)
        unsigned __int128 q5 = ((unsigned __int128)1 << 125) - 262143;  // 2^125 - 2^18 + 1
        unsigned __int128 inv5 = 1; for (int i = 0; i < 7; i++) inv5 *= 2 - q5 * inv5;
        ModC m5 = {}; for (int i = 0; i < 4; i++) { m5.q[i] = (uint32_t)(q5 >> (32 * i)); m5.r2[i] = (uint32_t)((2 * q5) >> (32 * i)); }
        m5.qinv0 = (uint32_t)(-inv5);
        ModC* dm5; CK(cudaMalloc(&dm5, sizeof(ModC))); CK(cudaMemcpy(dm5, &m5, sizeof(ModC), cudaMemcpyHostToDevice));
        const int blocks = sms * 3; size_t n = (size_t)threads * blocks * E;
        std::vector<uint4> h(n); for (size_t i = 0; i < n; i++) h[i] = make_uint4(i * 2654435761u, i, 77, 0x0fffffff);
        uint4* d; CK(cudaMalloc(&d, n * 16)); CK(cudaMemcpy(d, h.data(), n * 16, cudaMemcpyHostToDevice));
        for (int v : {0, 3, 5}) {
            auto launch = [&]() { if (v == 0) k_bfly<0, E><<<blocks, threads>>>(d, dtw, dm5, iters, dbad); else if (v == 3) k_bfly<3, E><<<blocks, threads>>>(d, dtw, dm5, iters, dbad); else k_bfly<5, E><<<blocks, threads>>>(d, dtw, dm5, iters, dbad); };
            launch(); CK(cudaDeviceSynchronize());
            float best = 1e30f;
            for (int r = 0; r < 3; r++) { cudaEventRecord(e0); launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms); }
            double bf = (double)threads * blocks * iters * (E == 4 ? 2 : 3) * (E / 2);
            printf("{\"q125_variant\":%d,\"bfly_per_clk_sm_at1965\":%.3f}\n", v, bf / (best * 1e-3) / (sms * 1.965e9));
        }
        // saturation curve: butterflies/clk/SM against resident warps (8 .. 32 per SM)
        for (int bpsm : {1, 2, 3, 4}) {
            const int blocks2 = sms * bpsm;
            for (int v : {0, 3}) {
                auto launch = [&]() { if (v == 0) k_bfly<0, E><<<blocks2, threads>>>(d, dtw, dm5, iters, dbad); else k_bfly<3, E><<<blocks2, threads>>>(d, dtw, dm5, iters, dbad); };
                if (bpsm > 3) { cudaFree(d); CK(cudaMalloc(&d, (size_t)threads * blocks2 * E * 16)); CK(cudaMemset(d, 0, (size_t)threads * blocks2 * E * 16)); }
                launch(); CK(cudaDeviceSynchronize());
                float best = 1e30f;
                for (int r = 0; r < 3; r++) { cudaEventRecord(e0); launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms); }
                double bf = (double)threads * blocks2 * iters * (E == 4 ? 2 : 3) * (E / 2);
                int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, v == 0 ? (const void*)k_bfly<0, E> : (const void*)k_bfly<3, E>, threads, 0);
                printf("{\"curve_variant\":%d,\"ept\":%d,\"warps_per_sm\":%d,\"occ_blocks\":%d,\"bfly_per_clk_sm_at1965\":%.3f}\n", v, E, bpsm * 8, occ, bf / (best * 1e-3) / (sms * 1.965e9));
            }
        }
        cudaFree(d);
    }
    for (int bpsm : {3}) {
        const int blocks = sms * bpsm;
        size_t n = (size_t)threads * blocks * E;
        std::vector<uint4> h(n); for (size_t i = 0; i < n; i++) h[i] = make_uint4(i * 2654435761u, i, 77, 0x7fffffff);
        uint4* d; CK(cudaMalloc(&d, n * 16));
        unsigned long long hsh[5];
        for (int v = 0; v < 5; v++) {
            CK(cudaMemcpy(d, h.data(), n * 16, cudaMemcpyHostToDevice));
            auto launch = [&]() { if (v == 0) k_bfly<0, E><<<blocks, threads>>>(d, dtw, dm, iters, dbad); else if (v == 1) k_bfly<1, E><<<blocks, threads>>>(d, dtw, dm, iters, dbad); else if (v == 2) k_bfly<2, E><<<blocks, threads>>>(d, dtw, dm, iters, dbad); else if (v == 3) k_bfly<4, E><<<blocks, threads>>>(d, dtw, dm, iters, dbad); else k_bfly<0, E><<<blocks, threads>>>(d, dtw, dm, iters, dbad); };
            launch(); CK(cudaDeviceSynchronize());
            std::vector<uint4> res(n); CK(cudaMemcpy(res.data(), d, n * 16, cudaMemcpyDeviceToHost));
            unsigned long long hs = 0; for (size_t i = 0; i < n; i++) hs = hs * 1000003ull + res[i].x + 7ull * res[i].w; hsh[v] = hs;
            float best = 1e30f;
            for (int r = 0; r < 3; r++) { cudaEventRecord(e0); launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms); }
            double bf = (double)threads * blocks * iters * (E == 4 ? 2 : 3) * (E / 2);
            printf("{\"variant\":%d,\"blocks_per_sm\":%d,\"ms\":%.4f,\"bfly_per_s\":%.4e,\"bfly_per_clk_sm_at1965\":%.3f}\n", v, bpsm, best, bf / (best * 1e-3), bf / (best * 1e-3) / (sms * 1.965e9));
        }
        printf("{\"blocks_per_sm\":%d,\"hash_equal\":%d}\n", bpsm, hsh[0] == hsh[1] && hsh[0] == hsh[2] && hsh[0] == hsh[3]);
        cudaFree(d);
    }
    return 0;
}
