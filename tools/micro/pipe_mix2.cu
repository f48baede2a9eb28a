// Which SASS classes contend with IMAD.WIDE.U32?  Streams (independent registers):
//  W: IMAD.WIDE carry chains, L: IMAD (lo) chains, A: IADD3.X carry chains, P: LOP3, H: IMAD.HI
#include <cstdio>
#include <cstdint>
#include <algorithm>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "CUDA %s\n", cudaGetErrorString(e)); return 1; } } while (0)

template <int W, int L, int A, int P, int H>
__global__ void k_mix(uint32_t* out, uint32_t seed, int iters) {
    uint32_t t[4][4], l[8], s[4][4], p[8], h[8];
    const uint32_t b0 = seed * 7u + blockIdx.x, b2 = b0 ^ 0x55u, c1 = b0 + 3;
#pragma unroll
    for (int k = 0; k < 4; k++)
#pragma unroll
        for (int j = 0; j < 4; j++) { t[k][j] = threadIdx.x * (k + 1) + j; s[k][j] = threadIdx.x ^ (k * 7 + j); }
#pragma unroll
    for (int k = 0; k < 8; k++) { l[k] = threadIdx.x + k; p[k] = threadIdx.x * 3 + k; h[k] = threadIdx.x * 5 + k; }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 4; k++)
            if (k < W)
                asm volatile("mad.lo.cc.u32 %0, %4, %5, %0;\n\t madc.hi.cc.u32 %1, %4, %5, %1;\n\t"
                             "madc.lo.cc.u32 %2, %4, %6, %2;\n\t madc.hi.u32 %3, %4, %6, %3;"
                             : "+r"(t[k][0]), "+r"(t[k][1]), "+r"(t[k][2]), "+r"(t[k][3]) : "r"(t[k][3]), "r"(b0), "r"(b2));
#pragma unroll
        for (int k = 0; k < 8; k++)
            if (k < L) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(l[k]) : "r"(b0), "r"(c1));
#pragma unroll
        for (int k = 0; k < 4; k++)
            if (k < A)
                asm volatile("add.cc.u32 %0, %0, %4;\n\t addc.cc.u32 %1, %1, %5;\n\t addc.cc.u32 %2, %2, %6;\n\t addc.u32 %3, %3, %7;"
                             : "+r"(s[k][0]), "+r"(s[k][1]), "+r"(s[k][2]), "+r"(s[k][3])
                             : "r"(s[(k + 1) % 4][3]), "r"(s[(k + 1) % 4][0]), "r"(b2), "r"(b0));
#pragma unroll
        for (int k = 0; k < 8; k++)
            if (k < P) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(p[k]) : "r"(p[(k + 1) % 8]), "r"(c1));
#pragma unroll
        for (int k = 0; k < 8; k++)
            if (k < H) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(h[k]) : "r"(b2), "r"(c1));
    }
    uint32_t x = 0;
#pragma unroll
    for (int k = 0; k < 4; k++)
#pragma unroll
        for (int j = 0; j < 4; j++) x ^= t[k][j] ^ s[k][j];
#pragma unroll
    for (int k = 0; k < 8; k++) x ^= l[k] ^ p[k] ^ h[k];
    if (x == 0x12345) out[0] = x;
}

template <int W, int L, int A, int P, int H>
int run(uint32_t* d, int sms, cudaEvent_t e0, cudaEvent_t e1) {
    const int threads = 256, blocks = sms * 8, iters = 4096;
    k_mix<W, L, A, P, H><<<blocks, threads>>>(d, 1, iters);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 3; r++) {
        cudaEventRecord(e0); k_mix<W, L, A, P, H><<<blocks, threads>>>(d, 1, iters); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
    }
    const double clk = best * 1e-3 * 1.965e9 * sms, lanes = (double)threads * blocks * iters;
    printf("{\"W\":%d,\"L\":%d,\"A\":%d,\"P\":%d,\"H\":%d,\"ms\":%.4f,\"wide/clk/sm\":%.1f,\"imad/clk/sm\":%.1f,\"add/clk/sm\":%.1f,\"lop/clk/sm\":%.1f,\"hi/clk/sm\":%.1f}\n",
           W, L, A, P, H, best, lanes * 2 * W / clk, lanes * L / clk, lanes * 4 * A / clk, lanes * P / clk, lanes * H / clk);
    return 0;
}

int main() {
    cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, 0)); int sms = pr.multiProcessorCount;
    uint32_t* d; CK(cudaMalloc(&d, 4));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    run<4, 0, 0, 0, 0>(d, sms, e0, e1);
    run<0, 8, 0, 0, 0>(d, sms, e0, e1);
    run<0, 0, 4, 0, 0>(d, sms, e0, e1);
    run<0, 0, 0, 8, 0>(d, sms, e0, e1);
    run<0, 0, 0, 0, 8>(d, sms, e0, e1);
    run<4, 8, 0, 0, 0>(d, sms, e0, e1);
    run<4, 0, 2, 0, 0>(d, sms, e0, e1);
    run<4, 0, 0, 8, 0>(d, sms, e0, e1);
    run<0, 8, 2, 0, 0>(d, sms, e0, e1);
    run<0, 8, 0, 8, 0>(d, sms, e0, e1);
    run<0, 0, 0, 8, 8>(d, sms, e0, e1);
    run<0, 0, 2, 0, 8>(d, sms, e0, e1);
    run<0, 8, 0, 0, 8>(d, sms, e0, e1);
    return 0;
}
