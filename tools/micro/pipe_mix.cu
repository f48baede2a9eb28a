// Does the IMAD.WIDE (fma-heavy) stream overlap with the IADD3.X (alu) stream?
// kernel M(w, a): per iteration w wide-product pairs (IMAD.WIDE carry chains) and
// a 4-word add-with-carry chains, on independent registers; time vs the parts alone.
#include <cstdio>
#include <cstdint>
#include <algorithm>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "CUDA %s\n", cudaGetErrorString(e)); return 1; } } while (0)

template <int W, int A>
__global__ void k_mix(uint32_t* out, uint32_t seed, int iters) {
    uint32_t t[4][4], s[4][4];
    uint32_t b0 = seed * 7u + blockIdx.x, b2 = b0 ^ 0x55u;
#pragma unroll
    for (int k = 0; k < 4; k++)
#pragma unroll
        for (int j = 0; j < 4; j++) { t[k][j] = threadIdx.x * (k + 1) + j; s[k][j] = threadIdx.x ^ (k * 7 + j); }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 4; k++) {
            if (k < W)
                asm volatile("mad.lo.cc.u32 %0, %4, %5, %0;\n\t madc.hi.cc.u32 %1, %4, %5, %1;\n\t"
                             "madc.lo.cc.u32 %2, %4, %6, %2;\n\t madc.hi.u32 %3, %4, %6, %3;"
                             : "+r"(t[k][0]), "+r"(t[k][1]), "+r"(t[k][2]), "+r"(t[k][3]) : "r"(t[k][3]), "r"(b0), "r"(b2));
        }
#pragma unroll
        for (int k = 0; k < 4; k++) {
            if (k < A)
                asm volatile("add.cc.u32 %0, %0, %4;\n\t addc.cc.u32 %1, %1, %5;\n\t addc.cc.u32 %2, %2, %6;\n\t addc.u32 %3, %3, %7;"
                             : "+r"(s[k][0]), "+r"(s[k][1]), "+r"(s[k][2]), "+r"(s[k][3])
                             : "r"(s[(k + 1) % 4][3]), "r"(s[(k + 1) % 4][0]), "r"(b2), "r"(b0));
        }
    }
    uint32_t x = 0;
#pragma unroll
    for (int k = 0; k < 4; k++)
#pragma unroll
        for (int j = 0; j < 4; j++) x ^= t[k][j] ^ s[k][j];
    if (x == 0x12345) out[0] = x;
}

template <int W, int A>
int run(uint32_t* d, int sms, cudaEvent_t e0, cudaEvent_t e1) {
    const int threads = 256, blocks = sms * 8, iters = 4096;
    k_mix<W, A><<<blocks, threads>>>(d, 1, iters);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 3; r++) {
        cudaEventRecord(e0); k_mix<W, A><<<blocks, threads>>>(d, 1, iters); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
    }
    double per_thread_iter_ns = best * 1e6 / ((double)iters);
    double wide = 2.0 * W, adds = 4.0 * A;   // IMAD.WIDE and 32-bit carry adds per iteration per thread
    double clk = best * 1e-3 * 1.965e9 * sms;  // SM-cycles available
    double lanes = (double)threads * blocks * iters;
    printf("{\"W\":%d,\"A\":%d,\"ms\":%.4f,\"wide_per_clk_sm\":%.2f,\"adds_per_clk_sm\":%.2f}\n", W, A, best,
           lanes * wide / clk, lanes * adds / clk);
    (void)per_thread_iter_ns;
    return 0;
}

int main() {
    cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0)); int sms = p.multiProcessorCount;
    uint32_t* d; CK(cudaMalloc(&d, 4));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    run<4, 0>(d, sms, e0, e1);
    run<0, 4>(d, sms, e0, e1);
    run<4, 4>(d, sms, e0, e1);
    run<4, 2>(d, sms, e0, e1);
    run<2, 4>(d, sms, e0, e1);
    run<4, 1>(d, sms, e0, e1);
    return 0;
}
