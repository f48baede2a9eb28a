// Does the modulus's location change the register-only butterfly rate?  Radix-4 register
// rounds (4 residues per thread, as the cfg3 pass kernel), 64 registers (16 warps... 32 warps
// per SM), FULL (canonical, q ~ 2^128) and LAZY (Harvey, q < 2^126) classes:
//   G: q, 2q, q' loaded from global memory (as k_ntt_pass does: vector registers);
//   P: q, 2q, q' in the kernel parameters (__grid_constant__: constant-bank operands / uniform registers);
//   A: an array of 64 moduli in the kernel parameters, indexed by a block-uniform index;
//   B: an array of 64 moduli in global memory, indexed by a block-uniform index.
// Results are checked equal between G and P.  Build: tools/micro/build.sh bfly_uniform
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "arith128.cuh"
using namespace ntt128;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

struct QC { uint32_t q[4], q2[4], qinv0; };

template <int V>   // 0 FULL, 3 LAZY
__device__ __forceinline__ void rounds(U128 (&x)[4], const U128 (&w)[2], const uint32_t q[4], const uint32_t q2[4], uint32_t qinv0, int iters) {
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int bit = 0; bit < 2; bit++) {
#pragma unroll
            for (int kk = 0; kk < 2; kk++) {
                const int k0 = ((kk >> bit) << (bit + 1)) | (kk & ((1 << bit) - 1));
                const int k1 = k0 | (1 << bit);
                const U128 u = x[k0];
                if (V == 3) {
                    const U128 us = reduce_2q(u, q2);
                    const U128 v = mont_mul_lazy(x[k1], w[(kk + bit) & 1], q, qinv0);
                    x[k0] = add_nored(us, v); x[k1] = sub_add_nored(us, v, q2);
                } else {
                    const U128 v = mont_mul(x[k1], w[(kk + bit) & 1], q, qinv0);
                    x[k0] = add_mod(u, v, q); x[k1] = sub_mod(u, v, q);
                }
            }
        }
    }
}

template <int V>
__global__ void __launch_bounds__(256, 4) k_g(uint4* io, const uint4* tw, const QC* qc, int iters) {
    const QC c = *qc;
    U128 x[4], w[2];
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
    for (int k = 0; k < 4; k++) x[k] = u128_from(io[tid * 4 + k]);
    w[0] = u128_from(tw[0]); w[1] = u128_from(tw[1]);
    rounds<V>(x, w, c.q, c.q2, c.qinv0, iters);
#pragma unroll
    for (int k = 0; k < 4; k++) io[tid * 4 + k] = u128_to(x[k]);
}
template <int V>
__global__ void __launch_bounds__(256, 4) k_p(uint4* io, const uint4* tw, const __grid_constant__ QC c, int iters) {
    U128 x[4], w[2];
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
    for (int k = 0; k < 4; k++) x[k] = u128_from(io[tid * 4 + k]);
    w[0] = u128_from(tw[0]); w[1] = u128_from(tw[1]);
    rounds<V>(x, w, c.q, c.q2, c.qinv0, iters);
#pragma unroll
    for (int k = 0; k < 4; k++) io[tid * 4 + k] = u128_to(x[k]);
}

struct QA { QC c[64]; };
template <int V>
__global__ void __launch_bounds__(256, 4) k_a(uint4* io, const uint4* tw, const __grid_constant__ QA qa, int iters) {
    const QC& c = qa.c[blockIdx.x & 63];
    U128 x[4], w[2];
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
    for (int k = 0; k < 4; k++) x[k] = u128_from(io[tid * 4 + k]);
    w[0] = u128_from(tw[0]); w[1] = u128_from(tw[1]);
    rounds<V>(x, w, c.q, c.q2, c.qinv0, iters);
#pragma unroll
    for (int k = 0; k < 4; k++) io[tid * 4 + k] = u128_to(x[k]);
}
template <int V>
__global__ void __launch_bounds__(256, 4) k_b(uint4* io, const uint4* tw, const QC* __restrict__ qa, int iters) {
    const QC c = qa[blockIdx.x & 63];
    U128 x[4], w[2];
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
    for (int k = 0; k < 4; k++) x[k] = u128_from(io[tid * 4 + k]);
    w[0] = u128_from(tw[0]); w[1] = u128_from(tw[1]);
    rounds<V>(x, w, c.q, c.q2, c.qinv0, iters);
#pragma unroll
    for (int k = 0; k < 4; k++) io[tid * 4 + k] = u128_to(x[k]);
}

int main() {
    cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0)); const int sms = p.multiProcessorCount;
    const int threads = 256, blocks = sms * 4, iters = 512;
    const size_t n = (size_t)threads * blocks * 4;
    std::vector<uint4> h(n); for (size_t i = 0; i < n; i++) h[i] = make_uint4(i * 2654435761u, i, 77, 0x0fffffff);
    uint4 *d, *dtw; QC* dq; QC* dqa;
    CK(cudaMalloc(&d, n * 16)); CK(cudaMalloc(&dtw, 32)); CK(cudaMalloc(&dq, sizeof(QC))); CK(cudaMalloc(&dqa, 64 * sizeof(QC)));
    static QA qa;
    uint4 tw[2] = {make_uint4(0x12345, 0x6789, 0xabcdef, 0x0fffffff), make_uint4(0x54321, 0x9876, 0xfedcba, 0x0ffffff0)};
    CK(cudaMemcpy(dtw, tw, 32, cudaMemcpyHostToDevice));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int cls : {0, 3}) {
        unsigned __int128 q = cls == 0 ? (~(unsigned __int128)0 - 8257535 + 1) : (((unsigned __int128)1 << 125) - 262143);
        unsigned __int128 inv = 1; for (int i = 0; i < 7; i++) inv *= 2 - q * inv;
        QC c = {}; for (int i = 0; i < 4; i++) { c.q[i] = (uint32_t)(q >> (32 * i)); c.q2[i] = (uint32_t)((2 * q) >> (32 * i)); }
        c.qinv0 = (uint32_t)(-inv);
        CK(cudaMemcpy(dq, &c, sizeof(QC), cudaMemcpyHostToDevice));
        for (int i = 0; i < 64; i++) qa.c[i] = c;
        CK(cudaMemcpy(dqa, qa.c, 64 * sizeof(QC), cudaMemcpyHostToDevice));
        unsigned long long hs[4];
        for (int v = 0; v < 4; v++) {
            CK(cudaMemcpy(d, h.data(), n * 16, cudaMemcpyHostToDevice));
            auto launch = [&]() {
                if (cls == 0) {
                    if (v == 0) k_g<0><<<blocks, threads>>>(d, dtw, dq, iters); else if (v == 1) k_p<0><<<blocks, threads>>>(d, dtw, c, iters);
                    else if (v == 2) k_a<0><<<blocks, threads>>>(d, dtw, qa, iters); else k_b<0><<<blocks, threads>>>(d, dtw, dqa, iters);
                } else {
                    if (v == 0) k_g<3><<<blocks, threads>>>(d, dtw, dq, iters); else if (v == 1) k_p<3><<<blocks, threads>>>(d, dtw, c, iters);
                    else if (v == 2) k_a<3><<<blocks, threads>>>(d, dtw, qa, iters); else k_b<3><<<blocks, threads>>>(d, dtw, dqa, iters);
                }
            };
            launch(); CK(cudaDeviceSynchronize());
            std::vector<uint4> r(n); CK(cudaMemcpy(r.data(), d, n * 16, cudaMemcpyDeviceToHost));
            unsigned long long x = 0; for (size_t i = 0; i < n; i++) x = x * 1000003ull + r[i].x + 7ull * r[i].w; hs[v] = x;
            float best = 1e30f;
            for (int k = 0; k < 3; k++) { cudaEventRecord(e0); launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms); }
            const double bf = (double)threads * blocks * iters * 4;
            printf("{\"class\":\"%s\",\"q_in\":\"%s\",\"bfly_per_clk_sm_at1965\":%.4f}\n", cls == 0 ? "FULL" : "LAZY", v == 0 ? "global" : (v == 1 ? "param" : (v == 2 ? "param_array_uniform_index" : "global_array_uniform_index")),
                   bf / (best * 1e-3) / (sms * 1.965e9));
        }
        printf("{\"class\":\"%s\",\"results_equal\":%d}\n", cls == 0 ? "FULL" : "LAZY", hs[0] == hs[1] && hs[0] == hs[2] && hs[0] == hs[3]);
    }
    return 0;
}
