// vec128.cu -- modular BLAS over one 128-bit modulus (§2.3):
// z = x + y, z = x - y, z = x * y, y = a x + y (all mod q), on [n][2] uint64 arrays.
//
// HBM-bound (48 bytes per element at ~6.5 TB/s vs <= 2 Montgomery products per
// element): a grid-stride loop over 16-byte elements, each thread
// keeping UNROLL independent elements in flight for memory-level parallelism.
// vec128_mul is a general product: mont(mont(x, y), R^2) = x y mod q.
// axpy uses the host-converted Montgomery scalar a R mod q: mont(x, aR) = a x.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <cstdlib>

#include "../../include/ntt128.h"
#include "arith128.cuh"
#include "barrett128.cuh"
#include "host128.h"

#ifndef NTT128_EXPERIMENTS
#define NTT128_EXPERIMENTS 0   // 1: experiment build (environment switches; never the product .so)
#endif

using namespace ntt128;
using ntt128h::u128;

void ntt128_count_launch(uint64_t k);

namespace {

struct VecConst {
    uint32_t q[4];
    uint32_t qinv0;
    uint32_t a_m[4];  // axpy scalar, Montgomery form
    uint32_t r2[4];   // R^2 mod q
    BarrettC bc;      // q and mu' = floor(2^256 / q) - 2^128 (OP_MULB: q > 2^127)
};

// OP_MUL: two Montgomery products (any odd q); OP_MULB: one Barrett product (q > 2^127,
// 43 word products instead of 72: barrett128.cuh).
enum Op { OP_ADD = 0, OP_SUB = 1, OP_MUL = 2, OP_AXPY = 3, OP_MULB = 4 };

__device__ __forceinline__ U128 mul_b(const U128& a, const U128& b, const BarrettC& bc) {
    U128 r;
    barrett_mul_dev(a.w, b.w, bc, r.w);
    return r;
}

constexpr int UNROLL = 4;
constexpr int THREADS = 256;

template <int OPK>
__global__ void __launch_bounds__(THREADS) k_vec(uint4* z, const uint4* __restrict__ x,
                                                 const uint4* y, uint64_t n, const VecConst c) {
    // programmatic dependent launch: wait for the previous kernel's writes, then let the
    // next one be scheduled as this grid drains (its launch latency overlaps our tail)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (UNROLL - 1) * stride < n; i += UNROLL * stride) {
        uint4 xv[UNROLL], yv[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; u++) {
            xv[u] = x[i + u * stride];
            yv[u] = y[i + u * stride];
        }
#pragma unroll
        for (int u = 0; u < UNROLL; u++) {
            U128 a = u128_from(xv[u]), b = u128_from(yv[u]), r;
            if (OPK == OP_ADD) r = add_mod(a, b, c.q);
            else if (OPK == OP_SUB) r = sub_mod(a, b, c.q);
            else if (OPK == OP_MUL) r = mont_mul(mont_mul(a, b, c.q, c.qinv0), U128{{c.r2[0], c.r2[1], c.r2[2], c.r2[3]}}, c.q, c.qinv0);
            else if (OPK == OP_MULB) r = mul_b(a, b, c.bc);
            else r = add_mod(mont_mul(a, U128{{c.a_m[0], c.a_m[1], c.a_m[2], c.a_m[3]}}, c.q, c.qinv0), b, c.q);
            z[i + u * stride] = u128_to(r);
        }
    }
    for (; i < n; i += stride) {
        U128 a = u128_from(x[i]), b = u128_from(y[i]), r;
        if (OPK == OP_ADD) r = add_mod(a, b, c.q);
        else if (OPK == OP_SUB) r = sub_mod(a, b, c.q);
        else if (OPK == OP_MUL) r = mont_mul(mont_mul(a, b, c.q, c.qinv0), U128{{c.r2[0], c.r2[1], c.r2[2], c.r2[3]}}, c.q, c.qinv0);
        else if (OPK == OP_MULB) r = mul_b(a, b, c.bc);
        else r = add_mod(mont_mul(a, U128{{c.a_m[0], c.a_m[1], c.a_m[2], c.a_m[3]}}, c.q, c.qinv0), b, c.q);
        z[i] = u128_to(r);
    }
}

__global__ void k_vec_check(const uint4* __restrict__ x, const uint4* __restrict__ y, uint64_t n, const VecConst c,
                            int* err) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        if (!lt_q(u128_from(x[i]), c.q) || !lt_q(u128_from(y[i]), c.q)) atomicOr(err, 1);
    }
}

void words(u128 v, uint32_t w[4]) {
    for (int i = 0; i < 4; i++) w[i] = (uint32_t)(v >> (32 * i));
}

int grid_for(uint64_t n) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint64_t want = (n + (uint64_t)THREADS * UNROLL - 1) / ((uint64_t)THREADS * UNROLL);
#if NTT128_EXPERIMENTS
    static const int per_sm = getenv("NTT128_VEC_CTAS_PER_SM") ? atoi(getenv("NTT128_VEC_CTAS_PER_SM")) : 8;
#else
    constexpr int per_sm = 8;
#endif
    uint64_t cap = (uint64_t)sms * per_sm;  // resident 256-thread CTAs per SM
    if (want > cap) want = cap;
    return want < 1 ? 1 : (int)want;
}

ntt128_status vec_op(int op, uint64_t* d_z, const uint64_t* d_x, const uint64_t* d_y, size_t n, const uint64_t* q_,
                     const uint64_t* a_, uint32_t flags, cudaStream_t stream) {
    if (!q_ || (op == OP_AXPY && !a_)) return NTT128_ERR_INVALID_ARG;
    if (flags & ~NTT128_FLAG_CHECK_INPUT) return NTT128_ERR_INVALID_ARG;
    const u128 q = ntt128h::make(q_[0], q_[1]);
    if ((q & 1) == 0 || q < 3) return NTT128_ERR_MODULUS;
    if (n == 0) return NTT128_OK;
    if (!d_z || !d_x || !d_y) return NTT128_ERR_INVALID_ARG;
    if (((uintptr_t)d_z | (uintptr_t)d_x | (uintptr_t)d_y) & 15u) return NTT128_ERR_ALIGNMENT;
    ntt128h::Mont M(q);
    VecConst c;
    words(q, c.q);
    c.qinv0 = (uint32_t)M.qp;
    words(M.r2, c.r2);
    u128 a = 0;
    if (op == OP_AXPY) {
        a = ntt128h::make(a_[0], a_[1]);
        if (a >= q) return NTT128_ERR_INPUT_RANGE;
    }
    words(M.to_m(a), c.a_m);
#if NTT128_EXPERIMENTS
    static const bool no_barrett = getenv("NTT128_NO_BARRETT") != nullptr;   // experiment build only (A/B)
#else
    constexpr bool no_barrett = false;
#endif
    const bool barrett = (q >> 127) != 0 && !no_barrett;
    if (barrett) {
        // mu = floor((2^256 - 1) / q) (= floor(2^256 / q), q odd) by restoring division
        u128 rem = 0, quo_lo = 0;
        uint32_t quo_hi = 0;   // quotient bit 128
        for (int i = 255; i >= 0; i--) {
            const bool top = (rem >> 127) != 0;
            rem = (rem << 1) | 1;
            quo_hi = (uint32_t)((quo_hi << 1) | (uint32_t)(quo_lo >> 127));
            quo_lo <<= 1;
            if (top || rem >= q) { rem -= q; quo_lo |= 1; }
        }
        (void)quo_hi;   // == 1 for 2^127 < q < 2^128: mu = 2^128 + quo_lo
        words(q, c.bc.q);
        words(quo_lo, c.bc.mu);
    }
    const uint4* x = (const uint4*)d_x;
    const uint4* y = (const uint4*)d_y;
    uint4* z = (uint4*)d_z;
    const int grid = grid_for(n);
    if (flags & NTT128_FLAG_CHECK_INPUT) {
        int* d_err = nullptr;
        int h = 0;
        if (cudaMallocAsync(&d_err, sizeof(int), stream) != cudaSuccess) return NTT128_ERR_OOM;
        cudaMemsetAsync(d_err, 0, sizeof(int), stream);
        k_vec_check<<<grid, THREADS, 0, stream>>>(x, y, n, c, d_err);
        ntt128_count_launch(1);
        cudaMemcpyAsync(&h, d_err, sizeof(int), cudaMemcpyDeviceToHost, stream);
        cudaFreeAsync(d_err, stream);
        if (cudaStreamSynchronize(stream) != cudaSuccess) return NTT128_ERR_CUDA;
        if (h) return NTT128_ERR_INPUT_RANGE;
    }
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(THREADS);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e;
    switch (op) {
        case OP_ADD: e = cudaLaunchKernelEx(&cfg, k_vec<OP_ADD>, z, x, y, (uint64_t)n, c); break;
        case OP_SUB: e = cudaLaunchKernelEx(&cfg, k_vec<OP_SUB>, z, x, y, (uint64_t)n, c); break;
        case OP_MUL:
            e = barrett ? cudaLaunchKernelEx(&cfg, k_vec<OP_MULB>, z, x, y, (uint64_t)n, c)
                        : cudaLaunchKernelEx(&cfg, k_vec<OP_MUL>, z, x, y, (uint64_t)n, c);
            break;
        default: e = cudaLaunchKernelEx(&cfg, k_vec<OP_AXPY>, z, x, y, (uint64_t)n, c); break;
    }
    ntt128_count_launch(1);
    return e == cudaSuccess && cudaGetLastError() == cudaSuccess ? NTT128_OK : NTT128_ERR_CUDA;
}

}  // namespace

extern "C" ntt128_status vec128_add(uint64_t* d_z, const uint64_t* d_x, const uint64_t* d_y, size_t n, const uint64_t* q,
                                    uint32_t flags, ntt128_stream_t stream) {
    return vec_op(OP_ADD, d_z, d_x, d_y, n, q, nullptr, flags, (cudaStream_t)stream);
}
extern "C" ntt128_status vec128_sub(uint64_t* d_z, const uint64_t* d_x, const uint64_t* d_y, size_t n, const uint64_t* q,
                                    uint32_t flags, ntt128_stream_t stream) {
    return vec_op(OP_SUB, d_z, d_x, d_y, n, q, nullptr, flags, (cudaStream_t)stream);
}
extern "C" ntt128_status vec128_mul(uint64_t* d_z, const uint64_t* d_x, const uint64_t* d_y, size_t n, const uint64_t* q,
                                    uint32_t flags, ntt128_stream_t stream) {
    return vec_op(OP_MUL, d_z, d_x, d_y, n, q, nullptr, flags, (cudaStream_t)stream);
}
// y <- a x + y: z = y (in place), "x" operand = d_x, "y" operand = d_y
extern "C" ntt128_status vec128_axpy(uint64_t* d_y, const uint64_t* a, const uint64_t* d_x, size_t n, const uint64_t* q,
                                     uint32_t flags, ntt128_stream_t stream) {
    return vec_op(OP_AXPY, d_y, d_x, d_y, n, q, a, flags, (cudaStream_t)stream);
}
