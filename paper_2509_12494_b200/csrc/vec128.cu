// vec128.cu -- modular BLAS over one 128-bit modulus (§2.3):
// z = x + y, z = x - y, z = x * y, y = a x + y (all mod q), on [n][2] uint64 arrays.
//
// HBM-bound (48 bytes per element at ~6.5 TB/s vs <= 2 Montgomery products per
// element): a grid-stride loop over 16-byte elements, each thread
// keeping UNROLL independent elements in flight (vec_unroll below).
// vec128_mul is a general product: mont(mont(x, y), R^2) = x y mod q.
// axpy uses the host-converted Montgomery scalar a R mod q: mont(x, aR) = a x.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <cstdlib>

#include "../../include/ntt128.h"
#include "arith128.cuh"
#include "barrett128.cuh"
#include "psm128.cuh"
#include "host128.h"
#include "ntt128_internal.h"

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
    uint32_t psm_s, psm_C;   // OP_MULP: s = 128 - bitlen(q), C = 2^128 - q 2^s (psm128.cuh)
};

// OP_MUL: two Montgomery products (any odd q); OP_MULB: one Barrett product (q > 2^127,
// 43 word products instead of 72: barrett128.cuh).
// OP_MULP: q = 2^b - c with c 2^(128-b) < 2^32 (pseudo-Mersenne, psm128.cuh): the 256-bit product
// folds 2^128 = C modulo q 2^(128-b), 21 word products, then one canonicalisation.
enum Op { OP_ADD = 0, OP_SUB = 1, OP_MUL = 2, OP_AXPY = 3, OP_MULB = 4, OP_MULP = 5 };

__device__ __forceinline__ U128 mul_p(const U128& a, const U128& b, const uint32_t q[4], uint32_t s, uint32_t C) {
    return psm_canon(psm_mul(a, b, C), q, s, C);   // b < q (an input residue): the product is < Q
}

__device__ __forceinline__ U128 mul_b(const U128& a, const U128& b, const BarrettC& bc) {
    U128 r;
    barrett_mul_dev(a.w, b.w, bc, r.w);
    return r;
}

// Residues per thread and resident-CTA cap (tools/exp_vec_graph.py sweeps, profiles/r02/vec_sweep.txt):
// many small CTAs over several waves beat one wave of 4-residue threads -- a CTA that finishes
// is replaced by one whose loads then overlap its neighbours' products.  mul keeps 2 residues
// per thread (its 43-product Barrett needs the in-flight loads), add / sub / axpy take 1.
#ifndef NTT_VEC_PSM
#define NTT_VEC_PSM 1         // 0: vec128_mul never takes the pseudo-Mersenne product (A/B build)
#endif
#ifndef NTT_VEC_UNROLL_MUL
#define NTT_VEC_UNROLL_MUL 2
#endif
#ifndef NTT_VEC_UNROLL
#define NTT_VEC_UNROLL 1
#endif
#ifndef NTT_VEC_CTAS_PER_SM
#define NTT_VEC_CTAS_PER_SM 16
#endif
template <int OPK>
constexpr int vec_unroll() { return (OPK == OP_MUL || OPK == OP_MULB || OPK == OP_MULP) ? NTT_VEC_UNROLL_MUL : NTT_VEC_UNROLL; }
#ifndef NTT_VEC_THREADS
#define NTT_VEC_THREADS 256
#endif
constexpr int THREADS = NTT_VEC_THREADS;

template <int OPK, int UNROLL = 4>
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
            else if (OPK == OP_MULP) r = mul_p(a, b, c.q, c.psm_s, c.psm_C);
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
        else if (OPK == OP_MULP) r = mul_p(a, b, c.q, c.psm_s, c.psm_C);
        else r = add_mod(mont_mul(a, U128{{c.a_m[0], c.a_m[1], c.a_m[2], c.a_m[3]}}, c.q, c.qinv0), b, c.q);
        z[i] = u128_to(r);
    }
}

// ---- bulk-copy pipeline (DESIGN.md §6 "BLAS"): one producer lane streams chunks of x and y
// into a ring of shared-memory stages with cp.async.bulk (SASS UBLKCP), completion counted
// on an mbarrier per stage (expect_tx); consumer warps compute and store z.  HBM reads run
// from the first cycle at full depth whatever the consumers are doing, so the modular
// products of chunk i overlap the loads of chunks i+1 .. i+S-1 (the one-wave kernel above
// issues every thread's loads, then computes: its compute tail is exposed).
// Shape <consumer warps, residues per stage and operand, stages>: two CTAs per SM.
template <int CW, int CHUNK, int STAGES>
struct PipeShape {
    static constexpr int CWARPS = CW, PCHUNK = CHUNK, PSTAGES = STAGES;
    static constexpr int THREADS = 32 * (CW + 1);            // warp CW is the producer
    static constexpr size_t SMEM = (size_t)STAGES * 2 * CHUNK * sizeof(uint4);
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra W;\n\t}" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <int OPK>
__device__ __forceinline__ U128 vec_op1(const U128& a, const U128& b, const VecConst& c) {
    if (OPK == OP_ADD) return add_mod(a, b, c.q);
    if (OPK == OP_SUB) return sub_mod(a, b, c.q);
    if (OPK == OP_MUL) return mont_mul(mont_mul(a, b, c.q, c.qinv0), U128{{c.r2[0], c.r2[1], c.r2[2], c.r2[3]}}, c.q, c.qinv0);
    if (OPK == OP_MULB) return mul_b(a, b, c.bc);
    if (OPK == OP_MULP) return mul_p(a, b, c.q, c.psm_s, c.psm_C);
    return add_mod(mont_mul(a, U128{{c.a_m[0], c.a_m[1], c.a_m[2], c.a_m[3]}}, c.q, c.qinv0), b, c.q);
}

template <int OPK, class PS>
__global__ void __launch_bounds__(PS::THREADS, 2) k_vec_pipe(uint4* z, const uint4* x, const uint4* y, uint64_t n,
                                                            const VecConst c) {
    constexpr int PIPE_CWARPS = PS::CWARPS, PIPE_CHUNK = PS::PCHUNK, PIPE_STAGES = PS::PSTAGES;
    extern __shared__ __align__(128) uint4 ring[];              // [STAGES][2][CHUNK]
    __shared__ __align__(8) uint64_t full[PIPE_STAGES], empty[PIPE_STAGES];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < PIPE_STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], PIPE_CWARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint64_t nchunks = (n + PIPE_CHUNK - 1) / PIPE_CHUNK;
    if (warp == PIPE_CWARPS) {                                    // producer
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (uint64_t k = blockIdx.x; k < nchunks; k += gridDim.x) {
                mbar_wait(&empty[s], ph ^ 1);                    // consumers released this stage
                const uint64_t e0 = k * PIPE_CHUNK;
                const uint32_t cnt = (uint32_t)(n - e0 < (uint64_t)PIPE_CHUNK ? n - e0 : PIPE_CHUNK);
                mbar_expect_tx(&full[s], 2 * cnt * 16);
                bulk_g2s(ring + (2 * s) * PIPE_CHUNK, x + e0, cnt * 16, &full[s]);
                bulk_g2s(ring + (2 * s + 1) * PIPE_CHUNK, y + e0, cnt * 16, &full[s]);
                if (++s == PIPE_STAGES) { s = 0; ph ^= 1; }
            }
        }
        return;
    }
    int s = 0;
    uint32_t ph = 0;
    constexpr int PER = PIPE_CHUNK / (32 * PIPE_CWARPS);        // residues per consumer thread per stage
    for (uint64_t k = blockIdx.x; k < nchunks; k += gridDim.x) {
        mbar_wait(&full[s], ph);
        const uint64_t e0 = k * PIPE_CHUNK;
        const uint4* xs = ring + (2 * s) * PIPE_CHUNK;
        const uint4* ys = ring + (2 * s + 1) * PIPE_CHUNK;
        uint4 xv[PER], yv[PER];
#pragma unroll
        for (int u = 0; u < PER; u++) {
            const int i = threadIdx.x + u * 32 * PIPE_CWARPS;
            xv[u] = xs[i];
            yv[u] = ys[i];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);                   // the stage may be refilled
#pragma unroll
        for (int u = 0; u < PER; u++) {
            const uint64_t i = e0 + threadIdx.x + u * 32 * PIPE_CWARPS;
            if (i < n) z[i] = u128_to(vec_op1<OPK>(u128_from(xv[u]), u128_from(yv[u]), c));
        }
        if (++s == PIPE_STAGES) { s = 0; ph ^= 1; }
    }
}
#ifndef NTT_VEC_PIPE_MASK
#define NTT_VEC_PIPE_MASK 0   // ops on the pipeline kernel (bit OPK); measured: DESIGN.md §6 "BLAS"
#endif
using Pipe0 = PipeShape<8, 512, 6>;
using Pipe1 = PipeShape<16, 1024, 3>;
using Pipe2 = PipeShape<16, 512, 6>;
#ifndef NTT_VEC_PIPE_CFG
#define NTT_VEC_PIPE_CFG 1
#endif
template <int OPK, class PS>
cudaError_t launch_pipe_s(cudaLaunchConfig_t& pc, uint4* z, const uint4* x, const uint4* y, uint64_t n, const VecConst& c) {
    static bool attr = false;   // > 48 KB of dynamic shared memory
    if (!attr) {
        cudaFuncSetAttribute(k_vec_pipe<OPK, PS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PS::SMEM);
        attr = true;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t nchunks = (n + PS::PCHUNK - 1) / PS::PCHUNK;
    uint64_t g = (uint64_t)sms * 2;
    if (g > nchunks) g = nchunks;
    pc.gridDim = dim3((unsigned)g);
    pc.blockDim = dim3(PS::THREADS);
    pc.dynamicSmemBytes = PS::SMEM;
    return cudaLaunchKernelEx(&pc, k_vec_pipe<OPK, PS>, z, x, y, n, c);
}
template <int OPK>
cudaError_t launch_pipe(cudaLaunchConfig_t& pc, uint4* z, const uint4* x, const uint4* y, uint64_t n, const VecConst& c) {
#if NTT128_EXPERIMENTS
    static const int cfg = getenv("NTT128_VEC_PIPE_CFG") ? atoi(getenv("NTT128_VEC_PIPE_CFG")) : NTT_VEC_PIPE_CFG;
    if (cfg == 0) return launch_pipe_s<OPK, Pipe0>(pc, z, x, y, n, c);
    if (cfg == 2) return launch_pipe_s<OPK, Pipe2>(pc, z, x, y, n, c);
    return launch_pipe_s<OPK, Pipe1>(pc, z, x, y, n, c);
#else
#if NTT_VEC_PIPE_CFG == 0
    return launch_pipe_s<OPK, Pipe0>(pc, z, x, y, n, c);
#elif NTT_VEC_PIPE_CFG == 2
    return launch_pipe_s<OPK, Pipe2>(pc, z, x, y, n, c);
#else
    return launch_pipe_s<OPK, Pipe1>(pc, z, x, y, n, c);
#endif
#endif
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

int grid_for(uint64_t n, int unroll) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint64_t want = (n + (uint64_t)THREADS * unroll - 1) / ((uint64_t)THREADS * unroll);
#if NTT128_EXPERIMENTS
    static const int per_sm = getenv("NTT128_VEC_CTAS_PER_SM") ? atoi(getenv("NTT128_VEC_CTAS_PER_SM")) : NTT_VEC_CTAS_PER_SM;
#else
    constexpr int per_sm = NTT_VEC_CTAS_PER_SM;
#endif
    uint64_t cap = (uint64_t)sms * per_sm;  // CTAs per SM over the launch (several waves)
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
    uint64_t g0, g1;
    ntt128_stream_gen(stream, &g0, &g1);   // NTT128_FLAG_CHAIN: other library work on the stream
    ntt128h::Mont M(q);
    VecConst c;
    c.psm_s = 0;
    c.psm_C = 0;
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
    // pseudo-Mersenne moduli (words 1..3 of q 2^s all ones, C != 2^32 - 1) take the folding product
    bool psm = false;
    if (NTT_VEC_PSM && op == OP_MUL) {
        int s = 0;
        while (((q << s) >> 127) == 0) s++;
        const u128 Q = q << s;
        psm = (Q >> 32) == (((u128)1 << 96) - 1) && (uint32_t)Q != 1u;
        c.psm_s = (uint32_t)s;
        c.psm_C = 0u - (uint32_t)Q;
    }
    const bool barrett = (q >> 127) != 0 && !no_barrett && !psm;
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
    const int grid = grid_for(n, op == OP_MUL ? NTT_VEC_UNROLL_MUL : NTT_VEC_UNROLL);
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
    // mul and axpy (compute ~70 % of their HBM time) run the bulk-copy pipeline; add / sub
    // (a handful of ALU ops per element) the one-wave kernel (DESIGN.md §6 "BLAS")
#if NTT128_EXPERIMENTS
    static const int pipe_mask = getenv("NTT128_VEC_PIPE") ? atoi(getenv("NTT128_VEC_PIPE")) : NTT_VEC_PIPE_MASK;
#else
    constexpr int pipe_mask = NTT_VEC_PIPE_MASK;
#endif
    const int opk = (op == OP_MUL && barrett) ? OP_MULB : op;
    if (!psm && ((pipe_mask >> opk) & 1)) {
        cudaLaunchConfig_t pc;
        memset(&pc, 0, sizeof(pc));
        pc.stream = stream;
        cudaLaunchAttribute pa[1];
        pa[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        pa[0].val.programmaticStreamSerializationAllowed = 1;
        pc.attrs = pa;
        pc.numAttrs = 1;
        cudaError_t e;
        switch (opk) {
            case OP_ADD: e = launch_pipe<OP_ADD>(pc, z, x, y, n, c); break;
            case OP_SUB: e = launch_pipe<OP_SUB>(pc, z, x, y, n, c); break;
            case OP_MUL: e = launch_pipe<OP_MUL>(pc, z, x, y, n, c); break;
            case OP_MULB: e = launch_pipe<OP_MULB>(pc, z, x, y, n, c); break;
            default: e = launch_pipe<OP_AXPY>(pc, z, x, y, n, c); break;
        }
        ntt128_count_launch(1);
        return e == cudaSuccess && cudaGetLastError() == cudaSuccess ? NTT128_OK : NTT128_ERR_CUDA;
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
        case OP_ADD: e = cudaLaunchKernelEx(&cfg, k_vec<OP_ADD, vec_unroll<OP_ADD>()>, z, x, y, (uint64_t)n, c); break;
        case OP_SUB: e = cudaLaunchKernelEx(&cfg, k_vec<OP_SUB, vec_unroll<OP_SUB>()>, z, x, y, (uint64_t)n, c); break;
        case OP_MUL:
            e = psm ? cudaLaunchKernelEx(&cfg, k_vec<OP_MULP, vec_unroll<OP_MULP>()>, z, x, y, (uint64_t)n, c)
                : barrett ? cudaLaunchKernelEx(&cfg, k_vec<OP_MULB, vec_unroll<OP_MULB>()>, z, x, y, (uint64_t)n, c)
                          : cudaLaunchKernelEx(&cfg, k_vec<OP_MUL, vec_unroll<OP_MUL>()>, z, x, y, (uint64_t)n, c);
            break;
        default: e = cudaLaunchKernelEx(&cfg, k_vec<OP_AXPY, vec_unroll<OP_AXPY>()>, z, x, y, (uint64_t)n, c); break;
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
