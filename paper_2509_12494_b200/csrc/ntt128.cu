// ntt128.cu -- 128-bit modular NTT for sm_100a behind the C ABI of include/ntt128.h.
//
// Method: the radix-2 NTT of Eq. ntt, log N stages of N/2
// butterflies, each "one modular addition, one modular subtraction, and one
// modular multiplication" (§3.2).  The paper's x86 dataflow (Pease
// with unpack/permute) is replaced by a GPU dataflow:
//
//  * Decimation in time (Cooley-Tukey): bit-reversed input order, natural output.
//    Stage s pairs elements whose index differs in bit s, with twiddle
//    omega^{(N/2^{s+1}) j}, j = index mod 2^s.  One table T[i] = omega^i, i < N/2,
//    serves every stage (stage s reads T[j << (n-1-s)]); Montgomery form.
//  * Stages are fused into passes of up to 9 (12 for a single pass) stages.  A CTA
//    owns C "groups" (the elements closed under the pass's stages), stages them
//    through shared memory, and runs them as register rounds of 4 stages on 16
//    elements per thread (8 independent butterflies per stage per thread).
//  * The bit reversal is folded into the first pass's gather (it reads strided
//    columns of x, coalesced across the C groups) and every later pass runs in
//    place, so no permutation pass exists.
//  * Inverse = same pass with T[i] = omega^{-i}; N^{-1} is folded into the last
//    stage (u N^{-1}, v (omega^{-j} N^{-1})), so the inverse costs N/2 log N mulmods.
//  * Stage 0 has twiddle 1 for every butterfly and skips the multiply.
//  * Negacyclic: twist x_j psi^j fused into the first pass's load, untwist
//    N^{-1} psi^{-j} fused into the last pass's store (reading c9).
#include <cuda.h>            // CUtensorMap (types only: the encoder comes from the driver entry point)
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <new>
#include <unordered_map>
#include <vector>

#include "../../include/ntt128.h"
#include "arith128.cuh"
#include "psm128.cuh"
#include "host128.h"
#include "ntt128_internal.h"

#ifndef NTT128_EXPERIMENTS
#define NTT128_EXPERIMENTS 0   // 1: experiment build (environment switches; never the product .so)
#endif
#ifndef NTT_COMPUTE_REPEAT
#define NTT_COMPUTE_REPEAT 1  // experiment: run a pass's register rounds k times (0: memory phases only)
#endif
#ifndef NTT_TRACE
#define NTT_TRACE 0           // experiment: per-tile timeline (tools/exp_trace.py)
#endif
#ifndef NTT_UNROLL_ROUNDS
#define NTT_UNROLL_ROUNDS 0   // 1: unroll the register rounds (compile-time windows)
#endif
// Groups per CTA of the multi-pass kernels (tools/gpu_sweep_variants.sh): one warp-owned
// (B = 8) or two-warp (B = 9) group per CTA avoids every cross-warp barrier and wins 5-8 %
// over C = 4; 8/16-thread groups (B = 6, 7) need C = 8 for occupancy (32 CTAs/SM cap).
#ifndef NTT_C8
#define NTT_C8 1
#endif
#ifndef NTT_C9
#define NTT_C9 1
#endif
#ifndef NTT_NC_C8
#define NTT_NC_C8 4           // permutation-free passes share one twiddle set per CTA when lo > 0
#endif
#ifndef NTT_NC_RB8
#define NTT_NC_RB8 3
#endif
#ifndef NTT_C7
#define NTT_C7 1
#endif
#ifndef NTT_C6
#define NTT_C6 8
#endif
#ifndef NTT_C5
#define NTT_C5 8
#endif
#ifndef NTT_OCC_THREADS
#define NTT_OCC_THREADS 768   // resident threads per SM the radix-8 pass kernels are register-budgeted for
#endif
#ifndef NTT_CARVEOUT
#define NTT_CARVEOUT -1       // >= 0: cudaFuncAttributePreferredSharedMemoryCarveout of the multi-pass kernels (experiment)
#endif
#ifndef NTT_OCC_THREADS_RB2
#define NTT_OCC_THREADS_RB2 1024   // ... and the radix-4 multi-pass kernels
#endif
#ifndef NTT_LDG_DATA
#define NTT_LDG_DATA 0        // 1: data tiles via LDG + STS instead of cp.async (experiment)
#endif
// radix-4 multi-pass rounds: XOR-swizzled layout (no bank conflicts) and unrolled rounds
// measured -1.3 % / -0.3 % against the padded layout and the rolled loop (fewer ALU ops
// per address, smaller code): both off
#ifndef NTT_RB2_XOR
#define NTT_RB2_XOR 0
#endif
#ifndef NTT_RB2_UNROLL
#define NTT_RB2_UNROLL 0
#endif
#ifndef NTT_RB9
#define NTT_RB9 3
#endif
#ifndef NTT_S9_C
#define NTT_S9_C 1    // single-pass N = 2^9: one group per CTA (+9 % over 4)
#endif
#ifndef NTT_S8_C
#define NTT_S8_C 8
#endif
#ifndef NTT_S10_C
#define NTT_S10_C 1    // single-pass N = 2^10: groups per CTA (1: +10 % over 2, 4) and register-round radix (log2)
#endif
#ifndef NTT_S10_RB
#define NTT_S10_RB 3
#endif
#ifndef NTT_RB7
#define NTT_RB7 2   // 7-stage passes: radix-4 rounds on one warp-owned group per CTA (NTT_C7 = 1):
                    // +2.4 % / +2.1 % at N = 2^14 / 2^15 over radix-8 with 8 groups per CTA
#endif
#ifndef NTT_RB6
#define NTT_RB6 3
#endif
#ifndef NTT_RB8
#define NTT_RB8 2   // register-round radix (log2) of the 8-stage multi-pass kernel: radix-4 rounds
                    // (smaller code, 32 warps/SM) beat radix-8 by 3.5 % with one group per CTA
#endif

using namespace ntt128;
using ntt128h::u128;

// ----------------------------------------------------------------------------- common
static std::atomic<uint64_t> g_launches{0};
static std::atomic<int> g_chain_plans{0};   // live plans with NTT128_FLAG_CHAIN (chained calls, below)
extern "C" uint64_t ntt128_launch_count(void) { return g_launches.load(); }
void ntt128_count_launch(uint64_t k) { g_launches += k; }

// Experiment builds only (-DNTT_TRACE=1): every multi-pass tile records globaltimer at its
// start, after its loads and after its stores, with its SM and pass, into a device buffer
// the caller provides (tools/exp_trace.py).  Not part of the product ABI.
#if NTT_TRACE
__device__ uint4* g_trace = nullptr;
__device__ unsigned long long g_trace_n = 0;
__device__ unsigned long long g_trace_cap = 0;
__device__ __forceinline__ uint32_t gtimer_lo() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return (uint32_t)(t & 0xffffffffu);
}
__device__ __forceinline__ uint32_t smid() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
extern "C" int ntt128_debug_trace(void* buf, unsigned long long cap) {
    unsigned long long z = 0;
    if (cudaMemcpyToSymbol(g_trace, &buf, sizeof(buf)) != cudaSuccess) return 1;
    if (cudaMemcpyToSymbol(g_trace_cap, &cap, sizeof(cap)) != cudaSuccess) return 1;
    if (cudaMemcpyToSymbol(g_trace_n, &z, sizeof(z)) != cudaSuccess) return 1;
    return 0;
}
#endif

extern "C" const char* ntt128_status_string(ntt128_status s) {
    switch (s) {
        case NTT128_OK: return "NTT128_OK";
        case NTT128_ERR_INVALID_ARG: return "NTT128_ERR_INVALID_ARG";
        case NTT128_ERR_MODULUS: return "NTT128_ERR_MODULUS";
        case NTT128_ERR_NOT_PRIME: return "NTT128_ERR_NOT_PRIME";
        case NTT128_ERR_NO_ROOT: return "NTT128_ERR_NO_ROOT";
        case NTT128_ERR_BAD_ROOT: return "NTT128_ERR_BAD_ROOT";
        case NTT128_ERR_ALIGNMENT: return "NTT128_ERR_ALIGNMENT";
        case NTT128_ERR_INPUT_RANGE: return "NTT128_ERR_INPUT_RANGE";
        case NTT128_ERR_OOM: return "NTT128_ERR_OOM";
        case NTT128_ERR_CUDA: return "NTT128_ERR_CUDA";
        case NTT128_ERR_UNSUPPORTED: return "NTT128_ERR_UNSUPPORTED";
    }
    return "NTT128_ERR_UNKNOWN";
}

static inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

static void to_words(u128 v, uint32_t w[4]) {
    for (int i = 0; i < 4; i++) w[i] = (uint32_t)(v >> (32 * i));
}

__device__ __forceinline__ uint32_t brev_bits(uint32_t x, int bits) { return bits == 0 ? 0u : (__brev(x) >> (32 - bits)); }

// 16-byte global -> shared copy without a register round trip (SASS LDGSTS)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Bulk copies (SASS UBLKCP) completing on an mbarrier (NTT_BULK, DESIGN.md §6 "Bulk staging").
#ifndef NTT_BULK
// bit 0: twiddle sets of 8- and 9-stage multi-pass passes by bulk copy (cfg3 +1.7 %, cfg4
// 2^14..2^17 +0.8..+1.4 %; with the 6/7-stage passes' eight small sets -1.3 % at 2^12: those
// keep cp.async); bit 1: first-pass stores by bulk copy (-3.4 %: off).  tools/exp_ab.py,
// profiles/r02/bulk_ab.txt
#define NTT_BULK 1
#endif
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
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
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
// Tensor (TMA) tile loads, SASS UTMALDG: one instruction moves a whole pass tile (DESIGN.md
// §6 "TMA staging"); the box lands in shared memory in box order, completing on `bar`.
__device__ __forceinline__ void tma_load5(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3, int c4,
                                          uint64_t* bar) {
    asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                 ::"r"(smem_u32(dst)), "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar)) : "memory");
}


// ----------------------------------------------------------------------------- twiddle generation
// out[m][i] = scale_m * base_m^i (Montgomery form), i < count; pow2[m][k] = base_m^{2^k}
// (Montgomery form), scale[m] Montgomery form.  Product over the set bits of i.
__global__ void k_gen_pow_table(uint4* out, uint64_t stride, uint64_t count, const uint4* pow2, int pow2_stride,
                                const uint4* scale, const ModC* mods) {
    const int m = blockIdx.y;
    const ModC& M = mods[m];
    uint32_t q[4] = {M.q[0], M.q[1], M.q[2], M.q[3]};
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x) {
        U128 r = u128_from(scale[m]);
        uint64_t e = i;
        int k = 0;
        while (e) {
            if (e & 1) r = mont_mul(r, u128_from(pow2[m * pow2_stride + k]), q, M.qinv0);
            e >>= 1;
            k++;
        }
        out[m * stride + i] = u128_to(r);
    }
}

// Per-pass twiddle tables in consumption order: out[m][L][k], L < 2^lo, k < 2^b - 1,
// k = (2^sl - 1) + jj for local stage sl (global s = lo + sl), holding the twiddle of
// the butterflies whose index mod 2^s is (jj << lo) | L, i.e. T[((jj << lo) | L) << (n-1-s)]
// (or T_last[(jj << lo) | L] for the final stage of a scaled inverse).
__global__ void k_gather_pass_tw(uint4* out, uint64_t out_stride, const uint4* T, const uint4* T_last,
                                 uint64_t tw_stride, uint32_t n, uint32_t lo, uint32_t b) {
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
        out[m * out_stride + e] = (T_last && s == n - 1) ? T_last[m * tw_stride + j] : T[m * tw_stride + (j << (n - 1 - s))];
    }
}

// Permutation-free negacyclic pass tables: out[m][H][k], k < 2^B - 1, local stage
// sl = B - 1 - floor(log2(k + 1)), block i = H 2^(B-1-sl) + (k - (2^(B-1-sl) - 1)),
// global stage b = lo + sl: psi^e (forward) or psi^-e (inverse), e = brev_n(2^(n-1-b) + i),
// from psi_pow[m][j] = psi^j R mod q (j < N; psi^-e = -psi^(N-e) since psi^N = -1); the
// inverse's b = n - 1 entries are multiplied by `scale` (Montgomery form) when given.
// Plain-residue copy of a Montgomery-form table (pseudo-Mersenne class): out = in R^-1 mod q.
__global__ void k_table_to_plain(uint4* out, const uint4* in, uint64_t stride, const ModC* mods) {
    const ModC& M = mods[blockIdx.y];
    const uint32_t q[4] = {M.q[0], M.q[1], M.q[2], M.q[3]};
    const U128 one = U128{{1u, 0u, 0u, 0u}};
    const uint64_t base = (uint64_t)blockIdx.y * stride;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < stride; i += (uint64_t)gridDim.x * blockDim.x)
        out[base + i] = u128_to(mont_mul(u128_from(in[base + i]), one, q, M.qinv0));
}

__global__ void k_gather_nc_tw(uint4* out, uint64_t out_stride, const uint4* psi_pow, uint32_t n, uint32_t lo,
                               uint32_t b, int inv, const uint4* scale, const ModC* mods) {
    const int m = blockIdx.y;
    const ModC& M = mods[m];
    const uint32_t K = (1u << b) - 1;
    const uint64_t count = ((uint64_t)1 << (n - lo - b)) * K;
    const uint64_t N = 1ull << n;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t H = e / K;
        const uint32_t k = (uint32_t)(e - H * K);
        const int lg = 31 - __clz(k + 1);            // = B - 1 - sl
        const uint32_t sl = b - 1 - lg;
        const uint64_t i = (H << lg) + (k + 1 - (1u << lg));
        const uint32_t gb = lo + sl;
        const uint64_t idx = ((uint64_t)1 << (n - 1 - gb)) + i;   // < N
        const uint64_t ex = __brevll(idx) >> (64 - n);
        U128 v;
        if (!inv) {
            v = u128_from(psi_pow[m * N + ex]);
        } else if (ex == 0) {
            v = U128{{M.one_m[0], M.one_m[1], M.one_m[2], M.one_m[3]}};
        } else {
            const U128 x = u128_from(psi_pow[m * N + (N - ex)]);
            const uint32_t z[4] = {0, 0, 0, 0};
            v = sub_mod(U128{{z[0], z[1], z[2], z[3]}}, x, M.q);
        }
        if (inv && scale && gb == n - 1) v = mont_mul(v, u128_from(scale[m]), M.q, M.qinv0);
        out[m * out_stride + e] = u128_to(v);
    }
}

// ----------------------------------------------------------------------------- pass kernel
// Per-modulus constants of one launch as KERNEL PARAMETERS (multi-pass kernels, DESIGN.md §5
// "Moduli in uniform registers"): indexed by a block-uniform polynomial index they load with
// LDCU into uniform registers, so every q-word operand of the Montgomery products and the
// mod-q adds is a uniform register -- no vector registers or vector register-file reads for
// q, 2q, q' (register-only butterfly rate +7.7 % LAZY, +2.6 % FULL, tools/micro/bfly_uniform.cu).
// A launch carries at most NTT_QMAX moduli: RNS plans with more polynomials launch each pass
// in chunks of NTT_QMAX polynomials.
#ifndef NTT_QMAX
#define NTT_QMAX 64
#endif
struct QPar {
    uint32_t q[4];
    uint32_t qinv0, pad[3];
    uint32_t ninv_m[4];   // N^-1 R mod q
    uint32_t ninv_rm[4];  // N^-1 R^2 mod q
};
struct PassArgs {
    // TMA kernels (k_ntt_pass<..., TMA>): the data tile's tensor map over src, encoded per
    // launch by the host (tma_map_*); unused otherwise.  First member: 64-byte aligned.
    CUtensorMap tm;
    QPar qp[NTT_QMAX];     // multi-pass kernels: the launch's moduli (qp[0] when nq == 1)
    uint16_t ord[NTT_QMAX];// multi-pass kernels, nq > 1: CTA polynomial slot -> polynomial (grouped by class)
    const uint4* src;      // [batch][N]
    uint4* dst;            // [batch][N]
    const uint4* pmul;     // optional point-wise multiplicand, same layout as src (Montgomery product)
    const uint4* pt;       // [nq][pt_stride] pass twiddles in consumption order: [L][k], k < 2^B - 1
    const uint4* fin;      // optional [nq][f_stride]: factor applied at load, by natural input index
    const uint4* fout;     // optional [nq][f_stride]: factor applied at store, by natural output index
    const ModC* mods;      // [nq]
    uint64_t pt_stride, f_stride;
    uint64_t total_groups; // batch << (n - B)
    uint32_t n, lo, nq;
    uint32_t ninv_r;       // SCALE_LAST multiplier: 0 -> ninv_m, 1 -> ninv_rm (point-wise R^-1 compensation)
    // Pass overlap (programmatic dependent launch, multi-pass plans): a later pass starts
    // on a polynomial once every CTA of the previous pass on it has signalled.
    const uint32_t* cnt_in;  // optional [batch]: previous pass's completion counters (wait for target)
    uint32_t* cnt_out;       // optional [batch]: this pass's completion counters (+1 per CTA)
    uint32_t target;         // cnt_in[poly] value that means "previous pass done" (wrap-safe compare)
    uint32_t pdl_wait;       // 1: griddepcontrol.wait before reading data (first pass of a PDL launch)
    // Four-step I/O (fourstep.cu; natural [batch][N] when left at the defaults):
    //  * the pass reads element idx of polynomial p at src[p in_ps + idx in_es] (default N, 1;
    //    a first pass may read the columns of a received [n][batch] matrix: in_ps 1, in_es batch);
    //  * fpoly: fin is indexed by polynomial instead of modulus, at fin[p f_ps + idx f_es];
    //  * r_lb != 0 (the transform's last pass): output k of polynomial p goes to
    //    rdst[k >> r_lb] + p r_ps + (k mod 2^r_lb) -- the destination rank's block of the
    //    all-to-all send buffer, or that rank's receive buffer itself (peer memory).
    uint64_t in_ps, in_es;
    uint64_t f_ps, f_es;     // fpoly: factor of (p, idx) at fin[p f_ps + idx f_es]
    uint32_t fpoly, r_lb;
    uint32_t psm, psm_pad;   // 1: pseudo-Mersenne class (MODE_PSM): pt holds plain twiddles (plain cyclic multi-pass only)
    uint64_t r_ps;
    uint4* rdst[NTT128_FS_MAX_RANKS];
};

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_gpu_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Shape of one pass: groups of G = 2^B elements, E = 2^RB elements per thread
// (register rounds of RB stages), T threads per group.  PADL selects the shared-memory
// layout of a group: padded (slot(l) = l + l/8, one empty 16-byte slot after every 8
// elements; multi-pass kernels) or XOR-swizzled (single-pass kernels, whose one-group
// CTAs gather bit-reversed rows).
template <int B, int RBMAX = 3, int C = 8, bool PADL = false>
struct PassShape {
    static constexpr int G = 1 << B;
    static constexpr int RB = B >= RBMAX ? RBMAX : B;  // radix-2^RB register rounds
    static constexpr int E = 1 << RB;
    static constexpr int T = G / E;
    // Strides between groups (data) and twiddle sets, in 16-byte slots: an 8-lane shared
    // memory phase covers min(C, 8) groups x 8/min(C, 8) adjacent rows, so the group
    // stride must be = 8/C (mod 8) for C in {2, 4} and odd for C >= 8.
    static constexpr int CM = C < 8 ? C : 8;
    static constexpr int GP = (PADL && !(RB == 2 && NTT_RB2_XOR)) ? G + G / 8 : G;   // slots a group's elements span
    static constexpr int PADG = PADL ? ((8 / CM) % 8 - GP % 8 + 8) % 8 : ((C >= 8 || C == 1) ? 1 : 8 / C);
    static constexpr int GS = GP + PADG;
    // twiddle-set stride: a warp-owned group (T <= 32) reads only its own set, so the sets
    // are 128-byte aligned (full-speed cp.async); otherwise staggered across banks
    static constexpr int TS = (PADL && T <= 32 && 32 % T == 0 && G >= 8) ? G : ((C >= 8 || C == 1) ? G - 1 : G + 8 / C);
    static constexpr int ROUNDS = (B + RB - 1) / RB;
    // every register-round window w is 0 or >= 3, so slot(l0 + k 2^w) is linear in k
    static constexpr bool LINEAR = PADL && (RB >= 3 || B == RB) && !(B - RB == 1 || B - RB == 2);
};

// XOR swizzle of the low 3 element-index bits (16-byte slots of a 128-byte bank
// row): conflict-free for the register-round patterns and, when B >= 9, for the
// bit-reversed gather of a single-group CTA.
template <int B>
__device__ __forceinline__ int swz(int l) {
    int f = l >> 3;
    if (B >= 9) f ^= l >> (B >= 9 ? B - 3 : 0);
    return l ^ (f & 7);
}
// Multi-pass layout: the padded slot l + l/8 (conflict-free for radix-8 windows w = 0, 3,
// 6 / B - 3; radix-4 windows w = 2 see 2-way conflicts).  NTT_RB2_XOR selects, for radix-4
// rounds, an XOR swizzle of the low three index bits, l ^ (bits 3..4 of l) ^ (bit 4 << 2),
// conflict-free for every radix-4 window and the load / store rows -- measured slower.
template <int B, bool PADL, int RB = 3>
__device__ __forceinline__ int slot(int l) {
    if (!PADL) return swz<B>(l);
    if (RB == 2 && NTT_RB2_XOR) return l ^ (((l >> 3) & 3) | ((l >> 2) & 4));
    return l + (l >> 3);
}

// Arithmetic mode of a multi-pass CTA, by modulus class (uniform per CTA):
//   MODE_FULL (q >= 2^127): canonical values in [0, q);
//   MODE_HALF (2^126 <= q < 2^127): values in [0, 2q), add/sub modulo 2q, lazy Montgomery;
//   MODE_LAZY (q < 2^126): values in [0, 4q), Harvey butterflies, lazy Montgomery.
// Single-pass CTAs (one CTA may hold several moduli) and the last pass's store keep the
// interface canonical.
enum { MODE_FULL = 0, MODE_HALF = 1, MODE_LAZY = 2, MODE_PSM = 3 };
// MODE_PSM (psm128.cuh): pseudo-Mersenne moduli q = 2^b - c in plain cyclic multi-pass
// transforms whose launch sets PassArgs::psm -- plain (non-Montgomery) twiddles, values are
// any 128-bit representative between stages, 21 word products per butterfly; q2[0] carries
// C = 2^128 - q 2^(128-b).  The inverse's u N^-1 is always the short digit (sh != 0).
#ifndef NTT_FORCE_FULL
#define NTT_FORCE_FULL 0      // 1: canonical arithmetic for every modulus (experiment)
#endif
__device__ __forceinline__ int mode_of(const uint32_t q[4]) {
    if (NTT_FORCE_FULL) return MODE_FULL;
    return (q[3] >> 30) == 0 ? MODE_LAZY : ((q[3] >> 31) == 0 ? MODE_HALF : MODE_FULL);
}

// One radix-2 CT butterfly (u, v) -> (u + w v, u - w v) in the given mode.  In the last
// stage of a scaled inverse u is multiplied by nf = N^-1 (Montgomery form) too.
#ifndef NTT_PSM
#define NTT_PSM 1             // 0: no pseudo-Mersenne class (A/B build)
#endif
#ifndef NTT_SHIFT_SCALE
#define NTT_SHIFT_SCALE 1     // 0: N^-1 always by the Montgomery product (A/B experiment)
#endif
// sh != 0 (a plain inverse, N = 2^sh): u N^-1 = u 2^-sh by one short digit (shr_mod, 8 word
// products) instead of the Montgomery product by nf (36); polymul's N^-1 R keeps nf.
template <int MODE, bool SCALE_U>
__device__ __forceinline__ void bfly(U128& u, U128& v, const U128& w, const uint32_t q[4], const uint32_t q2[4],
                                     uint32_t qinv0, const U128& nf, uint32_t sh = 0) {
    if (MODE == MODE_PSM) {
        const U128 us = SCALE_U ? shr_mod(u, sh, q, qinv0) : u;   // any u < 2^128 -> < max(q, 2^127)
        const U128 t = psm_mul(v, w, q2[0]);      // < Q: one fold in the add and the subtract
        u = psm_add1(us, t, q2[0]);
        v = psm_sub1(us, t, q2[0]);
    } else if (MODE == MODE_FULL) {
        const U128 us = SCALE_U ? (sh ? shr_mod(u, sh, q, qinv0) : mont_mul(u, nf, q, qinv0)) : u;
        const U128 t = mont_mul(v, w, q, qinv0);
        u = add_mod(us, t, q);
        v = sub_mod(us, t, q);
    } else if (MODE == MODE_HALF) {   // u, v in [0, 2q): t in [0, 2q); results mod 2q
        const U128 us = SCALE_U ? (sh ? shr_mod_lazy(u, sh, q, qinv0) : mont_mul_lazy(u, nf, q, qinv0)) : u;
        const U128 t = mont_mul_lazy(v, w, q, qinv0);
        u = add_mod(us, t, q2);
        v = sub_mod(us, t, q2);
    } else {                          // Harvey: u, v in [0, 4q); u' = u mod 2q; u' + t, u' - t + 2q
        const U128 us = SCALE_U ? (sh ? shr_mod_lazy(u, sh, q, qinv0) : mont_mul_lazy(u, nf, q, qinv0)) : reduce_2q(u, q2);
        const U128 t = mont_mul_lazy(v, w, q, qinv0);
        u = add_nored(us, t);
        v = sub_add_nored(us, t, q2);
    }
}
// Stage with twiddle 1 (first stage of a first pass): inputs canonical (< q).
template <int MODE>
__device__ __forceinline__ void bfly1(U128& u, U128& v, const uint32_t q[4], const uint32_t q2[4]) {
    if (MODE == MODE_PSM) {
        const U128 a = psm_add(u, v, q2[0]);
        v = psm_sub(u, v, q2[0]);
        u = a;
    } else if (MODE == MODE_FULL) {
        const U128 a = add_mod(u, v, q);
        v = sub_mod(u, v, q);
        u = a;
    } else {                          // u + v < 2q, u - v + q in (0, 2q): no reduction needed
        const U128 a = add_nored(u, v);
        v = sub_add_nored(u, v, q);
        u = a;
    }
}
// Butterfly with twiddle 1 on values in the mode's lazy range (a later stage's j = 0 block).
template <int MODE>
__device__ __forceinline__ void bfly_tw1(U128& u, U128& v, const uint32_t q[4], const uint32_t q2[4]) {
    if (MODE == MODE_PSM) {
        const U128 a = psm_add(u, v, q2[0]);
        v = psm_sub(u, v, q2[0]);
        u = a;
    } else if (MODE == MODE_FULL) {
        const U128 a = add_mod(u, v, q);
        v = sub_mod(u, v, q);
        u = a;
    } else if (MODE == MODE_HALF) {   // [0, 2q): arithmetic mod 2q
        const U128 a = add_mod(u, v, q2);
        v = sub_mod(u, v, q2);
        u = a;
    } else {                          // [0, 4q): both to [0, 2q), then Harvey's sums
        const U128 us = reduce_2q(u, q2), t = reduce_2q(v, q2);
        u = add_nored(us, t);
        v = sub_add_nored(us, t, q2);
    }
}

// Register rounds of one pass on a CTA's tile in shared memory: RB stages on E elements
// per thread (window [w, w + RB) of the group's index bits), 8-lane conflict-free
// addressing.  With the padded layout the E slots of a round are s0 + k st (one base,
// one stride per round), and a stage's distinct twiddles are loaded once: stage w + bit
// needs 2^bit of them (index (2^sl - 1) + tlo + (j << w), j < 2^bit).
// R0: the first round of a first pass (w = 0, global stage = local stage), peeled so the
// butterflies with twiddle index j = 0 (twiddle 1: all of stage 0, half of stage 1, a
// quarter of stage 2) skip their multiply at compile time.
template <int B, int C, bool FIRST, bool SCALE_LAST, int RBMAX, int MODE, bool WARPSYNC, bool PADL, bool R0>
__device__ __forceinline__ void round_body(const int rd, uint4* gsm, const uint4* tws, const int t, const uint32_t lo,
                                           const uint32_t n, const uint32_t q[4], const uint32_t q2[4],
                                           const uint32_t qinv0, const U128& nf, const uint32_t sh) {
    using S = PassShape<B, RBMAX, C, PADL>;
    constexpr int RB = S::RB, E = S::E;
    const int slo = R0 ? 0 : rd * RB;
    const int w = R0 ? 0 : ((slo + RB <= B) ? slo : B - RB);   // E-element window [w, w + RB)
    const int tlo = t & ((1 << w) - 1), thi = (t >> w) << (w + RB);
    const int l0 = thi | tlo;                                 // element k of this thread: l0 + (k << w)
    const int s0 = S::LINEAR ? slot<B, PADL, RB>(l0) : 0;
    const int st = S::LINEAR ? (w >= 3 ? (9 << (w - 3)) : (1 << w)) : 0;
    U128 x[E];
#pragma unroll
    for (int k = 0; k < E; k++) x[k] = u128_from(gsm[S::LINEAR ? s0 + k * st : slot<B, PADL, RB>(l0 | (k << w))]);
#pragma unroll
    for (int bit = 0; bit < RB; bit++) {
        const int sl = w + bit;                      // local stage
        if (sl < slo) continue;                      // overlap of the last window
        const bool last = SCALE_LAST && lo + sl == n - 1;
        if (R0 && bit == 0 && !last) {               // stage 0: twiddle 1, inputs canonical
#pragma unroll
            for (int kk = 0; kk < E / 2; kk++) {
                const int k0 = ((kk >> bit) << (bit + 1)) | (kk & ((1 << bit) - 1));
                bfly1<MODE>(x[k0], x[k0 | (1 << bit)], q, q2);
            }
            continue;
        }
        const uint4* tp = tws + tlo + ((1 << sl) - 1);
        U128 tw[E / 2];                              // the first 2^bit are used
#pragma unroll
        for (int j = 0; j < (1 << bit); j++) tw[j] = u128_from(tp[j << w]);
#pragma unroll
        for (int kk = 0; kk < E / 2; kk++) {
            const int k0 = ((kk >> bit) << (bit + 1)) | (kk & ((1 << bit) - 1));
            const int k1 = k0 | (1 << bit);
            const int j = kk & ((1 << bit) - 1);
            if (R0 && j == 0 && !last) bfly_tw1<MODE>(x[k0], x[k1], q, q2);
            else if (last) bfly<MODE, true>(x[k0], x[k1], tw[j], q, q2, qinv0, nf, sh);
            else bfly<MODE, false>(x[k0], x[k1], tw[j], q, q2, qinv0, nf);
        }
    }
#pragma unroll
    for (int k = 0; k < E; k++) gsm[S::LINEAR ? s0 + k * st : slot<B, PADL, RB>(l0 | (k << w))] = u128_to(x[k]);
    if (WARPSYNC) __syncwarp(); else __syncthreads();
}

template <int B, int C, bool FIRST, bool SCALE_LAST, int RBMAX, int MODE, bool WARPSYNC, bool PADL>
__device__ __forceinline__ void pass_rounds(uint4* gsm, const uint4* tws, const int t, const uint32_t lo, const uint32_t n,
                                            const uint32_t q[4], const uint32_t qinv0, const U128 nf, const uint32_t sh) {
    uint32_t q2[4] = {0, 0, 0, 0};
    if (MODE == MODE_PSM) {
        q2[0] = psm_C(q, psm_shift(q));
    } else if (MODE != MODE_FULL) {
        q2[0] = q[0] << 1;
        q2[1] = (q[1] << 1) | (q[0] >> 31);
        q2[2] = (q[2] << 1) | (q[1] >> 31);
        q2[3] = (q[3] << 1) | (q[2] >> 31);
    }
    using S = PassShape<B, RBMAX, C, PADL>;
    constexpr int rd0 = FIRST ? 1 : 0;
    if (FIRST)
        round_body<B, C, FIRST, SCALE_LAST, RBMAX, MODE, WARPSYNC, PADL, true>(0, gsm, tws, t, lo, n, q, q2, qinv0, nf, sh);
    if (S::RB == 2 && PADL && NTT_RB2_UNROLL) {
        // radix-4 rounds: unrolled, so every window and XOR-swizzle offset is a constant
#pragma unroll
        for (int rd = rd0; rd < S::ROUNDS; rd++)
            round_body<B, C, FIRST, SCALE_LAST, RBMAX, MODE, WARPSYNC, PADL, false>(rd, gsm, tws, t, lo, n, q, q2, qinv0, nf, sh);
    } else {
#if NTT_UNROLL_ROUNDS
#pragma unroll
#else
#pragma unroll 1
#endif
        for (int rd = rd0; rd < S::ROUNDS; rd++)
            round_body<B, C, FIRST, SCALE_LAST, RBMAX, MODE, WARPSYNC, PADL, false>(rd, gsm, tws, t, lo, n, q, q2, qinv0, nf, sh);
    }
}

// Resident threads per SM each pass kernel is register-budgeted for: radix-4 multi-pass
// kernels (16 data registers per thread, 64 registers) run 32 warps per SM, radix-8 ones
// (32 data registers, 80) 24 warps (tools/gpu_variants.sh).
template <int B, int RBMAX, bool SINGLE>
struct PassOcc {
    static constexpr int RB = PassShape<B, RBMAX>::RB;
    static constexpr int THREADS = (RB == 2 && !SINGLE) ? NTT_OCC_THREADS_RB2 : NTT_OCC_THREADS;
};
// TMA (later passes of 7-, 8- and 9-stage multi-pass plans, one group per CTA, DESIGN.md §6
// "TMA staging"): thread 0 moves the CTA's whole data tile with ONE tensor load (UTMALDG)
// and its twiddle set with one bulk copy (UBLKCP), both completing on mbarriers in shared
// memory; no thread issues a per-element copy.  The box {2 u64, 9 rows j from -1, 2^B/8
// chunks m} over the [poly][H][m][j][L] view (r = 8 m + j) lands as exactly the padded
// layout, slot 1 + l + l/8, the j = -1 rows being out of bounds (zero-filled, never read).
// First passes keep per-thread cp.async: their rows are the bit-reversed gather, which no
// affine box maps onto the padded layout.
template <int B, int C, bool FIRST, bool SCALE_LAST, bool SINGLE, int RBMAX, bool PM = false, bool TMA = false>
__global__ void __launch_bounds__(C * PassShape<B, RBMAX>::T,
                                  (PassOcc<B, RBMAX, SINGLE>::THREADS / (C * PassShape<B, RBMAX>::T)) > 0
                                      ? PassOcc<B, RBMAX, SINGLE>::THREADS / (C * PassShape<B, RBMAX>::T) : 1)
k_ntt_pass(const __grid_constant__ PassArgs a) {
    static_assert(!PM || (FIRST && !SINGLE), "polynomial-major groups: multi-pass first passes only");
    static_assert(!TMA || (C == 1 && !SINGLE && !PM && !FIRST && B >= 7 && B <= 9), "TMA: later passes, one group per CTA");
    constexpr bool PADL = !SINGLE;
    using S = PassShape<B, RBMAX, C, PADL>;
    constexpr int G = S::G, RB = S::RB, T = S::T, GS = S::GS, TS = S::TS;
    constexpr int NT = C * T;
    constexpr int NTW = (FIRST && !SINGLE) ? 1 : C;  // twiddle sets: a multi-pass first pass shares one (L = 0)
    constexpr int DOFF = TMA ? 1 : 0;                // TMA: slot 0 takes the box's first pad row
    extern __shared__ __align__(128) uint4 sm[];     // tensor-copy destinations: 128-byte aligned
    uint4* const dsm = sm + DOFF;                    // [C][GS] data tiles
    uint4* tsm = dsm + C * GS;                       // [NTW][TS] pass-local twiddles
    __shared__ __align__(8) uint64_t tw_bar_s;       // NTT_BULK: twiddle bulk copies (non-TMA kernels)
    // TMA kernels keep their barriers in dynamic shared memory: [0] twiddles, [1] data tile
    uint64_t* const bars = reinterpret_cast<uint64_t*>(tsm + NTW * TS);
    uint64_t* const twb = TMA ? bars : &tw_bar_s;

    const uint32_t n = a.n, lo = a.lo, gbits = n - B;
    const uint64_t N = 1ull << n;
    const uint64_t gmask = (1ull << gbits) - 1;
#if NTT_TRACE
    const uint32_t tr_t0 = gtimer_lo();
#endif
    uint64_t gg0 = (uint64_t)blockIdx.x * C;
    // multi-pass CTAs hold groups of one polynomial: visit polynomials in the plan's order
    // (grouped by arithmetic mode) so one code path at a time is hot in the I-cache
    // (a kernel-parameter table: the polynomial index stays block-uniform, in uniform registers)
    if (!SINGLE && !PM && a.nq > 1) gg0 = ((uint64_t)a.ord[gg0 >> gbits] << gbits) | (gg0 & gmask);
    // PM (polynomial-major first pass, four-step pass C over a received matrix whose
    // polynomials are adjacent in memory): the CTA's C groups are column g0
    // of the C consecutive polynomials [pc C, pc C + C), CTAs ordered g-major, so a row of
    // the gather is C adjacent residues (a full 32-byte sector at C = 2, 64 bytes at C = 4)
    // and consecutive CTAs read consecutive segments.  One modulus (nq == 1).
    const uint64_t pm_np = PM ? (a.total_groups >> gbits) / C : 1;
    const uint64_t pm_g0 = PM ? blockIdx.x / pm_np : 0, pm_pc = PM ? blockIdx.x % pm_np : 0;
    if (PM) gg0 = ((pm_pc * C) << gbits) | pm_g0;
    auto gg_of = [&](int c) -> uint64_t { return PM ? (((pm_pc * C + c) << gbits) | pm_g0) : gg0 + c; };
    const int tid = threadIdx.x;

    // ---------------- load phase: twiddles and data -> shared memory, all copies in flight
    // at once (cp.async 16-byte copies, LDGSTS), then one wait.  NT is a multiple of C, so a
    // thread keeps one group c = tid % C and visits rows t0 + i T: every address below is
    // a per-thread base plus a compile-time multiple of i.
    constexpr int LT = B - RB;                   // log2 T
    // multi-pass first pass: the rows of a lane pair/quad are T/2 (T/4) apart, so the
    // bit-reversed rows land in different banks (8-lane phase = CM groups x 8/CM rows)
    constexpr int RT0 = (!PADL || !FIRST) ? 0 : (S::CM == 8 ? 0 : (S::CM == 4 ? 1 : (S::CM == 2 ? 2 : 3)));
    constexpr int RT = RT0 < LT ? RT0 : LT;
    const int c_me = tid % C;
    const int u_me = tid / C;
    const int t0 = (RT == 0 || LT == 0) ? u_me : ((u_me >> RT) | ((u_me & ((1 << RT) - 1)) << (LT - RT)));
    const uint64_t gg_me = gg_of(c_me);
    const bool live = gg_me < a.total_groups;
    const uint64_t ggc_me = live ? gg_me : a.total_groups - 1;
    const uint64_t poly_me = ggc_me >> gbits, g_me = ggc_me & gmask;
    const uint32_t m_me = a.nq == 1 ? 0 : (uint32_t)poly_me;
    {
        // Twiddles: set c holds its group's 2^B - 1 twiddles in consumption order (slot
        // (2^sl - 1) + jj for local stage sl), precomputed per pass at plan time; the sets
        // of one CTA (consecutive L, same polynomial) are consecutive runs of the table.
        constexpr int TW_IT = (G - 1 + NT - 1) / NT;
        if (TMA || ((NTT_BULK & 1) && !SINGLE && B >= 8)) {
            // one thread streams the CTA's twiddle sets (contiguous runs of the pass table)
            // with bulk copies; the other threads wait on the mbarrier after the data phase
            if (tid == 0) {
                const uint64_t L0 = FIRST ? 0 : ((gg0 & gmask) & ((1ull << lo) - 1));
                const uint32_t m0 = a.nq == 1 ? 0 : (uint32_t)((gg0 < a.total_groups ? gg0 : a.total_groups - 1) >> gbits);
                const uint4* src = a.pt + m0 * a.pt_stride + L0 * (G - 1);
                mbar_init(twb, 1);
                if (TMA) mbar_init(bars + 1, 1);
                mbar_expect_tx(twb, NTW * (G - 1) * 16);
#pragma unroll
                for (int c = 0; c < NTW; c++) bulk_g2s(tsm + c * TS, src + c * (G - 1), (G - 1) * 16, twb);
            }
        } else if (NTW == 1 || !(FIRST && SINGLE)) {
            const uint64_t L0 = FIRST ? 0 : ((gg0 & gmask) & ((1ull << lo) - 1));
            const uint32_t m0 = a.nq == 1 ? 0 : (uint32_t)((gg0 < a.total_groups ? gg0 : a.total_groups - 1) >> gbits);
            const uint4* src = a.pt + m0 * a.pt_stride + L0 * (G - 1) + tid;
            uint4* dst = tsm + tid;
#pragma unroll
            for (int c = 0; c < NTW; c++)
#pragma unroll
                for (int i = 0; i < TW_IT; i++)
                    if ((G - 1) % NT == 0 || i + 1 < TW_IT || tid + i * NT < G - 1)
                        cp_async16(dst + c * TS + i * NT, src + c * (G - 1) + i * NT);
        } else {   // single pass, C polynomials per CTA, each with its own modulus
            constexpr int TW_PER = (NTW * (G - 1) + NT - 1) / NT;
#pragma unroll
            for (int i = 0; i < TW_PER; i++) {
                const int e = tid + i * NT;
                if (e < NTW * (G - 1)) {
                    const int c = e / (G - 1), k = e - c * (G - 1);
                    const uint64_t gg = gg0 + c;
                    const uint32_t m = a.nq == 1 ? 0 : (uint32_t)((gg < a.total_groups ? gg : a.total_groups - 1) >> gbits);
                    cp_async16(tsm + c * TS + k, a.pt + m * a.pt_stride + k);
                }
            }
        }
    }
    // ---------------- pass overlap: the twiddles (plan constants) are already in flight;
    // data may be read only once the producers of this polynomial are done
    {
        if (a.pdl_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
        if (a.cnt_in) {
            if (tid == 0) {
                const uint32_t* cp = a.cnt_in + (gg0 >> gbits);
                while ((int32_t)(ld_acquire_gpu(cp) - a.target) < 0) __nanosleep(128);
            }
            if (!TMA) __syncthreads();
        }
        if (TMA && tid == 0) {
            // the producers' generic-proxy stores (acquired above) before our async-proxy reads
            asm volatile("fence.proxy.async.global;" ::: "memory");
            // group (H, L): rows r = 8 m + j at stride 2^lo, box j from -1 (pad)
            const uint64_t poly = gg0 >> gbits, g = gg0 & gmask;
            const uint64_t H = g >> lo, L = g & ((1ull << lo) - 1);
            mbar_expect_tx(bars + 1, 9 * (G / 8) * 16);
            tma_load5(sm, &a.tm, (int)(2 * L), -1, 0, (int)H, (int)poly, bars + 1);
        }
        if (TMA) __syncthreads();   // mbarrier initialisation visible before anyone waits
        // our predecessors are complete (or their output for this polynomial is): the next
        // pass may be scheduled onto SMs as this grid drains
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
    constexpr int PER = (C * G) / NT;            // == E
    // element i of this thread: row r = t0 + i T
    uint64_t gbase;                              // natural index of row t0 of group c_me
    uint32_t gstride;                            // natural-index step per i (< 2^26)
    int lbase;                                   // local index of row t0
    if (FIRST) {   // gather column g of the (2^B x 2^gbits) view: row r -> local brev_B(r)
        gbase = ((uint64_t)t0 << gbits) | g_me;
        gstride = (uint32_t)T << gbits;
        lbase = (int)brev_bits((uint32_t)t0, B);
    } else {
        const uint64_t H = g_me >> lo, L = g_me & ((1ull << lo) - 1);
        gbase = (H << (lo + B)) | ((uint64_t)t0 << lo) | L;
        gstride = (uint32_t)T << lo;
        lbase = t0;
    }
    const uint4* srcp = a.src + poly_me * a.in_ps + gbase * a.in_es;
    const uint64_t sstride = (uint64_t)gstride * a.in_es;   // source step per i
    uint4* smc = dsm + c_me * GS;
    if (TMA) {
        // the tile is in flight (thread 0's tensor load)
    } else if (!a.fin && !a.pmul) {
        if (live) {
#if NTT_LDG_DATA
            // registers, then conflict-free STS: cp.async into the padded layout (lanes not
            // writing consecutive 16-byte slots) costs one L1 wavefront per lane
            uint4 v[PER];
#pragma unroll
            for (int i = 0; i < PER; i++) v[i] = __ldcg(srcp + (size_t)i * sstride);
#pragma unroll
            for (int i = 0; i < PER; i++) {
                const int l = FIRST ? (lbase | (int)(brev_bits((uint32_t)i, RB))) : (lbase + (i << LT));
                smc[slot<B, PADL, RB>(l)] = v[i];
            }
#else
#pragma unroll
            for (int i = 0; i < PER; i++) {
                const int l = FIRST ? (lbase | (int)(brev_bits((uint32_t)i, RB))) : (lbase + (i << LT));
                cp_async16(smc + slot<B, PADL, RB>(l), srcp + (size_t)i * sstride);
            }
#endif
        }
    } else if (FIRST && live) {   // load-side factors (twist, four-step, point-wise): first passes only
        uint4 stage[PER];
#pragma unroll
        for (int i = 0; i < PER; i++) stage[i] = srcp[(size_t)i * sstride];
        // multi-pass: the modulus from the kernel parameters (block-uniform: one polynomial per
        // CTA, or nq == 1 for the polynomial-major four-step CTAs); one-pass: the device table
        auto factors = [&](const uint32_t* qs, uint32_t qinv0) {
            const uint32_t q[4] = {qs[0], qs[1], qs[2], qs[3]};
#pragma unroll
            for (int i = 0; i < PER; i++) {
                const int l = FIRST ? (lbase | (int)(brev_bits((uint32_t)i, RB))) : (lbase + (i << LT));
                const uint64_t idx = gbase + (size_t)i * gstride;
                U128 x = u128_from(stage[i]);
                if (a.fin) x = mont_mul(x, u128_from(__ldg(a.fin + (a.fpoly ? poly_me * a.f_ps + idx * a.f_es : m_me * a.f_stride + idx))), q, qinv0);
                if (a.pmul) x = mont_mul(x, u128_from(__ldg(a.pmul + poly_me * N + idx)), q, qinv0);
                smc[slot<B, PADL, RB>(l)] = u128_to(x);
            }
        };
        if (SINGLE) {
            const ModC& M = a.mods[m_me];
            factors(M.q, M.qinv0);
        } else {
            const QPar& M = a.qp[a.nq == 1 ? 0 : (uint32_t)(gg0 >> gbits)];
            factors(M.q, M.qinv0);
        }
    }
    if (TMA) {
        mbar_wait(bars + 1, 0);   // data tile
        mbar_wait(bars, 0);       // twiddle set
    } else {
        cp_async_wait_all();
        __syncthreads();
        if ((NTT_BULK & 1) && !SINGLE && B >= 8) mbar_wait(twb, 0);
    }
#if NTT_TRACE
    const uint32_t tr_t1 = gtimer_lo();
#endif

    // ---------------- register rounds: RB stages on E elements per thread
    // Groups of at most 32 threads are owned by whole warps (c = tid / T), so the exchanges
    // between rounds never leave a warp and need only __syncwarp (pass_rounds); larger
    // groups keep the interleaved mapping and block barriers.
    {
        constexpr bool WARPMAP = T <= 32 && (32 % T) == 0;
        const int c = WARPMAP ? tid / T : tid % C, t = WARPMAP ? tid % T : tid / C;
        const uint64_t gg = gg_of(c);
        const uint64_t ggc = gg < a.total_groups ? gg : a.total_groups - 1;
        uint32_t q[4], qinv0;
        U128 nf;
        if (SINGLE) {   // one-pass CTAs may hold several moduli (lanes differ): the device table
            const uint32_t m = a.nq == 1 ? 0 : (uint32_t)(ggc >> gbits);
            const ModC& M = a.mods[m];
            q[0] = M.q[0]; q[1] = M.q[1]; q[2] = M.q[2]; q[3] = M.q[3];
            qinv0 = M.qinv0;
            if (SCALE_LAST) {
                const uint32_t* src = a.ninv_r ? M.ninv_rm : M.ninv_m;
                nf = U128{{src[0], src[1], src[2], src[3]}};
            }
        } else {        // multi-pass: the CTA's groups share one polynomial (PM: nq == 1) -- uniform
            const uint32_t m = a.nq == 1 ? 0 : (uint32_t)(gg0 >> gbits);
            const QPar& M = a.qp[m];
            q[0] = M.q[0]; q[1] = M.q[1]; q[2] = M.q[2]; q[3] = M.q[3];
            qinv0 = M.qinv0;
            if (SCALE_LAST) {
                const uint32_t* src = a.ninv_r ? M.ninv_rm : M.ninv_m;
                nf = U128{{src[0], src[1], src[2], src[3]}};
            }
        }
        uint4* gsm = dsm + c * GS;
        const uint4* tws = tsm + (NTW == 1 ? 0 : c) * TS;

        const int mode = a.psm ? MODE_PSM : (SINGLE ? MODE_FULL : mode_of(q));   // uniform per CTA: its groups share the polynomial
        const uint32_t sh = (NTT_SHIFT_SCALE && SCALE_LAST && !a.ninv_r && n >= 2) ? n : 0u;   // plain inverse: N^-1 by shifting
#if NTT_COMPUTE_REPEAT != 1
#pragma unroll 1
        for (int rep = 0; rep < NTT_COMPUTE_REPEAT; rep++)
#endif
        if (mode == MODE_PSM)
            pass_rounds<B, C, FIRST, SCALE_LAST, RBMAX, MODE_PSM, WARPMAP, PADL>(gsm, tws, t, lo, n, q, qinv0, nf, sh);
        else if (mode == MODE_LAZY)
            pass_rounds<B, C, FIRST, SCALE_LAST, RBMAX, MODE_LAZY, WARPMAP, PADL>(gsm, tws, t, lo, n, q, qinv0, nf, sh);
        else if (mode == MODE_HALF)
            pass_rounds<B, C, FIRST, SCALE_LAST, RBMAX, MODE_HALF, WARPMAP, PADL>(gsm, tws, t, lo, n, q, qinv0, nf, sh);
        else
            pass_rounds<B, C, FIRST, SCALE_LAST, RBMAX, MODE_FULL, WARPMAP, PADL>(gsm, tws, t, lo, n, q, qinv0, nf, sh);
        if (WARPMAP) __syncthreads();   // the store phase reads every group
    }

    // ---------------- store phase: shared -> global, coalesced; all smem reads first
    {
        uint4 outv[PER];
        if ((NTT_BULK & 2) && FIRST && !SINGLE && gbits > 0 && !a.fout) {
            // a group's output is one contiguous row of the working order (G residues at
            // brev(g) G): its 8-residue chunks (128 B, contiguous in the padded layout) leave
            // by bulk copies, one per thread; results must be visible to the async proxy first
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            constexpr int CH = G / 8;
            for (int j = tid; j < C * CH; j += NT) {
                const int c = j / CH, k = j - c * CH;
                const uint64_t gg = gg_of(c);
                if (gg >= a.total_groups) continue;
                const uint64_t poly = gg >> gbits, g = gg & gmask;
                uint4* dstp = a.dst + poly * N + ((uint64_t)brev_bits((uint32_t)g, gbits) << B) + 8 * k;
                bulk_s2g(dstp, dsm + c * GS + 9 * k, 128);
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");     // written (the next pass may read)
            asm volatile("fence.proxy.async.global;" ::: "memory");
        } else if (FIRST) {
            // groups are contiguous rows of the working order: e = tid + i NT -> (c, l), l fastest
#pragma unroll
            for (int i = 0; i < PER; i++) {
                const int e = tid + i * NT;
                outv[i] = dsm[(e / G) * GS + slot<B, PADL, RB>(e % G)];
            }
#pragma unroll
            for (int i = 0; i < PER; i++) {
                const int e = tid + i * NT;
                const int c = e / G, l = e % G;
                const uint64_t gg = gg_of(c);
                if (gg >= a.total_groups) continue;
                const uint64_t poly = gg >> gbits, g = gg & gmask;
                const uint64_t idx = ((uint64_t)brev_bits((uint32_t)g, gbits) << B) | (uint64_t)l;
                uint4 v = outv[i];
                if (SINGLE && a.psm && !a.fout) {   // pseudo-Mersenne class: any representative -> canonical
                    const ModC& M = a.mods[a.nq == 1 ? 0 : (uint32_t)poly];
                    const uint32_t q[4] = {M.q[0], M.q[1], M.q[2], M.q[3]};
                    const uint32_t s = psm_shift(q);
                    v = u128_to(psm_canon(u128_from(v), q, s, psm_C(q, s)));
                }
                if (!SINGLE && gbits == 0 && !a.fout) {
                    // the whole transform was this pass (four-step sub-transforms of 2^9 run the
                    // padded multi-pass kernel as their single pass): lazy classes -> canonical
                    const QPar& M = a.qp[a.nq == 1 ? 0 : (uint32_t)poly];
                    const uint32_t q[4] = {M.q[0], M.q[1], M.q[2], M.q[3]};
                    const int mode = a.psm ? MODE_PSM : mode_of(q);
                    if (mode == MODE_PSM) {
                        const uint32_t s = psm_shift(q);
                        v = u128_to(psm_canon(u128_from(v), q, s, psm_C(q, s)));
                    } else {
                        if (mode == MODE_LAZY) {
                            const uint32_t q2[4] = {q[0] << 1, (q[1] << 1) | (q[0] >> 31), (q[2] << 1) | (q[1] >> 31),
                                                    (q[3] << 1) | (q[2] >> 31)};
                            v = u128_to(reduce_2q(u128_from(v), q2));
                        }
                        if (mode != MODE_FULL) v = u128_to(reduce_2q(u128_from(v), q));
                    }
                }
                if (a.fout) {
                    const uint32_t m = a.nq == 1 ? 0 : (uint32_t)poly;
                    const ModC& M = a.mods[m];
                    const uint32_t q[4] = {M.q[0], M.q[1], M.q[2], M.q[3]};
                    v = u128_to(mont_mul(u128_from(v), u128_from(__ldg(a.fout + m * a.f_stride + idx)), q, M.qinv0));
                }
                if ((SINGLE || gbits == 0) && a.r_lb)   // four-step: straight into the destination rank's block
                    a.rdst[idx >> a.r_lb][poly * a.r_ps + (idx & ((1ull << a.r_lb) - 1))] = v;
                else
                    a.dst[poly * N + idx] = v;
            }
        } else {
            // same (c_me, rows t0 + i T) assignment as the load phase
#pragma unroll
            for (int i = 0; i < PER; i++) outv[i] = smc[slot<B, PADL, RB>(lbase + (i << LT))];
            if (!SINGLE && lo + B == n && !a.fout) {
                // lazy classes leave the last pass in [0, 4q) / [0, 2q): canonicalize
                const QPar& M = a.qp[a.nq == 1 ? 0 : (uint32_t)(gg0 >> gbits)];
                const uint32_t q[4] = {M.q[0], M.q[1], M.q[2], M.q[3]};
                const int mode = a.psm ? MODE_PSM : mode_of(q);
                if (mode == MODE_PSM) {
                    const uint32_t s = psm_shift(q), Cq = psm_C(q, s);
#pragma unroll
                    for (int i = 0; i < PER; i++) outv[i] = u128_to(psm_canon(u128_from(outv[i]), q, s, Cq));
                } else {
                    if (mode == MODE_LAZY) {
                        const uint32_t q2[4] = {q[0] << 1, (q[1] << 1) | (q[0] >> 31), (q[2] << 1) | (q[1] >> 31),
                                                (q[3] << 1) | (q[2] >> 31)};
#pragma unroll
                        for (int i = 0; i < PER; i++) outv[i] = u128_to(reduce_2q(u128_from(outv[i]), q2));
                    }
                    if (mode != MODE_FULL) {
#pragma unroll
                        for (int i = 0; i < PER; i++) outv[i] = u128_to(reduce_2q(u128_from(outv[i]), q));
                    }
                }
            }
            if (live) {
                uint4* dstp = a.dst + poly_me * N + gbase;
                if (a.fout) {   // !FIRST: a multi-pass kernel -- block-uniform modulus index
                    const QPar& M = a.qp[a.nq == 1 ? 0 : (uint32_t)(gg0 >> gbits)];
                    const uint32_t q[4] = {M.q[0], M.q[1], M.q[2], M.q[3]};
#pragma unroll
                    for (int i = 0; i < PER; i++)
                        outv[i] = u128_to(mont_mul(u128_from(outv[i]),
                                                   u128_from(__ldg(a.fout + m_me * a.f_stride + gbase + (size_t)i * gstride)), q, M.qinv0));
                }
                if (!SINGLE && a.r_lb && lo + B == n) {   // four-step: into the destination rank's block
#pragma unroll
                    for (int i = 0; i < PER; i++) {
                        const uint64_t k = gbase + (size_t)i * gstride;
                        a.rdst[k >> a.r_lb][poly_me * a.r_ps + (k & ((1ull << a.r_lb) - 1))] = outv[i];
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < PER; i++) dstp[(size_t)i * gstride] = outv[i];
                }
            }
        }
    }
    if (!SINGLE && a.cnt_out) {
        // all of this CTA's stores happen-before the release (barrier + cumulative release)
        __syncthreads();
        if (PM) {                         // one signal per polynomial of the CTA
            if (tid < C) red_release_gpu_add(a.cnt_out + (gg_of(tid) >> gbits), 1u);
        } else if (tid == 0) {
            red_release_gpu_add(a.cnt_out + (gg0 >> gbits), 1u);
        }
    }
#if NTT_TRACE
    if (tid == 0 && !SINGLE && g_trace) {
        const unsigned long long k = atomicAdd(&g_trace_n, 1ull);
        if (k < g_trace_cap) g_trace[k] = make_uint4(tr_t0, tr_t1, gtimer_lo(), (smid() << 16) | (a.lo << 8) | (FIRST ? 1u : 0u));
    }
#endif
}

// ----------------------------------------------------------------------------- first pass, TL groups per CTA
// (DESIGN.md §6 "Two tiles per CTA").  A multi-pass first pass shares ONE twiddle set among
// all its groups, so a CTA can own TL consecutive groups of one polynomial for the shared
// memory of TL data tiles + one set: every tile's gather is issued up front (one cp.async
// group per tile), tile k + 1's loads land while tile k computes, tile k's stores drain while
// tile k + 1 computes, and the CTA signals the pass-overlap counter once for TL groups (one
// release fence instead of TL).  Same arithmetic, addressing and layouts as k_ntt_pass's
// FIRST path with C = 1; plain cyclic I/O only (no load-side factors, natural layout).
#ifndef NTT_FIRST_TILES
#define NTT_FIRST_TILES 2
#endif
#ifndef NTT_FIRST_TILES9
#define NTT_FIRST_TILES9 2    // 9-stage first passes: two tiles with radix-4 rounds (128 threads, 64
#endif                        // registers, 8 CTAs per SM) +0.7..0.8 % at 2^15 / 2^17; with the radix-8
#ifndef NTT_FIRST9_RB         // rounds (80 registers) shared memory caps residency: -2.6 % (first_tiles_ab)
#define NTT_FIRST9_RB 2
#endif
template <int B, int RBMAX, int TL>
__global__ void __launch_bounds__(PassShape<B, RBMAX>::T,
                                  (PassOcc<B, RBMAX, false>::THREADS / PassShape<B, RBMAX>::T) > 0
                                      ? PassOcc<B, RBMAX, false>::THREADS / PassShape<B, RBMAX>::T : 1)
k_ntt_first_tl(const __grid_constant__ PassArgs a) {
    constexpr int C = 1;
    using S = PassShape<B, RBMAX, C, true>;
    constexpr int G = S::G, RB = S::RB, T = S::T, GS = S::GS;
    constexpr int LT = B - RB;
    constexpr int PER = G / T;                       // == E
    constexpr bool WARPMAP = T <= 32 && (32 % T) == 0;
    static_assert(B >= 8, "twiddles by bulk copy");
    static_assert(TL >= 1 && (TL & (TL - 1)) == 0, "a CTA's groups stay in one polynomial: TL a power of two");
    extern __shared__ __align__(128) uint4 sm[];
    uint4* const dsm = sm;                           // [TL][GS] data tiles
    uint4* const tsm = dsm + TL * GS;                // the pass's one twiddle set
    __shared__ __align__(8) uint64_t tw_bar;

    const uint32_t n = a.n, gbits = n - B;
    const uint64_t N = 1ull << n;
    const uint64_t gmask = (1ull << gbits) - 1;
    uint64_t gg0 = (uint64_t)blockIdx.x * TL;        // TL divides the groups of a polynomial
    if (a.nq > 1) gg0 = ((uint64_t)a.ord[gg0 >> gbits] << gbits) | (gg0 & gmask);
    const int tid = threadIdx.x;
    const uint64_t ggl = gg0 < a.total_groups ? gg0 : a.total_groups - 1;
    const uint64_t poly = ggl >> gbits;
    const uint32_t m = a.nq == 1 ? 0 : (uint32_t)poly;
    if (tid == 0) {
        mbar_init(&tw_bar, 1);
        mbar_expect_tx(&tw_bar, (G - 1) * 16);
        bulk_g2s(tsm, a.pt + m * a.pt_stride, (G - 1) * 16, &tw_bar);
    }
    if (a.pdl_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (a.cnt_in) {
        if (tid == 0) {
            const uint32_t* cp = a.cnt_in + poly;
            while ((int32_t)(ld_acquire_gpu(cp) - a.target) < 0) __nanosleep(128);
        }
        __syncthreads();
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // gathers: row r = t0 + i T of group g holds local index brev_B(r) (k_ntt_pass, C = 1)
    constexpr int RT = 3 < LT ? 3 : LT;
    const int t0 = (tid >> RT) | ((tid & ((1 << RT) - 1)) << (LT - RT));
    const int lbase = (int)brev_bits((uint32_t)t0, B);
    const uint64_t gstride = (uint64_t)T << gbits;
#pragma unroll
    for (int k = 0; k < TL; k++) {
        const uint64_t gg = gg0 + k;
        if (gg < a.total_groups) {
            const uint4* srcp = a.src + poly * N + (((uint64_t)t0 << gbits) | (gg & gmask));
            uint4* smc = dsm + k * GS;
#pragma unroll
            for (int i = 0; i < PER; i++)
                cp_async16(smc + slot<B, true, RB>(lbase | (int)brev_bits((uint32_t)i, RB)), srcp + (size_t)i * gstride);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    const QPar& M = a.qp[m];
    uint32_t q[4] = {M.q[0], M.q[1], M.q[2], M.q[3]};
    const uint32_t qinv0 = M.qinv0;
    const int mode = a.psm ? MODE_PSM : mode_of(q);
    const U128 nf = U128{{0, 0, 0, 0}};
#pragma unroll
    for (int k = 0; k < TL; k++) {
        // tile k's copies done (the later tiles' may still be in flight)
        if (k == 0) asm volatile("cp.async.wait_group %0;" ::"n"(TL - 1) : "memory");
        else if (k == 1) asm volatile("cp.async.wait_group %0;" ::"n"(TL > 2 ? TL - 2 : 0) : "memory");
        else asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        if (k == 0) mbar_wait(&tw_bar, 0);
        const uint64_t gg = gg0 + k;
        uint4* gsm = dsm + k * GS;
        if (mode == MODE_PSM)
            pass_rounds<B, C, true, false, RBMAX, MODE_PSM, WARPMAP, true>(gsm, tsm, tid, 0, n, q, qinv0, nf, 0);
        else if (mode == MODE_LAZY)
            pass_rounds<B, C, true, false, RBMAX, MODE_LAZY, WARPMAP, true>(gsm, tsm, tid, 0, n, q, qinv0, nf, 0);
        else if (mode == MODE_HALF)
            pass_rounds<B, C, true, false, RBMAX, MODE_HALF, WARPMAP, true>(gsm, tsm, tid, 0, n, q, qinv0, nf, 0);
        else
            pass_rounds<B, C, true, false, RBMAX, MODE_FULL, WARPMAP, true>(gsm, tsm, tid, 0, n, q, qinv0, nf, 0);
        if (WARPMAP) __syncthreads();
        if (gg < a.total_groups) {   // the group is one contiguous row of the working order
            uint4 outv[PER];
#pragma unroll
            for (int i = 0; i < PER; i++) outv[i] = gsm[slot<B, true, RB>(tid + i * T)];
            uint4* dstp = a.dst + poly * N + ((uint64_t)brev_bits((uint32_t)(gg & gmask), gbits) << B);
#pragma unroll
            for (int i = 0; i < PER; i++) dstp[tid + i * T] = outv[i];
        }
    }
    if (a.cnt_out) {
        __syncthreads();
        if (tid == 0) red_release_gpu_add(a.cnt_out + poly, 1u);
    }
}

// ----------------------------------------------------------------------------- later pass, TL polynomials per CTA
// One-modulus plans (nq == 1): the twiddle set of a later-pass group depends only on its L
// (and the modulus), so group g of TL consecutive polynomials shares one set -- the same
// two-tile scheme as k_ntt_first_tl for the later passes of plain cyclic one-modulus plans
// (BASELINE cfg 4 and 5 shapes).  The CTA signals each of its polynomials' counters once.
#ifndef NTT_LATER_TILES
#define NTT_LATER_TILES 2
#endif
template <int B, bool SCALE_LAST, int RBMAX, int TL>
__global__ void __launch_bounds__(PassShape<B, RBMAX>::T,
                                  (PassOcc<B, RBMAX, false>::THREADS / PassShape<B, RBMAX>::T) > 0
                                      ? PassOcc<B, RBMAX, false>::THREADS / PassShape<B, RBMAX>::T : 1)
k_ntt_later_tl(const __grid_constant__ PassArgs a) {
    constexpr int C = 1;
    using S = PassShape<B, RBMAX, C, true>;
    constexpr int G = S::G, RB = S::RB, T = S::T, GS = S::GS;
    constexpr int LT = B - RB;
    constexpr int PER = G / T;
    constexpr bool WARPMAP = T <= 32 && (32 % T) == 0;
    static_assert(B >= 8, "twiddles by bulk copy");
    extern __shared__ __align__(128) uint4 sm[];
    uint4* const dsm = sm;                           // [TL][GS] data tiles
    uint4* const tsm = dsm + TL * GS;                // the group's twiddle set (shared by the TL polynomials)
    __shared__ __align__(8) uint64_t tw_bar;

    const uint32_t n = a.n, lo = a.lo, gbits = n - B;
    const uint64_t N = 1ull << n;
    const uint64_t gpp = 1ull << gbits;              // groups per polynomial
    const uint64_t g = blockIdx.x & (gpp - 1);
    const uint64_t p0 = (uint64_t)(blockIdx.x >> gbits) * TL;   // TL divides the batch
    const int tid = threadIdx.x;
    const uint64_t H = g >> lo, L = g & ((1ull << lo) - 1);
    if (tid == 0) {
        mbar_init(&tw_bar, 1);
        mbar_expect_tx(&tw_bar, (G - 1) * 16);
        bulk_g2s(tsm, a.pt + L * (G - 1), (G - 1) * 16, &tw_bar);
    }
    if (a.pdl_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (a.cnt_in) {
        if (tid < TL) {
            const uint32_t* cp = a.cnt_in + p0 + tid;
            while ((int32_t)(ld_acquire_gpu(cp) - a.target) < 0) __nanosleep(128);
        }
        __syncthreads();
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // rows t + i T of group (H, L): elements H 2^(lo+B) + (t + i T) 2^lo + L
    const uint64_t gbase = (H << (lo + B)) | ((uint64_t)tid << lo) | L;
    const uint64_t gstride = (uint64_t)T << lo;
#pragma unroll
    for (int k = 0; k < TL; k++) {
        const uint4* srcp = a.src + (p0 + k) * N + gbase;
        uint4* smc = dsm + k * GS;
#pragma unroll
        for (int i = 0; i < PER; i++) cp_async16(smc + slot<B, true, RB>(tid + (i << LT)), srcp + (size_t)i * gstride);
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    const QPar& M = a.qp[0];
    uint32_t q[4] = {M.q[0], M.q[1], M.q[2], M.q[3]};
    const uint32_t qinv0 = M.qinv0;
    U128 nf = U128{{0, 0, 0, 0}};
    if (SCALE_LAST) {
        const uint32_t* src = a.ninv_r ? M.ninv_rm : M.ninv_m;
        nf = U128{{src[0], src[1], src[2], src[3]}};
    }
    const uint32_t sh = (NTT_SHIFT_SCALE && SCALE_LAST && !a.ninv_r && n >= 2) ? n : 0u;
    const int mode = a.psm ? MODE_PSM : mode_of(q);
    const bool last_pass = lo + B == n;
#pragma unroll
    for (int k = 0; k < TL; k++) {
        if (k == 0) asm volatile("cp.async.wait_group %0;" ::"n"(TL - 1) : "memory");
        else if (k == 1) asm volatile("cp.async.wait_group %0;" ::"n"(TL > 2 ? TL - 2 : 0) : "memory");
        else asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        if (k == 0) mbar_wait(&tw_bar, 0);
        uint4* gsm = dsm + k * GS;
        if (mode == MODE_PSM)
            pass_rounds<B, C, false, SCALE_LAST, RBMAX, MODE_PSM, WARPMAP, true>(gsm, tsm, tid, lo, n, q, qinv0, nf, sh);
        else if (mode == MODE_LAZY)
            pass_rounds<B, C, false, SCALE_LAST, RBMAX, MODE_LAZY, WARPMAP, true>(gsm, tsm, tid, lo, n, q, qinv0, nf, sh);
        else if (mode == MODE_HALF)
            pass_rounds<B, C, false, SCALE_LAST, RBMAX, MODE_HALF, WARPMAP, true>(gsm, tsm, tid, lo, n, q, qinv0, nf, sh);
        else
            pass_rounds<B, C, false, SCALE_LAST, RBMAX, MODE_FULL, WARPMAP, true>(gsm, tsm, tid, lo, n, q, qinv0, nf, sh);
        if (WARPMAP) __syncthreads();
        uint4 outv[PER];
#pragma unroll
        for (int i = 0; i < PER; i++) outv[i] = gsm[slot<B, true, RB>(tid + (i << LT))];
        if (last_pass && mode == MODE_PSM) {
            const uint32_t s = psm_shift(q), Cq = psm_C(q, s);
#pragma unroll
            for (int i = 0; i < PER; i++) outv[i] = u128_to(psm_canon(u128_from(outv[i]), q, s, Cq));
        } else if (last_pass && mode != MODE_FULL) {   // lazy classes leave the transform canonical
            if (mode == MODE_LAZY) {
                const uint32_t q2[4] = {q[0] << 1, (q[1] << 1) | (q[0] >> 31), (q[2] << 1) | (q[1] >> 31),
                                        (q[3] << 1) | (q[2] >> 31)};
#pragma unroll
                for (int i = 0; i < PER; i++) outv[i] = u128_to(reduce_2q(u128_from(outv[i]), q2));
            }
#pragma unroll
            for (int i = 0; i < PER; i++) outv[i] = u128_to(reduce_2q(u128_from(outv[i]), q));
        }
        uint4* dstp = a.dst + (p0 + k) * N + gbase;
#pragma unroll
        for (int i = 0; i < PER; i++) dstp[(size_t)i * gstride] = outv[i];
    }
    if (a.cnt_out) {
        __syncthreads();
        if (tid < TL) red_release_gpu_add(a.cnt_out + p0 + tid, 1u);
    }
}

// ----------------------------------------------------------------------------- permutation-free negacyclic passes
// SURVEY §8(f) f1 (DESIGN.md §6 "Bit-reversed negacyclic path").  Forward: Cooley-Tukey
// butterflies with psi-merged twiddles, natural-order input, stages from the top index
// bit down, output in bit-reversed order: Y[i] = a(psi^(2 brev(i) + 1)) -- no twist
// multiply and no permutation.  Inverse: Gentleman-Sande butterflies (u + v, (u - v) w)
// from bit-reversed input, stages from bit 0 up, psi^-1 twiddles, N^-1 folded into the
// last stage.  Stage on global bit b pairs j and j + 2^b (bit b of j clear) with twiddle
// psi^(+-brev_n(2^(n-1-b) + (j >> (b+1)))).  A pass covers bits [lo, lo + B) of the
// group (H, L): elements H 2^(lo+B) + r 2^lo + L; its twiddles depend on H and on r's
// bits above the stage, so a table holds per H the 2^B - 1 values in [local stage][block]
// order (offset 2^(B-1-sl) - 1 for local stage sl).

// GS butterfly (u, v) -> (u + v, (u - v) w) [* nf on u in the last stage], per mode:
// FULL canonical; HALF values in [0, 2q) (add/sub mod 2q); LAZY values in [0, 2q)
// (u + v reduced by 2q, u - v + 2q fed to the lazy product, which accepts < 4q).
template <int MODE, bool SCALE_U>
__device__ __forceinline__ void gs_bfly(U128& u, U128& v, const U128& w, const uint32_t q[4], const uint32_t q2[4],
                                        uint32_t qinv0, const U128& nf, uint32_t sh = 0) {
    if (MODE == MODE_FULL) {
        const U128 s = add_mod(u, v, q);
        const U128 d = sub_mod(u, v, q);
        u = SCALE_U ? (sh ? shr_mod(s, sh, q, qinv0) : mont_mul(s, nf, q, qinv0)) : s;
        v = mont_mul(d, w, q, qinv0);
    } else if (MODE == MODE_HALF) {
        const U128 s = add_mod(u, v, q2);
        const U128 d = sub_mod(u, v, q2);
        u = SCALE_U ? (sh ? shr_mod_lazy(s, sh, q, qinv0) : mont_mul_lazy(s, nf, q, qinv0)) : s;
        v = mont_mul_lazy(d, w, q, qinv0);
    } else {
        const U128 s = add_nored(u, v);                 // < 4q
        const U128 d = sub_add_nored(u, v, q2);         // in (0, 4q)
        u = SCALE_U ? (sh ? shr_mod_lazy(s, sh, q, qinv0) : mont_mul_lazy(s, nf, q, qinv0)) : reduce_2q(s, q2);
        v = mont_mul_lazy(d, w, q, qinv0);
    }
}

// Register rounds of a permutation-free pass: the windows of pass_rounds, visited top-down
// (forward, each window's stages from its top bit) or bottom-up (inverse).
template <int B, int C, bool INV, bool SCALE_LAST, int RBMAX, int MODE>
__device__ __forceinline__ void nc_rounds(uint4* gsm, const uint4* tws, const int t, const uint32_t lo, const uint32_t n,
                                          const uint32_t q[4], const uint32_t qinv0, const U128 nf, const uint32_t sh) {
    uint32_t q2[4] = {0, 0, 0, 0};
    if (MODE != MODE_FULL) {
        q2[0] = q[0] << 1;
        q2[1] = (q[1] << 1) | (q[0] >> 31);
        q2[2] = (q[2] << 1) | (q[1] >> 31);
        q2[3] = (q[3] << 1) | (q[2] >> 31);
    }
    using S = PassShape<B, RBMAX, C, true>;
    constexpr int RB = S::RB, E = S::E, R = S::ROUNDS;
#pragma unroll 1
    for (int it = 0; it < R; it++) {
        const int rd = INV ? it : R - 1 - it;
        const int slo = rd * RB;
        const int w = (slo + RB <= B) ? slo : B - RB;   // window [w, w + RB); its own stages are [slo, ..)
        const int tlo = t & ((1 << w) - 1);
        const int thi = (t >> w) << (w + RB);
        const int l0 = thi | tlo;
        const int s0 = S::LINEAR ? slot<B, true>(l0) : 0;
        const int st = S::LINEAR ? (w >= 3 ? (9 << (w - 3)) : (1 << w)) : 0;
        // window rd owns stages [slo, min(slo + RB, B)) (the last window overlaps the one
        // below it); the forward visits windows and their stages top-down
        U128 x[E];
#pragma unroll
        for (int k = 0; k < E; k++) x[k] = u128_from(gsm[S::LINEAR ? s0 + k * st : slot<B, true>(l0 | (k << w))]);
#pragma unroll
        for (int bb = 0; bb < RB; bb++) {
            const int bit = INV ? bb : RB - 1 - bb;
            const int sl = w + bit;
            if (sl < slo) continue;
            // twiddle (local stage sl, block r >> (sl + 1)): offset(sl) + (thi >> (w+RB) << (RB-1-bit)) + (k0 >> (bit+1))
            const uint4* tp = tws + ((1 << (B - 1 - sl)) - 1) + ((thi >> (w + RB)) << (RB - 1 - bit));
            U128 tw[E / 2];
#pragma unroll
            for (int j = 0; j < (E / 2 >> bit); j++) tw[j] = u128_from(tp[j]);
            const bool last = INV && SCALE_LAST && lo + sl == n - 1;
#pragma unroll
            for (int kk = 0; kk < E / 2; kk++) {
                const int k0 = ((kk >> bit) << (bit + 1)) | (kk & ((1 << bit) - 1));
                const int k1 = k0 | (1 << bit);
                const U128& wv = tw[k0 >> (bit + 1)];
                if (!INV) bfly<MODE, false>(x[k0], x[k1], wv, q, q2, qinv0, nf);
                else if (last) gs_bfly<MODE, true>(x[k0], x[k1], wv, q, q2, qinv0, nf, sh);
                else gs_bfly<MODE, false>(x[k0], x[k1], wv, q, q2, qinv0, nf);
            }
        }
#pragma unroll
        for (int k = 0; k < E; k++) gsm[S::LINEAR ? s0 + k * st : slot<B, true>(l0 | (k << w))] = u128_to(x[k]);
        if (S::T <= 32) __syncwarp(); else __syncthreads();
    }
}

template <int B, int C, bool INV, bool SCALE_LAST, int RBMAX>
__global__ void __launch_bounds__(C * PassShape<B, RBMAX>::T,
                                  (PassOcc<B, RBMAX, false>::THREADS / (C * PassShape<B, RBMAX>::T)) > 0
                                      ? PassOcc<B, RBMAX, false>::THREADS / (C * PassShape<B, RBMAX>::T) : 1)
k_nc_pass(const __grid_constant__ PassArgs a) {
    using S = PassShape<B, RBMAX, C, true>;
    constexpr int G = S::G, RB = S::RB, T = S::T, GS = S::GS, TS = S::TS;
    constexpr int NT = C * T;
    static_assert((T <= 32 && 32 % T == 0) || C == 1, "groups are warp-owned or alone in their CTA");
    extern __shared__ uint4 sm[];
    uint4* tsm = sm + C * GS;                        // [C][TS] twiddle sets (1 used when lo > 0)

    const uint32_t n = a.n, lo = a.lo, gbits = n - B;
    const uint64_t N = 1ull << n;
    const uint64_t gmask = (1ull << gbits) - 1;
    uint64_t gg0 = (uint64_t)blockIdx.x * C;
    if (a.nq > 1) gg0 = ((uint64_t)a.ord[gg0 >> gbits] << gbits) | (gg0 & gmask);   // kernel-parameter table: uniform
    const int tid = threadIdx.x;
    constexpr int LT = B - RB;
    const int c_me = tid % C, t0 = tid / C;
    const uint64_t poly = gg0 >> gbits;
    const uint64_t g_me = (gg0 + c_me) & gmask;
    const uint32_t m_me = a.nq == 1 ? 0 : (uint32_t)poly;
    // twiddle sets: indexed by H = g >> lo; the C groups share one set unless lo == 0
    const bool shared_set = lo > 0;
    {
        constexpr int TW_IT = (G - 1 + NT - 1) / NT;
        const uint64_t H0 = (gg0 & gmask) >> lo;
        const uint4* src = a.pt + m_me * a.pt_stride + H0 * (G - 1) + tid;
        uint4* dst = tsm + tid;
#pragma unroll
        for (int c = 0; c < C; c++) {
            if (c > 0 && shared_set) break;
#pragma unroll
            for (int i = 0; i < TW_IT; i++)
                if ((G - 1) % NT == 0 || i + 1 < TW_IT || tid + i * NT < G - 1)
                    cp_async16(dst + c * TS + i * NT, src + c * (G - 1) + i * NT);
        }
    }
    if (a.pdl_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (a.cnt_in) {
        if (tid == 0) {
            const uint32_t* cp = a.cnt_in + poly;
            while ((int32_t)(ld_acquire_gpu(cp) - a.target) < 0) __nanosleep(128);
        }
        __syncthreads();
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    constexpr int PER = (C * G) / NT;
    const uint64_t H = g_me >> lo, L = g_me & ((1ull << lo) - 1);
    const uint64_t gbase = (H << (lo + B)) | ((uint64_t)t0 << lo) | L;
    const uint32_t gstride = (uint32_t)T << lo;
    const int lbase = t0;
    const uint4* srcp = a.src + poly * N + gbase;
    uint4* smc = sm + c_me * GS;
    if (!a.pmul) {
#pragma unroll
        for (int i = 0; i < PER; i++) cp_async16(smc + slot<B, true>(lbase + (i << LT)), srcp + (size_t)i * gstride);
    } else {   // fused point-wise Montgomery product of two bit-reversed spectra
        uint4 va[PER], vb[PER];
        const uint4* pm = a.pmul + poly * N + gbase;
#pragma unroll
        for (int i = 0; i < PER; i++) { va[i] = __ldcg(srcp + (size_t)i * gstride); vb[i] = __ldcg(pm + (size_t)i * gstride); }
        const QPar& M = a.qp[m_me];   // kernel parameters, block-uniform index
        const uint32_t q[4] = {M.q[0], M.q[1], M.q[2], M.q[3]};
#pragma unroll
        for (int i = 0; i < PER; i++)
            smc[slot<B, true>(lbase + (i << LT))] = u128_to(mont_mul(u128_from(va[i]), u128_from(vb[i]), q, M.qinv0));
    }
    cp_async_wait_all();
    __syncthreads();
    {
        const int c = tid / T, t = tid % T;
        uint32_t q[4], qinv0;
        U128 nf;
        {
            const QPar& M = a.qp[m_me];   // kernel parameters, block-uniform index: uniform registers
            q[0] = M.q[0]; q[1] = M.q[1]; q[2] = M.q[2]; q[3] = M.q[3];
            qinv0 = M.qinv0;
            const uint32_t* src = a.ninv_r ? M.ninv_rm : M.ninv_m;
            nf = U128{{src[0], src[1], src[2], src[3]}};
        }
        uint4* gsm = sm + c * GS;
        const uint4* tws = tsm + (shared_set ? 0 : c) * TS;
        const int mode = mode_of(q);
        const uint32_t sh = (NTT_SHIFT_SCALE && SCALE_LAST && !a.ninv_r && n >= 2) ? n : 0u;   // plain inverse: N^-1 by shifting
        if (mode == MODE_LAZY) nc_rounds<B, C, INV, SCALE_LAST, RBMAX, MODE_LAZY>(gsm, tws, t, lo, n, q, qinv0, nf, sh);
        else if (mode == MODE_HALF) nc_rounds<B, C, INV, SCALE_LAST, RBMAX, MODE_HALF>(gsm, tws, t, lo, n, q, qinv0, nf, sh);
        else nc_rounds<B, C, INV, SCALE_LAST, RBMAX, MODE_FULL>(gsm, tws, t, lo, n, q, qinv0, nf, sh);
        __syncthreads();
    }
    {
        uint4 outv[PER];
#pragma unroll
        for (int i = 0; i < PER; i++) outv[i] = smc[slot<B, true>(lbase + (i << LT))];
        // the transform's last pass returns canonical values (lazy classes are in [0, 4q) / [0, 2q))
        const bool last_pass = INV ? (lo + B == n) : (lo == 0);
        if (last_pass) {
            const QPar& M = a.qp[m_me];
            const uint32_t q[4] = {M.q[0], M.q[1], M.q[2], M.q[3]};
            const int mode = mode_of(q);
            if (mode == MODE_LAZY && !INV) {
                const uint32_t q2[4] = {q[0] << 1, (q[1] << 1) | (q[0] >> 31), (q[2] << 1) | (q[1] >> 31),
                                        (q[3] << 1) | (q[2] >> 31)};
#pragma unroll
                for (int i = 0; i < PER; i++) outv[i] = u128_to(reduce_2q(u128_from(outv[i]), q2));
            }
            if (mode != MODE_FULL) {
#pragma unroll
                for (int i = 0; i < PER; i++) outv[i] = u128_to(reduce_2q(u128_from(outv[i]), q));
            }
        }
        uint4* dstp = a.dst + poly * N + gbase;
#pragma unroll
        for (int i = 0; i < PER; i++) dstp[(size_t)i * gstride] = outv[i];
    }
    if (a.cnt_out) {
        __syncthreads();
        if (tid == 0) red_release_gpu_add(a.cnt_out + poly, 1u);
    }
}

// ----------------------------------------------------------------------------- cluster latency kernel
// One polynomial on a cluster of 8 CTAs (8 SMs) with distributed shared memory, for the
// latency configuration (BASELINE cfg 1: one N = 2^10 transform; cyclic single-pass plans
// with N = 2^8 .. 2^11 and few polynomials).  One SM is throughput-bound on N/2 log N
// butterflies (3.7 us for N = 2^10 at 0.7 butterflies/clk); eight SMs leave the stage
// latency (one butterfly per thread per stage) as the bound.  N = 8 M, CTA r of the
// cluster owns positions [r M, (r + 1) M) of the bit-reversed working order:
//  * phase 1 (stages 0 .. LM - 1, LM = log2 M): positions p = r M + i, i < M, gathered
//    from x[brev_LM(i) 8 + brev_3(r)]; radix-2 stages in the CTA's shared memory, one
//    butterfly per thread per stage;
//  * phase 2 (stages LM .. LM + 2): the group of g < M is {g + k M : k < 8}, element k in
//    CTA k's shared memory at offset g.  CTA r takes groups [r M/8, (r + 1) M/8), reads its
//    first-stage pairs straight from the owners' shared memory (ld.shared::cluster), and
//    the last stage stores natural-order outputs p = g + k M to global memory.
// Every twiddle a thread uses (LM + 3 of them) is loaded into registers before the
// dependency wait.  Values stay canonical (any odd q < 2^128).
#include <cooperative_groups.h>
#ifndef NTT_CLU_LOG
#define NTT_CLU_LOG 3    // log2 CTAs per cluster (8: portable cluster size)
#endif
constexpr int CLU_LOG = NTT_CLU_LOG, CLU = 1 << CLU_LOG;

__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint4 ld_dsmem(const uint4* local, uint32_t rank) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(local);
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    uint4 v;
    asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(ra) : "memory");
    return v;
}

template <int LB, bool SCALE_LAST>
__global__ void __launch_bounds__(1 << (LB - CLU_LOG - 1)) k_ntt_cluster(const PassArgs a) {
    constexpr int LM = LB - CLU_LOG, M = 1 << LM, NT = M / 2, GPC = M / CLU;   // groups per CTA
    __shared__ uint4 loc[M];     // phase 1 working set, read by the whole cluster
    __shared__ uint4 buf[M];     // phase 2: [GPC][8]
    const uint32_t r = cluster_rank();
    const uint64_t poly = blockIdx.x >> CLU_LOG;
    const uint32_t m = a.nq == 1 ? 0 : (uint32_t)poly;
    const int t = threadIdx.x;
    const uint4* pt = a.pt + m * a.pt_stride;                   // stage s, twiddle j at (2^s - 1) + j
    const int gl = t >> (CLU_LOG - 1), bb = t & (CLU / 2 - 1);  // phase 2: group, butterfly in group
    const int g = (int)r * GPC + gl;
    U128 tw[LB];
#pragma unroll
    for (int s = 1; s < LM; s++) tw[s] = u128_from(__ldg(pt + (1 << s) - 1 + (t & ((1 << s) - 1))));
#pragma unroll
    for (int sp = 0; sp < CLU_LOG; sp++) {
        const int k0 = ((bb >> sp) << (sp + 1)) | (bb & ((1 << sp) - 1));
        tw[LM + sp] = u128_from(__ldg(pt + (1 << (LM + sp)) - 1 + g + ((k0 & ((1 << sp) - 1)) << LM)));
    }
    const ModC& MC = a.mods[m];
    const uint32_t q[4] = {MC.q[0], MC.q[1], MC.q[2], MC.q[3]};
    const uint32_t q2[4] = {0, 0, 0, 0};
    const uint32_t qinv0 = MC.qinv0;
    U128 nf = U128{{0, 0, 0, 0}};
    if (SCALE_LAST) {
        const uint32_t* sp = a.ninv_r ? MC.ninv_rm : MC.ninv_m;
        nf = U128{{sp[0], sp[1], sp[2], sp[3]}};
    }
    if (a.pdl_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    // ---- phase 1: stage 0 on the two gathered inputs in registers, then stages 1 .. LM - 1
    {
        const uint4* src = a.src + (poly << LB);
        const uint32_t br = brev_bits(r, CLU_LOG);
        U128 u = u128_from(__ldcg(src + ((brev_bits(2 * t, LM) << CLU_LOG) | br)));
        U128 v = u128_from(__ldcg(src + ((brev_bits(2 * t + 1, LM) << CLU_LOG) | br)));
        bfly1<MODE_FULL>(u, v, q, q2);
        loc[2 * t] = u128_to(u);
        loc[2 * t + 1] = u128_to(v);
        __syncthreads();
#pragma unroll
        for (int s = 1; s < LM; s++) {
            const int j = t & ((1 << s) - 1), i0 = ((t >> s) << (s + 1)) | j, i1 = i0 | (1 << s);
            u = u128_from(loc[i0]);
            v = u128_from(loc[i1]);
            bfly<MODE_FULL, false>(u, v, tw[s], q, q2, qinv0, nf);
            loc[i0] = u128_to(u);
            loc[i1] = u128_to(v);
            if (s + 1 < LM) __syncthreads();
        }
    }
    cluster_arrive();            // phase-1 values of every CTA visible cluster-wide
    cluster_wait();

    // ---- phase 2: stages LM .. LM + 2 on groups of 8 (one element per CTA)
    {
        U128 u = u128_from(ld_dsmem(loc + g, 2 * bb)), v = u128_from(ld_dsmem(loc + g, 2 * bb + 1));
        cluster_arrive();        // this CTA's remote reads are done (owners wait before exiting)
        bfly<MODE_FULL, false>(u, v, tw[LM], q, q2, qinv0, nf);   // LM < LB - 1: never the last stage
        uint4* gb = buf + gl * CLU;
        gb[2 * bb] = u128_to(u);
        gb[2 * bb + 1] = u128_to(v);
        constexpr unsigned WM = NT >= 32 ? 0xffffffffu : ((1u << NT) - 1);   // a group's 4 threads share a warp
        __syncwarp(WM);
#pragma unroll
        for (int sp = 1; sp < CLU_LOG; sp++) {
            const int k0 = ((bb >> sp) << (sp + 1)) | (bb & ((1 << sp) - 1)), k1 = k0 | (1 << sp);
            u = u128_from(gb[k0]);
            v = u128_from(gb[k1]);
            if (SCALE_LAST && LM + sp == LB - 1) bfly<MODE_FULL, true>(u, v, tw[LM + sp], q, q2, qinv0, nf, (NTT_SHIFT_SCALE && !a.ninv_r) ? LB : 0u);
            else bfly<MODE_FULL, false>(u, v, tw[LM + sp], q, q2, qinv0, nf);
            if (sp + 1 < CLU_LOG) {
                gb[k0] = u128_to(u);
                gb[k1] = u128_to(v);
                __syncwarp(WM);
            } else {             // natural-order outputs p = g + k M
                uint4* dst = a.dst + (poly << LB);
                dst[g + (k0 << LM)] = u128_to(u);
                dst[g + (k1 << LM)] = u128_to(v);
            }
        }
    }
    cluster_wait();              // nobody still reads this CTA's shared memory
}

// ----------------------------------------------------------------------------- launch table
typedef void (*PassKernel)(const PassArgs);

struct PassCfg {
    PassKernel fn;
    int B, C, threads;
    size_t smem;
    bool tma = false;     // k_ntt_pass<..., TMA>: the launch must carry the data tile's tensor map
    bool first = false;
    bool single = false;  // one-pass kernel (several moduli per CTA: the device table, not QPar)
    int tiles = 1;        // groups per CTA beyond C, handled one after another (k_ntt_first_tl / k_ntt_later_tl)
    bool tiles_across = false;   // the tiles are one group of `tiles` polynomials (k_ntt_later_tl)
};

template <int B, int C, bool FIRST, bool SCALE_LAST, bool SINGLE = false, int RBMAX = 3, bool PM = false, bool TMA = false>
static PassCfg make_cfg() {
    using S = PassShape<B, RBMAX, C, !SINGLE>;
    PassCfg c;
    c.fn = k_ntt_pass<B, C, FIRST, SCALE_LAST, SINGLE, RBMAX, PM, TMA>;
    c.B = B;
    c.C = C;
    c.threads = C * S::T;
    c.tma = TMA;
    c.first = FIRST;
    c.single = SINGLE;
    const size_t ntw = (size_t)((FIRST && !SINGLE) ? 1 : C) * S::TS;
    c.smem = ((size_t)C * S::GS + ntw + (TMA ? 2 : 0)) * sizeof(uint4);   // TMA: + the pad slot, + two mbarriers
    return c;
}

// multi-pass first pass over TL groups per CTA (k_ntt_first_tl): plain cyclic I/O, C = 1
template <int B, int RB, int TL>
static PassCfg first_tl_cfg_t() {
    using S = PassShape<B, RB, 1, true>;
    PassCfg c;
    c.fn = k_ntt_first_tl<B, RB, TL>;
    c.B = B;
    c.C = 1;
    c.threads = S::T;
    c.first = true;
    c.tiles = TL;
    c.smem = ((size_t)TL * S::GS + S::TS) * sizeof(uint4);
    return c;
}

// later pass over group g of TL polynomials per CTA (k_ntt_later_tl): one-modulus plain cyclic plans
template <int B, bool SL, int RB, int TL>
static PassCfg later_tl_cfg_t() {
    using S = PassShape<B, RB, 1, true>;
    PassCfg c;
    c.fn = k_ntt_later_tl<B, SL, RB, TL>;
    c.B = B;
    c.C = 1;
    c.threads = S::T;
    c.tiles = TL;
    c.tiles_across = true;
    c.smem = ((size_t)TL * S::GS + S::TS) * sizeof(uint4);
    return c;
}

// Single pass (n = B <= 12): C polynomials per CTA, the pass is both first and last.
template <bool SL>
static PassCfg single_cfg_t(int B) {
    switch (B) {
        case 1: return make_cfg<1, 64, true, SL, true>();
        case 2: return make_cfg<2, 64, true, SL, true>();
        case 3: return make_cfg<3, 64, true, SL, true>();
        case 4: return make_cfg<4, 32, true, SL, true>();
        case 5: return make_cfg<5, 16, true, SL, true>();
        case 6: return make_cfg<6, 16, true, SL, true>();
        case 7: return make_cfg<7, 16, true, SL, true>();
        case 8: return make_cfg<8, NTT_S8_C, true, SL, true>();
        case 9: return make_cfg<9, NTT_S9_C, true, SL, true>();
        case 10: return make_cfg<10, NTT_S10_C, true, SL, true, NTT_S10_RB>();
        case 11: return make_cfg<11, 1, true, SL, true>();
        default: return make_cfg<12, 1, true, SL, true>();
    }
}
// Single pass for a few polynomials (latency, BASELINE cfg 1): one polynomial per CTA and
// radix-4 register rounds, so N/4 threads share the work instead of N/8 with idle groups.
template <bool SL>
static PassCfg single_lat_cfg_t(int B) {
    switch (B) {
        case 6: return make_cfg<6, 1, true, SL, true, 2>();
        case 7: return make_cfg<7, 1, true, SL, true, 2>();
        case 8: return make_cfg<8, 1, true, SL, true, 2>();
        case 9: return make_cfg<9, 1, true, SL, true, 2>();
        case 10: return make_cfg<10, 1, true, SL, true, 2>();
        case 11: return make_cfg<11, 1, true, SL, true, 2>();
        default: return make_cfg<12, 1, true, SL, true, 2>();
    }
}
#ifndef NTT_LAT_CTAS
#define NTT_LAT_CTAS 148      // single-pass launches with fewer CTAs than this use the latency shape
#endif
static bool use_latency_shape(int B, uint32_t batch) {
    if (B < 6 || B > 12) return false;
    const PassCfg d = single_cfg_t<false>(B);
    return ((uint64_t)batch + d.C - 1) / d.C < (uint64_t)NTT_LAT_CTAS;
}
// Multi-pass: first pass (gather, stage 0), middle passes, last pass (optionally scaled).
// `wide`: rows of the pass are >= 2^NTT_WIDE_STRIDE elements apart; a one-group CTA then
// reads 16-byte pieces of rows megabytes apart, so 8- and 9-stage passes take 4 adjacent
// groups per CTA (64-byte row segments; N = 2^26: 12.1 -> 10.3 ms, tools/exp_large.py).
// `tma`: the pass may take the TMA kernel (natural-layout input, no load-side factor);
// one-group CTAs (7-, 8-, 9-stage passes, not wide) then load their tile by tensor copy.
#ifndef NTT_TMA
#define NTT_TMA 1
#endif
template <int B, bool FIRST, bool SL, int RB>
static PassCfg tma_cfg() {
    if constexpr (FIRST) return make_cfg<B, 1, FIRST, SL, false, RB>();
    else return make_cfg<B, 1, FIRST, SL, false, RB, false, true>();
}
template <bool FIRST, bool SL>
static PassCfg multi_cfg_t(int B, bool wide, bool tma) {
    tma = tma && NTT_TMA && !FIRST;
    switch (B) {
        case 5: return make_cfg<5, NTT_C5, FIRST, SL>();
        case 6: return make_cfg<6, NTT_C6, FIRST, SL, false, NTT_RB6>();
        case 7: return (tma && NTT_C7 == 1) ? tma_cfg<7, FIRST, SL, NTT_RB7>()
                                            : make_cfg<7, NTT_C7, FIRST, SL, false, NTT_RB7>();
        case 8:
            if (wide) return make_cfg<8, 4, FIRST, SL, false, NTT_RB8>();
            return (tma && NTT_C8 == 1) ? tma_cfg<8, FIRST, SL, NTT_RB8>()
                                        : make_cfg<8, NTT_C8, FIRST, SL, false, NTT_RB8>();
        default:
            if (wide) return make_cfg<9, 4, FIRST, SL, false, NTT_RB9>();
            return (tma && NTT_C9 == 1) ? tma_cfg<9, FIRST, SL, NTT_RB9>()
                                        : make_cfg<9, NTT_C9, FIRST, SL, false, NTT_RB9>();
    }
}
// Permutation-free negacyclic passes (B in [5, 8], warp-owned groups).
template <int B, int C, bool INV, bool SL>
static PassCfg make_nc_cfg() {
    constexpr int RBM = B == 8 ? NTT_NC_RB8 : 3;
    using S = PassShape<B, RBM, C, true>;
    PassCfg c;
    c.fn = k_nc_pass<B, C, INV, SL, RBM>;
    c.B = B;
    c.C = C;
    c.threads = C * S::T;
    c.smem = ((size_t)C * S::GS + (size_t)C * S::TS) * sizeof(uint4);
    return c;
}
template <bool INV, bool SL>
static PassCfg nc_cfg_t(int B) {
    switch (B) {
        case 5: return make_nc_cfg<5, 8, INV, SL>();
        case 6: return make_nc_cfg<6, 8, INV, SL>();
        case 7: return make_nc_cfg<7, 8, INV, SL>();
        default: return make_nc_cfg<8, NTT_NC_C8, INV, SL>();
    }
}
static PassCfg nc_cfg(bool inv, bool scale_last, int B) {
    if (!inv) return nc_cfg_t<false, false>(B);
    return scale_last ? nc_cfg_t<true, true>(B) : nc_cfg_t<true, false>(B);
}
// pass widths of the permutation-free path: ceil(n / 8) passes, widths as equal as possible
static std::vector<int> nc_pass_bits(int n) {
    std::vector<int> b;
    if (n < 10) return b;
    const int np = (n + 7) / 8 < 2 ? 2 : (n + 7) / 8;
    for (int i = 0; i < np; i++) b.push_back(n / np + (i < n % np ? 1 : 0));
    return b;
}

// Four-step pass C reads the columns of a received matrix (element stride = the number of
// polynomials, polynomials adjacent in memory): groups of adjacent polynomials per CTA.
//  * single pass: C polynomials per CTA (lanes c = tid % C are adjacent residues); B = 9
//    (cfg 5's 2^9-point pass C) takes 4 instead of the contiguous-layout 1;
//  * multi-pass first pass with 9 stages (cfg 5's inverse pass C, 2^17 = 9 + 8): the
//    polynomial-major kernel (PM, 4 polynomials per CTA); other widths keep their shape.
#ifndef NTT_FS_C
#define NTT_FS_C 4
#endif
static PassCfg strided_single_cfg(int B, bool scale_last, uint32_t batch) {
    if (B == 9 && batch % NTT_FS_C == 0)
        return scale_last ? make_cfg<9, NTT_FS_C, true, true, true>() : make_cfg<9, NTT_FS_C, true, false, true>();
    return scale_last ? single_cfg_t<true>(B) : single_cfg_t<false>(B);
}
static bool strided_pm_first(int B, uint32_t batch) { return B == 9 && batch % NTT_FS_C == 0; }
static PassCfg strided_pm_cfg() { return make_cfg<9, NTT_FS_C, true, false, false, NTT_RB9, true>(); }


#ifndef NTT_WIDE_STRIDE
#define NTT_WIDE_STRIDE 17
#endif
// lo = index bits below the pass (0 for the first pass); n = log2 N
static PassCfg pass_cfg(size_t npass, size_t i, int B, bool scale_last, int lo = 0, int n = 0, bool tma = true) {
    if (npass == 1) return scale_last ? single_cfg_t<true>(B) : single_cfg_t<false>(B);
    const bool wide = (i == 0 ? n - B : lo) >= NTT_WIDE_STRIDE;   // row stride of the pass, log2 elements
    if (i == 0) return multi_cfg_t<true, false>(B, wide, tma);
    if (i + 1 == npass && scale_last) return multi_cfg_t<false, true>(B, wide, tma);
    return multi_cfg_t<false, false>(B, wide, tma);
}

// Tensor map of a TMA pass's data tiles over a.src ([batch][N] residues, natural layout),
// encoded per launch (the map holds the buffer's address) through the driver's
// cuTensorMapEncodeTiled, reached via the runtime's entry-point query (no libcuda link).
static PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return (PFN_cuTensorMapEncodeTiled_v12000)f;
    }();
    return fn;
}
static bool tma_encode(PassArgs& a, bool first, int n, int B, int lo, uint32_t batch) {
    const PFN_cuTensorMapEncodeTiled_v12000 enc = tma_encoder();
    if (!enc) return false;
    const cuuint64_t N = 1ull << n;
    void* base = const_cast<uint4*>(a.src);
    CUresult r;
    if (first) {
        // [poly][r (2^B rows, as r_lo < 256 and r_hi)][g][2 u64]: box = column g, 128B swizzle
        const int gb = n - B;
        const cuuint32_t rl = B > 8 ? 256u : (1u << B), rh = (1u << B) / rl;
        const cuuint64_t dims[4] = {2ull << gb, rl, rh, batch};
        const cuuint64_t strides[3] = {16ull << gb, (16ull << gb) * rl, 16 * N};
        const cuuint32_t box[4] = {2, rl, rh, 1}, es[4] = {1, 1, 1, 1};
        r = enc(&a.tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        // [poly][H][m][j][L][2 u64], r = 8 m + j: box {2, 9 (j from -1), 2^B / 8, 1, 1}
        const cuuint64_t dims[5] = {2ull << lo, 8, 1ull << (B - 3), 1ull << (n - lo - B), batch};
        const cuuint64_t strides[4] = {16ull << lo, 16ull << (lo + 3), 16ull << (lo + B), 16 * N};
        const cuuint32_t box[5] = {2, 9, 1u << (B - 3), 1, 1}, es[5] = {1, 1, 1, 1, 1};
        r = enc(&a.tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    return r == CUDA_SUCCESS;
}

// ----------------------------------------------------------------------------- plan
struct ntt128_plan_s {
    uint32_t log2n, batch, nq, flags, kind;  // kind: 0 cyclic, 1 negacyclic
    int device;
    uint64_t N;
    std::vector<int> bits;                    // bits per pass, first pass first
    ModC* d_mods = nullptr;
    uint4* d_tw_fwd = nullptr;                // [nq][N/2]  omega^i
    uint4* d_tw_inv = nullptr;                // [nq][N/2]  omega^-i
    uint4* d_tw_inv_last = nullptr;           // [nq][N/2]  omega^-i N^-1          (cyclic)
    uint4* d_tw_inv_last_r = nullptr;         // [nq][N/2]  omega^-i N^-1 R        (cyclic polymul)
    uint4* d_f_twist = nullptr;               // [nq][N]    psi^j                  (negacyclic)
    uint4* d_f_untwist = nullptr;             // [nq][N]    N^-1 psi^-j            (negacyclic)
    uint4* d_f_untwist_r = nullptr;           // [nq][N]    N^-1 psi^-j R          (negacyclic polymul)
    std::vector<u128> q_host;
    std::vector<uint4*> d_pt_fwd, d_pt_inv, d_pt_inv_r;  // per pass, [nq][pt_stride]
    // pseudo-Mersenne class (psm128.cuh): every modulus is 2^b - c with c 2^(128-b) < 2^32 and the
    // plan is cyclic with >= 2 passes -- plain-residue copies of d_pt_fwd / d_pt_inv for the
    // plain forward / inverse calls (polymul, four-step I/O and negacyclic calls keep Montgomery)
    bool psm = false;
    std::vector<uint4*> d_pt_fwd_psm, d_pt_inv_psm;
    // permutation-free negacyclic path (n >= 10): pass widths bottom-up, per-pass tables
    // [nq][2^(n - lo - B)][2^B - 1] (psi, psi^-1; the top inverse pass N^-1 / N^-1 R scaled)
    std::vector<int> nc_bits;
    std::vector<uint4*> d_nc_fwd, d_nc_inv, d_nc_inv_r;
    std::vector<uint64_t> nc_stride;
    // multi-pass launches carry their moduli as kernel parameters (QPar, <= NTT_QMAX per launch):
    std::vector<QPar> qpar;                              // [nq] host copy of the per-modulus constants
    std::vector<uint32_t> order;                         // [batch] polynomials grouped by class (nq == batch)
    std::vector<uint64_t> pt_stride;
    // Pass-overlap completion counters, one set per stream (keyed by cudaStreamGetId):
    // counters only grow; the host keeps, per counter row, the value the row reaches once
    // every pass enqueued so far on the stream has signalled (a pass adds its CTAs per
    // polynomial), so in-stream order makes the targets exact without a reset, for any mix
    // of pass structures, and different streams never share a set.
    static constexpr int MAX_ROWS = 4;                 // passes of the deepest schedule (the last row: chained calls)
    // At most MAX_STREAMS entries are cached: a further stream evicts the least recently used
    // entry once the event recorded after that entry's last use has completed (entries used
    // under stream capture are pinned: a captured graph keeps referring to them).
    static constexpr int MAX_STREAMS = 8;
    struct StreamCtr {
        uint32_t* d = nullptr;                          // [MAX_ROWS][batch]
        uint32_t expected[MAX_ROWS] = {0, 0, 0, 0};
        // NTT128_FLAG_CHAIN: the last counter-signalling call of this plan on the stream --
        // its last pass's row and target, its buffers, and its library generation
        int last_row = -1;
        uint32_t last_target = 0;
        const void* last_bufs[3] = {nullptr, nullptr, nullptr};
        uint64_t gen = 0;
        uint4* scratch = nullptr;                       // polymul spectra [2][batch][N] / in-place copy [batch][N]
        size_t scratch_elems = 0;
        cudaEvent_t ev = nullptr;                       // recorded after the last enqueue that used the entry
        uint64_t tick = 0;                              // LRU clock
        bool pinned = false;
    };
    std::mutex mu;
    std::unordered_map<unsigned long long, StreamCtr> ctrs;
    uint64_t tick = 0;
};

static void plan_free(ntt128_plan_s* p) {
    if (!p) return;
    if (p->flags & NTT128_FLAG_CHAIN) g_chain_plans--;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(p->device);
    cudaFree(p->d_mods);
    cudaFree(p->d_tw_fwd);
    cudaFree(p->d_tw_inv);
    cudaFree(p->d_tw_inv_last);
    cudaFree(p->d_tw_inv_last_r);
    cudaFree(p->d_f_twist);
    cudaFree(p->d_f_untwist);
    cudaFree(p->d_f_untwist_r);
    for (auto& kv : p->ctrs) {
        cudaFree(kv.second.d);
        cudaFree(kv.second.scratch);
        if (kv.second.ev) cudaEventDestroy(kv.second.ev);
    }
    for (size_t i = 0; i < p->d_nc_fwd.size(); i++) {
        if (p->d_nc_inv_r[i] != p->d_nc_inv[i]) cudaFree(p->d_nc_inv_r[i]);
        cudaFree(p->d_nc_fwd[i]);
        cudaFree(p->d_nc_inv[i]);
    }
    for (uint4* t : p->d_pt_fwd_psm) cudaFree(t);
    for (uint4* t : p->d_pt_inv_psm) cudaFree(t);
    for (size_t i = 0; i < p->d_pt_fwd.size(); i++) {
        if (p->d_pt_inv_r[i] != p->d_pt_inv[i]) cudaFree(p->d_pt_inv_r[i]);
        cudaFree(p->d_pt_fwd[i]);
        cudaFree(p->d_pt_inv[i]);
    }
    cudaSetDevice(prev);
    delete p;
}

#ifndef NTT_SINGLE_MAX
#ifndef NTT_SINGLE_MAX
#define NTT_SINGLE_MAX 11   // largest log2 N done in one pass (measured: 2^12 is 25% faster as 6+6 passes)
#endif
#endif
// Two-pass splits measured over every (a, b) with 5 <= a, b <= 9 (tools/gpu_splits.sh,
// 1 GiB batches): 7-stage passes are the weak shape, so N = 2^13 runs 5 + 8 (+2.7 % over
// 6 + 7), 2^14 6 + 8 (+7 % over 7 + 7), 2^15 9 + 6 (+4.3 % over 7 + 8); 2^16 8 + 8 (9 + 7
// equal), 2^17 9 + 8 (3 % over 8 + 9), 2^18 9 + 9.  Three passes (tools/gpu_splits3.sh):
// 2^19 5+6+8 (+2 % over 7+6+6), 2^20 6+6+8 (+5.6 %), 2^21 9+6+6 (+7.5 %), 2^22 6+8+8 (+15 %
// over 8+7+7), 2^23 9+6+8 (+4.3 %); 2^24..2^26 widest first (8+8+8, 9+8+8, 9+9+8).
static std::vector<int> pass_bits(int n) {
#if NTT128_EXPERIMENTS
    if (const char* e = getenv("NTT128_SPLIT")) {   // experiment switch: "a,b[,c]" pass widths summing to n
        std::vector<int> v;
        int sum = 0;
        for (const char* c = e; *c;) {
            const int b = atoi(c);
            if (b < 5 || b > 9) { v.clear(); break; }
            v.push_back(b);
            sum += b;
            while (*c && *c != ',') c++;
            if (*c == ',') c++;
        }
        if (sum == n && v.size() > 1 && v.size() <= 4) return v;
    }
#endif
    if (n <= NTT_SINGLE_MAX) return {n};
    switch (n) {
        case 13: return {5, 8};
        case 14: return {6, 8};
        case 15: return {9, 6};
        case 19: return {5, 6, 8};
        case 20: return {6, 6, 8};
        case 21: return {9, 6, 6};
        case 22: return {6, 8, 8};
        case 23: return {9, 6, 8};
        default: break;
    }
    if (n <= 18) return {(n + 1) / 2, n / 2};
    int a = (n + 2) / 3, b = (n + 1) / 3, c = n / 3;
    return {a, b, c};
}

static inline uint4 to_uint4(u128 v) {
    uint32_t w[4];
    to_words(v, w);
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// Build one power table on the device: out[m][i] = scale_m * base_m^i, i < count.
static cudaError_t gen_table(uint4* out, uint64_t stride, uint64_t count, const std::vector<ntt128h::Mont>& mont,
                             const std::vector<u128>& base, const std::vector<u128>& scale, const ModC* d_mods) {
    const int nq = (int)mont.size();
    const int K = 40;
    std::vector<uint4> pow2((size_t)nq * K), sc(nq);
    for (int m = 0; m < nq; m++) {
        u128 b = mont[m].to_m(base[m]);
        for (int k = 0; k < K; k++) {
            pow2[(size_t)m * K + k] = to_uint4(b);
            b = mont[m].mul(b, b);
        }
        sc[m] = to_uint4(mont[m].to_m(scale[m]));
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
        k_gen_pow_table<<<dim3(gx, nq), 256>>>(out, stride, count, d_pow2, K, d_sc, d_mods);
        ntt128_count_launch(1);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
    }
    cudaFree(d_pow2);
    cudaFree(d_sc);
    return e;
}

// q = 2^b - c with c 2^(128-b) < 2^32 (psm128.cuh): words 1..3 of q 2^(128-b) are all ones.
static bool psm_eligible(u128 q) {
    int s = 0;
    while (((q << s) >> 127) == 0) s++;
    const u128 Q = q << s;
    return (Q >> 32) == (((u128)1 << 96) - 1) && (uint32_t)Q != 1u;   // C = 2^32 - 1 excluded (psm_mul's l4 + 1)
}

extern "C" ntt128_status ntt128_plan_create(ntt128_plan_t* out, uint32_t log2n, uint32_t batch, const uint64_t* q_host,
                                            const uint64_t* root_host, uint32_t n_moduli, uint32_t flags, int device) {
    if (!out || !q_host || !root_host) return NTT128_ERR_INVALID_ARG;
    *out = nullptr;
    if (log2n < 1 || log2n > 26 || batch == 0) return NTT128_ERR_INVALID_ARG;
    if (n_moduli != 1 && n_moduli != batch) return NTT128_ERR_INVALID_ARG;
    if (flags & ~(NTT128_NEGACYCLIC | NTT128_FLAG_CHECK_INPUT | NTT128_FLAG_CHAIN)) return NTT128_ERR_INVALID_ARG;
    const uint32_t kind = flags & NTT128_NEGACYCLIC;
    const uint64_t N = 1ull << log2n;

    // ---- validate every modulus and root on the host
    std::vector<ntt128h::Mont> mont;
    std::vector<u128> qs, roots;
    mont.reserve(n_moduli);
    for (uint32_t m = 0; m < n_moduli; m++) {
        u128 q = ntt128h::make(q_host[2 * m], q_host[2 * m + 1]);
        u128 r = ntt128h::make(root_host[2 * m], root_host[2 * m + 1]);
        if ((q & 1) == 0 || q < 3) return NTT128_ERR_MODULUS;
        if (!ntt128h::is_probable_prime(q)) return NTT128_ERR_NOT_PRIME;
        const u128 order = kind ? (u128)2 * N : (u128)N;
        if ((q - 1) % order != 0) return NTT128_ERR_NO_ROOT;
        if (r >= q) return NTT128_ERR_BAD_ROOT;
        mont.emplace_back(q);
        const ntt128h::Mont& M = mont.back();
        // exact order `order` (a power of two): r^order == 1 and r^(order/2) == q-1
        if (M.pow(r, order / 2) != q - 1) return NTT128_ERR_BAD_ROOT;
        qs.push_back(q);
        roots.push_back(r);
    }

    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(device) != cudaSuccess) return NTT128_ERR_INVALID_ARG;
    ntt128_plan_s* p = new (std::nothrow) ntt128_plan_s();
    if (!p) { cudaSetDevice(prev); return NTT128_ERR_OOM; }
    p->log2n = log2n;
    p->batch = batch;
    p->nq = n_moduli;
    p->flags = flags;
    if (flags & NTT128_FLAG_CHAIN) g_chain_plans++;   // plan_free undoes it
    p->kind = kind;
    p->device = device;
    p->N = N;
    p->bits = pass_bits((int)log2n);
    p->q_host = qs;

    // ---- per-modulus constants
    std::vector<ModC> mc(n_moduli);
    std::vector<u128> omega(n_moduli), omega_inv(n_moduli), ones(n_moduli), ninv(n_moduli), ninv_r(n_moduli);
    std::vector<u128> psi(n_moduli), psi_inv(n_moduli);
    for (uint32_t m = 0; m < n_moduli; m++) {
        const ntt128h::Mont& M = mont[m];
        const u128 q = qs[m];
        ModC& c = mc[m];
        memset(&c, 0, sizeof(c));
        to_words(q, c.q);
        c.qinv0 = (uint32_t)M.qp;
        to_words(M.r1, c.one_m);
        to_words(M.r2, c.r2);
        const u128 ni = M.inv((u128)(N % q));
        to_words(M.to_m(ni), c.ninv_m);
        to_words(M.to_m(M.mulmod(ni, M.r1)), c.ninv_rm);
        ones[m] = 1;
        ninv[m] = ni;
        ninv_r[m] = M.mulmod(ni, M.r1);
        if (kind) {
            psi[m] = roots[m];
            psi_inv[m] = M.inv(roots[m]);
            omega[m] = M.mulmod(roots[m], roots[m]);
        } else {
            omega[m] = roots[m];
        }
        omega_inv[m] = M.inv(omega[m]);
    }

    ntt128_status st = NTT128_OK;
    const uint64_t half = N / 2;
    auto alloc = [&](uint4** ptr, uint64_t per) -> bool {
        if (cudaMalloc(ptr, (size_t)per * n_moduli * sizeof(uint4)) != cudaSuccess) { st = NTT128_ERR_OOM; return false; }
        return true;
    };
    if (cudaMalloc(&p->d_mods, n_moduli * sizeof(ModC)) != cudaSuccess) st = NTT128_ERR_OOM;
    if (st == NTT128_OK && cudaMemcpy(p->d_mods, mc.data(), n_moduli * sizeof(ModC), cudaMemcpyHostToDevice) != cudaSuccess)
        st = NTT128_ERR_CUDA;
    std::vector<u128> scale_ninv(ninv), scale_ninv_r(ninv_r);
    if (st == NTT128_OK && alloc(&p->d_tw_fwd, half) && alloc(&p->d_tw_inv, half)) {
        if (gen_table(p->d_tw_fwd, half, half, mont, omega, ones, p->d_mods) != cudaSuccess ||
            gen_table(p->d_tw_inv, half, half, mont, omega_inv, ones, p->d_mods) != cudaSuccess)
            st = NTT128_ERR_CUDA;
    }
    if (st == NTT128_OK && !kind && alloc(&p->d_tw_inv_last, half) && alloc(&p->d_tw_inv_last_r, half)) {
        if (gen_table(p->d_tw_inv_last, half, half, mont, omega_inv, scale_ninv, p->d_mods) != cudaSuccess ||
            gen_table(p->d_tw_inv_last_r, half, half, mont, omega_inv, scale_ninv_r, p->d_mods) != cudaSuccess)
            st = NTT128_ERR_CUDA;
    }
    if (st == NTT128_OK && kind && alloc(&p->d_f_twist, N) && alloc(&p->d_f_untwist, N) && alloc(&p->d_f_untwist_r, N)) {
        if (gen_table(p->d_f_twist, N, N, mont, psi, ones, p->d_mods) != cudaSuccess ||
            gen_table(p->d_f_untwist, N, N, mont, psi_inv, scale_ninv, p->d_mods) != cudaSuccess ||
            gen_table(p->d_f_untwist_r, N, N, mont, psi_inv, scale_ninv_r, p->d_mods) != cudaSuccess)
            st = NTT128_ERR_CUDA;
    }
    // opt in to > 48 KB dynamic shared memory for every pass kernel this plan uses
    if (st == NTT128_OK) {
        for (size_t i = 0; i < p->bits.size(); i++) {
            for (int sl = 0; sl < 2; sl++) {
                int lo_i = 0;
                for (size_t k = 0; k < i; k++) lo_i += p->bits[k];
                for (int tma = 0; tma < 2; tma++) {   // the TMA kernel and its cp.async fallback
                    const PassCfg ct = pass_cfg(p->bits.size(), i, p->bits[i], sl == 1, lo_i, (int)log2n, tma == 1);
                    if (cudaFuncSetAttribute(ct.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ct.smem) != cudaSuccess)
                        st = NTT128_ERR_CUDA;
                    if (NTT_CARVEOUT >= 0)   // experiment: shared-memory carveout of the pass kernels
                        cudaFuncSetAttribute(ct.fn, cudaFuncAttributePreferredSharedMemoryCarveout, NTT_CARVEOUT);
                }
                PassCfg c;
                if (p->bits.size() == 1 && use_latency_shape(p->bits[i], batch)) {
                    c = sl ? single_lat_cfg_t<true>(p->bits[i]) : single_lat_cfg_t<false>(p->bits[i]);
                    if (cudaFuncSetAttribute(c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem) != cudaSuccess)
                        st = NTT128_ERR_CUDA;
                }
            }
        }
    }
    // polynomial order for multi-pass launches, grouped by arithmetic mode (q < 2^126,
    // q < 2^127, the rest) so one code path at a time is hot in the instruction cache
    if (st == NTT128_OK && n_moduli > 1) {
        for (int cls = 0; cls < 3; cls++)
            for (uint32_t m = 0; m < n_moduli; m++) {
                const int c = (qs[m] >> 126) == 0 ? 0 : ((qs[m] >> 127) == 0 ? 1 : 2);
                if (c == cls) p->order.push_back(m);
            }
    }
    if (st == NTT128_OK) {
        p->qpar.resize(n_moduli);
        for (uint32_t m = 0; m < n_moduli; m++) {
            QPar& d = p->qpar[m];
            memset(&d, 0, sizeof(d));
            for (int i = 0; i < 4; i++) {
                d.q[i] = mc[m].q[i];
                d.ninv_m[i] = mc[m].ninv_m[i];
                d.ninv_rm[i] = mc[m].ninv_rm[i];
            }
            d.qinv0 = mc[m].qinv0;
        }
    }
    // per-pass twiddle tables in consumption order (gathered from the power tables)
    if (st == NTT128_OK) {
        int lo = 0;
        const size_t np = p->bits.size();
        for (size_t i = 0; i < np && st == NTT128_OK; i++) {
            const int b = p->bits[i];
            const uint64_t stride = ((uint64_t)1 << lo) * (((uint64_t)1 << b) - 1);
            p->pt_stride.push_back(stride);
            const bool last = i + 1 == np;
            uint4 *f = nullptr, *v = nullptr, *vr = nullptr;
            const size_t bytes = (size_t)stride * n_moduli * sizeof(uint4);
            if (cudaMalloc(&f, bytes) != cudaSuccess || cudaMalloc(&v, bytes) != cudaSuccess) st = NTT128_ERR_OOM;
            if (st == NTT128_OK && last && !kind && cudaMalloc(&vr, bytes) != cudaSuccess) st = NTT128_ERR_OOM;
            if (!vr) vr = v;
            p->d_pt_fwd.push_back(f);
            p->d_pt_inv.push_back(v);
            p->d_pt_inv_r.push_back(vr);
            if (st != NTT128_OK) break;
            unsigned gx = (unsigned)((stride + 255) / 256);
            if (gx > 4096) gx = 4096;
            const dim3 grid(gx, n_moduli);
            k_gather_pass_tw<<<grid, 256>>>(f, stride, p->d_tw_fwd, nullptr, half, log2n, lo, b);
            k_gather_pass_tw<<<grid, 256>>>(v, stride, p->d_tw_inv, (last && !kind) ? p->d_tw_inv_last : nullptr, half,
                                            log2n, lo, b);
            if (vr != v) k_gather_pass_tw<<<grid, 256>>>(vr, stride, p->d_tw_inv, p->d_tw_inv_last_r, half, log2n, lo, b);
            ntt128_count_launch(vr != v ? 3 : 2);
            if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) st = NTT128_ERR_CUDA;
            lo += b;
        }
        // pseudo-Mersenne class: plain-residue copies of the forward / inverse pass tables
        p->psm = NTT_PSM && NTT_SHIFT_SCALE && !NTT_FORCE_FULL && !kind && log2n >= 2;
        for (uint32_t m = 0; m < n_moduli && p->psm; m++) p->psm = psm_eligible(qs[m]);
        for (size_t i = 0; i < np && st == NTT128_OK && p->psm; i++) {
            const uint64_t stride = p->pt_stride[i];
            const size_t bytes = (size_t)stride * n_moduli * sizeof(uint4);
            uint4 *f = nullptr, *v = nullptr;
            if (cudaMalloc(&f, bytes) != cudaSuccess || cudaMalloc(&v, bytes) != cudaSuccess) st = NTT128_ERR_OOM;
            p->d_pt_fwd_psm.push_back(f);
            p->d_pt_inv_psm.push_back(v);
            if (st != NTT128_OK) break;
            unsigned gx = (unsigned)((stride + 255) / 256);
            if (gx > 4096) gx = 4096;
            const dim3 grid(gx, n_moduli);
            k_table_to_plain<<<grid, 256>>>(f, p->d_pt_fwd[i], stride, p->d_mods);
            k_table_to_plain<<<grid, 256>>>(v, p->d_pt_inv[i], stride, p->d_mods);
            ntt128_count_launch(2);
            if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) st = NTT128_ERR_CUDA;
        }
        // permutation-free negacyclic tables (ntt128_forward_bitrev / inverse_bitrev, polymul)
        if (st == NTT128_OK && kind) {
            p->nc_bits = nc_pass_bits((int)log2n);
            std::vector<uint4> sc(n_moduli), scr(n_moduli);
            for (uint32_t m = 0; m < n_moduli; m++) {
                sc[m] = make_uint4(mc[m].ninv_m[0], mc[m].ninv_m[1], mc[m].ninv_m[2], mc[m].ninv_m[3]);
                scr[m] = make_uint4(mc[m].ninv_rm[0], mc[m].ninv_rm[1], mc[m].ninv_rm[2], mc[m].ninv_rm[3]);
            }
            uint4 *d_sc = nullptr, *d_scr = nullptr;
            if (!p->nc_bits.empty()) {
                if (cudaMalloc(&d_sc, n_moduli * sizeof(uint4)) != cudaSuccess ||
                    cudaMalloc(&d_scr, n_moduli * sizeof(uint4)) != cudaSuccess) st = NTT128_ERR_OOM;
                if (st == NTT128_OK && (cudaMemcpy(d_sc, sc.data(), n_moduli * sizeof(uint4), cudaMemcpyHostToDevice) != cudaSuccess ||
                                        cudaMemcpy(d_scr, scr.data(), n_moduli * sizeof(uint4), cudaMemcpyHostToDevice) != cudaSuccess))
                    st = NTT128_ERR_CUDA;
            }
            int nlo = 0;
            const size_t nnp = p->nc_bits.size();
            for (size_t i = 0; i < nnp && st == NTT128_OK; i++) {
                const int b = p->nc_bits[i];
                const uint64_t stride = ((uint64_t)1 << (log2n - nlo - b)) * (((uint64_t)1 << b) - 1);
                p->nc_stride.push_back(stride);
                const bool top = i + 1 == nnp;
                uint4 *f = nullptr, *v = nullptr, *vr = nullptr;
                const size_t bytes = (size_t)stride * n_moduli * sizeof(uint4);
                if (cudaMalloc(&f, bytes) != cudaSuccess || cudaMalloc(&v, bytes) != cudaSuccess) st = NTT128_ERR_OOM;
                if (st == NTT128_OK && top && cudaMalloc(&vr, bytes) != cudaSuccess) st = NTT128_ERR_OOM;
                if (!vr) vr = v;
                p->d_nc_fwd.push_back(f);
                p->d_nc_inv.push_back(v);
                p->d_nc_inv_r.push_back(vr);
                if (st != NTT128_OK) break;
                unsigned gx = (unsigned)((stride + 255) / 256);
                if (gx > 4096) gx = 4096;
                const dim3 grid(gx, n_moduli);
                k_gather_nc_tw<<<grid, 256>>>(f, stride, p->d_f_twist, log2n, nlo, b, 0, nullptr, p->d_mods);
                k_gather_nc_tw<<<grid, 256>>>(v, stride, p->d_f_twist, log2n, nlo, b, 1, top ? d_sc : nullptr, p->d_mods);
                if (vr != v) k_gather_nc_tw<<<grid, 256>>>(vr, stride, p->d_f_twist, log2n, nlo, b, 1, d_scr, p->d_mods);
                ntt128_count_launch(vr != v ? 3 : 2);
                if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) st = NTT128_ERR_CUDA;
                for (int iv = 0; iv < 2 && st == NTT128_OK; iv++)
                    for (int sl = 0; sl < 2; sl++) {
                        PassCfg c = nc_cfg(iv == 1, sl == 1, b);
                        if (cudaFuncSetAttribute(c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem) != cudaSuccess)
                            st = NTT128_ERR_CUDA;
                    }
                nlo += b;
            }
            cudaFree(d_sc);
            cudaFree(d_scr);
        }
        // the power tables are only the source of the pass tables
        cudaFree(p->d_tw_fwd); p->d_tw_fwd = nullptr;
        cudaFree(p->d_tw_inv); p->d_tw_inv = nullptr;
        cudaFree(p->d_tw_inv_last); p->d_tw_inv_last = nullptr;
        cudaFree(p->d_tw_inv_last_r); p->d_tw_inv_last_r = nullptr;
    }
    cudaSetDevice(prev);
    if (st != NTT128_OK) {
        plan_free(p);
        return st;
    }
    *out = p;
    return NTT128_OK;
}

extern "C" void ntt128_plan_destroy(ntt128_plan_t plan) { plan_free(plan); }

extern "C" ntt128_status ntt128_plan_info(const ntt128_plan_t p, uint32_t* log2n, uint32_t* batch, uint32_t* n_moduli,
                                          uint32_t* flags, uint32_t* num_passes) {
    if (!p) return NTT128_ERR_INVALID_ARG;
    if (log2n) *log2n = p->log2n;
    if (batch) *batch = p->batch;
    if (n_moduli) *n_moduli = p->nq;
    if (flags) *flags = p->flags;
    if (num_passes) *num_passes = (uint32_t)p->bits.size();
    return NTT128_OK;
}

extern "C" ntt128_status ntt128_plan_arith_class(const ntt128_plan_t p, uint32_t* cls) {
    if (!p || !cls) return NTT128_ERR_INVALID_ARG;
    *cls = p->psm ? NTT128_CLASS_PSEUDO_MERSENNE : NTT128_CLASS_MONTGOMERY;
    return NTT128_OK;
}

// ----------------------------------------------------------------------------- execution
struct RunOpts {
    bool inverse;
    const uint4* pmul;     // fused point-wise product (polymul inverse)
    bool polymul;          // use the R-compensated inverse tables
    const Ntt128IO* io = nullptr;   // four-step input / output layouts (fourstep.cu)
    // NTT128_FLAG_CHAIN: the stream's library generation before this API call and the one
    // it took (ntt128_stream_gen); 0 when unknown (stream capture)
    uint64_t gen_prev = 0, gen_new = 0;
};

static ntt128_status check_range(const ntt128_plan_s* p, const uint4* src, cudaStream_t stream);

// Experiment switches (A/B measurements in DESIGN.md).  The product library is built
// without NTT128_EXPERIMENTS and its behaviour does not depend on the environment; an
// experiment build (-DNTT128_EXPERIMENTS=1, a separate .so) reads, once per process,
// NTT128_NO_PDL (no pass overlap), NTT128_PDL_NOCNT (whole-grid programmatic dependencies
// only), NTT128_NO_NC (polymul through the natural-order path), NTT128_NO_CLUSTER.
struct Switches {
    bool no_pdl = false, pdl_nocnt = false, no_nc = false, no_cluster = false, no_tiles = false;
    Switches() {
#if NTT128_EXPERIMENTS
        no_tiles = getenv("NTT128_NO_TILES") != nullptr;
        no_pdl = getenv("NTT128_NO_PDL") != nullptr;
        pdl_nocnt = getenv("NTT128_PDL_NOCNT") != nullptr;
        no_nc = getenv("NTT128_NO_NC") != nullptr;
        no_cluster = getenv("NTT128_NO_CLUSTER") != nullptr;
#endif
    }
};
static const Switches& switches() {
    static const Switches s;
    return s;
}

static bool overlap_allowed(size_t npass, cudaStream_t stream, bool* ok) {
    *ok = npass > 1 && !switches().no_pdl;
    if (*ok) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess) return false;
        if (cs != cudaStreamCaptureStatusNone) *ok = false;
    }
    return true;
}
static cudaError_t launch_pass(const PassCfg& c, const PassArgs& a, uint64_t ctas, cudaStream_t stream, bool pdl) {
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3((unsigned)ctas);
    cfg.blockDim = dim3((unsigned)c.threads);
    cfg.dynamicSmemBytes = c.smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, c.fn, a);
}

// Launch one pass with its moduli as kernel parameters (QPar table).  Multi-pass
// kernels of an RNS plan with more than NTT_QMAX polynomials run as chunks of NTT_QMAX
// polynomials, each a launch over its own slice of every per-polynomial array (data,
// point-wise operand, completion counters) and per-modulus table (pass twiddles, factors,
// device constants).  TMA passes encode the chunk's tensor map; `alt` is the same pass
// without TMA, taken if the encode fails.
static ntt128_status launch_pass_q(const ntt128_plan_s* p, const PassCfg& c, const PassCfg& alt, const PassArgs& a0,
                                   int B, int lo, cudaStream_t stream, bool pdl) {
    const int n = (int)a0.n;
    const uint32_t nq = p->nq, batch = p->batch;
    const bool chunked = !c.single && nq > 1 && batch > NTT_QMAX;
    const uint32_t step = chunked ? NTT_QMAX : batch;
    for (uint32_t b0 = 0; b0 < batch; b0 += step) {
        const uint32_t nb = batch - b0 < step ? batch - b0 : step;
        PassArgs a = a0;
        if (nq == 1) {
            a.qp[0] = p->qpar[0];
        } else if (!c.single) {
            a.nq = nb;
            for (uint32_t i = 0; i < nb; i++) a.qp[i] = p->qpar[b0 + i];
            uint32_t k = 0;
            for (uint32_t m : p->order)
                if (m >= b0 && m < b0 + nb) a.ord[k++] = (uint16_t)(m - b0);
        }
        if (b0) {   // chunked (nq == batch, natural layout: no four-step I/O)
            a.src += (uint64_t)b0 * p->N;
            a.dst += (uint64_t)b0 * p->N;
            if (a.pmul) a.pmul += (uint64_t)b0 * p->N;
            a.pt += (uint64_t)b0 * a.pt_stride;
            a.mods += b0;
            if (a.fin) a.fin += (uint64_t)b0 * a.f_stride;
            if (a.fout) a.fout += (uint64_t)b0 * a.f_stride;
            if (a.cnt_in) a.cnt_in += b0;
            if (a.cnt_out) a.cnt_out += b0;
        }
        if (chunked) a.total_groups = (uint64_t)nb << (n - B);
        const PassCfg* cc = &c;
        if (c.tma && !tma_encode(a, c.first, n, B, lo, chunked ? nb : batch)) cc = &alt;   // per-thread cp.async tiles
        const uint64_t per_cta = (uint64_t)cc->C * cc->tiles;
        const uint64_t ctas = (a.total_groups + per_cta - 1) / per_cta;
        if (launch_pass(*cc, a, ctas, stream, pdl) != cudaSuccess) return NTT128_ERR_CUDA;
        ntt128_count_launch(1);
    }
    return NTT128_OK;
}

// The stream's cache entry (created on first use; `lk` must hold p->mu).  Creating an entry
// beyond MAX_STREAMS evicts the least recently used unpinned one after its last recorded
// use has completed on the device.
static ntt128_plan_s::StreamCtr* stream_entry(ntt128_plan_s* p, unsigned long long sid) {
    auto it = p->ctrs.find(sid);
    if (it == p->ctrs.end()) {
        if (p->ctrs.size() >= (size_t)ntt128_plan_s::MAX_STREAMS) {
            auto victim = p->ctrs.end();
            for (auto jt = p->ctrs.begin(); jt != p->ctrs.end(); ++jt)
                if (!jt->second.pinned && (victim == p->ctrs.end() || jt->second.tick < victim->second.tick)) victim = jt;
            if (victim != p->ctrs.end()) {
                if (victim->second.ev) {
                    cudaEventSynchronize(victim->second.ev);
                    cudaEventDestroy(victim->second.ev);
                }
                cudaFree(victim->second.d);
                cudaFree(victim->second.scratch);
                p->ctrs.erase(victim);
            }
        }
        it = p->ctrs.emplace(sid, ntt128_plan_s::StreamCtr()).first;
    }
    it->second.tick = ++p->tick;
    return &it->second;
}
static bool is_capturing(cudaStream_t stream) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess) return false;
    return cs != cudaStreamCaptureStatusNone;
}
// Record the end of this call's use of the stream's entry.  Under stream capture nothing of
// the cache is used (cudaStreamGetId would invalidate the capture; counters are bypassed and
// scratch comes from graph-owned stream-ordered allocations), so there is nothing to record.
static void stream_touch(ntt128_plan_s* p, cudaStream_t stream) {
    if (is_capturing(stream)) return;
    unsigned long long sid = 0;
    if (cudaStreamGetId(stream, &sid) != cudaSuccess) return;
    std::lock_guard<std::mutex> lk(p->mu);
    auto it = p->ctrs.find(sid);
    if (it == p->ctrs.end()) return;
    if (!it->second.ev && cudaEventCreateWithFlags(&it->second.ev, cudaEventDisableTiming) != cudaSuccess) {
        it->second.ev = nullptr;
        it->second.pinned = true;   // cannot prove it idle: never evict
        return;
    }
    cudaEventRecord(it->second.ev, stream);
}
// The stream's counter set (allocated and zeroed in stream order on first use); `lk` is
// locked and stays locked until the caller has enqueued every pass.
static ntt128_status stream_counters(ntt128_plan_s* p, cudaStream_t stream, std::unique_lock<std::mutex>& lk,
                                     ntt128_plan_s::StreamCtr** out) {
    unsigned long long sid = 0;
    if (cudaStreamGetId(stream, &sid) != cudaSuccess) return NTT128_ERR_CUDA;
    lk.lock();
    ntt128_plan_s::StreamCtr& c = *stream_entry(p, sid);
    if (!c.d) {
        const size_t bytes = (size_t)ntt128_plan_s::MAX_ROWS * p->batch * sizeof(uint32_t);
        if (cudaMalloc(&c.d, bytes) != cudaSuccess) { c.d = nullptr; return NTT128_ERR_OOM; }
        if (cudaMemsetAsync(c.d, 0, bytes, stream) != cudaSuccess) return NTT128_ERR_CUDA;
        memset(c.expected, 0, sizeof(c.expected));
    }
    *out = &c;
    return NTT128_OK;
}
// The stream's scratch of at least `elems` residues (polymul spectra 2 x batch x N, the
// in-place copy batch x N), kept with the entry: no per-call stream-ordered allocation (a
// memory pool trimmed at a synchronisation would re-grow inside the next call).  Work on
// one stream is ordered, so consecutive calls may reuse it.
static ntt128_status stream_scratch(ntt128_plan_s* p, cudaStream_t stream, size_t elems, uint4** out) {
    unsigned long long sid = 0;
    if (cudaStreamGetId(stream, &sid) != cudaSuccess) return NTT128_ERR_CUDA;
    std::lock_guard<std::mutex> lk(p->mu);
    ntt128_plan_s::StreamCtr& c = *stream_entry(p, sid);
    if (c.scratch_elems < elems) {
        // earlier work on this stream may still read the old buffer: cudaFree waits for it
        cudaFree(c.scratch);
        c.scratch = nullptr;
        c.scratch_elems = 0;
        if (cudaMalloc(&c.scratch, elems * sizeof(uint4)) != cudaSuccess) {
            c.scratch = nullptr;
            return NTT128_ERR_OOM;
        }
        c.scratch_elems = elems;
    }
    *out = c.scratch;
    return NTT128_OK;
}

// Scratch for one call: the stream's cached buffer, or -- under stream capture -- a
// stream-ordered allocation the caller frees on the same stream after its last use (a
// graph memory node: the captured graph owns it, so no cache entry is involved).
struct CallScratch {
    uint4* ptr = nullptr;
    bool graph_owned = false;
};
static ntt128_status acquire_scratch(ntt128_plan_s* p, cudaStream_t stream, size_t elems, CallScratch* cs) {
    if (is_capturing(stream)) {
        if (cudaMallocAsync(&cs->ptr, elems * sizeof(uint4), stream) != cudaSuccess) return NTT128_ERR_OOM;
        cs->graph_owned = true;
        return NTT128_OK;
    }
    return stream_scratch(p, stream, elems, &cs->ptr);
}
static void release_scratch(ntt128_plan_s* p, cudaStream_t stream, const CallScratch& cs) {
    if (cs.graph_owned) cudaFreeAsync(cs.ptr, stream);
    else stream_touch(p, stream);
}

// ---------------------------------------------------------------- chained calls
// NTT128_FLAG_CHAIN (include/ntt128.h, DESIGN.md §6 "Chained calls"): the first pass of a
// transform waits, per polynomial, on the previous call's last-pass counters instead of on
// the whole previous grid (griddepcontrol.wait) -- so the tail of one transform overlaps the
// start of the next, as consecutive passes of one transform already do.  Allowed only when
// (a) the previous library call on the stream was this plan's own counter-signalling
// transform (library-wide per-stream generation, ntt128_stream_gen) and (b) every buffer
// of this call either is a buffer of that call (same base) or is disjoint from all of them
// -- every pass touches only its own polynomial's [N] slice of each buffer, so the
// per-polynomial order then covers every read-after-write, write-after-read and
// write-after-write pair between the two calls.  Otherwise the first pass waits for the
// whole previous grid, as without the flag.
static std::mutex g_gen_mu;
static std::unordered_map<unsigned long long, uint64_t> g_gen;   // stream id -> generation
static uint64_t g_gen_next = 0;
// Every public entry point that enqueues device work calls this once per call (it is a no-op
// unless a chained plan exists).  Returns the stream's generation before the call in *prev
// and the call's own in *now (unique across streams; 0 / 0 under stream capture).
void ntt128_stream_gen(cudaStream_t stream, uint64_t* prev, uint64_t* now) {
    *prev = *now = 0;
    if (g_chain_plans.load(std::memory_order_relaxed) == 0) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
    unsigned long long sid = 0;
    if (cudaStreamGetId(stream, &sid) != cudaSuccess) return;
    std::lock_guard<std::mutex> lk(g_gen_mu);
    if (g_gen.size() > 4096) g_gen.clear();        // generations stay unique: a cleared stream never matches
    uint64_t& g = g_gen[sid];
    *prev = g;
    g = *now = ++g_gen_next;
}
static bool chain_bufs_ok(const ntt128_plan_s* p, const ntt128_plan_s::StreamCtr* c, const void* const cur[3]) {
    const uintptr_t bytes = (uintptr_t)p->N * p->batch * sizeof(uint4);
    for (int i = 0; i < 3; i++) {
        if (!cur[i]) continue;
        for (int j = 0; j < 3; j++) {
            const uintptr_t a = (uintptr_t)cur[i], b = (uintptr_t)c->last_bufs[j];
            if (!b || a == b || a + bytes <= b || b + bytes <= a) continue;
            return false;                          // partial overlap: polynomials would not line up
        }
    }
    return true;
}
// Decide whether this call's first pass may wait on the previous call's counters (the
// caller holds p->mu through `ctr`); `cur` are the call's buffers.
static bool chain_wait(const ntt128_plan_s* p, const ntt128_plan_s::StreamCtr* ctr, const RunOpts& o,
                       const void* const cur[3]) {
    if (!(p->flags & NTT128_FLAG_CHAIN) || o.gen_new == 0 || ctr->last_row < 0) return false;
    if (ctr->gen != o.gen_prev && ctr->gen != o.gen_new) return false;   // other library work in between
    return chain_bufs_ok(p, ctr, cur);
}
static void chain_first(const ntt128_plan_s* p, const ntt128_plan_s::StreamCtr* ctr, PassArgs& a) {
    a.pdl_wait = 0u;
    a.cnt_in = ctr->d + (size_t)ctr->last_row * p->batch;
    a.target = ctr->last_target;
}
// the last pass of a chained plan's transform signals row npass - 1; record the call
static void chain_last(ntt128_plan_s* p, ntt128_plan_s::StreamCtr* ctr, PassArgs& a, size_t npass,
                       uint32_t ctas_per_poly, const RunOpts& o, const void* const cur[3]) {
    const int row = (int)npass - 1;
    a.cnt_out = ctr->d + (size_t)row * p->batch;
    ctr->expected[row] += ctas_per_poly;
    ctr->last_row = row;
    ctr->last_target = ctr->expected[row];
    for (int j = 0; j < 3; j++) ctr->last_bufs[j] = cur[j];
    ctr->gen = o.gen_new;
}

// pass i (of npass, execution order) of an overlapped transform: the first pass waits for
// the previous grid; pass i > 0 waits on row i - 1 for the previous pass's CTAs per
// polynomial; every pass but the last signals row i.
static void set_overlap(ntt128_plan_s* p, ntt128_plan_s::StreamCtr* ctr, PassArgs& a, size_t i, size_t npass,
                        uint32_t prev_ctas_per_poly) {
    if (switches().pdl_nocnt) {   // experiment: whole-grid dependencies only
        a.pdl_wait = 1u;
        return;
    }
    a.pdl_wait = i == 0 ? 1u : 0u;
    if (i > 0) {
        ctr->expected[i - 1] += prev_ctas_per_poly;
        a.cnt_in = ctr->d + (i - 1) * (size_t)p->batch;
        a.target = ctr->expected[i - 1];
    }
    if (i + 1 < npass) a.cnt_out = ctr->d + i * (size_t)p->batch;
}

// Cluster path (k_ntt_cluster): cyclic single-pass plans, N = 2^8 .. 2^11, at most
// NTT_CLU_MAX_BATCH polynomials (8 CTAs each).  Measured at N = 2^10 (fwd+inv, graph
// replay, tools/exp_cluster_batch.py): clusters win up to 512 polynomials (B = 64: 9.2 vs
// 14.4 us, B = 512: 45 vs 58 us) and lose at 1024 (85 vs 72 us) to the batched pass.
#ifndef NTT_CLU_MAX_BATCH
#define NTT_CLU_MAX_BATCH 512
#endif
static bool use_cluster(const ntt128_plan_s* p, const RunOpts& o) {
    if (switches().no_cluster || p->kind != 0 || o.pmul || o.io || p->bits.size() != 1) return false;
    return p->log2n >= 8 && p->log2n <= 11 && p->batch <= NTT_CLU_MAX_BATCH;
}
template <bool SL>
static PassKernel cluster_fn(int B) {
    switch (B) {
        case 8: return k_ntt_cluster<8, SL>;
        case 9: return k_ntt_cluster<9, SL>;
        case 10: return k_ntt_cluster<10, SL>;
        default: return k_ntt_cluster<11, SL>;
    }
}
static ntt128_status run_cluster(ntt128_plan_s* p, const uint4* src, uint4* dst, cudaStream_t stream, const RunOpts& o) {
    const int n = (int)p->log2n;
    const bool scale_last = o.inverse;
    PassArgs a;
    memset(&a, 0, sizeof(a));
    a.src = src;
    a.dst = dst;
    a.mods = p->d_mods;
    a.pt = !o.inverse ? p->d_pt_fwd[0] : (o.polymul ? p->d_pt_inv_r[0] : p->d_pt_inv[0]);
    a.pt_stride = p->pt_stride[0];
    a.n = (uint32_t)n;
    a.nq = p->nq;
    a.ninv_r = o.polymul ? 1 : 0;
    const bool pdl = !switches().no_pdl;
    a.pdl_wait = pdl ? 1u : 0u;
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3(p->batch * CLU);
    cfg.blockDim = dim3(1u << (n - CLU_LOG - 1));
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CLU;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 2 : 1;
    const PassKernel fn = scale_last ? cluster_fn<true>(n) : cluster_fn<false>(n);
    if (CLU > 8) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (cudaLaunchKernelEx(&cfg, fn, a) != cudaSuccess) return NTT128_ERR_CUDA;
    ntt128_count_launch(1);
    return NTT128_OK;
}

static ntt128_status run_transform(ntt128_plan_s* p, const uint4* src, uint4* dst, cudaStream_t stream,
                                   const RunOpts& o) {
    if (use_cluster(p, o)) return run_cluster(p, src, dst, stream, o);
    const int n = (int)p->log2n;
    const size_t npass = p->bits.size();
    const bool scale_last = p->kind == 0 && o.inverse;
    // Multi-pass transforms overlap consecutive passes: every pass is a
    // programmatic dependent launch; pass i+1 CTAs wait per polynomial on pass i's
    // completion counters instead of on the whole grid.  Not under stream capture
    // (a captured launch would replay stale counter targets).
    bool overlap = false;
    if (!overlap_allowed(npass, stream, &overlap)) return NTT128_ERR_CUDA;
    ntt128_plan_s::StreamCtr* ctr = nullptr;
    std::unique_lock<std::mutex> lk(p->mu, std::defer_lock);
    if (overlap) {
        ntt128_status st = stream_counters(p, stream, lk, &ctr);
        if (st != NTT128_OK) return st;
    }
    // a single-pass transform is one programmatic dependent launch (no counters): its
    // launch and twiddle prologue overlap the previous kernel's tail, also under capture
    const bool pdl_single = npass == 1 && !switches().no_pdl;
    const void* const bufs[3] = {src, dst, o.pmul};
    const bool chain = overlap && (p->flags & NTT128_FLAG_CHAIN) && !o.io && !switches().pdl_nocnt;
    const bool wait_prev = chain && chain_wait(p, ctr, o, bufs);
    if (ctr && (p->flags & NTT128_FLAG_CHAIN) && !chain) ctr->last_row = -1;   // not signalling: no successor may chain
    int lo = 0;
    uint32_t prev_ctas_per_poly = 0;
    for (size_t i = 0; i < npass; i++) {
        const int B = p->bits[i];
        PassCfg c = pass_cfg(npass, i, B, scale_last, lo, n);
        if (npass == 1 && use_latency_shape(B, p->batch))
            c = scale_last ? single_lat_cfg_t<true>(B) : single_lat_cfg_t<false>(B);
        // plain cyclic first pass of 8 stages, one group per CTA: TL groups per CTA
        {
            const int tl = B == 8 ? NTT_FIRST_TILES : (B == 9 ? NTT_FIRST_TILES9 : 1);
            if (tl > 1 && i == 0 && npass > 1 && c.first && !c.single && !c.tma && c.C == 1 && !o.io && !o.pmul &&
                p->kind == 0 && ((1ull << (n - B)) % tl) == 0 && !switches().no_tiles) {
                c = B == 8 ? first_tl_cfg_t<8, NTT_RB8, (NTT_FIRST_TILES > 1 ? NTT_FIRST_TILES : 2)>()
                           : first_tl_cfg_t<9, NTT_FIRST9_RB, (NTT_FIRST_TILES9 > 1 ? NTT_FIRST_TILES9 : 2)>();
                if (cudaFuncSetAttribute(c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem) != cudaSuccess)
                    return NTT128_ERR_CUDA;
            }
            // one-modulus plans: a later 8-stage pass takes group g of NTT_LATER_TILES polynomials per CTA
            if (NTT_LATER_TILES > 1 && i > 0 && !c.single && c.C == 1 && B == 8 && p->nq == 1 && !o.io && !o.pmul &&
                p->kind == 0 && p->batch % NTT_LATER_TILES == 0 && !switches().no_tiles) {
                const bool sl = scale_last && i + 1 == npass;
                c = sl ? later_tl_cfg_t<8, true, NTT_RB8, (NTT_LATER_TILES > 1 ? NTT_LATER_TILES : 2)>()
                       : later_tl_cfg_t<8, false, NTT_RB8, (NTT_LATER_TILES > 1 ? NTT_LATER_TILES : 2)>();
                if (cudaFuncSetAttribute(c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem) != cudaSuccess)
                    return NTT128_ERR_CUDA;
            }
        }
        bool pm = false;
        if (i == 0 && o.io && npass == 1 && B == 9 && o.io->in_ps == 1 && strided_pm_first(B, p->batch)) {
            // four-step 2^9-point pass C: one polynomial-major pass of the padded multi-pass
            // kernel (2.0 vs 2.07 ms for the 4-polynomial single-pass kernel at cfg 5)
            c = strided_pm_cfg();
            pm = true;
            if (cudaFuncSetAttribute(c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem) != cudaSuccess)
                return NTT128_ERR_CUDA;
        } else if (i == 0 && o.io && o.io->in_ps == 1) {   // four-step pass C: adjacent polynomials per CTA
            if (npass == 1) {
                c = strided_single_cfg(B, scale_last, p->batch);
            } else if (strided_pm_first(B, p->batch)) {
                c = strided_pm_cfg();
                pm = true;
            }
            // > 48 KB of dynamic shared memory (set on the plan's device, as plan_create does)
            if (cudaFuncSetAttribute(c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem) != cudaSuccess)
                return NTT128_ERR_CUDA;
        }
        PassArgs a;
        memset(&a, 0, sizeof(a));
        a.src = i == 0 ? src : dst;
        a.dst = dst;
        a.mods = p->d_mods;
        a.pt_stride = p->pt_stride[i];
        a.f_stride = p->N;
        a.total_groups = (uint64_t)p->batch << (n - B);
        a.n = (uint32_t)n;
        a.lo = (uint32_t)lo;
        a.nq = p->nq;
        a.pt = !o.inverse ? p->d_pt_fwd[i] : (o.polymul ? p->d_pt_inv_r[i] : p->d_pt_inv[i]);
        if (p->psm && !o.pmul && !o.polymul) {   // cyclic call without a point-wise operand: pseudo-Mersenne class
            a.psm = 1;
            a.pt = !o.inverse ? p->d_pt_fwd_psm[i] : p->d_pt_inv_psm[i];
        }
        const bool first = i == 0, last = i + 1 == npass;
        if (first && o.pmul) a.pmul = o.pmul;
        if (scale_last && last) a.ninv_r = o.polymul ? 1 : 0;
        if (p->kind == 1) {
            if (!o.inverse && first) a.fin = p->d_f_twist;
            if (o.inverse && last) a.fout = o.polymul ? p->d_f_untwist_r : p->d_f_untwist;
        }
        a.in_ps = p->N;
        a.in_es = 1;
        if (o.io) {
            if (first && o.io->in_ps) {
                a.in_ps = o.io->in_ps;
                a.in_es = o.io->in_es;
            }
            if (first && o.io->fin) {
                a.fin = o.io->fin;
                a.fpoly = 1;
                a.f_ps = o.io->fin_ps;
                a.f_es = o.io->fin_es;
            }
            if (last && o.io->r_lb) {
                a.r_lb = o.io->r_lb;
                a.r_ps = o.io->r_ps;
                for (int h = 0; h < NTT128_FS_MAX_RANKS; h++) a.rdst[h] = o.io->rdst[h];
            }
        }
        PassCfg alt = c;
        if (c.tma) {
            alt = pass_cfg(npass, i, B, scale_last, lo, n, false);
            if (a.fin || a.pmul || a.in_ps != p->N || a.in_es != 1) c = alt;   // TMA passes read natural tiles only
        }
        // CTAs that signal each polynomial's counter (a PM CTA signals all of its C polynomials)
        const uint32_t ctas_per_poly =
            (uint32_t)(((uint64_t)1 << (n - B)) / (pm ? 1u : (uint64_t)c.C * (c.tiles_across ? 1 : c.tiles)));
        if (overlap) set_overlap(p, ctr, a, i, npass, prev_ctas_per_poly);
        if (i == 0 && wait_prev) chain_first(p, ctr, a);
        if (chain && last) chain_last(p, ctr, a, npass, ctas_per_poly, o, bufs);
        if (pdl_single) a.pdl_wait = 1u;
        const ntt128_status ls = launch_pass_q(p, c, alt, a, B, lo, stream, overlap || pdl_single);
        if (ls != NTT128_OK) return ls;
        lo += B;
        prev_ctas_per_poly = ctas_per_poly;
    }
    return NTT128_OK;
}

// Permutation-free negacyclic transform: forward = CT passes top-down,
// natural in, bit-reversed out; inverse = GS passes bottom-up, bit-reversed in, natural
// out, N^-1 in the last stage; `pmul` fuses the point-wise product into the inverse's
// first load (its R^-1 is cancelled by the R-scaled last-stage table).
static ntt128_status run_transform_nc(ntt128_plan_s* p, const uint4* src, uint4* dst, cudaStream_t stream,
                                      bool inverse, const uint4* pmul, const RunOpts& go) {
    const int n = (int)p->log2n;
    const size_t npass = p->nc_bits.size();
    bool overlap = false;
    if (!overlap_allowed(npass, stream, &overlap)) return NTT128_ERR_CUDA;
    ntt128_plan_s::StreamCtr* ctr = nullptr;
    std::unique_lock<std::mutex> lk(p->mu, std::defer_lock);
    if (overlap) {
        ntt128_status st = stream_counters(p, stream, lk, &ctr);
        if (st != NTT128_OK) return st;
    }
    const void* const bufs[3] = {src, dst, pmul};
    const bool chain = overlap && (p->flags & NTT128_FLAG_CHAIN) && !switches().pdl_nocnt;
    const bool wait_prev = chain && chain_wait(p, ctr, go, bufs);
    std::vector<int> los(npass);
    for (size_t k = 0, lo = 0; k < npass; k++) { los[k] = (int)lo; lo += p->nc_bits[k]; }
    uint32_t prev_ctas_per_poly = 0;
    for (size_t i = 0; i < npass; i++) {
        const size_t k = inverse ? i : npass - 1 - i;      // pass k covers bits [los[k], los[k] + B)
        const int B = p->nc_bits[k];
        const bool top = k + 1 == npass;
        PassCfg c = nc_cfg(inverse, inverse && top, B);
        PassArgs a;
        memset(&a, 0, sizeof(a));
        a.src = i == 0 ? src : dst;
        a.dst = dst;
        a.mods = p->d_mods;
        a.pt_stride = p->nc_stride[k];
        a.total_groups = (uint64_t)p->batch << (n - B);
        a.n = (uint32_t)n;
        a.lo = (uint32_t)los[k];
        a.nq = p->nq;
        a.pt = !inverse ? p->d_nc_fwd[k] : (pmul ? p->d_nc_inv_r[k] : p->d_nc_inv[k]);
        if (i == 0 && pmul) a.pmul = pmul;
        a.ninv_r = pmul ? 1 : 0;
        const uint32_t ctas_per_poly = (uint32_t)(((uint64_t)1 << (n - B)) / (uint64_t)c.C);
        if (overlap) set_overlap(p, ctr, a, i, npass, prev_ctas_per_poly);
        if (i == 0 && wait_prev) chain_first(p, ctr, a);
        if (chain && i + 1 == npass) chain_last(p, ctr, a, npass, ctas_per_poly, go, bufs);
        const ntt128_status ls = launch_pass_q(p, c, c, a, B, los[k], stream, overlap);
        if (ls != NTT128_OK) return ls;
        prev_ctas_per_poly = ctas_per_poly;
    }
    return NTT128_OK;
}

__global__ void k_check_range(const uint4* x, uint64_t per_poly, uint64_t total, const ModC* mods, uint32_t nq, int* err) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t m = nq == 1 ? 0 : (uint32_t)(i / per_poly);
        const ModC& M = mods[m];
        if (!lt_q(u128_from(x[i]), M.q)) atomicOr(err, 1);
    }
}

// The error flag is allocated per call in stream order, so concurrent checks on other
// streams (or threads) never share it.
static ntt128_status check_range(const ntt128_plan_s* p, const uint4* src, cudaStream_t stream) {
    int* d_err = nullptr;
    if (cudaMallocAsync(&d_err, sizeof(int), stream) != cudaSuccess) return NTT128_ERR_OOM;
    if (cudaMemsetAsync(d_err, 0, sizeof(int), stream) != cudaSuccess) { cudaFreeAsync(d_err, stream); return NTT128_ERR_CUDA; }
    const uint64_t total = p->N * p->batch;
    unsigned g = (unsigned)((total + 255) / 256);
    if (g > 148 * 16) g = 148 * 16;
    k_check_range<<<g, 256, 0, stream>>>(src, p->N, total, p->d_mods, p->nq, d_err);
    ntt128_count_launch(1);
    int h = 0;
    const cudaError_t e = cudaMemcpyAsync(&h, d_err, sizeof(int), cudaMemcpyDeviceToHost, stream);
    cudaFreeAsync(d_err, stream);
    if (e != cudaSuccess || cudaStreamSynchronize(stream) != cudaSuccess) return NTT128_ERR_CUDA;
    return h ? NTT128_ERR_INPUT_RANGE : NTT128_OK;
}

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int d) { cudaGetDevice(&prev); cudaSetDevice(d); }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

static ntt128_status transform(const ntt128_plan_t p, const uint64_t* d_in, uint64_t* d_out, cudaStream_t stream,
                               bool inverse) {
    if (!p || !d_in || !d_out) return NTT128_ERR_INVALID_ARG;
    if (!aligned16(d_in) || !aligned16(d_out)) return NTT128_ERR_ALIGNMENT;
    DeviceGuard g(p->device);
    const uint4* src = (const uint4*)d_in;
    uint4* dst = (uint4*)d_out;
    if (p->flags & NTT128_FLAG_CHECK_INPUT) {
        ntt128_status s = check_range(p, src, stream);
        if (s != NTT128_OK) return s;
    }
    RunOpts o{inverse, nullptr, false};
    ntt128_stream_gen(stream, &o.gen_prev, &o.gen_new);
    if (src == dst && p->bits.size() > 1) {
        // the first pass gathers bit-reversed columns: it cannot run in place
        const size_t bytes = (size_t)p->N * p->batch * sizeof(uint4);
        CallScratch cs;
        ntt128_status s = acquire_scratch(p, stream, (size_t)p->N * p->batch, &cs);
        if (s != NTT128_OK) return s;
        if (cudaMemcpyAsync(cs.ptr, src, bytes, cudaMemcpyDeviceToDevice, stream) != cudaSuccess) s = NTT128_ERR_CUDA;
        else s = run_transform(p, cs.ptr, dst, stream, o);
        release_scratch(p, stream, cs);
        return s;
    }
    const ntt128_status s = run_transform(p, src, dst, stream, o);
    if (p->bits.size() > 1) stream_touch(p, stream);
    return s;
}

extern "C" ntt128_status ntt128_forward(const ntt128_plan_t p, const uint64_t* d_in, uint64_t* d_out, ntt128_stream_t stream) {
    return transform(p, d_in, d_out, (cudaStream_t)stream, false);
}

extern "C" ntt128_status ntt128_inverse(const ntt128_plan_t p, const uint64_t* d_in, uint64_t* d_out, ntt128_stream_t stream) {
    return transform(p, d_in, d_out, (cudaStream_t)stream, true);
}

extern "C" ntt128_status ntt128_polymul(const ntt128_plan_t p, const uint64_t* d_a, const uint64_t* d_b, uint64_t* d_c,
                                        ntt128_stream_t stream_) {
    if (!p || !d_a || !d_b || !d_c) return NTT128_ERR_INVALID_ARG;
    if (!aligned16(d_a) || !aligned16(d_b) || !aligned16(d_c)) return NTT128_ERR_ALIGNMENT;
    cudaStream_t stream = (cudaStream_t)stream_;
    DeviceGuard g(p->device);
    if (p->flags & NTT128_FLAG_CHECK_INPUT) {
        ntt128_status s = check_range(p, (const uint4*)d_a, stream);
        if (s == NTT128_OK) s = check_range(p, (const uint4*)d_b, stream);
        if (s != NTT128_OK) return s;
    }
    CallScratch cs;
    ntt128_status s = acquire_scratch(p, stream, 2 * (size_t)p->N * p->batch, &cs);
    if (s != NTT128_OK) return s;
    uint4* fa = cs.ptr;
    uint4* fb = fa + (size_t)p->N * p->batch;
    RunOpts go{false, nullptr, false};
    ntt128_stream_gen(stream, &go.gen_prev, &go.gen_new);   // one API call: its transforms chain among themselves
    if (!p->nc_bits.empty() && !switches().no_nc) {
        // permutation-free pipeline: no twist / untwist multiplies, spectra stay bit-reversed
        s = run_transform_nc(p, (const uint4*)d_a, fa, stream, false, nullptr, go);
        if (s == NTT128_OK) s = run_transform_nc(p, (const uint4*)d_b, fb, stream, false, nullptr, go);
        if (s == NTT128_OK) s = run_transform_nc(p, fa, (uint4*)d_c, stream, true, fb, go);
    } else {
        RunOpts fwd{false, nullptr, false, nullptr, go.gen_prev, go.gen_new};
        s = run_transform(p, (const uint4*)d_a, fa, stream, fwd);
        if (s == NTT128_OK) s = run_transform(p, (const uint4*)d_b, fb, stream, fwd);
        // inverse with the point-wise Montgomery product fused into its first pass's load
        RunOpts inv{true, fb, true, nullptr, go.gen_prev, go.gen_new};
        if (s == NTT128_OK) s = run_transform(p, fa, (uint4*)d_c, stream, inv);
    }
    release_scratch(p, stream, cs);
    return s;
}

// Bit-reversed-order negacyclic transforms (include/ntt128.h): negacyclic plans, N >= 2^10.
static ntt128_status transform_bitrev(const ntt128_plan_t p, const uint64_t* d_in, uint64_t* d_out, cudaStream_t stream,
                                      bool inverse) {
    if (!p || !d_in || !d_out) return NTT128_ERR_INVALID_ARG;
    if (!aligned16(d_in) || !aligned16(d_out)) return NTT128_ERR_ALIGNMENT;
    if (p->kind != 1 || p->nc_bits.empty()) return NTT128_ERR_UNSUPPORTED;
    DeviceGuard g(p->device);
    if (p->flags & NTT128_FLAG_CHECK_INPUT) {
        ntt128_status s = check_range(p, (const uint4*)d_in, stream);
        if (s != NTT128_OK) return s;
    }
    RunOpts go{inverse, nullptr, false};
    ntt128_stream_gen(stream, &go.gen_prev, &go.gen_new);
    const ntt128_status s = run_transform_nc(p, (const uint4*)d_in, (uint4*)d_out, stream, inverse, nullptr, go);
    stream_touch(p, stream);
    return s;
}
extern "C" ntt128_status ntt128_forward_bitrev(const ntt128_plan_t p, const uint64_t* d_in, uint64_t* d_out,
                                               ntt128_stream_t stream) {
    return transform_bitrev(p, d_in, d_out, (cudaStream_t)stream, false);
}
extern "C" ntt128_status ntt128_inverse_bitrev(const ntt128_plan_t p, const uint64_t* d_in, uint64_t* d_out,
                                               ntt128_stream_t stream) {
    return transform_bitrev(p, d_in, d_out, (cudaStream_t)stream, true);
}

// Four-step sub-transform with non-natural input / output (ntt128_internal.h).
ntt128_status ntt128_transform_io(ntt128_plan_t p, const uint4* src, uint4* dst, cudaStream_t stream, bool inverse,
                                  const Ntt128IO& io) {
    if (!p || !src || p->kind != 0) return NTT128_ERR_INVALID_ARG;
    if (io.r_lb) {
        if (p->bits.size() > 1 && !io.tmp) return NTT128_ERR_INVALID_ARG;
        for (uint64_t h = 0; h < (p->N >> io.r_lb); h++)
            if (h >= NTT128_FS_MAX_RANKS || !io.rdst[h]) return NTT128_ERR_INVALID_ARG;
        if (p->bits.size() > 1) dst = io.tmp;
        else if (!dst) dst = io.rdst[0];
    }
    if (!dst) return NTT128_ERR_INVALID_ARG;
    if (src == dst && p->bits.size() > 1) return NTT128_ERR_INVALID_ARG;
    DeviceGuard g(p->device);
    RunOpts o{inverse, nullptr, false, &io};
    ntt128_stream_gen(stream, &o.gen_prev, &o.gen_new);
    const ntt128_status s = run_transform(p, src, dst, stream, o);
    if (p->bits.size() > 1) stream_touch(p, stream);
    return s;
}
