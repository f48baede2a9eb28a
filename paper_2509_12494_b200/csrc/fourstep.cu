// fourstep.cu -- distributed four-step NTT of one huge polynomial (include/ntt128.h,
// "Distributed four-step"; BASELINE cfg 5).
//
// N = n1 n2, j = j1 + n1 j2, k = k2 + n2 k1 (G ranks, R1 = n1/G, R2 = n2/G).  Since
// jk = j1 k2 + n2 j1 k1 + n1 j2 k2 (mod N), Eq. ntt factors as
//   pass A (rank g, columns j1 in [g R1, (g+1) R1)):
//       z[j1][k2] = sum_{j2} x[j1 + n1 j2] w^{n1 j2 k2}          (n2-point NTTs, batch R1)
//   exchange (block h = the k2 in [h R2, (h+1) R2)): all-to-all, or peer stores
//   pass C (rank h, rows k2 in [h R2, (h+1) R2)):
//       y[k2 + n2 k1] = sum_{j1} (w^{j1 k2} z[j1][k2]) w^{n2 j1 k1}  (n1-point NTTs, batch R2)
// Both passes are the library's own batched plans (ntt128.cu, k_ntt_pass) with non-natural
// I/O (ntt128_internal.h): pass A's LAST pass stores each output straight into the send
// block of its destination rank (or, with peers, into that rank's receive buffer over
// NVLink: the exchange is the epilogue of the transform); pass C's FIRST pass gathers the
// columns of the received [n1][R2] matrix directly (element stride R2) and multiplies the
// four-step twiddle w^{j1 k2} in as it loads -- one Montgomery product per element from a
// per-rank factor table [n1][R2] (plan time, laid out like the received matrix).  In the
// transposed layouts there is no separate twiddle, pack or transpose kernel and no extra HBM
// round trip: a direction is the same 3 passes as the single-GPU plan (n2 = 2^17 as 9 + 8,
// n1 = 2^9 as one pass at cfg 5).  The natural block layout (contiguous N/G slices, below)
// adds one pack kernel before and one transpose kernel after its two extra exchanges.
// The inverse swaps the roles: pass A = n1-point transforms with root w^{-n2} of the rows
// into the blocks of the destination of j1; pass C = N^{-1} w^{-j1 k2} at the load of the
// n2-point transforms with root w^{-n1} of the received [n2][R1] matrix's columns (forward
// kernels with inverse roots: the N^{-1} costs no stage of its own).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/ntt128.h"
#include "arith128.cuh"
#include "host128.h"
#include "ntt128_internal.h"

using namespace ntt128;
using ntt128h::u128;

void ntt128_count_launch(uint64_t k);

namespace {

struct FsConst {
    uint32_t q[4];
    uint32_t qinv0;
    uint32_t scale_m[4];   // factor every entry is multiplied by (Montgomery form)
};

// out[c][r] = s w^{((row0 + r) c) mod N} (Montgomery form), r < R, c < C -- laid out like the
// received matrix pass C reads (input index c major, polynomial r adjacent), from
// pw[b] = w^{2^b} (Montgomery form): square-and-multiply over the exponent's bits.
__global__ void k_fs_factors(uint4* out, uint64_t R, uint64_t C, uint64_t row0, uint64_t nmask, const uint4* pw,
                             const FsConst k) {
    const uint64_t total = R * C;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t c = i / R, r = i - c * R;
        uint64_t e = ((row0 + r) * c) & nmask;
        U128 v = U128{{k.scale_m[0], k.scale_m[1], k.scale_m[2], k.scale_m[3]}};
        for (int b = 0; e; b++, e >>= 1)
            if (e & 1) v = mont_mul(v, u128_from(pw[b]), k.q, k.qinv0);
        out[i] = u128_to(v);
    }
}

inline uint4 to4(u128 v) {
    return make_uint4((uint32_t)v, (uint32_t)(v >> 32), (uint32_t)(v >> 64), (uint32_t)(v >> 96));
}

// ---- natural block layout (SURVEY.md §8(e) "natural block layout ... +2 all-to-alls"):
// pure data movement around the exchanges, no arithmetic.
// Pack before an exchange: out[g][a][r] = in[a][g][r] (in [A][G][R], out [G][A][R]); runs of R
// residues are contiguous on both sides, so a warp moves 512 contiguous bytes per access.
__global__ void k_fs_pack(uint4* __restrict__ out, const uint4* __restrict__ in, uint64_t A, uint32_t G, uint64_t R) {
    const uint64_t total = A * G * R, AR = A * R;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t g = i / AR, rem = i - g * AR, a = rem / R, r = rem - a * R;
        out[i] = __ldcs(in + (a * G + g) * R + r);   // streamed: each residue is read once
    }
}

// Unpack after an exchange: out[k][m] = in[m][k] (in [M][K], out [K][M]), 32 x 32 tiles of
// 16-byte residues through shared memory (row pitch 33: conflict-free column reads).
constexpr int FS_TT = 32;
__global__ void __launch_bounds__(FS_TT * 8) k_fs_transpose(uint4* __restrict__ out, const uint4* __restrict__ in,
                                                            uint64_t M, uint64_t K) {
    __shared__ uint4 tile[FS_TT][FS_TT + 1];
    const uint64_t tiles_k = (K + FS_TT - 1) / FS_TT;
    const uint64_t m0 = (blockIdx.x / tiles_k) * FS_TT, k0 = (blockIdx.x % tiles_k) * FS_TT;
    const int tx = threadIdx.x % FS_TT, ty = threadIdx.x / FS_TT;   // 8 rows of 32 lanes
#pragma unroll
    for (int j = ty; j < FS_TT; j += 8)
        if (m0 + j < M && k0 + tx < K) tile[j][tx] = __ldcs(in + (m0 + j) * K + k0 + tx);
    __syncthreads();
#pragma unroll
    for (int j = ty; j < FS_TT; j += 8)
        if (k0 + j < K && m0 + tx < M) out[(k0 + j) * M + m0 + tx] = tile[tx][j];
}

}  // namespace

struct ntt128_fourstep_s {
    uint32_t log2n1, log2n2, rank, world;
    uint64_t n1, n2, N, R1, R2;
    int device;
    // n1-point x R2 rows: p1 root w^{n2} (forward pass C), p1i root w^{-n2} (inverse pass A);
    // n2-point x R1 columns: p2 root w^{n1} (forward pass A), p2i root w^{-n1} (inverse pass C).
    // The inverse runs FORWARD transforms with the inverse roots: no N^-1 stage in either
    // pass, the whole N^-1 = n1^-1 n2^-1 rides on pass C's factor table.
    ntt128_plan_t p1 = nullptr, p2 = nullptr, p1i = nullptr, p2i = nullptr;
    uint4* d_ff = nullptr;                     // [n1][R2]: w^{j1 (rank R2 + r)}          (forward pass C)
    uint4* d_fi = nullptr;                     // [n2][R1]: N^-1 w^{-(rank R1 + r) k2}    (inverse pass C)
    uint4* d_tmp = nullptr;                    // N/G: pass A's working buffer (multi-pass sub-transforms)
};

static void fs_free(ntt128_fourstep_s* f) {
    if (!f) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(f->device);
    ntt128_plan_destroy(f->p1);
    ntt128_plan_destroy(f->p2);
    ntt128_plan_destroy(f->p1i);
    ntt128_plan_destroy(f->p2i);
    cudaFree(f->d_ff);
    cudaFree(f->d_fi);
    cudaFree(f->d_tmp);
    cudaSetDevice(prev);
    delete f;
}

static cudaError_t gen_factors(uint4* out, uint64_t R, uint64_t C, uint64_t row0, u128 w, const ntt128h::Mont& M,
                               FsConst k, u128 scale, uint32_t logN) {
    for (int i = 0; i < 4; i++) k.scale_m[i] = (uint32_t)(M.to_m(scale) >> (32 * i));
    std::vector<uint4> pw(logN + 1);
    u128 b = M.to_m(w);
    for (uint32_t i = 0; i <= logN; i++) {
        pw[i] = to4(b);
        b = M.mul(b, b);
    }
    uint4* d_pw = nullptr;
    cudaError_t e = cudaMalloc(&d_pw, pw.size() * sizeof(uint4));
    if (e == cudaSuccess) e = cudaMemcpy(d_pw, pw.data(), pw.size() * sizeof(uint4), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        k_fs_factors<<<148 * 8, 256>>>(out, R, C, row0, (1ull << logN) - 1, d_pw, k);
        ntt128_count_launch(1);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
    }
    cudaFree(d_pw);
    return e;
}

extern "C" ntt128_status ntt128_fourstep_create(ntt128_fourstep_t* out, uint32_t log2n1, uint32_t log2n2,
                                                const uint64_t* q_, const uint64_t* omega_, uint32_t rank, uint32_t world,
                                                int device) {
    if (!out || !q_ || !omega_) return NTT128_ERR_INVALID_ARG;
    *out = nullptr;
    if (log2n1 < 1 || log2n2 < 1 || log2n1 + log2n2 > 26) return NTT128_ERR_INVALID_ARG;
    if (world == 0 || (world & (world - 1)) || rank >= world || world > NTT128_FS_MAX_RANKS) return NTT128_ERR_INVALID_ARG;
    const uint64_t n1 = 1ull << log2n1, n2 = 1ull << log2n2, N = n1 * n2;
    // every exchange block is at least 2 residues wide (a transform's destination-block
    // store keys on log2 of the block width, which must be >= 1)
    if (world > 1 && (2 * world > n1 || 2 * world > n2)) return NTT128_ERR_INVALID_ARG;
    const u128 q = ntt128h::make(q_[0], q_[1]), w = ntt128h::make(omega_[0], omega_[1]);
    if ((q & 1) == 0 || q < 3) return NTT128_ERR_MODULUS;
    if (!ntt128h::is_probable_prime(q)) return NTT128_ERR_NOT_PRIME;
    if ((q - 1) % N != 0) return NTT128_ERR_NO_ROOT;
    if (w >= q) return NTT128_ERR_BAD_ROOT;
    ntt128h::Mont M(q);
    if (M.pow(w, N / 2) != q - 1) return NTT128_ERR_BAD_ROOT;

    ntt128_fourstep_s* f = new (std::nothrow) ntt128_fourstep_s();
    if (!f) return NTT128_ERR_OOM;
    f->log2n1 = log2n1;
    f->log2n2 = log2n2;
    f->rank = rank;
    f->world = world;
    f->n1 = n1;
    f->n2 = n2;
    f->N = N;
    f->R1 = n1 / world;
    f->R2 = n2 / world;
    f->device = device;
    FsConst k;
    for (int i = 0; i < 4; i++) k.q[i] = (uint32_t)(q >> (32 * i));
    k.qinv0 = (uint32_t)M.qp;

    // sub-plans: n2-point over the R1 local columns (root w^{n1}), n1-point over the R2 rows (root w^{n2})
    const u128 wi = M.inv(w);
    const u128 w2 = M.pow(w, n1), w1 = M.pow(w, n2), w2i = M.pow(wi, n1), w1i = M.pow(wi, n2);
    const uint64_t qq[2] = {q_[0], q_[1]};
    const uint64_t r2[2] = {(uint64_t)w2, (uint64_t)(w2 >> 64)}, r1[2] = {(uint64_t)w1, (uint64_t)(w1 >> 64)};
    const uint64_t r2i[2] = {(uint64_t)w2i, (uint64_t)(w2i >> 64)}, r1i[2] = {(uint64_t)w1i, (uint64_t)(w1i >> 64)};
    ntt128_status st = ntt128_plan_create(&f->p2, log2n2, (uint32_t)f->R1, qq, r2, 1, NTT128_CYCLIC, device);
    if (st == NTT128_OK) st = ntt128_plan_create(&f->p1, log2n1, (uint32_t)f->R2, qq, r1, 1, NTT128_CYCLIC, device);
    if (st == NTT128_OK) st = ntt128_plan_create(&f->p2i, log2n2, (uint32_t)f->R1, qq, r2i, 1, NTT128_CYCLIC, device);
    if (st == NTT128_OK) st = ntt128_plan_create(&f->p1i, log2n1, (uint32_t)f->R2, qq, r1i, 1, NTT128_CYCLIC, device);
    if (st != NTT128_OK) { fs_free(f); return st; }

    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    const uint64_t local = N / world;
    if (cudaMalloc(&f->d_ff, local * 16) != cudaSuccess || cudaMalloc(&f->d_fi, local * 16) != cudaSuccess ||
        cudaMalloc(&f->d_tmp, local * 16) != cudaSuccess) {
        st = NTT128_ERR_OOM;
    } else if (gen_factors(f->d_ff, f->R2, n1, (uint64_t)rank * f->R2, w, M, k, 1, log2n1 + log2n2) != cudaSuccess ||
               gen_factors(f->d_fi, f->R1, n2, (uint64_t)rank * f->R1, wi, M, k, M.inv((u128)(N % q)), log2n1 + log2n2) !=
                   cudaSuccess) {
        st = NTT128_ERR_CUDA;
    }
    cudaSetDevice(prev);
    if (st != NTT128_OK) { fs_free(f); return st; }
    *out = f;
    return NTT128_OK;
}

extern "C" void ntt128_fourstep_destroy(ntt128_fourstep_t f) { fs_free(f); }

namespace {

inline bool al16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// pass A's output blocks: block h of `bases` receives the outputs k with k >> lb == h
ntt128_status pass_a(const ntt128_fourstep_s* f, ntt128_plan_t plan, bool inverse, const uint64_t* d_in,
                     uint4* const* bases, uint64_t R_out, uint64_t n_sub, cudaStream_t st) {
    Ntt128IO io;
    io.tmp = f->d_tmp;
    if (f->world > 1) {
        uint32_t lb = 0;
        while ((1ull << lb) < n_sub / f->world) lb++;   // log2 of the block width (R2 forward, R1 inverse)
        io.r_lb = lb;
        io.r_ps = R_out;
        for (uint32_t h = 0; h < f->world; h++) io.rdst[h] = bases[h];
    }
    return ntt128_transform_io(plan, (const uint4*)d_in, f->world > 1 ? nullptr : bases[0], st, inverse, io);
}

// pass C: columns of the received [n_sub][R_in] matrix, four-step factor at the load
ntt128_status pass_c(const ntt128_fourstep_s* f, ntt128_plan_t plan, bool inverse, const uint64_t* d_recv,
                     uint64_t* d_out, uint64_t R_in, const uint4* fac, cudaStream_t st) {
    Ntt128IO io;
    io.in_ps = 1;
    io.in_es = R_in;
    io.fin = fac;                 // [n_sub][R_in]: same layout as the received matrix
    io.fin_ps = 1;
    io.fin_es = R_in;
    (void)f;
    return ntt128_transform_io(plan, (const uint4*)d_recv, (uint4*)d_out, st, inverse, io);
}

}  // namespace

extern "C" ntt128_status ntt128_fourstep_forward_a(const ntt128_fourstep_t f, const uint64_t* d_cols, uint64_t* d_send,
                                                   ntt128_stream_t s) {
    if (!f || !d_cols || !d_send) return NTT128_ERR_INVALID_ARG;
    if (!al16(d_cols) || !al16(d_send)) return NTT128_ERR_ALIGNMENT;
    uint4* bases[NTT128_FS_MAX_RANKS] = {};
    for (uint32_t h = 0; h < f->world; h++) bases[h] = (uint4*)d_send + (uint64_t)h * f->R1 * f->R2;   // send[h][r][cc]
    return pass_a(f, f->p2, false, d_cols, bases, f->R2, f->n2, (cudaStream_t)s);
}

extern "C" ntt128_status ntt128_fourstep_forward_c(const ntt128_fourstep_t f, const uint64_t* d_recv, uint64_t* d_rows,
                                                   ntt128_stream_t s) {
    if (!f || !d_recv || !d_rows) return NTT128_ERR_INVALID_ARG;
    if (!al16(d_recv) || !al16(d_rows)) return NTT128_ERR_ALIGNMENT;
    if (d_recv == d_rows) return NTT128_ERR_INVALID_ARG;
    // recv [G][R1][R2] = z[j1][k2_local] with j1 = g R1 + r: column cc is row cc of the output
    return pass_c(f, f->p1, false, d_recv, d_rows, f->R2, f->d_ff, (cudaStream_t)s);
}

extern "C" ntt128_status ntt128_fourstep_inverse_a(const ntt128_fourstep_t f, const uint64_t* d_rows, uint64_t* d_send,
                                                   ntt128_stream_t s) {
    if (!f || !d_rows || !d_send) return NTT128_ERR_INVALID_ARG;
    if (!al16(d_rows) || !al16(d_send)) return NTT128_ERR_ALIGNMENT;
    uint4* bases[NTT128_FS_MAX_RANKS] = {};
    for (uint32_t h = 0; h < f->world; h++) bases[h] = (uint4*)d_send + (uint64_t)h * f->R2 * f->R1;   // send[h][r][m]
    return pass_a(f, f->p1i, false, d_rows, bases, f->R1, f->n1, (cudaStream_t)s);
}

extern "C" ntt128_status ntt128_fourstep_inverse_c(const ntt128_fourstep_t f, const uint64_t* d_recv, uint64_t* d_cols,
                                                   ntt128_stream_t s) {
    if (!f || !d_recv || !d_cols) return NTT128_ERR_INVALID_ARG;
    if (!al16(d_recv) || !al16(d_cols)) return NTT128_ERR_ALIGNMENT;
    if (d_recv == d_cols) return NTT128_ERR_INVALID_ARG;
    return pass_c(f, f->p2i, false, d_recv, d_cols, f->R1, f->d_fi, (cudaStream_t)s);
}

// Fused exchange (include/ntt128.h): peers[h] = rank h's receive buffer, mapped in this
// process (e.g. torch symmetric memory); the caller brackets the call with barriers.  Pass
// A's last pass stores each output into its destination rank's receive buffer at the
// offset the all-to-all would have used ([src rank][R][block width]).
static ntt128_status a_peers(const ntt128_fourstep_s* f, const uint64_t* d_in, const uint64_t* const* peers,
                             bool inverse, cudaStream_t st) {
    if (!f || !d_in || !peers) return NTT128_ERR_INVALID_ARG;
    if (!al16(d_in)) return NTT128_ERR_ALIGNMENT;
    uint4* bases[NTT128_FS_MAX_RANKS] = {};
    const uint64_t blk = f->R1 * f->R2;
    for (uint32_t h = 0; h < f->world; h++) {
        if (!peers[h]) return NTT128_ERR_INVALID_ARG;
        if (!al16(peers[h])) return NTT128_ERR_ALIGNMENT;
        bases[h] = (uint4*)peers[h] + (uint64_t)f->rank * blk;
    }
    return inverse ? pass_a(f, f->p1i, false, d_in, bases, f->R1, f->n1, st)
                   : pass_a(f, f->p2, false, d_in, bases, f->R2, f->n2, st);
}

// ---------------------------------------------------------------- natural block layout
// (include/ntt128.h "Natural block layout").  Rank g holds x[g N/G + i], i < N/G: viewed as
// [R2][n1] (j2 = g R2 + a) for the input, [R1][n2] (k1 = g R1 + b) for the output.  Each
// direction is pack -> exchange -> pass A (reading the received matrix's columns) ->
// exchange -> pass C (last pass into the blocks of the natural owners) -> exchange ->
// unpack: the transposed layouts' one exchange plus one at each end.
namespace {

ntt128_status launch_pack(const ntt128_fourstep_s* f, const uint64_t* d_in, uint64_t* d_out, uint64_t A, uint64_t R,
                          cudaStream_t st) {
    if (!f || !d_in || !d_out) return NTT128_ERR_INVALID_ARG;
    if (!al16(d_in) || !al16(d_out)) return NTT128_ERR_ALIGNMENT;
    if (d_in == d_out) return NTT128_ERR_INVALID_ARG;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(f->device);
    const uint64_t total = A * f->world * R;
    const uint64_t blocks = (total + 255) / 256 < 148ull * 16 ? (total + 255) / 256 : 148ull * 16;
    k_fs_pack<<<(unsigned)blocks, 256, 0, st>>>((uint4*)d_out, (const uint4*)d_in, A, f->world, R);
    ntt128_count_launch(1);
    const cudaError_t e = cudaGetLastError();
    cudaSetDevice(prev);
    return e == cudaSuccess ? NTT128_OK : NTT128_ERR_CUDA;
}

ntt128_status launch_unpack(const ntt128_fourstep_s* f, const uint64_t* d_in, uint64_t* d_out, uint64_t M, uint64_t K,
                            cudaStream_t st) {
    if (!f || !d_in || !d_out) return NTT128_ERR_INVALID_ARG;
    if (!al16(d_in) || !al16(d_out)) return NTT128_ERR_ALIGNMENT;
    if (d_in == d_out) return NTT128_ERR_INVALID_ARG;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(f->device);
    const uint64_t tiles = ((M + FS_TT - 1) / FS_TT) * ((K + FS_TT - 1) / FS_TT);
    k_fs_transpose<<<(unsigned)tiles, FS_TT * 8, 0, st>>>((uint4*)d_out, (const uint4*)d_in, M, K);
    ntt128_count_launch(1);
    const cudaError_t e = cudaGetLastError();
    cudaSetDevice(prev);
    return e == cudaSuccess ? NTT128_OK : NTT128_ERR_CUDA;
}

// pass A over the columns of a received [n_sub][R] matrix (element stride R), last pass into
// the send blocks [G][R][n_sub/G]
ntt128_status pass_a_nat(const ntt128_fourstep_s* f, ntt128_plan_t plan, const uint64_t* d_recv, uint64_t* d_send,
                         uint64_t R, uint64_t n_sub, cudaStream_t st) {
    if (!f || !d_recv || !d_send) return NTT128_ERR_INVALID_ARG;
    if (!al16(d_recv) || !al16(d_send)) return NTT128_ERR_ALIGNMENT;
    if (d_recv == d_send) return NTT128_ERR_INVALID_ARG;
    Ntt128IO io;
    io.tmp = f->d_tmp;
    io.in_ps = 1;
    io.in_es = R;
    uint32_t lb = 0;
    while ((1ull << lb) < n_sub / f->world) lb++;
    io.r_lb = lb;
    io.r_ps = n_sub / f->world;
    for (uint32_t h = 0; h < f->world; h++) io.rdst[h] = (uint4*)d_send + (uint64_t)h * R * (n_sub / f->world);
    if (f->world == 1) io.r_lb = 0;   // one rank: the block is the whole output row
    return ntt128_transform_io(plan, (const uint4*)d_recv, f->world == 1 ? (uint4*)d_send : nullptr, st, false, io);
}

// pass C (four-step factor at the load, as ntt128_fourstep_*_c) whose last pass stores output
// k of local polynomial p into block k / (n_out/G) of the send buffer [G][R][n_out/G] --
// the natural owner of k
ntt128_status pass_c_nat(const ntt128_fourstep_s* f, ntt128_plan_t plan, const uint64_t* d_recv, uint64_t* d_send,
                         uint64_t R_in, const uint4* fac, uint64_t R, uint64_t n_out, cudaStream_t st) {
    if (!f || !d_recv || !d_send) return NTT128_ERR_INVALID_ARG;
    if (!al16(d_recv) || !al16(d_send)) return NTT128_ERR_ALIGNMENT;
    if (d_recv == d_send) return NTT128_ERR_INVALID_ARG;
    Ntt128IO io;
    io.tmp = f->d_tmp;
    io.in_ps = 1;
    io.in_es = R_in;
    io.fin = fac;
    io.fin_ps = 1;
    io.fin_es = R_in;
    if (f->world > 1) {
        uint32_t lb = 0;
        while ((1ull << lb) < n_out / f->world) lb++;
        io.r_lb = lb;
        io.r_ps = n_out / f->world;
        for (uint32_t h = 0; h < f->world; h++) io.rdst[h] = (uint4*)d_send + (uint64_t)h * R * (n_out / f->world);
    }
    return ntt128_transform_io(plan, (const uint4*)d_recv, f->world > 1 ? nullptr : (uint4*)d_send, st, false, io);
}

}  // namespace

extern "C" ntt128_status ntt128_fourstep_forward_pack(const ntt128_fourstep_t f, const uint64_t* d_nat, uint64_t* d_send,
                                                      ntt128_stream_t s) {
    // x slice [R2][G][R1] -> send [G][R2][R1]: block g = the columns j1 rank g transforms
    return f ? launch_pack(f, d_nat, d_send, f->R2, f->R1, (cudaStream_t)s) : NTT128_ERR_INVALID_ARG;
}

extern "C" ntt128_status ntt128_fourstep_forward_a_nat(const ntt128_fourstep_t f, const uint64_t* d_recv, uint64_t* d_send,
                                                       ntt128_stream_t s) {
    // recv [G][R2][R1] = [n2][R1]: X_g[r][j2] = recv[j2 R1 + r] -> send [G][R1][R2] (as forward_a)
    return f ? pass_a_nat(f, f->p2, d_recv, d_send, f->R1, f->n2, (cudaStream_t)s) : NTT128_ERR_INVALID_ARG;
}

extern "C" ntt128_status ntt128_fourstep_forward_c_nat(const ntt128_fourstep_t f, const uint64_t* d_recv, uint64_t* d_send,
                                                       ntt128_stream_t s) {
    // recv [G][R1][R2] (as forward_c) -> send [G][R2][R1]: block h = the k1 in [h R1, (h+1) R1)
    return f ? pass_c_nat(f, f->p1, d_recv, d_send, f->R2, f->d_ff, f->R2, f->n1, (cudaStream_t)s)
             : NTT128_ERR_INVALID_ARG;
}

extern "C" ntt128_status ntt128_fourstep_forward_unpack(const ntt128_fourstep_t f, const uint64_t* d_recv, uint64_t* d_nat,
                                                        ntt128_stream_t s) {
    // recv [G][R2][R1] = [n2][R1] (k2, k1 - g R1) -> y slice [R1][n2]
    return f ? launch_unpack(f, d_recv, d_nat, f->n2, f->R1, (cudaStream_t)s) : NTT128_ERR_INVALID_ARG;
}

extern "C" ntt128_status ntt128_fourstep_inverse_pack(const ntt128_fourstep_t f, const uint64_t* d_nat, uint64_t* d_send,
                                                      ntt128_stream_t s) {
    // y slice [R1][G][R2] -> send [G][R1][R2]: block g = the k2 rank g holds in the rows layout
    return f ? launch_pack(f, d_nat, d_send, f->R1, f->R2, (cudaStream_t)s) : NTT128_ERR_INVALID_ARG;
}

extern "C" ntt128_status ntt128_fourstep_inverse_a_nat(const ntt128_fourstep_t f, const uint64_t* d_recv, uint64_t* d_send,
                                                       ntt128_stream_t s) {
    // recv [G][R1][R2] = [n1][R2]: Y_g[r][k1] = recv[k1 R2 + r] -> send [G][R2][R1] (as inverse_a)
    return f ? pass_a_nat(f, f->p1i, d_recv, d_send, f->R2, f->n1, (cudaStream_t)s) : NTT128_ERR_INVALID_ARG;
}

extern "C" ntt128_status ntt128_fourstep_inverse_c_nat(const ntt128_fourstep_t f, const uint64_t* d_recv, uint64_t* d_send,
                                                       ntt128_stream_t s) {
    // recv [G][R2][R1] (as inverse_c) -> send [G][R1][R2]: block h = the j2 in [h R2, (h+1) R2)
    return f ? pass_c_nat(f, f->p2i, d_recv, d_send, f->R1, f->d_fi, f->R1, f->n2, (cudaStream_t)s)
             : NTT128_ERR_INVALID_ARG;
}

extern "C" ntt128_status ntt128_fourstep_inverse_unpack(const ntt128_fourstep_t f, const uint64_t* d_recv, uint64_t* d_nat,
                                                        ntt128_stream_t s) {
    // recv [G][R1][R2] = [n1][R2] (j1, j2 - g R2) -> x slice [R2][n1]
    return f ? launch_unpack(f, d_recv, d_nat, f->n1, f->R2, (cudaStream_t)s) : NTT128_ERR_INVALID_ARG;
}

extern "C" ntt128_status ntt128_fourstep_forward_a_peers(const ntt128_fourstep_t f, const uint64_t* d_cols,
                                                         const uint64_t* const* peers, ntt128_stream_t s) {
    return a_peers(f, d_cols, peers, false, (cudaStream_t)s);
}

extern "C" ntt128_status ntt128_fourstep_inverse_a_peers(const ntt128_fourstep_t f, const uint64_t* d_rows,
                                                         const uint64_t* const* peers, ntt128_stream_t s) {
    return a_peers(f, d_rows, peers, true, (cudaStream_t)s);
}
