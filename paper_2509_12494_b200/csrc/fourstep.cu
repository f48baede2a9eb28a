// fourstep.cu -- distributed four-step NTT of one huge polynomial (include/ntt128.h,
// "Distributed four-step"; BASELINE cfg 5).
//
// N = n1 n2, j = j1 + n1 j2, k = k2 + n2 k1 (G ranks, R1 = n1/G, R2 = n2/G):
//   pass A  (rank g, columns j1 in [g R1, (g+1) R1)): n2-point NTTs of the columns
//           (batched ntt128 plan, root w^{n1}), then z *= w^{j1 k2}, packed by the
//           destination rank of k2                               -> send [G][R1][R2]
//   exchange: all-to-all of equal blocks (the caller's NCCL collective)
//   pass C  (rank h, rows k2 in [h R2, (h+1) R2)): transpose [G R1][R2] -> [R2][n1],
//           then n1-point NTTs (batched plan, root w^{n2})       -> rows [R2][n1]
// The inverse runs the same scheme with the roles of n1 and n2 swapped and w^{-1}.
// The twiddle w^{j1 k2} = w^e, e = j1 k2 mod N, is formed from two small tables
// TH[e >> s] TL[e & (2^s - 1)] with one extra Montgomery product per element
// ("two 2^13 tables for omega_N^{j1 k2}").
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/ntt128.h"
#include "arith128.cuh"
#include "host128.h"

using namespace ntt128;
using ntt128h::u128;

void ntt128_count_launch(uint64_t k);

namespace {

struct FsConst {
    uint32_t q[4];
    uint32_t qinv0;
};

// send[h][r][cc] = z[r][c] * w^{((row0 + r) c) mod N},  c = h * (C/G) + cc
__global__ void k_fs_twiddle_pack(const uint4* __restrict__ z, uint4* __restrict__ send, uint32_t R, uint32_t C,
                                  uint32_t G, uint64_t row0, const uint4* __restrict__ TH, const uint4* __restrict__ TL,
                                  uint32_t s, uint64_t nmask, const FsConst k) {
    const uint32_t CG = C / G;
    const uint64_t total = (uint64_t)R * C;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = i / C, c = i - r * C;
        const uint64_t e = ((row0 + r) * c) & nmask;
        const U128 w = mont_mul(u128_from(__ldg(TH + (e >> s))), u128_from(__ldg(TL + (e & ((1ull << s) - 1)))), k.q, k.qinv0);
        const U128 v = mont_mul(u128_from(z[i]), w, k.q, k.qinv0);
        const uint64_t h = c / CG, cc = c - h * CG;
        send[(h * R + r) * CG + cc] = u128_to(v);
    }
}

// Fused exchange: the same twiddle + pack, but block h is stored straight
// into rank h's receive buffer (peer memory over NVLink / NVSwitch), at the offset the
// all-to-all would have put it: recv_h[(src * R + r) * CG + cc].  One HBM round trip and
// the collective disappear; the transfer overlaps the twiddle multiplications.
#define NTT128_FS_MAX_PEERS 64
struct FsPeers {
    uint4* p[NTT128_FS_MAX_PEERS];
};
__global__ void k_fs_twiddle_pack_peers(const uint4* __restrict__ z, const FsPeers peers, uint32_t R, uint32_t C,
                                        uint32_t G, uint32_t src, uint64_t row0, const uint4* __restrict__ TH,
                                        const uint4* __restrict__ TL, uint32_t s, uint64_t nmask, const FsConst k) {
    const uint32_t CG = C / G;
    const uint64_t total = (uint64_t)R * C;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = i / C, c = i - r * C;
        const uint64_t e = ((row0 + r) * c) & nmask;
        const U128 w = mont_mul(u128_from(__ldg(TH + (e >> s))), u128_from(__ldg(TL + (e & ((1ull << s) - 1)))), k.q, k.qinv0);
        const U128 v = mont_mul(u128_from(z[i]), w, k.q, k.qinv0);
        const uint64_t h = c / CG, cc = c - h * CG;
        peers.p[h][((uint64_t)src * R + r) * CG + cc] = u128_to(v);
    }
}

// out[K][M] = transpose(in[M][K]) through 32 x 32 shared-memory tiles of 16-byte elements
__global__ void k_fs_transpose(const uint4* __restrict__ in, uint4* __restrict__ out, uint32_t M, uint32_t K) {
    __shared__ uint4 tile[32][33];
    const uint32_t bx = blockIdx.x * 32, by = blockIdx.y * 32;  // bx along K, by along M
    for (uint32_t j = threadIdx.y; j < 32; j += blockDim.y) {
        const uint32_t m = by + j, kk = bx + threadIdx.x;
        if (m < M && kk < K) tile[j][threadIdx.x] = in[(uint64_t)m * K + kk];
    }
    __syncthreads();
    for (uint32_t j = threadIdx.y; j < 32; j += blockDim.y) {
        const uint32_t kk = bx + j, m = by + threadIdx.x;
        if (m < M && kk < K) out[(uint64_t)kk * M + m] = tile[threadIdx.x][j];
    }
}

inline uint4 to4(u128 v) {
    return make_uint4((uint32_t)v, (uint32_t)(v >> 32), (uint32_t)(v >> 64), (uint32_t)(v >> 96));
}

}  // namespace

struct ntt128_fourstep_s {
    uint32_t log2n1, log2n2, rank, world, s;
    uint64_t n1, n2, N, R1, R2;
    int device;
    ntt128_plan_t p1 = nullptr, p2 = nullptr;  // n1-point x R2, n2-point x R1
    uint4 *d_TH = nullptr, *d_TL = nullptr, *d_THi = nullptr, *d_TLi = nullptr;
    uint4* d_tmp = nullptr;                    // N/G elements of scratch
    FsConst k;
};

static void fs_free(ntt128_fourstep_s* f) {
    if (!f) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(f->device);
    ntt128_plan_destroy(f->p1);
    ntt128_plan_destroy(f->p2);
    cudaFree(f->d_TH);
    cudaFree(f->d_TL);
    cudaFree(f->d_THi);
    cudaFree(f->d_TLi);
    cudaFree(f->d_tmp);
    cudaSetDevice(prev);
    delete f;
}

extern "C" ntt128_status ntt128_fourstep_create(ntt128_fourstep_t* out, uint32_t log2n1, uint32_t log2n2,
                                                const uint64_t* q_, const uint64_t* omega_, uint32_t rank, uint32_t world,
                                                int device) {
    if (!out || !q_ || !omega_) return NTT128_ERR_INVALID_ARG;
    *out = nullptr;
    if (log2n1 < 1 || log2n1 > 13 || log2n2 < 1 || log2n2 > 13) return NTT128_ERR_INVALID_ARG;
    if (world == 0 || (world & (world - 1)) || rank >= world) return NTT128_ERR_INVALID_ARG;
    const uint64_t n1 = 1ull << log2n1, n2 = 1ull << log2n2, N = n1 * n2;
    if (world > n1 || world > n2) return NTT128_ERR_INVALID_ARG;
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
    const uint32_t logN = log2n1 + log2n2;
    f->s = (logN + 1) / 2;
    for (int i = 0; i < 4; i++) f->k.q[i] = (uint32_t)(q >> (32 * i));
    f->k.qinv0 = (uint32_t)M.qp;

    // sub-plans: n2-point over the R1 local columns (root w^{n1}), n1-point over the R2 rows (root w^{n2})
    const u128 w2 = M.pow(w, n1), w1 = M.pow(w, n2);
    const uint64_t q2[2] = {q_[0], q_[1]};
    const uint64_t r2[2] = {(uint64_t)w2, (uint64_t)(w2 >> 64)}, r1[2] = {(uint64_t)w1, (uint64_t)(w1 >> 64)};
    ntt128_status st = ntt128_plan_create(&f->p2, log2n2, (uint32_t)f->R1, q2, r2, 1, NTT128_CYCLIC, device);
    if (st == NTT128_OK) st = ntt128_plan_create(&f->p1, log2n1, (uint32_t)f->R2, q2, r1, 1, NTT128_CYCLIC, device);
    if (st != NTT128_OK) { fs_free(f); return st; }

    // twiddle tables: TL[i] = w^i (i < 2^s), TH[i] = w^{i 2^s} (i < 2^(logN - s)); Montgomery form
    const uint64_t nl = 1ull << f->s, nh = 1ull << (logN - f->s);
    std::vector<uint4> TL(nl), TH(nh), TLi(nl), THi(nh);
    const u128 wi = M.inv(w);
    const u128 wm = M.to_m(w), wim = M.to_m(wi);
    u128 a = M.r1, b = M.r1;
    for (uint64_t i = 0; i < nl; i++) { TL[i] = to4(a); TLi[i] = to4(b); a = M.mul(a, wm); b = M.mul(b, wim); }
    const u128 ws = M.to_m(M.pow(w, nl)), wsi = M.to_m(M.pow(wi, nl));
    a = M.r1; b = M.r1;
    for (uint64_t i = 0; i < nh; i++) { TH[i] = to4(a); THi[i] = to4(b); a = M.mul(a, ws); b = M.mul(b, wsi); }
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    bool ok = cudaMalloc(&f->d_TL, nl * 16) == cudaSuccess && cudaMalloc(&f->d_TH, nh * 16) == cudaSuccess &&
              cudaMalloc(&f->d_TLi, nl * 16) == cudaSuccess && cudaMalloc(&f->d_THi, nh * 16) == cudaSuccess &&
              cudaMalloc(&f->d_tmp, (N / world) * 16) == cudaSuccess;
    if (ok) {
        ok = cudaMemcpy(f->d_TL, TL.data(), nl * 16, cudaMemcpyHostToDevice) == cudaSuccess &&
             cudaMemcpy(f->d_TH, TH.data(), nh * 16, cudaMemcpyHostToDevice) == cudaSuccess &&
             cudaMemcpy(f->d_TLi, TLi.data(), nl * 16, cudaMemcpyHostToDevice) == cudaSuccess &&
             cudaMemcpy(f->d_THi, THi.data(), nh * 16, cudaMemcpyHostToDevice) == cudaSuccess;
        if (!ok) st = NTT128_ERR_CUDA;
    } else {
        st = NTT128_ERR_OOM;
    }
    cudaSetDevice(prev);
    if (st != NTT128_OK) { fs_free(f); return st; }
    *out = f;
    return NTT128_OK;
}

extern "C" void ntt128_fourstep_destroy(ntt128_fourstep_t f) { fs_free(f); }

namespace {

struct Guard {
    int prev = 0;
    explicit Guard(int d) { cudaGetDevice(&prev); cudaSetDevice(d); }
    ~Guard() { cudaSetDevice(prev); }
};

inline bool al16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

ntt128_status pack(const ntt128_fourstep_s* f, const uint4* z, uint4* send, uint32_t R, uint32_t C, uint64_t row0,
                   bool inverse, cudaStream_t st) {
    const uint64_t total = (uint64_t)R * C;
    unsigned g = (unsigned)((total + 255) / 256);
    if (g > 148 * 8) g = 148 * 8;
    k_fs_twiddle_pack<<<g, 256, 0, st>>>(z, send, R, C, f->world, row0, inverse ? f->d_THi : f->d_TH,
                                         inverse ? f->d_TLi : f->d_TL, f->s, f->N - 1, f->k);
    ntt128_count_launch(1);
    return cudaGetLastError() == cudaSuccess ? NTT128_OK : NTT128_ERR_CUDA;
}

ntt128_status pack_peers(const ntt128_fourstep_s* f, const uint4* z, const uint64_t* const* peers, uint32_t R, uint32_t C,
                         uint64_t row0, bool inverse, cudaStream_t st) {
    if (f->world > NTT128_FS_MAX_PEERS) return NTT128_ERR_UNSUPPORTED;
    FsPeers pp;
    memset(&pp, 0, sizeof(pp));
    for (uint32_t h = 0; h < f->world; h++) {
        if (!peers[h]) return NTT128_ERR_INVALID_ARG;
        if (!al16(peers[h])) return NTT128_ERR_ALIGNMENT;
        pp.p[h] = (uint4*)peers[h];
    }
    const uint64_t total = (uint64_t)R * C;
    unsigned g = (unsigned)((total + 255) / 256);
    if (g > 148 * 8) g = 148 * 8;
    k_fs_twiddle_pack_peers<<<g, 256, 0, st>>>(z, pp, R, C, f->world, f->rank, row0, inverse ? f->d_THi : f->d_TH,
                                               inverse ? f->d_TLi : f->d_TL, f->s, f->N - 1, f->k);
    ntt128_count_launch(1);
    return cudaGetLastError() == cudaSuccess ? NTT128_OK : NTT128_ERR_CUDA;
}

ntt128_status transpose(const uint4* in, uint4* out, uint64_t M, uint64_t K, cudaStream_t st) {
    dim3 grid((unsigned)((K + 31) / 32), (unsigned)((M + 31) / 32)), block(32, 8);
    k_fs_transpose<<<grid, block, 0, st>>>(in, out, (uint32_t)M, (uint32_t)K);
    ntt128_count_launch(1);
    return cudaGetLastError() == cudaSuccess ? NTT128_OK : NTT128_ERR_CUDA;
}

}  // namespace

extern "C" ntt128_status ntt128_fourstep_forward_a(const ntt128_fourstep_t f, const uint64_t* d_cols, uint64_t* d_send,
                                                   ntt128_stream_t s) {
    if (!f || !d_cols || !d_send) return NTT128_ERR_INVALID_ARG;
    if (!al16(d_cols) || !al16(d_send)) return NTT128_ERR_ALIGNMENT;
    Guard g(f->device);
    cudaStream_t st = (cudaStream_t)s;
    ntt128_status r = ntt128_forward(f->p2, d_cols, (uint64_t*)f->d_tmp, s);                 // [R1][n2]: z[j1][k2]
    if (r != NTT128_OK) return r;
    return pack(f, f->d_tmp, (uint4*)d_send, (uint32_t)f->R1, (uint32_t)f->n2, (uint64_t)f->rank * f->R1, false, st);
}

extern "C" ntt128_status ntt128_fourstep_forward_c(const ntt128_fourstep_t f, const uint64_t* d_recv, uint64_t* d_rows,
                                                   ntt128_stream_t s) {
    if (!f || !d_recv || !d_rows) return NTT128_ERR_INVALID_ARG;
    if (!al16(d_recv) || !al16(d_rows)) return NTT128_ERR_ALIGNMENT;
    Guard g(f->device);
    // recv [G][R1][R2] is the (n1 x R2) matrix z[j1][k2_local]; rows of the n1-point NTTs are its columns
    ntt128_status r = transpose((const uint4*)d_recv, f->d_tmp, f->n1, f->R2, (cudaStream_t)s);
    if (r != NTT128_OK) return r;
    return ntt128_forward(f->p1, (const uint64_t*)f->d_tmp, d_rows, s);                       // [R2][n1]: y[k2 + n2 k1]
}

extern "C" ntt128_status ntt128_fourstep_inverse_a(const ntt128_fourstep_t f, const uint64_t* d_rows, uint64_t* d_send,
                                                   ntt128_stream_t s) {
    if (!f || !d_rows || !d_send) return NTT128_ERR_INVALID_ARG;
    if (!al16(d_rows) || !al16(d_send)) return NTT128_ERR_ALIGNMENT;
    Guard g(f->device);
    ntt128_status r = ntt128_inverse(f->p1, d_rows, (uint64_t*)f->d_tmp, s);                 // [R2][n1]: z[k2][j1] / n1
    if (r != NTT128_OK) return r;
    return pack(f, f->d_tmp, (uint4*)d_send, (uint32_t)f->R2, (uint32_t)f->n1, (uint64_t)f->rank * f->R2, true,
                (cudaStream_t)s);
}

extern "C" ntt128_status ntt128_fourstep_inverse_c(const ntt128_fourstep_t f, const uint64_t* d_recv, uint64_t* d_cols,
                                                   ntt128_stream_t s) {
    if (!f || !d_recv || !d_cols) return NTT128_ERR_INVALID_ARG;
    if (!al16(d_recv) || !al16(d_cols)) return NTT128_ERR_ALIGNMENT;
    Guard g(f->device);
    ntt128_status r = transpose((const uint4*)d_recv, f->d_tmp, f->n2, f->R1, (cudaStream_t)s);   // [R1][n2]
    if (r != NTT128_OK) return r;
    return ntt128_inverse(f->p2, (const uint64_t*)f->d_tmp, d_cols, s);                      // x columns, / n2
}

// Fused-exchange pass A (include/ntt128.h): peers[h] = rank h's receive buffer, mapped in
// this process (e.g. torch symmetric memory); the caller brackets the call with barriers.
extern "C" ntt128_status ntt128_fourstep_forward_a_peers(const ntt128_fourstep_t f, const uint64_t* d_cols,
                                                         const uint64_t* const* peers, ntt128_stream_t s) {
    if (!f || !d_cols || !peers) return NTT128_ERR_INVALID_ARG;
    if (!al16(d_cols)) return NTT128_ERR_ALIGNMENT;
    Guard g(f->device);
    ntt128_status r = ntt128_forward(f->p2, d_cols, (uint64_t*)f->d_tmp, s);
    if (r != NTT128_OK) return r;
    return pack_peers(f, f->d_tmp, peers, (uint32_t)f->R1, (uint32_t)f->n2, (uint64_t)f->rank * f->R1, false,
                      (cudaStream_t)s);
}

extern "C" ntt128_status ntt128_fourstep_inverse_a_peers(const ntt128_fourstep_t f, const uint64_t* d_rows,
                                                         const uint64_t* const* peers, ntt128_stream_t s) {
    if (!f || !d_rows || !peers) return NTT128_ERR_INVALID_ARG;
    if (!al16(d_rows)) return NTT128_ERR_ALIGNMENT;
    Guard g(f->device);
    ntt128_status r = ntt128_inverse(f->p1, d_rows, (uint64_t*)f->d_tmp, s);
    if (r != NTT128_OK) return r;
    return pack_peers(f, f->d_tmp, peers, (uint32_t)f->R2, (uint32_t)f->n1, (uint64_t)f->rank * f->R2, true,
                      (cudaStream_t)s);
}
