// Probe for the TMA tile loads of k_ntt_pass (DESIGN.md §6 "TMA staging"):
//  (a) later passes: a 5-D box {2 u64, 9 rows j from -1, 32 chunks m, 1, 1} over a
//      [poly][H][m][j][L] view whose j/m dims overlap (m stride = 8 j strides) must land
//      as the padded layout slot = 1 + l + l/8 with the j = -1 slots zero-filled (OOB);
//  (b) first pass: where does a box of 2^B rows x 16 B with SWIZZLE_128B land?  Checked
//      against two hypotheses: dense (row r at 16-byte slot r ^ ((r >> 3) & 7)) and pitched
//      (each row padded to the 128-byte swizzle span: slot 8 r + (r & 7)).
// Prints PASS/FAIL per case.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -cudart shared
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k5(const __grid_constant__ CUtensorMap map, uint4* out, int L, int H, int poly, uint32_t bytes) {
    __shared__ __align__(1024) uint4 sm[320];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 320; i++) sm[i] = make_uint4(0xdead, 0xdead, 0xdead, 0xdead);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(bytes));
        asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                     ::"r"(su(sm)), "l"(&map), "r"(2 * L), "r"(-1), "r"(0), "r"(H), "r"(poly), "r"(su(&bar)) : "memory");
        asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(su(&bar)));
        for (int i = 0; i < 320; i++) out[i] = sm[i];
    }
}

__global__ void k4(const __grid_constant__ CUtensorMap map, uint4* out, int g, int poly, uint32_t bytes) {
    extern __shared__ __align__(1024) uint4 dsm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4096; i++) dsm[i] = make_uint4(0xdead, 0xdead, 0xdead, 0xdead);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(bytes));
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                     ::"r"(su(dsm)), "l"(&map), "r"(2 * g), "r"(0), "r"(0), "r"(poly), "r"(su(&bar)) : "memory");
        asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(su(&bar)));
        out[4096] = make_uint4(su(dsm) & 1023u, 0, 0, 0);
        for (int i = 0; i < 4096; i++) out[i] = dsm[i];
    }
}

int main() {
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    if (!enc) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
    int fails = 0;
    // (a) later pass: n = 16, lo = 8, B = 8 -> H dim 1; use lo = 4, B = 8, n = 14: H = 4
    {
        const int n = 14, lo = 4, B = 8, P = 2;
        const uint64_t N = 1ull << n;
        std::vector<uint4> h(N * P);
        for (uint64_t i = 0; i < N * P; i++) h[i] = make_uint4((uint32_t)i, 1, 2, 3);
        uint4 *d, *o;
        cudaMalloc(&d, h.size() * 16); cudaMalloc(&o, 2048 * 16);
        cudaMemcpy(d, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
        CUtensorMap map;
        cuuint64_t dims[5] = {2ull << lo, 8, 1ull << (B - 3), 1ull << (n - lo - B), (cuuint64_t)P};
        cuuint64_t strides[4] = {16ull << lo, 16ull << (lo + 3), 16ull << (lo + B), 16 * N};
        cuuint32_t box[5] = {2, 9, 1u << (B - 3), 1, 1}, es[5] = {1, 1, 1, 1, 1};
        CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("(a) encode rc=%d\n", (int)cr);
        const int L = 5, H = 3, poly = 1;
        k5<<<1, 32>>>(map, o, L, H, poly, 9u * (1u << (B - 3)) * 16u);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<uint4> r(320);
        cudaMemcpy(r.data(), o, 320 * 16, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int l = 0; l < (1 << B); l++) {
            const uint64_t idx = poly * N + ((uint64_t)H << (lo + B)) + ((uint64_t)l << lo) + L;
            const uint4 v = r[1 + l + l / 8];
            if (v.x != (uint32_t)idx || v.y != 1 || v.z != 2 || v.w != 3) bad++;
        }
        for (int m = 0; m < (1 << (B - 3)); m++) {
            const uint4 v = r[9 * m];
            if (v.x | v.y | v.z | v.w) bad++;
        }
        printf("(a) padded box with OOB pad rows: %s (err=%s, bad=%d; r[0]=%x r[1]=%x r[9]=%x)\n", bad ? "FAIL" : "PASS",
               cudaGetErrorString(e), bad, r[0].x, r[1].x, r[9].x);
        fails += bad != 0 || e != cudaSuccess;
    }
    // (b) first pass: n = 16, B = 8, gbits = 8: view [poly][r][g]
    for (int B : {7, 8, 9}) {
        const int n = 16, gb = n - B, P = 2;
        const uint64_t N = 1ull << n;
        std::vector<uint4> h(N * P);
        for (uint64_t i = 0; i < N * P; i++) h[i] = make_uint4((uint32_t)i, 5, 6, 7);
        uint4 *d, *o;
        cudaMalloc(&d, h.size() * 16); cudaMalloc(&o, 4097 * 16);
        cudaMemcpy(d, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
        const uint32_t rl = B > 8 ? 256u : (1u << B), rh = (1u << B) / rl;
        CUtensorMap map;
        cuuint64_t dims[4] = {2ull << gb, rl, rh, (cuuint64_t)P};
        cuuint64_t strides[3] = {16ull << gb, (16ull << gb) * rl, 16 * N};
        cuuint32_t box[4] = {2, rl, rh, 1}, es[4] = {1, 1, 1, 1};
        CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("(b) B=%d encode rc=%d\n", B, (int)cr);
        cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * 16);
        const int g = 37, poly = 1;
        k4<<<1, 32, 4096 * 16>>>(map, o, g, poly, (1u << B) * 16u);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<uint4> r(4097);
        cudaMemcpy(r.data(), o, 4097 * 16, cudaMemcpyDeviceToHost);
        int bad_dense = 0, bad_pitch = 0;
        for (int row = 0; row < (1 << B); row++) {
            const uint64_t idx = poly * N + ((uint64_t)row << gb) + g;
            const uint4 v = r[row ^ ((row >> 3) & 7)], w = r[8 * row + (row & 7)];
            if (v.x != (uint32_t)idx || v.y != 5) bad_dense++;
            if (8 * row + (row & 7) >= 4096 || w.x != (uint32_t)idx || w.y != 5) bad_pitch++;
        }
        printf("(b) B=%d swizzle-128B rows: dense %s (bad=%d), 128-byte pitch %s (bad=%d); err=%s, smem base mod 1024 = %u\n", B,
               bad_dense ? "no" : "YES", bad_dense, bad_pitch ? "no" : "YES", bad_pitch, cudaGetErrorString(e), r[4096].x);
        fails += e != cudaSuccess;
    }
    printf("tma_layout: %s\n", fails ? "FAIL" : "PASS");
    return fails ? 1 : 0;
}
