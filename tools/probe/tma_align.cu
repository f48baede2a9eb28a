// Probe: does cp.async.bulk.tensor (TMA) accept shared-memory destinations that are only
// 16-byte aligned (the padded NTT layout puts 8-residue chunks 144 B apart)?  Copies a
// box of 8 rows x 16 B (row stride 4 KB) into smem at offsets 0, 144, 288, 16 and checks.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap map, uint4* out, int off_slots) {
    __shared__ __align__(1024) uint4 sm[64];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 64; i++) sm[i] = make_uint4(0xdead, 0, 0, 0);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(128));
        int c0 = 0, c1 = 3, c2 = 8, c3 = 0;   // u32 lane 0, column L = 3, rows 8..15, outer 0
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                     ::"r"(su(sm + off_slots)), "l"(&map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(su(&bar)) : "memory");
        asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(su(&bar)));
        for (int i = 0; i < 64; i++) out[i] = sm[i];
    }
}

int main() {
    const int L = 256, R = 256;                       // [R rows][L cols] of 16-byte residues
    std::vector<uint4> h(L * R);
    for (int r = 0; r < R; r++) for (int l = 0; l < L; l++) h[r * L + l] = make_uint4(r, l, 7, 9);
    uint4 *d, *o;
    cudaMalloc(&d, h.size() * 16); cudaMalloc(&o, 64 * 16);
    cudaMemcpy(d, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    if (!enc) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
    CUtensorMap map;
    cuuint64_t dims[4] = {4, (cuuint64_t)L, (cuuint64_t)R, 1};
    cuuint64_t strides[3] = {16, (cuuint64_t)L * 16, (cuuint64_t)L * R * 16};
    cuuint32_t box[4] = {4, 1, 8, 1}, es[4] = {1, 1, 1, 1};
    CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d\n", (int)cr);
    for (int off : {0, 9, 18, 1}) {
        k<<<1, 32>>>(map, o, off);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<uint4> r(64);
        cudaMemcpy(r.data(), o, 64 * 16, cudaMemcpyDeviceToHost);
        bool ok = e == cudaSuccess;
        for (int i = 0; i < 8 && ok; i++) ok = r[off + i].x == (unsigned)(8 + i) && r[off + i].y == 3;
        printf("smem offset %d bytes: %s (%s)\n", off * 16, ok ? "ok" : "WRONG", cudaGetErrorString(e));
        if (e != cudaSuccess) return 0;
    }
    return 0;
}
