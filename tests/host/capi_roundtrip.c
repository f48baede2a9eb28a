/* Plain-C consumer of the C ABI (include/ntt128.h): no Python, no torch.
 * usage: capi_roundtrip q_lo q_hi omega_lo omega_hi   (hex; a prime with 2^10 | q - 1 and
 * omega of order 2^10).  Forward + inverse of x_i = i (N = 1024) through ntt128_*, checks
 * y_0 = sum x_i = N (N - 1) / 2 (Eq. ntt at k = 0) and inverse(forward(x)) == x, then
 * vec128_add / vec128_sub round trip.  Prints "capi ok" and exits 0 on success. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <cuda_runtime_api.h>
#include "ntt128.h"

#define N 1024
#define CHECK(c, msg) do { if (!(c)) { fprintf(stderr, "FAIL: %s\n", msg); return 1; } } while (0)

int main(int argc, char** argv) {
    if (argc != 5) { fprintf(stderr, "usage: %s q_lo q_hi w_lo w_hi\n", argv[0]); return 2; }
    uint64_t q[2] = {strtoull(argv[1], NULL, 16), strtoull(argv[2], NULL, 16)};
    uint64_t w[2] = {strtoull(argv[3], NULL, 16), strtoull(argv[4], NULL, 16)};
    ntt128_plan_t plan = NULL;
    ntt128_status s = ntt128_plan_create(&plan, 10, 1, q, w, 1, NTT128_CYCLIC, 0);
    CHECK(s == NTT128_OK, ntt128_status_string(s));
    static uint64_t hx[2 * N], hy[2 * N], hz[2 * N];
    for (int i = 0; i < N; i++) { hx[2 * i] = (uint64_t)i; hx[2 * i + 1] = 0; }
    uint64_t *dx, *dy, *dz;
    CHECK(cudaMalloc((void**)&dx, sizeof hx) == cudaSuccess, "cudaMalloc");
    CHECK(cudaMalloc((void**)&dy, sizeof hx) == cudaSuccess, "cudaMalloc");
    CHECK(cudaMalloc((void**)&dz, sizeof hx) == cudaSuccess, "cudaMalloc");
    CHECK(cudaMemcpy(dx, hx, sizeof hx, cudaMemcpyHostToDevice) == cudaSuccess, "H2D");
    CHECK(ntt128_forward(plan, dx, dy, NULL) == NTT128_OK, "forward");
    CHECK(ntt128_inverse(plan, dy, dz, NULL) == NTT128_OK, "inverse");
    CHECK(cudaMemcpy(hy, dy, sizeof hy, cudaMemcpyDeviceToHost) == cudaSuccess, "D2H");
    CHECK(cudaMemcpy(hz, dz, sizeof hz, cudaMemcpyDeviceToHost) == cudaSuccess, "D2H");
    CHECK(hy[0] == (uint64_t)N * (N - 1) / 2 && hy[1] == 0, "y_0 != sum x_i");
    CHECK(memcmp(hx, hz, sizeof hx) == 0, "inverse(forward(x)) != x");
    /* BLAS: (x + y) - y == x on the spectrum y */
    CHECK(vec128_add(dz, dx, dy, N, q, 0, NULL) == NTT128_OK, "vec128_add");
    CHECK(vec128_sub(dz, dz, dy, N, q, 0, NULL) == NTT128_OK, "vec128_sub");
    CHECK(cudaMemcpy(hz, dz, sizeof hz, cudaMemcpyDeviceToHost) == cudaSuccess, "D2H");
    CHECK(memcmp(hx, hz, sizeof hx) == 0, "(x + y) - y != x");
    /* an error path: unaligned pointer */
    CHECK(ntt128_forward(plan, (const uint64_t*)((char*)dx + 8), dy, NULL) == NTT128_ERR_ALIGNMENT, "alignment check");
    ntt128_plan_destroy(plan);
    cudaFree(dx); cudaFree(dy); cudaFree(dz);
    printf("capi ok: launches %llu\n", (unsigned long long)ntt128_launch_count());
    return 0;
}
