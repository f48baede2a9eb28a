// Shoup vs Montgomery for the multiply-by-a-twiddle of the lazy class (q < 2^126), register
// only ("Shoup vs Montgomery").  Exploration tool, not the product path.
//  V0: arith128.cuh mont_mul_lazy (even/odd CIOS): 32 IMAD.WIDE + 4 IMAD, result in [0, 2q)
//  V1: Shoup, exact quotient: qh = hi128(v w'), w' = floor(w 2^128 / q) (16 products),
//      r = lo128(v w) + lo128(qh (2^128 - q)) (2 x (6 wide + 4 low)), r in [0, 2q)
//  V2: Shoup, truncated quotient: the 13 products of v w' at word positions >= 2 only
//      (qh short by at most 1), r in [0, 3q), one conditional subtraction of 2q -> [0, 2q)
// Every variant's results are checked on the host against (v w) mod q.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "../../paper_2509_12494_b200/csrc/arith128.cuh"
using namespace ntt128;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)
typedef unsigned __int128 u128;

__device__ __forceinline__ void mul256(uint32_t t[8], const uint32_t a[4], const uint32_t b[4]) {
  asm("mul.lo.u32 %0, %8, %12;\n\t mul.hi.u32 %1, %8, %12;\n\t mul.lo.u32 %2, %8, %14;\n\t mul.hi.u32 %3, %8, %14;\n\t"
      "mad.lo.cc.u32 %1, %8, %13, %1;\n\t madc.hi.cc.u32 %2, %8, %13, %2;\n\t madc.lo.cc.u32 %3, %8, %15, %3;\n\t madc.hi.u32 %4, %8, %15, 0;\n\t"
      "mad.lo.cc.u32 %1, %9, %12, %1;\n\t madc.hi.cc.u32 %2, %9, %12, %2;\n\t madc.lo.cc.u32 %3, %9, %14, %3;\n\t madc.hi.cc.u32 %4, %9, %14, %4;\n\t addc.u32 %5, 0, 0;\n\t"
      "mad.lo.cc.u32 %2, %9, %13, %2;\n\t madc.hi.cc.u32 %3, %9, %13, %3;\n\t madc.lo.cc.u32 %4, %9, %15, %4;\n\t madc.hi.u32 %5, %9, %15, %5;\n\t"
      "mad.lo.cc.u32 %2, %10, %12, %2;\n\t madc.hi.cc.u32 %3, %10, %12, %3;\n\t madc.lo.cc.u32 %4, %10, %14, %4;\n\t madc.hi.cc.u32 %5, %10, %14, %5;\n\t addc.u32 %6, 0, 0;\n\t"
      "mad.lo.cc.u32 %3, %10, %13, %3;\n\t madc.hi.cc.u32 %4, %10, %13, %4;\n\t madc.lo.cc.u32 %5, %10, %15, %5;\n\t madc.hi.u32 %6, %10, %15, %6;\n\t"
      "mad.lo.cc.u32 %3, %11, %12, %3;\n\t madc.hi.cc.u32 %4, %11, %12, %4;\n\t madc.lo.cc.u32 %5, %11, %14, %5;\n\t madc.hi.cc.u32 %6, %11, %14, %6;\n\t addc.u32 %7, 0, 0;\n\t"
      "mad.lo.cc.u32 %4, %11, %13, %4;\n\t madc.hi.cc.u32 %5, %11, %13, %5;\n\t madc.lo.cc.u32 %6, %11, %15, %6;\n\t madc.hi.u32 %7, %11, %15, %7;"
      : "=r"(t[0]), "=r"(t[1]), "=r"(t[2]), "=r"(t[3]), "=r"(t[4]), "=r"(t[5]), "=r"(t[6]), "=r"(t[7])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]));
}
// words 4..7 of the sum of the 13 partial products a_i b_j with i + j >= 2
__device__ __forceinline__ void mulhi_trunc(uint32_t h[4], const uint32_t a[4], const uint32_t b[4]) {
  uint32_t t2, t3;
  asm("{\n\t.reg .u32 t4, t5, t6, t7;\n\t"
      // row a0: b2 -> (2,3), b3 -> (3,4)
      "mul.lo.u32 %4, %8, %14;\n\t mul.hi.u32 %5, %8, %14;\n\t"
      "mad.lo.cc.u32 %5, %8, %15, %5;\n\t madc.hi.u32 t4, %8, %15, 0;\n\t"
      // row a1: b1 -> (2,3), b3 -> (4,5); then b2 -> (3,4)
      "mad.lo.cc.u32 %4, %9, %13, %4;\n\t madc.hi.cc.u32 %5, %9, %13, %5;\n\t madc.lo.cc.u32 t4, %9, %15, t4;\n\t madc.hi.cc.u32 t5, %9, %15, 0;\n\t addc.u32 t6, 0, 0;\n\t"
      "mad.lo.cc.u32 %5, %9, %14, %5;\n\t madc.hi.cc.u32 t4, %9, %14, t4;\n\t addc.cc.u32 t5, t5, 0;\n\t addc.u32 t6, t6, 0;\n\t"
      // row a2: b0 -> (2,3), b2 -> (4,5); b1 -> (3,4), b3 -> (5,6)
      "mad.lo.cc.u32 %4, %10, %12, %4;\n\t madc.hi.cc.u32 %5, %10, %12, %5;\n\t madc.lo.cc.u32 t4, %10, %14, t4;\n\t madc.hi.cc.u32 t5, %10, %14, t5;\n\t addc.cc.u32 t6, t6, 0;\n\t addc.u32 t7, 0, 0;\n\t"
      "mad.lo.cc.u32 %5, %10, %13, %5;\n\t madc.hi.cc.u32 t4, %10, %13, t4;\n\t madc.lo.cc.u32 t5, %10, %15, t5;\n\t madc.hi.cc.u32 t6, %10, %15, t6;\n\t addc.u32 t7, t7, 0;\n\t"
      // row a3: b0 -> (3,4), b2 -> (5,6); b1 -> (4,5), b3 -> (6,7)
      "mad.lo.cc.u32 %5, %11, %12, %5;\n\t madc.hi.cc.u32 t4, %11, %12, t4;\n\t madc.lo.cc.u32 t5, %11, %14, t5;\n\t madc.hi.cc.u32 t6, %11, %14, t6;\n\t addc.u32 t7, t7, 0;\n\t"
      "mad.lo.cc.u32 t4, %11, %13, t4;\n\t madc.hi.cc.u32 t5, %11, %13, t5;\n\t madc.lo.cc.u32 t6, %11, %15, t6;\n\t madc.hi.u32 t7, %11, %15, t7;\n\t"
      "mov.u32 %0, t4;\n\t mov.u32 %1, t5;\n\t mov.u32 %2, t6;\n\t mov.u32 %3, t7;\n\t}"
      : "=r"(h[0]), "=r"(h[1]), "=r"(h[2]), "=r"(h[3]), "=&r"(t2), "=&r"(t3)
      : "r"(0), "r"(0), "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]));
}
// low 128 bits of a b + c d (20 word products: 12 wide, 8 low)
__device__ __forceinline__ void mullo2(uint32_t r[4], const uint32_t a[4], const uint32_t b[4], const uint32_t c[4], const uint32_t d[4]) {
  asm("mul.lo.u32 %0, %4, %8;\n\t mul.hi.u32 %1, %4, %8;\n\t mul.lo.u32 %2, %4, %10;\n\t mul.hi.u32 %3, %4, %10;\n\t"
      "mad.lo.cc.u32 %1, %4, %9, %1;\n\t madc.hi.cc.u32 %2, %4, %9, %2;\n\t madc.lo.u32 %3, %4, %11, %3;\n\t"
      "mad.lo.cc.u32 %1, %5, %8, %1;\n\t madc.hi.cc.u32 %2, %5, %8, %2;\n\t madc.lo.u32 %3, %5, %10, %3;\n\t"
      "mad.lo.cc.u32 %2, %5, %9, %2;\n\t madc.hi.u32 %3, %5, %9, %3;\n\t"
      "mad.lo.cc.u32 %2, %6, %8, %2;\n\t madc.hi.u32 %3, %6, %8, %3;\n\t"
      "mad.lo.u32 %3, %6, %9, %3;\n\t mad.lo.u32 %3, %7, %8, %3;\n\t"
      "mad.lo.cc.u32 %0, %12, %16, %0;\n\t madc.hi.cc.u32 %1, %12, %16, %1;\n\t madc.lo.cc.u32 %2, %12, %18, %2;\n\t madc.hi.u32 %3, %12, %18, %3;\n\t"
      "mad.lo.cc.u32 %1, %12, %17, %1;\n\t madc.hi.cc.u32 %2, %12, %17, %2;\n\t madc.lo.u32 %3, %12, %19, %3;\n\t"
      "mad.lo.cc.u32 %1, %13, %16, %1;\n\t madc.hi.cc.u32 %2, %13, %16, %2;\n\t madc.lo.u32 %3, %13, %18, %3;\n\t"
      "mad.lo.cc.u32 %2, %13, %17, %2;\n\t madc.hi.u32 %3, %13, %17, %3;\n\t"
      "mad.lo.cc.u32 %2, %14, %16, %2;\n\t madc.hi.u32 %3, %14, %16, %3;\n\t"
      "mad.lo.u32 %3, %14, %17, %3;\n\t mad.lo.u32 %3, %15, %16, %3;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]),
        "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(d[0]), "r"(d[1]), "r"(d[2]), "r"(d[3]));
}
struct SC { uint32_t q[4], qn[4], q2[4], qinv0; };

template <int V>
__device__ __forceinline__ void mulw(uint32_t x[4], const uint32_t w[4], const uint32_t wp[4], const SC& c) {
  if (V == 0) {
    U128 a{{x[0], x[1], x[2], x[3]}}, b{{w[0], w[1], w[2], w[3]}};
    U128 r = mont_mul_lazy(a, b, c.q, c.qinv0);
    for (int i = 0; i < 4; i++) x[i] = r.w[i];
    return;
  }
  uint32_t h[4];
  if (V == 1) { uint32_t t[8]; mul256(t, x, wp); h[0] = t[4]; h[1] = t[5]; h[2] = t[6]; h[3] = t[7]; }
  else mulhi_trunc(h, x, wp);
  uint32_t r[4];
  mullo2(r, x, w, h, c.qn);
  if (V == 2) {   // [0, 3q) -> [0, 2q)
    U128 rr{{r[0], r[1], r[2], r[3]}};
    rr = reduce_2q(rr, c.q2);
    for (int i = 0; i < 4; i++) r[i] = rr.w[i];
  }
  for (int i = 0; i < 4; i++) x[i] = r[i];
}

template <int V>
__global__ void __launch_bounds__(256) k_rate(uint4* io, const uint4* tw, const SC c, int iters) {
  constexpr int ILP = 4;
  uint32_t x[ILP][4];
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int k = 0; k < ILP; k++) { uint4 v = io[tid * ILP + k]; x[k][0] = v.x; x[k][1] = v.y; x[k][2] = v.z; x[k][3] = v.w; }
  const uint4 wv = tw[V == 0 ? 2 : 0], pv = tw[1];
  const uint32_t w[4] = {wv.x, wv.y, wv.z, wv.w}, wp[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll 1
  for (int it = 0; it < iters; it++)
#pragma unroll
    for (int k = 0; k < ILP; k++) mulw<V>(x[k], w, wp, c);
  for (int k = 0; k < ILP; k++) io[tid * ILP + k] = make_uint4(x[k][0], x[k][1], x[k][2], x[k][3]);
}
// one product per element: v[i] * w[i] for the host check
template <int V>
__global__ void k_check(uint4* out, const uint4* v, const uint4* w, const uint4* wp, const SC c, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t x[4] = {v[i].x, v[i].y, v[i].z, v[i].w}, a[4] = {w[i].x, w[i].y, w[i].z, w[i].w}, b[4] = {wp[i].x, wp[i].y, wp[i].z, wp[i].w};
  mulw<V>(x, a, b, c);
  out[i] = make_uint4(x[0], x[1], x[2], x[3]);
}

static u128 U(uint4 v) { return ((u128)v.w << 96) | ((u128)v.z << 64) | ((u128)v.y << 32) | v.x; }
static uint4 P(u128 v) { return make_uint4((uint32_t)v, (uint32_t)(v >> 32), (uint32_t)(v >> 64), (uint32_t)(v >> 96)); }
static u128 mulmod(u128 a, u128 b, u128 q) {   // q < 2^126
  a %= q; u128 r = 0;
  for (int i = 127; i >= 0; i--) { r = (r << 1) % q; if ((b >> i) & 1) r = (r + a) % q; }
  return r;
}
static u128 shoup_wp(u128 w, u128 q) {         // floor(w 2^128 / q), w < q
  u128 rem = w, quo = 0;
  for (int i = 0; i < 128; i++) { rem <<= 1; quo <<= 1; if (rem >= q) { rem -= q; quo |= 1; } }
  return quo;
}
static uint64_t rng = 0x9E3779B97F4A7C15ull;
static uint64_t nx() { rng += 0x9E3779B97F4A7C15ull; uint64_t z = rng; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; return z ^ (z >> 31); }

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0)); const int sms = p.multiProcessorCount;
  const u128 q = ((u128)1 << 125) - 262143;                       // odd, < 2^126
  u128 inv = 1; for (int i = 0; i < 7; i++) inv *= 2 - q * inv;
  SC c; const uint4 qv = P(q), qnv = P((u128)0 - q), q2v = P(2 * q);
  c.q[0] = qv.x; c.q[1] = qv.y; c.q[2] = qv.z; c.q[3] = qv.w;
  c.qn[0] = qnv.x; c.qn[1] = qnv.y; c.qn[2] = qnv.z; c.qn[3] = qnv.w;
  c.q2[0] = q2v.x; c.q2[1] = q2v.y; c.q2[2] = q2v.z; c.q2[3] = q2v.w;
  c.qinv0 = (uint32_t)(0 - inv);
  // correctness: v < 2^128 (any), w < q; results must be = v w mod q and < 2q
  const int n = 1 << 16;
  std::vector<uint4> hv(n), hw(n), hp(n), ho(n);
  for (int i = 0; i < n; i++) {
    u128 v = ((u128)nx() << 64) | nx(), w = (((u128)nx() << 64) | nx()) % q;
    if (i < 64) { v = ~(u128)0 - (u128)i; w = q - 1 - (u128)(i % 3); }   // extreme operands
    hv[i] = P(v); hw[i] = P(w); hp[i] = P(shoup_wp(w, q));
  }
  uint4 *dv, *dw, *dp, *doo; CK(cudaMalloc(&dv, n * 16)); CK(cudaMalloc(&dw, n * 16)); CK(cudaMalloc(&dp, n * 16)); CK(cudaMalloc(&doo, n * 16));
  CK(cudaMemcpy(dv, hv.data(), n * 16, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dw, hw.data(), n * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dp, hp.data(), n * 16, cudaMemcpyHostToDevice));
  for (int v = 1; v <= 2; v++) {
    if (v == 1) k_check<1><<<n / 256, 256>>>(doo, dv, dw, dp, c, n); else k_check<2><<<n / 256, 256>>>(doo, dv, dw, dp, c, n);
    CK(cudaMemcpy(ho.data(), doo, n * 16, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int i = 0; i < n; i++) { const u128 r = U(ho[i]); if (r >= 2 * q || r % q != mulmod(U(hv[i]), U(hw[i]), q)) bad++; }
    printf("{\"check_variant\":%d,\"n\":%d,\"bad\":%d}\n", v, n, bad);
  }
  // throughput
  const int threads = 256, blocks = sms * 4, iters = 512;
  const size_t m = (size_t)threads * blocks * 4;
  std::vector<uint4> h(m); for (size_t i = 0; i < m; i++) h[i] = P((((u128)nx() << 64) | nx()) % q);
  uint4* d; CK(cudaMalloc(&d, m * 16));
  const u128 w = (((u128)nx() << 64) | nx()) % q;
  const uint4 twh[3] = {P(w), P(shoup_wp(w, q)), P(mulmod(w, (u128)0 - q, q) /* w R mod q, R = 2^128 */)};
  uint4* dt; CK(cudaMalloc(&dt, 48)); CK(cudaMemcpy(dt, twh, 48, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[3] = {"mont_mul_lazy", "shoup_exact", "shoup_trunc13"};
  for (int v = 0; v < 3; v++) {
    CK(cudaMemcpy(d, h.data(), m * 16, cudaMemcpyHostToDevice));
    auto launch = [&]() { if (v == 0) k_rate<0><<<blocks, threads>>>(d, dt, c, iters); else if (v == 1) k_rate<1><<<blocks, threads>>>(d, dt, c, iters); else k_rate<2><<<blocks, threads>>>(d, dt, c, iters); };
    launch(); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 3; r++) { cudaEventRecord(e0); launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms); }
    const double mm = (double)m * iters;
    printf("{\"kernel\":\"%s\",\"ms\":%.4f,\"mulmod_per_s\":%.4e,\"per_clk_per_sm_at1965\":%.3f}\n", names[v], best, mm / (best * 1e-3), mm / (best * 1e-3) / (sms * 1.965e9));
  }
  return 0;
}
