// Integer-pipe microbenchmark for the roofline denominator R:
// peak rate of 32x32->64-bit products on this B200, plus the ALU carry-add rate.
// Each kernel runs ILP independent dependency chains per thread over all SMs and
// reports SASS-instructions/clk/SM measured with clock64 and products/s by events.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>
#include <cstdlib>
#include <ctime>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ILP = 8;

// ---- 1. IMAD.WIDE.U32 (mad.wide.u32 with 64-bit addend), independent chains
__global__ void k_imad_wide(uint64_t* out, uint32_t seed, int iters, long long* cyc) {
  uint64_t acc[ILP]; uint32_t a = seed ^ threadIdx.x, b = seed * 7u + blockIdx.x;
#pragma unroll
  for (int k = 0; k < ILP; k++) acc[k] = k + threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int k = 0; k < ILP; k++) asm volatile("{\n\t.reg .u32 l, h;\n\tmov.b64 {l, h}, %1;\n\tmad.wide.u32 %0, h, %2, %0;\n\t}" : "+l"(acc[k]) : "l"(acc[(k+1)%ILP]), "r"(b));
  }
  long long t1 = clock64();
  uint64_t s = 0;
#pragma unroll
  for (int k = 0; k < ILP; k++) s ^= acc[k];
  if (s == 0x1234567) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// ---- 2. IMAD.HI.U32 (mad.hi.u32)
__global__ void k_imad_hi(uint64_t* out, uint32_t seed, int iters, long long* cyc) {
  uint32_t acc[ILP]; uint32_t a = seed ^ threadIdx.x, b = seed * 7u + blockIdx.x;
#pragma unroll
  for (int k = 0; k < ILP; k++) acc[k] = k + threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int k = 0; k < ILP; k++) asm volatile("mad.hi.u32 %0, %0, %1, %0;" : "+r"(acc[k]) : "r"(b));
  }
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < ILP; k++) s ^= acc[k];
  if (s == 0x1234567) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// ---- 3. IMAD (mad.lo.u32)
__global__ void k_imad_lo(uint64_t* out, uint32_t seed, int iters, long long* cyc) {
  uint32_t acc[ILP]; uint32_t a = seed ^ threadIdx.x, b = seed * 7u + blockIdx.x;
#pragma unroll
  for (int k = 0; k < ILP; k++) acc[k] = k + threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int k = 0; k < ILP; k++) asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(acc[k]) : "r"(b));
  }
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < ILP; k++) s ^= acc[k];
  if (s == 0x1234567) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// ---- 4. IMAD.WIDE.U32 carry chains: 4-product chain (mad.lo.cc / madc.hi.cc pairs)
__global__ void k_imad_wide_cc(uint64_t* out, uint32_t seed, int iters, long long* cyc) {
  uint32_t t[ILP][4]; uint32_t a = seed ^ threadIdx.x, b0 = seed * 7u + blockIdx.x, b1 = b0 ^ 0x55, b2 = b0 + 3, b3 = b0 * 5;
#pragma unroll
  for (int k = 0; k < ILP; k++) { t[k][0] = k; t[k][1] = threadIdx.x; t[k][2] = 3; t[k][3] = 4; }
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int k = 0; k < ILP; k++)
      asm volatile("mad.lo.cc.u32 %0, %4, %5, %0;\n\t madc.hi.cc.u32 %1, %4, %5, %1;\n\t"
                   "madc.lo.cc.u32 %2, %4, %6, %2;\n\t madc.hi.u32 %3, %4, %6, %3;"
                   : "+r"(t[k][0]), "+r"(t[k][1]), "+r"(t[k][2]), "+r"(t[k][3]) : "r"(t[k][3]), "r"(b0), "r"(b2));
  }
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < ILP; k++) s ^= t[k][0] ^ t[k][1] ^ t[k][2] ^ t[k][3];
  if (s == 0x1234567) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// ---- 5. IADD3 carry chain (add.cc / addc) 4 words
__global__ void k_iadd_cc(uint64_t* out, uint32_t seed, int iters, long long* cyc) {
  uint32_t t[ILP][4]; uint32_t b0 = seed * 7u + blockIdx.x, b1 = b0 ^ 0x55, b2 = b0 + 3, b3 = b0 * 5;
#pragma unroll
  for (int k = 0; k < ILP; k++) { t[k][0] = k; t[k][1] = threadIdx.x; t[k][2] = 3; t[k][3] = 4; }
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int k = 0; k < ILP; k++)
      asm volatile("add.cc.u32 %0, %0, %4;\n\t addc.cc.u32 %1, %1, %5;\n\t addc.cc.u32 %2, %2, %6;\n\t addc.u32 %3, %3, %7;"
                   : "+r"(t[k][0]), "+r"(t[k][1]), "+r"(t[k][2]), "+r"(t[k][3]) : "r"(t[(k+1)%ILP][3]), "r"(t[(k+1)%ILP][0]), "r"(b2), "r"(b3));
  }
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < ILP; k++) s ^= t[k][0] ^ t[k][1] ^ t[k][2] ^ t[k][3];
  if (s == 0x1234567) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// ---- 6. mixed: 1 IMAD.WIDE + 1 LOP3 per step (pipe overlap check)
__global__ void k_mixed(uint64_t* out, uint32_t seed, int iters, long long* cyc) {
  uint64_t acc[ILP]; uint32_t x[ILP]; uint32_t a = seed ^ threadIdx.x, b = seed * 7u + blockIdx.x;
#pragma unroll
  for (int k = 0; k < ILP; k++) { acc[k] = k + threadIdx.x; x[k] = k * 3; }
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int k = 0; k < ILP; k++) {
      asm volatile("{\n\t.reg .u32 l, h;\n\tmov.b64 {l, h}, %1;\n\tmad.wide.u32 %0, h, %2, %0;\n\t}" : "+l"(acc[k]) : "l"(acc[(k+1)%ILP]), "r"(b));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[k]) : "r"((uint32_t)acc[k]), "r"(x[(k+1)%ILP]));
    }
  }
  long long t1 = clock64();
  uint64_t s = 0;
#pragma unroll
  for (int k = 0; k < ILP; k++) s ^= acc[k] ^ x[k];
  if (s == 0x1234567) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

typedef void (*kfn)(uint64_t*, uint32_t, int, long long*);
struct K { const char* name; kfn f; double ops_per_step; const char* unit; };

// Every kernel is launched as exactly one wave (SMs x its measured occupancy), then re-launched
// back to back for >= 1 s of wall time (sustained clocks); tools/micro/int_peak.py reads the
// NVML clock samples of each kernel's [t_begin, t_end] window.  ops_per_clk_per_sm is
// computed from clock64 with the ACTUAL resident blocks per SM (round 1 assumed 8).
static double now_s() {
  timespec ts; clock_gettime(CLOCK_REALTIME, &ts); return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

int main(int argc, char** argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  const double min_s = argc > 1 ? atof(argv[1]) : 1.5;
  printf("{\"device\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"smem_per_sm\":%zu,\"regs_per_sm\":%d}\n", p.name, sms, p.l2CacheSize, p.sharedMemPerMultiprocessor, p.regsPerMultiprocessor);
  K ks[] = {
    {"imad_wide_u32", k_imad_wide, ILP, "32x32->64 products"},
    {"imad_hi_u32", k_imad_hi, ILP, "mul.hi"},
    {"imad_lo_u32", k_imad_lo, ILP, "mul.lo"},
    {"imad_wide_cc_chain", k_imad_wide_cc, 2.0 * ILP, "32x32->64 products (carry chain)"},
    {"iadd_cc_chain", k_iadd_cc, 4.0 * ILP, "32-bit adds with carry"},
    {"mixed_wide_lop3", k_mixed, ILP, "IMAD.WIDE (+1 LOP3 each)"},
  };
  uint64_t* d_out; long long* d_cyc; CK(cudaMalloc(&d_out, 8));
  const int threads = 256; const int iters = 4096;
  CK(cudaMalloc(&d_cyc, sizeof(long long) * sms * 32));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (auto& k : ks) {
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k.f, threads, 0));
    const int blocks = sms * occ;
    for (int w = 0; w < 3; w++) k.f<<<blocks, threads>>>(d_out, 1234u, iters, d_cyc);
    CK(cudaDeviceSynchronize());
    // sustained: back-to-back launches for >= min_s seconds
    const double t_begin = now_s();
    long launches = 0; float total_ms = 0.f;
    while (total_ms < 1e3 * min_s) {
      cudaEventRecord(e0);
      for (int r = 0; r < 50; r++) k.f<<<blocks, threads>>>(d_out, 1234u, iters, d_cyc);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
      total_ms += ms; launches += 50;
    }
    const double t_end = now_s();
    std::vector<long long> cyc(blocks);
    CK(cudaMemcpy(cyc.data(), d_cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost));
    std::sort(cyc.begin(), cyc.end());
    const double ops = (double)launches * blocks * threads * iters * k.ops_per_step;
    const double rate = ops / (total_ms * 1e-3);
    // one wave: each SM runs `occ` blocks concurrently over the median block's clock64 span
    const double med_cyc = (double)cyc[blocks / 2];
    const double per_sm_clk = (double)occ * threads * iters * k.ops_per_step / med_cyc;
    printf("{\"kernel\":\"%s\",\"unit\":\"%s\",\"blocks_per_sm\":%d,\"launches\":%ld,\"seconds\":%.3f,\"ops_per_s\":%.4e,"
           "\"ops_per_clk_per_sm\":%.3f,\"implied_mhz\":%.0f,\"t_begin\":%.3f,\"t_end\":%.3f}\n",
           k.name, k.unit, occ, launches, total_ms * 1e-3, rate, per_sm_clk, rate / (per_sm_clk * sms) / 1e6, t_begin, t_end);
    fflush(stdout);
  }
  return 0;
}
