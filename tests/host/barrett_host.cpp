// Host build of the product Barrett code (paper_2509_12494_b200/csrc/barrett128.cuh) for
// tests/test_barrett_host.py: the CUDA path's arithmetic, compiled for the CPU and checked
// against Python integers (this is not the oracle; the oracle shares no code with it).
#include "../../paper_2509_12494_b200/csrc/barrett128.cuh"
extern "C" void barrett_mul_batch(const uint32_t* a, const uint32_t* b, const uint32_t* q, const uint32_t* mu,
                                  uint32_t* r, long n) {
    ntt128::BarrettC c;
    for (int k = 0; k < 4; k++) { c.q[k] = q[k]; c.mu[k] = mu[k]; }
    for (long i = 0; i < n; i++) ntt128::barrett_mul(a + 4 * i, b + 4 * i, c, r + 4 * i);
}
