// ntt128_internal.h -- library-internal entry between the plan executor (ntt128.cu) and the
// distributed four-step (fourstep.cu).  Not part of the C ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/ntt128.h"

#ifndef NTT128_FS_MAX_RANKS
#define NTT128_FS_MAX_RANKS 8   // ranks of a distributed four-step (one box: <= 8 GPUs)
#endif

// Non-natural input / output of one batched cyclic transform (fourstep.cu):
//  * the first pass reads element idx of polynomial p at src[p in_ps + idx in_es]
//    (in_ps == 0: the natural [batch][N] layout);
//  * fin (optional): per-polynomial factors (Montgomery form), that of input idx of
//    polynomial p at fin[p fin_ps + idx fin_es], multiplied in as the first pass loads it;
//  * r_lb != 0: the last pass stores output k of polynomial p at
//    rdst[k >> r_lb] + p r_ps + (k mod 2^r_lb); a multi-pass transform then works in `tmp`
//    ([batch][N], natural) until its last pass.
struct Ntt128IO {
    uint64_t in_ps = 0, in_es = 1;
    const uint4* fin = nullptr;
    uint64_t fin_ps = 0, fin_es = 1;
    uint32_t r_lb = 0;
    uint64_t r_ps = 0;
    uint4* rdst[NTT128_FS_MAX_RANKS] = {};
    uint4* tmp = nullptr;
};

// NTT128_FLAG_CHAIN bookkeeping (ntt128.cu): every public entry point that enqueues device
// work takes its stream's next library generation (no-op while no chained plan exists).
void ntt128_stream_gen(cudaStream_t stream, uint64_t* prev, uint64_t* now);

ntt128_status ntt128_transform_io(ntt128_plan_t p, const uint4* src, uint4* dst, cudaStream_t stream, bool inverse,
                                  const Ntt128IO& io);
