// kernels.hpp -- launch interface of the pack/unpack/iov kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "desc.cuh"
#include "plan.hpp"

namespace mpx {

constexpr int kMaxJobs = 16;

struct ChainJob {
    Chain c;
    const uint8_t* src;
    uint8_t* dst;
    int64_t nwords;   // whole W-byte words to move
    int64_t limit;    // packed bytes to move (unpack may stop mid-word)
    int32_t w;        // word width in bytes
    int32_t blk0;     // first block of this job (filled by the launcher)
    int32_t nblk;     // blocks of this job (filled by the launcher)
    int32_t pad;
};

struct ChainBatch {
    int32_t njobs;
    int32_t pad;
    ChainJob job[kMaxJobs];
};

// widest word (<= plan alignment) that both pointers are aligned to
int chain_word(const Plan& p, const void* a, const void* b);

cudaError_t launch_chain_batch(ChainBatch& b, bool pack, int device, cudaStream_t stream);
cudaError_t launch_generic(const Plan& p, bool pack, const uint8_t* src, uint8_t* dst, int64_t limit,
                           cudaStream_t stream);
cudaError_t launch_iov(const Plan& p, int64_t k0, int64_t n, int64_t* out, cudaStream_t stream);

}  // namespace mpx
