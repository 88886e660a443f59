// kernels.hpp -- launch interface of the pack/unpack/iov kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "desc.cuh"
#include "plan.hpp"

namespace mpx {

constexpr int kMaxJobs = 16;

enum ChainMode : int32_t { CHAIN_ELEM = 0, CHAIN_ROW = 1, CHAIN_WIDE = 2 };

struct ChainJob {
    Chain c;
    const uint8_t* src;
    uint8_t* dst;
    int64_t rows;     // whole rows moved by the main path
    int64_t limit;    // packed bytes to move (unpack may stop mid-row: bytewise tail)
    int32_t w;        // element mode: word width in bytes
    int32_t mode;     // CHAIN_ELEM: thread per row; CHAIN_ROW: warp per row, 16 B + funnel;
                      // CHAIN_WIDE: thread per short row, aligned 16 B chunks on both sides
    int32_t blk0;     // first block of this job's interleave group (launcher)
    int32_t nblk;     // blocks of this job (launcher)
    int32_t gsize;    // jobs in the group; group blocks alternate between them
    int32_t gpos;     // this job's position in the group
    uint32_t m_g;     // magic divisor for gsize (32-bit, see host_magic32)
    int32_t s_g;
};

struct ChainBatch {
    int32_t njobs;
    int32_t pad;
    ChainJob job[kMaxJobs];
};

// fill mode / word width / row counts of a chain job from its plan and pointers
void chain_setup(const Plan& p, bool pack, ChainJob* j);

cudaError_t launch_chain_batch(ChainBatch& b, bool pack, int device, cudaStream_t stream);
cudaError_t launch_generic(const Plan& p, bool pack, const uint8_t* src, uint8_t* dst, int64_t limit,
                           cudaStream_t stream);
cudaError_t launch_span(const Plan& p, bool pack, const uint8_t* src, uint8_t* dst, int64_t limit,
                        cudaStream_t stream);
cudaError_t launch_runs(const Plan& p, bool pack, const uint8_t* src, uint8_t* dst, int64_t limit,
                        cudaStream_t stream);
// typed -> typed in one pass for two chain plans (copy_between, datatype.py:760-797)
cudaError_t launch_zip(const Plan& ps, const Plan& pd, const uint8_t* src, uint8_t* dst, int64_t bytes,
                       cudaStream_t stream);
cudaError_t launch_iov(const Plan& p, int64_t k0, int64_t n, int64_t* out, cudaStream_t stream);
// word-gather pack/unpack of span plans with PermSpecs (k_perm.cu)
cudaError_t launch_perm(const Plan& p, bool pack, const uint8_t* src, uint8_t* dst, int64_t limit,
                        cudaStream_t stream);
// force-load the pack/unpack/iov kernels on the current device (lazy loading)
// one warp polls *flag >= gen (volatile, nanosleep back-off): a stream wait
// that occupies one CTA slot instead of the stream's host-interface channel
cudaError_t launch_flag_wait(const uint32_t* flag, uint32_t gen, cudaStream_t stream);
cudaError_t preload_pack_kernels();
cudaError_t preload_perm_kernels();
int sm_count(int device);

}  // namespace mpx
