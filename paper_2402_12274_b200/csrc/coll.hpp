// coll.hpp -- native stream-ordered allreduce (rank-ordered one-shot kernel).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace mpx {

constexpr int kMaxCollRanks = 64;

constexpr int kCollSlots = 64;

// per-call pointer table in device memory (one copy per participating
// device); each rank's STREAM writes its two pointers with 64-bit stream
// memops before its "arrived" flag, so a slot is only rewritten once every
// rank's stream is past the previous use
struct CollTable {
    const void* send[kMaxCollRanks];
    void* recv[kMaxCollRanks];
};

// ring of collective slots of one communicator context
struct CollRing {
    CollTable table[kCollSlots];
    uint32_t arrive[kCollSlots][kMaxCollRanks];
    uint32_t finish[kCollSlots][kMaxCollRanks];
};

// Rank `rank` of `n` reduces its 1/n slice of the buffers: out = x0 + x1 + ...
// + x(n-1) in rank order (comm.py:582-588), accumulated in double for float
// types and in wrapping unsigned arithmetic for integers, and writes the
// result into every rank's receive buffer (peer stores over NVLink).
cudaError_t launch_allreduce_oneshot(const CollTable* table, int n, int rank, int64_t count, int dtype_code,
                                     int device, cudaStream_t stream);

// Same reduction with the n buffer pairs passed by value (multi-process
// worlds: the pointers are this process's mappings of the peers' buffers,
// known on the host at enqueue time).
constexpr int kMaxDirectRanks = 16;
cudaError_t launch_allreduce_direct(const void* const* send, void* const* recv, int n, int rank, int64_t count,
                                    int dtype_code, int device, cudaStream_t stream);

cudaError_t preload_coll_kernels();

}  // namespace mpx
