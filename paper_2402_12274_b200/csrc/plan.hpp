// plan.hpp -- lowering of a layout tree to a GPU execution plan.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "desc.cuh"
#include "typerep.hpp"

#include <cstdio>
#include <cstdlib>
#include <thread>

// MPX_TRACE=1: host-side progress markers on stderr (diagnosing stalls)
inline bool mpx_tracing() {
    static const bool on = std::getenv("MPX_TRACE") != nullptr;
    return on;
}
#define MPX_TRACE(...)                                                                        \
    do {                                                                                      \
        if (mpx_tracing()) {                                                                  \
            char mpx_tb_[320];                                                                \
            int mpx_tn_ = std::snprintf(mpx_tb_, sizeof mpx_tb_, "[mpx %04zx] ",               \
                                        std::hash<std::thread::id>()(std::this_thread::get_id()) & 0xffff); \
            mpx_tn_ += std::snprintf(mpx_tb_ + mpx_tn_, sizeof mpx_tb_ - mpx_tn_, __VA_ARGS__); \
            if (mpx_tn_ > (int)sizeof mpx_tb_ - 2) mpx_tn_ = (int)sizeof mpx_tb_ - 2;         \
            mpx_tb_[mpx_tn_++] = '\n';                                                        \
            std::fwrite(mpx_tb_, 1, (size_t)mpx_tn_, stderr);                                  \
        }                                                                                     \
    } while (0)

namespace mpx {

enum PlanKind : int32_t { PLAN_EMPTY = 0, PLAN_CHAIN = 1, PLAN_GENERIC = 2, PLAN_SPAN = 3, PLAN_RUNS = 4 };

// Flat run table for irregular layouts of many small runs (e.g. indexed types
// with thousands of short blocks): run r = layout bytes [src[r], src[r] +
// pk[r + 1] - pk[r]) at packed offset pk[r].  Runs longer than kRunPiece are
// split into pieces (then `split` is set and type_iov walks the descriptor).
constexpr int64_t kRunPiece = 512;
constexpr int64_t kMaxTableRuns = int64_t(1) << 23;

struct RunTable {
    const int64_t* src;
    const int64_t* pk;      // nruns + 1 entries
    int64_t nruns;
    int32_t g;              // largest power of two <= 16 dividing every offset and length
    int32_t split;
    int64_t avg_words;      // average run length in g-byte words (>= 16: warp per run)
};

struct Plan {
    int32_t kind = PLAN_EMPTY;
    int device = -1;
    int64_t runs = 0, nbytes = 0, min_off = 0, max_end = 0, node_count = 1;
    bool overlap = false;   // unpack must keep traversal order (last writer wins)
    Chain chain{};          // valid for PLAN_CHAIN
    int32_t chain_align = 16;  // largest power of two dividing base, L and strides
    DDesc desc{};           // device descriptor (always built, used by iov + generic)
    SpanPlan span{};        // valid for PLAN_SPAN (pointers into blob)
    RunTable rt{};          // valid for PLAN_RUNS (pointers into blob)
    std::vector<SpanChunk> span_chunks;   // host copies, uploaded with the descriptor
    std::vector<SpanBody> span_bodies;
    std::vector<PermSpec> perm_specs;     // host copies; tab = offset into perm_tab until upload
    std::vector<PermEntry> perm_tab;
    // per direction: (spec << 6 | layout phase << 2 | packed phase) of the
    // chunks (phases mod 4 relative to the buffers; bit 5 / bit 4: any
    // layout / packed phase)
    std::vector<int32_t> perm_use[2];
    std::vector<int64_t> span_iov;        // {segment prefix, raw run length} per chunk
    void* blob = nullptr;   // device allocation backing desc
    size_t blob_bytes = 0;
    cudaEvent_t ready = nullptr;     // upload finished (recorded on an internal stream)
    std::atomic<bool> ready_seen{false};
    ~Plan();
};

// make `stream` wait for the plan's descriptor upload (no-op once observed done)
cudaError_t plan_wait(Plan& p, cudaStream_t stream);

// Build (or fetch from the datatype's cache) the plan for (layout_for(count), device).
std::shared_ptr<Plan> get_plan(Datatype* dt, int64_t count, int device, cudaStream_t stream,
                               std::string* err);

// Lower one layout on the host (no device allocation); used by tests via the C ABI.
void analyze(const Node* layout, Plan* p);

}  // namespace mpx
