// capi_common.hpp -- helpers shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <string>

#include "mpx.h"
#include "plan.hpp"
#include "typerep.hpp"

namespace mpx {

extern thread_local std::string g_last_error;

// record a message for mpx_last_error() and return code
int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int cuda_fail(cudaError_t e, const char* what);

// handle -> live Datatype (nullptr when the handle is unknown)
Datatype* lookup(mpx_datatype h);

// validate a typed buffer and fetch its plan on the buffer's device
// (other_buf = the packed-side buffer, used to pick the execution device;
// pinned host buffers are addressed zero-copy)
int prepare(Datatype* d, int64_t count, const void* layout_buf, int64_t layout_bytes, const void* other_buf,
            cudaStream_t stream, std::shared_ptr<Plan>* plan, int* device);

// n fused pack (or unpack) operations on one stream
int movement(int n, const mpx_datatype* dts, const int64_t* counts, const void* const* srcs,
             const int64_t* src_bytes, void* const* dsts, const int64_t* dst_bytes, bool pack,
             cudaStream_t stream, int64_t* written_out);

// single pack/unpack of `limit` packed bytes executed on device `dev` (peer or
// pinned-host pointers allowed)
int launch_move(int dev, Datatype* d, int64_t count, bool pack, const void* src, void* dst, int64_t limit,
                cudaStream_t stream);
// typed -> typed transfer of `bytes` packed bytes in one pass (both layouts
// chains, destination without overlaps); MPX_ERR_PENDING when not applicable
int launch_zip_move(int dev, Datatype* sd, int64_t scount, const void* src, Datatype* rd, int64_t rcount, void* dst,
                    int64_t bytes, cudaStream_t stream);
// layout_for(count) is one run -> its offset
bool contiguous_run(Datatype* d, int64_t count, int64_t* off);
// count / usability / bounds checks of a typed buffer of `bytes` bytes
int check_layout_region(Datatype* d, int64_t count, int64_t bytes);
int set_device(int dev);

}  // namespace mpx
