// coll.cu -- native allreduce kernel (see coll.hpp).
#include <algorithm>

#include "coll.hpp"
#include "mpx.h"

namespace mpx {

namespace {

template <typename T, typename A>
__global__ void __launch_bounds__(256)
k_allreduce_oneshot(const CollTable* __restrict__ tab, int n, int64_t lo, int64_t hi) {
    __shared__ const T* src[kMaxCollRanks];
    __shared__ T* dst[kMaxCollRanks];
    if (threadIdx.x < n) {   // volatile: the slot is rewritten by later calls
        const volatile CollTable* vt = tab;
        src[threadIdx.x] = static_cast<const T*>(const_cast<const void*>(vt->send[threadIdx.x]));
        dst[threadIdx.x] = static_cast<T*>(const_cast<void*>(vt->recv[threadIdx.x]));
    }
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += stride) {
        A acc = (A)src[0][i];
        for (int j = 1; j < n; ++j) acc += (A)src[j][i];
        const T out = (T)acc;
        for (int j = 0; j < n; ++j) dst[j][i] = out;
    }
}

int sms(int device) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    return v > 0 ? v : 148;
}

}  // namespace

cudaError_t preload_coll_kernels() {
    cudaFuncAttributes a;
    cudaError_t e = cudaSuccess, r;
    if ((r = cudaFuncGetAttributes(&a, k_allreduce_oneshot<int32_t, uint32_t>)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_allreduce_oneshot<long long, unsigned long long>)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_allreduce_oneshot<float, double>)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_allreduce_oneshot<double, double>)) != cudaSuccess) e = r;
    return e;
}

cudaError_t launch_allreduce_oneshot(const CollTable* table, int n, int rank, int64_t count, int dtype_code,
                                     int device, cudaStream_t stream) {
    const int64_t chunk = (count + n - 1) / n;
    const int64_t lo = std::min<int64_t>(count, (int64_t)rank * chunk);
    const int64_t hi = std::min<int64_t>(count, lo + chunk);
    if (hi <= lo) return cudaSuccess;
    const int64_t want = (hi - lo + 255) / 256;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms(device) * 8));
    switch (dtype_code) {
    case MPX_INT32:
        k_allreduce_oneshot<int32_t, uint32_t><<<grid, 256, 0, stream>>>(table, n, lo, hi);
        break;
    case MPX_INT64:
        k_allreduce_oneshot<long long, unsigned long long><<<grid, 256, 0, stream>>>(table, n, lo, hi);
        break;
    case MPX_FLOAT32:
        k_allreduce_oneshot<float, double><<<grid, 256, 0, stream>>>(table, n, lo, hi);
        break;
    default:
        k_allreduce_oneshot<double, double><<<grid, 256, 0, stream>>>(table, n, lo, hi);
        break;
    }
    return cudaGetLastError();
}

}  // namespace mpx
