// coll.cu -- native allreduce kernel (see coll.hpp).
#include <algorithm>
#include <cstdint>

#include "coll.hpp"
#include "mpx.h"

namespace mpx {

namespace {

template <typename T, typename A>
__device__ __forceinline__ void reduce_one(const T* const* src, T* const* dst, int n, int64_t i) {
    A acc = (A)src[0][i];
    for (int j = 1; j < n; ++j) acc += (A)src[j][i];
    const T out = (T)acc;
    for (int j = 0; j < n; ++j) dst[j][i] = out;
}

// 16-byte vector form: V = 16 / sizeof(T) elements per access.  The loads of
// up to 8 ranks are issued together (peer loads over NVLink have ~us latency),
// then summed in rank order -- the reference's x0 + x1 + ... order.
template <typename T, typename A>
__device__ __forceinline__ void reduce_vec(const T* const* src, T* const* dst, int n, int64_t v) {
    constexpr int V = 16 / sizeof(T);
    constexpr int B = 8;
    union U { uint4 q; T e[V]; };
    A acc[V];
#pragma unroll
    for (int k = 0; k < V; ++k) acc[k] = (A)0;
    for (int j0 = 0; j0 < n; j0 += B) {
        U u[B];
#pragma unroll
        for (int b = 0; b < B; ++b)
            if (j0 + b < n) u[b].q = __ldg(reinterpret_cast<const uint4*>(src[j0 + b]) + v);
#pragma unroll
        for (int b = 0; b < B; ++b) {
            if (j0 + b >= n) break;
#pragma unroll
            for (int k = 0; k < V; ++k) acc[k] = (j0 + b == 0) ? (A)u[b].e[k] : acc[k] + (A)u[b].e[k];
        }
    }
    U u;
#pragma unroll
    for (int k = 0; k < V; ++k) u.e[k] = (T)acc[k];
    for (int j = 0; j < n; ++j) reinterpret_cast<uint4*>(dst[j])[v] = u.q;
}

// slice [lo, hi) of the n buffers whose pointers are in shared memory
template <typename T, typename A>
__device__ __forceinline__ void reduce_slice(const T* const* src, T* const* dst, int n, int aligned, int64_t lo,
                                             int64_t hi) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    constexpr int V = 16 / sizeof(T);
    if (aligned) {
        const int64_t vlo = (lo + V - 1) / V, vhi = hi / V;
        for (int64_t v = vlo + t0; v < vhi; v += stride) reduce_vec<T, A>(src, dst, n, v);
        for (int64_t i = lo + t0; i < min(hi, vlo * V); i += stride) reduce_one<T, A>(src, dst, n, i);
        for (int64_t i = max(lo, vhi * V) + t0; i < hi; i += stride) reduce_one<T, A>(src, dst, n, i);
    } else {
        for (int64_t i = lo + t0; i < hi; i += stride) reduce_one<T, A>(src, dst, n, i);
    }
}

template <typename T, typename A>
__global__ void __launch_bounds__(256)
k_allreduce_oneshot(const CollTable* __restrict__ tab, int n, int64_t lo, int64_t hi) {
    __shared__ const T* src[kMaxCollRanks];
    __shared__ T* dst[kMaxCollRanks];
    __shared__ int aligned;
    if (threadIdx.x == 0) aligned = 1;
    __syncthreads();
    if (threadIdx.x < n) {   // volatile: the slot is rewritten by later calls
        const volatile CollTable* vt = tab;
        src[threadIdx.x] = static_cast<const T*>(const_cast<const void*>(vt->send[threadIdx.x]));
        dst[threadIdx.x] = static_cast<T*>(const_cast<void*>(vt->recv[threadIdx.x]));
        if (((reinterpret_cast<uintptr_t>(src[threadIdx.x]) | reinterpret_cast<uintptr_t>(dst[threadIdx.x])) & 15) != 0)
            aligned = 0;
    }
    __syncthreads();
    reduce_slice<T, A>(src, dst, n, aligned, lo, hi);
}

struct DirectPtrs {
    const void* send[kMaxDirectRanks];
    void* recv[kMaxDirectRanks];
};

template <typename T, typename A>
__global__ void __launch_bounds__(256)
k_allreduce_direct(const DirectPtrs p, int n, int64_t lo, int64_t hi) {
    __shared__ const T* src[kMaxDirectRanks];
    __shared__ T* dst[kMaxDirectRanks];
    __shared__ int aligned;
    if (threadIdx.x == 0) aligned = 1;
    __syncthreads();
    if (threadIdx.x < n) {
        src[threadIdx.x] = static_cast<const T*>(p.send[threadIdx.x]);
        dst[threadIdx.x] = static_cast<T*>(p.recv[threadIdx.x]);
        if (((reinterpret_cast<uintptr_t>(src[threadIdx.x]) | reinterpret_cast<uintptr_t>(dst[threadIdx.x])) & 15) != 0)
            aligned = 0;
    }
    __syncthreads();
    reduce_slice<T, A>(src, dst, n, aligned, lo, hi);
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
    if ((r = cudaFuncGetAttributes(&a, k_allreduce_direct<int32_t, uint32_t>)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_allreduce_direct<long long, unsigned long long>)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_allreduce_direct<float, double>)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_allreduce_direct<double, double>)) != cudaSuccess) e = r;
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

cudaError_t launch_allreduce_direct(const void* const* send, void* const* recv, int n, int rank, int64_t count,
                                    int dtype_code, int device, cudaStream_t stream) {
    if (n > kMaxDirectRanks) return cudaErrorInvalidValue;
    DirectPtrs p{};
    for (int j = 0; j < n; ++j) {
        p.send[j] = send[j];
        p.recv[j] = recv[j];
    }
    const int64_t chunk = (count + n - 1) / n;
    const int64_t lo = std::min<int64_t>(count, (int64_t)rank * chunk);
    const int64_t hi = std::min<int64_t>(count, lo + chunk);
    if (hi <= lo) return cudaSuccess;
    const int64_t want = (hi - lo + 255) / 256;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms(device) * 8));
    switch (dtype_code) {
    case MPX_INT32:
        k_allreduce_direct<int32_t, uint32_t><<<grid, 256, 0, stream>>>(p, n, lo, hi);
        break;
    case MPX_INT64:
        k_allreduce_direct<long long, unsigned long long><<<grid, 256, 0, stream>>>(p, n, lo, hi);
        break;
    case MPX_FLOAT32:
        k_allreduce_direct<float, double><<<grid, 256, 0, stream>>>(p, n, lo, hi);
        break;
    default:
        k_allreduce_direct<double, double><<<grid, 256, 0, stream>>>(p, n, lo, hi);
        break;
    }
    return cudaGetLastError();
}

}  // namespace mpx
