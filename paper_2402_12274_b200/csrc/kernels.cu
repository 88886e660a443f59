// kernels.cu -- sm_100a pack / unpack / iov kernels.
//
// Pure data movement: no tensor cores.  Three families:
//
//  k_chain    closed-form strided copy for Rep^k(Run) layouts (vector, hvector,
//             subarray faces, contiguous).  One thread per W-byte word of the
//             packed stream (W = 16/8/4/2/1 chosen from the alignment of base,
//             strides, run length and both pointers), UNR independent words in
//             flight per thread, packed side perfectly coalesced.  A batch of up
//             to kMaxJobs layouts is fused into one launch (e.g. all six halo
//             faces), blocks partitioned across jobs by size.
//  k_generic  descriptor walk for arbitrary trees (struct / indexed / nested):
//             each warp owns a 4 KiB tile of the packed stream staged in shared
//             memory; lanes locate 32 consecutive runs in parallel (tree
//             descent by run index), then gather (pack) or scatter (unpack) the
//             tile's bytes with lane-contiguous accesses; the packed side moves
//             as 16-byte vectors.
//  k_ordered  unpack for layouts whose runs may overlap: one warp, runs in
//             traversal order, so the last writer wins exactly as in the
//             reference (datatype.py:705-728).
//  k_iov      (offset, length) pairs of runs [k0, k0+n) (type_iov).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>

#include "desc.cuh"
#include "kernels.hpp"

namespace mpx {

namespace {

template <int W> struct Vec;
template <> struct Vec<16> { using T = uint4; };
template <> struct Vec<8> { using T = uint2; };
template <> struct Vec<4> { using T = uint32_t; };
template <> struct Vec<2> { using T = uint16_t; };
template <> struct Vec<1> { using T = uint8_t; };

constexpr int kChainThreads = 256;
constexpr int kUnroll = 4;

template <int W, bool PACK>
__device__ __forceinline__ void chain_job_body(const ChainJob& j, int64_t blk, int64_t nblk) {
    using T = typename Vec<W>::T;
    const Chain& c = j.c;
    const int64_t T_ = nblk * kChainThreads;
    const int64_t nw = j.nwords;
    for (int64_t u = blk * kChainThreads + threadIdx.x; u < nw; u += T_ * kUnroll) {
        T v[kUnroll];
        int64_t lo[kUnroll];
#pragma unroll
        for (int q = 0; q < kUnroll; ++q) {
            const int64_t uu = u + q * T_;
            if (uu < nw) {
                const int64_t P = uu * W;
                lo[q] = chain_off(c, P);
                if (PACK) v[q] = *reinterpret_cast<const T*>(j.src + lo[q]);
                else v[q] = *reinterpret_cast<const T*>(j.src + P);
            }
        }
#pragma unroll
        for (int q = 0; q < kUnroll; ++q) {
            const int64_t uu = u + q * T_;
            if (uu < nw) {
                const int64_t P = uu * W;
                if (PACK) *reinterpret_cast<T*>(j.dst + P) = v[q];
                else *reinterpret_cast<T*>(j.dst + lo[q]) = v[q];
            }
        }
    }
    // unpack with a partial last word (data shorter than the layout): bytewise tail
    if (!PACK && blk == 0 && threadIdx.x == 0) {
        for (int64_t P = nw * W; P < j.limit; ++P) j.dst[chain_off(c, P)] = j.src[P];
    }
}

template <bool PACK>
__global__ void __launch_bounds__(kChainThreads) k_chain(const ChainBatch b) {
    int ji = 0;
    while (ji + 1 < b.njobs && (int)blockIdx.x >= b.job[ji + 1].blk0) ++ji;
    const ChainJob& j = b.job[ji];
    const int64_t blk = blockIdx.x - j.blk0;
    switch (j.w) {
    case 16: chain_job_body<16, PACK>(j, blk, j.nblk); break;
    case 8: chain_job_body<8, PACK>(j, blk, j.nblk); break;
    case 4: chain_job_body<4, PACK>(j, blk, j.nblk); break;
    case 2: chain_job_body<2, PACK>(j, blk, j.nblk); break;
    default: chain_job_body<1, PACK>(j, blk, j.nblk); break;
    }
}

// ---------------------------------------------------------------- generic
constexpr int kGenWarps = 8;
constexpr int kTile = 4096;
constexpr size_t kGenSmem = size_t(kGenWarps) * kTile + size_t(kGenWarps) * 96 * sizeof(int64_t);

__device__ __forceinline__ void tile_copy(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                                          int n, int lane) {
    if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
        const int nv = n >> 4;
        for (int i = lane; i < nv; i += 32)
            reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
        for (int i = (nv << 4) + lane; i < n; i += 32) dst[i] = src[i];
    } else {
        for (int i = lane; i < n; i += 32) dst[i] = src[i];
    }
}

template <bool PACK>
__global__ void __launch_bounds__(kGenWarps * 32)
k_generic(const DDesc d, const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t limit) {
    extern __shared__ __align__(16) uint8_t sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* tb = sm + warp * kTile;
    int64_t* tpo = reinterpret_cast<int64_t*>(sm + kGenWarps * kTile) + warp * 96;
    int64_t* tso = tpo + 32;
    int64_t* tln = tpo + 64;
    const int64_t ntiles = (limit + kTile - 1) / kTile;
    for (int64_t t = (int64_t)blockIdx.x * kGenWarps + warp; t < ntiles;
         t += (int64_t)gridDim.x * kGenWarps) {
        const int64_t P0 = t * kTile;
        const int64_t P1 = min(P0 + kTile, limit);
        const int n = (int)(P1 - P0);
        if (!PACK) {
            tile_copy(tb, src + P0, n, lane);
            __syncwarp();
        }
        int64_t kb = locate_byte(d, P0).k;
        for (;;) {
            const int64_t k = kb + lane;
            if (k < d.runs) {
                const RunLoc r = locate_run(d, k);
                tpo[lane] = r.poff;
                tso[lane] = r.src;
                tln[lane] = r.len;
            }
            __syncwarp();
            const int last = (int)min((int64_t)31, d.runs - 1 - kb);
            const int64_t bhi = tpo[last] + tln[last];
            const int64_t lo = max(P0, tpo[0]);
            const int64_t hi = min(P1, bhi);
            int jj = 0;
            for (int64_t p = lo + lane; p < hi; p += 32) {
                while (jj < last && tpo[jj + 1] <= p) ++jj;
                const int64_t a = tso[jj] + (p - tpo[jj]);
                if (PACK) tb[p - P0] = src[a];
                else dst[a] = tb[p - P0];
            }
            __syncwarp();
            if (bhi >= P1 || kb + 32 >= d.runs) break;
            kb += 32;
        }
        if (PACK) tile_copy(dst + P0, tb, n, lane);
        __syncwarp();
    }
}

// ------------------------------------------------------- ordered unpack
__global__ void __launch_bounds__(32)
k_ordered_unpack(const DDesc d, const uint8_t* __restrict__ src, uint8_t* dst, int64_t limit) {
    const int lane = threadIdx.x & 31;
    for (int64_t kb = 0; kb < d.runs; kb += 32) {
        RunLoc mine{0, 0, 0, LLONG_MAX};
        if (kb + lane < d.runs) mine = locate_run(d, kb + lane);
        const int cnt = (int)min((int64_t)32, d.runs - kb);
        for (int j = 0; j < cnt; ++j) {
            const int64_t so = __shfl_sync(0xffffffffu, mine.src, j);
            const int64_t ln = __shfl_sync(0xffffffffu, mine.len, j);
            const int64_t po = __shfl_sync(0xffffffffu, mine.poff, j);
            if (po >= limit) return;
            const int64_t take = min(ln, limit - po);
            for (int64_t x = lane; x < take; x += 32) dst[so + x] = src[po + x];
            __syncwarp();
        }
    }
}

// ---------------------------------------------------------------- iov
__global__ void __launch_bounds__(256)
k_iov(const DDesc d, int64_t k0, int64_t n, int64_t* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const RunLoc r = locate_run(d, k0 + i);
        reinterpret_cast<longlong2*>(out)[i] = make_longlong2(r.src, r.len);
    }
}

int sm_count(int device) {
    static int cached[64] = {0};
    if (device < 0 || device >= 64) return 148;
    if (!cached[device]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
        cached[device] = v > 0 ? v : 148;
    }
    return cached[device];
}

}  // namespace

int chain_word(const Plan& p, const void* a, const void* b) {
    int64_t w = p.chain_align;
    const uintptr_t m = reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b);
    while (w > 1 && (m & (uintptr_t)(w - 1))) w >>= 1;
    return (int)w;
}

cudaError_t launch_chain_batch(ChainBatch& b, bool pack, int device, cudaStream_t stream) {
    if (b.njobs == 0) return cudaSuccess;
    // blocks per job proportional to words, capped so one wave of the batch
    // covers ~8 CTAs per SM
    const int64_t cap = (int64_t)sm_count(device) * 8;
    int64_t total = 0;
    for (int i = 0; i < b.njobs; ++i) {
        ChainJob& j = b.job[i];
        const int64_t want = (j.nwords + (int64_t)kChainThreads * kUnroll - 1) / ((int64_t)kChainThreads * kUnroll);
        j.nblk = (int32_t)std::max<int64_t>(1, std::min<int64_t>(want, cap));
        j.blk0 = (int32_t)total;
        total += j.nblk;
    }
    if (pack) k_chain<true><<<(unsigned)total, kChainThreads, 0, stream>>>(b);
    else k_chain<false><<<(unsigned)total, kChainThreads, 0, stream>>>(b);
    return cudaGetLastError();
}

cudaError_t launch_generic(const Plan& p, bool pack, const uint8_t* src, uint8_t* dst, int64_t limit,
                           cudaStream_t stream) {
    if (limit <= 0) return cudaSuccess;
    if (!pack && p.overlap) {
        k_ordered_unpack<<<1, 32, 0, stream>>>(p.desc, src, dst, limit);
        return cudaGetLastError();
    }
    const int64_t tiles = (limit + kTile - 1) / kTile;
    const int64_t want = (tiles + kGenWarps - 1) / kGenWarps;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count(p.device) * 6));
    if (pack) k_generic<true><<<(unsigned)grid, kGenWarps * 32, kGenSmem, stream>>>(p.desc, src, dst, limit);
    else k_generic<false><<<(unsigned)grid, kGenWarps * 32, kGenSmem, stream>>>(p.desc, src, dst, limit);
    return cudaGetLastError();
}

cudaError_t launch_iov(const Plan& p, int64_t k0, int64_t n, int64_t* out, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    const int64_t want = (n + 255) / 256;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count(p.device) * 16));
    k_iov<<<(unsigned)grid, 256, 0, stream>>>(p.desc, k0, n, out);
    return cudaGetLastError();
}

}  // namespace mpx
