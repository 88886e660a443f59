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

// Chain kernels run 64-thread CTAs (A/B on one box, round 2, bench step =
// fused pack + unpack of the 12 halo faces): 256 threads 0.0767-0.0776 ms,
// 128 threads 0.0745-0.0751, 64 threads 0.0717-0.0718 with the caps below.
// Smaller CTAs retire and refill SMs at a finer grain, so the tail of the
// latency-bound x-face rows overlaps the y/z rows better; the vector(N/64,
// 32, 64) pack / unpack also gain (107.5 -> 87.6 / 98.4 -> 83.5 us) and the
// contiguous 256 MiB copy is unchanged (90.6 -> 89.2 us).  The
// MPX_* overrides exist for such A/B builds only (build.py MPX_NVCC_FLAGS).
#ifndef MPX_CHAIN_THREADS
#define MPX_CHAIN_THREADS 64
#endif
#ifndef MPX_PACK_MINB
#define MPX_PACK_MINB 24
#endif
constexpr int kChainThreads = MPX_CHAIN_THREADS;

// Scattered layout-side loads of short rows.  Measured on the fused halo
// pack (ncu, profiles/): L1-allocating loads 31.6 us, L2-only (.cg) 36.0 us,
// same DRAM bytes -- the 1- and 8-wide faces of a side reuse L1 lines.
#ifndef MPX_LAYOUT_LD
#define MPX_LAYOUT_LD 0
#endif
template <typename T>
__device__ __forceinline__ T ld_layout(const T* p) {
#if MPX_LAYOUT_LD == 1
    return __ldcg(p);
#elif MPX_LAYOUT_LD == 2
    return __ldcs(p);
#else
    return *p;
#endif
}

// bytes [a, a + 16) of the 32-byte concatenation lo || hi, 0 <= a < 16
__device__ __forceinline__ uint4 funnel16(const uint4& lo, const uint4& hi, int a) {
    const uint32_t w0 = lo.x, w1 = lo.y, w2 = lo.z, w3 = lo.w;
    const uint32_t w4 = hi.x, w5 = hi.y, w6 = hi.z, w7 = hi.w;
    const int r = (a & 3) * 8;
#define MPX_F(x, y) __funnelshift_r((x), (y), r)
    switch (a >> 2) {
    case 0: return make_uint4(MPX_F(w0, w1), MPX_F(w1, w2), MPX_F(w2, w3), MPX_F(w3, w4));
    case 1: return make_uint4(MPX_F(w1, w2), MPX_F(w2, w3), MPX_F(w3, w4), MPX_F(w4, w5));
    case 2: return make_uint4(MPX_F(w2, w3), MPX_F(w3, w4), MPX_F(w4, w5), MPX_F(w5, w6));
    default: return make_uint4(MPX_F(w3, w4), MPX_F(w4, w5), MPX_F(w5, w6), MPX_F(w6, w7));
    }
#undef MPX_F
}

__device__ __forceinline__ uint4 shfl_down16(const uint4& v, int d) {
    return make_uint4(__shfl_down_sync(0xffffffffu, v.x, d), __shfl_down_sync(0xffffffffu, v.y, d),
                      __shfl_down_sync(0xffffffffu, v.z, d), __shfl_down_sync(0xffffffffu, v.w, d));
}
__device__ __forceinline__ uint4 shfl_up16(const uint4& v, int d) {
    return make_uint4(__shfl_up_sync(0xffffffffu, v.x, d), __shfl_up_sync(0xffffffffu, v.y, d),
                      __shfl_up_sync(0xffffffffu, v.z, d), __shfl_up_sync(0xffffffffu, v.w, d));
}
__device__ __forceinline__ uint4 shfl16(const uint4& v, int src) {
    return make_uint4(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src),
                      __shfl_sync(0xffffffffu, v.z, src), __shfl_sync(0xffffffffu, v.w, src));
}

// store bytes [lo, hi) of v into the 16-byte aligned chunk at p
__device__ __forceinline__ void store_partial16(uint8_t* p, const uint4& v, int lo, int hi) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int b0 = 4 * i, b1 = 4 * i + 4;
        if (b0 >= lo && b1 <= hi) {
            *reinterpret_cast<uint32_t*>(p + b0) = w[i];
        } else {
#pragma unroll
            for (int b = b0; b < b1; ++b)
                if (b >= lo && b < hi) p[b] = (uint8_t)(w[i] >> (8 * (b - b0)));
        }
    }
}

// Unpack threads ask L2 for the destination line of a row (prefetch.global.L2)
// BEFORE loading the packed bytes: a partially written sector needs a DRAM
// fill, and issued this way the fill overlaps the load instead of trailing
// the store.  Measured on the bench step (A/B, round 2): fused unpack of the
// 12 halo faces 62.3 -> 52.1 us, same DRAM bytes.  MPX_UNPACK_PREFETCH=0 turns
// it off (experiments).
#ifndef MPX_UNPACK_PREFETCH
#define MPX_UNPACK_PREFETCH 1
#endif
__device__ __forceinline__ void prefetch_l2(const void* p) {
#if MPX_UNPACK_PREFETCH
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
#else
    (void)p;
#endif
}
// only the partially covered 32-byte sectors at the two ends of [d, d + len)
// need a fill; whole-sector writes never do (a prefetch there only costs:
// the vector(N/32,4,8) zipper, 32-byte aligned rows, slowed 0.146 -> 0.159 ms)
__device__ __forceinline__ void prefetch_partial(const uint8_t* d, int64_t len) {
    if (len <= 0) return;
    const uintptr_t a = reinterpret_cast<uintptr_t>(d), e = a + (uintptr_t)len;
    const bool head = (a & 31) != 0, tail = (e & 31) != 0;
    if (head) prefetch_l2(d);
    if (tail && (!head || ((e - 1) >> 5) != (a >> 5))) prefetch_l2(d + len - 1);
}

// Warp per row, 16-byte vectors on both sides.  The packed side is 16-byte
// aligned (L % 16 == 0); the layout side may start at any byte: aligned
// 16-byte loads (pack) or stores (unpack) are realigned with funnel shifts
// through neighbouring lanes, so no access is narrower than 16 bytes except
// the two partial chunks at the ends of an unpacked row.
// Work items are (row, piece): a piece is kRowPiece = 32 lanes x U x 16 B of a
// row, so long rows (a 64 MiB contiguous message is a single row) spread over
// the whole grid.
constexpr int kRowU = 4;
constexpr int kRowPieceChunks = 32 * kRowU;

template <bool PACK>
__device__ __forceinline__ void chain_rows(const ChainJob& j, int64_t warp0, int64_t nwarps) {
    const int lane = threadIdx.x & 31;
    const Chain& c = j.c;
    const int64_t nch = c.L >> 4;
    const int64_t npieces = (nch + kRowPieceChunks - 1) / kRowPieceChunks;
    const int64_t items = j.rows * npieces;
    for (int64_t it = warp0; it < items; it += nwarps) {
        const int64_t r = it / npieces;
        const int64_t k0 = (it - r * npieces) * kRowPieceChunks;
        const int64_t s = chain_row(c, r);
        if (PACK) {
            const uint8_t* srow = j.src + s;
            const int a = (int)(reinterpret_cast<uintptr_t>(srow) & 15);
            const uint4* s16 = reinterpret_cast<const uint4*>(srow - a);
            uint4* d16 = reinterpret_cast<uint4*>(j.dst + r * c.L);
            uint4 v[kRowU];
#pragma unroll
            for (int u = 0; u < kRowU; ++u) {
                const int64_t k = k0 + 32 * u + lane;
                v[u] = k < nch ? __ldg(s16 + k) : make_uint4(0, 0, 0, 0);
            }
            if (a) {
#pragma unroll
                for (int u = 0; u < kRowU; ++u) {
                    const int64_t k = k0 + 32 * u + lane;
                    uint4 c1 = shfl_down16(v[u], 1);
                    if (k < nch && (lane == 31 || k + 1 == nch)) c1 = __ldg(s16 + k + 1);
                    v[u] = funnel16(v[u], c1, a);
                }
            }
#pragma unroll
            for (int u = 0; u < kRowU; ++u) {
                const int64_t k = k0 + 32 * u + lane;
                if (k < nch) d16[k] = v[u];
            }
        } else {
            const uint4* p16 = reinterpret_cast<const uint4*>(j.src + r * c.L);
            uint8_t* drow = j.dst + s;
            const int a = (int)(reinterpret_cast<uintptr_t>(drow) & 15);
            uint8_t* d16 = drow - a;
            const int64_t nout = a ? nch + 1 : nch;
            if (a && lane == 0 && k0 == 0) prefetch_l2(d16);                       // partial first chunk
            if (a && lane == 31 && k0 + kRowPieceChunks >= nout) prefetch_l2(d16 + 16 * nch);   // partial last
            uint4 v[kRowU];
#pragma unroll
            for (int u = 0; u < kRowU; ++u) {
                const int64_t k = k0 + 32 * u + lane;
                v[u] = k < nch ? __ldg(p16 + k) : make_uint4(0, 0, 0, 0);
            }
            if (a == 0) {
#pragma unroll
                for (int u = 0; u < kRowU; ++u) {
                    const int64_t k = k0 + 32 * u + lane;
                    if (k < nch) reinterpret_cast<uint4*>(d16)[k] = v[u];
                }
                continue;
            }
            // the last piece also owns output chunk nch (the tail of the row)
            uint4 carry = (k0 > 0) ? __ldg(p16 + k0 - 1) : make_uint4(0, 0, 0, 0);
            const int64_t kend = min(k0 + (int64_t)kRowPieceChunks, nout);
#pragma unroll
            for (int u = 0; u < kRowU; ++u) {
                const int64_t k = k0 + 32 * u + lane;
                uint4 prev = shfl_up16(v[u], 1);
                if (lane == 0) prev = carry;
                carry = shfl16(v[u], 31);
                const uint4 out = funnel16(prev, v[u], 16 - a);
                if (k < kend) {
                    if (k == 0) store_partial16(d16, out, a, 16);
                    else if (k == nch) store_partial16(d16 + 16 * k, out, 0, a);
                    else reinterpret_cast<uint4*>(d16)[k] = out;
                }
            }
            // output chunk nch falls just past the last full piece
            if (nout > k0 + kRowPieceChunks && k0 + kRowPieceChunks == nch && lane == 0) {
                store_partial16(d16 + 16 * nch, funnel16(carry, make_uint4(0, 0, 0, 0), 16 - a), 0, a);
            }
        }
    }
}

// Thread per row (short rows): row offset computed once, W-byte words, four
// rows in flight per thread.
template <int W, bool PACK>
__device__ __forceinline__ void chain_elems(const ChainJob& j, int64_t t0, int64_t nthr) {
    using T = typename Vec<W>::T;
    const Chain& c = j.c;
    const int nw = (int)(c.L / W);
    constexpr int R = 4;
    for (int64_t r0 = t0; r0 < j.rows; r0 += nthr * R) {
        int64_t lo[R], po[R];
        bool ok[R];
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int64_t r = r0 + q * nthr;
            ok[q] = r < j.rows;
            lo[q] = ok[q] ? chain_row(c, r) : 0;
            po[q] = r * c.L;
            if (!PACK && ok[q]) prefetch_partial(j.dst + lo[q], c.L);
        }
        for (int w = 0; w < nw; ++w) {
            T v[R];
#pragma unroll
            for (int q = 0; q < R; ++q)
                if (ok[q])
                    v[q] = PACK ? ld_layout(reinterpret_cast<const T*>(j.src + lo[q] + w * W))
                                : *reinterpret_cast<const T*>(j.src + po[q] + w * W);
#pragma unroll
            for (int q = 0; q < R; ++q)
                if (ok[q]) *reinterpret_cast<T*>(j.dst + (PACK ? po[q] : lo[q]) + w * W) = v[q];
        }
    }
}

// Thread per short row (16 <= L <= 64, L % 16 == 0, rows 4-byte aligned,
// packed side 16-byte aligned): the row is moved as the aligned 16-byte
// chunks that cover it -- pack loads <= 5 chunks and realigns them with
// funnel shifts into L/16 full 16-byte packed stores; unpack loads L/16
// packed chunks and stores whole 16-byte chunks in the row's middle and
// 4-byte words at its two ends.  An x-face row of 8 floats at a 4 (mod 16)
// address takes 3 loads + 2 stores instead of 8 + 8 word accesses.
template <bool PACK>
__device__ __forceinline__ void chain_wide(const ChainJob& j, int64_t t0, int64_t nthr) {
    const Chain& c = j.c;
    const int nq = (int)(c.L >> 4);
    int64_t next_off = t0 < j.rows ? chain_row(c, t0) : 0;
    if (!PACK && t0 < j.rows) prefetch_partial(j.dst + next_off, c.L);
    for (int64_t r = t0; r < j.rows; r += nthr) {
        const int64_t off = next_off;
        if (r + nthr < j.rows) {   // the row this thread takes next: its fill starts now
            next_off = chain_row(c, r + nthr);
            if (!PACK) prefetch_partial(j.dst + next_off, c.L);
        }
        if (PACK) {
            const uint8_t* s = j.src + off;
            const int a = (int)(reinterpret_cast<uintptr_t>(s) & 15);
            const uint4* s16 = reinterpret_cast<const uint4*>(s - a);
            const int n16 = (a + (int)c.L + 15) >> 4;
            uint4 v[5];
#pragma unroll
            for (int i = 0; i < 5; ++i) v[i] = i < n16 ? ld_layout(s16 + i) : make_uint4(0, 0, 0, 0);
            uint4* d16 = reinterpret_cast<uint4*>(j.dst + r * c.L);
#pragma unroll
            for (int m = 0; m < 4; ++m)
                if (m < nq) d16[m] = funnel16(v[m], v[m + 1], a);
        } else {
            const uint4* p16 = reinterpret_cast<const uint4*>(j.src + r * c.L);
            uint8_t* d = j.dst + off;
            const int a = (int)(reinterpret_cast<uintptr_t>(d) & 15);
            uint8_t* d0 = d - a;
            const int end = a + (int)c.L;              // region bytes [a, end) of the chunks
            const int n16 = (end + 15) >> 4;
            uint4 p[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) p[i] = i < nq ? __ldg(p16 + i) : make_uint4(0, 0, 0, 0);
            const uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int m = 0; m < 5; ++m) {
                if (m >= n16) break;
                const uint4 lo = m == 0 ? z : p[m - 1 < 4 ? m - 1 : 3];
                const uint4 hi = m < nq ? p[m < 4 ? m : 3] : z;
                const uint4 v = a ? funnel16(lo, hi, 16 - a) : hi;
                const int blo = m == 0 ? a : 0, bhi = min(16, end - 16 * m);
                uint8_t* q = d0 + 16 * m;
                if (blo == 0 && bhi == 16) {
                    *reinterpret_cast<uint4*>(q) = v;
                } else {   // whole 8-byte halves as one store, the rest as 4-byte words
                    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (8 * h >= blo && 8 * h + 8 <= bhi) {
                            reinterpret_cast<uint2*>(q)[h] = make_uint2(w[2 * h], w[2 * h + 1]);
                        } else {
#pragma unroll
                            for (int k = 2 * h; k < 2 * h + 2; ++k)
                                if (4 * k >= blo && 4 * k + 4 <= bhi) reinterpret_cast<uint32_t*>(q)[k] = w[k];
                        }
                    }
                }
            }
        }
    }
}

template <bool PACK>
__device__ __forceinline__ void chain_job_body(const ChainJob& j, int64_t blk);

template <bool PACK>
__device__ __forceinline__ void chain_body(const ChainBatch& b) {
    // jobs with equal block counts are interleaved block by block, so e.g. the
    // lo and hi x-faces touch the same DRAM pages at the same time
    int ji = 0;
    const int bid = (int)blockIdx.x;
    uint32_t blk32 = 0;
    for (int i = 0; i < b.njobs; ++i) {
        const ChainJob& q = b.job[i];
        const int rel = bid - q.blk0;
        if (rel < 0 || rel >= q.nblk * q.gsize) continue;
        const uint32_t g = fdiv32((uint32_t)rel, q.m_g, q.s_g);
        if ((uint32_t)rel - g * (uint32_t)q.gsize == (uint32_t)q.gpos) {
            ji = i;
            blk32 = g;
            break;
        }
    }
    chain_job_body<PACK>(b.job[ji], blk32);
}

template <bool PACK>
__device__ __forceinline__ void chain_job_body(const ChainJob& j, int64_t blk) {
    if (j.mode == CHAIN_ROW) {
        chain_rows<PACK>(j, blk * (kChainThreads / 32) + (threadIdx.x >> 5),
                         (int64_t)j.nblk * (kChainThreads / 32));
    } else if (j.mode == CHAIN_WIDE) {
        chain_wide<PACK>(j, blk * kChainThreads + threadIdx.x, (int64_t)j.nblk * kChainThreads);
    } else {
        const int64_t t0 = blk * kChainThreads + threadIdx.x, nthr = (int64_t)j.nblk * kChainThreads;
        switch (j.w) {
        case 16: chain_elems<16, PACK>(j, t0, nthr); break;
        case 8: chain_elems<8, PACK>(j, t0, nthr); break;
        case 4: chain_elems<4, PACK>(j, t0, nthr); break;
        case 2: chain_elems<2, PACK>(j, t0, nthr); break;
        default: chain_elems<1, PACK>(j, t0, nthr); break;
        }
    }
    // unpack with data ending inside a row: bytewise tail
    if (!PACK && blk == 0 && threadIdx.x == 0) {
        for (int64_t P = j.rows * j.c.L; P < j.limit; ++P) j.dst[chain_off(j.c, P)] = j.src[P];
    }
}

// Separate entry points so each direction gets its own register budget
// (A/B on the bench step, round 2, then at 256 threads): pack at 1536
// threads/SM (40 registers) 33.8 -> 32.0 us; unpack (with the destination
// prefetches) at 1024 threads/SM (64 registers) 52.1 -> 48.5 us -- 1280
// threads 48.2 (spills), 1536 threads 49.4.  Same budgets at 64 threads.
__global__ void __launch_bounds__(kChainThreads, MPX_PACK_MINB) k_chain_pack(const ChainBatch b) { chain_body<true>(b); }
// one layout: the job by value (~250 B of parameters instead of the batch's
// ~4 KB: MPX_PROF measured 4.3-4.9 us of host time per single-layout launch)
__global__ void __launch_bounds__(kChainThreads, MPX_PACK_MINB) k_chain1_pack(const ChainJob j) {
    chain_job_body<true>(j, blockIdx.x);
}
#ifndef MPX_UNPACK_MINB
#define MPX_UNPACK_MINB 16
#endif
#if MPX_UNPACK_MINB
__global__ void __launch_bounds__(kChainThreads, MPX_UNPACK_MINB) k_chain_unpack(const ChainBatch b) { chain_body<false>(b); }
__global__ void __launch_bounds__(kChainThreads, MPX_UNPACK_MINB) k_chain1_unpack(const ChainJob j) {
    chain_job_body<false>(j, blockIdx.x);
}
#else
__global__ void __launch_bounds__(kChainThreads) k_chain_unpack(const ChainBatch b) { chain_body<false>(b); }
__global__ void __launch_bounds__(kChainThreads) k_chain1_unpack(const ChainJob j) { chain_job_body<false>(j, blockIdx.x); }
#endif

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

// ---------------------------------------------------------------- span
constexpr int kSpanWarps = 8;
constexpr int kSpanBuf = kSpanStage + 32;
constexpr size_t kSpanSmem = size_t(kSpanMaxBodies) * sizeof(SpanBody) + size_t(kSpanWarps) * 3 * kSpanBuf;

// global [g, g+len) -> smem buf[a, a+len) with aligned 16-byte loads (a = g & 15)
__device__ __forceinline__ int stage_in(uint8_t* buf, const uint8_t* g, int len, int lane) {
    const int a = (int)(reinterpret_cast<uintptr_t>(g) & 15);
    const uint4* g16 = reinterpret_cast<const uint4*>(g - a);
    const int nv = (a + len + 15) >> 4;
    for (int i = lane; i < nv; i += 32) reinterpret_cast<uint4*>(buf)[i] = __ldg(g16 + i);
    return a;
}

// smem buf[b, b+len) -> global [g, g+len) with aligned 16-byte stores
// (b = g & 15); mask (optional) selects the bytes to write (0xFF = write)
__device__ __forceinline__ void stage_out(uint8_t* g, const uint8_t* buf, const uint8_t* mask, int b, int len,
                                          int lane) {
    uint8_t* g0 = g - b;
    const int nv = (b + len + 15) >> 4;
    for (int k = lane; k < nv; k += 32) {
        const int lo = k == 0 ? b : 0;
        const int hi = min(16, b + len - 16 * k);
        const uint4 v = reinterpret_cast<const uint4*>(buf)[k];
        uint4 m = make_uint4(~0u, ~0u, ~0u, ~0u);
        if (mask) m = reinterpret_cast<const uint4*>(mask)[k];
        const bool full = lo == 0 && hi == 16 && (m.x & m.y & m.z & m.w) == ~0u;
        if (full) {
            reinterpret_cast<uint4*>(g0)[k] = v;
            continue;
        }
        const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
        const uint32_t mw[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int b0 = 4 * i;
            if (b0 >= lo && b0 + 4 <= hi && mw[i] == ~0u) {
                reinterpret_cast<uint32_t*>(g0 + 16 * k)[i] = vw[i];
            } else {
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int bb = b0 + t;
                    if (bb >= lo && bb < hi && ((mw[i] >> (8 * t)) & 0xFF))
                        g0[16 * k + bb] = (uint8_t)(vw[i] >> (8 * t));
                }
            }
        }
    }
}

// One warp per chunk, three phases:
//   1. the chunk's contiguous input (layout span for pack, packed bytes for
//      unpack) -> shared memory with aligned 16-byte loads;
//   2. shared -> shared permutation, one lane per element walking the body's
//      run table (unpack also marks the covered bytes);
//   3. shared -> global with aligned 16-byte stores; unpack writes only marked
//      bytes (bytes outside the runs are never touched).
template <bool PACK>
__global__ void __launch_bounds__(kSpanWarps * 32)
k_span(const SpanPlan sp, const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t limit) {
    extern __shared__ __align__(16) uint8_t sm[];
    SpanBody* bodies = reinterpret_cast<SpanBody*>(sm);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* A = sm + kSpanMaxBodies * sizeof(SpanBody) + warp * 3 * kSpanBuf;
    uint8_t* B = A + kSpanBuf;
    uint8_t* M = B + kSpanBuf;
    {
        const int nv = sp.nbodies * (int)(sizeof(SpanBody) / 16);
        const uint4* g = reinterpret_cast<const uint4*>(sp.bodies);
        for (int i = threadIdx.x; i < nv; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = __ldg(g + i);
    }
    __syncthreads();
    const int64_t stride_u = (int64_t)gridDim.x * kSpanWarps;
    for (int64_t u = (int64_t)blockIdx.x * kSpanWarps + warp; u < sp.nunits; u += stride_u) {
        const int64_t c = u % sp.nchunks;
        int64_t o = u / sp.nchunks, loff = 0, poff = 0;
        for (int i = sp.outer_depth - 1; i >= 0; --i) {
            const int64_t idx = o % sp.outer_cnt[i];
            o /= sp.outer_cnt[i];
            loff += idx * sp.outer_str[i];
            poff += idx * sp.outer_pk[i];
        }
        const SpanChunk* chp = sp.chunks + c;
        const int64_t lay0 = __ldg(&chp->src) + loff, pk0 = __ldg(&chp->pk) + poff;
        const int n = __ldg(&chp->n), body = __ldg(&chp->body), stride = __ldg(&chp->stride);
        const bool raw = body < 0;
        const SpanBody& Bd = bodies[raw ? 0 : body];
        const int span_len = raw ? stride : (n - 1) * stride + Bd.span_len;
        const int out_len = raw ? stride : n * Bd.nbytes;
        if (!PACK && pk0 >= limit) continue;
        const int qlim = (int)min((int64_t)out_len, limit - pk0);
        if (PACK) {
            const int a = stage_in(A, src + lay0, span_len, lane);
            const int b = (int)(reinterpret_cast<uintptr_t>(dst + pk0) & 15);
            __syncwarp();
            if (raw) {
                for (int i = lane; i < out_len; i += 32) B[b + i] = A[a + i];
            } else {
                const int nr = Bd.nruns, nb = Bd.nbytes;
                for (int e = lane; e < n; e += 32) {
                    const uint8_t* s0 = A + a + e * stride;
                    uint8_t* d0 = B + b + e * nb;
                    for (int r = 0; r < nr; ++r) {
                        const uint8_t* sr = s0 + Bd.roff[r];
                        uint8_t* dr = d0 + Bd.rpk[r];
                        const int len = Bd.rlen[r];
                        for (int x = 0; x < len; ++x) dr[x] = sr[x];
                    }
                }
            }
            __syncwarp();
            stage_out(dst + pk0, B, nullptr, b, out_len, lane);
        } else {
            const int a = stage_in(A, src + pk0, qlim, lane);
            const int b = (int)(reinterpret_cast<uintptr_t>(dst + lay0) & 15);
            const int nvm = (b + span_len + 15) >> 4;
            for (int i = lane; i < nvm; i += 32) reinterpret_cast<uint4*>(M)[i] = make_uint4(0, 0, 0, 0);
            __syncwarp();
            if (raw) {
                for (int i = lane; i < qlim; i += 32) {
                    B[b + i] = A[a + i];
                    M[b + i] = 0xFF;
                }
            } else {
                const int nr = Bd.nruns, nb = Bd.nbytes;
                for (int e = lane; e < n; e += 32) {
                    const int q0 = e * nb;
                    if (q0 >= qlim) break;
                    const uint8_t* s0 = A + a + q0;
                    const int d0 = b + e * stride;
                    for (int r = 0; r < nr; ++r) {
                        const int len = min((int)Bd.rlen[r], qlim - q0 - Bd.rpk[r]);
                        const uint8_t* sr = s0 + Bd.rpk[r];
                        const int dr = d0 + Bd.roff[r];
                        for (int x = 0; x < len; ++x) {
                            B[dr + x] = sr[x];
                            M[dr + x] = 0xFF;
                        }
                    }
                }
            }
            __syncwarp();
            stage_out(dst + lay0, B, M, b, span_len, lane);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- runs
// Flat run table (plan.hpp, RunTable): thread per run, G-byte words (G
// divides every offset and length), consecutive runs on consecutive lanes so
// the table loads and the packed side stay coalesced.  limit cuts the packed
// stream (unpack prefix semantics, datatype.py:719-724).
template <bool PACK, int G>
__global__ void __launch_bounds__(256)
k_runs(const RunTable t, const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t limit) {
    using T = typename Vec<G>::T;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < t.nruns; r += stride) {
        const int64_t so = __ldg(t.src + r), po = __ldg(t.pk + r);
        if (po >= limit) continue;
        const int64_t end = min(__ldg(t.pk + r + 1), limit);
        const int len = (int)(end - po);
        const uint8_t* s = src + (PACK ? so : po);
        uint8_t* d = dst + (PACK ? po : so);
        if (!PACK) prefetch_partial(d, len);   // destination fill before the load (see prefetch_l2)
        int w = 0;
        for (; w + G <= len; w += G) *reinterpret_cast<T*>(d + w) = *reinterpret_cast<const T*>(s + w);
        for (; w < len; ++w) d[w] = s[w];   // a run cut by the limit
    }
}

// Longer runs (>= 16 words on average): warp per run, lanes on consecutive
// words, so both sides move as coalesced 32 x G-byte accesses.  Lane l loads
// the table entry of run r0 + l; the warp then walks its 32 runs.
template <bool PACK, int G>
__global__ void __launch_bounds__(256)
k_runs_warp(const RunTable t, const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t limit) {
    using T = typename Vec<G>::T;
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * 8;
    for (int64_t r0 = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * 32; r0 < t.nruns; r0 += nw * 32) {
        int64_t so = 0, po = limit, end = limit;
        if (r0 + lane < t.nruns) {
            so = __ldg(t.src + r0 + lane);
            po = __ldg(t.pk + r0 + lane);
            end = min(__ldg(t.pk + r0 + lane + 1), limit);
        }
        const int cnt = (int)min((int64_t)32, t.nruns - r0);
        for (int j = 0; j < cnt; ++j) {
            const int64_t p0 = __shfl_sync(0xffffffffu, po, j);
            if (p0 >= limit) break;
            const int64_t s0 = __shfl_sync(0xffffffffu, so, j);
            const int len = (int)(__shfl_sync(0xffffffffu, end, j) - p0);
            const uint8_t* s = src + (PACK ? s0 : p0);
            uint8_t* d = dst + (PACK ? p0 : s0);
            const int nwd = len / G;
            for (int w = lane; w < nwd; w += 32)
                reinterpret_cast<T*>(d)[w] = reinterpret_cast<const T*>(s)[w];
            for (int b = nwd * G + lane; b < len; b += 32) d[b] = s[b];   // a run cut by the limit
        }
    }
}

__global__ void __launch_bounds__(256)
k_iov_runs(const RunTable t, int64_t k0, int64_t n, int64_t* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int64_t r = k0 + i;
        reinterpret_cast<longlong2*>(out)[i] = make_longlong2(__ldg(t.src + r), __ldg(t.pk + r + 1) - __ldg(t.pk + r));
    }
}

// ---------------------------------------------------------------- zipper
// Typed -> typed transfer in one pass (datatype.py:760-797 copy_between, the
// reference's zipper): both layouts are chains, so packed byte P maps to a
// source and a destination offset in closed form.  The packed stream is cut
// into pieces of g = gcd(L_src, L_dst) bytes that are contiguous on both
// sides; a thread moves a piece with W-byte words, two pieces in flight.
// No staging buffer: HBM (or NVLink for a peer buffer) is touched once per
// side.
template <int W>
__global__ void __launch_bounds__(256)
k_zip(const Chain cs, const Chain cd, const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
      int64_t npieces, int g) {
    using T = typename Vec<W>::T;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p0 < npieces; p0 += 2 * nthr) {
        int64_t so[2], dof[2];
        bool ok[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int64_t p = p0 + q * nthr;
            ok[q] = p < npieces;
            so[q] = ok[q] ? chain_off(cs, p * g) : 0;
            dof[q] = ok[q] ? chain_off(cd, p * g) : 0;
            if (ok[q]) prefetch_partial(dst + dof[q], g);
        }
        for (int w = 0; w < g; w += W) {
            T v[2];
#pragma unroll
            for (int q = 0; q < 2; ++q)
                if (ok[q]) v[q] = *reinterpret_cast<const T*>(src + so[q] + w);
#pragma unroll
            for (int q = 0; q < 2; ++q)
                if (ok[q]) *reinterpret_cast<T*>(dst + dof[q] + w) = v[q];
        }
    }
}

// bytes [from, to) of the packed stream, one thread, byte by byte (the tail
// that is not a whole piece)
__global__ void __launch_bounds__(32)
k_zip_tail(const Chain cs, const Chain cd, const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
           int64_t from, int64_t to) {
    for (int64_t P = from + threadIdx.x; P < to; P += 32) dst[chain_off(cd, P)] = src[chain_off(cs, P)];
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
// Chains: segment k is row k (closed form).
__global__ void __launch_bounds__(256)
k_iov_chain(const Chain c, int64_t k0, int64_t n, int64_t* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        reinterpret_cast<longlong2*>(out)[i] = make_longlong2(chain_row(c, k0 + i), c.L);
}

// Span plans: the segments of a (outer element, chunk) unit are its
// elements' body runs in order (raw pieces of one run form one segment).  A
// warp takes 32 units at a time: lane l loads unit l's metadata (one round
// trip for 32 units), then the warp walks the units, broadcasting each one's
// metadata and emitting its segments with lanes on consecutive segments --
// coalesced 16-byte stores, no tree descent.
__global__ void __launch_bounds__(256)
k_iov_span(const SpanPlan sp, int64_t k0, int64_t n, int64_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    longlong2* o2 = reinterpret_cast<longlong2*>(out);
    // an even split of the units over the warps (a grid-stride over 32-unit
    // batches left a third of the launch in a tail of a few warps: ~2.1
    // batches per warp on cfg3)
    const int64_t nw = (int64_t)gridDim.x * 8, gw = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int64_t ua = sp.nunits / nw * gw + min(gw, sp.nunits % nw);
    const int64_t uz = ua + sp.nunits / nw + (gw < sp.nunits % nw ? 1 : 0);
    for (int64_t ub = ua; ub < uz; ub += 32) {
        // lane l: metadata of unit ub + l
        int64_t seg0 = 0, lay0 = 0, rlen = 0;
        int32_t segs = 0, body = -1, stride = 0;
        const int64_t u = ub + lane;
        if (u < uz) {
            const uint64_t o = fdiv((uint64_t)u, sp.m_nchunks, sp.s_nchunks);
            const int64_t c = u - (int64_t)o * sp.nchunks;
            const longlong2 ic = __ldg(sp.iovc + c);
            const int64_t next = c + 1 < sp.nchunks ? __ldg(&sp.iovc[c + 1].x) : sp.segs_outer;
            int64_t loff = 0;
            if (sp.outer_depth == 1) {
                loff = (int64_t)o * sp.outer_str[0];
            } else if (sp.outer_depth == 2) {
                const uint64_t o0 = fdiv(o, sp.m_outer1, sp.s_outer1);
                loff = (int64_t)o0 * sp.outer_str[0] +
                       (int64_t)(o - o0 * (uint64_t)sp.outer_cnt[1]) * sp.outer_str[1];
            }
            const SpanChunk* ch = sp.chunks + c;
            seg0 = (int64_t)o * sp.segs_outer + ic.x;
            segs = (int32_t)(next - ic.x);
            lay0 = __ldg(&ch->src) + loff;
            body = __ldg(&ch->body);
            stride = __ldg(&ch->stride);
            rlen = ic.y;
            if (seg0 + segs <= k0 || seg0 >= k0 + n) segs = 0;
        }
        const int cnt = (int)min((int64_t)32, uz - ub);
        // Flat batch: when every unit of the batch repeats ONE body of <= 4
        // runs (cfg3: 2-run struct elements, ~26 per unit), the warp walks the
        // batch's elements as one sequence -- lane per element, its unit found
        // by a 5-step search over the units' element prefix held in the
        // lanes -- instead of unit by unit (per-unit set-up dominated: ~52
        // segments per unit).  Consecutive elements are consecutive in the
        // output, so a warp store covers 32 whole elements.
        {
            const int bd0 = __shfl_sync(0xffffffffu, body, 0);
            int nr0 = 0;
            if (bd0 >= 0) nr0 = __ldg(&sp.bodies[bd0].nruns);
            const int ne = nr0 == 2 ? segs >> 1 : nr0 > 0 ? segs / nr0 : 0;
            const bool ok = segs == 0 || (body == bd0 && nr0 > 0 && nr0 <= 4 && ne * nr0 == segs);
            if (__all_sync(0xffffffffu, ok) && bd0 >= 0 && nr0 <= 4) {
                const SpanBody* B = sp.bodies + bd0;
                int64_t ro[4];
                int64_t rl[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    ro[r] = r < nr0 ? (int64_t)__ldg(&B->roff[r]) : 0;
                    rl[r] = r < nr0 ? (int64_t)__ldg(&B->rlen[r]) : 0;
                }
                int incl = ne;   // inclusive prefix of elements over the units (lanes)
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, incl, d);
                    if (lane >= d) incl += v;
                }
                const int excl = incl - ne;
                const int total = __shfl_sync(0xffffffffu, incl, 31);
                longlong2* const ob = o2 - k0;
                for (int t0 = 0; t0 < total; t0 += 32) {   // warp-uniform trips: the shuffles need every lane
                    const int t = t0 + lane;
                    int uu = 0;   // last unit whose first element is <= t (it holds element t)
#pragma unroll
                    for (int step = 16; step; step >>= 1)
                        if (__shfl_sync(0xffffffffu, excl, uu + step) <= t) uu += step;
                    const int e = t - __shfl_sync(0xffffffffu, excl, uu);
                    const int64_t g = __shfl_sync(0xffffffffu, seg0, uu) + (int64_t)e * nr0;
                    const int64_t b = __shfl_sync(0xffffffffu, lay0, uu) +
                                      (int64_t)e * __shfl_sync(0xffffffffu, stride, uu);
                    longlong2* const p = ob + g;
                    if (t >= total) continue;
                    if (nr0 == 2 && g >= k0 && g + 2 <= k0 + n && !(reinterpret_cast<uintptr_t>(p) & 31)) {
                        asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(b + ro[0]), "l"(rl[0]),
                                     "l"(b + ro[1]), "l"(rl[1])
                                     : "memory");
                    } else {
#pragma unroll
                        for (int r = 0; r < 4; ++r)
                            if (r < nr0 && g + r >= k0 && g + r < k0 + n) p[r] = make_longlong2(b + ro[r], rl[r]);
                    }
                }
                continue;
            }
        }
        for (int j = 0; j < cnt; ++j) {
            const int32_t sg = __shfl_sync(0xffffffffu, segs, j);
            if (sg == 0) continue;
            const int64_t s0 = __shfl_sync(0xffffffffu, seg0, j);
            const int64_t l0 = __shfl_sync(0xffffffffu, lay0, j);
            const int32_t bd = __shfl_sync(0xffffffffu, body, j);
            if (bd < 0) {   // a raw run: one segment of the whole run
                const int64_t rl = __shfl_sync(0xffffffffu, rlen, j);
                if (lane == 0 && s0 >= k0) o2[s0 - k0] = make_longlong2(l0, rl);
                continue;
            }
            const int32_t st = __shfl_sync(0xffffffffu, stride, j);
            const SpanBody* B = sp.bodies + bd;
            const int nr = __ldg(&B->nruns);
            const int q32 = 32 / nr, r32 = 32 % nr;
            int e = lane / nr, r = lane - e * nr;
            const int64_t lo = max((int64_t)0, k0 - s0), hi = min((int64_t)sg, k0 + n - s0);
            for (int64_t i = lane; i < hi; i += 32) {
                if (i >= lo)
                    o2[s0 + i - k0] = make_longlong2(l0 + (int64_t)e * st + __ldg(&B->roff[r]), __ldg(&B->rlen[r]));
                e += q32;
                r += r32;
                if (r >= nr) {
                    r -= nr;
                    ++e;
                }
            }
        }
    }
}

__global__ void __launch_bounds__(256)
k_iov(const DDesc d, int64_t k0, int64_t n, int64_t* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const RunLoc r = locate_run(d, k0 + i);
        reinterpret_cast<longlong2*>(out)[i] = make_longlong2(r.src, r.len);
    }
}

}  // namespace

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

void chain_setup(const Plan& p, bool pack, ChainJob* j) {
    const Chain& c = p.chain;
    const uint8_t* layout_ptr = pack ? j->src : j->dst;
    const uint8_t* packed_ptr = pack ? j->dst : j->src;
    j->rows = j->limit / c.L;
    const bool packed_aligned = (reinterpret_cast<uintptr_t>(packed_ptr) & 15) == 0;
    if (c.L >= 64 && (c.L & 15) == 0 && packed_aligned) {
        j->mode = CHAIN_ROW;
        j->w = 16;
        return;
    }
    int64_t w = p.chain_align;
    const uintptr_t m = reinterpret_cast<uintptr_t>(layout_ptr) | reinterpret_cast<uintptr_t>(packed_ptr);
    while (w > 1 && (m & (uintptr_t)(w - 1))) w >>= 1;
    if (w >= 4 && w < 16 && (c.L & 15) == 0 && c.L <= 64 && packed_aligned) {
        j->mode = CHAIN_WIDE;    // short rows at 4/8-byte alignment: aligned 16-byte chunks
        j->w = 16;
        return;
    }
    j->mode = CHAIN_ELEM;
    j->w = (int32_t)w;
}

#ifndef MPX_ELEM_RPT
#define MPX_ELEM_RPT 2
#endif
#ifndef MPX_WIDE_RPT
#define MPX_WIDE_RPT 2
#endif

cudaError_t launch_chain_batch(ChainBatch& b, bool pack, int device, cudaStream_t stream) {
    if (b.njobs == 0) return cudaSuccess;
    // Enough CTAs that every row gets its own warp (row mode, <= 2 KiB per
    // warp pass) or its own thread (element mode) up to a cap of CTAs per SM
    // per job; bigger jobs loop (grid-stride) with 4 rows / 4 chunks in
    // flight.  Caps (64-thread CTAs): unpack 8, element / wide-mode pack 16,
    // row mode 8 (A/B: pack caps 8 / 12 / 16 / 24 -> bench-step pack 31.7 /
    // 31.6 / 30.3 / 31.7 us; a row-mode pack cap of 16 slows the contiguous
    // 256 MiB pack 89.2 -> 92.7 us; an unpack cap of 6 gains nothing).
#ifndef MPX_CHAIN_CAP
#define MPX_CHAIN_CAP 8
#endif
#ifndef MPX_CHAIN_PACK_CAP
#define MPX_CHAIN_PACK_CAP 16
#endif
#ifndef MPX_CHAIN_ROW_CAP
#define MPX_CHAIN_ROW_CAP 8
#endif
    const int64_t cap = (int64_t)sm_count(device) * (pack ? MPX_CHAIN_PACK_CAP : MPX_CHAIN_CAP);
    const int64_t row_cap = (int64_t)sm_count(device) * MPX_CHAIN_ROW_CAP;
    int64_t total = 0;
    for (int i = 0; i < b.njobs; ++i) {
        ChainJob& j = b.job[i];
        int64_t want;
        if (j.mode == CHAIN_ROW) {
            const int64_t nch = j.c.L >> 4;
            const int64_t items = j.rows * ((nch + kRowPieceChunks - 1) / kRowPieceChunks);
            want = (items + kChainThreads / 32 - 1) / (kChainThreads / 32);
        } else {
            // element-mode unpack: MPX_ELEM_RPT rows per thread (their
            // destination lines prefetched together); 1 = a thread per row
            const bool big = j.rows >= (int64_t)kChainThreads * sm_count(device) * 4;
            // unpack of large faces: 2 rows per thread, the next row's
            // destination prefetched while the current one is stored (wide
            // mode 48.3 -> 44.6 us on the bench step); pack keeps a thread per
            // row (2 per thread measured 32.1 -> 35.6 us)
            const int64_t per = (!pack && big) ? (j.mode == CHAIN_ELEM ? MPX_ELEM_RPT : MPX_WIDE_RPT) : 1;
            want = (j.rows + per * kChainThreads - 1) / (per * kChainThreads);
        }
        j.nblk = (int32_t)std::max<int64_t>(1, std::min<int64_t>(want, j.mode == CHAIN_ROW ? row_cap : cap));
        j.gsize = 1;
        j.gpos = 0;
        j.blk0 = -1;
        j.m_g = 0;
        j.s_g = 0;
    }
    for (int i = 0; i < b.njobs; ++i) {   // groups of equal nblk, interleaved
        ChainJob& j = b.job[i];
        if (j.blk0 >= 0) continue;
        int g = 0;
        for (int k = i; k < b.njobs; ++k)
            if (b.job[k].blk0 < 0 && b.job[k].nblk == j.nblk) ++g;
        int pos = 0;
        for (int k = i; k < b.njobs; ++k) {
            ChainJob& q = b.job[k];
            if (q.blk0 >= 0 || q.nblk != j.nblk) continue;
            q.blk0 = (int32_t)total;
            q.gsize = g;
            q.gpos = pos++;
            host_magic32((uint32_t)g, &q.m_g, &q.s_g);
        }
        total += (int64_t)j.nblk * g;
    }
    if (b.njobs == 1) {   // blocks map 1:1 onto the job (blk0 = 0, one-job group)
        if (pack) k_chain1_pack<<<(unsigned)total, kChainThreads, 0, stream>>>(b.job[0]);
        else k_chain1_unpack<<<(unsigned)total, kChainThreads, 0, stream>>>(b.job[0]);
    } else if (pack) {
        k_chain_pack<<<(unsigned)total, kChainThreads, 0, stream>>>(b);
    } else {
        k_chain_unpack<<<(unsigned)total, kChainThreads, 0, stream>>>(b);
    }
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

// Force-load every kernel of this translation unit on the current device.
// With CUDA lazy module loading, the first launch of a kernel loads its module
// and that load waits behind any stream parked in a stream-memop wait (even on
// other streams): a rank's first pack could then deadlock against a peer.
__global__ void k_flag_wait(const uint32_t* flag, uint32_t gen);

cudaError_t preload_pack_kernels() {
    cudaFuncAttributes a;
    cudaError_t e = cudaSuccess, r;
    if ((r = cudaFuncGetAttributes(&a, k_chain_pack)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_chain_unpack)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_chain1_pack)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_chain1_unpack)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_generic<true>)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_generic<false>)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_ordered_unpack)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_iov)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_iov_chain)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_iov_span)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_span<true>)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_span<false>)) != cudaSuccess) e = r;
    if ((r = preload_perm_kernels()) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_flag_wait)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_zip<16>)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_zip<8>)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_zip<4>)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_zip<2>)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_zip<1>)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_zip_tail)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_iov_runs)) != cudaSuccess) e = r;
#define MPX_PRE(PK, G)                                                                     \
    if ((r = cudaFuncGetAttributes(&a, k_runs<PK, G>)) != cudaSuccess) e = r;              \
    if ((r = cudaFuncGetAttributes(&a, k_runs_warp<PK, G>)) != cudaSuccess) e = r
    MPX_PRE(true, 16); MPX_PRE(true, 8); MPX_PRE(true, 4); MPX_PRE(true, 2); MPX_PRE(true, 1);
    MPX_PRE(false, 16); MPX_PRE(false, 8); MPX_PRE(false, 4); MPX_PRE(false, 2); MPX_PRE(false, 1);
#undef MPX_PRE
    return e;
}

cudaError_t launch_span(const Plan& p, bool pack, const uint8_t* src, uint8_t* dst, int64_t limit,
                        cudaStream_t stream) {
    if (limit <= 0 || p.span.nunits == 0) return cudaSuccess;
    if (p.span.perms) return launch_perm(p, pack, src, dst, limit, stream);
    const int64_t want = (p.span.nunits + kSpanWarps - 1) / kSpanWarps;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count(p.device) * 4));
    static bool attr_set[64][2] = {};   // the opt-in is per device
    const int d = p.device >= 0 && p.device < 64 ? p.device : 0;
    if (!attr_set[d][pack]) {   // > 48 KiB of dynamic shared memory needs an opt-in
        cudaError_t e = pack ? cudaFuncSetAttribute(k_span<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSpanSmem)
                             : cudaFuncSetAttribute(k_span<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSpanSmem);
        if (e != cudaSuccess) return e;
        attr_set[d][pack] = true;
    }
    if (pack) k_span<true><<<(unsigned)grid, kSpanWarps * 32, kSpanSmem, stream>>>(p.span, src, dst, limit);
    else k_span<false><<<(unsigned)grid, kSpanWarps * 32, kSpanSmem, stream>>>(p.span, src, dst, limit);
    return cudaGetLastError();
}

cudaError_t launch_runs(const Plan& p, bool pack, const uint8_t* src, uint8_t* dst, int64_t limit,
                        cudaStream_t stream) {
    if (limit <= 0 || p.rt.nruns == 0) return cudaSuccess;
    int g = p.rt.g;
    const uintptr_t m = reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst);
    while (g > 1 && (m & (uintptr_t)(g - 1))) g >>= 1;
    const int64_t want = (p.rt.nruns + 255) / 256;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count(p.device) * 16));
    const bool coop = p.rt.avg_words >= 16;
    const int64_t wgrid = std::max<int64_t>(1, std::min<int64_t>((p.rt.nruns + 255) / 256, (int64_t)sm_count(p.device) * 8));
#define MPX_RUNS(PK, G)                                                                     \
    do {                                                                                    \
        if (coop) k_runs_warp<PK, G><<<(unsigned)wgrid, 256, 0, stream>>>(p.rt, src, dst, limit); \
        else k_runs<PK, G><<<(unsigned)grid, 256, 0, stream>>>(p.rt, src, dst, limit);     \
    } while (0)
    if (pack) {
        switch (g) {
        case 16: MPX_RUNS(true, 16); break;
        case 8: MPX_RUNS(true, 8); break;
        case 4: MPX_RUNS(true, 4); break;
        case 2: MPX_RUNS(true, 2); break;
        default: MPX_RUNS(true, 1); break;
        }
    } else {
        switch (g) {
        case 16: MPX_RUNS(false, 16); break;
        case 8: MPX_RUNS(false, 8); break;
        case 4: MPX_RUNS(false, 4); break;
        case 2: MPX_RUNS(false, 2); break;
        default: MPX_RUNS(false, 1); break;
        }
    }
#undef MPX_RUNS
    return cudaGetLastError();
}

__global__ void __launch_bounds__(32) k_flag_wait(const uint32_t* flag, uint32_t gen) {
    if (threadIdx.x != 0) return;
    const volatile uint32_t* f = flag;
    unsigned ns = 64;
    while (*f < gen) {
        __nanosleep(ns);
        ns = ns < 2048 ? 2 * ns : ns;
    }
    __threadfence_system();
}

cudaError_t launch_flag_wait(const uint32_t* flag, uint32_t gen, cudaStream_t stream) {
    k_flag_wait<<<1, 32, 0, stream>>>(flag, gen);
    return cudaGetLastError();
}

cudaError_t launch_zip(const Plan& ps, const Plan& pd, const uint8_t* src, uint8_t* dst, int64_t bytes,
                       cudaStream_t stream) {
    if (bytes <= 0) return cudaSuccess;
    int64_t a = ps.chain.L, b = pd.chain.L;
    while (b) {
        const int64_t t = a % b;
        a = b;
        b = t;
    }
    const int64_t g = a;
    const int64_t npieces = bytes / g;
    int64_t w = std::min<int64_t>(ps.chain_align, pd.chain_align);
    const uintptr_t m = reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) | (uintptr_t)g;
    while (w > 1 && (m & (uintptr_t)(w - 1))) w >>= 1;
    if (npieces > 0) {
        // 128-thread CTAs, <= 8 per SM (A/B on the 2-rank vector(N/32,4,8)
        // ring, `profiles/r02l_ab_zip.txt`: 256 threads 0.147-0.154 / 1.66-1.68
        // ms at 64 MiB / 1 GiB, 128 threads 0.138-0.141 / 1.61-1.62, 64
        // threads x 16 the same, 64 x 32 or 128 x 16 no gain)
#ifndef MPX_ZIP_THREADS
#define MPX_ZIP_THREADS 128
#endif
#ifndef MPX_ZIP_CAP
#define MPX_ZIP_CAP 8
#endif
        constexpr int kZipThreads = MPX_ZIP_THREADS;
        const int64_t want = (npieces + 2 * kZipThreads - 1) / (2 * kZipThreads);
        const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count(ps.device) * MPX_ZIP_CAP));
        const int gi = (int)g;
        switch (w) {
        case 16: k_zip<16><<<(unsigned)grid, kZipThreads, 0, stream>>>(ps.chain, pd.chain, src, dst, npieces, gi); break;
        case 8: k_zip<8><<<(unsigned)grid, kZipThreads, 0, stream>>>(ps.chain, pd.chain, src, dst, npieces, gi); break;
        case 4: k_zip<4><<<(unsigned)grid, kZipThreads, 0, stream>>>(ps.chain, pd.chain, src, dst, npieces, gi); break;
        case 2: k_zip<2><<<(unsigned)grid, kZipThreads, 0, stream>>>(ps.chain, pd.chain, src, dst, npieces, gi); break;
        default: k_zip<1><<<(unsigned)grid, kZipThreads, 0, stream>>>(ps.chain, pd.chain, src, dst, npieces, gi); break;
        }
    }
    if (npieces * g < bytes) k_zip_tail<<<1, 32, 0, stream>>>(ps.chain, pd.chain, src, dst, npieces * g, bytes);
    return cudaGetLastError();
}

cudaError_t launch_iov(const Plan& p, int64_t k0, int64_t n, int64_t* out, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    const int64_t want = (n + 255) / 256;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count(p.device) * 16));
    if (p.kind == PLAN_CHAIN) {
        k_iov_chain<<<(unsigned)grid, 256, 0, stream>>>(p.chain, k0, n, out);
    } else if (p.kind == PLAN_RUNS && !p.rt.split) {
        k_iov_runs<<<(unsigned)grid, 256, 0, stream>>>(p.rt, k0, n, out);
    } else if (p.kind == PLAN_SPAN && p.span.iovc) {
        // one wave of resident CTAs: every warp takes an equal share of the units
        static int resident = 0;
        if (!resident) {
            int b = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_iov_span, 256, 0) != cudaSuccess || b < 1) {
                cudaGetLastError();
                b = 4;
            }
            resident = b;
        }
        const int64_t g = std::max<int64_t>(1, std::min<int64_t>((p.span.nunits + 255) / 256, (int64_t)sm_count(p.device) * resident));
        k_iov_span<<<(unsigned)g, 256, 0, stream>>>(p.span, k0, n, out);
    } else {
        k_iov<<<(unsigned)grid, 256, 0, stream>>>(p.desc, k0, n, out);
    }
    return cudaGetLastError();
}

}  // namespace mpx
