// k_perm.cu -- periodic word-gather pack / unpack for span plans (sm_100a).
//
// Layouts lowered to span chunks (plan.cpp: struct / indexed / nested types,
// e.g. BASELINE cfg3) move through this kernel whenever every chunk has a
// PermSpec (desc.cuh).  Data movement per warp and chunk:
//
//   1. the chunk's contiguous input (the layout span for pack, the packed
//      bytes for unpack) streams into shared memory with 16-byte cp.async,
//      double-buffered: chunk i+1 loads while chunk i is permuted;
//   2. each lane assembles whole aligned 32-bit output words from a window of
//      <= 4 staged input words with byte_perm (selectors precomputed per slot
//      and address phase on the host) and stores them straight to global
//      memory, a warp step covering W consecutive words;
//   3. words at the two ends of a chunk, words straddling a layout gap
//      (unpack) and chunks cut by the data limit take a per-byte path, so no
//      byte outside the layout (or past the limit) is ever written.
//
// Reference semantics: datatype.py:695-702 (pack) and :705-728 (unpack, prefix
// writes for short data); span plans never hold overlapping runs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "desc.cuh"
#include "kernels.hpp"

namespace mpx {

namespace {

constexpr int kWarps = 8;
constexpr int kBuf = kSpanStage + 32;     // staged input + window slack at the end
constexpr int kFront = 16;                // window slack before the staged input
constexpr int kSlot = kFront + kBuf;
#ifndef MPX_PERM_BPS2
#define MPX_PERM_BPS2 4
#endif
#ifndef MPX_PERM_BPS1
#define MPX_PERM_BPS1 4
#endif
template <int NS> constexpr int blocks_per_sm() { return NS <= 1 ? MPX_PERM_BPS1 : NS == 2 ? MPX_PERM_BPS2 : 3; }
constexpr size_t kSmem = size_t(kWarps) * 2 * kSlot;

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
// shared loads by 32-bit shared-window address; ordered after the
// cp.async wait / __syncwarp by the asm volatile chain
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1];\n" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
    uint16_t v;
    asm volatile("ld.shared.u8 %0, [%1];\n" : "=h"(v) : "r"(a));
    return v;
}

struct Unit {
    const uint8_t* in;   // chunk input
    uint8_t* out;        // chunk output
    int32_t in_len;      // input bytes present (unpack: cut by the data limit)
    int32_t out_len;     // output bytes (pack: cut by the limit)
    int32_t flags;       // bit 0: live (starts before the limit), bit 1: input holds the
                         // whole chunk, bits 8+: PermSpec index
};

// Unpack: ask L2 for the destination lines of the NEXT unit while this one is
// permuted -- its layout bytes are mostly partial sectors (a struct's gaps),
// whose DRAM fills then overlap the current unit's work instead of trailing
// its stores (the chain unpack gained 16 % this way).  MPX_UNPACK_PREFETCH=0
// turns it off.
#ifndef MPX_UNPACK_PREFETCH
#define MPX_UNPACK_PREFETCH 1
#endif
__device__ __forceinline__ void prefetch_out(const Unit& u, int lane) {
#if MPX_UNPACK_PREFETCH
    const uintptr_t first = reinterpret_cast<uintptr_t>(u.out) & ~uintptr_t(127);
    const uintptr_t last = (reinterpret_cast<uintptr_t>(u.out) + (uintptr_t)u.out_len - 1) & ~uintptr_t(127);
    for (uintptr_t a = first + (uintptr_t)lane * 128; a <= last; a += 32 * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
#else
    (void)u;
    (void)lane;
#endif
}

// Walks one warp's contiguous range of units in order without per-unit
// division: unit = (outer indices o0, o1; chunk c).
struct UnitIter {
    int32_t left;        // units after the current one
    int32_t c, o1;
    int64_t loff, poff;
};

__device__ __forceinline__ void iter_init(UnitIter& it, const SpanPlan& sp, int64_t u0, int64_t u1) {
    it.left = (int32_t)(u1 - u0 - 1);
    const uint64_t o = fdiv((uint64_t)u0, sp.m_nchunks, sp.s_nchunks);
    it.c = (int32_t)(u0 - (int64_t)o * sp.nchunks);
    it.o1 = 0;
    it.loff = it.poff = 0;
    if (sp.outer_depth == 1) {
        it.loff = (int64_t)o * sp.outer_str[0];
        it.poff = (int64_t)o * sp.outer_pk[0];
    } else if (sp.outer_depth == 2) {
        const uint64_t o0 = fdiv(o, sp.m_outer1, sp.s_outer1);
        it.o1 = (int32_t)(o - o0 * (uint64_t)sp.outer_cnt[1]);
        it.loff = (int64_t)o0 * sp.outer_str[0] + (int64_t)it.o1 * sp.outer_str[1];
        it.poff = (int64_t)o0 * sp.outer_pk[0] + (int64_t)it.o1 * sp.outer_pk[1];
    }
}

__device__ __forceinline__ void iter_next(UnitIter& it, const SpanPlan& sp) {
    --it.left;
    if (++it.c < sp.nchunks) return;
    it.c = 0;
    if (sp.outer_depth == 1) {
        it.loff += sp.outer_str[0];
        it.poff += sp.outer_pk[0];
    } else if (sp.outer_depth == 2) {
        it.loff += sp.outer_str[1];
        it.poff += sp.outer_pk[1];
        if (++it.o1 == sp.outer_cnt[1]) {
            it.o1 = 0;
            it.loff += sp.outer_str[0] - sp.outer_cnt[1] * sp.outer_str[1];
            it.poff += sp.outer_pk[0] - sp.outer_cnt[1] * sp.outer_pk[1];
        }
    }
}

template <bool PACK>
__device__ __forceinline__ Unit make_unit(const UnitIter& it, const SpanPlan& sp, const uint8_t* src, uint8_t* dst,
                                          int64_t limit) {
    const SpanChunk* ch = sp.chunks + it.c;
    const longlong2 sp0 = __ldg(reinterpret_cast<const longlong2*>(ch));          // src, pk
    const int64_t lay0 = sp0.x + it.loff, pk0 = sp0.y + it.poff;
    const int2 sl = __ldg(reinterpret_cast<const int2*>(&ch->span));   // span, plen
    const int32_t pp = __ldg(reinterpret_cast<const int32_t*>(&ch->perm[0]));
    const int32_t spec = PACK ? (pp >> 16) : (int32_t)(int16_t)(pp & 0xFFFF);
    Unit r;
    const int32_t avail = (int32_t)min((int64_t)sl.y, limit - pk0);
    const int32_t live = pk0 < limit ? 1 : 0;
    if (PACK) {
        r.in = src + lay0;
        r.out = dst + pk0;
        r.in_len = sl.x;
        r.out_len = avail;
        r.flags = live | 2 | (spec << 8);
    } else {
        r.in = src + pk0;
        r.out = dst + lay0;
        r.in_len = avail;
        r.out_len = sl.x;
        r.flags = live | (avail >= sl.y ? 2 : 0) | (spec << 8);
    }
    return r;
}

// Unit metadata for 32 consecutive units at once: lane l computes unit
// ub + l (one decomposition and one round of loads for 32 units); the warp
// then walks the batch broadcasting one unit at a time with shuffles.
template <bool PACK>
__device__ __forceinline__ Unit load_batch(const SpanPlan& sp, int64_t ub, int64_t u_end, const uint8_t* src,
                                           uint8_t* dst, int64_t limit, int lane) {
    Unit r;
    r.in = nullptr;
    r.out = nullptr;
    r.in_len = r.out_len = 0;
    r.flags = 0;
    const int64_t u = ub + lane;
    if (u < u_end) {
        UnitIter it;
        iter_init(it, sp, u, u + 1);
        r = make_unit<PACK>(it, sp, src, dst, limit);
    }
    return r;
}

__device__ __forceinline__ Unit bcast(const Unit& m, int i) {
    Unit r;
    r.in = reinterpret_cast<const uint8_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(m.in), i));
    r.out = reinterpret_cast<uint8_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(m.out), i));
    r.in_len = __shfl_sync(0xffffffffu, m.in_len, i);
    r.out_len = __shfl_sync(0xffffffffu, m.out_len, i);
    r.flags = __shfl_sync(0xffffffffu, m.flags, i);
    return r;
}

__device__ __forceinline__ void stage(uint32_t sbuf, const Unit& U, int lane) {
    const int a = (int)(reinterpret_cast<uintptr_t>(U.in) & 15);
    const uint8_t* g = U.in - a;
    const int nv = (a + U.in_len + 15) >> 4;
    for (int i = lane; i < nv; i += 32) cp_async16(sbuf + 16 * i, g + 16 * i);
}

// ---- TMA (bulk async copy) staging: one elected lane moves a chunk with
// one cp.async.bulk completing on the buffer's mbarrier.
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "MPX_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra MPX_WAIT_%=;\n}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_1d(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// Double-buffered staging of a warp's units: cp.async (any address: peer /
// host memory too) or TMA bulk copies (device-local buffers).
template <bool TMA>
struct Pipe {
    uint32_t bar;     // shared address of this warp's two mbarriers (TMA)
    uint32_t parity;  // bit b: phase to wait for on buffer b
    __device__ __forceinline__ void init(uint32_t bars, int lane) {
        bar = bars;
        parity = 0;
        if (TMA) {
            if (lane == 0) {
                mbar_init(bar, 1);
                mbar_init(bar + 8, 1);
                asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
            }
            __syncwarp();
        }
    }
    __device__ __forceinline__ void issue(uint32_t sbuf, int b, const Unit& U, int lane) {
        if (TMA) {
            if (lane == 0) {
                const int a = (int)(reinterpret_cast<uintptr_t>(U.in) & 15);
                const uint32_t bytes = (uint32_t)((a + U.in_len + 15) & ~15);
                // the buffer was last read through the generic proxy
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                mbar_expect_tx(bar + 8 * b, bytes);
                tma_load_1d(sbuf, U.in - a, bytes, bar + 8 * b);
            }
        } else {
            stage(sbuf, U, lane);
        }
    }
    __device__ __forceinline__ void commit() {
        if (!TMA) cp_async_commit();
    }
    // the current buffer b (issued iff live) is ready for every lane
    __device__ __forceinline__ void wait(int b, bool live) {
        if (TMA) {
            if (live) {
                mbar_wait(bar + 8 * b, (parity >> b) & 1);
                parity ^= 1u << b;
            }
        } else {
            cp_async_wait<1>();
            __syncwarp();
        }
    }
    __device__ __forceinline__ void drain() {
        if (!TMA) cp_async_wait<0>();
    }
};

__device__ __forceinline__ uint32_t prmt(uint32_t x, uint32_t y, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;\n" : "=r"(r) : "r"(x), "r"(y), "r"(sel));
    return r;
}

// Bytes of output word gw written this step: cover, minus bytes before the
// chunk (first word) and past its end (last word).
__device__ __forceinline__ uint32_t valid_mask(uint32_t cov, int gw, int po, int out_len) {
    const uint32_t lo = gw == 0 ? (0xFu << po) & 0xFu : 0xFu;
    const int nb = out_len + po - 4 * gw;
    const uint32_t hi = nb >= 4 ? 0xFu : (nb > 0 ? (1u << nb) - 1 : 0u);
    return cov & lo & hi;
}

// one table slot, as loaded: window address at step 0 + the three selectors
struct Slot {
    uint32_t w, lo, hi, mix;
};

// MPX_DEBUG_BOUNDS builds trap on a shared window outside the warp's two
// staging slots (the library ships without the check)
#ifdef MPX_DEBUG_BOUNDS
__device__ __forceinline__ uint8_t* sm_base_dbg();
#define MPX_CHECK_WIN(w)                                                                        \
    do {                                                                                        \
        const uint32_t lo_ = (uint32_t)__cvta_generic_to_shared(sm_base_dbg()) +                 \
                             (uint32_t)((threadIdx.x >> 5) * 2 * kSlot);                          \
        if ((w) < lo_ || (w) + 16 > lo_ + 2 * kSlot) {                                           \
            printf("k_perm window %u outside [%u, %u)\n", (w), lo_, lo_ + 2 * kSlot);             \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
#else
#define MPX_CHECK_WIN(w) ((void)0)
#endif

// output word of a slot whose window starts at shared address w
#ifdef MPX_DEBUG_BOUNDS
__device__ __forceinline__ uint8_t* sm_base_dbg() {
    extern __shared__ __align__(16) uint8_t sm[];
    return sm;
}
#endif

// byte form: input byte i of the word at shared address w + delta_i
__device__ __forceinline__ int byte_delta(const Slot& e, int i) {
    return i == 0 ? 0 : i == 1 ? (int)(int16_t)(e.hi & 0xFFFF) : i == 2 ? (int)(int16_t)(e.hi >> 16)
                                                                        : (int)(int16_t)(e.mix & 0xFFFF);
}

// byte form gather; addresses clamped into [lo, hi] (edge steps)
__device__ __forceinline__ uint32_t gather_bytes(uint32_t w, const Slot& e, uint32_t lo, uint32_t hi) {
    uint32_t b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = lds8(min(max(w + (uint32_t)byte_delta(e, i), lo), hi));
    return prmt(prmt(b[0], b[1], 0x0040u), prmt(b[2], b[3], 0x0040u), 0x5410u);
}

__device__ __forceinline__ uint32_t gather_word(uint32_t w, const Slot& e) {
    MPX_CHECK_WIN(w);
    const uint32_t a = prmt(lds32(w), lds32(w + 4), e.lo);
    const uint32_t b = prmt(lds32(w + 8), lds32(w + 12), e.hi);
    return prmt(a, b, e.mix);
}

__device__ __forceinline__ void store_bytes(uint8_t* p, uint32_t r, uint32_t m) {
    if (m & 1) p[0] = (uint8_t)r;
    if (m & 2) p[1] = (uint8_t)(r >> 8);
    if (m & 4) p[2] = (uint8_t)(r >> 16);
    if (m & 8) p[3] = (uint8_t)(r >> 24);
}

template <bool PACK, int NS, bool MIXED>
__device__ __forceinline__ void permute(const PermSpec& S, const Unit& U, uint32_t sbuf, int lane) {
    const int a = (int)(reinterpret_cast<uintptr_t>(U.in) & 15);
    const int ap = a & 3;
    const int po = (int)(reinterpret_cast<uintptr_t>(U.out) & 3);
    const int W = S.W;
    const bool bytes = MIXED && S.pad != 0;           // per-byte gathers (uniform per chunk)
    const int wc = S.wc[po * 4 + ap];                 // entries (words with a written byte) this phase
    const uint32_t Dw4 = 4u * (uint32_t)S.Dw;
    const uint4* tab = reinterpret_cast<const uint4*>(S.tab) + (po * 4 + ap) * W;
    const uint32_t A = sbuf + (uint32_t)(a & ~3);      // shared address of input word 0
    uint32_t* ow = reinterpret_cast<uint32_t*>(U.out - po);
    Slot e[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const int j = lane + 32 * s;
        uint4 t = make_uint4(0, 0, 0, 0);
        if (j < wc) t = __ldg(tab + j);
        e[s].w = A + t.x;
        e[s].lo = t.y;
        e[s].hi = t.z;
        e[s].mix = t.w;
    }
    const int words = (po + U.out_len + 3) >> 2;

    if (!(U.flags & 2)) {
        // input cut by the data limit (one chunk per call): bytes whose input
        // is missing are skipped one by one
        for (int kw = 0, kd = 0; kw < words; kw += W, kd += (int)Dw4) {
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                const int gw = kw + (int)(e[s].lo >> 24);
                const uint32_t vm = valid_mask((e[s].lo >> 16) & 0xF, gw, po, U.out_len);
                if (!vm || gw >= words) continue;
                const int wb = (int)(e[s].w - A) + kd;     // window start, bytes from input word 0
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if (!((vm >> i) & 1)) continue;
                    int in_off;
                    if (bytes) {
                        in_off = wb + byte_delta(e[s], i) - ap;
                    } else {
                        const uint32_t pr = (e[s].lo >> (20 + i)) & 1;
                        const uint32_t nib = ((pr ? e[s].hi : e[s].lo) >> (4 * i)) & 7;
                        in_off = wb + 8 * (int)pr + 4 * (int)(nib >> 2) + (int)(nib & 3) - ap;
                    }
                    if (in_off < U.in_len)
                        reinterpret_cast<uint8_t*>(ow + gw)[i] = (uint8_t)lds8(A + (uint32_t)(in_off + ap));
                }
            }
        }
        return;
    }

    // One step covers output words [kw, kw + W).  Words [w_lo, w_hi) are whole
    // (the first word is partial when po > 0); a window of a word that has a
    // valid byte lies within [sbuf - 16, sbuf + kBuf) (front slack), windows of
    // words past the end are clamped into the buffer and never stored.
    const int w_lo = po ? 1 : 0, w_hi = (U.out_len + po) >> 2;
    const uint32_t wmax = sbuf + (uint32_t)(kBuf - 16);
    auto edge = [&](int kw, uint32_t kd) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            if (32 * s >= wc) break;
            const uint32_t r = bytes ? gather_bytes(e[s].w + kd, e[s], sbuf - kFront, wmax + 15)
                                     : gather_word(min(e[s].w + kd, wmax), e[s]);
            const int gw = kw + (int)(e[s].lo >> 24);
            const uint32_t cov = (e[s].lo >> 16) & 0xF;
            uint32_t* p = ow + gw;
            if (gw >= w_lo && gw < w_hi) {
                if (cov == 0xF) *p = r;
                else if (!PACK && cov) store_bytes(reinterpret_cast<uint8_t*>(p), r, cov);   // layout gap
            } else if (cov && gw < words) {
                store_bytes(reinterpret_cast<uint8_t*>(p), r, valid_mask(cov, gw, po, U.out_len));
            }
        }
    };
    // interior steps (every word whole, so every window inside the staged
    // input) need no clamp and no bounds checks
    int kw = 0;
    uint32_t kd = 0;
    if (po && words > 0) {
        edge(0, 0);
        kw = W;
        kd = Dw4;
    }
    if (NS == 1 && !bytes) {
        // one slot per lane: window address and store pointer advance by a
        // constant per step
        if (kw + W <= w_hi) {
            const uint32_t cov = (e[0].lo >> 16) & 0xF;
            uint32_t wa = e[0].w + kd;
            uint32_t* p = ow + kw + (int)(e[0].lo >> 24);
            int left = w_hi - kw;
            do {
                const uint32_t r = gather_word(wa, e[0]);
                if (cov == 0xF) *p = r;
                else if (!PACK && cov) store_bytes(reinterpret_cast<uint8_t*>(p), r, cov);   // layout gap
                wa += Dw4;
                p += W;
                left -= W;
            } while (left >= W);
            kw = w_hi - left;
            kd = wa - e[0].w;
        }
    } else {
        for (; kw + W <= w_hi; kw += W, kd += Dw4) {
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                if (32 * s >= wc) break;
                const uint32_t r = bytes ? gather_bytes(e[s].w + kd, e[s], 0u, 0xFFFFFFFFu)
                                         : gather_word(e[s].w + kd, e[s]);
                const uint32_t cov = (e[s].lo >> 16) & 0xF;
                uint32_t* p = ow + kw + (int)(e[s].lo >> 24);
                if (cov == 0xF) *p = r;
                else if (!PACK && cov) store_bytes(reinterpret_cast<uint8_t*>(p), r, cov);   // layout gap
            }
        }
    }
    for (; kw < words; kw += W, kd += Dw4) edge(kw, kd);
}

#ifndef MPX_PACK_CARRY
#define MPX_PACK_CARRY 1
#endif
constexpr bool kPackCarry = MPX_PACK_CARRY != 0;   // A/B switch (-DMPX_PACK_CARRY=0: per-unit edges)

// Pack of one unit with a carried partial word.  A warp's units are
// consecutive chunks whose packed outputs abut, so the last, partial output
// word of unit u and the first, partial word of unit u + 1 are the same
// word: its bytes from unit u ride in `carry` (every lane) to unit u + 1,
// which merges them (one prmt) and stores the word whole.  The steps of a
// unit are then interior steps, the last ones with clamped windows -- no
// per-unit edge steps with byte masks.  Units whose head has no carry (the
// warp's first unit) or whose tail cannot be handed over (the warp's last
// unit, a unit cut by the limit) take the generic path, after storing any
// carried bytes.
//   head_ok:   `carry` holds bytes [0, po) of this unit's first output word
//   tail_keep: the next unit abuts this one in the packed output
// Returns whether the tail word was handed over in `carry`.
template <int NS, bool MIXED>
__device__ __forceinline__ bool permute_pack(const PermSpec& S, const Unit& U, uint32_t sbuf, int lane,
                                             uint32_t& carry, bool head_ok, bool tail_keep) {
    const int po = (int)(reinterpret_cast<uintptr_t>(U.out) & 3);
    const int tb = (po + U.out_len) & 3;                  // bytes of the tail word (0: none)
    const int w_hi = (U.out_len + po) >> 2;
    head_ok = head_ok && po != 0;
    tail_keep = tail_keep && tb != 0 && (w_hi > 0 || head_ok);
    const bool bytes = MIXED && S.pad != 0;
    if (bytes || (po && !head_ok) || (tb && !tail_keep) || !(U.flags & 2)) {
        // carried bytes [0, po) of the first word are stored here; the rest
        // of the unit by the generic path
        if (head_ok && lane == 0) store_bytes(U.out - po, carry, (1u << po) - 1);
        permute<true, NS, MIXED>(S, U, sbuf, lane);
        return false;
    }
    const int a = (int)(reinterpret_cast<uintptr_t>(U.in) & 15);
    const int ap = a & 3;
    const int W = S.W;
    const int wc = S.wc[po * 4 + ap];
    const uint32_t Dw4 = 4u * (uint32_t)S.Dw;
    const uint4* tab = reinterpret_cast<const uint4*>(S.tab) + (po * 4 + ap) * W;
    const uint32_t A = sbuf + (uint32_t)(a & ~3);
    uint32_t* ow = reinterpret_cast<uint32_t*>(U.out - po);
    Slot e[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const int j = lane + 32 * s;
        uint4 t = make_uint4(0, 0, 0, 0);
        if (j < wc) t = __ldg(tab + j);
        e[s].w = A + t.x;
        e[s].lo = t.y;
        e[s].hi = t.z;
        e[s].mix = t.w;
    }
    const int words = (po + U.out_len + 3) >> 2;
    const uint32_t wmax = sbuf + (uint32_t)(kBuf - 16);
    const uint32_t hsel = po == 1 ? 0x7650u : po == 2 ? 0x7610u : 0x7210u;   // bytes [0, po) from the carry
    uint32_t tail = 0;
    int kw = 0;
    uint32_t kd = 0;
    // the step holding word 0 merges the carry into it (po > 0); windows of
    // steps that reach past the last whole word are clamped into the buffer
    auto last_steps = [&](int kw, uint32_t kd) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            if (32 * s >= wc) break;
            uint32_t r = gather_word(min(e[s].w + kd, wmax), e[s]);
            const int gw = kw + (int)(e[s].lo >> 24);
            uint32_t cov = (e[s].lo >> 16) & 0xF;   // 0: an unused slot (lanes past wc alias word kw)
            if (gw == 0 && po && cov) {
                r = prmt(carry, r, hsel);
                cov = 0xF;
            }
            if (gw < w_hi) {
                if (cov == 0xF) ow[gw] = r;
            } else if (gw == w_hi && cov) {
                tail = r;
            }
        }
    };
    if (po) {
        if (W <= w_hi) {
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                if (32 * s >= wc) break;
                uint32_t r = gather_word(e[s].w, e[s]);
                const int gw = (int)(e[s].lo >> 24);
                uint32_t cov = (e[s].lo >> 16) & 0xF;
                if (gw == 0 && cov) {
                    r = prmt(carry, r, hsel);
                    cov = 0xF;
                }
                if (cov == 0xF) ow[gw] = r;
            }
        } else {
            last_steps(0, 0);
        }
        kw = W;
        kd = Dw4;
    }
    if (NS == 1) {
        // one slot per lane: window address and store pointer advance by a
        // constant per step (no per-step index math)
        if (kw + W <= w_hi) {
            const bool act = ((e[0].lo >> 16) & 0xF) == 0xF;
            uint32_t wa = e[0].w + kd;
            uint32_t* p = ow + kw + (int)(e[0].lo >> 24);
            int left = w_hi - kw;
            do {
                const uint32_t r = gather_word(wa, e[0]);
                if (act) *p = r;
                wa += Dw4;
                p += W;
                left -= W;
            } while (left >= W);
            kw = w_hi - left;
            kd = wa - e[0].w;
        }
    } else {
        for (; kw + W <= w_hi; kw += W, kd += Dw4) {
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                if (32 * s >= wc) break;
                const uint32_t r = gather_word(e[s].w + kd, e[s]);
                if (((e[s].lo >> 16) & 0xF) == 0xF) ow[kw + (int)(e[s].lo >> 24)] = r;
            }
        }
    }
    for (; kw < words; kw += W, kd += Dw4) last_steps(kw, kd);
    carry = __reduce_or_sync(0xffffffffu, tail_keep ? tail : 0u);
    return tail_keep;
}

template <bool PACK, int NS, bool TMA, bool MIXED>
__global__ void __launch_bounds__(kWarps * 32, blocks_per_sm<NS>())
k_perm(const SpanPlan sp, const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t limit) {
    extern __shared__ __align__(16) uint8_t sm[];
    __shared__ PermSpec specs[2 * kPermMaxSpecs];
    __shared__ __align__(8) uint64_t bars[kWarps][2];
    for (int i = threadIdx.x; i < sp.nperms; i += blockDim.x) specs[i] = sp.perms[i];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm) + (uint32_t)(warp * 2 * kSlot + kFront);
    // a contiguous range of units per warp: consecutive chunks, no per-unit division
    const int64_t nw = (int64_t)gridDim.x * kWarps, gwid = (int64_t)blockIdx.x * kWarps + warp;
    const int64_t u0 = sp.nunits / nw * gwid + min(gwid, sp.nunits % nw);
    const int64_t u1 = u0 + sp.nunits / nw + (gwid < sp.nunits % nw ? 1 : 0);
    if (u0 >= u1) return;
    Pipe<TMA> pipe;
    pipe.init((uint32_t)__cvta_generic_to_shared(&bars[warp][0]), lane);
    uint32_t pb = 0;
    uint32_t carry = 0;    // pack: the previous unit's tail word (permute_pack)
    bool have = false;
#ifndef MPX_UNPACK_BATCH
#define MPX_UNPACK_BATCH 0
#endif
    if (NS == 1 && (PACK || MPX_UNPACK_BATCH)) {
        // unit metadata 32 units per batch, distributed over the lanes (one
        // round of dependent loads per 32 units instead of per unit; measured
        // faster for pack, slower for unpack)
        Unit batch = load_batch<PACK>(sp, u0, u1, src, dst, limit, lane);
        Unit cur = bcast(batch, 0);
        if (cur.flags & 1) pipe.issue(sbase, 0, cur, lane);
        pipe.commit();
        for (int64_t u = u0;; ++u) {
            const bool more = u + 1 < u1;
            Unit nxt;
            nxt.flags = 0;
            if (more) {
                const int i = (int)((u + 1 - u0) & 31);
                if (i == 0) batch = load_batch<PACK>(sp, u + 1, u1, src, dst, limit, lane);
                nxt = bcast(batch, i);
                if (nxt.flags & 1) pipe.issue(sbase + (pb ^ kSlot), pb ? 0 : 1, nxt, lane);
                if (!PACK && (nxt.flags & 1)) prefetch_out(nxt, lane);
            }
            pipe.commit();
            pipe.wait(pb ? 1 : 0, cur.flags & 1);
            if (cur.flags & 1) {
                if (PACK && kPackCarry) {
                    const bool abut = (nxt.flags & 1) && nxt.out == cur.out + cur.out_len;
                    have = permute_pack<NS, MIXED>(specs[cur.flags >> 8], cur, sbase + pb, lane, carry, have, abut);
                } else {
                    permute<PACK, NS, MIXED>(specs[cur.flags >> 8], cur, sbase + pb, lane);
                }
            }
            __syncwarp();
            if (!more) break;
            cur = nxt;
            pb ^= kSlot;
        }
    } else {
        // walk units one by one (more slots leave no registers for a batch)
        UnitIter it;
        iter_init(it, sp, u0, u1);
        Unit cur = make_unit<PACK>(it, sp, src, dst, limit);
        if (cur.flags & 1) pipe.issue(sbase, 0, cur, lane);
        pipe.commit();
        for (;;) {
            const bool more = it.left > 0;
            Unit nxt;
            nxt.flags = 0;
            if (more) {
                iter_next(it, sp);
                nxt = make_unit<PACK>(it, sp, src, dst, limit);
                if (nxt.flags & 1) pipe.issue(sbase + (pb ^ kSlot), pb ? 0 : 1, nxt, lane);
                if (!PACK && (nxt.flags & 1)) prefetch_out(nxt, lane);
            }
            pipe.commit();
            pipe.wait(pb ? 1 : 0, cur.flags & 1);
            if (cur.flags & 1) {
                if (PACK && kPackCarry) {
                    const bool abut = (nxt.flags & 1) && nxt.out == cur.out + cur.out_len;
                    have = permute_pack<NS, MIXED>(specs[cur.flags >> 8], cur, sbase + pb, lane, carry, have, abut);
                } else {
                    permute<PACK, NS, MIXED>(specs[cur.flags >> 8], cur, sbase + pb, lane);
                }
            }
            __syncwarp();
            if (!more) break;
            cur = nxt;
            pb ^= kSlot;
        }
    }
    pipe.drain();
}

// The staged input is read from `ptr` (the layout side for pack, the packed
// side for unpack): plain device memory of `device`?
bool local_device_memory(const void* ptr, int device) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice && at.device == device;
}

template <typename F>
cudaError_t set_smem(F f) {
    return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
}

bool disable_tma() {
    static const bool off = getenv("MPX_NO_TMA") != nullptr;   // A/B switch
    return off;
}

template <bool PACK>
cudaError_t launch_dir(const Plan& p, const uint8_t* src, uint8_t* dst, int64_t limit, cudaStream_t stream) {
    // slots this launch needs: the phase variants its chunks actually take
    // given the buffer addresses (aligned buffers touch few variants)
    int ns = 0;
    {
        const int lp = (int)(reinterpret_cast<uintptr_t>(PACK ? src : dst) & 3);
        const int pp = (int)(reinterpret_cast<uintptr_t>(PACK ? dst : src) & 3);
        for (const int32_t u : p.perm_use[PACK ? 1 : 0]) {
            const PermSpec& S = p.perm_specs[(size_t)(u >> 6)];
            int wc = 0;
            for (int v = 0; v < 16; ++v) {
                const int po = v >> 2, ap = v & 3;
                const int lay = PACK ? ap : po, pk = PACK ? po : ap;   // phases of this variant
                const bool lay_ok = (u & 32) || lay == ((((u >> 2) & 3) + lp) & 3);
                const bool pk_ok = (u & 16) || pk == (((u & 3) + pp) & 3);
                if (lay_ok && pk_ok) wc = std::max<int>(wc, S.wc[v]);
            }
            ns = std::max(ns, (wc + 31) / 32);
        }
        ns = std::max(ns, 1);
        static const bool dbg = getenv("MPX_DEBUG_PLAN") != nullptr;
        if (dbg) fprintf(stderr, "[mpx k_perm] %s: %d slots (plan max %d), %zu spec/phase uses\n",
                         PACK ? "pack" : "unpack", ns, p.span.ns_max[PACK ? 1 : 0], p.perm_use[PACK ? 1 : 0].size());
    }
    const int64_t want = (p.span.nunits + kWarps - 1) / kWarps;
    const int64_t grid = std::max<int64_t>(
        1, std::min<int64_t>(want, (int64_t)sm_count(p.device) * (ns <= 1 ? blocks_per_sm<1>() : ns == 2 ? blocks_per_sm<2>() : blocks_per_sm<4>())));
    // TMA bulk staging for pack when the layout side is memory of this device
    // (peer and pinned-host buffers keep cp.async).  Measured (ncu, cfg3):
    // pack 290 us with TMA vs 299 us with cp.async; unpack -- small packed
    // chunks -- 433 vs 402-415 us, so unpack stays on cp.async.
    static const bool unpack_tma = getenv("MPX_UNPACK_TMA") != nullptr;   // A/B switch
    const bool tma = (PACK || unpack_tma) && local_device_memory(src, p.device) && !disable_tma();
    // byte-form specs need the mixed kernel; word-window-only plans get the
    // leaner one (no byte path compiled in)
    bool mixed = false;
    for (const int32_t u : p.perm_use[PACK ? 1 : 0]) mixed = mixed || p.perm_specs[(size_t)(u >> 6)].pad != 0;
    // > 48 KiB of dynamic shared memory needs the opt-in, per device and kernel
    static bool smem_set[64][4][4] = {};
    const int dslot = p.device >= 0 && p.device < 64 ? p.device : 0;
    const int nsi = std::min(std::max(ns, 1), 4) - 1, vi = (tma ? 1 : 0) | (mixed ? 2 : 0);
    if (!smem_set[dslot][nsi][vi]) {
        cudaError_t e = cudaSuccess;
#define MPX_PERM_ATTR(N)                                                                             \
        do {                                                                                         \
            if (mixed) e = tma ? set_smem(k_perm<PACK, N, true, true>) : set_smem(k_perm<PACK, N, false, true>); \
            else e = tma ? set_smem(k_perm<PACK, N, true, false>) : set_smem(k_perm<PACK, N, false, false>); \
        } while (0)
        switch (nsi) {
        case 0: MPX_PERM_ATTR(1); break;
        case 1: MPX_PERM_ATTR(2); break;
        case 2: MPX_PERM_ATTR(3); break;
        default: MPX_PERM_ATTR(4); break;
        }
#undef MPX_PERM_ATTR
        if (e != cudaSuccess) return e;
        smem_set[dslot][nsi][vi] = true;
    }
#define MPX_PERM(N)                                                                              \
    do {                                                                                         \
        if (mixed) {                                                                             \
            if (tma) k_perm<PACK, N, true, true><<<(unsigned)grid, kWarps * 32, kSmem, stream>>>(p.span, src, dst, limit); \
            else k_perm<PACK, N, false, true><<<(unsigned)grid, kWarps * 32, kSmem, stream>>>(p.span, src, dst, limit); \
        } else {                                                                                 \
            if (tma) k_perm<PACK, N, true, false><<<(unsigned)grid, kWarps * 32, kSmem, stream>>>(p.span, src, dst, limit); \
            else k_perm<PACK, N, false, false><<<(unsigned)grid, kWarps * 32, kSmem, stream>>>(p.span, src, dst, limit); \
        }                                                                                        \
    } while (0)
    switch (ns) {
    case 1: MPX_PERM(1); break;
    case 2: MPX_PERM(2); break;
    case 3: MPX_PERM(3); break;
    default: MPX_PERM(4); break;
    }
#undef MPX_PERM
    return cudaGetLastError();
}

template <typename F>
cudaError_t attr(F f, cudaFuncAttributes* a) {
    return cudaFuncGetAttributes(a, f);
}

}  // namespace

static_assert(kPermMaxSlots == 4, "launch_dir instantiates NS = 1..4");

cudaError_t launch_perm(const Plan& p, bool pack, const uint8_t* src, uint8_t* dst, int64_t limit,
                        cudaStream_t stream) {
    if (limit <= 0 || p.span.nunits == 0) return cudaSuccess;
    return pack ? launch_dir<true>(p, src, dst, limit, stream) : launch_dir<false>(p, src, dst, limit, stream);
}

cudaError_t preload_perm_kernels() {
    cudaFuncAttributes a;
    cudaError_t e = cudaSuccess, r;
#define MPX_PRE(PK, N)                                                        \
    if ((r = attr(k_perm<PK, N, false, false>, &a)) != cudaSuccess) e = r;    \
    if ((r = attr(k_perm<PK, N, true, false>, &a)) != cudaSuccess) e = r;     \
    if ((r = attr(k_perm<PK, N, false, true>, &a)) != cudaSuccess) e = r;     \
    if ((r = attr(k_perm<PK, N, true, true>, &a)) != cudaSuccess) e = r
    MPX_PRE(true, 1); MPX_PRE(true, 2); MPX_PRE(true, 3); MPX_PRE(true, 4);
    MPX_PRE(false, 1); MPX_PRE(false, 2); MPX_PRE(false, 3); MPX_PRE(false, 4);
#undef MPX_PRE
    return e;
}

}  // namespace mpx
