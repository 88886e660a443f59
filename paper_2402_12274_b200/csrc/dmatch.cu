// dmatch.cu -- device-resident matching kernels (see dmatch.hpp).
//
// Matching rules: transport.py:191-201 (a receive pattern matches a message
// when the contexts are equal and source / tag are equal or ANY_*), the
// earliest candidate wins (posting order for receives, arrival order for
// messages: transport.py:399-428, :509-516).  Box entries are read with
// volatile (L1-bypassing) loads: a box is written by kernels of several
// ranks, possibly on peer GPUs over NVLink, and published under its lock
// with system-scope fences.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <cstring>

#include "dmatch.hpp"
#include "kernels.hpp"
#include "mpx.h"

namespace mpx {

namespace {

constexpr int kThreads = 256;

template <int W> struct DVec;
template <> struct DVec<16> { using T = uint4; };
template <> struct DVec<8> { using T = uint2; };
template <> struct DVec<4> { using T = uint32_t; };
template <> struct DVec<2> { using T = uint16_t; };
template <> struct DVec<1> { using T = uint8_t; };
constexpr unsigned long long kNone = ~0ull;
constexpr uint64_t kGiveUpNs = 20ull * 1000000000ull;   // a full queue for 20 s: report and drop

__device__ __forceinline__ uint64_t now_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void lock(DmBox* b) {
    while (atomicCAS_system(&b->lock, 0, 1) != 0) __nanosleep(64);
    __threadfence_system();
}

__device__ __forceinline__ void unlock(DmBox* b) {
    __threadfence_system();
    atomicExch_system(&b->lock, 0);
}

__device__ __forceinline__ bool pat_match(int psrc, int ptag, int pctx, int src, int tag, int ctx) {
    return pctx == ctx && (psrc == MPX_ANY_SOURCE || psrc == src) && (ptag == MPX_ANY_TAG || ptag == tag);
}

// block-wide: the key (seq << 12 | index) of the earliest live entry accepted
// by `ok`, or kNone
template <typename F>
__device__ __forceinline__ unsigned long long earliest(int hw, F ok, unsigned long long* sh) {
    if (threadIdx.x == 0) *sh = kNone;
    __syncthreads();
    unsigned long long mine = kNone;
    for (int i = threadIdx.x; i < hw; i += blockDim.x) {
        const unsigned long long k = ok(i);
        mine = k < mine ? k : mine;
    }
    if (mine != kNone) atomicMin(sh, mine);
    __syncthreads();
    const unsigned long long r = *sh;
    __syncthreads();
    return r;
}

// block-wide: the lowest free index below min(hw + 1, kDmSlots), or -1
template <typename F>
__device__ __forceinline__ int first_free(int hw, F is_free, int* sh) {
    if (threadIdx.x == 0) *sh = INT_MAX;
    __syncthreads();
    const int lim = hw + 1 < kDmSlots ? hw + 1 : kDmSlots;
    for (int i = threadIdx.x; i < lim; i += blockDim.x)
        if (is_free(i)) {
            atomicMin(sh, i);
            break;
        }
    __syncthreads();
    const int r = *sh;
    __syncthreads();
    return r == INT_MAX ? -1 : r;
}

// 8-byte word copies of the plain-old-data box records (volatile: another
// rank's kernel may read them over NVLink)
template <typename T>
__device__ __forceinline__ void vput(volatile T* dst, const T& src) {
    static_assert(sizeof(T) % 8 == 0, "8-byte words");
    const uint64_t* s = reinterpret_cast<const uint64_t*>(&src);
    volatile uint64_t* d = reinterpret_cast<volatile uint64_t*>(dst);
#pragma unroll 4
    for (int i = 0; i < (int)(sizeof(T) / 8); ++i) d[i] = s[i];
}

// block-cooperative copy of a layout record: one 8-byte word per thread, so
// the volatile loads (L2 / NVLink round trips) overlap instead of queueing
constexpr int kLayWords = (int)(sizeof(DmLay) / 8);
static_assert(kLayWords <= kThreads, "one word per thread");
__device__ __forceinline__ void coop_lay(volatile DmLay* dst, const volatile DmLay* src) {
    if (threadIdx.x < kLayWords)
        reinterpret_cast<volatile uint64_t*>(dst)[threadIdx.x] =
            reinterpret_cast<const volatile uint64_t*>(src)[threadIdx.x];
}

// a contiguous run of `bytes` at offset 0 (device side; lay_off never
// divides on a depth-0 chain, so no magic numbers)
__device__ __forceinline__ DmLay dm_contig_lay_dev(int64_t bytes) {
    DmLay l;
    memset(&l, 0, sizeof l);
    l.c.L = bytes > 0 ? bytes : 1;
    l.align = 16;
    return l;
}

// layout offset of packed byte P (a depth-0 chain is one run covering every P)
__device__ __forceinline__ int64_t lay_off(const Chain& c, int64_t P) {
    return c.depth == 0 ? c.base + P : chain_off(c, P);
}

__device__ __forceinline__ int64_t gcd64(int64_t a, int64_t b) {
    while (b) {
        const int64_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}

template <int W>
__device__ __forceinline__ void chain_pieces(const Chain& sc, const uint8_t* sb, const Chain& dc, uint8_t* db,
                                             int64_t np, int64_t g, int64_t tid, int64_t nth) {
    using T = typename DVec<W>::T;
    for (int64_t p = tid; p < np; p += nth) {
        const int64_t so = lay_off(sc, p * g), dof = lay_off(dc, p * g);
        for (int64_t w = 0; w < g; w += W)
            *reinterpret_cast<T*>(db + dof + w) = *reinterpret_cast<const T*>(sb + so + w);
    }
}

// grid-stride byte copy, 16 / 4-byte words when both sides allow
__device__ __forceinline__ void copy_bytes(const uint8_t* src, uint8_t* dst, int64_t n, int64_t tid, int64_t nth) {
    const uintptr_t mis = (reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst));
    int64_t head = 0;
    if ((mis & 15) == 0) {
        const int64_t nv = n >> 4;
        const uint4* s4 = reinterpret_cast<const uint4*>(src);
        uint4* d4 = reinterpret_cast<uint4*>(dst);
        for (int64_t i = tid; i < nv; i += nth) d4[i] = s4[i];
        head = nv << 4;
    } else if ((mis & 3) == 0) {
        const int64_t nv = n >> 2;
        const uint32_t* s4 = reinterpret_cast<const uint32_t*>(src);
        uint32_t* d4 = reinterpret_cast<uint32_t*>(dst);
        for (int64_t i = tid; i < nv; i += nth) d4[i] = s4[i];
        head = nv << 2;
    }
    for (int64_t i = head + tid; i < n; i += nth) dst[i] = src[i];
}

// packed bytes [0, n) from layout s of buffer sb to layout d of buffer db
// (copy_between semantics, datatype.py:760-797): the packed stream cut into
// pieces of g = gcd(run lengths, 64) bytes, contiguous on both sides, moved
// with the widest word both sides allow; the < g tail byte by byte
__device__ __forceinline__ void chain_copy(const DmLay& s, const uint8_t* sb, const DmLay& d, uint8_t* db, int64_t n,
                                           int64_t tid, int64_t nth) {
    if (n <= 0) return;
    if (s.c.depth == 0 && d.c.depth == 0) {   // contiguous on both sides: a plain copy
        copy_bytes(sb + s.c.base, db + d.c.base, n, tid, nth);
        return;
    }
    const int64_t g = gcd64(gcd64(s.c.L, d.c.L), 64);
    int w = s.align < d.align ? s.align : d.align;
    w = w > 16 ? 16 : w;
    const uintptr_t m = reinterpret_cast<uintptr_t>(sb) | reinterpret_cast<uintptr_t>(db) | (uintptr_t)g;
    while (w > 1 && (m & (uintptr_t)(w - 1))) w >>= 1;
    const int64_t np = n / g;
    switch (w) {
    case 16: chain_pieces<16>(s.c, sb, d.c, db, np, g, tid, nth); break;
    case 8: chain_pieces<8>(s.c, sb, d.c, db, np, g, tid, nth); break;
    case 4: chain_pieces<4>(s.c, sb, d.c, db, np, g, tid, nth); break;
    case 2: chain_pieces<2>(s.c, sb, d.c, db, np, g, tid, nth); break;
    default: chain_pieces<1>(s.c, sb, d.c, db, np, g, tid, nth); break;
    }
    for (int64_t P = np * g + tid; P < n; P += nth) db[lay_off(d.c, P)] = sb[lay_off(s.c, P)];
}

__device__ __forceinline__ void publish(DmResult* res, int src, int tag, int64_t bytes, const uint8_t* data,
                                        uint32_t* consumed, uint32_t cgen, int rdv, uint8_t* dst, int64_t cap,
                                        int copier) {
    volatile DmResult* r = res;   // slay / dlay: copied by the block before (coop_lay)
    r->src = src;
    r->tag = tag;
    r->bytes = bytes;
    r->data = data;
    r->consumed = consumed;
    r->cgen = cgen;
    r->rdv = rdv;
    r->dst = dst;
    r->n = bytes < cap ? bytes : cap;
    r->copier = copier;
    r->copied = 0;
    r->xdone = 0;
    __threadfence_system();
    r->ready = 1;
}

// the rendezvous copy is complete: release the sender, then the receiver
__device__ __forceinline__ void rdv_complete(volatile DmResult* r) {
    __threadfence_system();
    *reinterpret_cast<volatile uint32_t*>(r->consumed) = r->cgen;
    __threadfence_system();
    r->copied = 1;
}

struct SendArgs {
    DmBox* box;
    int32_t src, tag, ctx;
    uint32_t cgen;
    const uint8_t* data;
    int64_t bytes;
    uint32_t* consumed;
    int32_t* record;      // rendezvous: the matched result slot, or -1 (sender's own box)
    int32_t rdv, pad;
    DmLay lay;            // relative to data
    uint8_t* bounce;      // eager, chain layout: the block packs data (lay) into bounce first
};

// a message arrives at the receiving rank's box
__global__ void __launch_bounds__(kThreads) k_dm_send(SendArgs a) {
    __shared__ unsigned long long best;
    __shared__ int slot;
    DmBox* b = a.box;
    volatile DmBox* vb = b;
    if (a.bounce) {   // eager message of a chain layout: pack it here (no separate pack launch)
        chain_copy(a.lay, a.data, dm_contig_lay_dev(a.bytes), a.bounce, a.bytes, threadIdx.x, blockDim.x);
        __threadfence();
        __syncthreads();
        a.data = a.bounce;
        a.lay = dm_contig_lay_dev(a.bytes);
    }
    const uint64_t t0 = now_ns();
    for (;;) {
        if (threadIdx.x == 0) lock(b);
        __syncthreads();
        const int hw = vb->hw_recv;
        const unsigned long long k = earliest(hw, [&](int i) -> unsigned long long {
            volatile const DmRecv& r = vb->recv[i];
            if (r.state != 1 || !pat_match(r.src, r.tag, r.ctx, a.src, a.tag, a.ctx)) return kNone;
            return ((unsigned long long)r.seq << 12) | (unsigned)i;
        }, &best);
        bool done = true;
        if (k != kNone) {   // the earliest posted receive takes it
            {
                const int i = (int)(k & 0xFFF);
                volatile DmResult* rr = &b->result[vb->recv[i].result];
                coop_lay(&rr->slay, &a.lay);
                coop_lay(&rr->dlay, &vb->recv[i].lay);
                __syncthreads();
            }
            if (threadIdx.x == 0) {
                const int i = (int)(k & 0xFFF);
                volatile DmRecv& rv = vb->recv[i];
                publish(&b->result[rv.result], a.src, a.tag, a.bytes, a.data, a.consumed, a.cgen, a.rdv,
                        rv.dst, rv.cap, 0);
                if (a.record) *reinterpret_cast<volatile int32_t*>(a.record) = rv.result;
                vb->recv[i].state = 0;
                int h = hw;
                while (h > 0 && vb->recv[h - 1].state == 0) --h;
                vb->hw_recv = h;
            }
        } else {            // unexpected: queue it
            const int hm = vb->hw_msg;
            const int f = first_free(hm, [&](int i) { return vb->msg[i].state == 0; }, &slot);
            if (threadIdx.x == 0) {
                if (f >= 0) {
                    volatile DmMsg& m = vb->msg[f];
                    m.src = a.src;
                    m.tag = a.tag;
                    m.ctx = a.ctx;
                    m.seq = vb->next_seq;
                    vb->next_seq = vb->next_seq + 1;
                    m.data = a.data;
                    m.bytes = a.bytes;
                    m.consumed = a.consumed;
                    m.cgen = a.cgen;
                    m.rdv = a.rdv;
                    vput(&m.lay, a.lay);
                    if (a.record) *reinterpret_cast<volatile int32_t*>(a.record) = -1;
                    __threadfence_system();
                    m.state = 1;
                    if (f + 1 > hm) vb->hw_msg = f + 1;
                } else if (now_ns() - t0 < kGiveUpNs) {
                    done = false;   // full: let receivers drain it, retry
                } else {
                    vb->err = MPX_ERR_EXHAUSTED;
                }
            }
        }
        if (threadIdx.x == 0) {
            unlock(b);
            slot = done ? 1 : 0;
        }
        __syncthreads();
        if (slot) return;
        __nanosleep(1000);
    }
}

struct PostArgs {
    DmBox* box;
    int32_t src, tag, ctx;   // patterns
    int32_t result;
    uint8_t* dst;            // where the message lands
    int64_t cap;
    int32_t big, pad;        // big: a k_dm_xfer follows this post
    DmLay lay;               // relative to dst
};

// a receive is posted at its stream position
__global__ void __launch_bounds__(kThreads) k_dm_post(const PostArgs a) {
    __shared__ unsigned long long best;
    __shared__ int slot, small_copy;
    DmBox* b = a.box;
    volatile DmBox* vb = b;
    const uint64_t t0 = now_ns();
    if (threadIdx.x == 0) small_copy = 0;
    for (;;) {
        if (threadIdx.x == 0) {
            lock(b);
            volatile DmResult* r = &b->result[a.result];
            r->ready = 0;
            r->ndone = 0;
            r->copied = 0;
            r->xdone = 0;
        }
        __syncthreads();
        const int hm = vb->hw_msg;
        const unsigned long long k = earliest(hm, [&](int i) -> unsigned long long {
            volatile const DmMsg& m = vb->msg[i];
            if (m.state != 1 || !pat_match(a.src, a.tag, a.ctx, m.src, m.tag, m.ctx)) return kNone;
            return ((unsigned long long)m.seq << 12) | (unsigned)i;
        }, &best);
        bool done = true;
        if (k != kNone) {   // the earliest unexpected message
            coop_lay(&b->result[a.result].slay, &vb->msg[(int)(k & 0xFFF)].lay);
            coop_lay(&b->result[a.result].dlay, &a.lay);
            __syncthreads();
            if (threadIdx.x == 0) {
                const int i = (int)(k & 0xFFF);
                volatile DmMsg& m = vb->msg[i];
                publish(&b->result[a.result], m.src, m.tag, m.bytes, m.data, m.consumed, m.cgen, m.rdv, a.dst,
                        a.cap, 1);
                small_copy = m.rdv && !a.big;   // a receive within the eager limit copies here
                m.state = 0;
                int h = hm;
                while (h > 0 && vb->msg[h - 1].state == 0) --h;
                vb->hw_msg = h;
            }
        } else {
            const int hr = vb->hw_recv;
            const int f = first_free(hr, [&](int i) { return vb->recv[i].state == 0; }, &slot);
            if (threadIdx.x == 0) {
                if (f >= 0) {
                    volatile DmRecv& r = vb->recv[f];
                    r.src = a.src;
                    r.tag = a.tag;
                    r.ctx = a.ctx;
                    r.result = a.result;
                    r.dst = a.dst;
                    r.cap = a.cap;
                    vput(&r.lay, a.lay);
                    r.seq = vb->next_seq;
                    vb->next_seq = vb->next_seq + 1;
                    __threadfence_system();
                    r.state = 1;
                    if (f + 1 > hr) vb->hw_recv = f + 1;
                } else if (now_ns() - t0 < kGiveUpNs) {
                    done = false;
                } else {
                    vb->err = MPX_ERR_EXHAUSTED;
                }
            }
        }
        if (threadIdx.x == 0) {
            unlock(b);
            slot = done ? 1 : 0;
        }
        __syncthreads();
        if (slot) break;
        __nanosleep(1000);
    }
    if (small_copy) {   // rendezvous message into a receive of <= eager-limit bytes
        __shared__ DmLay sl;
        volatile DmResult* r = &b->result[a.result];
        coop_lay(&sl, &r->slay);
        __syncthreads();
        chain_copy(sl, (const uint8_t*)r->data, a.lay, a.dst, r->n, threadIdx.x, blockDim.x);
        __syncthreads();
        if (threadIdx.x == 0) rdv_complete(r);
    }
}

// the rendezvous copy of the side that matched second: after k_dm_send on
// the sender's stream (record: the slot the send matched, or -1) or after a
// big receive's k_dm_post on the receiver's stream (record == nullptr: the
// post's own slot `res`)
__global__ void __launch_bounds__(kThreads) k_dm_xfer(DmBox* b, int res, const int32_t* record) {
    // one thread decides for the block: a sender may publish into this slot
    // while the block starts (the decision must be uniform for the barriers)
    __shared__ int go, slot_sh;
    if (threadIdx.x == 0) {
        const int side = record ? 0 : 1;
        const int rs = record ? *reinterpret_cast<const volatile int32_t*>(record) : res;
        int ok = 0;
        if (rs >= 0) {
            volatile DmResult* q = &b->result[rs];
            ok = q->ready && q->rdv && q->copier == side;
        }
        go = ok;
        slot_sh = rs;
    }
    __syncthreads();
    if (!go) return;
    res = slot_sh;
    volatile DmResult* r = &b->result[res];
    __threadfence_system();
    __shared__ DmLay sl, dl;
    coop_lay(&sl, &r->slay);
    coop_lay(&dl, &r->dlay);
    __syncthreads();
    chain_copy(sl, (const uint8_t*)r->data, dl, (uint8_t*)r->dst, r->n, (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
               (int64_t)gridDim.x * blockDim.x);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        if (atomicAdd((unsigned*)&b->result[res].xdone, 1u) == gridDim.x - 1) rdv_complete(r);
    }
}

// wait for a receive's match (one thread spins; the GPU stays free for the
// senders' kernels) and record its status
__global__ void __launch_bounds__(32) k_dm_wait(DmBox* b, int res, DmStatus* st, int64_t cap) {
    if (threadIdx.x) return;
    volatile DmResult* r = &b->result[res];
    volatile DmBox* vb = b;
    unsigned ns = 32;
    while (r->ready == 0) {
        if (vb->err) {
            volatile DmStatus* s = st;
            s->err = vb->err;
            s->src = -1;
            s->tag = -1;
            s->bytes = 0;
            return;
        }
        __nanosleep(ns);
        ns = ns < 1024 ? 2 * ns : ns;
    }
    if (r->rdv)   // rendezvous: the side that matched second is copying
        while (r->copied == 0) {
            __nanosleep(ns);
            ns = ns < 1024 ? 2 * ns : ns;
        }
    __threadfence_system();
    volatile DmStatus* s = st;
    s->src = r->src;
    s->tag = r->tag;
    s->bytes = r->bytes;
    s->err = r->bytes > cap ? MPX_ERR_TRUNCATE : MPX_SUCCESS;
}

// a receive within the eager limit: wait and copy in ONE single-CTA kernel
// (one launch per receive instead of two)
__global__ void __launch_bounds__(kThreads) k_dm_wait_copy(DmBox* b, int res, DmStatus* st, int64_t cap) {
    __shared__ int state;   // 0: failed (box error), 1: copy, 2: rendezvous (already copied)
    __shared__ DmLay sl, dl;
    volatile DmResult* r = &b->result[res];
    volatile DmBox* vb = b;
    if (threadIdx.x == 0) {
        unsigned ns = 32;
        state = 1;
        while (r->ready == 0) {
            if (vb->err) {
                state = 0;
                break;
            }
            __nanosleep(ns);
            ns = ns < 1024 ? 2 * ns : ns;
        }
        if (state && r->rdv) {
            state = 2;
            while (r->copied == 0) {
                __nanosleep(ns);
                ns = ns < 1024 ? 2 * ns : ns;
            }
        }
        __threadfence_system();
    }
    __syncthreads();
    const int stt = state;
    int64_t n = 0;
    if (stt == 1) {
        n = r->bytes < cap ? r->bytes : cap;
        coop_lay(&sl, &r->slay);
        coop_lay(&dl, &r->dlay);
        __syncthreads();
        chain_copy(sl, (const uint8_t*)r->data, dl, (uint8_t*)r->dst, n, threadIdx.x, blockDim.x);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile DmStatus* s = st;
        if (stt == 0) {
            s->err = vb->err;
            s->src = -1;
            s->tag = -1;
            s->bytes = 0;
        } else {
            s->src = r->src;
            s->tag = r->tag;
            s->bytes = r->bytes;
            s->err = r->bytes > cap ? MPX_ERR_TRUNCATE : MPX_SUCCESS;
            if (stt == 1) {
                __threadfence_system();
                *reinterpret_cast<volatile uint32_t*>(r->consumed) = r->cgen;
            }
        }
        __threadfence_system();
        s->done = 1;
    }
}

// copy the part of the message that fits; the last CTA releases the bounce
// buffer and completes the status
__global__ void __launch_bounds__(kThreads) k_dm_copy(DmBox* b, int res, int64_t cap, DmStatus* st) {
    volatile DmResult* r = &b->result[res];
    const bool ok = r->ready != 0;
    const bool rdv = ok && r->rdv;   // already copied at match time (k_dm_wait saw it complete)
    const int64_t n = ok && !rdv ? (r->bytes < cap ? r->bytes : cap) : 0;
    if (n > 0) {   // the bounce buffer (contiguous) into the receive's layout
        __shared__ DmLay sl, dl;
        coop_lay(&sl, &r->slay);
        coop_lay(&dl, &r->dlay);
        __syncthreads();
        chain_copy(sl, (const uint8_t*)r->data, dl, (uint8_t*)r->dst, n, (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                   (int64_t)gridDim.x * blockDim.x);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        if (atomicAdd((unsigned*)&b->result[res].ndone, 1u) == gridDim.x - 1) {
            if (ok && !rdv) {
                uint32_t* c = r->consumed;
                *reinterpret_cast<volatile uint32_t*>(c) = r->cgen;
            }
            __threadfence_system();
            reinterpret_cast<volatile DmStatus*>(st)->done = 1;
        }
    }
}

}  // namespace

namespace {
unsigned xfer_grid(int64_t bytes, int device) {
    const int64_t want = (bytes + (int64_t)kThreads * 64 - 1) / ((int64_t)kThreads * 64);
    const int64_t cap = (int64_t)sm_count(device) * 4;
    return (unsigned)(want < 1 ? 1 : want > cap ? cap : want);
}
}  // namespace

cudaError_t dm_send(DmBox* box, int src, int tag, int ctx, const uint8_t* data, int64_t bytes, uint32_t* consumed,
                    uint32_t cgen, cudaStream_t stream) {
    SendArgs a{box, src, tag, ctx, cgen, data, bytes, consumed, nullptr, 0, 0, dm_contig_lay(0, bytes), nullptr};
    k_dm_send<<<1, kThreads, 0, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t dm_send_packed(DmBox* box, int src, int tag, int ctx, const uint8_t* data, const DmLay& lay,
                           uint8_t* bounce, int64_t bytes, uint32_t* consumed, uint32_t cgen, cudaStream_t stream) {
    SendArgs a{box, src, tag, ctx, cgen, data, bytes, consumed, nullptr, 0, 0, lay, bounce};
    k_dm_send<<<1, kThreads, 0, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t dm_wait_copy(DmBox* box, int result, DmStatus* status, int64_t cap, cudaStream_t stream) {
    k_dm_wait_copy<<<1, kThreads, 0, stream>>>(box, result, status, cap);
    return cudaGetLastError();
}

cudaError_t dm_send_rdv(DmBox* box, int src, int tag, int ctx, const uint8_t* data, const DmLay& lay, int64_t bytes,
                        uint32_t* consumed, uint32_t cgen, int32_t* record, int device, cudaStream_t stream) {
    SendArgs a{box, src, tag, ctx, cgen, data, bytes, consumed, record, 1, 0, lay, nullptr};
    k_dm_send<<<1, kThreads, 0, stream>>>(a);
    k_dm_xfer<<<xfer_grid(bytes, device), kThreads, 0, stream>>>(box, -1, record);
    return cudaGetLastError();
}

cudaError_t dm_post(DmBox* box, int src, int tag, int ctx, int result, uint8_t* dst, const DmLay& lay, int64_t cap,
                    bool big, int device, cudaStream_t stream) {
    PostArgs a{box, src, tag, ctx, result, dst, cap, big ? 1 : 0, 0, lay};
    k_dm_post<<<1, kThreads, 0, stream>>>(a);
    if (big) k_dm_xfer<<<xfer_grid(cap, device), kThreads, 0, stream>>>(box, result, nullptr);
    return cudaGetLastError();
}

cudaError_t dm_wait(DmBox* box, int result, DmStatus* status, int64_t cap, cudaStream_t stream) {
    k_dm_wait<<<1, 32, 0, stream>>>(box, result, status, cap);
    return cudaGetLastError();
}

cudaError_t dm_copy(DmBox* box, int result, int64_t cap, DmStatus* status, int device, cudaStream_t stream) {
    const int64_t want = (cap + (int64_t)kThreads * 64 - 1) / ((int64_t)kThreads * 64);
    const int64_t grid = want < 1 ? 1 : (want > (int64_t)sm_count(device) * 4 ? (int64_t)sm_count(device) * 4 : want);
    k_dm_copy<<<(unsigned)grid, kThreads, 0, stream>>>(box, result, cap, status);
    return cudaGetLastError();
}

DmLay dm_contig_lay(int64_t off, int64_t bytes) {
    DmLay l;
    memset(&l, 0, sizeof l);
    l.c.base = off;
    l.c.L = bytes > 0 ? bytes : 1;
    l.c.depth = 0;
    host_magic((uint64_t)l.c.L, &l.c.m_L, &l.c.s_L);
    int64_t a = 16;
    while (a > 1 && ((off | l.c.L) & (a - 1))) a >>= 1;
    l.align = (int32_t)a;
    return l;
}

cudaError_t preload_dm_kernels() {
    cudaFuncAttributes a;
    cudaError_t e = cudaSuccess, r;
    if ((r = cudaFuncGetAttributes(&a, k_dm_send)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_dm_post)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_dm_wait)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_dm_copy)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_dm_xfer)) != cudaSuccess) e = r;
    if ((r = cudaFuncGetAttributes(&a, k_dm_wait_copy)) != cudaSuccess) e = r;
    return e;
}

}  // namespace mpx
