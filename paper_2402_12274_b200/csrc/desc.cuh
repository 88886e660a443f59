// desc.cuh -- GPU-resident layout descriptors and their device-side walkers.
//
// Two lowered forms of a layout tree (typerep.hpp):
//
//  * Chain: the tree is Rep^k(Run), k <= 4 (vector / hvector / subarray faces
//    / contiguous).  Packed byte P maps to layout offset in closed form:
//      row = P / L, col = P % L, row -> (idx_0..idx_{k-1}) mixed radix,
//      off = base + col + sum idx_i * stride_i.
//    All divisions are by launch constants and use precomputed 64-bit
//    multiply-high magic numbers (Granlund-Montgomery, N = 63).
//
//  * DDesc: the whole DAG flattened into a node array (96 B per node), a
//    child-index table and per-Seq run/byte prefix tables.  Device code
//    descends it exactly like the reference's emit_from / prefix_within
//    (datatype.py:145-153, 155-163, 202-215): divide at Rep nodes, binary
//    search at Seq nodes.
#pragma once

#include <cstdint>

#include <vector_types.h>

namespace mpx {

constexpr int kMaxChain = 4;

struct Chain {
    int64_t base;           // total displacement of the innermost run
    int64_t L;              // run length in bytes
    int32_t depth;          // number of Rep levels (0 = a single run)
    int32_t pad0;
    int64_t cnt[kMaxChain]; // outermost first
    int64_t str[kMaxChain];
    uint64_t m_cnt[kMaxChain];
    int32_t s_cnt[kMaxChain];
    uint64_t m_L;
    int32_t s_L;
    int32_t small;          // rows < 2^31 and counts < 2^31: 32-bit index math
    uint32_t m32_cnt[kMaxChain];
    int32_t s32_cnt[kMaxChain];
};

// ---- span lowering (struct / indexed / nested types with small elements) ----
// Outer Rep levels stay symbolic; everything below is decomposed on the host
// into chunks of consecutive elements of a small "body" (<= kSpanMaxBody bytes
// of span).  A chunk's source span is contiguous, so a warp stages it in
// shared memory with aligned 16-byte loads and produces the other side word by
// word through the body's byte maps.
constexpr int kSpanMaxBody = 256;
constexpr int kSpanMaxRuns = 32;
constexpr int kSpanMaxBodies = 8;
#ifndef MPX_SPAN_STAGE
#define MPX_SPAN_STAGE 3072
#endif
constexpr int kSpanStage = MPX_SPAN_STAGE;     // bytes staged per warp per buffer (plus 32 B slack): one
                                      // chunk per cfg3 block (<= 64 x 40 B) -- fewer, larger units
constexpr int kSpanMaxOuter = 2;

// one element of a span chunk: its runs relative to the element's span start
struct SpanBody {
    int32_t span_len;       // element span bytes (<= kSpanMaxBody)
    int32_t nbytes;         // payload bytes per element
    int32_t nruns;
    int32_t pad;
    int16_t roff[kSpanMaxRuns];  // run offset in the element span
    int16_t rpk[kSpanMaxRuns];   // run offset in the element's packed bytes
    int16_t rlen[kSpanMaxRuns];
};
static_assert(sizeof(SpanBody) % 16 == 0, "SpanBody must be 16-byte sized");

struct SpanChunk {
    int64_t src;            // span start of element 0 (layout offset)
    int64_t pk;             // packed offset of element 0
    int32_t span;           // layout bytes covered: (n - 1) * stride + span_len (raw: stride)
    int32_t plen;           // packed bytes: n * nbytes (raw: stride)
    int32_t n;              // elements
    int32_t body;           // body index, -1 = raw contiguous piece of `stride` bytes
    int32_t stride;         // element stride in bytes (>= span_len when n > 1)
    int16_t perm[2];        // word-gather spec for [unpack, pack] (index into SpanPlan::perms)
    int32_t pad[2];
};
static_assert(sizeof(SpanChunk) == 48, "SpanChunk layout");

// ---- periodic word gather (k_perm) ----
// For a chunk of n equal elements the output stream (packed bytes for pack,
// the layout span for unpack) is a periodic function of the input stream:
// output element size Eo, input element size Ei, and every E elements
// (E in {1,2,4}, chosen so E*Eo and E*Ei are multiples of 4) the pattern of
// 32-bit output words repeats with the input advanced by E*Ei bytes.  A warp
// step produces W = M*E*Eo/4 consecutive aligned output words (lane l owns
// words l, l+32, ... < W: its "slots"); each output word is assembled from a
// window of <= 4 consecutive input words with byte_perm selectors.  The
// selectors depend only on the slot and on the two address phases
// (output address & 3, input address & 3), so the host precomputes them:
// tab[(po * 4 + ap) * W + j].  byte_perm reads only the low 16 bits of its
// selector, so the entry words feed it directly.
constexpr int kPermMaxSlots = 4;     // W <= 128 words per step
constexpr int kPermMaxSpecs = 16;

// Byte form (PermSpec::pad == 1, bodies whose words spread over > 16 input
// bytes): wo4 = input offset of byte 0, lo = cover / j as below, hi = int16
// deltas of bytes 1 and 2, mix = int16 delta of byte 3.
struct PermEntry {
    int32_t wo4;            // window start: byte offset from the staged input's word 0 (+ step * 4 * Dw)
    uint32_t lo;            // bits 0-15: byte_perm selector over window words (0, 1);
                            // 16-19: cover (byte i is written; unpack leaves layout gaps alone);
                            // 20-23: byte i comes from window words (2, 3); 24-31: the word's
                            // index j in the step (entries are compacted: uncovered words dropped)
    uint32_t hi;            // byte_perm selector over window words (2, 3)
    uint32_t mix;           // byte_perm selector merging the two halves
};
static_assert(sizeof(PermEntry) == 16, "PermEntry layout");

struct PermSpec {
    int32_t W;              // output words per warp step
    int32_t Dw;             // input words advanced per step
    int32_t ns;             // slots per lane: ceil(max(wc) / 32)
    int32_t pad;            // 0: word windows; 1: per-byte gathers (PermEntry byte form)
    const PermEntry* tab;   // [16][W]: per phase variant, the words with a written byte first
    uint8_t wc[16];         // per phase variant: words with a written byte (entries used)
};
static_assert(sizeof(PermSpec) == 40, "PermSpec layout");

struct SpanPlan {
    const SpanChunk* chunks;
    const SpanBody* bodies;
    const PermSpec* perms;              // nullptr: no word-gather form (k_span fallback)
    int32_t nchunks, nbodies;
    int32_t nperms, outer_depth;
    int64_t outer_cnt[kSpanMaxOuter];
    int64_t outer_str[kSpanMaxOuter];   // layout stride per outer level
    int64_t outer_pk[kSpanMaxOuter];    // packed stride per outer level
    int64_t nunits;                     // prod(outer_cnt) * nchunks
    uint64_t m_nchunks;                 // magic divisors for the unit decode
    uint64_t m_outer1;
    int32_t s_nchunks, s_outer1;
    int32_t ns_max[2];                  // most slots any spec needs, [unpack, pack]
    // iov enumeration (k_iov_span): per chunk {segments before it within one
    // outer element, run length if it starts a raw run (0 otherwise)}; raw
    // pieces that continue a run add no segment
    const longlong2* iovc;
    int64_t segs_outer;                 // segments per outer element
};

struct DNode {
    int32_t kind;           // 0 empty, 1 run, 2 rep, 3 seq
    int32_t nkids;          // seq
    int32_t child;          // rep: body node index; seq: first index in kid table
    int32_t pref;           // seq: first index in the prefix tables
    int64_t a, b, c;        // run: off, len ; rep: count, stride, base
    int64_t runs, nbytes;
    int64_t body_runs, body_nbytes;
    uint64_t m_runs, m_bytes;
    int32_t s_runs, s_bytes;
};
static_assert(sizeof(DNode) == 96, "DNode layout");

struct DDesc {
    const DNode* nodes;
    const int32_t* kids;
    const int64_t* rp;
    const int64_t* bp;
    int32_t root;
    int32_t pad;
    int64_t runs;
    int64_t nbytes;
};

// magic for q = floor(n / d), 0 <= n < 2^63: m = ceil(2^(63+l)/d), l = ceil(log2 d)
inline void host_magic(uint64_t d, uint64_t* m, int32_t* s) {
    if (d <= 1) { *m = 0; *s = 0; return; }
    const int l = 64 - __builtin_clzll(d - 1);
    const unsigned __int128 num = (unsigned __int128)1 << (63 + l);
    *m = (uint64_t)((num + d - 1) / d);
    *s = l - 1;
}

// 32-bit variant, 0 <= n < 2^31: m = ceil(2^(31+l)/d)
inline void host_magic32(uint32_t d, uint32_t* m, int32_t* s) {
    if (d <= 1) { *m = 0; *s = 0; return; }
    const int l = 32 - __builtin_clz(d - 1);
    const uint64_t num = (uint64_t)1 << (31 + l);
    *m = (uint32_t)((num + d - 1) / d);
    *s = l - 1;
}

#ifdef __CUDACC__
__device__ __forceinline__ uint32_t fdiv32(uint32_t n, uint32_t m, int32_t s) {
    return m ? (__umulhi(n, m) >> s) : n;
}

// layout offset of the start of row r of a chain
__device__ __forceinline__ int64_t chain_row(const Chain& c, int64_t r) {
    int64_t off = c.base;
    if (c.depth == 0) return off;
    if (c.small) {
        uint32_t rr = (uint32_t)r;
#pragma unroll
        for (int i = kMaxChain - 1; i >= 1; --i) {
            if (i < c.depth) {
                const uint32_t q = fdiv32(rr, c.m32_cnt[i], c.s32_cnt[i]);
                off += (int64_t)(int32_t)(rr - q * (uint32_t)c.cnt[i]) * c.str[i];
                rr = q;
            }
        }
        return off + (int64_t)rr * c.str[0];
    }
    uint64_t rr = (uint64_t)r;
#pragma unroll
    for (int i = kMaxChain - 1; i >= 1; --i) {
        if (i < c.depth) {
            const uint64_t q = __umul64hi(rr, c.m_cnt[i]) >> c.s_cnt[i];
            const uint64_t qq = c.m_cnt[i] ? q : rr;
            off += (int64_t)(rr - qq * (uint64_t)c.cnt[i]) * c.str[i];
            rr = qq;
        }
    }
    return off + (int64_t)rr * c.str[0];
}

__device__ __forceinline__ uint64_t fdiv(uint64_t n, uint64_t m, int32_t s) {
    return m ? (__umul64hi(n, m) >> s) : n;
}

struct RunLoc {
    int64_t k;      // run index
    int64_t src;    // layout offset of the run start
    int64_t len;    // run length
    int64_t poff;   // packed offset of the run start
};

// largest i in [0, n) with a[i] <= key (a[0] == 0 <= key)
__device__ __forceinline__ int prefix_search(const int64_t* __restrict__ a, int n, int64_t key) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(a + mid) <= key) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// run k -> (layout offset, length, packed offset); emit_from seek, datatype.py:145-153,202-206
__device__ __forceinline__ RunLoc locate_run(const DDesc& d, int64_t k) {
    int32_t ni = d.root;
    int64_t shift = 0, poff = 0, kk = k;
    for (;;) {
        const DNode* nd = d.nodes + ni;
        const int kind = __ldg(&nd->kind);
        if (kind == 1) return RunLoc{k, shift + __ldg(&nd->a), __ldg(&nd->b), poff};
        if (kind == 2) {
            const uint64_t q = fdiv((uint64_t)kk, __ldg(&nd->m_runs), __ldg(&nd->s_runs));
            kk -= (int64_t)q * __ldg(&nd->body_runs);
            shift += __ldg(&nd->c) + (int64_t)q * __ldg(&nd->b);
            poff += (int64_t)q * __ldg(&nd->body_nbytes);
            ni = __ldg(&nd->child);
        } else {
            const int pref = __ldg(&nd->pref);
            const int i = prefix_search(d.rp + pref, __ldg(&nd->nkids), kk);
            kk -= __ldg(d.rp + pref + i);
            poff += __ldg(d.bp + pref + i);
            ni = __ldg(d.kids + __ldg(&nd->child) + i);
        }
    }
}

// packed byte p (< nbytes) -> the run containing it; prefix_within-style descent
__device__ __forceinline__ RunLoc locate_byte(const DDesc& d, int64_t p) {
    int32_t ni = d.root;
    int64_t shift = 0, poff = 0, k = 0, pp = p;
    for (;;) {
        const DNode* nd = d.nodes + ni;
        const int kind = __ldg(&nd->kind);
        if (kind == 1) return RunLoc{k, shift + __ldg(&nd->a), __ldg(&nd->b), poff};
        if (kind == 2) {
            const uint64_t q = fdiv((uint64_t)pp, __ldg(&nd->m_bytes), __ldg(&nd->s_bytes));
            const int64_t bn = __ldg(&nd->body_nbytes);
            pp -= (int64_t)q * bn;
            k += (int64_t)q * __ldg(&nd->body_runs);
            shift += __ldg(&nd->c) + (int64_t)q * __ldg(&nd->b);
            poff += (int64_t)q * bn;
            ni = __ldg(&nd->child);
        } else {
            const int pref = __ldg(&nd->pref);
            const int i = prefix_search(d.bp + pref, __ldg(&nd->nkids), pp);
            pp -= __ldg(d.bp + pref + i);
            k += __ldg(d.rp + pref + i);
            poff += __ldg(d.bp + pref + i);
            ni = __ldg(d.kids + __ldg(&nd->child) + i);
        }
    }
}

// closed-form layout offset of packed byte P for a chain
__device__ __forceinline__ int64_t chain_off(const Chain& c, int64_t P) {
    const uint64_t row = fdiv((uint64_t)P, c.m_L, c.s_L);
    int64_t off = c.base + (P - (int64_t)row * c.L);
    if (c.depth == 0) return off;
    uint64_t r = row;
#pragma unroll
    for (int i = kMaxChain - 1; i >= 1; --i) {
        if (i < c.depth) {
            const uint64_t q = fdiv(r, c.m_cnt[i], c.s_cnt[i]);
            off += (int64_t)(r - q * (uint64_t)c.cnt[i]) * c.str[i];
            r = q;
        }
    }
    return off + (int64_t)r * c.str[0];
}
#endif

}  // namespace mpx
