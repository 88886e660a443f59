// plan.cpp -- tree -> {chain | device descriptor} lowering and overlap analysis.
#include "plan.hpp"

#include <algorithm>
#include <deque>
#include <climits>
#include <cstring>
#include <tuple>
#include <map>
#include <set>
#include <mutex>
#include <unordered_map>

namespace mpx {

namespace {
cudaStream_t upload_stream(int device);
cudaMemPool_t desc_pool(int device);
}  // namespace

// Never blocks: the descriptor goes back to its stream-ordered pool on the
// upload stream (cudaFree would synchronise the device, which may hold
// streams parked in stream-memop waits on other ranks).
Plan::~Plan() {
    if (blob || ready) {
        int cur = -1;
        cudaGetDevice(&cur);
        if (device >= 0 && cur != device) cudaSetDevice(device);
        if (blob) cudaFreeAsync(blob, upload_stream(device));
        if (ready) cudaEventDestroy(ready);
        if (device >= 0 && cur != device && cur >= 0) cudaSetDevice(cur);
    }
}

// Order `stream` after the plan's descriptor upload.  The host never blocks
// on the upload: another rank of this process may hold a stream parked in a
// stream-memop wait that this very call is about to release, and a host wait
// on GPU work could then stall behind it (hardware queues are shared once a
// process has more streams than CUDA_DEVICE_MAX_CONNECTIONS).
cudaError_t plan_wait(Plan& p, cudaStream_t stream) {
    if (!p.ready || p.ready_seen.load(std::memory_order_acquire)) return cudaSuccess;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaError_t ce = cudaStreamIsCapturing(stream, &cs);
    if (ce != cudaSuccess) return ce;
    // inside stream capture no event may be queried: the graph waits on the
    // (long completed) upload event as an external dependency
    if (cs != cudaStreamCaptureStatusNone) return cudaStreamWaitEvent(stream, p.ready, cudaEventWaitExternal);
    cudaError_t q = cudaEventQuery(p.ready);
    if (q == cudaSuccess) {
        p.ready_seen.store(true, std::memory_order_release);
        return cudaSuccess;
    }
    if (q != cudaErrorNotReady) return q;
    cudaGetLastError();
    return cudaStreamWaitEvent(stream, p.ready, 0);
}

namespace {
// stream-ordered pool for descriptors (no hidden inter-stream dependencies)
cudaMemPool_t desc_pool(int device) {
    static std::mutex mu;
    static std::map<int, cudaMemPool_t> pools;
    std::lock_guard<std::mutex> g(mu);
    auto it = pools.find(device);
    if (it != pools.end()) return it->second;
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    int zero = 0;
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &zero);
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    pools[device] = pool;
    return pool;
}

// Pinned staging for descriptor uploads.  A cudaMemcpyAsync from pageable
// memory may hold the calling thread until the copy engine has drained the
// driver's bounded staging buffers -- and with several ranks of one process
// on a device, that drain can sit behind work that only another (blocked)
// rank thread would release.  From pinned memory the call returns at once.
// A chunk is reused only once its latest upload has completed (checked with
// cudaEventQuery, never waited for); otherwise another chunk is added.
class UploadArena {
  public:
    cudaError_t copy(cudaStream_t up, void* dst, const void* src, size_t n) {
        std::lock_guard<std::mutex> g(mu_);
        Chunk* c = nullptr;
        for (auto& k : chunks_)
            if (k.cap - k.used >= n) { c = &k; break; }
        if (!c)
            for (auto& k : chunks_)
                if (k.cap >= n && cudaEventQuery(k.last) == cudaSuccess) { k.used = 0; c = &k; break; }
        cudaGetLastError();
        if (!c) {
            Chunk k;
            k.cap = std::max<size_t>(n, size_t(8) << 20);
            cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&k.base), k.cap, cudaHostAllocPortable);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&k.last, cudaEventDisableTiming);
            if (e != cudaSuccess) return e;
            chunks_.push_back(k);
            c = &chunks_.back();
        }
        uint8_t* at = c->base + c->used;
        std::memcpy(at, src, n);
        c->used += (n + 255) & ~size_t(255);
        if (c->used > c->cap) c->used = c->cap;
        cudaError_t e = cudaMemcpyAsync(dst, at, n, cudaMemcpyHostToDevice, up);
        if (e == cudaSuccess) e = cudaEventRecord(c->last, up);
        return e;
    }

  private:
    struct Chunk {
        uint8_t* base = nullptr;
        size_t cap = 0, used = 0;
        cudaEvent_t last = nullptr;
    };
    std::mutex mu_;
    std::deque<Chunk> chunks_;   // stable addresses
};

UploadArena& upload_arena(int device) {
    static std::mutex mu;
    static std::map<int, UploadArena*> arenas;   // never destroyed
    std::lock_guard<std::mutex> g(mu);
    auto& a = arenas[device];
    if (!a) a = new UploadArena();
    return *a;
}

// one internal upload stream per device: descriptor uploads never
// synchronise (or even touch) the caller's stream
cudaStream_t upload_stream(int device) {
    static std::mutex mu;
    static std::map<int, cudaStream_t> streams;
    std::lock_guard<std::mutex> g(mu);
    auto it = streams.find(device);
    if (it != streams.end()) return it->second;
    cudaStream_t s = nullptr;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    streams[device] = s;
    return s;
}
}  // namespace

namespace {

int64_t pow2_div(int64_t v) {  // largest power of two (<=16) dividing v
    v = v < 0 ? -v : v;
    if (v == 0) return 16;
    int64_t a = 1;
    while (a < 16 && (v % (a * 2)) == 0) a *= 2;
    return a;
}

// Conservative structural test: can two runs of this subtree touch the same byte?
bool may_overlap(const Node* n) {
    switch (n->kind) {
    case Kind::Empty:
    case Kind::Run: return false;
    case Kind::Rep: {
        const int64_t span = n->body->max_end - n->body->min_off;
        const int64_t st = n->stride < 0 ? -n->stride : n->stride;
        return st < span || may_overlap(n->body.get());
    }
    case Kind::Seq: {
        std::vector<std::pair<int64_t, int64_t>> iv;
        iv.reserve(n->kids.size());
        for (const auto& c : n->kids) {
            if (may_overlap(c.get())) return true;
            iv.emplace_back(c->min_off, c->max_end);
        }
        std::sort(iv.begin(), iv.end());
        for (size_t i = 1; i < iv.size(); ++i)
            if (iv[i].first < iv[i - 1].second) return true;
        return false;
    }
    }
    return true;
}

// Exact test on small layouts: sort the iov and look for intersecting runs.
bool exact_overlap(const Node* n) {
    std::vector<int64_t> flat;
    tree::enumerate(n, 0, flat, n->runs);
    const size_t r = flat.size() / 2;
    std::vector<std::pair<int64_t, int64_t>> iv(r);
    for (size_t i = 0; i < r; ++i) iv[i] = {flat[2 * i], flat[2 * i] + flat[2 * i + 1]};
    std::sort(iv.begin(), iv.end());
    for (size_t i = 1; i < r; ++i)
        if (iv[i].first < iv[i - 1].second) return true;
    return false;
}

struct Flattener {
    std::vector<DNode> nodes;
    std::vector<int32_t> kids;
    std::vector<int64_t> rp, bp;
    std::unordered_map<const Node*, int32_t> memo;

    int32_t add(const Node* n) {
        auto it = memo.find(n);
        if (it != memo.end()) return it->second;
        DNode d;
        std::memset(&d, 0, sizeof d);
        d.kind = (int32_t)n->kind;
        d.runs = n->runs;
        d.nbytes = n->nbytes;
        if (n->kind == Kind::Run) {
            d.a = n->off;
            d.b = n->len;
        } else if (n->kind == Kind::Rep) {
            d.a = n->count;
            d.b = n->stride;
            d.c = n->base;
            d.body_runs = n->body->runs;
            d.body_nbytes = n->body->nbytes;
            host_magic((uint64_t)d.body_runs, &d.m_runs, &d.s_runs);
            host_magic((uint64_t)d.body_nbytes, &d.m_bytes, &d.s_bytes);
            d.child = add(n->body.get());
        } else if (n->kind == Kind::Seq) {
            std::vector<int32_t> ids;
            ids.reserve(n->kids.size());
            for (const auto& c : n->kids) ids.push_back(add(c.get()));
            d.nkids = (int32_t)n->kids.size();
            d.child = (int32_t)kids.size();
            kids.insert(kids.end(), ids.begin(), ids.end());
            d.pref = (int32_t)rp.size();
            rp.insert(rp.end(), n->run_prefix.begin(), n->run_prefix.end());
            bp.insert(bp.end(), n->byte_prefix.begin(), n->byte_prefix.end());
        }
        const int32_t id = (int32_t)nodes.size();
        nodes.push_back(d);
        memo.emplace(n, id);
        return id;
    }
};

// ------------------------------------------------------------ span lowering
class SpanBuilder {
  public:
    static constexpr int64_t kMaxChunks = int64_t(1) << 21;
    std::vector<SpanChunk> chunks;
    std::vector<SpanBody> bodies;
    bool ok = true;

    bool small(const Node* n) const {
        return n->runs > 0 && n->runs <= 32 && n->max_end - n->min_off <= kSpanMaxBody;
    }

    void emit(const Node* n, int64_t shift, int64_t poff) {
        if (!ok || n->runs == 0) return;
        if ((int64_t)chunks.size() > kMaxChunks) { ok = false; return; }
        // a small Rep of small elements stays a strided chunk (one shared body
        // and word-gather period) rather than becoming a one-element body
        const bool strided = n->kind == Kind::Rep && n->count > 1 && small(n->body.get()) &&
                             n->stride >= n->body->max_end - n->body->min_off;
        if (small(n) && !strided) {   // chunk src = span start of the element
            add(shift + n->min_off, poff, 1, body_of(n), 0);
            return;
        }
        switch (n->kind) {
        case Kind::Run: {   // large contiguous run: raw pieces
            const int64_t piece = kSpanStage - 16;
            for (int64_t o = 0; o < n->len; o += piece)
                add_raw(shift + n->off + o, poff + o, std::min(piece, n->len - o));
            return;
        }
        case Kind::Rep: {
            const Node* b = n->body.get();
            if (small(b)) {
                const int64_t span = b->max_end - b->min_off;
                if (n->stride < span) {   // element spans interleave or stride < 0
                    ok = false;
                    return;
                }
                const int64_t room = kSpanStage - 16;
                int64_t epc = n->stride > 0 ? (room - span) / n->stride + 1 : 1;
                epc = std::max<int64_t>(1, std::min({epc, room / std::max<int64_t>(1, b->nbytes), n->count}));
                const int body = body_of(b);
                for (int64_t k = 0; k < n->count && ok; k += epc)
                    add(shift + n->base + b->min_off + k * n->stride, poff + k * b->nbytes,
                        std::min(epc, n->count - k), body, n->stride);
                return;
            }
            for (int64_t k = 0; k < n->count && ok; ++k)
                emit(b, shift + n->base + k * n->stride, poff + k * b->nbytes);
            return;
        }
        case Kind::Seq:
            for (size_t i = 0; i < n->kids.size() && ok; ++i) emit(n->kids[i].get(), shift, poff + n->byte_prefix[i]);
            return;
        default: return;
        }
    }

  private:
    std::map<std::vector<int64_t>, int> ids_;

    // body = the element's runs relative to its span start (dedupe key)
    int body_of(const Node* n) {
        std::vector<int64_t> runs;
        tree::enumerate(n, -n->min_off, runs, 64);
        auto it = ids_.find(runs);
        if (it != ids_.end()) return it->second;
        const int nr = (int)(runs.size() / 2);
        if ((int)bodies.size() >= kSpanMaxBodies || nr > kSpanMaxRuns) { ok = false; return 0; }
        SpanBody b;
        std::memset(&b, 0, sizeof b);
        b.span_len = (int32_t)(n->max_end - n->min_off);
        b.nbytes = (int32_t)n->nbytes;
        b.nruns = nr;
        std::vector<bool> seen((size_t)b.span_len, false);
        int64_t q = 0;
        for (int r = 0; r < nr; ++r) {
            b.roff[r] = (int16_t)runs[2 * r];
            b.rlen[r] = (int16_t)runs[2 * r + 1];
            b.rpk[r] = (int16_t)q;
            for (int64_t x = 0; x < runs[2 * r + 1]; ++x) {
                if (seen[(size_t)(runs[2 * r] + x)]) { ok = false; return 0; }   // self-overlapping element
                seen[(size_t)(runs[2 * r] + x)] = true;
            }
            q += runs[2 * r + 1];
        }
        const int id = (int)bodies.size();
        bodies.push_back(b);
        ids_[runs] = id;
        return id;
    }

    void add(int64_t src, int64_t pk, int64_t n, int body, int64_t stride) {
        if (!ok) return;
        SpanChunk c;
        std::memset(&c, 0, sizeof c);
        c.src = src;
        c.pk = pk;
        c.n = (int32_t)n;
        c.body = body;
        c.stride = (int32_t)(n > 1 ? stride : 0);
        c.span = (int32_t)((n - 1) * c.stride + bodies[body].span_len);
        c.plen = (int32_t)(n * bodies[body].nbytes);
        chunks.push_back(c);
    }

    void add_raw(int64_t src, int64_t pk, int64_t len) {
        SpanChunk c;
        std::memset(&c, 0, sizeof c);
        c.src = src;
        c.pk = pk;
        c.n = 1;
        c.body = -1;
        c.stride = (int32_t)len;
        c.span = (int32_t)len;
        c.plen = (int32_t)len;
        chunks.push_back(c);
    }
};

int64_t floor_div(int64_t a, int64_t b) {   // b > 0
    return a >= 0 ? a / b : -((-a + b - 1) / b);
}

// One table entry from the input offsets r[i] of output bytes i (cov[i]:
// byte written) at input phase ap; false if the bytes span >= 16 input bytes.
bool make_entry(const int64_t r[4], const bool cov[4], int ap, PermEntry* en, bool bytes) {
    std::memset(en, 0, sizeof *en);
    int64_t mn = INT64_MAX;
    for (int i = 0; i < 4; ++i)
        if (cov[i]) mn = std::min(mn, ap + r[i]);
    if (mn == INT64_MAX) return true;
    if (bytes) {   // byte gather: byte 0's offset + int16 deltas of bytes 1-3
        int64_t first = 0;      // input offset of the first covered byte (may be negative)
        bool have = false;
        uint32_t cover = 0;
        for (int i = 0; i < 4; ++i)
            if (cov[i]) {
                if (!have) first = ap + r[i];
                have = true;
                cover |= 1u << i;
            }
        int64_t d[4];
        for (int i = 0; i < 4; ++i) {
            d[i] = cov[i] ? ap + r[i] - first : 0;   // uncovered bytes re-read byte 0's address
            if (d[i] < INT16_MIN || d[i] > INT16_MAX) return false;
        }
        if (first < INT32_MIN || first > INT32_MAX) return false;
        en->wo4 = (int32_t)first;
        en->lo = cover << 16;
        en->hi = ((uint32_t)d[1] & 0xFFFF) | ((uint32_t)d[2] << 16);
        en->mix = ((uint32_t)d[3] & 0xFFFF) | ((uint32_t)d[0] << 16);
        return true;
    }
    const int64_t wo = floor_div(mn, 4);
    if (wo < INT16_MIN || wo > INT16_MAX) return false;
    en->wo4 = (int32_t)(4 * wo);
    uint32_t s01 = 0, s23 = 0, pairs = 0, cover = 0;
    for (int i = 0; i < 4; ++i) {
        if (!cov[i]) continue;
        const int64_t rel = ap + r[i] - 4 * wo;
        if (rel < 0 || rel >= 16) return false;
        const uint32_t wi = (uint32_t)(rel >> 2), bi = (uint32_t)(rel & 3);
        const uint32_t nib = (wi & 1) * 4 + bi;
        if (wi >> 1) {
            s23 |= nib << (4 * i);
            pairs |= 1u << i;
        } else {
            s01 |= nib << (4 * i);
        }
        cover |= 1u << i;
    }
    uint32_t mixsel = 0;
    for (int i = 0; i < 4; ++i) mixsel |= (uint32_t)(i + ((pairs >> i) & 1) * 4) << (4 * i);
    en->lo = s01 | (cover << 16) | (pairs << 20);
    en->hi = s23;
    en->mix = mixsel;
    return true;
}

// Append one phase variant (W entries, entry j for step word j) with the
// words that write a byte first; returns their count.
int push_variant(std::vector<PermEntry>& var, std::vector<PermEntry>* tab) {
    int wc = 0;
    for (size_t j = 0; j < var.size(); ++j) {
        var[j].lo |= (uint32_t)j << 24;
        if ((var[j].lo >> 16) & 0xF) tab->push_back(var[j]), ++wc;
    }
    PermEntry z;
    std::memset(&z, 0, sizeof z);
    for (size_t j = (size_t)wc; j < var.size(); ++j) tab->push_back(z);
    return wc;
}

// Word-gather tables for one (element map, direction): output element of Eo
// bytes, input element of Ei bytes, map[t] = input offset of output byte t
// within its element (-1: not written).  False if the period or a word's
// input window is too wide for k_perm.
// Tables for M periods per step (W = M * P words) into `out`; false if a
// word's input bytes spread over >= 16 bytes.
bool perm_tables(int64_t Eo, int64_t Ei, int64_t E, int64_t M, const std::vector<int64_t>& map, PermSpec* spec,
                 std::vector<PermEntry>* out, bool bytes) {
    const int64_t W = M * E * Eo / 4;
    const int64_t Din = M * E * Ei;      // input bytes per step (multiple of 4)
    spec->W = (int32_t)W;
    spec->Dw = (int32_t)(Din / 4);
    spec->pad = bytes ? 1 : 0;
    int wcmax = 0;
    for (int po = 0; po < 4; ++po) {
        for (int ap = 0; ap < 4; ++ap) {
            std::vector<PermEntry> var((size_t)W);
            for (int64_t j = 0; j < W; ++j) {
                int64_t r[4];
                bool cov[4];
                for (int i = 0; i < 4; ++i) {
                    // one step later, so every byte of the slot is a real byte
                    const int64_t q = 4 * j + i - po + 4 * W;
                    const int64_t e = q / Eo, t = q % Eo;
                    cov[i] = map[(size_t)t] >= 0;
                    r[i] = cov[i] ? e * Ei + map[(size_t)t] - Din : 0;
                }
                if (!make_entry(r, cov, ap, &var[(size_t)j], bytes)) return false;
            }
            const int wc = push_variant(var, out);
            spec->wc[po * 4 + ap] = (uint8_t)wc;
            wcmax = std::max(wcmax, wc);
        }
    }
    spec->ns = (wcmax + 31) / 32;
    return true;
}

bool build_perm(int64_t Eo, int64_t Ei, const std::vector<int64_t>& map, PermSpec* spec,
                std::vector<PermEntry>* tab) {
    int64_t E = 1;
    while (((E * Eo) % 4) || ((E * Ei) % 4)) E *= 2;
    const int64_t P = E * Eo / 4;
    const int64_t wmax = 32 * kPermMaxSlots;
    if (P > wmax) return false;
    // Periods per step: fewest slots per lane first (registers / occupancy),
    // then the best lane use at address phase (0, 0) -- the common case of
    // aligned buffers -- counting only words that write a byte.
    PermSpec best{};
    std::vector<PermEntry> best_tab;
    double best_eff = -1;
    // word windows when every output word's bytes lie within 16 input bytes,
    // else per-byte gathers (structs with wide padding)
    bool bytes = false;
    {
        PermSpec probe{};
        std::vector<PermEntry> t;
        if (!perm_tables(Eo, Ei, E, 1, map, &probe, &t, false)) bytes = true;
    }
    static const int64_t force_m = getenv("MPX_PERM_M") ? atoll(getenv("MPX_PERM_M")) : 0;   // A/B experiments
    for (int64_t m = 1; m * P <= wmax; ++m) {
        if (force_m > 0 && m != force_m && force_m * P <= wmax) continue;
        PermSpec sp{};
        std::vector<PermEntry> t;
        if (!perm_tables(Eo, Ei, E, m, map, &sp, &t, bytes)) return false;
        const int wc0 = sp.wc[0];
        const double eff = wc0 ? double(wc0) / double(32 * ((wc0 + 31) / 32)) : 0.0;
        if (best_eff < 0 || sp.ns < best.ns || (sp.ns == best.ns && eff > best_eff + 1e-9)) {
            best = sp;
            best_tab.swap(t);
            best_eff = eff;
        }
    }
    *spec = best;
    spec->tab = reinterpret_cast<const PermEntry*>((uintptr_t)tab->size());   // patched at upload
    tab->insert(tab->end(), best_tab.begin(), best_tab.end());
    return true;
}

// Single-element chunks have no period: one step of W >= ceil((Eo + 3) / 4)
// words covers the element at any output phase; bytes outside it are left
// uncovered.
bool build_perm_single(int64_t Eo, const std::vector<int64_t>& map, PermSpec* spec,
                       std::vector<PermEntry>* tab) {
    const int64_t need = (Eo + 3 + 3) / 4;
    if (need > 32 * kPermMaxSlots) return false;
    const int64_t W = need;
    auto build = [&](bool bytes, PermSpec* sp, std::vector<PermEntry>* out) {
        sp->W = (int32_t)W;
        sp->Dw = 0;
        sp->pad = bytes ? 1 : 0;
        int wcmax = 0;
        for (int po = 0; po < 4; ++po) {
            for (int ap = 0; ap < 4; ++ap) {
                std::vector<PermEntry> var((size_t)W);
                for (int64_t j = 0; j < W; ++j) {
                    int64_t r[4];
                    bool cov[4];
                    for (int i = 0; i < 4; ++i) {
                        const int64_t q = 4 * j + i - po;
                        cov[i] = q >= 0 && q < Eo && map[(size_t)q] >= 0;
                        r[i] = cov[i] ? map[(size_t)q] : 0;
                    }
                    if (!make_entry(r, cov, ap, &var[(size_t)j], bytes)) return false;
                }
                const int wc = push_variant(var, out);
                sp->wc[po * 4 + ap] = (uint8_t)wc;
                wcmax = std::max(wcmax, wc);
            }
        }
        sp->ns = (wcmax + 31) / 32;
        return true;
    };
    std::vector<PermEntry> t;
    if (!build(false, spec, &t)) {   // word windows, else per-byte gathers
        t.clear();
        if (!build(true, spec, &t)) return false;
    }
    spec->tab = reinterpret_cast<const PermEntry*>((uintptr_t)tab->size());
    tab->insert(tab->end(), t.begin(), t.end());
    return true;
}

// Attach word-gather specs to every chunk; false leaves the plan on k_span.
bool build_perms(std::vector<SpanChunk>& chunks, const std::vector<SpanBody>& bodies, Plan* p) {
    std::map<std::tuple<int, int64_t, int>, int> ids;   // (body, stride, pack) -> spec
    std::vector<PermSpec> specs;
    std::vector<PermEntry> tab;
    for (auto& c : chunks) {
        for (int pack = 0; pack < 2; ++pack) {
            int64_t S;
            if (c.body < 0) S = 4;
            else if (c.n > 1) S = c.stride;
            else S = -1;                          // single element: no period
            const auto key = std::make_tuple(c.body, S, pack);
            auto it = ids.find(key);
            if (it == ids.end()) {
                if ((int)specs.size() >= 2 * kPermMaxSpecs) return false;
                std::vector<int64_t> map;
                int64_t Eo, Ei;
                if (c.body < 0) {
                    Eo = Ei = 4;
                    map = {0, 1, 2, 3};
                } else {
                    const SpanBody& b = bodies[c.body];
                    if (S < 0) {
                        Eo = pack ? b.nbytes : b.span_len;
                        map.assign((size_t)Eo, -1);
                        for (int r = 0; r < b.nruns; ++r)
                            for (int x = 0; x < b.rlen[r]; ++x) {
                                if (pack) map[(size_t)(b.rpk[r] + x)] = b.roff[r] + x;
                                else map[(size_t)(b.roff[r] + x)] = b.rpk[r] + x;
                            }
                        PermSpec sp;
                        if (!build_perm_single(Eo, map, &sp, &tab)) return false;
                        it = ids.emplace(key, (int)specs.size()).first;
                        specs.push_back(sp);
                        c.perm[pack] = (int16_t)it->second;
                        continue;
                    }
                    if (pack) {
                        Eo = b.nbytes;
                        Ei = S;
                        map.assign((size_t)Eo, -1);
                        for (int r = 0; r < b.nruns; ++r)
                            for (int x = 0; x < b.rlen[r]; ++x) map[(size_t)(b.rpk[r] + x)] = b.roff[r] + x;
                    } else {
                        Eo = S;
                        Ei = b.nbytes;
                        map.assign((size_t)Eo, -1);
                        for (int r = 0; r < b.nruns; ++r)
                            for (int x = 0; x < b.rlen[r]; ++x) map[(size_t)(b.roff[r] + x)] = b.rpk[r] + x;
                    }
                }
                PermSpec sp;
                if (!build_perm(Eo, Ei, map, &sp, &tab)) return false;
                it = ids.emplace(key, (int)specs.size()).first;
                specs.push_back(sp);
            }
            c.perm[pack] = (int16_t)it->second;
        }
    }
    p->perm_specs = std::move(specs);
    p->perm_tab = std::move(tab);
    return true;
}

// Try the span lowering; true when it applies.
bool build_span(const Node* layout, Plan* p) {
    if (layout->runs == 0) return false;
    SpanPlan sp;
    std::memset(&sp, 0, sizeof sp);
    const Node* n = layout;
    SpanBuilder b;
    int64_t base = 0;
    while (n->kind == Kind::Rep && !b.small(n->body.get()) && sp.outer_depth < kSpanMaxOuter) {
        sp.outer_cnt[sp.outer_depth] = n->count;
        sp.outer_str[sp.outer_depth] = n->stride;
        sp.outer_pk[sp.outer_depth] = n->body->nbytes;
        base += n->base;
        ++sp.outer_depth;
        n = n->body.get();
    }
    b.emit(n, base, 0);
    if (!b.ok || b.chunks.empty()) return false;
    sp.nchunks = (int32_t)b.chunks.size();
    sp.nbodies = (int32_t)b.bodies.size();
    int64_t units = sp.nchunks;
    for (int i = 0; i < sp.outer_depth; ++i) units *= sp.outer_cnt[i];
    sp.nunits = units;
    host_magic((uint64_t)sp.nchunks, &sp.m_nchunks, &sp.s_nchunks);
    if (sp.outer_depth == 2) host_magic((uint64_t)sp.outer_cnt[1], &sp.m_outer1, &sp.s_outer1);
    if (!build_perms(b.chunks, b.bodies, p)) {
        p->perm_specs.clear();
        p->perm_tab.clear();
    }
    sp.nperms = (int32_t)p->perm_specs.size();
    sp.ns_max[0] = sp.ns_max[1] = 0;
    for (const auto& c : b.chunks)
        for (int d = 0; d < 2 && sp.nperms; ++d)
            sp.ns_max[d] = std::max(sp.ns_max[d], p->perm_specs[(size_t)c.perm[d]].ns);
    if (sp.nperms) {
        // (spec, layout phase, packed phase) of every chunk; an outer stride
        // that is not a multiple of 4 makes every phase of that side possible
        bool lay_al = true, pk_al = true;
        for (int i = 0; i < sp.outer_depth; ++i) {
            lay_al = lay_al && (sp.outer_str[i] & 3) == 0;
            pk_al = pk_al && (sp.outer_pk[i] & 3) == 0;
        }
        for (int d = 0; d < 2; ++d) {
            std::set<int32_t> use;
            for (const auto& c : b.chunks)
                use.insert((c.perm[d] << 6) | (lay_al ? (int32_t)((c.src & 3) << 2) : 32) |
                           (pk_al ? (int32_t)(c.pk & 3) : 16));
            p->perm_use[d].assign(use.begin(), use.end());
        }
    }
    // iov segments per chunk: body chunks n * nruns; a raw piece starts a
    // segment unless it continues the previous raw piece (one split run)
    {
        std::vector<int64_t> iov(2 * b.chunks.size(), 0);
        int64_t seg = 0, first_raw = -1;
        for (size_t i = 0; i < b.chunks.size(); ++i) {
            const SpanChunk& c = b.chunks[i];
            iov[2 * i] = seg;
            if (c.body >= 0) {
                seg += (int64_t)c.n * b.bodies[(size_t)c.body].nruns;
                first_raw = -1;
                continue;
            }
            const bool cont = first_raw >= 0 && i > 0 && b.chunks[i - 1].body < 0 &&
                              b.chunks[i - 1].src + b.chunks[i - 1].stride == c.src &&
                              b.chunks[i - 1].pk + b.chunks[i - 1].stride == c.pk;
            if (cont) {
                iov[2 * (size_t)first_raw + 1] += c.stride;
            } else {
                first_raw = (int64_t)i;
                iov[2 * i + 1] = c.stride;
                ++seg;
            }
        }
        sp.segs_outer = seg;
        p->span_iov = std::move(iov);
    }
    p->span = sp;
    p->span_chunks = std::move(b.chunks);
    p->span_bodies = std::move(b.bodies);
    return true;
}

}  // namespace

void analyze(const Node* layout, Plan* p) {
    p->runs = layout->runs;
    p->nbytes = layout->nbytes;
    p->min_off = layout->min_off;
    p->max_end = layout->max_end;
    p->node_count = layout->node_count;
    if (layout->runs == 0) {
        p->kind = PLAN_EMPTY;
        return;
    }
    // chain: Rep^k(Run), k <= kMaxChain
    const Node* n = layout;
    Chain c;
    std::memset(&c, 0, sizeof c);
    int64_t align = 16;
    while (n->kind == Kind::Rep && c.depth < kMaxChain) {
        c.cnt[c.depth] = n->count;
        c.str[c.depth] = n->stride;
        c.base += n->base;
        align = std::min(align, pow2_div(n->stride));
        ++c.depth;
        n = n->body.get();
    }
    if (n->kind == Kind::Run) {
        c.base += n->off;
        c.L = n->len;
        align = std::min(align, pow2_div(c.L));
        align = std::min(align, pow2_div(c.base));
        int64_t rows = 1;
        bool small = true;
        for (int i = 0; i < c.depth; ++i) {
            host_magic((uint64_t)c.cnt[i], &c.m_cnt[i], &c.s_cnt[i]);
            rows *= c.cnt[i];
            small = small && c.cnt[i] < (int64_t(1) << 31);
            if (c.cnt[i] < (int64_t(1) << 31)) host_magic32((uint32_t)c.cnt[i], &c.m32_cnt[i], &c.s32_cnt[i]);
        }
        c.small = small && rows < (int64_t(1) << 31);
        host_magic((uint64_t)c.L, &c.m_L, &c.s_L);
        p->kind = PLAN_CHAIN;
        p->chain = c;
        p->chain_align = (int32_t)align;
    } else {
        const bool span = build_span(layout, p);
        // many small irregular runs: tiny span chunks (or no span form at
        // all) lose to a flat run table, one thread per run
        const int64_t units = span ? std::max<int64_t>(1, p->span.nunits) : 1;
        const bool tiny = !span || p->perm_specs.empty() || layout->nbytes / units < 128;
        if (tiny && layout->runs <= kMaxTableRuns && layout->nbytes / std::max<int64_t>(1, layout->runs) <= 1024) {
            p->kind = PLAN_RUNS;
            p->span_chunks.clear();
            p->span_bodies.clear();
            p->perm_specs.clear();
            p->perm_tab.clear();
            p->span_iov.clear();
            p->perm_use[0].clear();
            p->perm_use[1].clear();
        } else {
            p->kind = span ? PLAN_SPAN : PLAN_GENERIC;
        }
    }
    p->overlap = may_overlap(layout);
    if (p->overlap && layout->runs <= (int64_t(1) << 22)) p->overlap = exact_overlap(layout);
}

std::shared_ptr<Plan> get_plan(Datatype* dt, int64_t count, int device, cudaStream_t stream,
                               std::string* err) {
    {
        std::lock_guard<std::mutex> g(dt->mu);
        auto it = dt->plans.find({device, count});
        if (it != dt->plans.end()) return it->second;
    }
    NodeP lay = dt->layout_for(count);
    auto p = std::make_shared<Plan>();
    p->device = device;
    analyze(lay.get(), p.get());
    std::vector<int64_t> rt_src, rt_pk;
    if (p->kind == PLAN_RUNS) {
        std::vector<int64_t> flat;
        tree::enumerate(lay.get(), 0, flat, lay->runs);
        const size_t n = flat.size() / 2;
        rt_src.reserve(n);
        rt_pk.reserve(n + 1);
        int64_t pk = 0, all = 0;
        bool split = false;
        for (size_t i = 0; i < n; ++i) {
            const int64_t off = flat[2 * i], len = flat[2 * i + 1];
            all |= off | len;
            for (int64_t o = 0; o < len; o += kRunPiece) {
                rt_src.push_back(off + o);
                rt_pk.push_back(pk + o);
                split = split || o > 0;
            }
            pk += len;
        }
        rt_pk.push_back(pk);
        int32_t g = 16;
        while (g > 1 && (all & (g - 1))) g >>= 1;
        p->rt.nruns = (int64_t)rt_src.size();
        p->rt.g = g;
        p->rt.avg_words = p->rt.nruns ? pk / p->rt.nruns / g : 0;
        p->rt.split = split ? 1 : 0;
    }
    if (p->kind != PLAN_EMPTY) {
        Flattener f;
        const int32_t root = f.add(lay.get());
        const size_t nb = f.nodes.size() * sizeof(DNode);
        const size_t kb = ((f.kids.size() * sizeof(int32_t)) + 15) & ~size_t(15);
        const size_t pb = f.rp.size() * sizeof(int64_t);
        const size_t bo = (nb + kb + 2 * pb + 15) & ~size_t(15);           // span bodies
        const size_t bb = p->span_bodies.size() * sizeof(SpanBody);
        const size_t co = (bo + bb + 15) & ~size_t(15);                     // span chunks
        const size_t cb = p->span_chunks.size() * sizeof(SpanChunk);
        const size_t so = (co + cb + 15) & ~size_t(15);                     // perm specs
        const size_t sb = p->perm_specs.size() * sizeof(PermSpec);
        const size_t to = (so + sb + 15) & ~size_t(15);                     // perm tables
        const size_t tb = p->perm_tab.size() * sizeof(PermEntry);
        const size_t io = (to + tb + 15) & ~size_t(15);                     // iov chunk info
        const size_t ib = p->span_iov.size() * sizeof(int64_t);
        const size_t ro = (io + ib + 15) & ~size_t(15);                     // run table
        const size_t rb = rt_src.size() * sizeof(int64_t);
        const size_t qo = (ro + rb + 15) & ~size_t(15);
        const size_t qb = rt_pk.size() * sizeof(int64_t);
        std::vector<uint8_t> host(qo + qb + 16, 0);
        std::memcpy(host.data(), f.nodes.data(), nb);
        if (!f.kids.empty()) std::memcpy(host.data() + nb, f.kids.data(), f.kids.size() * sizeof(int32_t));
        if (pb) {
            std::memcpy(host.data() + nb + kb, f.rp.data(), pb);
            std::memcpy(host.data() + nb + kb + pb, f.bp.data(), pb);
        }
        if (bb) std::memcpy(host.data() + bo, p->span_bodies.data(), bb);
        if (cb) std::memcpy(host.data() + co, p->span_chunks.data(), cb);
        if (tb) std::memcpy(host.data() + to, p->perm_tab.data(), tb);
        if (ib) std::memcpy(host.data() + io, p->span_iov.data(), ib);
        if (rb) std::memcpy(host.data() + ro, rt_src.data(), rb);
        if (qb) std::memcpy(host.data() + qo, rt_pk.data(), qb);
        (void)stream;
        void* dev = nullptr;
        MPX_TRACE("plan create: blob %zu B", host.size());
        cudaStream_t up = upload_stream(device);
        cudaMemPool_t pool = desc_pool(device);
        cudaError_t e = pool ? cudaMallocFromPoolAsync(&dev, host.size(), pool, up) : cudaErrorMemoryAllocation;
        if (e != cudaSuccess) {
            *err = std::string("descriptor allocation: ") + cudaGetErrorString(e);
            return nullptr;
        }
        if (sb) {   // table pointers are device addresses inside the blob
            std::vector<PermSpec> specs = p->perm_specs;
            for (auto& sp : specs)
                sp.tab = reinterpret_cast<const PermEntry*>(static_cast<uint8_t*>(dev) + to) +
                         reinterpret_cast<uintptr_t>(sp.tab);
            std::memcpy(host.data() + so, specs.data(), sb);
        }
        p->blob = dev;
        // through pinned staging: returns at once, only the (private) upload
        // stream is involved
        MPX_TRACE("plan upload %zu B", host.size());
        e = upload_arena(device).copy(up, dev, host.data(), host.size());
        MPX_TRACE("plan upload issued");
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ready, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventRecord(p->ready, up);
        if (e != cudaSuccess) {
            *err = std::string("descriptor upload: ") + cudaGetErrorString(e);
            return nullptr;
        }
        p->blob_bytes = host.size();
        uint8_t* b = (uint8_t*)dev;
        p->desc.nodes = (const DNode*)b;
        p->desc.kids = (const int32_t*)(b + nb);
        p->desc.rp = (const int64_t*)(b + nb + kb);
        p->desc.bp = (const int64_t*)(b + nb + kb + pb);
        p->desc.root = root;
        p->span.bodies = (const SpanBody*)(b + bo);
        p->span.chunks = (const SpanChunk*)(b + co);
        p->span.perms = sb ? (const PermSpec*)(b + so) : nullptr;
        p->span.iovc = ib ? (const longlong2*)(b + io) : nullptr;
        p->rt.src = rb ? (const int64_t*)(b + ro) : nullptr;
        p->rt.pk = qb ? (const int64_t*)(b + qo) : nullptr;
        p->desc.runs = lay->runs;
        p->desc.nbytes = lay->nbytes;
    }
    std::lock_guard<std::mutex> g(dt->mu);
    auto ins = dt->plans.emplace(std::make_pair(device, count), p);
    return ins.first->second;
}

}  // namespace mpx
