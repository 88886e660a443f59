// ipc.cpp -- shared segment, matching, flags, arenas, buffer export/import
// and progress thread of multi-process worlds (see ipc.hpp).
#include "ipc.hpp"

#include <cuda.h>
#include <cuda_runtime.h>
#include <fcntl.h>
#include <pthread.h>
#include <sys/mman.h>
#include <sys/prctl.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include <atomic>
#include <cerrno>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>

#include "capi_common.hpp"

namespace mpx {

namespace {
constexpr uint32_t kMagic = 0x4d505832;   // "MPX2"
constexpr int kMaxRanks = 16;
constexpr int kSlots = 512;               // mailbox entries per receiving rank
constexpr int kFlags = 1 << 16;           // completion flags per rank
constexpr int kCollFlags = 2 * IpcWorld::kCollCtx;   // the last flags of each rank: collective counters
constexpr int kCollDepth = 4;             // collective calls in flight per context slot
constexpr int kBlobs = 16;

enum : int32_t { FREE = 0, SEND = 1, RECV = 2, MATCHED = 3 };

struct Entry {
    int32_t state;
    int32_t ctx, src, tag;      // RECV: patterns; SEND/MATCHED: the send's
    int64_t seq;
    int64_t bytes;              // SEND: message bytes; RECV: capacity
    int64_t off;                // eager: sender's arena offset
    uint32_t ready_idx, ready_gen;   // in the sender's flag range
    uint32_t cons_idx, cons_gen;
    int32_t sender;
    int32_t rndv;
    uint64_t cookie;            // RECV / MATCHED: receiver-process pointer
    cudaIpcMemHandle_t handle;  // rendezvous: the sender's allocation
    uint64_t bufid;
    int64_t buf_off;
    IpcLayout layout;
};

struct Box {
    pthread_mutex_t mu;
    int64_t next_seq;
    Entry e[kSlots];
};

struct CollPost {
    std::atomic<int64_t> seq;   // call number published (+1; 0 = none)
    cudaIpcMemHandle_t h[2];    // send, recv allocations
    uint64_t id[2];
    int64_t off[2];
    int64_t count;
    int32_t code, pad;
};

struct Blob {
    std::atomic<int64_t> key;   // key + 1 once written
    unsigned char data[128];
};

#define MPX_CU_RET(x)                                      \
    do {                                                   \
        cudaError_t e_ = (x);                              \
        if (e_ != cudaSuccess) return cuda_fail(e_, #x);   \
    } while (0)

void nap(long ns) {
    struct timespec ts{0, ns};
    nanosleep(&ts, nullptr);
}

// restores the calling thread's device on every exit path
struct DeviceGuard {
    int cur = -1;
    DeviceGuard() { cudaGetDevice(&cur); }
    ~DeviceGuard() {
        if (cur >= 0) cudaSetDevice(cur);
    }
};

using RangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
using AttrFn = CUresult (*)(void*, CUpointer_attribute, CUdeviceptr);

template <typename F>
F driver_fn(const char* name) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPointByVersion(name, &f, 12000, cudaEnableDefault, &q);
    cudaGetLastError();
    return reinterpret_cast<F>(f);
}
}  // namespace

constexpr int kWins = 32;   // window slots (window id mod kWins) per job

struct WinEntry {
    cudaIpcMemHandle_t handle;
    uint64_t bufid;
    int64_t off, bytes, unit;
    int64_t id;
};

struct IpcShared {
    std::atomic<uint32_t> magic;
    int32_t size;
    std::atomic<int32_t> joined, mapped, left, failed;
    std::atomic<int64_t> bar_count, bar_gen;
    int32_t device[kMaxRanks];
    int64_t arena_bytes[kMaxRanks];
    cudaIpcMemHandle_t arena[kMaxRanks];
    Box box[kMaxRanks];
    WinEntry win[kWins][kMaxRanks];
    CollPost coll[kMaxRanks][IpcWorld::kCollCtx][kCollDepth];
    Blob blob[kBlobs];
    alignas(64) uint32_t flags[kMaxRanks][kFlags];
};

int IpcWorld::join(const char* name, int size, int rank, int device, int64_t arena_bytes, IpcOnMatch cb,
                   IpcWorld** out) {
    if (size < 1 || size > kMaxRanks) return fail(MPX_ERR_ARG, "multi-process worlds hold 1..%d ranks", kMaxRanks);
    if (rank < 0 || rank >= size) return fail(MPX_ERR_ARG, "rank %d outside job of %d", rank, size);
    DeviceGuard guard;
    std::unique_ptr<IpcWorld> w(new IpcWorld());
    w->name_ = std::string("/mpx-") + name;
    for (auto& ch : w->name_)
        if (ch == '/' && &ch != &w->name_[0]) ch = '_';
    w->size_ = size;
    w->rank_ = rank;
    w->device_ = device;
    w->cb_ = cb;
    w->map_bytes_ = (sizeof(IpcShared) + 4095) & ~size_t(4095);
    // rank 0 creates and initialises the segment (and removes it again if its
    // own join fails); the others wait for it
    struct Unlinker {
        const std::string* name = nullptr;
        ~Unlinker() {
            if (name) shm_unlink(name->c_str());
        }
    } unlink_on_fail;
    if (rank == 0) {
        shm_unlink(w->name_.c_str());   // a stale segment of a crashed job
        w->fd_ = shm_open(w->name_.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
        if (w->fd_ < 0) return fail(MPX_ERR_TRANSPORT, "shm_open(%s): %s", w->name_.c_str(), strerror(errno));
        unlink_on_fail.name = &w->name_;
        if (ftruncate(w->fd_, (off_t)w->map_bytes_) != 0)
            return fail(MPX_ERR_TRANSPORT, "ftruncate: %s", strerror(errno));
    } else {
        for (int t = 0; t < 120000 && w->fd_ < 0; ++t) {
            w->fd_ = shm_open(w->name_.c_str(), O_RDWR, 0600);
            if (w->fd_ < 0) nap(1000000);
        }
        if (w->fd_ < 0) return fail(MPX_ERR_TRANSPORT, "job %s: rank 0 never created its segment", name);
        struct stat st{};
        for (int t = 0; t < 120000; ++t) {
            if (fstat(w->fd_, &st) == 0 && (size_t)st.st_size >= w->map_bytes_) break;
            nap(1000000);
        }
    }
    void* p = mmap(nullptr, w->map_bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, w->fd_, 0);
    if (p == MAP_FAILED) return fail(MPX_ERR_TRANSPORT, "mmap: %s", strerror(errno));
    w->sh_ = static_cast<IpcShared*>(p);
    IpcShared* sh = w->sh_;
    if (rank == 0) {
        std::memset(static_cast<void*>(sh), 0, sizeof(IpcShared));
        sh->size = size;
        pthread_mutexattr_t a;
        pthread_mutexattr_init(&a);
        pthread_mutexattr_setpshared(&a, PTHREAD_PROCESS_SHARED);
        for (int r = 0; r < kMaxRanks; ++r) pthread_mutex_init(&sh->box[r].mu, &a);
        pthread_mutexattr_destroy(&a);
        sh->magic.store(kMagic, std::memory_order_release);
    } else {
        // A segment left behind by a crashed job of the same name may be found
        // before rank 0 replaces it (unlink + create): one whose size differs,
        // that is already full, or that a failed rank marked, is stale -- drop
        // it and open the name again.
        for (int t = 0;; ++t) {
            const bool ready = sh->magic.load(std::memory_order_acquire) == kMagic;
            const bool stale = ready && (sh->size != size || sh->joined.load() >= size || sh->failed.load() > 0);
            if (ready && !stale) break;
            if (t >= 120000) {
                if (stale) return fail(MPX_ERR_ARG, "job %s has %d ranks, not %d (or is a dead job's segment)", name,
                                       sh->size, size);
                return fail(MPX_ERR_TRANSPORT, "job %s: segment never initialised", name);
            }
            nap(1000000);
            if (stale || t % 1000 == 999) {   // reopen the name: rank 0 may have replaced the segment
                int fd = shm_open(w->name_.c_str(), O_RDWR, 0600);
                struct stat st{};
                if (fd >= 0 && fstat(fd, &st) == 0 && (size_t)st.st_size >= w->map_bytes_) {
                    void* q = mmap(nullptr, w->map_bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
                    if (q != MAP_FAILED) {
                        munmap(w->sh_, w->map_bytes_);
                        close(w->fd_);
                        w->fd_ = fd;
                        w->sh_ = sh = static_cast<IpcShared*>(q);
                        p = q;
                        fd = -1;
                    }
                }
                if (fd >= 0) close(fd);
            }
        }
    }
    // a rank that fails from here on tells the others, so they fail fast
    struct FailFlag {
        IpcShared* sh;
        bool ok = false;
        ~FailFlag() {
            if (!ok) sh->failed.fetch_add(1);
        }
    } failed{sh};
    // this rank's arena, exported; the whole segment registered with CUDA
    MPX_CU_RET(cudaSetDevice(device));
    w->arena_bytes_ = arena_bytes;
    MPX_CU_RET(cudaMalloc(reinterpret_cast<void**>(&w->arena_), (size_t)arena_bytes));
    MPX_CU_RET(cudaIpcGetMemHandle(&sh->arena[rank], w->arena_));
    MPX_CU_RET(cudaHostRegister(p, w->map_bytes_, cudaHostRegisterMapped | cudaHostRegisterPortable));
    w->registered_ = true;
    sh->device[rank] = device;
    sh->arena_bytes[rank] = arena_bytes;
    w->shadow_.assign(kFlags, 0);
    sh->joined.fetch_add(1);
    for (int t = 0; t < 1200000 && sh->joined.load() < size && !sh->failed.load(); ++t) nap(100000);
    if (sh->joined.load() < size) return fail(MPX_ERR_TRANSPORT, "job %s: not every rank joined", name);
    w->peer_.assign(size, nullptr);
    for (int r = 0; r < size; ++r) {
        if (r == rank) {
            w->peer_[r] = w->arena_;
            continue;
        }
        void* q = nullptr;
        MPX_CU_RET(cudaIpcOpenMemHandle(&q, sh->arena[r], cudaIpcMemLazyEnablePeerAccess));
        w->peer_[r] = static_cast<const uint8_t*>(q);
    }
    sh->mapped.fetch_add(1);
    for (int t = 0; t < 1200000 && sh->mapped.load() < size && !sh->failed.load(); ++t) nap(100000);
    if (sh->mapped.load() < size)
        return fail(MPX_ERR_TRANSPORT, "job %s: a peer failed to map the staging arenas", name);
    failed.ok = true;
    unlink_on_fail.name = nullptr;
    IpcWorld* raw = w.release();
    raw->thread_ = new std::thread([raw] { raw->progress_loop(); });
    *out = raw;
    return MPX_SUCCESS;
}

void IpcWorld::release_all() {
    for (int r = 0; r < (int)peer_.size(); ++r)
        if (r != rank_ && peer_[r]) cudaIpcCloseMemHandle(const_cast<uint8_t*>(peer_[r]));
    peer_.clear();
    for (auto& kv : imported_) cudaIpcCloseMemHandle(kv.second);
    imported_.clear();
}

IpcWorld::~IpcWorld() {
    release_all();
    if (arena_) cudaFree(arena_);
    if (registered_) cudaHostUnregister(sh_);
    if (sh_) munmap(sh_, map_bytes_);
    if (fd_ >= 0) close(fd_);
}

int IpcWorld::device_of(int r) const { return sh_->device[r]; }

int IpcWorld::barrier() {
    IpcShared* sh = sh_;
    const int64_t gen = sh->bar_gen.load(std::memory_order_acquire);
    if (sh->bar_count.fetch_add(1) + 1 == size_) {
        sh->bar_count.store(0);
        sh->bar_gen.fetch_add(1, std::memory_order_release);
        return MPX_SUCCESS;
    }
    for (long t = 0; sh->bar_gen.load(std::memory_order_acquire) == gen; ++t) {
        if (t > 2400000) return fail(MPX_ERR_TRANSPORT, "barrier of job %s timed out", name_.c_str());
        nap(50000);
    }
    return MPX_SUCCESS;
}

int IpcWorld::leave() {
    stop_ = true;
    if (thread_) {
        auto* t = static_cast<std::thread*>(thread_);
        t->join();
        delete t;
        thread_ = nullptr;
    }
    DeviceGuard guard;
    cudaSetDevice(device_);
    int rc = barrier();
    release_all();
    rc = rc ? rc : barrier();   // nobody frees its arena while a peer still maps it
    if (arena_) cudaFree(arena_);
    cudaHostUnregister(sh_);
    const bool last = sh_->left.fetch_add(1) + 1 == size_;
    munmap(sh_, map_bytes_);
    close(fd_);
    if (last) shm_unlink(name_.c_str());
    arena_ = nullptr;           // all released above: the destructor has nothing left to do
    registered_ = false;
    sh_ = nullptr;
    fd_ = -1;
    delete this;
    return rc;
}

uint32_t* IpcWorld::local_flag(uint32_t* gen) {
    std::lock_guard<std::mutex> g(mu_);
    return flag_locked(gen);
}

uint32_t IpcWorld::flag_index(const uint32_t* f) const { return static_cast<uint32_t>(f - &sh_->flags[rank_][0]); }

uint32_t* IpcWorld::coll_arrive(int r, int cs) { return &sh_->flags[r][kFlags - 1 - 2 * cs]; }
uint32_t* IpcWorld::coll_finish(int r, int cs) { return &sh_->flags[r][kFlags - 2 - 2 * cs]; }

uint32_t* IpcWorld::flag_locked(uint32_t* gen) {
    const uint32_t i = next_flag_++ % (kFlags - kCollFlags);   // the last ones are the collective counters
    *gen = ++shadow_[i];
    return &sh_->flags[rank_][i];
}

int IpcWorld::reserve(int64_t bytes, uint8_t** dst, int64_t* off, uint32_t** ready, uint32_t* ready_gen,
                      uint32_t* cons_idx, uint32_t* cons_gen) {
    std::lock_guard<std::mutex> g(mu_);
    const int64_t len = std::max<int64_t>(256, (bytes + 255) & ~int64_t(255));
    if (len > arena_bytes_)
        return fail(MPX_ERR_EXHAUSTED, "staged message of %lld bytes exceeds the %lld-byte staging arena "
                    "(MPX_IPC_ARENA)", (long long)bytes, (long long)arena_bytes_);
    // Room is made by receivers consuming earlier messages (they write the
    // consumed flags from their streams).  The host runs ahead of the GPUs, so
    // when the ring is full wait for that (polling the flags; no GPU call),
    // up to MPX_IPC_WAIT seconds, before reporting the arena exhausted.
    static const double limit_s = std::getenv("MPX_IPC_WAIT") ? std::atof(std::getenv("MPX_IPC_WAIT")) : 60.0;
    int64_t o = 0;
    for (long spins = 0;; ++spins) {
        size_t k = 0;   // reclaim consumed slots from the head of the ring
        while (k < inflight_.size() &&
               *reinterpret_cast<volatile uint32_t*>(&sh_->flags[rank_][inflight_[k].idx]) >= inflight_[k].gen)
            ++k;
        if (k) {
            inflight_.erase(inflight_.begin(), inflight_.begin() + (long)k);
            if (inflight_.empty()) head_ = tail_ = 0;
            else head_ = inflight_.front().off;
        }
        // place [o, o+len): after tail_, wrapping to 0 when it does not fit.
        // Used space is [head_, tail_) when tail_ > head_, and wraps past the
        // end when tail_ <= head_ with messages in flight (tail_ == head_:
        // completely full -- the wrapped message exactly filled the gap).
        o = tail_;
        bool fits;
        const bool wrapped = !inflight_.empty() && tail_ <= head_;
        if (!wrapped) {
            fits = o + len <= arena_bytes_;
            if (!fits && (inflight_.empty() || len <= head_)) {
                o = 0;
                fits = true;
            }
        } else {
            fits = o + len <= head_;
        }
        if (fits) break;
        if (spins * 20e-6 > limit_s)
            return fail(MPX_ERR_EXHAUSTED, "staging arena full for %.0f s: receivers have not consumed earlier messages",
                        limit_s);
        nap(20000);
    }
    tail_ = o + len;
    uint32_t cgen;
    uint32_t* cons = flag_locked(&cgen);
    inflight_.push_back({o, len, static_cast<uint32_t>(cons - &sh_->flags[rank_][0]), cgen});
    *dst = arena_ + o;
    *off = o;
    *ready = flag_locked(ready_gen);
    *cons_idx = inflight_.back().idx;
    *cons_gen = cgen;
    return MPX_SUCCESS;
}

namespace {
bool matches(int pat_src, int pat_tag, int ctx, int src, int tag, int mctx) {
    return ctx == mctx && (pat_src == MPX_ANY_SOURCE || pat_src == src) && (pat_tag == MPX_ANY_TAG || pat_tag == tag);
}
int free_slot(Box& b) {
    for (int i = 0; i < kSlots; ++i)
        if (b.e[i].state == FREE) return i;
    return -1;
}
}  // namespace

void IpcWorld::msg_of(int box, int slot, IpcMsg* m) {
    const Entry& e = sh_->box[box].e[slot];
    m->src = e.sender;
    m->tag = e.tag;
    m->bytes = e.bytes;
    m->rndv = e.rndv;
    m->data = e.rndv ? nullptr : peer_[e.sender] + e.off;
    m->ready = &sh_->flags[e.sender][e.ready_idx];
    m->ready_gen = e.ready_gen;
    m->consumed = &sh_->flags[e.sender][e.cons_idx];
    m->consumed_gen = e.cons_gen;
    m->handle = e.handle;
    m->bufid = e.bufid;
    m->buf_off = e.buf_off;
    m->layout = e.layout;
}

int IpcWorld::post_send(const IpcSend& s) {
    if (s.dest < 0 || s.dest >= size_) return fail(MPX_ERR_ARG, "dest %d out of range", s.dest);
    Box& b = sh_->box[s.dest];
    pthread_mutex_lock(&b.mu);
    // the oldest posted receive this send matches
    int best = -1;
    for (int i = 0; i < kSlots; ++i) {
        const Entry& e = b.e[i];
        if (e.state == RECV && matches(e.src, e.tag, e.ctx, rank_, s.tag, s.ctx) && (best < 0 || e.seq < b.e[best].seq))
            best = i;
    }
    int i = best >= 0 ? best : free_slot(b);
    if (i < 0) {
        pthread_mutex_unlock(&b.mu);
        return fail(MPX_ERR_EXHAUSTED, "mailbox of rank %d full", s.dest);
    }
    Entry& e = b.e[i];
    if (best < 0) {
        e.seq = b.next_seq++;
        e.ctx = s.ctx;
        e.src = rank_;
        e.cookie = 0;
    }
    e.tag = s.tag;
    e.bytes = s.bytes;
    e.off = s.off;
    e.ready_idx = flag_index(s.ready);
    e.ready_gen = s.ready_gen;
    e.cons_idx = s.cons_idx;
    e.cons_gen = s.cons_gen;
    e.sender = rank_;
    e.rndv = s.rndv;
    e.handle = s.handle;
    e.bufid = s.bufid;
    e.buf_off = s.buf_off;
    e.layout = s.layout;
    e.state = best >= 0 ? MATCHED : SEND;
    pthread_mutex_unlock(&b.mu);
    return MPX_SUCCESS;
}

int IpcWorld::recv(int ctx, int src, int tag, int64_t cap, void* cookie, bool* matched, IpcMsg* m) {
    Box& b = sh_->box[rank_];
    pthread_mutex_lock(&b.mu);
    int best = -1;
    for (int i = 0; i < kSlots; ++i) {
        const Entry& e = b.e[i];
        if (e.state == SEND && matches(src, tag, ctx, e.sender, e.tag, e.ctx) && (best < 0 || e.seq < b.e[best].seq))
            best = i;
    }
    if (best >= 0) {
        msg_of(rank_, best, m);
        b.e[best].state = FREE;
        pthread_mutex_unlock(&b.mu);
        *matched = true;
        return MPX_SUCCESS;
    }
    const int i = free_slot(b);
    if (i < 0) {
        pthread_mutex_unlock(&b.mu);
        return fail(MPX_ERR_EXHAUSTED, "mailbox of rank %d full", rank_);
    }
    Entry& e = b.e[i];
    e.seq = b.next_seq++;
    e.ctx = ctx;
    e.src = src;
    e.tag = tag;
    e.bytes = cap;
    e.cookie = reinterpret_cast<uint64_t>(cookie);
    e.state = RECV;
    pthread_mutex_unlock(&b.mu);
    *matched = false;
    return MPX_SUCCESS;
}

int IpcWorld::resolve(IpcMsg* m) {
    if (!m->rndv || m->data) return MPX_SUCCESS;
    uint8_t* base = nullptr;
    if (int rc = import_buffer(m->src, m->handle, m->bufid, &base)) return rc;
    m->data = base + m->buf_off;
    return MPX_SUCCESS;
}

int IpcWorld::export_buffer(const void* p, cudaIpcMemHandle_t* h, uint64_t* id, int64_t* off) {
    static RangeFn range = driver_fn<RangeFn>("cuMemGetAddressRange");
    static AttrFn attr = driver_fn<AttrFn>("cuPointerGetAttribute");
    if (!range || !attr) return fail(MPX_ERR_UNSUPPORTED, "cuMemGetAddressRange / cuPointerGetAttribute unavailable");
    unsigned long long bid = 0;
    if (attr(&bid, CU_POINTER_ATTRIBUTE_BUFFER_ID, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS)
        return fail(MPX_ERR_UNSUPPORTED, "buffer is not device memory of this process");
    CUdeviceptr alloc = 0;
    size_t len = 0;
    if (range(&alloc, &len, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS)
        return fail(MPX_ERR_UNSUPPORTED, "buffer is not device memory of this process");
    *id = bid;
    *off = static_cast<int64_t>(reinterpret_cast<uintptr_t>(p) - static_cast<uintptr_t>(alloc));
    std::lock_guard<std::mutex> g(buf_mu_);
    auto it = exported_.find(bid);
    if (it != exported_.end()) {
        *h = it->second;
        return MPX_SUCCESS;
    }
    cudaError_t e = cudaIpcGetMemHandle(h, reinterpret_cast<void*>(alloc));
    if (e != cudaSuccess) {   // e.g. stream-ordered pool memory: not exportable this way
        cudaGetLastError();
        return fail(MPX_ERR_UNSUPPORTED, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    }
    exported_[bid] = *h;
    return MPX_SUCCESS;
}

int IpcWorld::import_buffer(int rank, const cudaIpcMemHandle_t& h, uint64_t id, uint8_t** base) {
    if (rank == rank_) return fail(MPX_ERR_ARG, "a process cannot import its own allocation");
    std::lock_guard<std::mutex> g(buf_mu_);
    auto key = std::make_pair(rank, id);
    auto it = imported_.find(key);
    if (it != imported_.end()) {
        *base = it->second;
        return MPX_SUCCESS;
    }
    DeviceGuard guard;
    MPX_CU_RET(cudaSetDevice(device_));
    void* q = nullptr;
    MPX_CU_RET(cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess));
    imported_[key] = static_cast<uint8_t*>(q);
    *base = static_cast<uint8_t*>(q);
    return MPX_SUCCESS;
}

int IpcWorld::coll_exchange(int cs, int64_t seq, const void* send, void* recv, int64_t count, int code,
                            std::vector<const void*>* sends, std::vector<void*>* recvs) {
    CollPost& mine = sh_->coll[rank_][cs][seq % kCollDepth];
    if (int rc = export_buffer(send, &mine.h[0], &mine.id[0], &mine.off[0])) return rc;
    if (int rc = export_buffer(recv, &mine.h[1], &mine.id[1], &mine.off[1])) return rc;
    mine.count = count;
    mine.code = code;
    mine.seq.store(seq + 1, std::memory_order_release);
    sends->assign(size_, nullptr);
    recvs->assign(size_, nullptr);
    for (int r = 0; r < size_; ++r) {
        if (r == rank_) {
            (*sends)[r] = send;
            (*recvs)[r] = recv;
            continue;
        }
        CollPost& p = sh_->coll[r][cs][seq % kCollDepth];
        for (long t = 0; p.seq.load(std::memory_order_acquire) != seq + 1; ++t) {
            if (t > 6000000) return fail(MPX_ERR_TRANSPORT, "collective %lld: rank %d never arrived", (long long)seq, r);
            if (t > 1000) nap(20000);
        }
        if (p.count != count || p.code != code)
            return fail(MPX_ERR_ARG, "collective %lld: rank %d passed count %lld / type %d, this rank %lld / %d",
                        (long long)seq, r, (long long)p.count, p.code, (long long)count, code);
        uint8_t* b = nullptr;
        if (int rc = import_buffer(r, p.h[0], p.id[0], &b)) return rc;
        (*sends)[r] = b + p.off[0];
        if (int rc = import_buffer(r, p.h[1], p.id[1], &b)) return rc;
        (*recvs)[r] = b + p.off[1];
    }
    return MPX_SUCCESS;
}

int IpcWorld::share_blob(int slot, int64_t key, void* blob, size_t n) {
    if (n > sizeof(Blob::data)) return fail(MPX_ERR_ARG, "blob too large");
    Blob& b = sh_->blob[slot % kBlobs];
    if (rank_ == 0) {
        std::memcpy(b.data, blob, n);
        b.key.store(key + 1, std::memory_order_release);
        return MPX_SUCCESS;
    }
    for (long t = 0; b.key.load(std::memory_order_acquire) != key + 1; ++t) {
        if (t > 6000000) return fail(MPX_ERR_TRANSPORT, "rank 0 never published blob %lld", (long long)key);
        nap(20000);
    }
    std::memcpy(blob, b.data, n);
    return MPX_SUCCESS;
}

int IpcWorld::win_expose(int64_t id, const void* base, int64_t bytes, int64_t unit, std::vector<const void*>* bases,
                         std::vector<int64_t>* sizes, std::vector<int64_t>* units) {
    WinEntry& mine = sh_->win[id % kWins][rank_];
    std::memset(static_cast<void*>(&mine), 0, sizeof mine);
    if (bytes > 0) {
        if (export_buffer(base, &mine.handle, &mine.bufid, &mine.off))
            return fail(MPX_ERR_ARG, "window region is not device memory of this process");
    }
    mine.bytes = bytes;
    mine.unit = unit;
    mine.id = id;
    if (int rc = barrier()) return rc;   // every rank's entry is in place
    bases->assign(size_, nullptr);
    sizes->assign(size_, 0);
    units->assign(size_, 1);
    for (int r = 0; r < size_; ++r) {
        const WinEntry& e = sh_->win[id % kWins][r];
        if (e.id != id) return fail(MPX_ERR_STATE, "window %lld: ranks disagree on the window order", (long long)id);
        (*sizes)[r] = e.bytes;
        (*units)[r] = e.unit;
        if (e.bytes == 0) continue;
        if (r == rank_) {
            (*bases)[r] = base;
            continue;
        }
        uint8_t* mapped = nullptr;   // one mapping per (rank, allocation)
        if (int rc = import_buffer(r, e.handle, e.bufid, &mapped)) return rc;
        (*bases)[r] = mapped + e.off;
    }
    return barrier();    // nobody reuses the slot before every rank has read it
}

void IpcWorld::defer(void* cookie, const IpcMsg& m) {
    std::lock_guard<std::mutex> g(later_mu_);
    later_in_.emplace_back(cookie, m);
}

void IpcWorld::progress_loop() {
    prctl(PR_SET_TIMERSLACK, 1UL, 0, 0, 0);   // short naps really are short (default slack: 50 us)
    cudaSetDevice(device_);
    Box& b = sh_->box[rank_];
    // matched receives whose delivery the receiver's stream cannot take yet
    // (its post point is still behind earlier work): retried every pass, so a
    // delivery never sits on the side stream ahead of a later, independent
    // one (MPI lets receives complete out of posting order across tags)
    std::vector<std::pair<void*, IpcMsg>> later;
    long idle = 0;
    while (!stop_) {
        bool did = false;
        {
            std::lock_guard<std::mutex> g(later_mu_);
            for (auto& x : later_in_) later.push_back(x);
            later_in_.clear();
        }
        for (size_t k = 0; k < later.size();) {
            if (cb_(later[k].first, later[k].second)) {
                later.erase(later.begin() + (long)k);
                did = true;
            } else {
                ++k;
            }
        }
        IpcMsg m;
        void* cookie = nullptr;
        pthread_mutex_lock(&b.mu);
        for (int i = 0; i < kSlots; ++i)
            if (b.e[i].state == MATCHED) {
                msg_of(rank_, i, &m);
                cookie = reinterpret_cast<void*>(b.e[i].cookie);
                b.e[i].state = FREE;
                break;
            }
        pthread_mutex_unlock(&b.mu);
        if (cookie) {
            if (!cb_(cookie, m)) later.emplace_back(cookie, m);
            did = true;
        }
        if (did) {
            idle = 0;
        } else {
            nap(idle < 1000 ? 2000 : 50000);
            ++idle;
        }
    }
}

}  // namespace mpx
