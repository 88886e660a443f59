// ipc.cpp -- shared segment, matching, flags, arenas and progress thread of
// multi-process worlds (see ipc.hpp).
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
constexpr uint32_t kMagic = 0x4d505849;   // "MPXI"
constexpr int kMaxRanks = 16;
constexpr int kSlots = 512;               // mailbox entries per receiving rank
constexpr int kFlags = 1 << 16;           // completion flags per rank

enum : int32_t { FREE = 0, SEND = 1, RECV = 2, MATCHED = 3 };

struct Entry {
    int32_t state;
    int32_t ctx, src, tag;      // RECV: patterns; SEND/MATCHED: the send's
    int64_t seq;
    int64_t bytes;              // SEND: message bytes; RECV: capacity
    int64_t off;                // sender's arena offset
    uint32_t ready_idx, ready_gen;   // in the sender's flag range
    uint32_t cons_idx, cons_gen;
    int32_t sender;
    int32_t pad;
    uint64_t cookie;            // RECV / MATCHED: receiver-process pointer
};

struct Box {
    pthread_mutex_t mu;
    int64_t next_seq;
    Entry e[kSlots];
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
}  // namespace

constexpr int kWins = 32;   // window slots (window id mod kWins) per job

struct WinEntry {
    cudaIpcMemHandle_t handle;
    int64_t off, bytes, unit;
    int64_t id;
};

struct IpcShared {
    std::atomic<uint32_t> magic;
    int32_t size;
    std::atomic<int32_t> joined, mapped, left;
    std::atomic<int64_t> bar_count, bar_gen;
    int32_t device[kMaxRanks];
    int64_t arena_bytes[kMaxRanks];
    cudaIpcMemHandle_t arena[kMaxRanks];
    Box box[kMaxRanks];
    WinEntry win[kWins][kMaxRanks];
    alignas(64) uint32_t flags[kMaxRanks][kFlags];
};

int IpcWorld::join(const char* name, int size, int rank, int device, int64_t arena_bytes, IpcOnMatch cb,
                   IpcWorld** out) {
    if (size < 1 || size > kMaxRanks) return fail(MPX_ERR_ARG, "multi-process worlds hold 1..%d ranks", kMaxRanks);
    if (rank < 0 || rank >= size) return fail(MPX_ERR_ARG, "rank %d outside job of %d", rank, size);
    std::unique_ptr<IpcWorld> w(new IpcWorld());
    w->name_ = std::string("/mpx-") + name;
    for (auto& ch : w->name_)
        if (ch == '/' && &ch != &w->name_[0]) ch = '_';
    w->size_ = size;
    w->rank_ = rank;
    w->device_ = device;
    w->cb_ = cb;
    w->map_bytes_ = (sizeof(IpcShared) + 4095) & ~size_t(4095);
    // rank 0 creates and initialises the segment; the others wait for it
    if (rank == 0) {
        shm_unlink(w->name_.c_str());   // a stale segment of a crashed job
        w->fd_ = shm_open(w->name_.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
        if (w->fd_ < 0) return fail(MPX_ERR_TRANSPORT, "shm_open(%s): %s", w->name_.c_str(), strerror(errno));
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
        for (int t = 0; t < 120000 && sh->magic.load(std::memory_order_acquire) != kMagic; ++t) nap(1000000);
        if (sh->magic.load() != kMagic) return fail(MPX_ERR_TRANSPORT, "job %s: segment never initialised", name);
        if (sh->size != size) return fail(MPX_ERR_ARG, "job %s has %d ranks, not %d", name, sh->size, size);
    }
    // this rank's arena, exported; the whole segment registered with CUDA
    int cur = -1;
    cudaGetDevice(&cur);
    MPX_CU_RET(cudaSetDevice(device));
    w->arena_bytes_ = arena_bytes;
    w->coll_off_ = (arena_bytes - arena_bytes / 4) & ~int64_t(255);
    MPX_CU_RET(cudaMalloc(reinterpret_cast<void**>(&w->arena_), (size_t)arena_bytes));
    MPX_CU_RET(cudaIpcGetMemHandle(&sh->arena[rank], w->arena_));
    MPX_CU_RET(cudaHostRegister(p, w->map_bytes_, cudaHostRegisterMapped | cudaHostRegisterPortable));
    w->registered_ = true;
    sh->device[rank] = device;
    sh->arena_bytes[rank] = arena_bytes;
    w->shadow_.assign(kFlags, 0);
    sh->joined.fetch_add(1);
    for (int t = 0; t < 1200000 && sh->joined.load() < size; ++t) nap(100000);
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
    for (int t = 0; t < 1200000 && sh->mapped.load() < size; ++t) nap(100000);
    if (cur >= 0) cudaSetDevice(cur);
    IpcWorld* raw = w.release();
    raw->thread_ = new std::thread([raw] { raw->progress_loop(); });
    *out = raw;
    return MPX_SUCCESS;
}

IpcWorld::~IpcWorld() {
    for (int r = 0; r < (int)peer_.size(); ++r)
        if (r != rank_ && peer_[r]) cudaIpcCloseMemHandle(const_cast<uint8_t*>(peer_[r]));
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
    int rc = barrier();
    for (int r = 0; r < size_; ++r)
        if (r != rank_ && peer_[r]) cudaIpcCloseMemHandle(const_cast<uint8_t*>(peer_[r]));
    for (auto& kv : opened_) cudaIpcCloseMemHandle(kv.second);
    rc = rc ? rc : barrier();   // nobody frees its arena while a peer still maps it
    if (arena_) cudaFree(arena_);
    cudaHostUnregister(sh_);
    const bool last = sh_->left.fetch_add(1) + 1 == size_;
    munmap(sh_, map_bytes_);
    close(fd_);
    if (last) shm_unlink(name_.c_str());
    peer_.clear();           // all released above: the destructor has nothing left to do
    arena_ = nullptr;
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

uint32_t* IpcWorld::coll_ready(int r) { return &sh_->flags[r][kFlags - 1]; }
uint32_t* IpcWorld::coll_read(int r) { return &sh_->flags[r][kFlags - 2]; }

uint32_t* IpcWorld::flag_locked(uint32_t* gen) {
    const uint32_t i = next_flag_++ % (kFlags - 2);   // the last two are the collective counters
    *gen = ++shadow_[i];
    return &sh_->flags[rank_][i];
}

int IpcWorld::reserve(int64_t bytes, uint8_t** dst, int64_t* off, uint32_t** ready, uint32_t* ready_gen,
                      uint32_t* cons_idx, uint32_t* cons_gen) {
    std::lock_guard<std::mutex> g(mu_);
    const int64_t len = std::max<int64_t>(256, (bytes + 255) & ~int64_t(255));
    if (len > coll_off_)
        return fail(MPX_ERR_EXHAUSTED, "message of %lld bytes exceeds the %lld-byte staging ring (3/4 of MPX_IPC_ARENA)",
                    (long long)bytes, (long long)coll_off_);
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
            head_ = inflight_.empty() ? tail_ : inflight_.front().off;
            if (inflight_.empty()) head_ = tail_ = 0;
        }
        // place [o, o+len): after tail_, wrapping to 0 when it does not fit
        o = tail_;
        bool fits;
        const bool wrapped = !inflight_.empty() && tail_ < head_;
        if (!wrapped) {
            fits = o + len <= coll_off_;
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
    m->data = peer_[e.sender] + e.off;
    m->ready = &sh_->flags[e.sender][e.ready_idx];
    m->ready_gen = e.ready_gen;
    m->consumed = &sh_->flags[e.sender][e.cons_idx];
    m->consumed_gen = e.cons_gen;
}

int IpcWorld::post_send(int dest, int ctx, int tag, int64_t bytes, int64_t off, uint32_t* ready, uint32_t ready_gen,
                        uint32_t cons_idx, uint32_t cons_gen) {
    if (dest < 0 || dest >= size_) return fail(MPX_ERR_ARG, "dest %d out of range", dest);
    Box& b = sh_->box[dest];
    pthread_mutex_lock(&b.mu);
    // the oldest posted receive this send matches
    int best = -1;
    for (int i = 0; i < kSlots; ++i) {
        const Entry& e = b.e[i];
        if (e.state == RECV && matches(e.src, e.tag, e.ctx, rank_, tag, ctx) && (best < 0 || e.seq < b.e[best].seq))
            best = i;
    }
    int i = best >= 0 ? best : free_slot(b);
    if (i < 0) {
        pthread_mutex_unlock(&b.mu);
        return fail(MPX_ERR_EXHAUSTED, "mailbox of rank %d full", dest);
    }
    Entry& e = b.e[i];
    if (best < 0) {
        e.seq = b.next_seq++;
        e.ctx = ctx;
        e.src = rank_;
        e.cookie = 0;
    }
    e.tag = tag;
    e.bytes = bytes;
    e.off = off;
    e.ready_idx = static_cast<uint32_t>(ready - &sh_->flags[rank_][0]);
    e.ready_gen = ready_gen;
    e.cons_idx = cons_idx;
    e.cons_gen = cons_gen;
    e.sender = rank_;
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

int IpcWorld::win_expose(int64_t id, const void* base, int64_t bytes, int64_t unit, std::vector<const void*>* bases,
                         std::vector<int64_t>* sizes, std::vector<int64_t>* units) {
    using RangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static RangeFn range = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &f, 12000, cudaEnableDefault, &q);
        cudaGetLastError();
        return reinterpret_cast<RangeFn>(f);
    }();
    if (!range) return fail(MPX_ERR_UNSUPPORTED, "cuMemGetAddressRange unavailable");
    WinEntry& mine = sh_->win[id % kWins][rank_];
    std::memset(static_cast<void*>(&mine), 0, sizeof mine);
    if (bytes > 0) {
        CUdeviceptr alloc = 0;
        size_t len = 0;
        if (range(&alloc, &len, reinterpret_cast<CUdeviceptr>(base)) != CUDA_SUCCESS)
            return fail(MPX_ERR_ARG, "window region is not device memory of this process");
        MPX_CU_RET(cudaIpcGetMemHandle(&mine.handle, reinterpret_cast<void*>(alloc)));
        mine.off = static_cast<int64_t>(reinterpret_cast<uintptr_t>(base) - static_cast<uintptr_t>(alloc));
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
        // one mapping per (rank, allocation): a handle opens once per process
        std::string key = std::to_string(r) + ":" + std::string(e.handle.reserved, sizeof e.handle.reserved);
        void* mapped = nullptr;
        for (auto& kv : opened_)
            if (kv.first == key) mapped = kv.second;
        if (!mapped) {
            MPX_CU_RET(cudaIpcOpenMemHandle(&mapped, e.handle, cudaIpcMemLazyEnablePeerAccess));
            opened_.emplace_back(key, mapped);
        }
        (*bases)[r] = static_cast<const uint8_t*>(mapped) + e.off;
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
