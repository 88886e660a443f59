// enqueue.cpp -- stream-ordered point-to-point and allreduce engine.
//
// B200 counterpart of the reference's offload path
// (/root/reference/pkg/src/minimpi/offload.py:49-304, p2p.py:84-185,
// transport.py:313-602): the DeviceQueue executor thread becomes the caller's
// cudaStream_t, the eager/rendezvous frame protocol becomes device-side
// ordering between the two ranks' streams, and the payload moves with the
// pack/unpack kernels over peer (NVLink) or local pointers.
//
// Matching happens on the host when an operation is enqueued, with MPI rules
// (context, source incl. ANY_SOURCE, tag incl. ANY_TAG, FIFO per channel,
// transport.py:191-201,399-428), in a per-destination mailbox guarded by its
// own mutex (no global lock on the data path).  Whichever side is enqueued
// second knows both buffers and issues the transfer:
//
//   first side publishes an event recorded at its stream position (buffer
//   ready) and, if it must wait for completion, a flag in pinned host memory
//   waited on with cuStreamWaitValue32;
//   second side waits for that event (cudaStreamWaitEvent), moves the data,
//   and writes the flag with cuStreamWriteValue32.
//
// Eager (<= eager_limit bytes, and every self-send): the sender packs into a
// staging buffer at its stream position and never waits, exactly like the
// reference's eager frames (transport.py:355-375).  Rendezvous: a blocking
// send waits until its data has been delivered (the reference's RTS/CTS wait).
// Nonblocking forms run their deferred part on a per-communicator side stream
// forked from the user stream, joined again by wait_enqueue.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <execinfo.h>
#include <signal.h>
#include <sys/prctl.h>
#include <sys/syscall.h>
#include <unistd.h>
#include <time.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <functional>
#include <thread>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "capi_common.hpp"
#include "coll.hpp"
#include "dmatch.hpp"
#include "ipc.hpp"
#include "kernels.hpp"
#include "mpx.h"

namespace mpx {

namespace {

// MPX_PROF=1 (diagnosis): host time spent in selected CUDA calls of the
// enqueue path, per category, printed at exit
struct ProfCat {
    std::atomic<int64_t> ns{0}, n{0};
};
enum { P_ORDER, P_RECORD, P_MALLOC, P_FREE, P_LAUNCH, P_WAITEV, P_MEMOP, P_QUERY, P_NCAT };
ProfCat g_prof[P_NCAT];
const char* const g_prof_name[P_NCAT] = {"stream_order", "event_record", "malloc_async", "free_async",
                                         "launch_move", "stream_wait_event", "memop", "event_query"};
inline bool profiling() {
    static const bool on = std::getenv("MPX_PROF") != nullptr;
    return on;
}
struct ProfScope {
    int cat;
    struct timespec t0;
    explicit ProfScope(int c) : cat(c) {
        if (profiling()) clock_gettime(CLOCK_MONOTONIC, &t0);
    }
    ~ProfScope() {
        if (!profiling()) return;
        struct timespec t1;
        clock_gettime(CLOCK_MONOTONIC, &t1);
        g_prof[cat].ns += (t1.tv_sec - t0.tv_sec) * 1000000000LL + (t1.tv_nsec - t0.tv_nsec);
        g_prof[cat].n += 1;
    }
};
struct ProfReport {
    ~ProfReport() {
        if (!profiling()) return;
        for (int i = 0; i < P_NCAT; ++i)
            if (g_prof[i].n.load())
                std::fprintf(stderr, "[mpx prof] %-18s %9lld calls %8.2f us/call\n", g_prof_name[i],
                             (long long)g_prof[i].n.load(), g_prof[i].ns.load() / 1e3 / (double)g_prof[i].n.load());
    }
} g_prof_report;

// ------------------------------------------------------------------ flags
// Completion flags live in pinned, mapped host memory (device address = host
// address under UVA).  Slot values only grow, so a waiter on (slot, gen) with
// GEQ is released by exactly the write of gen.
class FlagPool {
  public:
    explicit FlagPool(size_t n) : n_(n), shadow_(n, 0) {}
    int init() {
        cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&base_), n_ * sizeof(uint32_t),
                                      cudaHostAllocMapped | cudaHostAllocPortable);
        if (e != cudaSuccess) return cuda_fail(e, "cudaHostAlloc(flags)");
        std::fill(base_, base_ + n_, 0u);
        return MPX_SUCCESS;
    }
    ~FlagPool() {
        if (base_) cudaFreeHost(base_);
    }
    void take(uint32_t** addr, uint32_t* gen) {
        std::lock_guard<std::mutex> g(mu_);
        const size_t i = next_++ % n_;
        *addr = base_ + i;
        *gen = ++shadow_[i];
    }

  private:
    std::mutex mu_;
    size_t n_, next_ = 0;
    uint32_t* base_ = nullptr;
    std::vector<uint32_t> shadow_;
};

// Driver-API stream memory operations, resolved through the runtime so the
// library does not link libcuda (it must load on GPU-less hosts).
using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WriteValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using ErrStrFn = CUresult (*)(CUresult, const char**);

using WriteValue64Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);

struct MemOps {
    WaitValueFn wait = nullptr;
    WriteValueFn write = nullptr;
    WriteValue64Fn write64 = nullptr;
    ErrStrFn err = nullptr;
};

const MemOps& memops() {
    static MemOps m = [] {
        MemOps r;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", reinterpret_cast<void**>(&r.wait), 12000,
                                         cudaEnableDefault, &q);
        cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", reinterpret_cast<void**>(&r.write), 12000,
                                         cudaEnableDefault, &q);
        cudaGetDriverEntryPointByVersion("cuStreamWriteValue64", reinterpret_cast<void**>(&r.write64), 12000,
                                         cudaEnableDefault, &q);
        cudaGetDriverEntryPointByVersion("cuGetErrorString", reinterpret_cast<void**>(&r.err), 6000,
                                         cudaEnableDefault, &q);
        cudaGetLastError();
        return r;
    }();
    return m;
}

int memop_fail(CUresult r, const char* what) {
    const char* m = nullptr;
    if (memops().err) memops().err(r, &m);
    return fail(MPX_ERR_OTHER, "%s: %s", what, m ? m : "driver error");
}

// MPX_TRACE: every stream wait on a flag is remembered, so a stalled run can
// list the waits whose flag was never written (mpx_debug_flags)
struct FlagWait {
    cudaStream_t s;
    uint32_t* addr;
    uint32_t gen;
};
std::mutex g_waits_mu;
std::vector<FlagWait> g_waits;
struct SideOp {            // a second-side transfer: runs on `side` after both events
    cudaStream_t side;
    cudaEvent_t fork;
    cudaStream_t fork_on;
    cudaEvent_t peer;
    cudaStream_t peer_on;
    uint32_t* flag;        // written when the transfer is done
    int rank;
};
std::vector<SideOp> g_sideops;
void note_side(const SideOp& o) {
    std::lock_guard<std::mutex> g(g_waits_mu);
    g_sideops.push_back(o);
}

int wait_flag(cudaStream_t s, uint32_t* addr, uint32_t gen) {
    // MPX_SPIN_WAIT=1 (diagnosis): poll the flag from a one-warp kernel
    // instead of parking the stream in cuStreamWaitValue32
    static const bool spin = std::getenv("MPX_SPIN_WAIT") != nullptr;
    if (spin) {
        cudaError_t e = launch_flag_wait(addr, gen, s);
        return e == cudaSuccess ? MPX_SUCCESS : cuda_fail(e, "flag wait kernel");
    }
    if (!memops().wait) return fail(MPX_ERR_UNSUPPORTED, "cuStreamWaitValue32 unavailable");
    if (mpx_tracing()) {
        std::lock_guard<std::mutex> g(g_waits_mu);
        g_waits.push_back({s, addr, gen});
        MPX_TRACE("wait stream %p flag %p >= %u", (void*)s, (void*)addr, gen);
    }
    CUresult r = memops().wait(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), gen,
                               CU_STREAM_WAIT_VALUE_GEQ);
    return r == CUDA_SUCCESS ? MPX_SUCCESS : memop_fail(r, "cuStreamWaitValue32");
}

int write_ptr(cudaStream_t s, const void* const* addr, const void* value) {
    if (!memops().write64) return fail(MPX_ERR_UNSUPPORTED, "cuStreamWriteValue64 unavailable");
    CUresult r = memops().write64(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr),
                                  (cuuint64_t) reinterpret_cast<uintptr_t>(value), CU_STREAM_WRITE_VALUE_DEFAULT);
    return r == CUDA_SUCCESS ? MPX_SUCCESS : memop_fail(r, "cuStreamWriteValue64");
}

int write_flag(cudaStream_t s, uint32_t* addr, uint32_t gen) {
    ProfScope ps(P_MEMOP);
    if (!memops().write) return fail(MPX_ERR_UNSUPPORTED, "cuStreamWriteValue32 unavailable");
    MPX_TRACE("write stream %p flag %p = %u", (void*)s, (void*)addr, gen);
    CUresult r = memops().write(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), gen,
                                CU_STREAM_WRITE_VALUE_DEFAULT);
    return r == CUDA_SUCCESS ? MPX_SUCCESS : memop_fail(r, "cuStreamWriteValue32");
}

#define MPX_CU(x)                                               \
    do {                                                        \
        cudaError_t e_ = (x);                                   \
        if (e_ != cudaSuccess) return cuda_fail(e_, #x);        \
    } while (0)
#define MPX_RC(x)                 \
    do {                          \
        int rc_ = (x);            \
        if (rc_) return rc_;      \
    } while (0)

// Staging memory comes from a private per-device pool that never inserts
// hidden stream dependencies (cudaMemPoolReuseAllowInternalDependencies = 0):
// the default pool may make an allocation on one rank's stream wait for a
// free on another rank's stream, which can be blocked in a memop wait on the
// first -- a deadlock the protocol must never contain.
cudaMemPool_t staging_pool(int dev) {
    static std::mutex mu;
    static std::map<int, cudaMemPool_t> pools;
    std::lock_guard<std::mutex> g(mu);
    auto it = pools.find(dev);
    if (it != pools.end()) return it->second;
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    int zero = 0, one = 1;
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &zero);
    cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowOpportunistic, &one);
    cudaMemPoolSetAttribute(pool, cudaMemPoolReuseFollowEventDependencies, &one);
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    pools[dev] = pool;
    return pool;
}

int staging_alloc(int dev, size_t bytes, cudaStream_t st, void** out) {
    cudaMemPool_t pool = staging_pool(dev);
    if (!pool) return fail(MPX_ERR_OTHER, "cannot create the staging memory pool on device %d", dev);
    ProfScope ps(P_MALLOC);
    MPX_CU(cudaMallocFromPoolAsync(out, bytes ? bytes : 1, pool, st));
    return MPX_SUCCESS;
}

// Events are recycled through a per-device free list: creating and
// destroying one per stream point cost ~2 us of host time per operation.
// An event goes back to the list only when its last user is done with it
// (every wait on it enqueued, every query done) -- the points where the code
// used to destroy it -- so re-recording it later cannot be observed.
class EventPool {
  public:
    cudaError_t get(cudaEvent_t* ev) {
        int dev = -1;
        cudaGetDevice(&dev);
        {
            std::lock_guard<std::mutex> g(mu_);
            auto& f = free_[dev];
            if (!f.empty()) {
                *ev = f.back();
                f.pop_back();
                return cudaSuccess;
            }
        }
        cudaError_t e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
        if (e == cudaSuccess) {
            std::lock_guard<std::mutex> g(mu_);
            dev_of_[*ev] = dev;
        }
        return e;
    }
    void put(cudaEvent_t ev) {
        if (!ev) return;
        std::lock_guard<std::mutex> g(mu_);
        auto it = dev_of_.find(ev);
        if (it == dev_of_.end()) {   // not one of ours
            cudaEventDestroy(ev);
            return;
        }
        free_[it->second].push_back(ev);
    }

  private:
    std::mutex mu_;
    std::unordered_map<int, std::vector<cudaEvent_t>> free_;
    std::unordered_map<cudaEvent_t, int> dev_of_;
};

EventPool& event_pool() {
    static EventPool* p = new EventPool();   // never destroyed: events outlive late users
    return *p;
}

void release_event(cudaEvent_t ev) { event_pool().put(ev); }

int record_new_event(cudaStream_t s, cudaEvent_t* ev) {
    ProfScope ps(P_RECORD);
    MPX_CU(event_pool().get(ev));
    MPX_CU(cudaEventRecord(*ev, s));
    return MPX_SUCCESS;
}

// has the stream position recorded in `e` been reached (and passed)?
bool ev_done(cudaEvent_t e) {
    ProfScope ps(P_QUERY);
    const cudaError_t q = cudaEventQuery(e);
    if (q != cudaSuccess) cudaGetLastError();
    return q != cudaErrorNotReady;
}

// ------------------------------------------------------------ stream pool
// Communicator side streams come from a per-device pool and go back to it
// when the communicator dies, so the number of streams alive stays small: the
// device spreads streams over its CUDA_DEVICE_MAX_CONNECTIONS hardware queues,
// and two streams sharing a queue are serialised -- a stream parked in a
// cuStreamWaitValue32 would then also park the stream that is to write the
// flag.  (The Python layer's queue / communicator streams are torch pool
// streams kept distinct per owner, _lib.own_stream.)
class StreamPool {
  public:
    // The free stream made earliest: the first batch sits on distinct
    // hardware queues, so while at most that many streams are live (<= 10
    // in-process ranks per device) no two live streams share a queue, however
    // many streams leaked owners have made the pool grow.
    cudaError_t acquire(int dev, cudaStream_t* out) {
        {
            std::lock_guard<std::mutex> g(mu_);
            auto& f = free_[dev];
            if (!f.empty()) {
                size_t best = 0;
                for (size_t i = 1; i < f.size(); ++i)
                    if (ordinal_[f[i]] < ordinal_[f[best]]) best = i;
                *out = f[best];
                f.erase(f.begin() + (long)best);
                return cudaSuccess;
            }
        }
        MPX_TRACE("stream pool of device %d empty: creating a stream on the data path", dev);
        static const bool dbg = std::getenv("MPX_POOL_DEBUG") != nullptr;
        if (dbg) fprintf(stderr, "[mpx pool] device %d: stream created on the data path\n", dev);
        int cur = -1;
        cudaGetDevice(&cur);
        if (cur != dev) cudaSetDevice(dev);
        cudaError_t e = cudaStreamCreateWithFlags(out, cudaStreamNonBlocking);
        if (cur != dev && cur >= 0) cudaSetDevice(cur);
        if (e == cudaSuccess) {
            std::lock_guard<std::mutex> g(mu_);
            made_.insert(*out);
            ordinal_[*out] = made_.size();
        }
        return e;
    }
    // Top the device's free list up to n streams.  Called at world join:
    // creating a stream can stall inside the driver (holding a lock that
    // cudaEventCreate also takes) while another rank's stream is parked in a
    // memop wait -- measured, with native backtraces -- so streams are made
    // ahead of time, never on the data path.
    cudaError_t reserve(int dev, size_t n) {
        {   // the first reserve of a device creates one batch covering every
            // hardware queue but two (the legacy default stream and one spare):
            // the driver hands queues out round-robin at stream creation, so
            // streams created together sit on distinct queues -- a stream
            // parked in a wait then never parks another of ours, whatever
            // stream (re)use later brings (tools/stall_probe.py: a shared queue
            // deadlocks the 8-ranks-per-GPU ring)
            std::lock_guard<std::mutex> g(mu_);
            if (!batched_.count(dev)) {
                batched_.insert(dev);
                const char* env = std::getenv("CUDA_DEVICE_MAX_CONNECTIONS");
                const int conn = env ? std::max(1, std::min(32, std::atoi(env))) : 8;
                n = std::max(n, (size_t)std::max(1, conn - 2));
            }
        }
        for (;;) {
            {
                std::lock_guard<std::mutex> g(mu_);
                if (free_[dev].size() >= n) return cudaSuccess;
            }
            int cur = -1;
            cudaGetDevice(&cur);
            if (cur != dev) cudaSetDevice(dev);
            cudaStream_t s = nullptr;
            cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
            if (cur != dev && cur >= 0) cudaSetDevice(cur);
            if (e != cudaSuccess) return e;
            std::lock_guard<std::mutex> g(mu_);
            free_[dev].push_back(s);
            made_.insert(s);
            ordinal_[s] = made_.size();
            static const bool dbg = std::getenv("MPX_POOL_DEBUG") != nullptr;
            if (dbg) fprintf(stderr, "[mpx pool] device %d: stream #%zu created (reserve %zu)\n", dev, made_.size(), n);
        }
    }
    // queued work on a released stream simply runs ahead of its next owner's
    void release(int dev, cudaStream_t s) {
        std::lock_guard<std::mutex> g(mu_);
        free_[dev].push_back(s);
    }
    // a stream handed out by mpx_stream_new, returned by its owner once
    // drained (queue destroyed, communicator freed); false if not ours or
    // already free
    bool give_back(int dev, cudaStream_t s) {
        std::lock_guard<std::mutex> g(mu_);
        if (!made_.count(s)) return false;
        auto& f = free_[dev];
        if (std::find(f.begin(), f.end(), s) != f.end()) return false;
        f.push_back(s);
        return true;
    }

  private:
    std::mutex mu_;
    std::map<int, std::vector<cudaStream_t>> free_;
    std::set<cudaStream_t> made_;
    std::map<cudaStream_t, size_t> ordinal_;   // creation order (queue placement)
    std::set<int> batched_;
};

StreamPool& stream_pool() {
    static StreamPool* p = new StreamPool();  // never destroyed: outlives late frees
    return *p;
}

}  // namespace

struct World;
struct Comm;

// Host-side completion record of a nonblocking operation (Request,
// progress.py:34-60; EnqueuedRequest, offload.py:34-46).
struct ReqState {
    std::shared_ptr<Comm> comm;
    bool is_send = false;
    bool matched = false;     // host match done: status known
    int source = -1, tag = -1;
    int64_t count = 0;        // elements of this request's datatype
    int err = MPX_SUCCESS;
    // how the request's stream joins completion at wait_enqueue
    uint32_t* flag = nullptr;  // wait flag >= gen (first side)
    uint32_t gen = 0;
    cudaEvent_t done_ev = nullptr;  // or wait this event (second side, side stream)
    // or run this delivery on the waiting stream: a nonblocking receive
    // matched at initiation moves its data when its stream reaches the wait
    // (the stream then waits only for the sender's data point, which the
    // wait has to anyway -- no side stream, no deferral thread)
    std::function<int(cudaStream_t)> at_wait;
    bool needs_wait = false;
    bool waited = false;
    // device-matched receive (dmatch.hpp): the status lives in pinned host
    // memory, written by the GPU when the match and the copy happen
    DmStatus* dm = nullptr;
    int64_t dm_cap = 0, dm_size = 0;
    std::mutex mu;
};

// one side of a message as known on the host
struct Side {
    int rank = 0, device = 0;
    std::shared_ptr<Comm> comm;   // keeps a freed communicator alive while referenced
    Datatype* dt = nullptr;
    int64_t count = 0;
    void* buf = nullptr;
    int64_t bytes = 0;        // send: message bytes; recv: capacity
};

struct PendingSend {
    int ctx, src, tag;
    Side s;
    bool eager;
    void* staging = nullptr;  // eager: packed copy (sender device)
    cudaEvent_t ev = nullptr; // sender stream position (data ready / staged)
    uint32_t* flag = nullptr; // rendezvous: delivered
    uint32_t gen = 0;
    std::shared_ptr<ReqState> req;
};

struct PendingRecv {
    int ctx, src, tag;        // patterns
    Side r;
    cudaEvent_t ev = nullptr; // receiver stream position (buffer ready)
    uint32_t* flag = nullptr; // delivered
    uint32_t gen = 0;
    bool blocking = false;
    std::shared_ptr<ReqState> req;
};

struct Mailbox {
    std::mutex mu;
    std::deque<PendingSend> sends;  // unexpected (unmatched) sends to this rank
    std::deque<PendingRecv> recvs;  // posted (unmatched) recvs of this rank
};

struct World {
    std::string group;
    IpcWorld* ipc = nullptr;   // multi-process job (ipc.hpp); null: ranks are threads of this process
    int size = 0;
    // matching mode (mpx_world_set_matching): -1 unset (host), 0 host, 1 device
    int dm_mode = -1;
    std::mutex dm_mu;
    std::vector<DmBox*> dm_box;               // per rank, in that rank's device memory
    std::vector<DmStatus*> dm_status;         // per rank, kDmResults, pinned host memory
    std::vector<uint32_t> dm_next;            // per rank: next result slot
    std::vector<uint32_t> dm_rec_next;        // per rank: next rendezvous match record (DmBox::srec)
    std::vector<std::vector<std::weak_ptr<Comm>>> dm_owner;   // blocking receive of a slot, to check for truncation
    int64_t eager_limit = 65536;
    std::vector<int> devices;
    std::vector<bool> joined;
    int live = 0;
    std::vector<std::unique_ptr<Mailbox>> mbox;
    FlagPool flags{1u << 20};
    std::mutex peer_mu;
    std::set<std::pair<int, int>> peer_on;
    // collective rings live in DEVICE memory, one copy per participating
    // device (system-scope reads of pinned host memory serialise across the
    // GPU); kMaxRings ring slots per device are allocated when the device is
    // set up, context ids map to a ring index at comm creation
    static constexpr int kMaxRings = 16;
    std::mutex coll_mu;
    std::map<int, CollRing*> area;      // device -> kMaxRings rings
    std::map<int, int> ring_index;      // context id -> ring index
    std::mutex nccl_mu;
    std::condition_variable nccl_cv;
    std::vector<ncclComm_t> nccl;   // per rank, by ncclCommInitAll
    int nccl_state = 0;             // 0 none, 1 building, 2 ready, -1 failed
    std::map<int, ncclComm_t> nccl_ctx;   // multi-process: this rank's communicator per context
    // passive-target read windows (onesided.py): window k = every rank's k-th
    // mpx_win_create; created / freed collectively
    struct Win {
        std::vector<const void*> base;
        std::vector<int64_t> bytes, unit;
        int registered = 0, released = 0;
    };
    std::mutex win_mu;
    std::condition_variable win_cv;
    std::map<int64_t, Win> wins;
    std::vector<int64_t> next_win;   // per rank
    std::mutex svc_mu;
    std::map<int, cudaStream_t> svc;  // per-device service streams (deferred frees)
    // Deliveries whose inputs are not reachable yet (a receive's post point,
    // or a send's staging point, still behind earlier work on that rank's
    // stream) wait here instead of on a side stream, where they would hold
    // up every later, independent delivery queued behind them -- MPI lets
    // receives complete out of posting order across tags.  One host thread
    // per world retries them until their events have completed; it is only
    // started when the first such delivery appears.
    std::mutex defer_mu;
    std::vector<std::function<bool()>> deferred_ops;
    std::thread defer_thread;
    bool defer_stop = false;
    std::condition_variable defer_cv;
    void defer(std::function<bool()> op) {
        MPX_TRACE("delivery deferred");
        std::lock_guard<std::mutex> g(defer_mu);
        deferred_ops.push_back(std::move(op));
        if (!defer_thread.joinable()) defer_thread = std::thread([this] { defer_loop(); });
        defer_cv.notify_one();   // an idle thread sleeps on the cv: no wake-up latency
    }
    void defer_loop() {
        prctl(PR_SET_TIMERSLACK, 1UL, 0, 0, 0);   // short naps really are short (default slack: 50 us)
        std::vector<std::function<bool()>> mine;
        long idle = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> g(defer_mu);
                if (mine.empty())   // nothing pending: sleep until a delivery is deferred
                    defer_cv.wait(g, [&] { return defer_stop || !deferred_ops.empty(); });
                if (defer_stop && deferred_ops.empty() && mine.empty()) return;
                for (auto& f : deferred_ops) mine.push_back(std::move(f));
                deferred_ops.clear();
            }
            bool did = false;
            for (size_t k = 0; k < mine.size();) {
                if (mine[k]()) {
                    MPX_TRACE("deferred delivery issued (%zu left)", mine.size() - 1);
                    mine.erase(mine.begin() + (long)k);
                    did = true;
                } else {
                    ++k;
                }
            }
            if (did) idle = 0;
            if (mine.empty()) continue;
            struct timespec ts{0, ++idle > 1000 ? 20000L : 2000L};   // inputs pending on the GPU: poll
            nanosleep(&ts, nullptr);
        }
    }
    void stop_deferred() {
        {
            std::lock_guard<std::mutex> g(defer_mu);
            defer_stop = true;
        }
        defer_cv.notify_one();
        if (defer_thread.joinable()) defer_thread.join();
    }
    std::mutex late_mu;
    std::map<int, cudaStream_t> late;   // device -> the world's late stream there
    cudaError_t take_late(int dev) {
        std::lock_guard<std::mutex> g(late_mu);
        if (late.count(dev)) return cudaSuccess;
        cudaStream_t st = nullptr;
        cudaError_t e = stream_pool().acquire(dev, &st);
        if (e == cudaSuccess) late[dev] = st;
        return e;
    }
    cudaStream_t late_on(int dev) {
        std::lock_guard<std::mutex> g(late_mu);
        auto it = late.find(dev);
        return it == late.end() ? nullptr : it->second;
    }
    cudaStream_t service(int dev) {
        std::lock_guard<std::mutex> g(svc_mu);
        auto it = svc.find(dev);
        if (it != svc.end()) return it->second;
        cudaStream_t st = nullptr;
        if (stream_pool().acquire(dev, &st) != cudaSuccess) {
            cudaGetLastError();
            st = nullptr;
        }
        svc[dev] = st;
        return st;
    }
};

struct Comm {
    ~Comm();
    World* w = nullptr;
    int rank = 0, ctx = 0, device = 0;
    cudaStream_t stream = nullptr;  // the user's stream
    cudaStream_t side = nullptr;    // internal, same device; created on first use (side_stream)
    std::once_flag side_once;
    cudaError_t side_err = cudaSuccess;
    // Nonblocking operations run their deferred part here.  Taken lazily
    // from the device's stream pool (reserved at world join, so no stream is
    // created on the data path): most communicators never need one.
    cudaStream_t side_stream() {
        std::call_once(side_once, [this] {
            side_err = stream_pool().acquire(device, &side);
            if (side_err != cudaSuccess) side = nullptr;
        });
        return side;
    }
    // Deferred deliveries (World::defer) are enqueued here, and only once
    // every stream point they depend on has been reached: they never wait,
    // so they can never sit behind -- or hold up -- the side stream's
    // program-ordered work.
    // One per (world, device), shared by the device's communicators -- safe
    // because nothing on it ever waits -- and taken at world join (never on
    // the deferral / progress thread), so the streams alive per device stay
    // few: more streams than the device's CUDA_DEVICE_MAX_CONNECTIONS
    // hardware queues put two streams on one queue, and a stream parked in a
    // wait then parks the other (measured: tools/stall_probe.py, 4 ranks with
    // 4 queues stall every time, with 8+ queues never).
    cudaError_t late_err = cudaErrorNotReady;
    cudaStream_t late_stream();
    // Host run-ahead bound: a mark (pooled event) is recorded on the user
    // stream every kMarkEvery enqueue calls, and a call finding more than
    // kMaxMarks marks outstanding first polls the oldest until the GPU has
    // passed it.  Without it a loop of thousands of enqueue calls fills the
    // CUDA work queues; a rank thread then blocks INSIDE a CUDA call while
    // the work its queue is parked on needs that very thread's later calls
    // (measured: a 2000-iteration 8-byte ring of 2 in-process ranks hung in
    // cuLaunchKernel / cuEventRecord).  Waiting for the own stream is safe
    // for any program that is deadlock-free executed in order.
    static constexpr int kMarkEvery = 16;
    static constexpr size_t kMaxMarks = 4;
    std::mutex mark_mu;
    std::deque<cudaEvent_t> marks;
    int since_mark = 0;
    // false (mpx_comm_set_host_wait): throttle returns MPX_WOULD_BLOCK instead
    // of waiting, before the call has any effect -- a binding that holds a
    // language lock across its calls (Python's GIL, ctypes.PyDLL) waits with
    // the lock released (mpx_comm_throttle_wait) and repeats the call
    std::atomic<bool> host_may_wait{true};
    int throttle();
    int throttle_wait();
    std::mutex err_mu;
    std::deque<std::pair<int, std::string>> deferred;
    std::atomic<int64_t> outstanding{0};
    int64_t coll_seq = 0;
    int ring = -1;                  // index into every device's ring area
    // device matching: this communicator's bounce buffers not yet known to be
    // consumed, and its blocking receives not yet checked for truncation
    struct Bounce {
        void* p;
        uint32_t* flag;
        uint32_t gen;
    };
    std::mutex dm_mu;
    std::deque<Bounce> dm_bounce;
    std::vector<int> dm_blocking;
};

Comm::~Comm() {
    if (side) stream_pool().release(device, side);
    for (cudaEvent_t e : marks) release_event(e);
}

int Comm::throttle() {
    std::unique_lock<std::mutex> g(mark_mu);
    if (++since_mark >= kMarkEvery) {
        since_mark = 0;
        MPX_RC(set_device(device));
        cudaEvent_t ev;
        MPX_RC(record_new_event(stream, &ev));
        marks.push_back(ev);
    }
    long ns = 500;
    while (marks.size() > kMaxMarks) {
        const cudaError_t q = cudaEventQuery(marks.front());
        if (q == cudaErrorNotReady) {
            if (!host_may_wait.load(std::memory_order_relaxed)) return MPX_WOULD_BLOCK;
            struct timespec ts{0, ns};
            nanosleep(&ts, nullptr);
            if (ns < 50000) ns *= 2;
            continue;
        }
        if (q != cudaSuccess) cudaGetLastError();
        release_event(marks.front());
        marks.pop_front();
    }
    return MPX_SUCCESS;
}

int Comm::throttle_wait() {
    std::unique_lock<std::mutex> g(mark_mu);
    long ns = 500;
    while (marks.size() > kMaxMarks) {
        const cudaError_t q = cudaEventQuery(marks.front());
        if (q == cudaErrorNotReady) {
            g.unlock();
            struct timespec ts{0, ns};
            nanosleep(&ts, nullptr);
            if (ns < 50000) ns *= 2;
            g.lock();
            continue;
        }
        if (q != cudaSuccess) cudaGetLastError();
        release_event(marks.front());
        marks.pop_front();
    }
    return MPX_SUCCESS;
}

cudaStream_t Comm::late_stream() {
    cudaStream_t st = w->late_on(device);
    late_err = st ? cudaSuccess : cudaErrorInvalidResourceHandle;
    return st;
}

namespace {

std::mutex g_worlds_mu;
std::map<std::string, World*> g_worlds;
std::mutex g_handles_mu;
std::map<const void*, std::shared_ptr<Comm>> g_comms;
std::map<const void*, std::shared_ptr<ReqState>> g_reqs;

std::shared_ptr<Comm> comm_of(mpx_comm h) {
    std::lock_guard<std::mutex> g(g_handles_mu);
    auto it = g_comms.find(h);
    return it == g_comms.end() ? nullptr : it->second;
}

std::shared_ptr<ReqState> req_of(mpx_request h) {
    std::lock_guard<std::mutex> g(g_handles_mu);
    auto it = g_reqs.find(h);
    return it == g_reqs.end() ? nullptr : it->second;
}

void defer_error(const std::shared_ptr<Comm>& c, int code, const std::string& msg) {
    std::lock_guard<std::mutex> g(c->err_mu);
    c->deferred.emplace_back(code, msg);
}

// Per-device setup done once, at world join (never on the data path: these
// calls may synchronise with streams that are parked in memop waits):
// peer access to every peer device, the staging pool readable from them, the
// world's service stream.
int setup_device(World* w, int dev, int ndev) {
    static std::mutex mu;
    static std::set<int> done;
    std::lock_guard<std::mutex> g(mu);
    MPX_RC(set_device(dev));
    if (!done.count(dev)) {
        cudaMemPool_t pool = staging_pool(dev);
        if (!pool) return fail(MPX_ERR_OTHER, "cannot create the staging memory pool on device %d", dev);
        for (int peer = 0; peer < ndev; ++peer) {
            if (peer == dev) continue;
            int can = 0;
            MPX_CU(cudaDeviceCanAccessPeer(&can, dev, peer));
            if (!can) continue;
            cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
            cudaMemAccessDesc d{};
            d.location.type = cudaMemLocationTypeDevice;
            d.location.id = peer;
            d.flags = cudaMemAccessFlagsProtReadWrite;
            MPX_CU(cudaMemPoolSetAccess(pool, &d, 1));
        }
        done.insert(dev);
    }
    w->service(dev);
    MPX_CU(w->take_late(dev));
    {
        std::lock_guard<std::mutex> g2(w->coll_mu);
        if (!w->area.count(dev)) {
            CollRing* area = nullptr;
            const size_t bytes = sizeof(CollRing) * World::kMaxRings;
            MPX_CU(cudaMalloc(reinterpret_cast<void**>(&area), bytes));
            cudaStream_t svc = w->service(dev);
            MPX_CU(cudaMemsetAsync(area, 0, bytes, svc));
            MPX_CU(cudaStreamSynchronize(svc));   // only the private service stream
            w->area[dev] = area;
        }
    }
    return set_device(dev);
}

int ensure_peer(World* w, int a, int b) {
    (void)w;
    if (a == b) return MPX_SUCCESS;
    int can = 0;
    MPX_CU(cudaDeviceCanAccessPeer(&can, a, b));
    if (!can) return fail(MPX_ERR_TRANSPORT, "device %d cannot access device %d", a, b);
    return MPX_SUCCESS;
}

bool matches(int pat_src, int pat_tag, int ctx, int src, int tag, int mctx) {
    return ctx == mctx && (pat_src == MPX_ANY_SOURCE || pat_src == src) &&
           (pat_tag == MPX_ANY_TAG || pat_tag == tag);
}

// Move min(send bytes, recv capacity) packed bytes from the send layout to
// the recv layout, executed on `st` (device `dev`).  copy_between semantics
// (datatype.py:760-797) with a contiguous side used in place and a packed
// staging buffer otherwise.
int transfer(int dev, cudaStream_t st, const Side& s, const Side& r, int64_t moved) {
    if (moved <= 0) return MPX_SUCCESS;
    int64_t off = 0;
    if (contiguous_run(s.dt, s.count, &off))
        return launch_move(dev, r.dt, r.count, false, static_cast<uint8_t*>(s.buf) + off, r.buf, moved, st);
    if (moved == s.bytes && contiguous_run(r.dt, r.count, &off))
        return launch_move(dev, s.dt, s.count, true, s.buf, static_cast<uint8_t*>(r.buf) + off, s.bytes, st);
    // both typed: one-pass zipper when both layouts are chains
    const int z = launch_zip_move(dev, s.dt, s.count, s.buf, r.dt, r.count, r.buf, moved, st);
    if (z != MPX_ERR_PENDING) return z;
    MPX_RC(set_device(dev));
    void* tmp = nullptr;
    MPX_RC(staging_alloc(dev, (size_t)s.bytes, st, &tmp));
    MPX_RC(launch_move(dev, s.dt, s.count, true, s.buf, tmp, s.bytes, st));
    MPX_RC(launch_move(dev, r.dt, r.count, false, tmp, r.buf, moved, st));
    MPX_CU(cudaFreeAsync(tmp, st));
    return MPX_SUCCESS;
}

void fill_status(const std::shared_ptr<ReqState>& q, const Side& mine, int src, int tag, int64_t moved,
                 bool trunc) {
    if (!q) return;
    std::lock_guard<std::mutex> g(q->mu);
    q->matched = true;
    q->source = src;
    q->tag = tag;
    const int64_t sz = mine.dt->size;
    q->count = sz ? moved / sz : 0;
    q->err = trunc ? MPX_ERR_TRUNCATE : MPX_SUCCESS;
}

// Eager send: pack at the sender's stream position into a staging buffer.
int stage_send(const std::shared_ptr<Comm>& c, PendingSend& ps) {
    MPX_RC(set_device(c->device));
    MPX_RC(staging_alloc(c->device, (size_t)ps.s.bytes, c->stream, &ps.staging));
    MPX_TRACE("staged %lld B", (long long)ps.s.bytes);
    ProfScope pl(P_LAUNCH);
    MPX_RC(launch_move(c->device, ps.s.dt, ps.s.count, true, ps.s.buf, ps.staging, ps.s.bytes, c->stream));
    return MPX_SUCCESS;
}

// Consume an eager staging buffer on stream `st` (device of st = `dev`):
// unpack into the receiver, then free the staging on the world's service
// stream of the owner's device (the sender may have freed its communicator).
// The free never parks a stream: on the consuming stream itself when the
// staging lives on that device, else (a peer device's pool) by the world's
// deferral thread once the unpack has run.  (A service stream waiting for the
// unpack would sit parked -- possibly thousands of operations ahead of the
// GPU when the host runs ahead -- and a parked stream also parks every stream
// that shares its hardware queue: measured as a ring deadlock.)
int consume_staging(World* w, int dev, cudaStream_t st, const PendingSend& ps, const Side& r, int64_t moved) {
    {
        ProfScope pl(P_LAUNCH);
        MPX_RC(launch_move(dev, r.dt, r.count, false, ps.staging, r.buf, moved, st));
    }
    MPX_TRACE("consume: unpack launched");
    if (ps.s.device == dev) {
        MPX_RC(set_device(dev));
        ProfScope pf(P_FREE);
        MPX_CU(cudaFreeAsync(ps.staging, st));
        return MPX_SUCCESS;
    }
    cudaEvent_t used;
    MPX_RC(record_new_event(st, &used));
    const int sdev = ps.s.device;
    void* staging = ps.staging;
    w->defer([w, sdev, staging, used]() {
        if (!ev_done(used)) return false;
        set_device(sdev);
        cudaFreeAsync(staging, w->service(sdev));
        release_event(used);
        return true;
    });
    return MPX_SUCCESS;
}

// -------------------------------------------------------------- send path
int ipc_send(const std::shared_ptr<Comm>& c, const void* buf, int64_t count, Datatype* dt, int dest, int tag,
             bool blocking, std::shared_ptr<ReqState>* out_req);
int ipc_recv(const std::shared_ptr<Comm>& c, void* buf, int64_t count, Datatype* dt, int source, int tag,
             bool blocking, std::shared_ptr<ReqState>* out_req);

int dm_send_op(const std::shared_ptr<Comm>& c, const void* buf, int64_t count, Datatype* dt, int dest, int tag,
               bool blocking, std::shared_ptr<ReqState>* out_req);
int dm_recv_op(const std::shared_ptr<Comm>& c, void* buf, int64_t count, Datatype* dt, int source, int tag,
               bool blocking, std::shared_ptr<ReqState>* out_req);

int do_send(const std::shared_ptr<Comm>& c, const void* buf, int64_t buf_bytes, int64_t count, Datatype* dt, int dest, int tag,
            bool blocking, std::shared_ptr<ReqState>* out_req) {
    World* w = c->w;
    if (w->ipc) {
        if (dest < 0 || dest >= w->size) return fail(MPX_ERR_ARG, "dest %d out of range for size-%d communicator", dest, w->size);
        if (tag < 0) return fail(MPX_ERR_ARG, "tag %d out of range [0, 2147483647]", tag);
        MPX_RC(check_layout_region(dt, count, buf_bytes));
        return ipc_send(c, buf, count, dt, dest, tag, blocking, out_req);
    }
    if (dest < 0 || dest >= w->size) return fail(MPX_ERR_ARG, "dest %d out of range for size-%d communicator", dest, w->size);
    if (tag < 0) return fail(MPX_ERR_ARG, "tag %d out of range [0, 2147483647]", tag);
    MPX_RC(check_layout_region(dt, count, buf_bytes));
    if (w->dm_mode == 1) return dm_send_op(c, buf, count, dt, dest, tag, blocking, out_req);
    Side s;
    s.rank = c->rank;
    s.device = c->device;
    s.comm = c;
    s.dt = dt;
    s.count = count;
    s.buf = const_cast<void*>(buf);
    s.bytes = dt->size * count;
    std::shared_ptr<ReqState> req;
    if (!blocking) {
        req = std::make_shared<ReqState>();
        req->comm = c;
        req->is_send = true;
        req->matched = true;  // a send's status is known at initiation
    }
    const bool eager = s.bytes <= w->eager_limit || dest == c->rank;
    Mailbox& mb = *w->mbox[dest];
    std::unique_lock<std::mutex> lk(mb.mu);
    auto it = std::find_if(mb.recvs.begin(), mb.recvs.end(), [&](const PendingRecv& pr) {
        return matches(pr.src, pr.tag, pr.ctx, c->rank, tag, c->ctx);
    });
    MPX_TRACE("send r%d -> %d tag %d %lld B (%s) %s side", c->rank, dest, tag, (long long)s.bytes,
              eager ? "eager" : "rndv", it == mb.recvs.end() ? "first" : "second");
    if (it == mb.recvs.end()) {
        // --- first side: publish the send -----------------------------------
        PendingSend ps{c->ctx, c->rank, tag, s, eager};
        ps.req = req;
        MPX_RC(set_device(c->device));
        if (eager) MPX_RC(stage_send(c, ps));
        MPX_RC(record_new_event(c->stream, &ps.ev));
        if (!eager) w->flags.take(&ps.flag, &ps.gen);
        uint32_t* flag = ps.flag;
        const uint32_t gen = ps.gen;
        mb.sends.push_back(ps);
        lk.unlock();
        if (!eager) {  // rendezvous: complete when the receiver has pulled the data
            if (blocking) MPX_RC(wait_flag(c->stream, flag, gen));
            else {
                req->flag = flag;
                req->gen = gen;
                req->needs_wait = true;
            }
        }
        if (req) c->outstanding++;
        if (out_req) *out_req = req;
        return MPX_SUCCESS;
    }
    // --- second side: the receive was posted first ---------------------------
    PendingRecv pr = *it;
    mb.recvs.erase(it);
    lk.unlock();
    const int64_t moved = std::min(s.bytes, pr.r.bytes);
    const bool trunc = s.bytes > pr.r.bytes;
    fill_status(pr.req, pr.r, c->rank, tag, moved, trunc);
    if (trunc && pr.blocking)
        defer_error(pr.r.comm, MPX_ERR_TRUNCATE, "message truncated: incoming data larger than the posted receive");
    MPX_RC(ensure_peer(w, c->device, pr.r.device));
    MPX_RC(set_device(c->device));
    if (eager) {
        PendingSend ps{c->ctx, c->rank, tag, s, true};
        MPX_RC(stage_send(c, ps));
        cudaEvent_t staged;
        MPX_RC(record_new_event(c->stream, &staged));
        ps.ev = staged;
        if (pr.req) {   // a nonblocking receive not waited yet: it unpacks at its wait
            std::unique_lock<std::mutex> rl(pr.req->mu);
            if (!pr.req->waited) {
                World* wd = w;
                Side rr = pr.r;
                cudaEvent_t post = pr.ev;
                pr.req->at_wait = [wd, ps, rr, moved, post](cudaStream_t ws) -> int {
                    MPX_RC(set_device(rr.device));
                    {
                        ProfScope pw(P_WAITEV);
                        MPX_CU(cudaStreamWaitEvent(ws, ps.ev, 0));
                    }
                    MPX_RC(consume_staging(wd, rr.device, ws, ps, rr, moved));
                    MPX_RC(set_device(rr.device));
                    release_event(ps.ev);
                    release_event(post);
                    return MPX_SUCCESS;
                };
                rl.unlock();
                MPX_TRACE("send r%d -> %d: eager, delivered at the receiver's wait", c->rank, dest);
                if (req) c->outstanding++;
                if (out_req) *out_req = req;
                return MPX_SUCCESS;
            }
        }
        if (!c->side_stream()) return cuda_fail(c->side_err, "cudaStreamCreate(side)");
        auto deliver = [c, staged, ev = pr.ev, r = pr.r, flag = pr.flag, gen = pr.gen, staging = ps.staging,
                        moved](cudaStream_t st) -> int {
            MPX_RC(set_device(c->device));
            if (!st) return cuda_fail(c->late_err, "cudaStreamCreate(late)");
            MPX_CU(cudaStreamWaitEvent(st, staged, 0));
            MPX_CU(cudaStreamWaitEvent(st, ev, 0));
            MPX_RC(launch_move(c->device, r.dt, r.count, false, staging, r.buf, moved, st));
            MPX_RC(set_device(c->device));
            MPX_CU(cudaFreeAsync(staging, st));
            MPX_RC(write_flag(st, flag, gen));
            release_event(staged);
            release_event(ev);
            return MPX_SUCCESS;
        };
        if (ev_done(pr.ev)) {   // the side stream waits only for this rank's own staging point
            MPX_RC(deliver(c->side_stream()));
        } else {   // the receive's post point is behind earlier work: deliver later
            w->defer([deliver, c, ev = pr.ev, staged]() {
                if (!ev_done(ev) || !ev_done(staged)) return false;
                if (int rc = deliver(c->late_stream())) defer_error(c, rc, "deferred delivery failed: " + g_last_error);
                return true;
            });
        }
        if (req) c->outstanding++;
        if (out_req) *out_req = req;
        return MPX_SUCCESS;
    } else if (blocking) {
        MPX_CU(cudaStreamWaitEvent(c->stream, pr.ev, 0));
        MPX_RC(transfer(c->device, c->stream, s, pr.r, moved));
        MPX_RC(write_flag(c->stream, pr.flag, pr.gen));
    } else {
        cudaEvent_t fork;
        MPX_RC(record_new_event(c->stream, &fork));
        if (!c->side_stream()) return cuda_fail(c->side_err, "cudaStreamCreate(side)");
        if (!ev_done(pr.ev)) {
            // the receive's post point is still behind earlier work on the
            // receiver's stream: the world's deferral thread enqueues it on the
            // late stream once every input is reached; the send request
            // completes on a flag
            uint32_t* done = nullptr;
            uint32_t dgen = 0;
            w->flags.take(&done, &dgen);
            req->flag = done;
            req->gen = dgen;
            req->needs_wait = true;
            w->defer([c, fork, ev = pr.ev, s, r = pr.r, flag = pr.flag, gen = pr.gen, moved, done, dgen]() {
                if (!ev_done(ev) || !ev_done(fork)) return false;
                int rc = set_device(c->device);
                cudaStream_t side = c->late_stream();
                if (!rc && !side) rc = cuda_fail(c->late_err, "cudaStreamCreate(late)");
                if (!rc && cudaStreamWaitEvent(side, fork, 0) != cudaSuccess) rc = fail(MPX_ERR_OTHER, "wait");
                if (!rc) rc = transfer(c->device, side, s, r, moved);
                if (!rc) rc = set_device(c->device);
                if (!rc) rc = write_flag(side, flag, gen);
                if (!rc) rc = write_flag(side, done, dgen);
                if (rc) defer_error(c, rc, "deferred delivery failed: " + g_last_error);
                release_event(fork);
                release_event(ev);
                return true;
            });
            c->outstanding++;
            if (out_req) *out_req = req;
            return MPX_SUCCESS;
        }
        MPX_CU(cudaStreamWaitEvent(c->side_stream(), fork, 0));
        MPX_CU(cudaStreamWaitEvent(c->side_stream(), pr.ev, 0));
        MPX_RC(transfer(c->device, c->side_stream(), s, pr.r, moved));
        MPX_RC(write_flag(c->side_stream(), pr.flag, pr.gen));
        MPX_RC(record_new_event(c->side_stream(), &req->done_ev));
        req->needs_wait = true;
        if (mpx_tracing()) note_side({c->side_stream(), fork, c->stream, pr.ev, pr.r.comm->stream, pr.flag, c->rank});
        else release_event(fork);
    }
    if (!mpx_tracing()) release_event(pr.ev);  // the waits above captured it
    if (req) c->outstanding++;
    if (out_req) *out_req = req;
    MPX_TRACE("send r%d -> %d issued", c->rank, dest);
    return MPX_SUCCESS;
}

// -------------------------------------------------------------- recv path
int do_recv(const std::shared_ptr<Comm>& c, void* buf, int64_t buf_bytes, int64_t count, Datatype* dt, int source, int tag,
            bool blocking, std::shared_ptr<ReqState>* out_req) {
    World* w = c->w;
    if (source != MPX_ANY_SOURCE && (source < 0 || source >= w->size))
        return fail(MPX_ERR_ARG, "source %d out of range for size-%d communicator", source, w->size);
    if (tag < 0 && tag != MPX_ANY_TAG) return fail(MPX_ERR_ARG, "tag %d out of range [0, 2147483647]", tag);
    MPX_RC(check_layout_region(dt, count, buf_bytes));  // DtypeSink check at post time (p2p.py:63-64)
    if (w->ipc) return ipc_recv(c, buf, count, dt, source, tag, blocking, out_req);
    if (w->dm_mode == 1) return dm_recv_op(c, buf, count, dt, source, tag, blocking, out_req);
    Side r;
    r.rank = c->rank;
    r.device = c->device;
    r.comm = c;
    r.dt = dt;
    r.count = count;
    r.buf = buf;
    r.bytes = dt->size * count;
    std::shared_ptr<ReqState> req;
    if (!blocking) {
        req = std::make_shared<ReqState>();
        req->comm = c;
    }
    Mailbox& mb = *w->mbox[c->rank];
    std::unique_lock<std::mutex> lk(mb.mu);
    auto it = std::find_if(mb.sends.begin(), mb.sends.end(), [&](const PendingSend& ps) {
        return matches(source, tag, c->ctx, ps.src, ps.tag, ps.ctx);
    });
    MPX_TRACE("recv r%d <- %d tag %d %s side", c->rank, source, tag, it == mb.sends.end() ? "first" : "second");
    if (it == mb.sends.end()) {
        // --- first side: post the receive ------------------------------------
        PendingRecv pr{c->ctx, source, tag, r};
        pr.blocking = blocking;
        pr.req = req;
        MPX_RC(set_device(c->device));
        MPX_RC(record_new_event(c->stream, &pr.ev));
        MPX_TRACE("recv r%d posted", c->rank);
        w->flags.take(&pr.flag, &pr.gen);
        uint32_t* flag = pr.flag;
        const uint32_t gen = pr.gen;
        mb.recvs.push_back(pr);
        lk.unlock();
        if (blocking) MPX_RC(wait_flag(c->stream, flag, gen));
        else {
            req->flag = flag;
            req->gen = gen;
            req->needs_wait = true;
            c->outstanding++;
        }
        if (out_req) *out_req = req;
        return MPX_SUCCESS;
    }
    // --- second side: the send was enqueued first ----------------------------
    PendingSend ps = *it;
    mb.sends.erase(it);
    lk.unlock();
    const int64_t moved = std::min(ps.s.bytes, r.bytes);
    const bool trunc = ps.s.bytes > r.bytes;
    fill_status(req, r, ps.src, ps.tag, moved, trunc);
    if (trunc && blocking)
        defer_error(c, MPX_ERR_TRUNCATE, "message truncated: incoming data larger than the posted receive");
    MPX_RC(ensure_peer(w, c->device, ps.s.device));
    MPX_RC(set_device(c->device));
    cudaStream_t st = c->stream;
    if (!blocking && ps.eager) {
        // an eager message (its sender never waits for it) matched at
        // initiation: the data moves when this stream reaches wait_enqueue,
        // waiting there only for the sender's staging point -- no side
        // stream, no deferral thread.  (Not for rendezvous: the sender's
        // completion would then hang on this rank's wait, which MPI lets
        // depend on the sender's later operations.)
        req->at_wait = [w, c, ps, r, moved](cudaStream_t ws) -> int {
            MPX_RC(set_device(c->device));
            MPX_CU(cudaStreamWaitEvent(ws, ps.ev, 0));
            MPX_RC(consume_staging(w, c->device, ws, ps, r, moved));
            MPX_RC(set_device(c->device));
            release_event(ps.ev);
            return MPX_SUCCESS;
        };
        req->needs_wait = true;
        c->outstanding++;
        if (out_req) *out_req = req;
        MPX_TRACE("recv r%d matched an eager send at initiation: delivery at wait", c->rank);
        return MPX_SUCCESS;
    }
    cudaEvent_t fork0 = nullptr;
    if (!blocking) MPX_RC(record_new_event(c->stream, &fork0));
    if (!blocking && !ev_done(ps.ev)) {
        // the send's data point is still behind earlier work on the
        // sender's stream: the world's deferral thread enqueues it on the late
        // stream once every input is reached (complete on a flag).  The side
        // stream only ever waits for this rank's own, program-ordered stream
        // points; nothing ever waits for a peer point that is not reached,
        // so no delivery can hold up another queued behind it.
        cudaEvent_t fork = fork0;
        uint32_t* done = nullptr;
        uint32_t dgen = 0;
        w->flags.take(&done, &dgen);
        req->flag = done;
        req->gen = dgen;
        req->needs_wait = true;
        w->defer([c, fork, ps, r, moved, done, dgen]() {
            if (!ev_done(ps.ev) || !ev_done(fork)) return false;
            int rc = set_device(c->device);
            cudaStream_t side = c->late_stream();
            if (!rc && !side) rc = cuda_fail(c->late_err, "late stream");
            if (!rc && cudaStreamWaitEvent(side, fork, 0) != cudaSuccess) rc = fail(MPX_ERR_OTHER, "wait");
            if (!rc && cudaStreamWaitEvent(side, ps.ev, 0) != cudaSuccess) rc = fail(MPX_ERR_OTHER, "wait");
            if (!rc) rc = transfer(c->device, side, ps.s, r, moved);
            if (!rc) rc = write_flag(side, ps.flag, ps.gen);
            if (!rc) rc = set_device(c->device);
            if (!rc) rc = write_flag(side, done, dgen);
            if (rc) defer_error(c, rc, "deferred delivery failed: " + g_last_error);
            release_event(fork);
            release_event(ps.ev);
            return true;
        });
        c->outstanding++;
        if (out_req) *out_req = req;
        return MPX_SUCCESS;
    }
    if (!blocking) {   // rendezvous, the sender's data point reached: the side stream
        if (!c->side_stream()) return cuda_fail(c->side_err, "cudaStreamCreate(side)");
        MPX_CU(cudaStreamWaitEvent(c->side_stream(), fork0, 0));
        if (mpx_tracing()) note_side({c->side_stream(), fork0, c->stream, ps.ev, ps.s.comm->stream, ps.flag, c->rank});
        else release_event(fork0);
        st = c->side_stream();
    }
    MPX_CU(cudaStreamWaitEvent(st, ps.ev, 0));
    MPX_TRACE("recv r%d second side on the %s stream", c->rank, blocking ? "user" : "side");
    if (ps.eager) {
        MPX_RC(consume_staging(w, c->device, st, ps, r, moved));
        MPX_TRACE("recv r%d consumed staging", c->rank);
    } else {
        MPX_RC(transfer(c->device, st, ps.s, r, moved));
        MPX_RC(write_flag(st, ps.flag, ps.gen));
    }
    MPX_RC(set_device(c->device));
    if (!blocking) {
        MPX_RC(record_new_event(st, &req->done_ev));
        req->needs_wait = true;
        c->outstanding++;
    }
    if (!mpx_tracing()) release_event(ps.ev);
    if (out_req) *out_req = req;
    MPX_TRACE("recv r%d issued", c->rank);
    return MPX_SUCCESS;
}


// ------------------------------------------------ device matching (dmatch.hpp)
// The receiving rank's box (allocated on first use, on that rank's device;
// a rank that has not joined yet is waited for) and its status array.
int dm_box_of(World* w, int rank, DmBox** out) {
    for (long t = 0;; ++t) {
        {
            std::lock_guard<std::mutex> g(w->dm_mu);
            if (w->dm_box[(size_t)rank]) {
                *out = w->dm_box[(size_t)rank];
                return MPX_SUCCESS;
            }
            const int dev = w->devices[(size_t)rank];
            if (dev >= 0) {
                int cur = 0;
                cudaGetDevice(&cur);
                MPX_RC(set_device(dev));
                DmBox* b = nullptr;
                MPX_CU(cudaMalloc(reinterpret_cast<void**>(&b), sizeof(DmBox)));
                cudaStream_t svc = w->service(dev);
                MPX_CU(cudaMemsetAsync(b, 0, sizeof(DmBox), svc));
                MPX_CU(cudaStreamSynchronize(svc));   // only the private service stream
                DmStatus* st = nullptr;
                MPX_CU(cudaHostAlloc(reinterpret_cast<void**>(&st), sizeof(DmStatus) * kDmResults,
                                     cudaHostAllocMapped | cudaHostAllocPortable));
                std::memset(static_cast<void*>(st), 0, sizeof(DmStatus) * kDmResults);
                for (int i = 0; i < kDmResults; ++i) st[i].done = 1;   // every slot free
                w->dm_status[(size_t)rank] = st;
                w->dm_box[(size_t)rank] = b;
                *out = b;
                return set_device(cur);
            }
        }
        if (t > 120000) return fail(MPX_ERR_STATE, "rank %d never joined world %s", rank, w->group.c_str());
        struct timespec ts{0, 1000000L};
        nanosleep(&ts, nullptr);
    }
}

// Check a blocking receive's status for truncation (deferred error of its
// communicator, raised at synchronize like the host path's).  w->dm_mu held.
void dm_settle_locked(World* w, int rank, int slot) {
    auto& own = w->dm_owner[(size_t)rank][(size_t)slot];
    auto c = own.lock();
    own.reset();
    if (!c) return;
    const volatile DmStatus* st = &w->dm_status[(size_t)rank][slot];
    if (st->done && st->err == MPX_ERR_TRUNCATE)
        defer_error(c, MPX_ERR_TRUNCATE, "message truncated: incoming data larger than the posted receive");
    else if (st->done && st->err)
        defer_error(c, st->err, "device matching: the unexpected-message queue overflowed");
}

// A result slot for a new receive of `rank`: the next one round-robin, which
// must have completed its previous use.
int dm_take_slot(World* w, int rank, int* slot) {
    std::lock_guard<std::mutex> g(w->dm_mu);
    const int s = (int)(w->dm_next[(size_t)rank]++ % (uint32_t)kDmResults);
    volatile DmStatus* st = &w->dm_status[(size_t)rank][s];
    if (!st->done)
        return fail(MPX_ERR_EXHAUSTED, "device matching: more than %d receives of rank %d in flight", kDmResults, rank);
    dm_settle_locked(w, rank, s);
    st->done = 0;
    st->err = 0;
    st->src = -1;
    st->tag = -1;
    st->bytes = 0;
    *slot = s;
    return MPX_SUCCESS;
}

// Free this communicator's bounce buffers whose receivers have copied them
// out (stream-ordered on its own stream: after the pack that wrote them).
int dm_reclaim(const std::shared_ptr<Comm>& c) {
    std::lock_guard<std::mutex> g(c->dm_mu);
    for (auto it = c->dm_bounce.begin(); it != c->dm_bounce.end();) {
        if (*reinterpret_cast<volatile uint32_t*>(it->flag) >= it->gen) {
            ProfScope pf(P_FREE);
            MPX_CU(cudaFreeAsync(it->p, c->stream));
            it = c->dm_bounce.erase(it);
        } else {
            ++it;
        }
    }
    return MPX_SUCCESS;
}

// The layout of (dt, count) as a chain for the device copies (dmatch.hpp):
// contiguous or Rep^k(Run), non-overlapping; false for other layouts.
bool dm_chain_lay(int dev, Datatype* dt, int64_t count, cudaStream_t st, DmLay* out) {
    std::string err;
    auto p = get_plan(dt, count, dev, st, &err);
    if (!p || p->kind != PLAN_CHAIN || p->overlap) return false;
    std::memset(out, 0, sizeof *out);
    out->c = p->chain;
    out->align = p->chain_align;
    return true;
}

// Eager: the message is packed into a bounce buffer at the sender's stream
// position, then announced to the receiver's box (k_dm_send): the send is
// complete at that point, blocking or not.  Rendezvous (nonblocking,
// contiguous, above the eager limit): the sender's own buffer is announced
// and copied once by the side that matches second (k_dm_xfer); the send's
// wait_enqueue waits for the copy's completion flag.
int dm_send_op(const std::shared_ptr<Comm>& c, const void* buf, int64_t count, Datatype* dt, int dest, int tag,
               bool blocking, std::shared_ptr<ReqState>* out_req) {
    World* w = c->w;
    DmBox* box = nullptr;
    MPX_RC(dm_box_of(w, dest, &box));
    MPX_RC(set_device(c->device));
    MPX_RC(dm_reclaim(c));
    const int64_t bytes = dt->size * count;
    DmLay lay;
    if (!blocking && bytes > w->eager_limit && dest != c->rank && dm_chain_lay(c->device, dt, count, c->stream, &lay)) {
        DmBox* own = nullptr;
        MPX_RC(dm_box_of(w, c->rank, &own));
        uint32_t idx = 0;
        {
            std::lock_guard<std::mutex> g(w->dm_mu);
            idx = w->dm_rec_next[(size_t)c->rank]++ % (uint32_t)kDmRecords;
        }
        uint32_t* flag = nullptr;
        uint32_t gen = 0;
        w->flags.take(&flag, &gen);
        MPX_RC(set_device(c->device));
        {
            ProfScope pl(P_LAUNCH);
            MPX_CU(dm_send_rdv(box, c->rank, tag, c->ctx, static_cast<const uint8_t*>(buf), lay, bytes, flag, gen,
                               &own->srec[idx], c->device, c->stream));
        }
        MPX_TRACE("dm send r%d -> %d tag %d %lld B (rendezvous)", c->rank, dest, tag, (long long)bytes);
        auto req = std::make_shared<ReqState>();
        req->comm = c;
        req->is_send = true;
        req->matched = true;
        req->flag = flag;      // wait_enqueue: the stream waits for the copy
        req->gen = gen;
        req->needs_wait = true;
        c->outstanding++;
        if (out_req) *out_req = req;
        return MPX_SUCCESS;
    }
    void* bounce = nullptr;
    MPX_RC(staging_alloc(c->device, (size_t)bytes, c->stream, &bounce));
    // a small message of a chain layout is packed by k_dm_send itself
    const bool fused = bytes > 0 && bytes <= kDmFusedBytes && dm_chain_lay(c->device, dt, count, c->stream, &lay);
    if (bytes > 0 && !fused) {
        ProfScope pl(P_LAUNCH);
        MPX_RC(launch_move(c->device, dt, count, true, buf, bounce, bytes, c->stream));
        MPX_RC(set_device(c->device));
    }
    uint32_t* flag = nullptr;
    uint32_t gen = 0;
    w->flags.take(&flag, &gen);
    {
        ProfScope pl(P_LAUNCH);
        MPX_RC(set_device(c->device));
        if (fused)
            MPX_CU(dm_send_packed(box, c->rank, tag, c->ctx, static_cast<const uint8_t*>(buf), lay,
                                  static_cast<uint8_t*>(bounce), bytes, flag, gen, c->stream));
        else
            MPX_CU(dm_send(box, c->rank, tag, c->ctx, static_cast<const uint8_t*>(bounce), bytes, flag, gen, c->stream));
    }
    {
        std::lock_guard<std::mutex> g(c->dm_mu);
        c->dm_bounce.push_back({bounce, flag, gen});
    }
    MPX_TRACE("dm send r%d -> %d tag %d %lld B", c->rank, dest, tag, (long long)bytes);
    if (!blocking) {
        auto req = std::make_shared<ReqState>();
        req->comm = c;
        req->is_send = true;
        req->matched = true;   // buffered: complete at its stream position
        c->outstanding++;
        if (out_req) *out_req = req;
    }
    return MPX_SUCCESS;
}

// The receive is posted at its stream position (k_dm_post); its data moves
// at the wait (blocking: right away): k_dm_wait, then the copy -- straight
// into the buffer for a contiguous layout; for a typed one into a landing
// buffer pre-filled with the layout's current bytes (so a short message
// leaves the rest of the layout as it was), unpacked afterwards.
int dm_recv_op(const std::shared_ptr<Comm>& c, void* buf, int64_t count, Datatype* dt, int source, int tag,
               bool blocking, std::shared_ptr<ReqState>* out_req) {
    World* w = c->w;
    const int64_t cap = dt->size * count;
    DmLay lay;
    // chain layouts (contiguous, vector, subarray faces ...) receive in place
    const bool direct = dm_chain_lay(c->device, dt, count, c->stream, &lay);
    if (!direct && cap > 0) {
        int64_t q[8];
        MPX_RC(mpx_layout_query(reinterpret_cast<mpx_datatype>(dt), count, q));
        if (q[6]) return fail(MPX_ERR_UNSUPPORTED, "device matching: receive layouts with overlapping bytes are not supported");
    }
    DmBox* box = nullptr;
    MPX_RC(dm_box_of(w, c->rank, &box));
    int slot = 0;
    MPX_RC(dm_take_slot(w, c->rank, &slot));
    DmStatus* st = &w->dm_status[(size_t)c->rank][slot];
    MPX_RC(set_device(c->device));
    const int dev = c->device;
    // other typed receives land in a buffer holding the layout's current
    // bytes (a short message leaves the rest of the layout as it was),
    // prepared at the post (a rendezvous message may be copied in at match
    // time) and unpacked at the wait
    void* landing = nullptr;
    if (!direct) {
        MPX_RC(staging_alloc(dev, (size_t)cap, c->stream, &landing));
        if (cap > 0) MPX_RC(launch_move(dev, dt, count, true, buf, landing, cap, c->stream));
        MPX_RC(set_device(dev));
        lay = dm_contig_lay(0, cap);
    }
    uint8_t* land = direct ? static_cast<uint8_t*>(buf) : static_cast<uint8_t*>(landing);
    {
        ProfScope pl(P_LAUNCH);
        MPX_CU(dm_post(box, source, tag, c->ctx, slot, land, lay, cap, cap > w->eager_limit, dev, c->stream));
    }
    auto deliver = [dev, box, slot, st, cap, direct, dt, count, buf, landing](cudaStream_t ws) -> int {
        MPX_RC(set_device(dev));
        ProfScope pl(P_LAUNCH);
        if (cap <= kDmFusedBytes) {   // wait and copy in one single-CTA kernel
            MPX_CU(dm_wait_copy(box, slot, st, cap, ws));
        } else {
            MPX_CU(dm_wait(box, slot, st, cap, ws));
            MPX_CU(dm_copy(box, slot, cap, st, dev, ws));
        }
        if (direct) return MPX_SUCCESS;
        if (cap > 0) MPX_RC(launch_move(dev, dt, count, false, landing, buf, cap, ws));
        MPX_RC(set_device(dev));
        MPX_CU(cudaFreeAsync(landing, ws));
        return MPX_SUCCESS;
    };
    MPX_TRACE("dm recv r%d <- %d tag %d posted (slot %d)", c->rank, source, tag, slot);
    if (blocking) {
        {
            std::lock_guard<std::mutex> g(w->dm_mu);
            w->dm_owner[(size_t)c->rank][(size_t)slot] = c;
        }
        {
            std::lock_guard<std::mutex> g(c->dm_mu);
            c->dm_blocking.push_back(slot);
        }
        return deliver(c->stream);
    }
    auto req = std::make_shared<ReqState>();
    req->comm = c;
    req->dm = st;
    req->dm_cap = cap;
    req->dm_size = dt->size;
    req->at_wait = deliver;
    req->needs_wait = true;
    c->outstanding++;
    if (out_req) *out_req = req;
    return MPX_SUCCESS;
}

// after the communicator's stream is drained: free consumed bounce buffers,
// report truncated blocking receives
int dm_after_sync(const std::shared_ptr<Comm>& c) {
    World* w = c->w;
    if (w->dm_mode != 1) return MPX_SUCCESS;
    MPX_RC(dm_reclaim(c));
    std::vector<int> slots;
    {
        std::lock_guard<std::mutex> g(c->dm_mu);
        slots.swap(c->dm_blocking);
    }
    std::lock_guard<std::mutex> g(w->dm_mu);
    for (int s : slots) {
        auto o = w->dm_owner[(size_t)c->rank][(size_t)s].lock();
        if (o.get() == c.get()) dm_settle_locked(w, c->rank, s);
    }
    return MPX_SUCCESS;
}

// ------------------------------------------------ multi-process (ipc.hpp)
// Eager messages (<= eager_limit, self-sends, and layouts a peer cannot
// rebuild) are packed into the sender's staging arena at its stream
// position; the receiving process unpacks from that arena and releases the
// space with the consumed flag (sends complete locally, like the reference's
// eager frames).  Larger messages whose layout is contiguous or a strided
// chain go rendezvous (transport.py:355-375,548-602): the sender publishes a
// cached IPC handle of its buffer's allocation plus its layout, the receiver
// pulls the bytes straight from the sender's buffer in ONE transfer kernel
// (typed -> typed through the zipper) over NVLink and writes the done flag
// the send completes on.  No staging copy, no size cap.
struct IpcPending {          // a receive posted before its send arrived
    std::shared_ptr<Comm> c;
    Side r;
    std::shared_ptr<ReqState> req;
    cudaEvent_t ev = nullptr;   // receiver stream position (buffer ready)
    uint32_t* flag = nullptr;   // completion, in this rank's flag range
    uint32_t gen = 0;
    bool blocking = false;
};

// the sender's layout in a form the receiving process can rebuild (chains)
bool ipc_layout_of(Datatype* dt, int64_t count, IpcLayout* out) {
    NodeP lay = dt->layout_for(count);
    const Node* n = lay.get();
    IpcLayout L;
    L.nrep = 0;
    while (n->kind == Kind::Rep) {
        if (L.nrep == kIpcMaxRep) return false;
        L.rep[L.nrep][0] = n->count;
        L.rep[L.nrep][1] = n->stride;
        L.rep[L.nrep][2] = n->base;
        L.nrep++;
        n = n->body.get();
    }
    if (n->kind != Kind::Run) return false;
    L.run_off = n->off;
    L.run_len = n->len;
    *out = L;
    return true;
}

// a datatype with exactly a peer sender's layout (receiving side; cached for
// the process lifetime -- its plans may be in use by queued transfers)
Datatype* ipc_layout_type(const IpcLayout& L) {
    static std::mutex mu;
    static std::map<std::string, std::unique_ptr<Datatype>>* cache =
        new std::map<std::string, std::unique_ptr<Datatype>>();
    const std::string key(reinterpret_cast<const char*>(&L), sizeof L);
    std::lock_guard<std::mutex> g(mu);
    auto it = cache->find(key);
    if (it != cache->end()) return it->second.get();
    NodeP n = tree::run(L.run_off, L.run_len);
    for (int i = L.nrep - 1; i >= 0; --i) n = tree::rep(L.rep[i][0], L.rep[i][1], n, L.rep[i][2]);
    auto d = std::make_unique<Datatype>();
    d->layout = n;
    d->size = n->nbytes;
    d->lb = n->min_off;
    d->ub = n->max_end;
    d->committed = true;
    d->desc = "peer-layout";
    Datatype* raw = d.get();
    cache->emplace(key, std::move(d));
    return raw;
}

int ipc_deliver(const std::shared_ptr<Comm>& c, cudaStream_t st, const Side& r, IpcMsg m, int64_t* moved) {
    *moved = std::min(m.bytes, r.bytes);
    if (m.rndv) MPX_RC(c->w->ipc->resolve(&m));   // map the sender's allocation (cached)
    MPX_RC(wait_flag(st, m.ready, m.ready_gen));
    if (*moved > 0) {
        if (m.rndv) {   // pull from the sender's buffer
            Side s;
            s.rank = m.src;
            s.device = c->w->devices[(size_t)m.src];
            s.dt = ipc_layout_type(m.layout);
            s.count = 1;
            s.buf = const_cast<uint8_t*>(m.data);
            s.bytes = m.bytes;
            MPX_RC(transfer(c->device, st, s, r, *moved));
        } else {
            MPX_RC(launch_move(c->device, r.dt, r.count, false, m.data, r.buf, *moved, st));
        }
    }
    MPX_RC(set_device(c->device));
    return write_flag(st, m.consumed, m.consumed_gen);
}

bool ipc_on_match(void* cookie, const IpcMsg& m) {
    auto* raw = static_cast<IpcPending*>(cookie);
    if (!m.rndv && raw->req) {
        // an eager message for a nonblocking receive not waited yet: it
        // unpacks when the receiver's stream reaches the wait
        std::unique_lock<std::mutex> rl(raw->req->mu);
        if (!raw->req->waited) {
            std::unique_ptr<IpcPending> p(raw);
            const int64_t moved = std::min(m.bytes, p->r.bytes);
            auto& q = p->req;
            q->matched = true;
            q->source = m.src;
            q->tag = m.tag;
            q->count = p->r.dt->size ? moved / p->r.dt->size : 0;
            q->err = m.bytes > p->r.bytes ? MPX_ERR_TRUNCATE : MPX_SUCCESS;
            auto c = p->c;
            const Side r = p->r;
            q->at_wait = [c, r, m](cudaStream_t ws) -> int {
                int64_t mv = 0;
                return ipc_deliver(c, ws, r, m, &mv);
            };
            release_event(p->ev);
            return true;
        }
    }
    set_device(raw->c->device);
    // deliver only once the receiver's stream has reached the receive's
    // post point: a delivery waiting for it on the side stream would hold up
    // every later delivery queued behind it
    const cudaError_t q = cudaEventQuery(raw->ev);
    if (q == cudaErrorNotReady || *reinterpret_cast<volatile uint32_t*>(m.ready) < m.ready_gen) {
        cudaGetLastError();
        return false;   // the post point or the sender's data is not there yet
    }
    std::unique_ptr<IpcPending> p(raw);
    const auto& c = p->c;
    int64_t moved = 0;
    int rc = q == cudaSuccess ? MPX_SUCCESS : cuda_fail(q, "cudaEventQuery");
    // every input is reached: the late stream (never behind a waiting op)
    cudaStream_t st = c->late_stream();
    if (!rc && !st) rc = cuda_fail(c->late_err, "cudaStreamCreate(late)");
    if (!rc) rc = ipc_deliver(c, st, p->r, m, &moved);
    if (!rc) rc = write_flag(st, p->flag, p->gen);
    release_event(p->ev);
    const bool trunc = m.bytes > p->r.bytes;
    fill_status(p->req, p->r, m.src, m.tag, moved, trunc);
    if (rc) defer_error(c, rc, "multi-process delivery failed: " + g_last_error);
    else if (trunc && p->blocking)
        defer_error(c, MPX_ERR_TRUNCATE, "message truncated: incoming data larger than the posted receive");
    return true;
}

int ipc_send(const std::shared_ptr<Comm>& c, const void* buf, int64_t count, Datatype* dt, int dest, int tag,
             bool blocking, std::shared_ptr<ReqState>* out_req) {
    IpcWorld* ipc = c->w->ipc;
    const int64_t bytes = dt->size * count;
    IpcSend s;
    s.dest = dest;
    s.ctx = c->ctx;
    s.tag = tag;
    s.bytes = bytes;
    const bool rndv = bytes > c->w->eager_limit && dest != c->rank && ipc_layout_of(dt, count, &s.layout) &&
                      ipc->export_buffer(buf, &s.handle, &s.bufid, &s.buf_off) == MPX_SUCCESS;
    MPX_RC(set_device(c->device));
    uint32_t* done = nullptr;
    uint32_t dgen = 0;
    if (rndv) {
        s.rndv = 1;
        s.ready = ipc->local_flag(&s.ready_gen);
        done = ipc->local_flag(&dgen);
        s.cons_idx = ipc->flag_index(done);
        s.cons_gen = dgen;
        MPX_RC(write_flag(c->stream, s.ready, s.ready_gen));   // the buffer is ready at this stream position
    } else {
        uint8_t* slot = nullptr;
        MPX_RC(ipc->reserve(bytes, &slot, &s.off, &s.ready, &s.ready_gen, &s.cons_idx, &s.cons_gen));
        if (bytes > 0) MPX_RC(launch_move(c->device, dt, count, true, buf, slot, bytes, c->stream));
        MPX_RC(set_device(c->device));
        MPX_RC(write_flag(c->stream, s.ready, s.ready_gen));
    }
    MPX_RC(ipc->post_send(s));
    MPX_TRACE("ipc send r%d -> %d tag %d %lld B (%s)", c->rank, dest, tag, (long long)bytes, rndv ? "rndv" : "eager");
    if (rndv && blocking) MPX_RC(wait_flag(c->stream, done, dgen));   // complete once the receiver has pulled it
    if (!blocking) {
        auto req = std::make_shared<ReqState>();
        req->comm = c;
        req->is_send = true;
        req->matched = true;
        if (rndv) {
            req->flag = done;
            req->gen = dgen;
            req->needs_wait = true;
        }
        c->outstanding++;
        if (out_req) *out_req = req;
    }
    return MPX_SUCCESS;
}

int ipc_recv(const std::shared_ptr<Comm>& c, void* buf, int64_t count, Datatype* dt, int source, int tag,
             bool blocking, std::shared_ptr<ReqState>* out_req) {
    IpcWorld* ipc = c->w->ipc;
    auto p = std::make_unique<IpcPending>();
    p->c = c;
    p->r.rank = c->rank;
    p->r.device = c->device;
    p->r.comm = c;
    p->r.dt = dt;
    p->r.count = count;
    p->r.buf = buf;
    p->r.bytes = dt->size * count;
    p->blocking = blocking;
    if (!blocking) {
        p->req = std::make_shared<ReqState>();
        p->req->comm = c;
    }
    auto req = p->req;
    MPX_RC(set_device(c->device));
    MPX_RC(record_new_event(c->stream, &p->ev));
    p->flag = ipc->local_flag(&p->gen);
    uint32_t* flag = p->flag;
    const uint32_t gen = p->gen;
    const Side r = p->r;
    bool matched = false;
    IpcMsg m;
    IpcPending* raw = p.release();   // owned by the mailbox entry unless matched now
    int rc = ipc->recv(c->ctx, source, tag, r.bytes, raw, &matched, &m);
    if (rc || matched) p.reset(raw);
    if (rc) {
        release_event(p->ev);
        return rc;
    }
    MPX_TRACE("ipc recv r%d <- %d tag %d %s", c->rank, source, tag, matched ? "matched" : "posted");
    if (matched && !blocking && !m.rndv) {
        // an eager message matched at initiation: the data moves when this
        // stream reaches wait_enqueue (waiting there for the sender's ready
        // flag, which the wait needs anyway; the sender never waits for it)
        release_event(p->ev);
        const int64_t moved = std::min(m.bytes, r.bytes);
        fill_status(req, r, m.src, m.tag, moved, m.bytes > r.bytes);
        req->at_wait = [c, r, m](cudaStream_t ws) -> int {
            int64_t mv = 0;
            MPX_RC(ipc_deliver(c, ws, r, m, &mv));
            return MPX_SUCCESS;
        };
        req->needs_wait = true;
        c->outstanding++;
        if (out_req) *out_req = req;
        return MPX_SUCCESS;
    }
    if (matched && !blocking && *reinterpret_cast<volatile uint32_t*>(m.ready) < m.ready_gen) {
        // rendezvous whose sender has not reached its data point: a
        // side-stream wait for that could hold up later deliveries (and the
        // sender's completion must not hang on this rank's wait), so the
        // progress thread delivers it once the ready flag is written
        req->flag = flag;
        req->gen = gen;
        req->needs_wait = true;
        ipc->defer(p.release(), m);
        c->outstanding++;
        if (out_req) *out_req = req;
        return MPX_SUCCESS;
    }
    if (matched) {
        release_event(p->ev);
        cudaStream_t st = c->stream;
        if (!blocking) {   // rendezvous with the sender's data point reached: the side stream
            cudaEvent_t fork;
            MPX_RC(record_new_event(c->stream, &fork));
            st = c->side_stream();
            if (!st) return cuda_fail(c->side_err, "cudaStreamCreate(side)");
            MPX_CU(cudaStreamWaitEvent(st, fork, 0));
            release_event(fork);
        }
        int64_t moved = 0;
        MPX_RC(ipc_deliver(c, st, r, m, &moved));
        const bool trunc = m.bytes > r.bytes;
        fill_status(req, r, m.src, m.tag, moved, trunc);
        if (trunc && blocking)
            defer_error(c, MPX_ERR_TRUNCATE, "message truncated: incoming data larger than the posted receive");
        if (!blocking) {
            MPX_RC(record_new_event(st, &req->done_ev));
            req->needs_wait = true;
        }
    } else if (blocking) {
        MPX_RC(wait_flag(c->stream, flag, gen));
    } else {
        req->flag = flag;
        req->gen = gen;
        req->needs_wait = true;
    }
    if (req) {
        c->outstanding++;
        if (out_req) *out_req = req;
    }
    return MPX_SUCCESS;
}

// Multi-process native allreduce: every rank publishes IPC handles of its
// send and receive buffers on the host (cached mappings; the call is
// collective), then on its stream: "arrived" (my buffers are ready), wait
// for every rank's arrival, reduce MY slice of every rank's send buffer in
// rank order and store it into every rank's receive buffer (peer loads and
// stores over NVLink), "finished", wait for every rank to finish (my receive
// buffer is complete and nobody reads my send buffer any more).  Flags and
// sequence numbers are per communicator context, so collectives of
// different communicators never alias.
int ipc_allreduce_native(const std::shared_ptr<Comm>& c, const void* sendbuf, void* recvbuf, int64_t count,
                         int dtype_code) {
    World* w = c->w;
    IpcWorld* ipc = w->ipc;
    const int n = w->size, me = c->rank;
    if (n > kMaxDirectRanks) return fail(MPX_ERR_UNSUPPORTED, "native allreduce supports <= %d ranks", kMaxDirectRanks);
    const int cs = (c->ctx >> 1) % IpcWorld::kCollCtx;
    const int64_t seq = ++c->coll_seq;
    std::vector<const void*> sends;
    std::vector<void*> recvs;
    MPX_RC(ipc->coll_exchange(cs, seq, sendbuf, recvbuf, count, dtype_code, &sends, &recvs));
    MPX_RC(set_device(c->device));
    cudaStream_t st = c->stream;
    const uint32_t g = static_cast<uint32_t>(seq);
    MPX_RC(write_flag(st, ipc->coll_arrive(me, cs), g));
    for (int q = 0; q < n; ++q)
        if (q != me) MPX_RC(wait_flag(st, ipc->coll_arrive(q, cs), g));
    cudaError_t e = launch_allreduce_direct(sends.data(), recvs.data(), n, me, count, dtype_code, c->device, st);
    if (e != cudaSuccess) return cuda_fail(e, "allreduce kernel");
    MPX_RC(write_flag(st, ipc->coll_finish(me, cs), g));
    for (int q = 0; q < n; ++q)
        if (q != me) MPX_RC(wait_flag(st, ipc->coll_finish(q, cs), g));
    return MPX_SUCCESS;
}

mpx_request publish_req(const std::shared_ptr<ReqState>& q) {
    std::lock_guard<std::mutex> g(g_handles_mu);
    g_reqs[q.get()] = q;
    return reinterpret_cast<mpx_request>(q.get());
}

int wait_one(const std::shared_ptr<ReqState>& q) {
    Comm* c = q->comm.get();
    std::lock_guard<std::mutex> g(q->mu);
    if (q->waited) return MPX_SUCCESS;
    q->waited = true;
    MPX_RC(set_device(c->device));
    if (q->at_wait) {
        auto f = std::move(q->at_wait);
        q->at_wait = nullptr;
        int rc = f(c->stream);
        if (rc) {
            c->outstanding--;
            return rc;
        }
    } else if (q->needs_wait) {
        if (q->done_ev) {
            MPX_CU(cudaStreamWaitEvent(c->stream, q->done_ev, 0));
            release_event(q->done_ev);
            q->done_ev = nullptr;
        } else {
            MPX_RC(wait_flag(c->stream, q->flag, q->gen));
        }
    }
    c->outstanding--;
    return MPX_SUCCESS;
}

// ---------------------------------------------------------- NCCL loading
struct Nccl {
    bool tried = false, ok = false;
    ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char* (*errStr)(ncclResult_t) = nullptr;
    // multi-process worlds: one communicator per context, id through the segment
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
};
Nccl g_nccl;
std::mutex g_nccl_mu;

bool nccl_bind(void* h) {
    g_nccl.commInitAll = (decltype(g_nccl.commInitAll))dlsym(h, "ncclCommInitAll");
    g_nccl.allReduce = (decltype(g_nccl.allReduce))dlsym(h, "ncclAllReduce");
    g_nccl.commDestroy = (decltype(g_nccl.commDestroy))dlsym(h, "ncclCommDestroy");
    g_nccl.errStr = (decltype(g_nccl.errStr))dlsym(h, "ncclGetErrorString");
    g_nccl.getUniqueId = (decltype(g_nccl.getUniqueId))dlsym(h, "ncclGetUniqueId");
    g_nccl.commInitRank = (decltype(g_nccl.commInitRank))dlsym(h, "ncclCommInitRank");
    return g_nccl.commInitAll && g_nccl.allReduce && g_nccl.commDestroy && g_nccl.errStr;
}

bool nccl_available() {
    std::lock_guard<std::mutex> g(g_nccl_mu);
    if (!g_nccl.tried) {
        g_nccl.tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
        g_nccl.ok = h && nccl_bind(h);
    }
    return g_nccl.ok;
}

// all ranks of the world call this; the first builds every comm with ncclCommInitAll
int nccl_comm_for(const std::shared_ptr<Comm>& c, ncclComm_t* out) {
    World* w = c->w;
    std::unique_lock<std::mutex> lk(w->nccl_mu);
    if (w->nccl_state == 0) {
        w->nccl_state = 1;
        lk.unlock();
        w->nccl.assign(w->size, nullptr);
        ncclResult_t r = g_nccl.commInitAll(w->nccl.data(), w->size, w->devices.data());
        lk.lock();
        w->nccl_state = r == ncclSuccess ? 2 : -1;
        w->nccl_cv.notify_all();
        if (r != ncclSuccess) return fail(MPX_ERR_TRANSPORT, "ncclCommInitAll: %s", g_nccl.errStr(r));
    }
    w->nccl_cv.wait(lk, [&] { return w->nccl_state != 1; });
    if (w->nccl_state != 2) return fail(MPX_ERR_TRANSPORT, "NCCL communicator creation failed");
    *out = w->nccl[c->rank];
    return MPX_SUCCESS;
}

// multi-process worlds: the communicator of this context, created on its
// first allreduce (collective: every rank makes the same calls in the same
// order); rank 0's unique id reaches the others through the job's segment
int nccl_comm_ipc(const std::shared_ptr<Comm>& c, ncclComm_t* out) {
    World* w = c->w;
    std::lock_guard<std::mutex> g(w->nccl_mu);
    auto it = w->nccl_ctx.find(c->ctx);
    if (it != w->nccl_ctx.end()) {
        *out = it->second;
        return MPX_SUCCESS;
    }
    if (!g_nccl.getUniqueId || !g_nccl.commInitRank)
        return fail(MPX_ERR_UNSUPPORTED, "libnccl lacks ncclGetUniqueId / ncclCommInitRank");
    ncclUniqueId id;
    std::memset(&id, 0, sizeof id);
    if (c->rank == 0) {
        ncclResult_t r = g_nccl.getUniqueId(&id);
        if (r != ncclSuccess) return fail(MPX_ERR_TRANSPORT, "ncclGetUniqueId: %s", g_nccl.errStr(r));
    }
    MPX_RC(w->ipc->share_blob(c->ctx >> 1, c->ctx, &id, sizeof id));
    MPX_RC(set_device(c->device));
    ncclComm_t nc = nullptr;
    ncclResult_t r = g_nccl.commInitRank(&nc, w->size, id, c->rank);
    if (r != ncclSuccess) return fail(MPX_ERR_TRANSPORT, "ncclCommInitRank: %s", g_nccl.errStr(r));
    w->nccl_ctx[c->ctx] = nc;
    *out = nc;
    return MPX_SUCCESS;
}

ncclDataType_t nccl_type(int code) {
    return code == MPX_INT32 ? ncclInt32 : code == MPX_INT64 ? ncclInt64 : code == MPX_FLOAT32 ? ncclFloat32
                                                                                             : ncclFloat64;
}

int elem_size(int code) {
    switch (code) {
    case MPX_INT32: case MPX_FLOAT32: return 4;
    case MPX_INT64: case MPX_FLOAT64: return 8;
    default: return 0;
    }
}

}  // namespace
}  // namespace mpx

using namespace mpx;

extern "C" {

int mpx_world_join(const char* group, int size, int rank, int device, int64_t eager_limit, mpx_world* out) {
    if (!group || size < 1 || rank < 0 || rank >= size)
        return fail(MPX_ERR_ARG, "rank %d outside job of %d", rank, size);
    if (eager_limit < 0) return fail(MPX_ERR_ARG, "eager_limit/chunk_size out of range");
    int ndev = 0;
    MPX_CU(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(MPX_ERR_ARG, "device %d not present (%d devices)", device, ndev);
    MPX_RC(set_device(device));
    MPX_CU(preload_pack_kernels());
    MPX_CU(preload_coll_kernels());
    (void)staging_pool(device);
    std::lock_guard<std::mutex> g(g_worlds_mu);
    World*& w = g_worlds[group];
    if (!w) {
        w = new World();
        w->group = group;
        w->size = size;
        w->eager_limit = eager_limit;
        w->devices.assign(size, -1);
        w->joined.assign(size, false);
        for (int i = 0; i < size; ++i) w->mbox.emplace_back(new Mailbox());
        w->next_win.assign(size, 0);
        int rc = w->flags.init();
        if (rc) {
            delete w;
            g_worlds.erase(group);
            return rc;
        }
    }
    if (w->size != size) return fail(MPX_ERR_ARG, "world %s has %d ranks, not %d", group, w->size, size);
    if (w->joined[rank]) return fail(MPX_ERR_STATE, "rank %d already joined world %s", rank, group);
    // streams for the queue, world communicator and side stream of this rank
    // and of the ranks still to join (+ the device's late and service
    // streams), made now (see StreamPool::reserve) -- and no more: every
    // extra stream shares a hardware queue sooner.  (Topping the free list up
    // to 3 x size at every join made the pool grow by ~3 streams per joined
    // rank: 120 streams over the test suite, where two ranks' streams on one
    // hardware queue can park each other in a memop handshake.)
    int still = 0;
    for (int r = 0; r < size; ++r) still += w->joined[r] ? 0 : 1;
    MPX_CU(stream_pool().reserve(device, (size_t)std::min(64, 3 * still + 2)));
    MPX_RC(setup_device(w, device, ndev));
    w->joined[rank] = true;
    w->devices[rank] = device;
    w->live++;
    *out = reinterpret_cast<mpx_world>(w);
    return MPX_SUCCESS;
}

int mpx_ipc_world_join(const char* job, int size, int rank, int device, int64_t eager_limit, int64_t arena_bytes,
                       mpx_world* out) {
    if (!job || size < 1 || rank < 0 || rank >= size) return fail(MPX_ERR_ARG, "rank %d outside job of %d", rank, size);
    if (eager_limit < 0 || arena_bytes <= 0) return fail(MPX_ERR_ARG, "eager_limit / arena size out of range");
    int ndev = 0;
    MPX_CU(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(MPX_ERR_ARG, "device %d not present (%d devices)", device, ndev);
    MPX_RC(set_device(device));
    MPX_CU(preload_pack_kernels());
    MPX_CU(preload_coll_kernels());
    (void)staging_pool(device);
    IpcWorld* ipc = nullptr;
    MPX_RC(IpcWorld::join(job, size, rank, device, arena_bytes, ipc_on_match, &ipc));
    auto* w = new World();
    w->group = job;
    w->ipc = ipc;
    w->size = size;
    w->eager_limit = eager_limit;
    w->joined.assign(size, false);
    w->devices.resize(size);
    for (int r = 0; r < size; ++r) w->devices[r] = ipc->device_of(r);
    w->next_win.assign(size, 0);
    int rc = stream_pool().reserve(device, 8) != cudaSuccess ? fail(MPX_ERR_OTHER, "stream reserve") : MPX_SUCCESS;
    if (!rc) rc = setup_device(w, device, ndev);
    if (rc) return rc;
    w->joined[rank] = true;
    w->live = 1;
    *out = reinterpret_cast<mpx_world>(w);
    return MPX_SUCCESS;
}

int mpx_world_barrier(mpx_world h) {
    auto* w = reinterpret_cast<World*>(h);
    if (!w) return fail(MPX_ERR_STATE, "not a live world");
    if (!w->ipc) return fail(MPX_ERR_UNSUPPORTED, "in-process worlds synchronise their rank threads in the caller");
    return w->ipc->barrier();
}

int mpx_world_set_matching(mpx_world h, int device_side) {
    auto* w = reinterpret_cast<World*>(h);
    if (!w) return fail(MPX_ERR_STATE, "not a live world");
    if (device_side != 0 && device_side != 1) return fail(MPX_ERR_ARG, "matching mode must be 0 (host) or 1 (device)");
    if (w->ipc && device_side) return fail(MPX_ERR_UNSUPPORTED, "device matching is built for in-process worlds");
    std::lock_guard<std::mutex> g(w->dm_mu);
    if (w->dm_mode < 0) {
        if (device_side) {
            MPX_CU(preload_dm_kernels());
            w->dm_box.assign((size_t)w->size, nullptr);
            w->dm_status.assign((size_t)w->size, nullptr);
            w->dm_next.assign((size_t)w->size, 0);
            w->dm_rec_next.assign((size_t)w->size, 0);
            w->dm_owner.assign((size_t)w->size, std::vector<std::weak_ptr<Comm>>((size_t)kDmResults));
        }
        w->dm_mode = device_side;
    } else if (w->dm_mode != device_side) {
        return fail(MPX_ERR_ARG, "ranks of world %s disagree on the matching mode (%s here)", w->group.c_str(),
                    device_side ? "device" : "host");
    }
    return MPX_SUCCESS;
}

int mpx_world_leave(mpx_world h, int rank) {
    auto* w = reinterpret_cast<World*>(h);
    if (w && w->ipc) {
        if (rank < 0 || rank >= w->size || !w->joined[rank]) return fail(MPX_ERR_STATE, "rank %d not in world", rank);
        for (auto& kv : w->nccl_ctx) g_nccl.commDestroy(kv.second);
        w->nccl_ctx.clear();
        int rc = w->ipc->leave();
        for (auto& kv : w->area) {
            set_device(kv.first);
            cudaFree(kv.second);
        }
        for (auto& kv : w->late) stream_pool().release(kv.first, kv.second);
        for (auto& kv : w->svc)
            if (kv.second) stream_pool().release(kv.first, kv.second);
        delete w;
        return rc;
    }
    std::lock_guard<std::mutex> g(g_worlds_mu);
    auto it = g_worlds.find(w ? w->group : std::string());
    if (!w || it == g_worlds.end() || it->second != w) return fail(MPX_ERR_STATE, "not a live world");
    if (rank < 0 || rank >= w->size || !w->joined[rank]) return fail(MPX_ERR_STATE, "rank %d not in world", rank);
    w->joined[rank] = false;
    if (--w->live == 0) {
        w->stop_deferred();
        for (size_t r = 0; r < w->dm_box.size(); ++r) {
            if (w->dm_box[r]) {
                set_device(w->devices[r]);
                cudaFree(w->dm_box[r]);
            }
            if (w->dm_status[r]) cudaFreeHost(w->dm_status[r]);
        }
        for (auto& kv : w->area) {
            set_device(kv.first);
            cudaFree(kv.second);
        }
        if (w->nccl_state == 2)
            for (auto cm : w->nccl)
                if (cm) g_nccl.commDestroy(cm);
        for (auto& kv : w->late) stream_pool().release(kv.first, kv.second);
        for (auto& kv : w->svc)
            if (kv.second) stream_pool().release(kv.first, kv.second);
        g_worlds.erase(it);
        delete w;
    }
    return MPX_SUCCESS;
}

int mpx_comm_create(mpx_world h, int rank, int ctx, void* stream, mpx_comm* out) {
    auto* w = reinterpret_cast<World*>(h);
    if (!w || rank < 0 || rank >= w->size) return fail(MPX_ERR_ARG, "bad world / rank");
    const int dev = w->devices[rank];
    MPX_RC(set_device(dev));
    auto c = std::make_shared<Comm>();
    c->w = w;
    c->rank = rank;
    c->ctx = ctx;
    c->device = dev;
    c->stream = reinterpret_cast<cudaStream_t>(stream);
    // the side stream is created on first use (Comm::side_stream)
    {   // ring index of this context (the same in every device's area)
        std::lock_guard<std::mutex> g(w->coll_mu);
        auto it = w->ring_index.find(ctx);
        if (it == w->ring_index.end()) {
            const int idx = (int)w->ring_index.size();
            if (idx >= World::kMaxRings) return fail(MPX_ERR_EXHAUSTED, "too many communicator contexts with collectives");
            it = w->ring_index.emplace(ctx, idx).first;
        }
        c->ring = it->second;
    }
    std::lock_guard<std::mutex> g(g_handles_mu);
    g_comms[c.get()] = c;
    *out = reinterpret_cast<mpx_comm>(c.get());
    return MPX_SUCCESS;
}

int mpx_comm_free(mpx_comm h) {
    auto c = comm_of(h);
    if (!c) return fail(MPX_ERR_STATE, "communicator already freed");
    if (c->outstanding.load() > 0)
        return fail(MPX_ERR_PENDING, "communicator has %lld outstanding operations", (long long)c->outstanding.load());
    std::lock_guard<std::mutex> g(g_handles_mu);
    g_comms.erase(h);   // destroyed once no pending operation references it
    return MPX_SUCCESS;
}

int mpx_send_enqueue(mpx_comm h, const void* buf, int64_t bb, int64_t count, mpx_datatype dt, int dest, int tag) {
    auto c = comm_of(h);
    if (!c) return fail(MPX_ERR_STATE, "communicator already freed");
    MPX_RC(c->throttle());
    Datatype* d = lookup(dt);
    if (!d) return fail(MPX_ERR_ARG, "not a datatype handle");
    return do_send(c, buf, bb, count, d, dest, tag, true, nullptr);
}

int mpx_recv_enqueue(mpx_comm h, void* buf, int64_t bb, int64_t count, mpx_datatype dt, int source, int tag) {
    auto c = comm_of(h);
    if (!c) return fail(MPX_ERR_STATE, "communicator already freed");
    MPX_RC(c->throttle());
    Datatype* d = lookup(dt);
    if (!d) return fail(MPX_ERR_ARG, "not a datatype handle");
    return do_recv(c, buf, bb, count, d, source, tag, true, nullptr);
}

int mpx_isend_enqueue(mpx_comm h, const void* buf, int64_t bb, int64_t count, mpx_datatype dt, int dest, int tag,
                      mpx_request* out) {
    auto c = comm_of(h);
    if (!c) return fail(MPX_ERR_STATE, "communicator already freed");
    MPX_RC(c->throttle());
    Datatype* d = lookup(dt);
    if (!d) return fail(MPX_ERR_ARG, "not a datatype handle");
    std::shared_ptr<ReqState> q;
    MPX_RC(do_send(c, buf, bb, count, d, dest, tag, false, &q));
    *out = publish_req(q);
    return MPX_SUCCESS;
}

int mpx_irecv_enqueue(mpx_comm h, void* buf, int64_t bb, int64_t count, mpx_datatype dt, int source, int tag,
                      mpx_request* out) {
    auto c = comm_of(h);
    if (!c) return fail(MPX_ERR_STATE, "communicator already freed");
    MPX_RC(c->throttle());
    Datatype* d = lookup(dt);
    if (!d) return fail(MPX_ERR_ARG, "not a datatype handle");
    std::shared_ptr<ReqState> q;
    MPX_RC(do_recv(c, buf, bb, count, d, source, tag, false, &q));
    *out = publish_req(q);
    return MPX_SUCCESS;
}

int mpx_wait_enqueue(mpx_request h) {
    auto q = req_of(h);
    if (!q) return fail(MPX_ERR_ARG, "wait_enqueue needs a request produced by an _enqueue operation");
    MPX_RC(q->comm->throttle());
    return wait_one(q);
}

int mpx_waitall_enqueue(int n, const mpx_request* hs) {
    std::vector<std::shared_ptr<ReqState>> qs;
    for (int i = 0; i < n; ++i) {
        auto q = req_of(hs[i]);
        if (!q) return fail(MPX_ERR_ARG, "waitall_enqueue needs requests produced by _enqueue operations");
        qs.push_back(q);
    }
    for (auto& q : qs)
        if (q->comm->stream != qs[0]->comm->stream)
            return fail(MPX_ERR_ARG, "waitall_enqueue cannot mix device queues");
    if (!qs.empty()) MPX_RC(qs[0]->comm->throttle());
    for (auto& q : qs) MPX_RC(wait_one(q));
    return MPX_SUCCESS;
}

int mpx_request_status(mpx_request h, int64_t out[5]) {
    auto q = req_of(h);
    if (!q) return fail(MPX_ERR_ARG, "unknown request");
    std::lock_guard<std::mutex> g(q->mu);
    if (q->dm) {   // device-matched receive: known once the GPU has matched and copied it
        const volatile DmStatus* st = q->dm;
        const bool done = st->done != 0;
        const int64_t nb = st->bytes;
        const int64_t moved = done ? std::min<int64_t>(nb, q->dm_cap) : 0;
        out[0] = done;
        out[1] = done ? st->src : -1;
        out[2] = done ? st->tag : -1;
        out[3] = done && q->dm_size ? moved / q->dm_size : 0;
        out[4] = done ? st->err : MPX_SUCCESS;
        return MPX_SUCCESS;
    }
    out[0] = q->matched;
    out[1] = q->source;
    out[2] = q->tag;
    out[3] = q->count;
    out[4] = q->err;
    return MPX_SUCCESS;
}

int mpx_request_free(mpx_request h) {
    std::lock_guard<std::mutex> g(g_handles_mu);
    if (!g_reqs.erase(h)) return fail(MPX_ERR_ARG, "unknown request");
    return MPX_SUCCESS;
}

int mpx_comm_synchronize(mpx_comm h) {
    auto c = comm_of(h);
    if (!c) return fail(MPX_ERR_STATE, "device queue already destroyed");
    MPX_RC(set_device(c->device));
    MPX_RC(mpx_stream_wait(c->stream));
    MPX_RC(dm_after_sync(c));
    std::lock_guard<std::mutex> g(c->err_mu);
    if (!c->deferred.empty()) {
        auto e = c->deferred.front();
        c->deferred.clear();  // raise the first, drop the rest (offload.py:116-119)
        return fail(e.first, "%s", e.second.c_str());
    }
    return MPX_SUCCESS;
}

int mpx_comm_set_host_wait(mpx_comm h, int may_wait) {
    auto c = comm_of(h);
    if (!c) return fail(MPX_ERR_STATE, "communicator already freed");
    c->host_may_wait.store(may_wait != 0);
    return MPX_SUCCESS;
}

int mpx_comm_throttle_wait(mpx_comm h) {
    auto c = comm_of(h);
    if (!c) return fail(MPX_ERR_STATE, "communicator already freed");
    return c->throttle_wait();
}

int mpx_comm_progress(mpx_comm h, int64_t* outstanding) {
    auto c = comm_of(h);
    if (!c) return fail(MPX_ERR_STATE, "communicator already freed");
    if (outstanding) *outstanding = c->outstanding.load();
    return MPX_SUCCESS;
}

int mpx_stream_device(void* stream, int* device) {
    MPX_CU(cudaStreamGetDevice(reinterpret_cast<cudaStream_t>(stream), device));
    return MPX_SUCCESS;
}

// Host wait for a stream by polling cudaStreamQuery (with a short back-off)
// instead of cudaStreamSynchronize: with several ranks of one process on a
// device, a thread blocked in cudaStreamSynchronize on a stream parked in a
// stream-memop wait was seen to stall other threads' enqueue calls -- the
// very calls that would release the wait.
int mpx_stream_wait(void* stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    long ns = 1000;
    for (;;) {
        cudaError_t e = cudaStreamQuery(s);
        if (e == cudaSuccess) return MPX_SUCCESS;
        if (e != cudaErrorNotReady) return mpx::cuda_fail(e, "cudaStreamQuery");
        struct timespec ts{0, ns};
        nanosleep(&ts, nullptr);
        if (ns < 100000) ns *= 2;
    }
}

int mpx_stream_order(void* after, void* stream) {
    if (after == stream) return MPX_SUCCESS;
    mpx::ProfScope ps(mpx::P_ORDER);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int dev = 0;
    MPX_CU(cudaStreamGetDevice(s, &dev));
    MPX_RC(mpx::set_device(dev));
    cudaEvent_t ev;
    MPX_RC(mpx::record_new_event(reinterpret_cast<cudaStream_t>(after), &ev));
    cudaError_t e = cudaStreamWaitEvent(s, ev, 0);
    mpx::release_event(ev);
    return e == cudaSuccess ? MPX_SUCCESS : mpx::cuda_fail(e, "cudaStreamWaitEvent");
}

int mpx_stream_release(void* stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int dev = 0;
    MPX_CU(cudaStreamGetDevice(s, &dev));
    mpx::stream_pool().give_back(dev, s);
    return MPX_SUCCESS;
}

int mpx_stream_new(int device, void** stream) {
    if (!stream) return fail(MPX_ERR_ARG, "null output pointer");
    int ndev = 0;
    MPX_CU(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(MPX_ERR_ARG, "device %d out of range", device);
    cudaStream_t st = nullptr;
    cudaError_t e = mpx::stream_pool().acquire(device, &st);   // reserved at world join
    if (e != cudaSuccess) return mpx::cuda_fail(e, "cudaStreamCreate");
    *stream = st;
    return MPX_SUCCESS;
}

// MPX_BT=1 (diagnosis): SIGUSR2 makes the receiving thread print its native
// backtrace (with /proc/self/maps offsets resolvable by addr2line)
namespace {
void bt_handler(int) {
    void* fr[64];
    const int n = backtrace(fr, 64);
    char head[64];
    const int k = std::snprintf(head, sizeof head, "=== bt tid %ld\n", (long)syscall(SYS_gettid));
    if (write(2, head, (size_t)k) < 0) return;
    backtrace_symbols_fd(fr, n, 2);
}
struct BtInstall {
    BtInstall() {
        if (std::getenv("MPX_BT")) signal(SIGUSR2, bt_handler);
    }
} g_bt_install;
}  // namespace

int mpx_debug_flags(void) {
    std::lock_guard<std::mutex> g(mpx::g_waits_mu);
    int n = 0;
    for (const auto& w : mpx::g_waits) {
        const uint32_t v = *reinterpret_cast<volatile uint32_t*>(w.addr);
        if (v < w.gen) {
            std::fprintf(stderr, "[mpx] unmet wait: stream %p flag %p = %u < %u (stream %s)\n", (void*)w.s,
                         (void*)w.addr, v, w.gen, cudaStreamQuery(w.s) == cudaSuccess ? "idle" : "busy");
            n++;
        }
    }
    std::fprintf(stderr, "[mpx] %zu waits recorded, %d unmet\n", mpx::g_waits.size(), n);
    auto q = [](cudaEvent_t e) { return cudaEventQuery(e) == cudaSuccess ? "done" : "PENDING"; };
    for (const auto& o : mpx::g_sideops) {
        const uint32_t v = *reinterpret_cast<volatile uint32_t*>(o.flag);
        std::fprintf(stderr, "[mpx] side op r%d on %p -> flag %p (=%u): fork@%p %s, peer@%p %s, side %s\n", o.rank,
                     (void*)o.side, (void*)o.flag, v, (void*)o.fork_on, q(o.fork), (void*)o.peer_on, q(o.peer),
                     cudaStreamQuery(o.side) == cudaSuccess ? "idle" : "busy");
    }
    std::lock_guard<std::mutex> gw(mpx::g_worlds_mu);
    for (auto& kv : mpx::g_worlds) {
        for (size_t r = 0; r < kv.second->mbox.size(); ++r) {
            auto& mb = *kv.second->mbox[r];
            std::lock_guard<std::mutex> gm(mb.mu);
            for (auto& ps : mb.sends)
                std::fprintf(stderr, "[mpx] world %s rank %zu: unmatched send from %d tag %d flag %p gen %u\n",
                             kv.first.c_str(), r, ps.src, ps.tag, (void*)ps.flag, ps.gen);
            for (auto& pr : mb.recvs)
                std::fprintf(stderr, "[mpx] world %s rank %zu: unmatched recv from %d tag %d flag %p gen %u\n",
                             kv.first.c_str(), r, pr.src, pr.tag, (void*)pr.flag, pr.gen);
        }
    }
    return n;
}

int mpx_nccl_load(const char* path) {
    std::lock_guard<std::mutex> g(g_nccl_mu);
    void* h = dlopen(path, RTLD_NOW);
    if (!h) return fail(MPX_ERR_UNSUPPORTED, "dlopen(%s): %s", path, dlerror());
    g_nccl.tried = true;
    g_nccl.ok = nccl_bind(h);
    return g_nccl.ok ? MPX_SUCCESS : fail(MPX_ERR_UNSUPPORTED, "%s lacks NCCL symbols", path);
}

int mpx_allreduce_enqueue(mpx_comm h, const void* sendbuf, void* recvbuf, int64_t count, int dtype_code, int op,
                          int algo) {
    auto c = comm_of(h);
    if (!c) return fail(MPX_ERR_STATE, "communicator already freed");
    if (op != MPX_OP_SUM) return fail(MPX_ERR_ARG, "unsupported reduction op %d (only SUM)", op);
    const int es = elem_size(dtype_code);
    if (!es) return fail(MPX_ERR_ARG, "allreduce supports INT32, INT64, FLOAT32 and FLOAT64");
    if (count < 0) return fail(MPX_ERR_ARG, "count must be a nonnegative int");
    if (count == 0) return MPX_SUCCESS;  // comm.py:572-574
    MPX_RC(c->throttle());
    (void)es;
    World* w = c->w;
    MPX_RC(set_device(c->device));
    bool distinct = true;
    {
        std::set<int> ds(w->devices.begin(), w->devices.end());
        distinct = (int)ds.size() == w->size && !ds.count(-1);
    }
    if (algo == 0) algo = (w->size > 1 && distinct && nccl_available()) ? 2 : 1;
    if (algo == 2) {
        if (!distinct) return fail(MPX_ERR_UNSUPPORTED, "NCCL allreduce needs one device per rank");
        if (!nccl_available()) return fail(MPX_ERR_UNSUPPORTED, "libnccl.so.2 not available");
        ncclComm_t nc = nullptr;
        MPX_RC(w->ipc ? nccl_comm_ipc(c, &nc) : nccl_comm_for(c, &nc));
        MPX_RC(set_device(c->device));
        ncclResult_t r = g_nccl.allReduce(sendbuf, recvbuf, (size_t)count, nccl_type(dtype_code), ncclSum, nc,
                                          c->stream);
        if (r != ncclSuccess) return fail(MPX_ERR_TRANSPORT, "ncclAllReduce: %s", g_nccl.errStr(r));
        return MPX_SUCCESS;
    }
    if (w->ipc) return ipc_allreduce_native(c, sendbuf, recvbuf, count, dtype_code);
    // native one-shot: every rank's stream publishes its buffers and arrives
    // (memops into every participating device's ring copy), waits for all on
    // its own device's copy, reduces its slice into every rank, meets again
    if (w->size > kMaxCollRanks) return fail(MPX_ERR_UNSUPPORTED, "native allreduce supports <= %d ranks", kMaxCollRanks);
    const int64_t seq = c->coll_seq++;
    const int slot = (int)(seq % kCollSlots);
    const uint32_t gen = (uint32_t)(seq / kCollSlots + 1);
    std::vector<CollRing*> copies;
    CollRing* mine = nullptr;
    {
        std::lock_guard<std::mutex> g(w->coll_mu);
        std::set<int> devs(w->devices.begin(), w->devices.end());
        for (int d : devs) {
            auto it = w->area.find(d);
            if (it == w->area.end()) return fail(MPX_ERR_STATE, "device %d of the world is not set up", d);
            copies.push_back(it->second + c->ring);
            if (d == c->device) mine = it->second + c->ring;
        }
    }
    for (int j = 0; j < w->size; ++j)
        if (w->devices[j] != c->device) MPX_RC(ensure_peer(w, c->device, w->devices[j]));
    MPX_RC(set_device(c->device));
    for (CollRing* r : copies) {
        CollTable* tab = &r->table[slot];
        MPX_RC(write_ptr(c->stream, &tab->send[c->rank], sendbuf));
        MPX_RC(write_ptr(c->stream, (const void* const*)&tab->recv[c->rank], recvbuf));
        MPX_RC(write_flag(c->stream, &r->arrive[slot][c->rank], gen));
    }
    for (int j = 0; j < w->size; ++j) MPX_RC(wait_flag(c->stream, &mine->arrive[slot][j], gen));
    cudaError_t e = launch_allreduce_oneshot(&mine->table[slot], w->size, c->rank, count, dtype_code, c->device,
                                             c->stream);
    if (e != cudaSuccess) return cuda_fail(e, "allreduce launch");
    for (CollRing* r : copies) MPX_RC(write_flag(c->stream, &r->finish[slot][c->rank], gen));
    for (int j = 0; j < w->size; ++j) MPX_RC(wait_flag(c->stream, &mine->finish[slot][j], gen));
    return MPX_SUCCESS;
}

// ---------------------------------------------------------- read windows
// onesided.py:146-163 (win_create), :76-125 (get), :136-144 (free).  Every
// rank of the world exposes [base, base + bytes); a get moves target bytes
// described by (target_disp * target unit, target type) into the origin
// layout on the communicator's stream, reading the target's device memory
// directly (peer access) -- no target-side action, as in the reference's
// passive target.

int mpx_win_create(mpx_comm h, const void* base, int64_t bytes, int64_t disp_unit, int64_t* win_id) {
    auto c = comm_of(h);
    if (!c) return fail(MPX_ERR_STATE, "communicator already freed");
    if (disp_unit < 1) return fail(MPX_ERR_ARG, "disp_unit must be a positive int");
    if (bytes < 0 || (bytes > 0 && !base)) return fail(MPX_ERR_ARG, "bad window region");
    World* w = c->w;
    if (w->ipc) {   // one rank per process: exchange IPC handles through the job's segment
        const int64_t id = w->next_win[(size_t)c->rank]++;
        World::Win win;
        MPX_RC(set_device(c->device));
        MPX_RC(w->ipc->win_expose(id, base, bytes, disp_unit, &win.base, &win.bytes, &win.unit));
        win.registered = w->size;
        std::lock_guard<std::mutex> g(w->win_mu);
        w->wins[id] = win;
        *win_id = id;
        return MPX_SUCCESS;
    }
    std::unique_lock<std::mutex> lk(w->win_mu);
    const int64_t id = w->next_win[(size_t)c->rank]++;
    World::Win& win = w->wins[id];
    if (win.base.empty()) {
        win.base.assign((size_t)w->size, nullptr);
        win.bytes.assign((size_t)w->size, 0);
        win.unit.assign((size_t)w->size, 1);
    }
    win.base[(size_t)c->rank] = base;
    win.bytes[(size_t)c->rank] = bytes;
    win.unit[(size_t)c->rank] = disp_unit;
    win.registered++;
    w->win_cv.notify_all();
    w->win_cv.wait(lk, [&] { return w->wins[id].registered >= w->size; });   // collective
    *win_id = id;
    return MPX_SUCCESS;
}

// out = {bytes, disp_unit} of `rank`'s region of window `id`
int mpx_win_info(mpx_comm h, int64_t id, int rank, int64_t out[2]) {
    auto c = comm_of(h);
    if (!c) return fail(MPX_ERR_STATE, "communicator already freed");
    World* w = c->w;
    std::lock_guard<std::mutex> g(w->win_mu);
    auto it = w->wins.find(id);
    if (it == w->wins.end() || rank < 0 || rank >= w->size) return fail(MPX_ERR_ARG, "no such window / rank");
    out[0] = it->second.bytes[(size_t)rank];
    out[1] = it->second.unit[(size_t)rank];
    return MPX_SUCCESS;
}

int mpx_win_get(mpx_comm h, int64_t id, void* origin, int64_t origin_bytes, int64_t ocount, mpx_datatype odt,
                int target, int64_t tdisp, int64_t tcount, mpx_datatype tdt) {
    auto c = comm_of(h);
    if (!c) return fail(MPX_ERR_STATE, "communicator already freed");
    World* w = c->w;
    if (target < 0 || target >= w->size) return fail(MPX_ERR_ARG, "target rank %d out of range", target);
    Datatype* od = lookup(odt);
    Datatype* td = lookup(tdt);
    if (!od || !td) return fail(MPX_ERR_ARG, "bad datatype handle");
    const void* tbase;
    int64_t tbytes, tunit;
    {
        std::lock_guard<std::mutex> g(w->win_mu);
        auto it = w->wins.find(id);
        if (it == w->wins.end()) return fail(MPX_ERR_STATE, "window already freed");
        tbase = it->second.base[(size_t)target];
        tbytes = it->second.bytes[(size_t)target];
        tunit = it->second.unit[(size_t)target];
    }
    MPX_RC(check_layout_region(od, ocount, origin_bytes));
    const int64_t total = td->size * tcount;
    if (od->size * ocount != total)
        return fail(MPX_ERR_ARG, "origin and target type signatures disagree (%lld vs %lld bytes)",
                    (long long)(od->size * ocount), (long long)total);
    const int64_t off = tdisp * tunit;
    MPX_RC(check_layout_region(td, tcount, tbytes - off));   // the target's bounds check (_serve_get)
    if (total == 0) return MPX_SUCCESS;
    Side s;
    s.rank = target;
    s.device = w->devices[(size_t)target];
    s.dt = td;
    s.count = tcount;
    s.buf = const_cast<uint8_t*>(static_cast<const uint8_t*>(tbase)) + off;
    s.bytes = total;
    Side r;
    r.rank = c->rank;
    r.device = c->device;
    r.dt = od;
    r.count = ocount;
    r.buf = origin;
    r.bytes = total;
    MPX_RC(ensure_peer(w, c->device, s.device));
    MPX_RC(set_device(c->device));
    return transfer(c->device, c->stream, s, r, total);
}

int mpx_win_free(mpx_comm h, int64_t id) {
    auto c = comm_of(h);
    if (!c) return fail(MPX_ERR_STATE, "communicator already freed");
    World* w = c->w;
    if (w->ipc) {   // collective; the mappings stay cached until the world ends
        {
            std::lock_guard<std::mutex> g(w->win_mu);
            if (!w->wins.count(id)) return fail(MPX_ERR_STATE, "window already freed");
            w->wins.erase(id);
        }
        return w->ipc->barrier();
    }
    std::unique_lock<std::mutex> lk(w->win_mu);
    auto it = w->wins.find(id);
    if (it == w->wins.end()) return fail(MPX_ERR_STATE, "window already freed");
    it->second.released++;
    w->win_cv.notify_all();
    w->win_cv.wait(lk, [&] {   // collective (the reference's barrier)
        auto j = w->wins.find(id);
        return j == w->wins.end() || j->second.released >= w->size;
    });
    w->wins.erase(id);
    w->win_cv.notify_all();
    return MPX_SUCCESS;
}

}  // extern "C"
