// ipc.hpp -- multi-process worlds on one node.
//
// One process per rank (e.g. launched by torchrun), the ranks of a job share
// a POSIX shared-memory segment holding, per receiving rank, a mailbox of
// posted receives and unexpected sends (process-shared mutex, sequence
// numbers for MPI's non-overtaking rule, transport.py:191-201,399-428) and
// the completion flags (registered with CUDA in every process, so streams
// wait on / write them with stream memory operations).
//
// Two ways a message moves (the reference's eager / rendezvous split,
// transport.py:355-375,548-602):
//  * eager (<= eager_limit, self-sends, and layouts the receiver cannot
//    rebuild): the sender packs into its own device staging arena (exported
//    with cudaIpcGetMemHandle at join, mapped by every peer before join
//    returns) and publishes (offset, bytes, ready flag); the receiving process
//    unpacks straight from the peer arena and writes the consumed flag that
//    frees the space.  Sends complete locally.
//  * rendezvous (larger messages whose layout is contiguous or a strided
//    chain): nothing is staged.  The sender publishes an IPC handle of the
//    allocation holding its buffer (cached per allocation), the offset, its
//    layout and a ready flag written at its stream position; the receiver
//    maps the allocation once (cached per (rank, allocation id)), pulls the
//    data with ONE transfer kernel over NVLink -- typed -> typed through the
//    one-pass zipper -- and writes the done flag the send completes on.
//
// Collectives exchange the IPC handles of every rank's send / receive
// buffers on the host (cached mappings), then run entirely on the streams
// (arrive / finish flags); NCCL communicators get their unique id through
// the segment.
//
// This file owns the shared segment, matching, flags, arenas, buffer
// export/import and the progress thread; the CUDA work (pack/unpack launches,
// memops) is issued by enqueue.cpp through the IpcMsg it is handed.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <vector>

namespace mpx {

constexpr int kIpcMaxRep = 4;

// A sender layout the receiving process can rebuild without the sender's
// datatype object: Rep^k(Run), k <= kIpcMaxRep (contiguous, vector, hvector,
// subarray faces ...).  nrep < 0: not transportable (the message is staged).
struct IpcLayout {
    int32_t nrep = -1;
    int32_t pad = 0;
    int64_t rep[kIpcMaxRep][3] = {};   // (count, stride, base), outermost first
    int64_t run_off = 0, run_len = 0;
};

// a send as seen by the receiving process
struct IpcMsg {
    int src = 0, tag = 0;
    int64_t bytes = 0;
    int32_t rndv = 0;                // 1: pull from the sender's buffer (data = its base)
    const uint8_t* data = nullptr;   // eager: packed bytes in the sender's arena; rendezvous: after resolve()
    uint32_t* ready = nullptr;       // wait >= ready_gen before reading data
    uint32_t ready_gen = 0;
    uint32_t* consumed = nullptr;    // write consumed_gen once data is read (frees arena space / completes the send)
    uint32_t consumed_gen = 0;
    // rendezvous: the sender's allocation and layout
    cudaIpcMemHandle_t handle{};
    uint64_t bufid = 0;
    int64_t buf_off = 0;             // buffer start inside the allocation
    IpcLayout layout;
};

// what a sender publishes (post_send)
struct IpcSend {
    int dest = 0, ctx = 0, tag = 0;
    int64_t bytes = 0;
    int32_t rndv = 0;
    int64_t off = 0;                 // eager: arena offset
    uint32_t* ready = nullptr;
    uint32_t ready_gen = 0;
    uint32_t cons_idx = 0, cons_gen = 0;
    cudaIpcMemHandle_t handle{};
    uint64_t bufid = 0;
    int64_t buf_off = 0;
    IpcLayout layout;
};

// called (by the progress thread of the receiving process) for a receive
// that was posted first and has now been matched by a send; returns false
// when the delivery cannot be enqueued yet (called again later)
using IpcOnMatch = bool (*)(void* cookie, const IpcMsg& m);

struct IpcShared;

class IpcWorld {
  public:
    static constexpr int kCollCtx = 16;     // context slots with collective state
    // collective over the `size` processes of job `name`; returns once every
    // rank has joined and mapped every peer's arena
    static int join(const char* name, int size, int rank, int device, int64_t arena_bytes, IpcOnMatch cb,
                    IpcWorld** out);
    int leave();       // collective; the last rank removes the segment
    int barrier();     // host barrier over the job's processes
    int size() const { return size_; }
    int rank() const { return rank_; }
    int device_of(int r) const;

    // sender (eager): room for `bytes` in this rank's arena (reclaims
    // consumed space; MPX_ERR_EXHAUSTED when receivers have not drained it)
    // and the flags of the message: `ready` to write after packing,
    // `consumed` set by the receiver.
    int reserve(int64_t bytes, uint8_t** dst, int64_t* off, uint32_t** ready, uint32_t* ready_gen,
                uint32_t* cons_idx, uint32_t* cons_gen);
    int64_t arena_bytes() const { return arena_bytes_; }
    // sender: publish a message (after enqueueing the pack / the ready write)
    int post_send(const IpcSend& s);
    // receiver: take the oldest matching unexpected send (matched = true,
    // *m filled) or post the receive with `cookie` (matched = false)
    int recv(int ctx, int src, int tag, int64_t cap, void* cookie, bool* matched, IpcMsg* m);
    // receiver: map a rendezvous message's buffer (m->data); cached
    int resolve(IpcMsg* m);
    // a completion flag in this rank's range; index of a flag of this rank
    uint32_t* local_flag(uint32_t* gen);
    uint32_t flag_index(const uint32_t* f) const;
    // hand a matched receive to the progress thread (the callback is retried
    // until it reports the delivery enqueued)
    void defer(void* cookie, const IpcMsg& m);

    // buffers of this process shared with peers: the allocation holding p
    // (IPC handle + allocation id + offset of p), cached per allocation;
    // MPX_ERR_UNSUPPORTED when p is not cudaMalloc'd device memory
    int export_buffer(const void* p, cudaIpcMemHandle_t* h, uint64_t* id, int64_t* off);
    // a peer's allocation mapped into this process (cached per (rank, id))
    int import_buffer(int rank, const cudaIpcMemHandle_t& h, uint64_t id, uint8_t** base);

    // collectives on context slot cs: publish this rank's buffers of call
    // `seq` and wait until every rank has published the same call; returns
    // every rank's send / receive buffer mapped in this process
    int coll_exchange(int cs, int64_t seq, const void* send, void* recv, int64_t count, int code,
                      std::vector<const void*>* sends, std::vector<void*>* recvs);
    uint32_t* coll_arrive(int r, int cs);   // r's stream reached call seq (value = seq)
    uint32_t* coll_finish(int r, int cs);   // r finished writing its slices of call seq
    // small blob (<= 128 B, e.g. an NCCL unique id) from rank 0 to every
    // rank, under `key` (collective)
    int share_blob(int slot, int64_t key, void* blob, size_t n);

    // windows: collective; publishes this rank's region (an IPC handle of the
    // allocation that holds it + offset) and maps every peer's.  base[r] is
    // rank r's region in this process (nullptr for an empty region).
    int win_expose(int64_t id, const void* base, int64_t bytes, int64_t unit, std::vector<const void*>* bases,
                   std::vector<int64_t>* sizes, std::vector<int64_t>* units);

    ~IpcWorld();       // frees what a failed join left behind (leave() empties it first)

  private:
    IpcWorld() = default;
    void progress_loop();
    uint32_t* flag_locked(uint32_t* gen);
    void msg_of(int entry_box, int slot, IpcMsg* m);
    void release_all();

    std::string name_;
    int size_ = 0, rank_ = 0, device_ = 0;
    int fd_ = -1;
    IpcShared* sh_ = nullptr;
    bool registered_ = false;   // sh_ registered with CUDA
    size_t map_bytes_ = 0;
    uint8_t* arena_ = nullptr;
    int64_t arena_bytes_ = 0;
    std::vector<const uint8_t*> peer_;
    IpcOnMatch cb_ = nullptr;
    struct Slot {
        int64_t off, len;
        uint32_t idx, gen;   // consumed flag
    };
    std::vector<Slot> inflight_;   // FIFO of arena slots awaiting consumption
    int64_t head_ = 0, tail_ = 0;  // ring: used space is [head_, tail_) mod arena (full when tail_ == head_)
    uint32_t next_flag_ = 0;
    std::vector<uint32_t> shadow_;
    std::mutex mu_;             // arena ring and flag allocation
    std::mutex later_mu_;
    std::vector<std::pair<void*, IpcMsg>> later_in_;
    std::mutex buf_mu_;         // export / import caches
    std::map<uint64_t, cudaIpcMemHandle_t> exported_;           // allocation id -> handle
    std::map<std::pair<int, uint64_t>, uint8_t*> imported_;     // (rank, allocation id) -> mapping
    void* thread_ = nullptr;
    volatile bool stop_ = false;
};

}  // namespace mpx
