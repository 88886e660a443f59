// ipc.hpp -- multi-process worlds on one node.
//
// One process per rank (e.g. launched by torchrun), the ranks of a job share
// a POSIX shared-memory segment holding, per receiving rank, a mailbox of
// posted receives and unexpected sends (process-shared mutex, sequence
// numbers for MPI's non-overtaking rule, transport.py:191-201,399-428) and
// the completion flags (registered with CUDA in every process, so streams
// wait on / write them with stream memory operations).  Every process
// exports one device staging arena with cudaIpcGetMemHandle at join and maps
// its peers' arenas before the join completes -- no IPC call on the data
// path.  A send packs into the sender's own arena at its stream position
// and publishes (offset, bytes, ready flag); the receiving process unpacks
// straight from the peer arena (NVLink or local HBM) and then writes the
// consumed flag that lets the sender reuse the space.  The unpack is
// enqueued by the receiver's own thread when its receive is posted second,
// and by the receiving process's progress thread when the send is.
//
// This file owns the shared segment, matching, flags, arenas and the
// progress thread; the CUDA work (pack/unpack launches, memops) is issued by
// enqueue.cpp through the IpcMsg it is handed.
#pragma once

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

namespace mpx {

// a send as seen by the receiving process
struct IpcMsg {
    int src = 0, tag = 0;
    int64_t bytes = 0;
    const uint8_t* data = nullptr;   // in the sender's arena, mapped in this process
    uint32_t* ready = nullptr;       // wait >= ready_gen before reading data
    uint32_t ready_gen = 0;
    uint32_t* consumed = nullptr;    // write consumed_gen once data is read
    uint32_t consumed_gen = 0;
};

// called (by the progress thread of the receiving process) for a receive
// that was posted first and has now been matched by a send; returns false
// when the delivery cannot be enqueued yet (called again later)
using IpcOnMatch = bool (*)(void* cookie, const IpcMsg& m);

struct IpcShared;

class IpcWorld {
  public:
    // collective over the `size` processes of job `name`; returns once every
    // rank has joined and mapped every peer's arena
    static int join(const char* name, int size, int rank, int device, int64_t arena_bytes, IpcOnMatch cb,
                    IpcWorld** out);
    int leave();       // collective; the last rank removes the segment
    int barrier();     // host barrier over the job's processes
    int size() const { return size_; }
    int rank() const { return rank_; }
    int device_of(int r) const;

    // sender: room for `bytes` in this rank's arena (reclaims consumed space;
    // MPX_ERR_EXHAUSTED when receivers have not drained it) and the flags of
    // the message: `ready` to write after packing, `consumed` set by the
    // receiver.
    int reserve(int64_t bytes, uint8_t** dst, int64_t* off, uint32_t** ready, uint32_t* ready_gen,
                uint32_t* cons_idx, uint32_t* cons_gen);
    // sender: publish the packed message to `dest` (after enqueueing the
    // pack and the ready write)
    int post_send(int dest, int ctx, int tag, int64_t bytes, int64_t off, uint32_t* ready, uint32_t ready_gen,
                  uint32_t cons_idx, uint32_t cons_gen);
    // receiver: take the oldest matching unexpected send (matched = true,
    // *m filled) or post the receive with `cookie` (matched = false)
    int recv(int ctx, int src, int tag, int64_t cap, void* cookie, bool* matched, IpcMsg* m);
    // a completion flag in this rank's range
    uint32_t* local_flag(uint32_t* gen);
    // hand a matched receive to the progress thread (the callback is retried
    // until it reports the delivery enqueued)
    void defer(void* cookie, const IpcMsg& m);

    // collectives: the last quarter of every rank's arena is its
    // contribution area (mapped by every peer); per rank two flags in shared
    // memory count the collectives whose contribution is in place (ready)
    // and whose peer contributions it has finished reading (read)
    const uint8_t* coll_area(int r) const { return peer_[r] + coll_off_; }
    uint8_t* my_coll_area() const { return arena_ + coll_off_; }
    int64_t coll_bytes() const { return arena_bytes_ - coll_off_; }
    uint32_t* coll_ready(int r);
    uint32_t* coll_read(int r);
    uint32_t next_coll_seq() { return ++coll_seq_; }

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

    std::string name_;
    int size_ = 0, rank_ = 0, device_ = 0;
    int fd_ = -1;
    IpcShared* sh_ = nullptr;
    bool registered_ = false;   // sh_ registered with CUDA
    size_t map_bytes_ = 0;
    uint8_t* arena_ = nullptr;
    int64_t arena_bytes_ = 0;
    int64_t coll_off_ = 0;      // [0, coll_off_): point-to-point ring; rest: collective area
    uint32_t coll_seq_ = 0;
    std::vector<std::pair<std::string, void*>> opened_;   // (rank + handle bytes) -> mapping
    std::vector<const uint8_t*> peer_;
    IpcOnMatch cb_ = nullptr;
    struct Slot {
        int64_t off, len;
        uint32_t idx, gen;   // consumed flag
    };
    std::vector<Slot> inflight_;   // FIFO of arena slots awaiting consumption
    int64_t head_ = 0, tail_ = 0;  // ring: used space is [head_, tail_) mod arena
    uint32_t next_flag_ = 0;
    std::vector<uint32_t> shadow_;
    std::mutex mu_;             // arena ring and flag allocation
    std::mutex later_mu_;
    std::vector<std::pair<void*, IpcMsg>> later_in_;
    void* thread_ = nullptr;
    volatile bool stop_ = false;
};

}  // namespace mpx
