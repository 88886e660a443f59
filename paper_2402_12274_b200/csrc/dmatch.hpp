// dmatch.hpp -- device-resident message matching.
//
// In a world joined with device matching (mpx_world_set_matching), the MPI
// matching of stream-communicator point-to-point traffic happens on the GPU,
// at the moment each rank's STREAM reaches the operation -- the B200 form of
// the reference's executor-thread matching (offload.py:87-102 ->
// transport.py:399-428 for receives, :191-201 / :509-516 for arriving
// frames): every receiving rank owns a DmBox in its device memory holding the
// two MPI queues,
//
//   msg[]  -- the unexpected queue: messages that arrived before a matching
//             receive was posted (transport.py `_unexpected`);
//   recv[] -- the posted-receive queue (transport.py `_posted`);
//
// each entry stamped with a box-wide sequence number, so "earliest" is
// arrival / posting order.  One single-CTA kernel per operation, serialised
// by a spin lock in the box (system-scope atomics: senders on peer GPUs
// reach the box over NVLink):
//
//   k_dm_send  (sender's stream, after packing the message into its bounce
//              buffer): earliest posted receive that matches (source / tag /
//              context, ANY_SOURCE / ANY_TAG on the receive) -> hand the
//              message to its result slot; none -> append to msg[];
//   k_dm_post  (receiver's stream, at the receive's position): earliest
//              unexpected message that matches -> result slot; none ->
//              append to recv[];
//   k_dm_wait  (receiver's stream, at wait / blocking receive): spin until
//              the result slot is filled (a single CTA: never starves the
//              sender's kernels of SMs), write the status;
//   k_dm_copy  grid-wide copy of the message prefix that fits out of the
//              bounce buffer; its last CTA marks the bounce buffer consumed
//              (the sender's host frees it lazily) and the status done.
//
// Messages and receives of <= 64 KiB take fused single-CTA forms: k_dm_send
// packs a chain-layout message into its bounce buffer itself (no pack
// launch), and k_dm_wait_copy waits and copies in one kernel -- the same
// launch count per message as host matching.
//
// Every message and every posted receive carries its layout as a chain
// (DmLay: contiguous or Rep^k(Run) -- vector, hvector, subarray faces), and
// every copy is a chain-to-chain zipper (`chain_copy`: the packed stream cut
// into pieces contiguous on both sides), so a strided message lands in a
// strided receive in one pass.  Receives of other layouts (struct / indexed)
// land in a contiguous buffer unpacked at the wait.
//
// Eager messages (<= the eager limit, every blocking send, send layouts that
// are not chains) are buffered: packed into a bounce buffer at the sender's
// stream position, so a blocking send never waits for its receiver (rings of
// blocking sends are safe at every size; the reference guarantees it up to
// its eager limit), and copied out at the receiver's wait.
//
// Rendezvous (a nonblocking send of a chain layout above the eager limit):
// no bounce buffer -- the message announces the sender's own buffer and
// layout, and the data moves ONCE, at match time, on the stream of whichever
// side matched second (transport.py's RTS/CTS pull, :355-375 / :548-602):
//
//   k_dm_xfer  after k_dm_send (sender's stream): copies into the posted
//              receive's destination if the send matched one;
//              after k_dm_post of a receive larger than the eager limit
//              (receiver's stream): copies if the post matched a waiting
//              rendezvous message (a smaller receive's k_dm_post copies the
//              <= eager-limit prefix itself);
//
// then marks the result copied and writes the send's completion flag, which
// the send's wait_enqueue waits for (cuStreamWaitValue32).  Copies never wait
// for a wait_enqueue, so `irecv; isend; wait(send); wait(recv)` on every
// rank cannot deadlock.  A typed receive's destination is a landing buffer
// allocated and pre-filled with the layout's bytes at post time, unpacked
// at the wait.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "desc.cuh"

namespace mpx {

// a side's layout relative to its buffer pointer: a chain (desc.cuh; a
// contiguous run is a chain of depth 0) and the widest word every run start
// and length allow
struct DmLay {
    Chain c;
    int32_t align, pad;
};

constexpr int kDmSlots = 2048;        // per receiving rank: unexpected messages + posted receives, each
constexpr int kDmResults = 1 << 14;   // per receiving rank: receives in flight (posted, not yet copied)

struct DmMsg {            // an unexpected message
    int32_t state;        // 0 free, 1 queued
    int32_t src, tag, ctx;
    int64_t seq;
    const uint8_t* data;  // bounce buffer, or the sender's buffer (rendezvous)
    int64_t bytes;
    uint32_t* consumed;   // pinned host word: set to cgen once the bytes are copied out
    uint32_t cgen;
    int32_t rdv;          // 1: rendezvous (copied at match time)
    DmLay lay;            // the message's layout relative to data (bounce: contiguous)
};

struct DmRecv {           // a posted receive
    int32_t state;
    int32_t src, tag, ctx;    // patterns
    int64_t seq;
    int32_t result, pad;
    uint8_t* dst;             // where a message lands (buffer or landing)
    int64_t cap;
    DmLay lay;                // relative to dst
};

struct DmResult {         // a receive's match, written by whichever side matched
    int32_t ready;        // 1 once the fields below are valid
    int32_t src, tag;
    uint32_t ndone;       // k_dm_copy CTAs finished
    int64_t bytes;
    const uint8_t* data;
    uint32_t* consumed;
    uint32_t cgen;
    int32_t rdv;          // rendezvous: the copy happens at match time ...
    uint8_t* dst;         // ... into dst (n = min(bytes, cap) bytes)
    int64_t n;
    int32_t copier;       // 0: the sender's k_dm_xfer, 1: the receiver's (k_dm_xfer or k_dm_post)
    int32_t copied;       // 1 once the rendezvous copy is complete
    uint32_t xdone;       // k_dm_xfer CTAs finished
    uint32_t pad2;
    DmLay slay, dlay;     // the message's layout (relative to data), the receive's (relative to dst)
};

struct DmStatus {         // pinned host memory, one per result slot
    int32_t done;         // 1: matched and copied
    int32_t src, tag, err;
    int64_t bytes;        // message bytes
    int64_t pad;
};

constexpr int kDmRecords = 1 << 14;   // per sending rank: match records of rendezvous sends (ring)

struct DmBox {
    int32_t lock;
    int32_t hw_msg, hw_recv;  // entries at or above the high-water marks are free
    int32_t err;              // sticky: an unexpected-queue overflow
    int64_t next_seq;
    DmMsg msg[kDmSlots];
    DmRecv recv[kDmSlots];
    DmResult result[kDmResults];
    int32_t srec[kDmRecords];   // sends FROM this box's rank: the result slot a rendezvous send matched (-1: none)
};

// launchers (dmatch.cu); `box` is the receiving rank's box
// eager send: `data` = the bounce buffer (packed, contiguous)
cudaError_t dm_send(DmBox* box, int src, int tag, int ctx, const uint8_t* data, int64_t bytes, uint32_t* consumed,
                    uint32_t cgen, cudaStream_t stream);
// rendezvous send: `data` is the sender's buffer, `lay` its layout; the
// match is recorded in *record (in the sender's own box) and k_dm_xfer
// copies right behind it
cudaError_t dm_send_rdv(DmBox* box, int src, int tag, int ctx, const uint8_t* data, const DmLay& lay, int64_t bytes,
                        uint32_t* consumed, uint32_t cgen, int32_t* record, int device, cudaStream_t stream);
// `dst` / `lay` / `cap`: where the message lands; big: a k_dm_xfer follows
// the post (cap above the eager limit), else k_dm_post copies itself
cudaError_t dm_post(DmBox* box, int src, int tag, int ctx, int result, uint8_t* dst, const DmLay& lay, int64_t cap,
                    bool big, int device, cudaStream_t stream);
// messages and receives up to this size take the fused single-CTA kernels:
// pack inside k_dm_send, wait + copy in one k_dm_wait_copy
constexpr int64_t kDmFusedBytes = 64 << 10;
// eager send of a chain layout <= kDmFusedBytes: k_dm_send packs `data`
// (layout `lay`) into `bounce` itself
cudaError_t dm_send_packed(DmBox* box, int src, int tag, int ctx, const uint8_t* data, const DmLay& lay,
                           uint8_t* bounce, int64_t bytes, uint32_t* consumed, uint32_t cgen, cudaStream_t stream);
// a receive of <= kDmFusedBytes: k_dm_wait + k_dm_copy in one kernel
cudaError_t dm_wait_copy(DmBox* box, int result, DmStatus* status, int64_t cap, cudaStream_t stream);
// a layout that is one contiguous run of `bytes` at offset `off`
DmLay dm_contig_lay(int64_t off, int64_t bytes);
cudaError_t dm_wait(DmBox* box, int result, DmStatus* status, int64_t cap, cudaStream_t stream);
// eager messages: copy into the receive's destination (its layout, recorded
// at the post); rendezvous: already there
cudaError_t dm_copy(DmBox* box, int result, int64_t cap, DmStatus* status, int device,
                    cudaStream_t stream);
cudaError_t preload_dm_kernels();

}  // namespace mpx
