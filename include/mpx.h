/*
 * mpx.h -- C ABI of libmpx.so, the B200-native datatype / enqueue hot path.
 *
 * Plain C: opaque handles, int64 sizes, raw device pointers, cudaStream_t
 * passed as void*.  Every function returns an MPX_* status code (0 = OK);
 * mpx_last_error() gives the calling thread's message for the last failure.
 * Codes map 1:1 onto the reference's error taxonomy
 * (/root/reference/pkg/src/minimpi/errors.py:9-70).
 *
 * Each entry point names the reference interface it replaces.  Reference
 * paths are relative to /root/reference/pkg/src/minimpi/.
 */
#ifndef MPX_H
#define MPX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (errors.py:9-70) */
#define MPX_SUCCESS          0
#define MPX_ERR_ARG          1   /* ArgError        "ERR_ARG"         */
#define MPX_ERR_STATE        2   /* StateError      "ERR_STATE"       */
#define MPX_ERR_PENDING      3   /* PendingError    "ERR_PENDING"     */
#define MPX_ERR_TRUNCATE     4   /* TruncateError   "ERR_TRUNCATE"    */
#define MPX_ERR_UNSUPPORTED  5   /* UnsupportedError"ERR_UNSUPPORTED" */
#define MPX_ERR_EXHAUSTED    6   /* ExhaustedError  "ERR_EXHAUSTED"   */
#define MPX_ERR_TRANSPORT    7   /* TransportError  "ERR_TRANSPORT"   */
#define MPX_ERR_OTHER        8   /* MinimpiError    "ERR_OTHER" (CUDA failures) */
#define MPX_WOULD_BLOCK      9   /* not an error: see mpx_comm_set_host_wait */

/* builtin datatypes (datatype.py:410-422; INT8 is new) */
#define MPX_BYTE     0
#define MPX_CHAR     1
#define MPX_INT8     2
#define MPX_INT32    3
#define MPX_INT64    4
#define MPX_FLOAT32  5
#define MPX_FLOAT64  6

typedef struct mpx_type_s *mpx_datatype;

int mpx_abi_version(void);
/* thread-local message of the last failing call */
const char *mpx_last_error(void);

/* Device tuning: L2 fetch granularity (cudaLimitMaxL2FetchGranularity,
 * 0/32/64/128 bytes) for the calling process on `device`.  Sparse layouts
 * (single-element halo faces) read 32 B sectors; a larger fetch size would
 * drag in bytes that are never used.  Returns the previous value in *prev. */
int mpx_device_set_l2_fetch(int device, int bytes, int *prev);

/* ---- datatype constructors (datatype.py:444-610) ------------------------ */
/* builtins: datatype.py:410-422 */
int mpx_type_builtin(int which, mpx_datatype *out);
/* type_contiguous: datatype.py:444-455 */
int mpx_type_contiguous(int64_t count, mpx_datatype child, mpx_datatype *out);
/* type_vector: datatype.py:458-475 (stride in child extents) */
int mpx_type_vector(int64_t count, int64_t blocklength, int64_t stride,
                    mpx_datatype child, mpx_datatype *out);
/* type_hvector: datatype.py:478-495 (stride in bytes) */
int mpx_type_hvector(int64_t count, int64_t blocklength, int64_t stride_bytes,
                     mpx_datatype child, mpx_datatype *out);
/* type_indexed_block: datatype.py:498-516 */
int mpx_type_indexed_block(int64_t blocklength, int64_t n, const int64_t *displs,
                           mpx_datatype child, mpx_datatype *out);
/* MPI_Type_indexed (absent from the reference: SURVEY 8a a3; semantics of
 * type_create_struct with byte displacement displs[i]*extent, one child) */
int mpx_type_indexed(int64_t n, const int64_t *blocklengths, const int64_t *displs,
                     mpx_datatype child, mpx_datatype *out);
/* type_create_struct: datatype.py:519-547 */
int mpx_type_create_struct(int64_t n, const int64_t *blocklengths,
                           const int64_t *byte_displs, const mpx_datatype *children,
                           mpx_datatype *out);
/* type_create_subarray (C order): datatype.py:550-583 */
int mpx_type_create_subarray(int ndims, const int64_t *full, const int64_t *sub,
                             const int64_t *offs, mpx_datatype child, mpx_datatype *out);
/* type_create_resized: datatype.py:586-591 */
int mpx_type_create_resized(mpx_datatype child, int64_t lb, int64_t extent,
                            mpx_datatype *out);
/* type_commit / type_free: datatype.py:594-610 */
int mpx_type_commit(mpx_datatype dt);
int mpx_type_free(mpx_datatype dt);

/* Datatype attributes (datatype.py:345-401):
 * info[0..7] = size_bytes, lb, ub, extent_bytes, segment_count, node_count,
 *              committed, freed */
int mpx_type_get_info(mpx_datatype dt, int64_t info[8]);

/* ---- queries --------------------------------------------------------- */
/* type_iov_len: datatype.py:618-628 (host, O(depth * log)) */
int mpx_type_iov_len(mpx_datatype dt, int64_t max_iov_bytes, int64_t *n, int64_t *bytes);
/* type_iov: datatype.py:631-650, computed on the device.  Writes *n_out
 * (offset, length) int64 pairs to dev_pairs (device memory, room for
 * cap_pairs pairs) for segments [iov_offset, iov_offset + max_iov_len) of
 * the layout replicated count times (count = 1 is the reference call). */
int mpx_type_iov(mpx_datatype dt, int64_t count, int64_t iov_offset, int64_t max_iov_len,
                 int64_t *dev_pairs, int64_t cap_pairs, int64_t *n_out, void *stream);
/* packed_size: datatype.py:731-734 */
int mpx_packed_size(mpx_datatype dt, int64_t count, int64_t *out);
/* Host-side lowering summary of layout_for(count) (datatype.py:658-661):
 * out[0..7] = runs, nbytes, min_off, max_end, node_count,
 *             plan kind (0 empty, 1 chain, 2 descriptor walk, 3 span, 4 run table),
 *             overlap, chain alignment (span plans: word-gather spec count) */
int mpx_layout_query(mpx_datatype dt, int64_t count, int64_t out[8]);
/* Host-side span lowering of layout_for(count) as int64 words (plan kind,
 * outer levels, chunks, word-gather specs and tables) for tests that
 * emulate the tables on the CPU; *n = words needed. */
int mpx_plan_dump(mpx_datatype dt, int64_t count, int64_t *out, int64_t cap, int64_t *n);

/* ---- data movement (device buffers, asynchronous on `stream`) ----------- */
/* pack: datatype.py:695-702 with _checked_view bounds (:680-692).
 * src = device buffer of src_bytes; dst = device buffer of >= packed bytes. */
int mpx_pack(mpx_datatype dt, int64_t count, const void *src, int64_t src_bytes,
             void *dst, int64_t dst_bytes, void *stream);
/* unpack: datatype.py:705-728.  *written = min(src_bytes, packed size) is
 * known at call time; when src_bytes exceeds the layout the full layout is
 * written and MPX_ERR_TRUNCATE is returned (after the launch), exactly as the
 * reference raises TruncateError after filling. */
int mpx_unpack(mpx_datatype dt, int64_t count, const void *src, int64_t src_bytes,
               void *dst, int64_t dst_bytes, int64_t *written, void *stream);
/* Batched forms: n independent pack (unpack) operations fused into as few
 * launches as possible (one launch for up to 16 strided layouts, e.g. the
 * six faces of a halo exchange).  B200 extension; no reference equivalent
 * beyond calling pack/unpack n times.  The n operations run concurrently:
 * unpack destinations of different operations must be disjoint or carry the
 * same bytes where they overlap (as in the halo bench, whose 1-wide faces lie
 * inside the 8-wide faces); with conflicting overlaps which value survives
 * is unspecified, as for concurrent MPI receives into overlapping buffers.
 * Overlaps WITHIN one layout keep the reference's last-writer-wins order. */
int mpx_pack_multi(int n, const mpx_datatype *dts, const int64_t *counts,
                   const void *const *srcs, const int64_t *src_bytes,
                   void *const *dsts, const int64_t *dst_bytes, void *stream);
int mpx_unpack_multi(int n, const mpx_datatype *dts, const int64_t *counts,
                     const void *const *srcs, const int64_t *src_bytes,
                     void *const *dsts, const int64_t *dst_bytes, void *stream);

/* ---- worlds, stream communicators, enqueue (offload.py, comm.py) ------------
 * A world is one job of `size` ranks hosted in this process (one host thread
 * per rank, each rank bound to a CUDA device; ranks may share a device) --
 * the B200 counterpart of the reference's in-process fabric
 * (transport.py:653-715, tests/_twin.py:15-58).  A stream communicator binds
 * one rank to a cudaStream_t (comm.py:619-648 with runtime.py:173-188's
 * "cudaStream_t" branch implemented).  Enqueue operations are matched on the
 * host at call time with MPI rules and ordered on the device with events and
 * stream memory operations only: no host synchronisation, no spinning
 * kernels. */
typedef struct mpx_world_s *mpx_world;
typedef struct mpx_comm_s *mpx_comm;
typedef struct mpx_request_s *mpx_request;

#define MPX_ANY_SOURCE (-1)
#define MPX_ANY_TAG    (-1)

/* InProcFabric.join (transport.py:653-715): create or join the named world. */
int mpx_world_join(const char *group, int size, int rank, int device,
                   int64_t eager_limit, mpx_world *out);
/* Instance.finalize counterpart: the last rank to leave destroys the world. */
int mpx_world_leave(mpx_world w, int rank);
/* stream_comm_create (comm.py:619-648) for one rank: stream = cudaStream_t */
int mpx_comm_create(mpx_world w, int rank, int context_id, void *stream, mpx_comm *out);
/* comm_free (comm.py:178-190): ERR_PENDING while requests are outstanding */
int mpx_comm_free(mpx_comm c);
/* send_enqueue / recv_enqueue (offload.py:184-195).  buf_bytes = size of the
 * buffer (bounds check, datatype.py:680-692 / p2p.py:63-64). */
int mpx_send_enqueue(mpx_comm c, const void *buf, int64_t buf_bytes, int64_t count,
                     mpx_datatype dt, int dest, int tag);
int mpx_recv_enqueue(mpx_comm c, void *buf, int64_t buf_bytes, int64_t count,
                     mpx_datatype dt, int source, int tag);
/* isend_enqueue / irecv_enqueue (offload.py:198-227): initiation only */
int mpx_isend_enqueue(mpx_comm c, const void *buf, int64_t buf_bytes, int64_t count,
                      mpx_datatype dt, int dest, int tag, mpx_request *out);
int mpx_irecv_enqueue(mpx_comm c, void *buf, int64_t buf_bytes, int64_t count,
                      mpx_datatype dt, int source, int tag, mpx_request *out);
/* wait_enqueue / waitall_enqueue (offload.py:241-268): completion is placed on
 * the request's stream; waitall requires one stream (ERR_ARG otherwise). */
int mpx_wait_enqueue(mpx_request r);
int mpx_waitall_enqueue(int n, const mpx_request *rs);
/* status of a request (transport.py:605-621): out[0..4] = matched, source,
 * tag, count (elements of the request's datatype), error code (MPX_*).
 * Valid once the request's stream has passed its wait. */
int mpx_request_status(mpx_request r, int64_t out[5]);
int mpx_request_free(mpx_request r);
/* allreduce (comm.py:560-595) as a stream operation: SUM over
 * MPX_INT32/INT64/FLOAT32/FLOAT64; algo 0 = auto, 1 = native rank-ordered
 * one-shot kernel (bit-identical to the reference order x0+x1+...), 2 = NCCL */
#define MPX_OP_SUM 0
int mpx_allreduce_enqueue(mpx_comm c, const void *sendbuf, void *recvbuf, int64_t count,
                          int dtype_code, int op, int algo);
/* DeviceQueue.synchronize (offload.py:111-119): stream sync, then return the
 * first deferred error (and clear it); its message via mpx_last_error(). */
int mpx_comm_synchronize(mpx_comm c);
/* explicit progress (runtime.py:141-146): reclaim staging buffers and events
 * of completed operations; never blocks.  *outstanding = live requests. */
int mpx_comm_progress(mpx_comm c, int64_t *outstanding);
/* give a stream from mpx_stream_new back to libmpx once its owner is done
 * with it and it is drained (queue destroyed, communicator freed): the
 * number of streams per device then stays that of the live owners -- more
 * streams than CUDA_DEVICE_MAX_CONNECTIONS hardware queues let a stream
 * parked in a wait park its queue-mates.  Unknown streams are ignored. */
int mpx_stream_release(void *stream);
/* Host run-ahead bound: every communicator keeps its host thread at most
 * ~64 enqueue calls ahead of its stream, waiting (polling) when further.
 * mpx_comm_set_host_wait(c, 0): such a call instead returns MPX_WOULD_BLOCK
 * before it has any effect; the caller then runs mpx_comm_throttle_wait(c)
 * (with its own locks released, e.g. Python's GIL) and repeats the call. */
int mpx_comm_set_host_wait(mpx_comm c, int may_wait);
int mpx_comm_throttle_wait(mpx_comm c);
/* order `stream` after the work already issued on `after` (same device):
 * one pooled event recorded on `after`, waited on by `stream`; no host wait */
int mpx_stream_order(void *after, void *stream);
/* device owning a cudaStream_t (for wrapping a raw handle from an Info) */
int mpx_stream_device(void *stream, int *device);
/* ---- multi-process worlds (csrc/ipc.hpp) -----------------------
 * One process per rank on one node (e.g. under torchrun): collective over
 * the `size` processes that join job name `job`.  Matching and flags live in
 * a shared-memory segment.  Eager messages (<= eager_limit, self-sends, and
 * layouts that are not strided chains) are packed into the sender's device
 * staging arena of `arena_bytes` (exported with CUDA IPC) at its stream
 * position and unpacked by the receiving process straight from there;
 * larger contiguous / chain-layout messages are pulled by the receiver
 * directly from the sender's buffer (cached IPC mapping of its allocation)
 * in one transfer kernel, and the send completes when it has been read
 * (transport.py:355-375,548-602).  Stream communicators and the send / recv
 * / isend / irecv / wait enqueue calls, allreduce_enqueue (NCCL through
 * ncclCommInitRank when every rank has its own GPU, else the rank-ordered
 * native kernel over the peers' mapped buffers) and read windows work
 * unchanged on such a world. */
int mpx_ipc_world_join(const char *job, int size, int rank, int device, int64_t eager_limit,
                       int64_t arena_bytes, mpx_world *out);
/* host barrier over the processes of a multi-process world */
int mpx_world_barrier(mpx_world w);
/* Matching mode of an in-process world (csrc/dmatch.hpp), set
 * by every rank right after mpx_world_join, before any point-to-point call:
 * 0 = on the host when an operation is enqueued (default), 1 = on the GPU
 * when each rank's stream reaches the operation (posted / unexpected queues
 * in the receiver's device memory; eager messages buffered, nonblocking
 * sends of chain layouts above the eager limit copied once at match time,
 * layout to layout).  The ranks must
 * agree (MPX_ERR_ARG otherwise); multi-process worlds: host only
 * (MPX_ERR_UNSUPPORTED).  Replaces the matching of transport.py:191-201,
 * 399-428 (executor-thread order, offload.py:87-102). */
int mpx_world_set_matching(mpx_world w, int device_side);
/* a non-blocking stream on `device` for the caller alone, owned by the
 * process (never destroyed by the library); taken from the streams libmpx
 * creates ahead of time at world join (creating a stream while another
 * rank's stream is parked in a memop wait can stall in the driver).  The Python layer gives every queue,
 * communicator and serial context its own: torch's stream pool hands out 32
 * streams round-robin, and two ranks sharing a stream would park each other
 * behind their stream-memop waits. */
int mpx_stream_new(int device, void **stream);
/* block the calling host thread until all work queued on `stream` is done,
 * polling cudaStreamQuery (never cudaStreamSynchronize: a thread blocked in
 * it on a stream parked by a peer rank was seen to stall the enqueue calls
 * of the other rank threads that would release it) */
int mpx_stream_wait(void *stream);
/* diagnostics (with MPX_TRACE set): print every recorded stream wait whose
 * flag has not been written yet; returns how many */
int mpx_debug_flags(void);
/* optional: path of libnccl.so.2 when it is not already loaded */
int mpx_nccl_load(const char *path);

/* ---- passive-target read windows (onesided.py) ------------------------- */
/* win_create (onesided.py:146-163): collective over the communicator's world;
 * every rank exposes [base, base + bytes) with its own displacement unit;
 * *win_id = the window number (k-th create of every rank). */
int mpx_win_create(mpx_comm c, const void *base, int64_t bytes, int64_t disp_unit, int64_t *win_id);
/* out = {bytes, disp_unit} of `rank`'s region of window win_id */
int mpx_win_info(mpx_comm c, int64_t win_id, int rank, int64_t out[2]);
/* Window.get (onesided.py:76-125): tcount x tdt at target displacement
 * tdisp (in the target's unit) of `target`'s region -> ocount x odt into
 * `origin`, enqueued on the communicator's stream (the target's device
 * memory is read directly: passive target).  Signatures must agree. */
int mpx_win_get(mpx_comm c, int64_t win_id, void *origin, int64_t origin_bytes, int64_t ocount,
                mpx_datatype odt, int target, int64_t tdisp, int64_t tcount, mpx_datatype tdt);
/* Window.free (onesided.py:136-144): collective */
int mpx_win_free(mpx_comm c, int64_t win_id);

#ifdef __cplusplus
}
#endif

#endif /* MPX_H */
