"""Communicators, point-to-point, enqueue operations and allreduce -- the
reference's ``comm.py`` / ``p2p.py`` / ``offload.py`` / ``progress.py``
surface for the GPU-stream path, backed by libmpx.so (csrc/enqueue.cpp).

* A stream communicator (``stream_comm_create(world, stream)``,
  comm.py:619-648) bound to a CUDA-stream-backed Stream turns every user p2p
  call into an enqueue operation (p2p.py:151-185): ``send``/``recv``/
  ``isend``/``irecv`` become ``send_enqueue`` ... on the stream.
* Conventional communicators (the world) and SERIAL_CONTEXT stream
  communicators are host-blocking: their operations run on a private CUDA
  stream and return after it synchronises, which gives the reference's host
  semantics (including Status results) on the same engine.

Buffers of enqueue operations are CUDA tensors or pinned CPU tensors (the
kernels address the latter zero-copy); host-blocking operations also accept
plain host buffers (staged through the GPU).
"""

import ctypes

import numpy as np
import torch

from . import runtime as _rt
from ._lib import GIL_FASTPATH, WOULD_BLOCK, check, fast, lib, own_stream, release_stream, stream_wait
from .queues import order_after_caller
from .datatypes import FLOAT32, FLOAT64, INT32, INT64, Datatype, _host_view
from .errors import ArgError, MinimpiError, PendingError, StateError, for_status

CONVENTIONAL = "conventional"
STREAM_SINGLE = "stream_single"

ANY = -1
ANY_SOURCE = ANY
ANY_TAG = ANY
MAX_TAG = (1 << 31) - 1
SUM = "sum"

_ERR_NAMES = {1: "ERR_ARG", 2: "ERR_STATE", 3: "ERR_PENDING", 4: "ERR_TRUNCATE",
              5: "ERR_UNSUPPORTED", 6: "ERR_EXHAUSTED", 7: "ERR_TRANSPORT", 8: "ERR_OTHER"}
_DT_CODES = {id(INT32): 3, id(INT64): 4, id(FLOAT32): 5, id(FLOAT64): 6}
_ALGOS = {None: 0, "auto": 0, "native": 1, "nccl": 2}


class Status:
    """Completion record (transport.py:605-621)."""

    __slots__ = ("source", "tag", "count", "source_stream_idx", "error")

    def __init__(self, source=ANY, tag=ANY, count=0, source_stream_idx=ANY, error=None):
        self.source = source
        self.tag = tag
        self.count = count
        self.source_stream_idx = source_stream_idx
        self.error = error

    def __repr__(self):
        return ("Status(source={}, tag={}, count={}, source_stream_idx={}, error={!r})"
                .format(self.source, self.tag, self.count, self.source_stream_idx, self.error))


# ---------------------------------------------------------------- checks
# p2p.py:25-43


def _check_count(count):
    if type(count) is not int and (not isinstance(count, int) or isinstance(count, bool)) or count < 0:
        raise ArgError("count must be a nonnegative int, got %r" % (count,))


def _check_tag(tag, allow_any):
    if type(tag) is not int and (not isinstance(tag, int) or isinstance(tag, bool)):
        raise ArgError("tag must be an int, got %r" % (tag,))
    if allow_any and tag == ANY_TAG:
        return
    if not 0 <= tag <= MAX_TAG:
        raise ArgError("tag %d out of range [0, %d]" % (tag, MAX_TAG))


def _check_rank(name, value, size, allow_any=False):
    if allow_any and value == ANY:
        return
    if type(value) is not int and (not isinstance(value, int) or isinstance(value, bool)) or not 0 <= value < size:
        raise ArgError("%s %r out of range for size-%d communicator" % (name, value, size))


def _check_dtype(dtype):
    if not isinstance(dtype, Datatype):
        raise ArgError("expected a Datatype, got %r" % (dtype,))


_Tensor = torch.Tensor


def _dev_buffer(buf):
    """Enqueue operations need device-addressable memory."""
    if isinstance(buf, _Tensor) and (buf.is_cuda or buf.is_pinned()):
        if not buf.is_contiguous():
            raise ArgError("buffer must be C-contiguous")
        return buf
    raise ArgError("enqueue operations need a CUDA tensor or a pinned CPU tensor, got %s"
                   % type(buf).__name__)


def _nbytes(t):
    return t.nbytes


def _call_blocking(comm, name, *args):
    """A call that may wait on the host (collectives: peers, NCCL set-up):
    always with the GIL released."""
    f = getattr(lib, name)
    rc = f(*args)
    while rc == WOULD_BLOCK:
        check(lib.mpx_comm_throttle_wait(comm._h))
        rc = f(*args)
    return check(rc)


def _call(comm, name, *args):
    """One enqueue call on `comm`; when its host thread is too far ahead of
    the stream the call returns MPX_WOULD_BLOCK untouched: wait with the GIL
    released, then repeat it."""
    f = getattr(getattr(comm, "_lib", lib), name)
    rc = f(*args)
    while rc == WOULD_BLOCK:
        check(lib.mpx_comm_throttle_wait(comm._h))
        rc = f(*args)
    return check(rc)


# ---------------------------------------------------------------- requests


class Request:
    """Host-side request of a host-blocking communicator (progress.py:34-60)."""

    kind = "p2p"
    enqueued = False

    def __init__(self, comm, handle, finish=None, keep=()):
        self.comm = comm
        self._h = handle
        self._finish = finish
        self._keep = list(keep)
        self.complete = False
        self.status = Status()

    def _complete(self):
        if self.complete:
            return
        stream_wait(self.comm._stream)
        self.status = _status_of(self._h)
        if self._finish is not None:
            self._finish()
        self.complete = True
        self.comm._drop(self)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.mpx_request_free(h)


class EnqueuedRequest(Request):
    """Completion handle owned by a device queue (offload.py:34-46): host
    wait/test refuse it; wait_enqueue / waitall_enqueue put the wait on the
    queue; .status is valid once the queue has passed that wait."""

    kind = "enqueued"
    enqueued = True

    def __init__(self, comm, handle, keep=()):
        # hot path (one per isend/irecv_enqueue): plain attribute stores
        self.comm = comm
        self._h = handle
        self._finish = None
        self._keep = keep
        self.complete = False
        self.queue = comm._device_queue

    @property
    def status(self):
        return _status_of(self._h)

    @status.setter
    def status(self, value):
        pass


def _status_of(h):
    out = (ctypes.c_int64 * 5)()
    check(lib.mpx_request_status(h, out))
    matched, src, tag, count, err = list(out)
    return Status(source=src, tag=tag, count=count,
                  error=_ERR_NAMES.get(err) if err else None)


def completed_request():
    r = Request.__new__(Request)
    r.comm, r._h, r._finish, r._keep = None, None, None, []
    r.complete = True
    r.status = Status()
    return r


# ---------------------------------------------------------------- comms


class Communicator:
    """Conventional communicator (comm.py:60-203); host-blocking p2p through a
    private CUDA stream of this rank's device."""

    kind = CONVENTIONAL

    def __init__(self, instance, context_id, rank, size, stream=None):
        self.instance = instance
        self.context_id = context_id
        self.coll_context_id = context_id + 1
        self._rank = rank
        self.size = size
        self.freed = False
        self._device_queue = None
        self.local_stream = stream
        self._owns_stream = stream is None
        if stream is None:
            self._stream = own_stream(instance.device)
        else:
            self._stream = stream.torch_stream
        h = ctypes.c_void_p()
        check(lib.mpx_comm_create(instance._world, rank, context_id, self._stream.cuda_stream,
                                  ctypes.byref(h)))
        self._h = h.value
        # in-process ranks share one GIL: short enqueue calls keep it held
        # (_lib.fast) and a throttled call hands back MPX_WOULD_BLOCK instead
        # of waiting inside (see _call)
        self._lib = fast if (GIL_FASTPATH and instance.transport == _rt.TRANSPORT_INPROC) else lib
        if self._lib is fast:
            check(lib.mpx_comm_set_host_wait(self._h, 0))
        self._live = []           # requests / buffers kept alive until completion
        self._coll = None

    def __repr__(self):
        return "<%s kind=%s ctx=%d rank=%d/%d>" % (type(self).__name__, self.kind,
                                                   self.context_id, self._rank, self.size)

    @property
    def rank(self):
        return self._rank

    def _check_live(self):
        if self.freed:
            raise StateError("communicator already freed")

    def _drop(self, req):
        try:
            self._live.remove(req)
        except ValueError:
            pass

    def outstanding(self):
        if self.freed or not self._h:
            return 0
        out = ctypes.c_int64()
        check(lib.mpx_comm_progress(self._h, ctypes.byref(out)))
        return out.value + sum(1 for r in self._live if isinstance(r, Request) and not r.complete
                               and not r.enqueued)

    def _synchronize(self):
        """Stream sync + first deferred error of this communicator."""
        rc = lib.mpx_comm_synchronize(self._h)
        self._live = [r for r in self._live if isinstance(r, EnqueuedRequest)]
        check(rc)

    def _coll_comm(self):
        """Host collectives run on the odd (collective) context, never matching
        user traffic (comm.py:15-17)."""
        if self._coll is None:
            self._coll = Communicator.__new__(Communicator)
            c = self._coll
            c.instance, c.context_id, c.coll_context_id = self.instance, self.coll_context_id, -1
            c._rank, c.size, c.freed, c._device_queue = self._rank, self.size, False, None
            c.local_stream, c._stream, c._live, c._coll = None, self._stream, [], None
            h = ctypes.c_void_p()
            check(lib.mpx_comm_create(self.instance._world, self._rank, self.coll_context_id,
                                      self._stream.cuda_stream, ctypes.byref(h)))
            c._h = h.value
        return self._coll

    def _release(self):
        for c in (self._coll, self):
            if c is not None and c._h:
                check(lib.mpx_comm_free(c._h))
                c._h = None
        self.freed = True
        if getattr(self, "_owns_stream", False):
            self._owns_stream = False
            release_stream(self._stream)

    # p2p surface (comm.py:129-155)
    def send(self, buf, count, dtype, dest, tag):
        return send(self, buf, count, dtype, dest, tag)

    def recv(self, buf, count, dtype, source=ANY, tag=ANY):
        return recv(self, buf, count, dtype, source, tag)

    def isend(self, buf, count, dtype, dest, tag):
        return isend(self, buf, count, dtype, dest, tag)

    def irecv(self, buf, count, dtype, source=ANY, tag=ANY):
        return irecv(self, buf, count, dtype, source, tag)

    def barrier(self):
        return barrier(self)

    def allreduce(self, sendbuf, recvbuf, count, dtype, op=SUM):
        return allreduce(self, sendbuf, recvbuf, count, dtype, op)

    def free(self):
        comm_free(self)

    def get_stream(self, idx):
        self._check_live()
        if not isinstance(idx, int) or isinstance(idx, bool) or idx != 0:
            raise ArgError("communicator exposes a single stream slot, index %r is invalid" % (idx,))
        return self.local_stream if self.local_stream is not None else _rt.NULL_STREAM


class StreamComm(Communicator):
    """Single-stream communicator (comm.py:205-261) bound to a CUDA stream."""

    kind = STREAM_SINGLE


def comm_free(comm):
    """comm.py:178-190"""
    comm._check_live()
    if comm.context_id == 0:
        raise ArgError("cannot free the world communicator")
    n = comm.outstanding()
    if n:
        raise PendingError("communicator has %d outstanding operations" % n)
    comm._release()
    if comm.local_stream is not None:
        comm.local_stream.attach_count -= 1


def comm_get_stream(comm, idx):
    return comm.get_stream(idx)


def stream_comm_create(parent, stream):
    """Collective: derive a single-stream communicator (comm.py:619-648).
    A CUDA-stream or device-queue stream makes it an enqueue communicator."""
    parent._check_live()
    if parent.kind != CONVENTIONAL:
        raise ArgError("stream communicators derive from conventional ones")
    inst = parent.instance
    if stream is not _rt.NULL_STREAM:
        if not isinstance(stream, _rt.Stream):
            raise ArgError("expected a stream or NULL_STREAM, got %r" % (stream,))
        if stream.freed:
            raise PendingError("stream is being freed")
    ctx = inst.next_context_id
    inst.next_context_id += 2
    local = None if stream is _rt.NULL_STREAM else stream
    child = StreamComm(inst, ctx, parent.rank, parent.size, local)
    if local is not None:
        local.attach_count += 1
        if local.kind in (_rt.DEVICE_QUEUE, _rt.CUDA_STREAM):
            from .queues import DeviceQueue, queue_from_hex
            q = local.queue
            if q is None:
                try:
                    q = queue_from_hex("%016x" % local.cuda_stream)
                except ArgError:
                    q = DeviceQueue(device=local.device, stream=local.torch_stream)
            child._device_queue = q
            q._comms.append(child)
    inst._comms.append(child)
    inst._barrier()
    return child


# ------------------------------------------------------------- enqueue ops
# offload.py:172-268


def _queue_of(comm):
    q = comm._device_queue
    if q is None:
        raise ArgError("communicator is not bound to a device queue")
    if q.destroyed:
        raise StateError("device queue already destroyed")
    if comm.freed:
        raise StateError("communicator already freed")
    order_after_caller(comm._stream)     # the operation follows the caller's earlier work
    return q


def send_enqueue(comm, buf, count, dtype, dest, tag):
    """Blocking send as a stream operation (offload.py:184-189)."""
    _queue_of(comm)
    _check_dtype(dtype)
    _check_count(count)
    _check_tag(tag, allow_any=False)
    _check_rank("dest", dest, comm.size)
    b = _dev_buffer(buf)
    _call(comm, "mpx_send_enqueue", comm._h, b.data_ptr(), _nbytes(b), count, dtype._h, dest, tag)
    comm._live.append(b)


def recv_enqueue(comm, buf, count, dtype, source=ANY_SOURCE, tag=ANY_TAG):
    """Blocking receive as a stream operation (offload.py:192-195); returns
    None like the reference; truncation is deferred to queue_synchronize."""
    _queue_of(comm)
    _check_dtype(dtype)
    _check_count(count)
    _check_tag(tag, allow_any=True)
    _check_rank("source", source, comm.size, allow_any=True)
    b = _dev_buffer(buf)
    _call(comm, "mpx_recv_enqueue", comm._h, b.data_ptr(), _nbytes(b), count, dtype._h, source, tag)
    comm._live.append(b)


def isend_enqueue(comm, buf, count, dtype, dest, tag):
    """Initiation only (offload.py:198-212)."""
    _queue_of(comm)
    _check_dtype(dtype)
    _check_count(count)
    _check_tag(tag, allow_any=False)
    _check_rank("dest", dest, comm.size)
    b = _dev_buffer(buf)
    h = ctypes.c_void_p()
    _call(comm, "mpx_isend_enqueue", comm._h, b.data_ptr(), _nbytes(b), count, dtype._h, dest, tag,
          ctypes.byref(h))
    r = EnqueuedRequest(comm, h.value, keep=(b,))
    comm._live.append(r)
    return r


def irecv_enqueue(comm, buf, count, dtype, source=ANY_SOURCE, tag=ANY_TAG):
    """offload.py:215-227"""
    _queue_of(comm)
    _check_dtype(dtype)
    _check_count(count)
    _check_tag(tag, allow_any=True)
    _check_rank("source", source, comm.size, allow_any=True)
    b = _dev_buffer(buf)
    h = ctypes.c_void_p()
    _call(comm, "mpx_irecv_enqueue", comm._h, b.data_ptr(), _nbytes(b), count, dtype._h, source, tag,
          ctypes.byref(h))
    r = EnqueuedRequest(comm, h.value, keep=(b,))
    comm._live.append(r)
    return r


def wait_enqueue(request):
    """Put the completion wait on the request's own queue (offload.py:241-248)."""
    if not isinstance(request, EnqueuedRequest):
        raise ArgError("wait_enqueue needs a request produced by an _enqueue operation")
    _call(request.comm, "mpx_wait_enqueue", request._h)


def waitall_enqueue(requests):
    """offload.py:251-268: every request must share one queue."""
    requests = list(requests)
    if not requests:
        return
    for r in requests:
        if not isinstance(r, EnqueuedRequest):
            raise ArgError("waitall_enqueue needs requests produced by _enqueue operations")
    q = requests[0].queue
    for r in requests[1:]:
        if r.queue is not q:
            raise ArgError("waitall_enqueue cannot mix device queues")
    hs = (ctypes.c_void_p * len(requests))(*[r._h for r in requests])
    _call(requests[0].comm, "mpx_waitall_enqueue", len(requests), hs)


# ------------------------------------------------------ host p2p surface
# p2p.py:151-185: device-queue communicators redirect to the enqueue forms


def _host_buffer(buf, device, writable):
    """(device tensor, finish-callback) for a host-blocking operation."""
    if isinstance(buf, torch.Tensor) and (buf.is_cuda or buf.is_pinned()):
        if not buf.is_contiguous():
            raise ArgError("buffer must be C-contiguous")
        return buf, None
    view = _host_view(buf, writable)
    host = np.frombuffer(view, dtype=np.uint8) if len(view) else np.zeros(0, np.uint8)
    dev = torch.from_numpy(host.copy()).to(device) if len(view) else \
        torch.zeros(1, dtype=torch.uint8, device=device)
    if not writable:
        return dev, None

    def finish():
        if len(view):
            view[:] = dev.cpu().numpy().tobytes()
    return dev, finish


def _host_isend(comm, buf, count, dtype, dest, tag):
    comm._check_live()
    _check_dtype(dtype)
    _check_count(count)
    _check_tag(tag, allow_any=False)
    _check_rank("dest", dest, comm.size)
    b, _ = _host_buffer(buf, comm.instance.device, writable=False)
    order_after_caller(comm._stream)      # the upload above ran on the caller's stream
    h = ctypes.c_void_p()
    _call(comm, "mpx_isend_enqueue", comm._h, b.data_ptr(), _nbytes(b), count, dtype._h, dest, tag,
          ctypes.byref(h))
    _call(comm, "mpx_wait_enqueue", h.value)
    r = Request(comm, h.value, keep=(b,))
    comm._live.append(r)
    return r


def _host_irecv(comm, buf, count, dtype, source, tag):
    comm._check_live()
    _check_dtype(dtype)
    _check_count(count)
    _check_tag(tag, allow_any=True)
    _check_rank("source", source, comm.size, allow_any=True)
    b, finish = _host_buffer(buf, comm.instance.device, writable=True)
    order_after_caller(comm._stream)
    h = ctypes.c_void_p()
    _call(comm, "mpx_irecv_enqueue", comm._h, b.data_ptr(), _nbytes(b), count, dtype._h, source, tag,
          ctypes.byref(h))
    _call(comm, "mpx_wait_enqueue", h.value)
    r = Request(comm, h.value, finish=finish, keep=(b,))
    comm._live.append(r)
    return r


def isend(comm, buf, count, dtype, dest, tag):
    if comm._device_queue is not None:
        return isend_enqueue(comm, buf, count, dtype, dest, tag)
    return _host_isend(comm, buf, count, dtype, dest, tag)


def irecv(comm, buf, count, dtype, source=ANY_SOURCE, tag=ANY_TAG):
    if comm._device_queue is not None:
        return irecv_enqueue(comm, buf, count, dtype, source, tag)
    return _host_irecv(comm, buf, count, dtype, source, tag)


def send(comm, buf, count, dtype, dest, tag):
    if comm._device_queue is not None:
        return send_enqueue(comm, buf, count, dtype, dest, tag)
    wait(_host_isend(comm, buf, count, dtype, dest, tag))


def recv(comm, buf, count, dtype, source=ANY_SOURCE, tag=ANY_TAG):
    """Blocking receive; returns the Status (p2p.py:180-185)."""
    if comm._device_queue is not None:
        return recv_enqueue(comm, buf, count, dtype, source, tag)
    return wait(_host_irecv(comm, buf, count, dtype, source, tag))


def _finalize(req):
    st = req.status
    if st.error:
        raise for_status(st)
    return st


def wait(request):
    """Block until complete; enqueued requests are refused (progress.py:195-212)."""
    if request.enqueued:
        raise ArgError("request belongs to a device queue; use wait_enqueue")
    if not request.complete:
        request._complete()
    return _finalize(request)


def test(request):
    """progress.py:215-223"""
    if request.enqueued:
        raise ArgError("request belongs to a device queue; use wait_enqueue")
    if not request.complete and request.comm is not None:
        if request.comm._stream.query():
            request._complete()
    if request.complete:
        return True, _finalize(request)
    return False, Status()


def waitall(requests):
    """progress.py:241-288 (host requests only)."""
    requests = list(requests)
    for r in requests:
        if r.enqueued:
            raise ArgError("request belongs to a device queue; use waitall_enqueue")
    statuses, failure = [], None
    for r in requests:
        try:
            statuses.append(wait(r))
        except MinimpiError as exc:
            failure = failure or exc
            statuses.append(exc.status)
    if failure is not None:
        raise failure
    return statuses


# ------------------------------------------------------------- collectives


def barrier(comm):
    """Host barrier of the in-process job (comm.py:536-557)."""
    comm._check_live()
    if comm.size > 1:
        comm.instance._barrier()


def _ar_check(comm, count, dtype, op):
    comm._check_live()
    if op != SUM:
        raise ArgError("unsupported reduction op %r (only SUM)" % (op,))
    code = _DT_CODES.get(id(dtype))
    if code is None:
        raise ArgError("allreduce supports INT32, INT64, FLOAT32 and FLOAT64, got %s" % (dtype,))
    _check_count(count)
    return code


def allreduce_enqueue(comm, sendbuf, recvbuf, count, dtype, op=SUM, algo=None):
    """MPIX_Allreduce_enqueue: SUM on the communicator's stream, no host
    synchronisation.  algo: None/"auto" (NCCL when every rank has its own
    device, else native), "native" (rank-ordered one-shot kernel, same
    summation order as comm.py:582-588), "nccl"."""
    _queue_of(comm)
    code = _ar_check(comm, count, dtype, op)
    if count == 0:
        return
    s, r = _dev_buffer(sendbuf), _dev_buffer(recvbuf)
    need = count * dtype.size_bytes
    if _nbytes(s) < need or _nbytes(r) < need:
        raise ArgError("allreduce buffers hold %d/%d bytes, need %d" % (_nbytes(s), _nbytes(r), need))
    _call_blocking(comm, "mpx_allreduce_enqueue", comm._h, s.data_ptr(), r.data_ptr(), count, code, 0,
                   _ALGOS.get(algo, 0))
    comm._live.extend((s, r))


def allreduce(comm, sendbuf, recvbuf, count, dtype, op=SUM, algo=None):
    """Host-blocking allreduce (comm.py:560-595) on the communicator's
    stream; returns when every rank's result is in recvbuf."""
    code = _ar_check(comm, count, dtype, op)
    if count == 0:
        return
    dev = comm.instance.device
    s, _ = _host_buffer(sendbuf, dev, writable=False)
    r, finish = _host_buffer(recvbuf, dev, writable=True)
    need = count * dtype.size_bytes
    if _nbytes(s) < need or _nbytes(r) < need:
        raise ArgError("allreduce buffers hold %d/%d bytes, need %d" % (_nbytes(s), _nbytes(r), need))
    c = comm if comm._device_queue is None else comm
    order_after_caller(comm._stream)      # the uploads above ran on the caller's stream
    _call_blocking(c, "mpx_allreduce_enqueue", c._h, s.data_ptr(), r.data_ptr(), count, code, 0,
                   _ALGOS.get(algo, 0))
    stream_wait(comm._stream)
    if finish is not None:
        finish()
