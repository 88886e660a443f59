"""Device queues -- the reference's ``offload.py`` DeviceQueue
(/root/reference/pkg/src/minimpi/offload.py:49-169,271-304) made real: a
queue IS a CUDA stream.  Its 16-hex-character handle is the cudaStream_t
value, so ``{"type": "devstream", "value": queue.handle}`` and
``{"type": "cudaStream_t", ...}`` infos both resolve to it.

compute_enqueue(queue, fn, *args) runs ``fn`` on the host with the queue's
stream current, so the torch kernels it launches are ordered on the queue;
MinimpiErrors it raises are deferred to the next queue_synchronize exactly
like the reference's executor (offload.py:97-100, 111-119).
"""

import threading

import torch

from .errors import ArgError, MinimpiError, StateError
from ._lib import check, lib, own_stream, release_stream, stream_wait

_raw_stream = torch._C._cuda_getCurrentRawStream
_QUEUES = {}
_lock = threading.Lock()


class DeviceQueue:
    """A CUDA stream with the reference's queue lifecycle."""

    def __init__(self, instance=None, device=None, stream=None):
        if device is None:
            device = instance.device if instance is not None else torch.device(
                "cuda", torch.cuda.current_device())
        self.instance = instance
        self._owned = stream is None
        self.torch_stream = stream if stream is not None else own_stream(device)
        self.device = self.torch_stream.device
        self.handle = "%016x" % self.torch_stream.cuda_stream
        self.destroyed = False
        self._errors = []
        self._comms = []          # stream communicators bound to this queue
        with _lock:
            _QUEUES[self.handle] = self

    def __repr__(self):
        return "DeviceQueue(handle=%s)" % self.handle

    @property
    def cuda_stream(self):
        return self.torch_stream.cuda_stream

    def _check_live(self):
        if self.destroyed:
            raise StateError("device queue already destroyed")

    def _defer(self, exc):
        self._errors.append(exc)

    def synchronize(self):
        """Block until every enqueued operation has run; raise the first
        deferred error since the last sync, once (offload.py:111-119)."""
        self._check_live()
        stream_wait(self.torch_stream)
        first = self._errors[0] if self._errors else None
        del self._errors[:]
        for c in list(self._comms):
            if c.freed:
                self._comms.remove(c)
                continue
            try:
                c._synchronize()
            except MinimpiError as exc:
                if first is None:
                    first = exc
        if first is not None:
            raise first

    def destroy(self):
        """Drain, then invalidate (offload.py:121-133)."""
        self._check_live()
        stream_wait(self.torch_stream)
        self.destroyed = True
        with _lock:
            _QUEUES.pop(self.handle, None)
        if self._owned:
            release_stream(self.torch_stream)

    def stream_info(self):
        return {"type": "devstream", "value": self.handle}


def queue_create(instance=None):
    return DeviceQueue(instance)


def queue_destroy(queue):
    queue.destroy()


def queue_synchronize(queue):
    queue.synchronize()


def queue_from_hex(value):
    """offload.py:152-169: any case, optional left padding; unknown -> ArgError."""
    if not isinstance(value, str) or not value:
        raise ArgError("device queue handle must be hex text, got %r" % (value,))
    try:
        num = int(value, 16)
    except ValueError:
        raise ArgError("malformed device queue handle %r" % (value,))
    if num < 0 or num >> 64:
        raise ArgError("device queue handle %r out of range" % (value,))
    with _lock:
        q = _QUEUES.get("%016x" % num)
    if q is None:
        raise ArgError("unknown device queue handle %r" % (value,))
    return q


def _nbytes(t):
    return t.numel() * t.element_size()


def order_after_caller(stream):
    """Enqueued work runs after what the calling thread already issued on its
    current stream (program order, as the reference's serial queue gives):
    the queue's stream waits on an event of the current stream when they
    differ."""
    dev = stream.device.index
    cur = _raw_stream(dev if dev is not None else torch.cuda.current_device())
    s = stream.cuda_stream
    if cur != s:
        rc = lib.mpx_stream_order(cur, s)   # one pooled event, no Python objects
        if rc:
            check(rc)


def memcpy_enqueue(queue, dst, src, nbytes):
    """Ordered byte copy on the queue; bounds checked at enqueue
    (offload.py:271-285)."""
    queue._check_live()
    if not isinstance(nbytes, int) or isinstance(nbytes, bool) or nbytes < 0:
        raise ArgError("nbytes must be a nonnegative int")
    if not isinstance(dst, torch.Tensor) or not isinstance(src, torch.Tensor):
        raise ArgError("memcpy_enqueue needs tensors")
    if nbytes > _nbytes(dst) or nbytes > _nbytes(src):
        raise ArgError("memcpy of %d bytes overruns a %d/%d byte buffer"
                       % (nbytes, _nbytes(src), _nbytes(dst)))
    order_after_caller(queue.torch_stream)
    with torch.cuda.stream(queue.torch_stream):
        dst.reshape(-1).view(torch.uint8)[:nbytes].copy_(
            src.reshape(-1).view(torch.uint8)[:nbytes], non_blocking=True)


def compute_enqueue(queue, fn, *args):
    """Run fn with the queue's stream current: the device work it launches
    is ordered on the queue (offload.py:288-293)."""
    queue._check_live()
    if not callable(fn):
        raise ArgError("compute_enqueue needs a callable")
    order_after_caller(queue.torch_stream)
    with torch.cuda.stream(queue.torch_stream):
        try:
            fn(*args)
        except MinimpiError as exc:
            queue._defer(exc)


def saxpy(a, x, y, count):
    """y[i] = a*x[i] + y[i] (offload.py:296-304) as a device kernel on the
    current stream."""
    if count > x.numel() or count > y.numel():
        raise ArgError("saxpy count %d overruns operand buffers" % count)
    y[:count].add_(x[:count], alpha=a)
