"""Passive-target read windows -- the reference's ``onesided.py``
(/root/reference/pkg/src/minimpi/onesided.py), on the GPU.

The reference ships a GET_REQ frame of flattened target segments and the
target gathers them in its progress path (:76-125, :198-239).  Here every rank
exposes device memory -- peer-accessible over NVLink in an in-process world,
mapped through CUDA IPC handles exchanged at win_create in a multi-process one --
so a read is fully origin-driven: ``get`` moves the target bytes described by
(target_disp x the target's unit, target type) straight into the origin
layout with the datatype kernels -- the one-pass zipper when both layouts are
chains -- on the origin communicator's stream; the target does nothing.
``unlock`` completes the epoch (stream synchronisation) and raises the first
rejected read, exactly where the reference does.

Window memory: a CUDA (or pinned) tensor is exposed in place; any other
buffer is uploaded once at ``win_create`` (the window then serves that
snapshot).  The exposing rank's pending work on the window buffer must be
finished before reads are served; ``win_create`` synchronises the device, as
the reference's collective ``barrier`` orders the exposure.
"""

import ctypes

import numpy as np
import torch

from ._lib import check, lib, stream_wait
from .comms import CONVENTIONAL, Status
from .datatypes import Datatype, _count, _host_view, packed_size
from .errors import ArgError, PendingError, StateError, UnsupportedError

LOCK_SHARED = "shared"
LOCK_EXCLUSIVE = "exclusive"


def _nbytes(t):
    return t.numel() * t.element_size()


def _check_type(d, what):
    if not isinstance(d, Datatype):
        raise ArgError("%s must be a Datatype" % what)
    d.layout_query(1)          # raises for freed / uncommitted types (_check_usable)


class GetRequest:
    """One read of an epoch; completes at unlock (onesided.py:102-106)."""

    kind = "get"
    enqueued = False

    def __init__(self, target, count, finish=None, error=None, keep=()):
        self.target = target
        self.count = count
        self._finish = finish
        self._error = error
        self._keep = list(keep)
        self.complete = False
        self.status = Status(source=target)

    def _complete(self):
        if self.complete:
            return
        if self._error is not None:
            self.status = Status(source=self.target, error="ERR_ARG")
        else:
            if self._finish is not None:
                self._finish()
            self.status = Status(source=self.target, count=self.count)
        self.complete = True


class Window:
    """One rank's view of a read window (onesided.py:39-144)."""

    def __init__(self, comm, exposed, disp_unit, win_id, remote_units, remote_sizes):
        self.comm = comm
        self._exposed = exposed          # keeps the exposed buffer alive
        self.size_bytes = _nbytes(exposed)
        self.disp_unit = disp_unit
        self.win_id = win_id
        self.remote_units = remote_units  # displacement arithmetic uses the TARGET's unit
        self.remote_sizes = remote_sizes
        self.epochs = {}
        self.freed = False

    def __repr__(self):
        return "Window(id=%d, bytes=%d, comm=%r)" % (self.win_id, self.size_bytes, self.comm)

    def _check_live(self):
        if self.freed:
            raise StateError("window already freed")

    def lock(self, target_rank, lock_type=LOCK_SHARED):
        self._check_live()
        if lock_type == LOCK_EXCLUSIVE:
            raise UnsupportedError("exclusive window locks are not implemented; use shared epochs")
        if lock_type != LOCK_SHARED:
            raise ArgError("unknown lock type %r" % (lock_type,))
        if not isinstance(target_rank, int) or not 0 <= target_rank < self.comm.size:
            raise ArgError("target rank %r out of range" % (target_rank,))
        if target_rank in self.epochs:
            raise StateError("an epoch to rank %d is already open" % target_rank)
        self.epochs[target_rank] = []

    def get(self, origin_buf, origin_count, origin_dtype, target_rank, target_disp, target_count,
            target_dtype):
        """Start one read; completes at unlock (onesided.py:76-125)."""
        self._check_live()
        ops = self.epochs.get(target_rank)
        if ops is None:
            raise StateError("no access epoch open to rank %d (win_lock first)" % target_rank)
        _check_type(origin_dtype, "origin_dtype")
        _check_type(target_dtype, "target_dtype")
        _count(origin_count, "origin_count")
        _count(target_count, "target_count")
        if not isinstance(target_disp, int) or isinstance(target_disp, bool) or target_disp < 0:
            raise ArgError("target_disp must be a nonnegative int")
        total = packed_size(target_dtype, target_count)
        if packed_size(origin_dtype, origin_count) != total:
            raise ArgError("origin and target type signatures disagree (%d vs %d bytes)"
                           % (packed_size(origin_dtype, origin_count), total))
        dst, finish = self._landing_zone(origin_buf)
        # the target's bounds check (_serve_get): a rejected read fails at unlock
        base = target_disp * self.remote_units[target_rank]
        q = target_dtype.layout_query(target_count)
        if q["runs"] and (base + q["min_off"] < 0 or base + q["max_end"] > self.remote_sizes[target_rank]):
            req = GetRequest(target_rank, origin_count, error="ERR_ARG")
        else:
            if total:
                # ordered after the caller's work on the origin buffer
                self.comm._stream.wait_stream(torch.cuda.current_stream(self.comm.instance.device))
                check(lib.mpx_win_get(self.comm._h, self.win_id, dst.data_ptr(), _nbytes(dst),
                                      origin_count, origin_dtype._h, target_rank, target_disp,
                                      target_count, target_dtype._h))
            req = GetRequest(target_rank, origin_count, finish=finish, keep=(dst,))
        ops.append(req)
        return req

    def _landing_zone(self, buf):
        """Origin buffer as a device-visible tensor (+ copy-back callback)."""
        if isinstance(buf, torch.Tensor) and (buf.is_cuda or buf.is_pinned()):
            if not buf.is_contiguous():
                raise ArgError("buffer must be C-contiguous")
            return buf, None
        view = _host_view(buf, writable=True)      # validated now, filled at unlock
        dev = self.comm.instance.device
        host = np.frombuffer(view, dtype=np.uint8) if len(view) else np.zeros(0, np.uint8)
        d = torch.from_numpy(host.copy()).to(dev) if len(view) else \
            torch.zeros(1, dtype=torch.uint8, device=dev)[:0]

        def finish():
            if len(view):
                view[:] = d.cpu().numpy().tobytes()
        return d, finish

    def unlock(self, target_rank):
        """Close the epoch: wait for every read to target_rank; raise the
        first rejected read's error (onesided.py:127-134)."""
        self._check_live()
        ops = self.epochs.pop(target_rank, None)
        if ops is None:
            raise StateError("no epoch open to rank %d" % target_rank)
        stream_wait(self.comm._stream)
        first = None
        for r in ops:
            r._complete()
            if r.status.error and first is None:
                first = r
        if first is not None:
            raise ArgError("read from rank %d rejected by the target: region outside its window"
                           % first.target)

    def free(self):
        """Collective (onesided.py:136-144)."""
        self._check_live()
        if self.epochs:
            raise PendingError("window has %d open epoch(s)" % len(self.epochs))
        check(lib.mpx_win_free(self.comm._h, self.win_id))
        self.freed = True


def win_create(comm, buf, disp_unit=1):
    """Collective: expose buf for remote reads over comm (onesided.py:146-163)."""
    comm._check_live()
    if comm.kind != CONVENTIONAL:
        raise ArgError("windows attach to conventional communicators")
    if not isinstance(disp_unit, int) or isinstance(disp_unit, bool) or disp_unit < 1:
        raise ArgError("disp_unit must be a positive int")
    dev = comm.instance.device
    if isinstance(buf, torch.Tensor) and (buf.is_cuda or buf.is_pinned()):
        if not buf.is_contiguous():
            raise ArgError("buffer must be C-contiguous")
        exposed = buf
    else:
        view = _host_view(buf, writable=False)
        host = np.frombuffer(view, dtype=np.uint8) if len(view) else np.zeros(0, np.uint8)
        exposed = torch.from_numpy(host.copy()).to(dev)
    torch.cuda.synchronize(dev)        # the exposed bytes are final before any read
    wid = ctypes.c_int64()
    check(lib.mpx_win_create(comm._h, exposed.data_ptr() if _nbytes(exposed) else None,
                             _nbytes(exposed), disp_unit, ctypes.byref(wid)))
    units, sizes = [], []
    info = (ctypes.c_int64 * 2)()
    for r in range(comm.size):
        check(lib.mpx_win_info(comm._h, wid.value, r, info))
        sizes.append(info[0])
        units.append(info[1])
    return Window(comm, exposed, disp_unit, wid.value, units, sizes)


def win_lock(window, target_rank, lock_type=LOCK_SHARED):
    window.lock(target_rank, lock_type)


def win_unlock(window, target_rank):
    window.unlock(target_rank)


def win_get(window, origin_buf, origin_count, origin_dtype, target_rank, target_disp, target_count,
            target_dtype):
    return window.get(origin_buf, origin_count, origin_dtype, target_rank, target_disp, target_count,
                      target_dtype)


def win_free(window):
    window.free()
