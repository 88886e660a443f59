"""Runtime lifecycle, Info objects and MPIX streams -- the reference's
``runtime.py`` / ``stream.py`` surface for the enqueue hot path.

An Instance is one rank.  ``init(transport="inproc", rank=r, ranks=n,
group=g, device=d)`` joins the named in-process world (one host thread per
rank, as the reference's InProcFabric and tests/_twin.py host them); each rank
is bound to a CUDA device (ranks may share one).  Configuration precedence is
the reference's: explicit argument > MINIMPI_* environment > default
(runtime.py:44-53, 217-257).

``Instance.stream_create(info)`` implements the branch the reference refuses
(runtime.py:186-187): ``{"type": "cudaStream_t", "value": <hex handle>}``
wraps a CUDA stream; ``"devstream"`` resolves a DeviceQueue handle (itself a
CUDA stream, see queues.py); no type gives a SERIAL_CONTEXT stream backed by
a private CUDA stream used for host-blocking communication.
"""

import ctypes
import os
import threading

import torch

from ._lib import check, lib, own_stream, release_stream
from .errors import ArgError, ExhaustedError, PendingError, StateError, UnsupportedError

TRANSPORT_INPROC = "inproc"
TRANSPORT_IPC = "ipc"          # one process per rank on one node
DEFAULT_IPC_ARENA = 256 << 20  # per-rank staging arena of a multi-process world
MATCH_HOST = "host"            # matching at enqueue time (default)
MATCH_DEVICE = "device"        # matching on the GPU at stream time (csrc/dmatch.hpp)
SERIAL_CONTEXT = "serial_context"
DEVICE_QUEUE = "device_queue"
CUDA_STREAM = "cuda_stream"

DEFAULT_EAGER_LIMIT = 65536        # transport.py:63
DEFAULT_POOL_CAPACITY = 64         # stream.py:22


def _cfg(flag, env, default, convert):
    """runtime.py:44-53"""
    if flag is not None:
        return flag
    raw = os.environ.get(env)
    if raw is not None:
        try:
            return convert(raw)
        except (TypeError, ValueError):
            raise ArgError("bad %s value %r" % (env, raw))
    return default


# ------------------------------------------------------------------ Info


class Info:
    """Ordered string key/value hints (runtime.py:264-289)."""

    def __init__(self):
        self._entries = {}

    def set(self, key, value):
        if not isinstance(key, str) or not key:
            raise ArgError("info key must be a nonempty string")
        if not isinstance(value, str):
            raise ArgError("info value must be a string")
        self._entries[key] = value

    def get(self, key, default=None):
        return self._entries.get(key, default)

    def delete(self, key):
        if key not in self._entries:
            raise ArgError("info has no key %r" % (key,))
        del self._entries[key]

    def keys(self):
        return list(self._entries)

    def __repr__(self):
        return "Info(%r)" % (self._entries,)


def info_create():
    return Info()


def info_set(info, key, value):
    info.set(key, value)


def info_set_hex(info, key, value, length=None):
    """Binary handle as lowercase hex, memory byte order kept; ints are
    zero-padded to 8 bytes unless length says otherwise (runtime.py:300-328)."""
    if length is not None and (not isinstance(length, int) or isinstance(length, bool)
                               or length < 0):
        raise ArgError("length must be a nonnegative int, got %r" % (length,))
    if isinstance(value, int) and not isinstance(value, bool):
        if value < 0:
            raise ArgError("hex info value must be nonnegative")
        width = 8 if length is None else length
        if value >> (8 * width):
            raise ArgError("value %#x does not fit in %d bytes" % (value, width))
        info.set(key, "%0*x" % (2 * width, value) if width else "")
    elif isinstance(value, (bytes, bytearray, memoryview)):
        raw = bytes(value)
        if length is not None:
            if length > len(raw):
                raise ArgError("length %d exceeds value size %d" % (length, len(raw)))
            raw = raw[:length]
        info.set(key, raw.hex())
    else:
        raise ArgError("expected int or bytes for hex value, got %r" % (value,))


def _hex_handle(value):
    if not isinstance(value, str) or not value:
        raise ArgError("stream handle must be hex text, got %r" % (value,))
    try:
        num = int(value, 16)
    except ValueError:
        raise ArgError("malformed stream handle %r" % (value,))
    if num < 0 or num >> 64:
        raise ArgError("stream handle %r out of range" % (value,))
    return num


# ---------------------------------------------------------------- streams


class _NullStream:
    _instance = None

    def __new__(cls):
        if cls._instance is None:
            cls._instance = super().__new__(cls)
        return cls._instance

    def __repr__(self):
        return "NULL_STREAM"


NULL_STREAM = _NullStream()


class Stream:
    """An MPIX stream (stream.py:43-62) backed by a CUDA stream."""

    __slots__ = ("id", "kind", "instance", "torch_stream", "device", "queue",
                 "attach_count", "freed")

    def __init__(self, sid, kind, instance, torch_stream, queue=None):
        self.id = sid
        self.kind = kind
        self.instance = instance
        self.torch_stream = torch_stream
        self.device = torch_stream.device
        self.queue = queue
        self.attach_count = 0
        self.freed = False

    @property
    def cuda_stream(self):
        return self.torch_stream.cuda_stream

    def _check_live(self, what="use"):
        if self.freed:
            raise ArgError("stream %s after free" % what)

    def __repr__(self):
        return "Stream(id=%d, kind=%s)" % (self.id, self.kind)


def free_stream(stream):
    """stream.py:137-152"""
    if stream is NULL_STREAM:
        raise ArgError("cannot free NULL_STREAM")
    if not isinstance(stream, Stream):
        raise ArgError("expected a stream, got %r" % (stream,))
    stream._check_live("free")
    if stream.attach_count > 0:
        raise PendingError("stream %d still attached to %d communicator(s)"
                           % (stream.id, stream.attach_count))
    stream.freed = True
    if stream.kind == SERIAL_CONTEXT:
        stream.instance._pool_in_use -= 1
        release_stream(stream.torch_stream)     # its own CUDA stream goes back to libmpx


# -------------------------------------------------------------- instance


class _Group:
    """In-process job: ranks of one world joined by name."""

    _lock = threading.Lock()
    _groups = {}

    def __init__(self, name, size):
        self.name = name
        self.size = size
        self.barrier = threading.Barrier(size)
        self.members = 0

    @classmethod
    def join(cls, name, size):
        with cls._lock:
            g = cls._groups.get(name)
            if g is None or g.members == 0:
                g = cls._groups[name] = _Group(name, size)
            if g.size != size:
                raise ArgError("group %s has %d ranks, not %d" % (name, g.size, size))
            g.members += 1
            return g

    def leave(self):
        with self._lock:
            self.members -= 1
            if self.members == 0 and self._groups.get(self.name) is self:
                del self._groups[self.name]


class _IpcGroup:
    """The processes of a multi-process job: barrier through libmpx's shared
    segment (mpx_world_barrier)."""

    def __init__(self, inst):
        self._inst = inst
        self.barrier = self

    def wait(self, timeout=None):
        check(lib.mpx_world_barrier(self._inst._world))

    def leave(self):
        pass


class Instance:
    """One rank of a running job (runtime.py:56-214)."""

    def __init__(self, rank, size, group, device, eager_limit, vci_pool, transport=TRANSPORT_INPROC,
                 arena=DEFAULT_IPC_ARENA, matching=MATCH_HOST):
        self.transport = transport
        self.matching = matching
        self.rank = rank
        self.size = size
        self.group = group
        self.device = torch.device("cuda", device)
        self.eager_limit = eager_limit
        self.pool_capacity = vci_pool
        self._pool_in_use = 0
        self.finalized = False
        self.next_context_id = 2
        self.next_stream_id = 0
        if transport == TRANSPORT_IPC:
            h = ctypes.c_void_p()
            check(lib.mpx_ipc_world_join(group.encode(), size, rank, device, eager_limit, arena,
                                         ctypes.byref(h)))
            self._world = h.value
            self._group = _IpcGroup(self)
            from .comms import Communicator
            self.world = Communicator(self, 0, rank, size)
            self._comms = [self.world]
            return
        self._group = _Group.join(group, size)
        h = ctypes.c_void_p()
        check(lib.mpx_world_join(group.encode(), size, rank, device, eager_limit,
                                 ctypes.byref(h)))
        self._world = h.value
        try:
            check(lib.mpx_world_set_matching(self._world, 1 if matching == MATCH_DEVICE else 0))
        except BaseException:
            lib.mpx_world_leave(self._world, rank)
            self._group.leave()
            raise
        from .comms import Communicator
        self.world = Communicator(self, 0, rank, size)
        self._comms = [self.world]

    def __repr__(self):
        return "<Instance rank=%d/%d device=%s>" % (self.rank, self.size, self.device)

    def _check_live(self):
        if self.finalized:
            raise StateError("instance already finalized")

    def _barrier(self):
        try:
            self._group.barrier.wait(timeout=float(os.environ.get("MINIMPI_BARRIER_TIMEOUT", "120")))
        except threading.BrokenBarrierError:
            raise StateError("barrier of group %s broken (a rank failed or timed out)" % self.group)

    # ---- streams (runtime.py:173-191) ----
    def stream_create(self, info=None):
        self._check_live()
        kind_val = info.get("type") if info is not None else None
        sid = self.next_stream_id
        if kind_val is None:
            if self._pool_in_use >= self.pool_capacity:
                raise ExhaustedError("VCI pool exhausted (%d in use)" % self.pool_capacity)
            self._pool_in_use += 1
            self.next_stream_id += 1
            return Stream(sid, SERIAL_CONTEXT, self, own_stream(self.device))
        if kind_val == "devstream":
            from .queues import queue_from_hex
            q = queue_from_hex(info.get("value"))
            self.next_stream_id += 1
            return Stream(sid, DEVICE_QUEUE, self, q.torch_stream, queue=q)
        if kind_val == "cudaStream_t":
            handle = _hex_handle(info.get("value"))
            dev = ctypes.c_int()
            check(lib.mpx_stream_device(handle, ctypes.byref(dev)))
            ts = torch.cuda.ExternalStream(handle, device=torch.device("cuda", dev.value))
            self.next_stream_id += 1
            return Stream(sid, CUDA_STREAM, self, ts)
        raise ArgError("unknown stream type %r" % (kind_val,))

    def stream_free(self, stream):
        free_stream(stream)

    def progress(self, stream=None):
        """One explicit progress pass (runtime.py:141-146): reclaims resources
        of completed stream operations; never blocks."""
        self._check_live()
        out = ctypes.c_int64()
        for c in list(self._comms):
            if getattr(c, "_h", None):
                check(lib.mpx_comm_progress(c._h, ctypes.byref(out)))

    def finalize(self):
        """Collective teardown; refuses while anything is outstanding."""
        self._check_live()
        pending = sum(c.outstanding() for c in self._comms if not c.freed)
        if pending:
            raise PendingError("%d operations still outstanding" % pending)
        self._barrier()
        for c in self._comms:
            if not c.freed and c is not self.world:
                c._release()
        self.world._release()
        check(lib.mpx_world_leave(self._world, self.rank))
        self._group.leave()
        self.finalized = True


def init(transport=None, rank=None, ranks=None, group=None, device=None,
         eager_limit=None, vci_pool=None, matching=None, **_ignored):
    """Bring up this rank (runtime.py:217-257).  transport must be "inproc"
    (the only in-scope transport: socket / multi-host bootstrap is out of
    scope)."""
    transport = _cfg(transport, "MINIMPI_TRANSPORT", TRANSPORT_INPROC, str).replace("-", "")
    if transport not in (TRANSPORT_INPROC, TRANSPORT_IPC):
        raise UnsupportedError("transport %r is out of scope for the B200 build" % transport)
    # where point-to-point messages are matched (csrc/dmatch.hpp): "host" at
    # enqueue time, or "device" when each rank's stream reaches the operation
    matching = _cfg(matching, "MINIMPI_MATCHING", MATCH_HOST, str)
    if matching not in (MATCH_HOST, MATCH_DEVICE):
        raise ArgError("matching must be %r or %r, got %r" % (MATCH_HOST, MATCH_DEVICE, matching))
    if matching == MATCH_DEVICE and transport == TRANSPORT_IPC:
        raise UnsupportedError("device matching is built for in-process worlds (transport 'inproc')")
    if transport == TRANSPORT_IPC:
        # one process per rank: torchrun's RANK / WORLD_SIZE / LOCAL_RANK unless given
        rank = _cfg(rank, "MINIMPI_RANK", int(os.environ.get("RANK", "0")), int)
        ranks = _cfg(ranks, "MINIMPI_SIZE", int(os.environ.get("WORLD_SIZE", "1")), int)
        group = _cfg(group, "MINIMPI_GROUP", "job%s%s" % (os.environ.get("MASTER_PORT", ""),
                                                         os.environ.get("TORCHELASTIC_RUN_ID", "")), str)
        if device is None and "LOCAL_RANK" in os.environ:
            device = int(os.environ["LOCAL_RANK"]) % max(1, torch.cuda.device_count())
    rank = _cfg(rank, "MINIMPI_RANK", 0, int)
    size = _cfg(ranks, "MINIMPI_SIZE", 1, int)
    group = _cfg(group, "MINIMPI_GROUP", "default", str)
    eager_limit = _cfg(eager_limit, "MINIMPI_EAGER_LIMIT", DEFAULT_EAGER_LIMIT, int)
    vci_pool = _cfg(vci_pool, "MINIMPI_VCI_POOL", DEFAULT_POOL_CAPACITY, int)
    if size < 1:
        raise ArgError("ranks must be >= 1, got %d" % size)
    if not 0 <= rank < size:
        raise ArgError("rank %d outside job of %d" % (rank, size))
    if eager_limit < 0:
        raise ArgError("eager_limit/chunk_size out of range")
    if device is None:
        ndev = torch.cuda.device_count()
        if ndev == 0:
            raise UnsupportedError("no CUDA device: the B200 build has no CPU data path")
        device = rank % ndev
    if isinstance(device, torch.device):
        device = device.index or 0
    arena = int(os.environ.get("MPX_IPC_ARENA", DEFAULT_IPC_ARENA))
    return Instance(rank, size, group, int(device), eager_limit, vci_pool, transport, arena, matching)
