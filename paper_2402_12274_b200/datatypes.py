"""Derived datatypes, iov queries and pack/unpack -- the reference's
``minimpi.datatype`` surface (/root/reference/pkg/src/minimpi/datatype.py)
backed by libmpx.so.

Layout trees are compiled and lowered in C++ (csrc/typerep.cpp, plan.cpp);
iov enumeration, pack and unpack run as sm_100a kernels (csrc/kernels.cu).

Buffers:
  * CUDA tensors (any dtype, C-contiguous) are used in place; work is enqueued
    on the tensor device's current torch stream and results are CUDA uint8
    tensors.
  * Host buffer-protocol objects (bytes, bytearray, numpy, array.array, CPU
    tensors) keep the reference contract (``pack`` returns ``bytes``,
    ``unpack`` writes the host buffer): they are staged through the current
    CUDA device.  There is no CPU implementation of the data movement.
"""

import ctypes
import warnings
from typing import NamedTuple

import numpy as np
import torch

from . import _lib
from ._lib import check, lib, i64_array
from .errors import ArgError, TruncateError


class IovSegment(NamedTuple):
    """One maximal contiguous byte run (datatype.py:28-32)."""

    base_offset: int
    length: int


def _is_int(v):
    return isinstance(v, int) and not isinstance(v, bool)


def _count(n, what):
    # _check_count, datatype.py:434-436
    if not _is_int(n) or n < 0:
        raise ArgError("%s must be an integer >= 0" % what)
    return n


def _anyint(v, msg):
    if not _is_int(v):
        raise ArgError(msg)
    return v


class Datatype:
    """Handle to a C++ datatype (datatype.py:345-407)."""

    __slots__ = ("_h", "_builtin_name", "__weakref__")

    def __init__(self, handle, builtin_name=None):
        self._h = handle
        self._builtin_name = builtin_name

    def _info(self):
        out = (ctypes.c_int64 * 8)()
        check(lib.mpx_type_get_info(self._h, out))
        return out

    @property
    def size_bytes(self):
        return self._info()[0]

    @property
    def lb(self):
        return self._info()[1]

    @property
    def ub(self):
        return self._info()[2]

    @property
    def extent_bytes(self):
        return self._info()[3]

    @property
    def segment_count(self):
        return self._info()[4]

    @property
    def node_count(self):
        return self._info()[5]

    @property
    def committed(self):
        i = self._info()
        return bool(i[6]) and not i[7]

    def __repr__(self):
        i = self._info()
        return "<Datatype %s size=%d extent=%d segments=%d>" % (
            self._builtin_name or "derived", i[0], i[3], i[4])

    def commit(self):
        return type_commit(self)

    def free(self):
        type_free(self)

    def iov_len(self, max_iov_bytes=-1):
        return type_iov_len(self, max_iov_bytes)

    def iov(self, iov_offset=0, max_iov_len=-1):
        return type_iov(self, iov_offset, max_iov_len)

    def layout_query(self, count=1):
        """Host-side lowering summary (runs, nbytes, min_off, max_end,
        node_count, plan kind (0 empty, 1 chain, 2 descriptor walk, 3 span,
        4 run table), overlap, and chain alignment -- or, for span plans,
        the number of word-gather specs (0: k_span fallback))."""
        out = (ctypes.c_int64 * 8)()
        check(lib.mpx_layout_query(self._h, count, out))
        keys = ("runs", "nbytes", "min_off", "max_end", "node_count", "plan",
                "overlap", "chain_align")
        return dict(zip(keys, list(out)))


def _builtin(which, name):
    h = ctypes.c_void_p()
    check(lib.mpx_type_builtin(which, ctypes.byref(h)))
    return Datatype(h.value, name)


BYTE = _builtin(0, "byte")
CHAR = _builtin(1, "char")
INT8 = _builtin(2, "int8")
INT32 = _builtin(3, "int32")
INT64 = _builtin(4, "int64")
FLOAT32 = _builtin(5, "float32")
FLOAT64 = _builtin(6, "float64")
BUILTINS = (BYTE, CHAR, INT8, INT32, INT64, FLOAT32, FLOAT64)


def _child(c):
    if not isinstance(c, Datatype):
        raise ArgError("child must be a Datatype")
    return c._h


def _new(fn, *args):
    h = ctypes.c_void_p()
    check(fn(*args, ctypes.byref(h)))
    return Datatype(h.value)


# ---------------------------------------------------------------- constructors


def type_contiguous(count, child):
    """datatype.py:444-455"""
    return _new(lib.mpx_type_contiguous, _count(count, "count"), _child(child))


def type_vector(count, blocklength, stride_elems, child):
    """datatype.py:458-475"""
    _count(count, "count")
    _count(blocklength, "blocklength")
    _anyint(stride_elems, "stride must be an integer")
    return _new(lib.mpx_type_vector, count, blocklength, stride_elems, _child(child))


def type_hvector(count, blocklength, stride_bytes, child):
    """datatype.py:478-495"""
    _count(count, "count")
    _count(blocklength, "blocklength")
    _anyint(stride_bytes, "stride must be an integer")
    return _new(lib.mpx_type_hvector, count, blocklength, stride_bytes, _child(child))


def type_indexed_block(blocklength, displacements, child):
    """datatype.py:498-516"""
    _count(blocklength, "blocklength")
    ds = [_anyint(d, "displacements must be integers") for d in displacements]
    return _new(lib.mpx_type_indexed_block, blocklength, len(ds), i64_array(ds),
                _child(child))


def type_indexed(blocklengths, displacements, child):
    """MPI_Type_indexed: variable block lengths, displacements in child
    extents.  Absent from the reference; semantics equal
    type_create_struct(bls, [d * extent], [child] * n)."""
    bls = [_count(b, "blocklength") for b in blocklengths]
    ds = [_anyint(d, "displacements must be integers") for d in displacements]
    if len(bls) != len(ds):
        raise ArgError("indexed arrays must have equal length")
    return _new(lib.mpx_type_indexed, len(bls), i64_array(bls), i64_array(ds),
                _child(child))


def type_create_struct(blocklengths, byte_displacements, children):
    """datatype.py:519-547"""
    bls, ds, kids = list(blocklengths), list(byte_displacements), list(children)
    if not (len(bls) == len(ds) == len(kids)):
        raise ArgError("struct arrays must have equal length")
    for b in bls:
        _count(b, "blocklength")
    for d in ds:
        _anyint(d, "byte displacements must be integers")
    hs = (ctypes.c_void_p * max(1, len(kids)))(*[_child(k) for k in kids])
    return _new(lib.mpx_type_create_struct, len(bls), i64_array(bls), i64_array(ds), hs)


def type_create_subarray(full_sizes, sub_sizes, sub_offsets, child):
    """C-order subarray, datatype.py:550-583"""
    full, sub, offs = list(full_sizes), list(sub_sizes), list(sub_offsets)
    if not full or not (len(full) == len(sub) == len(offs)):
        raise ArgError("subarray dimension arrays must match and be non-empty")
    for f, s, o in zip(full, sub, offs):
        _count(f, "full size")
        _count(s, "sub size")
        _count(o, "offset")
    return _new(lib.mpx_type_create_subarray, len(full), i64_array(full),
                i64_array(sub), i64_array(offs), _child(child))


def type_create_resized(child, lb, extent):
    """datatype.py:586-591"""
    if not _is_int(lb) or not _is_int(extent) or extent < 0:
        raise ArgError("resized needs integer lb and extent >= 0")
    return _new(lib.mpx_type_create_resized, _child(child), lb, extent)


def type_commit(d):
    """datatype.py:594-600"""
    if not isinstance(d, Datatype):
        raise ArgError("type_commit expects a Datatype")
    check(lib.mpx_type_commit(d._h))
    return d


def type_free(d):
    """datatype.py:603-610"""
    if not isinstance(d, Datatype):
        raise ArgError("type_free expects a Datatype")
    check(lib.mpx_type_free(d._h))


# ---------------------------------------------------------------- queries


def type_iov_len(d, max_iov_bytes=-1):
    """(whole leading segments within the budget, their bytes); datatype.py:618-628"""
    if not isinstance(d, Datatype):
        raise ArgError("expected a Datatype")
    if not _is_int(max_iov_bytes):
        raise ArgError("max_iov_bytes must be an integer >= -1")
    n = ctypes.c_int64()
    b = ctypes.c_int64()
    check(lib.mpx_type_iov_len(d._h, max_iov_bytes, ctypes.byref(n), ctypes.byref(b)))
    return n.value, b.value


def _stream_ptr(device):
    return torch.cuda.current_stream(device).cuda_stream


def type_iov_tensor(d, iov_offset=0, max_iov_len=-1, count=1, device=None):
    """Device-resident iov: a (n, 2) int64 CUDA tensor of (base_offset,
    length) for segments [iov_offset, iov_offset + max_iov_len) of the
    layout replicated ``count`` times.  Enqueued on the current stream."""
    if not isinstance(d, Datatype):
        raise ArgError("expected a Datatype")
    for v, what in ((iov_offset, "iov_offset"), (max_iov_len, "max_iov_len"), (count, "count")):
        if not _is_int(v):
            raise ArgError("%s must be an integer" % what)
    q = d.layout_query(count)     # validates usability / count
    total = q["runs"]
    n = total - iov_offset if 0 <= iov_offset <= total else 0
    if max_iov_len >= 0:
        n = min(n, max_iov_len)
    dev = torch.device("cuda", torch.cuda.current_device() if device is None
                       else torch.device(device).index or 0)
    out = torch.empty((max(n, 1), 2), dtype=torch.int64, device=dev)
    got = ctypes.c_int64()
    check(lib.mpx_type_iov(d._h, count, iov_offset, max_iov_len, out.data_ptr(),
                           max(n, 0), ctypes.byref(got), _stream_ptr(dev)))
    return out[:got.value]


def type_iov(d, iov_offset=0, max_iov_len=-1):
    """(segments[iov_offset : iov_offset + max_iov_len], count); datatype.py:631-650.
    Enumerated on the GPU, returned as a list of IovSegment."""
    t = type_iov_tensor(d, iov_offset, max_iov_len)
    rows = t.cpu().tolist()
    return [IovSegment(o, l) for o, l in rows], len(rows)


def packed_size(d, count=1):
    """datatype.py:731-734"""
    out = ctypes.c_int64()
    check(lib.mpx_packed_size(d._h, _count(count, "count"), ctypes.byref(out)))
    return out.value


# ---------------------------------------------------------------- buffers


def _cuda_tensor(obj):
    if isinstance(obj, torch.Tensor) and obj.is_cuda:
        if not obj.is_contiguous():
            raise ArgError("buffer must be C-contiguous")
        return obj
    return None


def _gpu_visible(obj):
    """CUDA tensor, or pinned CPU tensor (kernels address it zero-copy)."""
    t = _cuda_tensor(obj)
    if t is not None:
        return t
    if isinstance(obj, torch.Tensor) and obj.is_pinned():
        if not obj.is_contiguous():
            raise ArgError("buffer must be C-contiguous")
        return obj
    return None


def _exec_device(*tensors):
    for t in tensors:
        if t is not None and t.is_cuda:
            return t.device
    return _default_device()


def _host_view(buf, writable):
    """Reference as_byte_view (datatype.py:664-677), plus CPU tensors."""
    if isinstance(buf, torch.Tensor):
        if not buf.is_contiguous():
            raise ArgError("buffer must be C-contiguous")
        buf = buf.view(torch.uint8).numpy() if buf.numel() else np.empty(0, np.uint8)
    try:
        mv = memoryview(buf)
    except TypeError:
        raise ArgError("object of type %s is not a buffer" % type(buf).__name__)
    if writable and mv.readonly:
        raise ArgError("buffer is read-only but a writable one is required")
    if mv.format != "B" or mv.ndim != 1:
        try:
            mv = mv.cast("B")
        except TypeError:
            raise ArgError("buffer must be C-contiguous")
    return mv


def _nbytes(t):
    return t.numel() * t.element_size()


def _upload(view, device):
    n = len(view)
    if n == 0:
        return torch.empty(1, dtype=torch.uint8, device=device)[:0]
    arr = np.frombuffer(view, dtype=np.uint8)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        host = torch.from_numpy(arr)
    return host.to(device)


def _to_cuda_bytes(obj, device, writable=False):
    t = _cuda_tensor(obj)
    if t is not None:
        return t
    if isinstance(obj, torch.Tensor) and obj.is_pinned():
        if not obj.is_contiguous():
            raise ArgError("buffer must be C-contiguous")
        return obj.view(torch.uint8).reshape(-1).to(device, non_blocking=True)
    return _upload(_host_view(obj, writable), device)


def _default_device():
    return torch.device("cuda", torch.cuda.current_device())


# ---------------------------------------------------------------- pack


def pack_into(d, buf, out, count=1):
    """Pack ``buf`` (CUDA tensor) into the CUDA tensor ``out`` (>= packed
    size bytes); asynchronous on the current stream of buf's device.
    Returns the number of packed bytes."""
    if not isinstance(d, Datatype):
        raise ArgError("expected a Datatype")
    src = _cuda_tensor(buf)
    dst = _cuda_tensor(out)
    if src is None or dst is None:
        raise ArgError("pack_into needs CUDA tensors")
    _count(count, "count")
    check(lib.mpx_pack(d._h, count, src.data_ptr(), _nbytes(src), dst.data_ptr(),
                       _nbytes(dst), _stream_ptr(src.device)))
    return packed_size(d, count)


def pack(d, buf, count=1):
    """Gather the layout's bytes in traversal order (datatype.py:695-702).

    CUDA tensor in -> CUDA uint8 tensor out (asynchronous).  Host buffer in
    -> ``bytes`` out (staged through the GPU, synchronous)."""
    if not isinstance(d, Datatype):
        raise ArgError("expected a Datatype")
    _count(count, "count")
    src = _gpu_visible(buf)
    if src is not None:
        n = packed_size(d, count)
        if src.is_cuda:
            out = torch.empty(max(n, 1), dtype=torch.uint8, device=src.device)[:n]
        else:
            out = torch.empty(max(n, 1), dtype=torch.uint8, pin_memory=True)[:n]
        dev = _exec_device(src)
        check(lib.mpx_pack(d._h, count, src.data_ptr(), _nbytes(src),
                           out.data_ptr() if n else src.data_ptr(), n, _stream_ptr(dev)))
        if not src.is_cuda:          # host-facing result: complete before returning
            torch.cuda.current_stream(dev).synchronize()
        return out
    # reference contract for host buffers: validate like _checked_view first
    view = _host_view(buf, writable=False)
    n = packed_size(d, count)
    q = d.layout_query(count)
    if q["runs"]:
        if q["min_off"] < 0:
            raise ArgError("layout reaches before the start of the buffer")
        if q["max_end"] > len(view):
            raise ArgError("buffer too small: layout spans %d bytes, buffer has %d"
                           % (q["max_end"], len(view)))
    if n == 0:
        return b""
    dev = _default_device()
    dsrc = _upload(view, dev)
    out = torch.empty(n, dtype=torch.uint8, device=dev)
    check(lib.mpx_pack(d._h, count, dsrc.data_ptr(), _nbytes(dsrc), out.data_ptr(), n,
                       _stream_ptr(dev)))
    return out.cpu().numpy().tobytes()


def unpack(d, data, buf, count=1):
    """Scatter packed bytes into ``buf`` (datatype.py:705-728); returns
    bytes written.  Last writer wins on overlapping layouts; short data
    writes a prefix; excess data writes the full layout and then raises
    TruncateError."""
    if not isinstance(d, Datatype):
        raise ArgError("expected a Datatype")
    _count(count, "count")
    dst = _gpu_visible(buf)
    written = ctypes.c_int64()
    if dst is not None:
        src = _gpu_visible(data)
        dev = _exec_device(dst, src)
        if src is None:
            src = _to_cuda_bytes(data, dev)
        rc = lib.mpx_unpack(d._h, count, src.data_ptr(), _nbytes(src), dst.data_ptr(),
                            _nbytes(dst), ctypes.byref(written), _stream_ptr(dev))
        if not dst.is_cuda:
            torch.cuda.current_stream(dev).synchronize()
        if rc and rc != 4:
            check(rc)
        if rc == 4:
            raise TruncateError("%d bytes offered but layout holds %d"
                                % (_nbytes(src), packed_size(d, count)))
        return written.value
    # host destination: stage the whole buffer through the GPU and write back
    view = _host_view(buf, writable=True)
    dev = _default_device()
    src = _to_cuda_bytes(data, dev)
    q = d.layout_query(count)
    if q["runs"]:
        if q["min_off"] < 0:
            raise ArgError("layout reaches before the start of the buffer")
        if q["max_end"] > len(view):
            raise ArgError("buffer too small: layout spans %d bytes, buffer has %d"
                           % (q["max_end"], len(view)))
    ddst = _upload(view, dev) if len(view) else torch.empty(1, dtype=torch.uint8, device=dev)
    rc = lib.mpx_unpack(d._h, count, src.data_ptr(), _nbytes(src), ddst.data_ptr(),
                        len(view), ctypes.byref(written), _stream_ptr(dev))
    if rc and rc != 4:
        check(rc)
    if len(view):
        view[:] = ddst.cpu().numpy().tobytes()
    if rc == 4:
        raise TruncateError("%d bytes offered but layout holds %d"
                            % (_nbytes(src), packed_size(d, count)))
    return written.value


def _multi(fn, dts, counts, srcs, dsts):
    n = len(dts)
    if not (len(counts) == len(srcs) == len(dsts) == n):
        raise ArgError("multi arrays must have equal length")
    hs = (ctypes.c_void_p * max(1, n))(*[_child(d) for d in dts])
    sp = (ctypes.c_void_p * max(1, n))(*[s.data_ptr() for s in srcs])
    dp = (ctypes.c_void_p * max(1, n))(*[t.data_ptr() for t in dsts])
    sb = i64_array([_nbytes(s) for s in srcs])
    db = i64_array([_nbytes(t) for t in dsts])
    cs = i64_array(counts)
    for t in list(srcs) + list(dsts):
        if _gpu_visible(t) is None:
            raise ArgError("multi operations need CUDA or pinned CPU tensors")
    stream = _stream_ptr(_exec_device(*srcs, *dsts)) if n else 0
    return fn(n, hs, cs, sp, sb, dp, db, stream)


def pack_multi(dts, bufs, outs, counts=None):
    """Fused pack of several (datatype, buffer) pairs into their outputs --
    one launch for up to 16 strided layouts (e.g. six halo faces).  Buffers
    are CUDA tensors or pinned CPU tensors (zero-copy over PCIe).
    Asynchronous on the current stream.  B200 extension of pack()."""
    counts = counts or [1] * len(dts)
    check(_multi(lib.mpx_pack_multi, dts, counts, bufs, outs))


def unpack_multi(dts, datas, bufs, counts=None):
    """Fused unpack counterpart of pack_multi.  The unpacks run concurrently:
    destinations of different layouts must be disjoint or agree where they
    overlap (include/mpx.h); overlaps within one layout are last-writer-wins
    as in unpack."""
    counts = counts or [1] * len(dts)
    check(_multi(lib.mpx_unpack_multi, dts, counts, datas, bufs))


def check_region(d, buf, count=1, writable=False):
    """Validate that buf covers d's layout replicated count times
    (datatype.py:737-740)."""
    _count(count, "count")
    t = _cuda_tensor(buf)
    size = _nbytes(t) if t is not None else len(_host_view(buf, writable))
    q = d.layout_query(count)
    if q["runs"]:
        if q["min_off"] < 0:
            raise ArgError("layout reaches before the start of the buffer")
        if q["max_end"] > size:
            raise ArgError("buffer too small: layout spans %d bytes, buffer has %d"
                           % (q["max_end"], size))


def set_l2_fetch_granularity(nbytes, device=None):
    """Set cudaLimitMaxL2FetchGranularity (bytes) on a device; returns the
    previous value.  nbytes = -1 only queries."""
    dev = torch.cuda.current_device() if device is None else torch.device(device).index or 0
    prev = ctypes.c_int()
    check(lib.mpx_device_set_l2_fetch(dev, nbytes, ctypes.byref(prev)))
    return prev.value


# ------------------------------------------------------- type expressions

_EXPR = {
    "byte": BYTE, "char": CHAR, "int8": INT8, "int32": INT32, "int64": INT64,
    "float32": FLOAT32, "float64": FLOAT64,
    "contiguous": lambda *a: type_contiguous(*a).commit(),
    "vector": lambda *a: type_vector(*a).commit(),
    "hvector": lambda *a: type_hvector(*a).commit(),
    "indexed_block": lambda *a: type_indexed_block(*a).commit(),
    "indexed": lambda *a: type_indexed(*a).commit(),
    "struct": lambda *a: type_create_struct(*a).commit(),
    "subarray": lambda *a: type_create_subarray(*a).commit(),
    "resized": lambda *a: type_create_resized(*a).commit(),
}


def parse_type_expr(text):
    """Constructor expression -> committed Datatype (datatype.py:818-831)."""
    try:
        value = eval(text, {"__builtins__": {}}, dict(_EXPR))  # noqa: S307 (no builtins)
    except ArgError:
        raise
    except Exception as exc:
        raise ArgError("bad type expression: %s" % exc) from exc
    if not isinstance(value, Datatype):
        raise ArgError("expression did not produce a datatype")
    return value
