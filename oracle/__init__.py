"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the datatype hot path.

This package is the *checker*, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import it.  The product package
(``paper_2402_12274_b200``) never imports anything from here and fails loudly
when its CUDA library is missing.

Contents
  * ``liboracle.so`` (built from ``dt_oracle.c``): a C restatement of
    ``/root/reference/pkg/src/minimpi/datatype.py`` (layout tree, merge
    builders, iov, pack/unpack, copy_between) and of the rank-ordered
    allreduce SUM in ``comm.py:582-588``.
  * ``brute.py``: an independent brute-force flattener restating
    ``/root/reference/pkg/tests/flatten_oracle.py`` (leaf enumeration plus
    adjacent merge) for small cross-checks.

Parity pin: ``tests/test_oracle_golden.py`` checks this oracle against
golden vectors produced by the real Python reference
(``tests/golden/make_golden.py``).

Type specs use the flatten_oracle tuple forms
(``flatten_oracle.py:8-16``) plus ``("indexed", bls, displs, child)``.
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "dt_oracle.c")

_KIND = {"basic": 0, "contiguous": 1, "vector": 2, "hvector": 3,
         "indexed_block": 4, "struct": 5, "subarray": 6, "resized": 7,
         "indexed": 8}


def build(force=False):
    """Compile dt_oracle.c -> liboracle.so with gcc (no GPU needed)."""
    if (not force and os.path.exists(_SO)
            and os.path.getmtime(_SO) >= os.path.getmtime(_SRC)):
        return _SO
    subprocess.check_call(["gcc", "-O2", "-g", "-fPIC", "-shared", "-std=c99",
                           "-Wall", "-o", _SO, _SRC])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        i64, p64 = ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)
        vp = ctypes.c_void_p
        L.orc_build.argtypes = [p64, i64]
        L.orc_build.restype = i64
        L.orc_info.argtypes = [i64, p64]
        L.orc_layout_info.argtypes = [i64, i64, p64]
        L.orc_iov_len.argtypes = [i64, i64, p64, p64]
        L.orc_iov.argtypes = [i64, i64, i64, i64, p64]
        L.orc_iov.restype = i64
        L.orc_pack.argtypes = [i64, i64, vp, i64, vp]
        L.orc_pack.restype = i64
        L.orc_unpack.argtypes = [i64, i64, vp, i64, vp, i64,
                                 ctypes.POINTER(ctypes.c_int)]
        L.orc_unpack.restype = i64
        L.orc_copy_between.argtypes = [i64, i64, vp, i64, i64, i64, vp, i64]
        L.orc_copy_between.restype = i64
        L.orc_reset.argtypes = []
        _lib = L
    return _lib


def encode(spec):
    """Tuple spec -> flat int64 prefix program understood by orc_build."""
    out = []

    def enc(t):
        kind = t[0]
        out.append(_KIND[kind])
        if kind == "basic":
            out.append(t[1])
        elif kind == "contiguous":
            out.append(t[1]); enc(t[2])
        elif kind in ("vector", "hvector"):
            out.extend([t[1], t[2], t[3]]); enc(t[4])
        elif kind == "indexed_block":
            out.extend([t[1], len(t[2])]); out.extend(t[2]); enc(t[3])
        elif kind == "struct":
            out.append(len(t[1])); out.extend(t[1]); out.extend(t[2])
            for c in t[3]:
                enc(c)
        elif kind == "subarray":
            out.append(len(t[1])); out.extend(t[1]); out.extend(t[2])
            out.extend(t[3]); enc(t[4])
        elif kind == "resized":
            out.extend([t[1], t[2]]); enc(t[3])
        elif kind == "indexed":
            out.append(len(t[1])); out.extend(t[1]); out.extend(t[2]); enc(t[3])
        else:
            raise ValueError(kind)

    enc(spec)
    return out


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleType:
    """A committed reference-semantics datatype living in the C oracle."""

    def __init__(self, spec):
        prog = np.asarray(encode(spec), dtype=np.int64)
        L = lib()
        h = L.orc_build(prog.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                        len(prog))
        if h < 0:
            raise ValueError("oracle could not build spec %r" % (spec,))
        self.h = h
        info = (ctypes.c_int64 * 8)()
        L.orc_info(h, info)
        (self.size_bytes, self.lb, self.ub, self.extent_bytes,
         self.segment_count, self.node_count, self.min_off,
         self.max_end) = list(info)

    def layout_info(self, count=1):
        out = (ctypes.c_int64 * 5)()
        if lib().orc_layout_info(self.h, count, out) != 0:
            raise ValueError("bad count")
        return dict(runs=out[0], nbytes=out[1], min_off=out[2],
                    max_end=out[3], node_count=out[4])

    def iov_len(self, max_bytes=-1):
        n = ctypes.c_int64()
        b = ctypes.c_int64()
        if lib().orc_iov_len(self.h, max_bytes, ctypes.byref(n),
                             ctypes.byref(b)) != 0:
            raise ValueError("bad max_bytes")
        return n.value, b.value

    def iov(self, offset=0, maxlen=-1, count=1):
        """(n, 2) int64 array of (base_offset, length)."""
        runs = self.layout_info(count)["runs"]
        n = runs - offset
        if maxlen != -1:
            n = min(n, maxlen)
        n = max(n, 0)
        out = np.empty((n, 2), dtype=np.int64)
        got = lib().orc_iov(self.h, count, offset, maxlen,
                            out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
        if got < 0:
            raise ValueError("bad iov arguments")
        return out[:got]

    def pack(self, buf, count=1):
        src = np.frombuffer(buf, dtype=np.uint8) if not isinstance(
            buf, np.ndarray) else buf.view(np.uint8).reshape(-1)
        nbytes = self.layout_info(count)["nbytes"]
        out = np.empty(nbytes, dtype=np.uint8)
        got = lib().orc_pack(self.h, count, _ptr(src), src.size, _ptr(out))
        if got < 0:
            raise ValueError("buffer too small / layout out of bounds")
        return out

    def unpack(self, data, dst, count=1):
        """Scatter data into dst (a writable uint8 ndarray).  Returns
        (bytes_written, truncated)."""
        d = np.frombuffer(data, dtype=np.uint8) if not isinstance(
            data, np.ndarray) else data.view(np.uint8).reshape(-1)
        tr = ctypes.c_int()
        got = lib().orc_unpack(self.h, count, _ptr(d), d.size, _ptr(dst),
                               dst.size, ctypes.byref(tr))
        if got < 0:
            raise ValueError("buffer too small / layout out of bounds")
        return got, bool(tr.value)


def copy_between(src_t, src_count, src, dst_t, dst_count, dst):
    """Zipper transfer (datatype.py:760-797); dst_t None = plain bytes."""
    got = lib().orc_copy_between(
        src_t.h, src_count, _ptr(src), src.size,
        -1 if dst_t is None else dst_t.h, dst_count, _ptr(dst), dst.size)
    if got < 0:
        raise ValueError("bad copy_between arguments")
    return got


def reset():
    """Drop every oracle type (frees the node arena)."""
    lib().orc_reset()


def allreduce_sum(bufs):
    """Rank-ordered SUM (comm.py:582-588): x0 + x1 + ... in int64 or
    float64.  float32 inputs are upcast to float64 (the reference has no
    float32 allreduce)."""
    acc = np.array(bufs[0], copy=True)
    if acc.dtype == np.float32:
        acc = acc.astype(np.float64)
    for b in bufs[1:]:
        acc = acc + (b.astype(np.float64) if b.dtype == np.float32 else b)
    return acc
