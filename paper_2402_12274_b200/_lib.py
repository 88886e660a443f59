"""ctypes binding of libmpx.so (the C ABI declared in include/mpx.h).

The product has no CPU fallback: if libmpx.so is missing or fails to load,
importing the package raises immediately.  Build it with
``python paper_2402_12274_b200/build.py``.
"""

import ctypes
import os

from .errors import error_for_code

_HERE = os.path.dirname(os.path.abspath(__file__))
# MPX_LIB_PATH: an A/B build of the same sources (experiments only)
SO_PATH = os.environ.get("MPX_LIB_PATH") or os.path.join(_HERE, "libmpx.so")

if not os.path.exists(SO_PATH):
    raise ImportError(
        "libmpx.so not found at %s -- build it with "
        "`python paper_2402_12274_b200/build.py` (no CPU fallback exists)" % SO_PATH)

# torch first: it loads the CUDA runtime / NCCL this library talks to
import torch  # noqa: E402,F401

lib = ctypes.CDLL(SO_PATH, mode=ctypes.RTLD_GLOBAL)

i64 = ctypes.c_int64
p64 = ctypes.POINTER(ctypes.c_int64)
vp = ctypes.c_void_p
pvp = ctypes.POINTER(ctypes.c_void_p)
cint = ctypes.c_int
dt_t = ctypes.c_void_p
pdt = ctypes.POINTER(ctypes.c_void_p)

_SIGS = {
    "mpx_abi_version": ([], cint),
    "mpx_last_error": ([], ctypes.c_char_p),
    "mpx_device_set_l2_fetch": ([cint, cint, ctypes.POINTER(cint)], cint),
    "mpx_type_builtin": ([cint, pdt], cint),
    "mpx_type_contiguous": ([i64, dt_t, pdt], cint),
    "mpx_type_vector": ([i64, i64, i64, dt_t, pdt], cint),
    "mpx_type_hvector": ([i64, i64, i64, dt_t, pdt], cint),
    "mpx_type_indexed_block": ([i64, i64, p64, dt_t, pdt], cint),
    "mpx_type_indexed": ([i64, p64, p64, dt_t, pdt], cint),
    "mpx_type_create_struct": ([i64, p64, p64, pdt, pdt], cint),
    "mpx_type_create_subarray": ([cint, p64, p64, p64, dt_t, pdt], cint),
    "mpx_type_create_resized": ([dt_t, i64, i64, pdt], cint),
    "mpx_type_commit": ([dt_t], cint),
    "mpx_type_free": ([dt_t], cint),
    "mpx_type_get_info": ([dt_t, p64], cint),
    "mpx_type_iov_len": ([dt_t, i64, p64, p64], cint),
    "mpx_type_iov": ([dt_t, i64, i64, i64, vp, i64, p64, vp], cint),
    "mpx_packed_size": ([dt_t, i64, p64], cint),
    "mpx_layout_query": ([dt_t, i64, p64], cint),
    "mpx_plan_dump": ([dt_t, i64, p64, i64, p64], cint),
    "mpx_pack": ([dt_t, i64, vp, i64, vp, i64, vp], cint),
    "mpx_unpack": ([dt_t, i64, vp, i64, vp, i64, p64, vp], cint),
    "mpx_pack_multi": ([cint, pdt, p64, pvp, p64, pvp, p64, vp], cint),
    "mpx_unpack_multi": ([cint, pdt, p64, pvp, p64, pvp, p64, vp], cint),
    "mpx_stream_order": ([vp, vp], cint),
    "mpx_comm_set_host_wait": ([vp, cint], cint),
    "mpx_comm_throttle_wait": ([vp], cint),
    "mpx_stream_release": ([vp], cint),
    "mpx_world_join": ([ctypes.c_char_p, cint, cint, cint, i64, pvp], cint),
    "mpx_world_leave": ([vp, cint], cint),
    "mpx_comm_create": ([vp, cint, cint, vp, pvp], cint),
    "mpx_comm_free": ([vp], cint),
    "mpx_send_enqueue": ([vp, vp, i64, i64, dt_t, cint, cint], cint),
    "mpx_recv_enqueue": ([vp, vp, i64, i64, dt_t, cint, cint], cint),
    "mpx_isend_enqueue": ([vp, vp, i64, i64, dt_t, cint, cint, pvp], cint),
    "mpx_irecv_enqueue": ([vp, vp, i64, i64, dt_t, cint, cint, pvp], cint),
    "mpx_wait_enqueue": ([vp], cint),
    "mpx_waitall_enqueue": ([cint, pvp], cint),
    "mpx_request_status": ([vp, p64], cint),
    "mpx_request_free": ([vp], cint),
    "mpx_allreduce_enqueue": ([vp, vp, vp, i64, cint, cint, cint], cint),
    "mpx_comm_synchronize": ([vp], cint),
    "mpx_comm_progress": ([vp, p64], cint),
    "mpx_stream_device": ([vp, ctypes.POINTER(cint)], cint),
    "mpx_stream_new": ([cint, pvp], cint),
    "mpx_ipc_world_join": ([ctypes.c_char_p, cint, cint, cint, i64, i64, pvp], cint),
    "mpx_world_barrier": ([vp], cint),
    "mpx_world_set_matching": ([vp, cint], cint),
    "mpx_stream_wait": ([vp], cint),
    "mpx_debug_flags": ([], cint),
    "mpx_nccl_load": ([ctypes.c_char_p], cint),
    "mpx_win_create": ([vp, vp, i64, i64, p64], cint),
    "mpx_win_info": ([vp, i64, cint, p64], cint),
    "mpx_win_get": ([vp, i64, vp, i64, i64, dt_t, cint, i64, i64, dt_t], cint),
    "mpx_win_free": ([vp, i64], cint),
}

for _name, (_args, _res) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res

# The enqueue calls that never wait on the host (in-process worlds, whose
# communicators return MPX_WOULD_BLOCK instead of throttling, see
# mpx_comm_set_host_wait) are also bound through ctypes.PyDLL: the GIL stays
# held across them.  Releasing and re-taking it around every short call costs
# a thread hand-off per call when several rank threads of one process are
# busy (measured: ~8 us each, 2-rank 8-byte ring 68 -> 40 us/iteration).
# MPX_GIL_FASTPATH=0 turns this off.
WOULD_BLOCK = 9
FAST_CALLS = ("mpx_send_enqueue", "mpx_recv_enqueue", "mpx_isend_enqueue", "mpx_irecv_enqueue",
              "mpx_wait_enqueue", "mpx_waitall_enqueue", "mpx_stream_order", "mpx_request_status",
              "mpx_request_free")
GIL_FASTPATH = os.environ.get("MPX_GIL_FASTPATH", "1") != "0"
fast = ctypes.PyDLL(SO_PATH, mode=ctypes.RTLD_GLOBAL) if GIL_FASTPATH else lib
if GIL_FASTPATH:
    for _name in FAST_CALLS:
        _args, _res = _SIGS[_name]
        _f = getattr(fast, _name)
        _f.argtypes = _args
        _f.restype = _res


def last_error():
    m = lib.mpx_last_error()
    return m.decode(errors="replace") if m else ""


def check(rc):
    """Raise the MinimpiError subclass matching a nonzero MPX_* code."""
    if rc:
        raise error_for_code(rc, last_error())
    return rc


def own_stream(device):
    """A dedicated CUDA stream (cudaStreamCreateWithFlags, non-blocking) for
    one rank-side owner: a queue, a communicator or a serial context.  Never
    one of torch's pooled streams -- torch hands its 32 out round-robin, so
    two ranks can end up on the SAME stream and one rank's stream-memop wait
    then parks the other rank's flag write behind it (tools/diag_alias.py).
    The stream is never destroyed (the C side may still order work on it
    after the Python owner is gone); owners that end explicitly and drained
    hand it back with release_stream, so a later owner reuses it."""
    import torch
    dev = torch.device(device)
    h = ctypes.c_void_p()
    check(lib.mpx_stream_new(dev.index if dev.index is not None else torch.cuda.current_device(),
                             ctypes.byref(h)))
    return torch.cuda.ExternalStream(h.value, device=dev)


def release_stream(ts):
    """Drain a stream from own_stream and give it back to libmpx's pool (the
    owner is done with it): streams per device stay those of live owners."""
    check(lib.mpx_stream_wait(ts.cuda_stream))
    check(lib.mpx_stream_release(ts.cuda_stream))


def stream_wait(ts):
    """Host-wait for a torch stream through libmpx's polling wait (see
    mpx_stream_wait); the GIL is released while waiting."""
    check(lib.mpx_stream_wait(ts.cuda_stream))


def exported_symbols():
    """Names of every function this binding declares (test helper)."""
    return sorted(_SIGS)


def i64_array(values):
    vals = list(values)
    return (ctypes.c_int64 * max(1, len(vals)))(*vals)
