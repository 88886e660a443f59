"""paper_2402_12274_b200 -- B200-native MPIX datatype / enqueue hot path.

A drop-in for the data path of the reference package ``minimpi``
(/root/reference/pkg/src/minimpi/__init__.py:13-63): the same flat API names
for derived datatypes, iov queries, pack/unpack, CUDA-stream communicators and
the enqueue operations, executed by hand-written sm_100a kernels in
libmpx.so (C ABI: include/mpx.h).  Buffers are PyTorch CUDA tensors (host
buffers are accepted and staged through the GPU).

Passive-target read windows (``win_create`` / ``win_get``, onesided.py) read
peer device memory directly with the same datatype kernels.

Out of scope: socket transport and launcher,
thread communicators, stream-multiplex communicators, generalized requests,
VCI lock studies, the message-rate benchmarks.
"""

import os as _os

# Stream communicators order ranks' streams with stream memory operations;
# give every stream its own hardware queue so a waiting stream never blocks
# an unrelated one (takes effect if set before the CUDA context exists).
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# Lazy module loading makes the first launch of any kernel wait behind a
# stream parked in a stream-memop wait -- even on other streams (measured with
# tools/diag_memop.py).  libmpx force-loads its own kernels at world join;
# eager loading covers the caller's kernels too.
_os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

from .errors import (  # noqa: F401,E402
    MinimpiError, StateError, PendingError, ArgError, TransportError,
    SpawnError, ExhaustedError, UnsupportedError, TruncateError,
)
from .datatypes import (  # noqa: F401,E402
    Datatype, IovSegment,
    BYTE, CHAR, INT8, INT32, INT64, FLOAT32, FLOAT64,
    type_contiguous, type_vector, type_hvector, type_indexed_block,
    type_indexed, type_create_struct, type_create_subarray,
    type_create_resized, type_commit, type_free, type_iov_len, type_iov,
    type_iov_tensor, pack, pack_into, unpack, pack_multi, unpack_multi,
    packed_size, check_region, parse_type_expr, set_l2_fetch_granularity,
)
from .runtime import (  # noqa: F401,E402
    Instance, init, Info, info_create, info_set, info_set_hex,
    Stream, NULL_STREAM, SERIAL_CONTEXT, DEVICE_QUEUE, CUDA_STREAM,
    free_stream, TRANSPORT_INPROC,
)
from .queues import (  # noqa: F401,E402
    DeviceQueue, queue_create, queue_destroy, queue_synchronize,
    queue_from_hex, memcpy_enqueue, compute_enqueue, saxpy,
)
from .comms import (  # noqa: F401,E402
    Communicator, StreamComm, Status, Request, EnqueuedRequest,
    CONVENTIONAL, STREAM_SINGLE, SUM,
    stream_comm_create, comm_free, comm_get_stream, barrier, allreduce,
    allreduce_enqueue,
    send, recv, isend, irecv, wait, test, waitall,
    send_enqueue, recv_enqueue, isend_enqueue, irecv_enqueue,
    wait_enqueue, waitall_enqueue,
)

from .onesided import (  # noqa: F401,E402
    Window, LOCK_SHARED, LOCK_EXCLUSIVE,
    win_create, win_lock, win_unlock, win_get, win_free,
)

ANY_SOURCE = -1
ANY_TAG = -1

__version__ = "0.1.0"
