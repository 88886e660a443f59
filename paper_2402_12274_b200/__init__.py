"""paper_2402_12274_b200 -- B200-native MPIX datatype / enqueue hot path.

A drop-in for the data path of the reference package ``minimpi``
(/root/reference/pkg/src/minimpi/__init__.py:13-63): the same flat API names
for derived datatypes, iov queries, pack/unpack, CUDA-stream communicators and
the enqueue operations, executed by hand-written sm_100a kernels in
libmpx.so (C ABI: include/mpx.h).  Buffers are PyTorch CUDA tensors (host
buffers are accepted and staged through the GPU).
"""

from .errors import (  # noqa: F401
    MinimpiError, StateError, PendingError, ArgError, TransportError,
    SpawnError, ExhaustedError, UnsupportedError, TruncateError,
)
from .datatypes import (  # noqa: F401
    Datatype, IovSegment,
    BYTE, CHAR, INT8, INT32, INT64, FLOAT32, FLOAT64,
    type_contiguous, type_vector, type_hvector, type_indexed_block,
    type_indexed, type_create_struct, type_create_subarray,
    type_create_resized, type_commit, type_free, type_iov_len, type_iov,
    type_iov_tensor, pack, pack_into, unpack, pack_multi, unpack_multi,
    packed_size, check_region, parse_type_expr, set_l2_fetch_granularity,
)

ANY_SOURCE = -1
ANY_TAG = -1

__version__ = "0.1.0"
