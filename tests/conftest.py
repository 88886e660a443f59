import gzip
import json
import os
import sys

# one hardware queue per stream (set before any CUDA context exists): stream
# communicators block streams in memop waits, which must never stall an
# unrelated stream that shares a hardware queue
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# eager module loading: with lazy loading the first launch of any kernel waits
# behind a stream parked in a stream-memop wait (measured: tools/diag_memop.py)
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, GOLDEN):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


_cache = {}


def load_golden(name):
    if name not in _cache:
        with gzip.open(os.path.join(GOLDEN, "%s.json.gz" % name), "rt") as f:
            _cache[name] = json.load(f)
    return _cache[name]


def to_tuple_spec(spec):
    """JSON lists -> the tuple forms (first element is the kind)."""
    if isinstance(spec, list) and spec and isinstance(spec[0], str):
        kind = spec[0]
        if kind == "struct":
            return (kind, list(spec[1]), list(spec[2]), [to_tuple_spec(c) for c in spec[3]])
        return tuple([kind] + [to_tuple_spec(x) if isinstance(x, list) and x and
                               isinstance(x[0], str) else x for x in spec[1:]])
    return spec


@pytest.fixture(autouse=True)
def _release_leftover_queues():
    """Test hygiene: device queues a test did not destroy go back to libmpx's
    stream pool when the test ends.  A queue's stream is never reclaimed by
    the garbage collector (work may still be ordered on it), so leaked queues
    used to grow the pool past the device's hardware queues over a long
    suite; two ranks' streams sharing a hardware queue can then park each
    other in a stream-memop handshake."""
    yield
    qmod = sys.modules.get("paper_2402_12274_b200.queues")
    if qmod is None:
        return
    with qmod._lock:
        left = [q for q in qmod._QUEUES.values() if not q.destroyed]
    for q in left:
        try:
            q.destroy()
        except Exception:
            pass
