"""GPU timeline of the 2-rank in-process ring (64 MiB u8 by default) via the
torch profiler (CUPTI activity records; no nsys on the box): per-kernel and
per-memcpy start / duration / stream, to see where an iteration's time goes
beyond the copies themselves.  Development probe."""
import json
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tools")]
import torch  # noqa: E402
from torch.profiler import profile, ProfilerActivity  # noqa: E402

import enqueue_bench as eb  # noqa: E402

nbytes = int(sys.argv[1]) if len(sys.argv) > 1 else 64 << 20
kind = sys.argv[2] if len(sys.argv) > 2 else "u8"
eb.ring(2, nbytes, iters=3, warmup=3, group="tl-warm", kind=kind)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    r = eb.ring(2, nbytes, iters=5, warmup=1, group="tl", kind=kind)
print(json.dumps({k: r[k] for k in ("ms_per_iter", "GBps_per_rank", "correct")}))
evs = []
for e in prof.events():
    if e.device_type.name == "CUDA" or getattr(e, "device_type", None) == torch.autograd.DeviceType.CUDA:
        evs.append((e.time_range.start, e.time_range.end - e.time_range.start, e.name[:60]))
evs.sort()
t0 = evs[0][0] if evs else 0
for s, d, n in evs[-60:]:
    print("%10.1f us  dur %8.1f us  %s" % (s - t0, d, n))
