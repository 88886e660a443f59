"""Latency of cross-stream ping-pong through stream memory operations:
flags in pinned host memory vs device memory (diagnostic)."""
import os
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import time
import torch
from cuda.bindings import driver as cu

GEQ = cu.CUstreamWaitValue_flags.CU_STREAM_WAIT_VALUE_GEQ
torch.cuda.init()
dev = torch.device("cuda", 0)
for where in ("host", "device"):
    if where == "host":
        f = torch.zeros(64, dtype=torch.int32).pin_memory()
    else:
        f = torch.zeros(64, dtype=torch.int32, device=dev)
    a1, a2 = f.data_ptr(), f.data_ptr() + 128
    sa, sb = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    torch.cuda.synchronize()
    N = 500
    t0 = time.perf_counter()
    for i in range(1, N + 1):
        cu.cuStreamWriteValue32(sa.cuda_stream, a1, i, 0)
        cu.cuStreamWaitValue32(sa.cuda_stream, a2, i, GEQ)
        cu.cuStreamWaitValue32(sb.cuda_stream, a1, i, GEQ)
        cu.cuStreamWriteValue32(sb.cuda_stream, a2, i, 0)
    t1 = time.perf_counter()
    sa.synchronize(); sb.synchronize()
    t2 = time.perf_counter()
    print("%-6s enqueue %.1f us/iter, total %.1f us/iter (round trip)" % (
        where, 1e6 * (t1 - t0) / N, 1e6 * (t2 - t0) / N), flush=True)
    # one-way latency with the host as writer
    e = torch.cuda.Event(enable_timing=True)
