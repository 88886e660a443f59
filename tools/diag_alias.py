"""Does a stream parked in cuStreamWaitValue32 block other streams that share
its hardware queue?  Parks stream 0, then launches a kernel on each of N
later-created streams and reports which never complete."""
import os
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import sys, time
import torch
from cuda.bindings import driver as cu
from cuda.bindings import runtime as cr

torch.cuda.init()
dev = torch.device("cuda", 0)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 40
mode = sys.argv[2] if len(sys.argv) > 2 else "raw"


def mk():
    if mode == "torch":
        return torch.cuda.Stream(dev)
    err, h = cr.cudaStreamCreateWithFlags(1)
    return torch.cuda.ExternalStream(int(h), device=dev)


x = torch.ones(1 << 10, device=dev)
x.mul_(2)
torch.cuda.synchronize()
streams = [mk() for _ in range(N)]
flag = torch.zeros(4, dtype=torch.int32).pin_memory()
cu.cuStreamWaitValue32(streams[0].cuda_stream, flag.data_ptr(), 1, cu.CUstreamWaitValue_flags.CU_STREAM_WAIT_VALUE_GEQ)
evs = []
for i, s in enumerate(streams[1:], 1):
    with torch.cuda.stream(s):
        x.add_(0)
    e = torch.cuda.Event()
    e.record(s)
    evs.append((i, e))
time.sleep(1.0)
blocked = [i for i, e in evs if not e.query()]
print(mode, "N", N, "blocked behind stream 0:", blocked, flush=True)
flag[0] = 1
torch.cuda.synchronize()
print("released", flush=True)
