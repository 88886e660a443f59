"""Which host calls block while a stream is parked in cuStreamWaitValue32?"""
import os
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import sys, threading, time
import torch
from cuda.bindings import driver as cu

torch.cuda.init()
dev = torch.device("cuda", 0)
A = cu.CUdevice_attribute
for name in ["CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_WAIT_VALUE_NOR",
             "CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS",
             "CU_DEVICE_ATTRIBUTE_CAN_USE_HOST_POINTER_FOR_REGISTERED_MEM",
             "CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES"]:
    try:
        print(name, cu.cuDeviceGetAttribute(getattr(A, name), 0), flush=True)
    except Exception as e:
        print(name, "n/a", e, flush=True)

mode = sys.argv[1] if len(sys.argv) > 1 else "host"
if mode == "host":
    flag = torch.zeros(4, dtype=torch.int32).pin_memory()
else:
    flag = torch.zeros(4, dtype=torch.int32, device=dev)
s = torch.cuda.Stream(dev)
x = torch.ones(16, device=dev)
s2 = torch.cuda.Stream(dev)
if "warm" in sys.argv:
    with torch.cuda.stream(s2):
        torch.arange(1000, device=dev).mul_(2)
        x.add_(0)
        flag.fill_(0) if flag.is_cuda else None
torch.cuda.synchronize()
r = cu.cuStreamWaitValue32(s.cuda_stream, flag.data_ptr(), 1, cu.CUstreamWaitValue_flags.CU_STREAM_WAIT_VALUE_GEQ)
print(mode, "wait enqueued", r, flush=True)


def probe(name, fn, t=3.0):
    done = threading.Event()
    err = []
    def run():
        try:
            fn()
        except Exception as e:
            err.append(repr(e))
        done.set()
    th = threading.Thread(target=run, daemon=True)
    th.start()
    ok = done.wait(t)
    print("%-50s %s %s" % (name, "ok" if ok else "BLOCKED", err), flush=True)
    return ok

def on_s2():
    with torch.cuda.stream(s2):
        torch.arange(1000, device=dev).mul_(2)
ok = probe("kernel on another stream s2", on_s2)
ok = ok and probe("event record on s (behind wait)", lambda: torch.cuda.Event().record(s))
def on_s():
    with torch.cuda.stream(s):
        x.add_(1)
ok = ok and probe("kernel on s (behind wait)", on_s)
ok = ok and probe("kernel on s2 after that", on_s2)
ok = ok and probe("torch.empty 64MB", lambda: torch.empty(64 << 20, dtype=torch.uint8, device=dev))
from cuda.bindings import runtime as cr
def new_stream():
    err, h = cr.cudaStreamCreateWithFlags(1)
    assert err == cr.cudaError_t.cudaSuccess, err
    return torch.cuda.ExternalStream(int(h), device=dev)
ok = ok and probe("cudaStreamCreate (new stream)", new_stream)
ok = ok and probe("cudaEventCreate", lambda: cr.cudaEventCreate())
def on_new():
    ns = new_stream()
    with torch.cuda.stream(ns):
        torch.arange(1000, device=dev).mul_(2)
    ev = torch.cuda.Event()
    ev.record(ns)
    ns.synchronize()
ok = ok and probe("kernel on a NEW stream (+ its sync)", on_new)
def wait_on_new():
    ns = new_stream()
    e = torch.cuda.Event()
    e.record(s2)
    ns.wait_event(e)
    with torch.cuda.stream(ns):
        torch.arange(1000, device=dev).mul_(2)
    ns.synchronize()
ok = ok and probe("event wait + kernel on a NEW stream", wait_on_new)
print("releasing flag", flush=True)
if mode == "host":
    flag[0] = 1
else:
    def rel():
        with torch.cuda.stream(s2):
            flag.fill_(1)
    probe("device flag write on s2", rel)
t0 = time.time()
done = threading.Event()
threading.Thread(target=lambda: (s.synchronize(), done.set()), daemon=True).start()
print("stream released" if done.wait(10) else "stream STILL BLOCKED", "%.3fs" % (time.time() - t0), flush=True)
os._exit(0)
