import os, sys, json, time, threading
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tools")]
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch
import paper_2402_12274_b200 as mp
import enqueue_bench as eb

def probe(n, count, iters=5):
    def body(inst, bar):
        q = mp.queue_create(inst)
        info = mp.info_create(); info.set("type", "devstream"); mp.info_set_hex(info, "value", bytes.fromhex(q.handle))
        s = inst.stream_create(info); c = mp.stream_comm_create(inst.world, s)
        x = torch.full((count,), 1.0, device=inst.device); y = torch.zeros_like(x)
        mp.allreduce_enqueue(c, x, y, count, mp.FLOAT32, algo="native"); mp.queue_synchronize(q)
        bar.wait()
        evs = []
        th = 0.0
        for _ in range(iters):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(q.torch_stream)
            t0 = time.perf_counter()
            mp.allreduce_enqueue(c, x, y, count, mp.FLOAT32, algo="native")
            th += time.perf_counter() - t0
            b.record(q.torch_stream)
            evs.append((a, b))
        mp.queue_synchronize(q)
        dev_ms = [a.elapsed_time(b) for a, b in evs]
        mp.comm_free(c); mp.free_stream(s)
        return {"rank": inst.rank, "host_us_per_call": 1e6 * th / iters, "device_ms": [round(d, 3) for d in dev_ms]}
    return eb._run_ranks(n, body, "probe-%d-%d" % (n, count))

for n, count in ((1, 16 << 20), (2, 1 << 10), (2, 16 << 20)):
    print(n, count, json.dumps(probe(n, count)), flush=True)
