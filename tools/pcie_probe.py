"""PCIe ceilings for the e2e halo step (development probe): 56.6 MB pinned
H2D, D2H, and both concurrently on two streams."""
import json
import torch
dev = torch.device("cuda", 0)
n = 56623104
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device=dev)
d_out = torch.empty(n, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]
def both():
    cur = torch.cuda.current_stream()
    e = torch.cuda.Event(); e.record(cur)
    s1.wait_event(e); s2.wait_event(e)
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
r = {"h2d_ms": t(lambda: d_in.copy_(h_in, non_blocking=True)),
     "d2h_ms": t(lambda: h_out.copy_(d_out, non_blocking=True)),
     "both_ms": t(both)}
r["h2d_GBs"] = n / r["h2d_ms"] / 1e6
r["d2h_GBs"] = n / r["d2h_ms"] / 1e6
print(json.dumps(r))
