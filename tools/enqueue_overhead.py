"""Host cost of the enqueue calls (development probe): one rank, self
send/recv of 8 bytes, per-call wall time of each API call."""
import os, sys, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2402_12274_b200 as mp

inst = mp.init(rank=0, ranks=1, group="ovh", device=0)
q = mp.queue_create(inst)
info = mp.info_create()
info.set("type", "devstream")
mp.info_set_hex(info, "value", bytes.fromhex(q.handle))
s = inst.stream_create(info)
c = mp.stream_comm_create(inst.world, s)
src = torch.ones(8, dtype=torch.uint8, device="cuda")
dst = torch.zeros_like(src)
T = {"irecv": 0.0, "isend": 0.0, "waitall": 0.0}
N = 2000
for it in range(N + 100):
    t0 = time.perf_counter()
    rr = mp.irecv_enqueue(c, dst, 8, mp.BYTE, 0, 0)
    t1 = time.perf_counter()
    sr = mp.isend_enqueue(c, src, 8, mp.BYTE, 0, 0)
    t2 = time.perf_counter()
    mp.waitall_enqueue([rr, sr])
    t3 = time.perf_counter()
    if it >= 100:
        T["irecv"] += t1 - t0
        T["isend"] += t2 - t1
        T["waitall"] += t3 - t2
    if it % 200 == 0:
        mp.queue_synchronize(q)
mp.queue_synchronize(q)
print(json.dumps({k: round(v / N * 1e6, 2) for k, v in T.items()}))
import cProfile, pstats
pr = cProfile.Profile()
pr.enable()
for it in range(500):
    rr = mp.irecv_enqueue(c, dst, 8, mp.BYTE, 0, 0)
    sr = mp.isend_enqueue(c, src, 8, mp.BYTE, 0, 0)
    mp.waitall_enqueue([rr, sr])
pr.disable()
mp.queue_synchronize(q)
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
