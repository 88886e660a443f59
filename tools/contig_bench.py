"""Contiguous pack (one 256 MiB run, the ring's send path) vs torch copy_
(development probe)."""
import json, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2402_12274_b200 as mp

dev = torch.device("cuda", 0)
n = 256 << 20
a = torch.empty(n, dtype=torch.uint8, device=dev)
b = torch.empty_like(a)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
dt = mp.type_contiguous(n, mp.BYTE).commit()
vec = mp.type_vector(n // 64, 32, 64, mp.BYTE).commit()
vb = torch.empty(n // 2, dtype=torch.uint8, device=dev)


def t(fn, reps=8):
    fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        torch.cuda._sleep(100000)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))

res = {}
for name, fn, by in (("torch_copy", lambda: b.copy_(a), 2 * n),
                     ("mpx_pack_contig", lambda: mp.pack_into(dt, a, b), 2 * n),
                     ("mpx_unpack_contig", lambda: mp.unpack(dt, b, a), 2 * n),
                     ("mpx_pack_vector32of64", lambda: mp.pack_into(vec, a, vb), n),
                     ("mpx_unpack_vector32of64", lambda: mp.unpack(vec, vb, a), n)):
    ms = t(fn)
    res[name] = {"us": round(ms * 1e3, 1), "GBs_rw": round(by / ms / 1e6, 1)}
print(json.dumps(res))
