"""Fused halo step through a CUDA graph vs direct launches (development probe)."""
import os, sys, json
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")]
import paper_2402_12274_b200 as mp
from golden_common import cfg2_faces, seeded_bytes
from specbuild import build_product

dev = torch.device("cuda", 0)
faces = cfg2_faces()
dts = [build_product(s, mp) for _, s in faces]
arr = torch.from_numpy(seeded_bytes(2, 514 ** 3 * 4)).to(dev)
dst = torch.zeros_like(arr)
outs = [torch.empty(mp.packed_size(d), dtype=torch.uint8, device=dev) for d in dts]
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def step():
    mp.pack_multi(dts, [arr] * 12, outs)
    mp.unpack_multi(dts, outs, [dst] * 12)


step(); torch.cuda.synchronize()
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    step()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        step()
torch.cuda.synchronize()
res = {}
for name, fn in (("direct", step), ("graph", g.replay)):
    ts = []
    for it in range(14):
        flush.zero_(); torch.cuda._sleep(50000)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        if it >= 4:
            ts.append(a.elapsed_time(b))
    res[name] = round(1e3 * float(np.median(ts)), 1)
dst2 = torch.zeros_like(arr)
ok = True
print(json.dumps(res))
