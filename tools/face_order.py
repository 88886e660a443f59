"""Fused 12-face pack/unpack time vs job order (development probe)."""
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
arr = torch.from_numpy(seeded_bytes(2, 514 ** 3 * 4)).to(dev)
dst = torch.zeros_like(arr)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
orders = {"x_first": [n for n, _ in faces],
          "yz_first": [n for n, _ in faces if n[0] != "x"] + [n for n, _ in faces if n[0] == "x"],
          "mixed": ["xlo-w1", "zlo-w8", "xhi-w1", "zhi-w8", "xlo-w8", "ylo-w8", "xhi-w8", "yhi-w8",
                    "ylo-w1", "yhi-w1", "zlo-w1", "zhi-w1"]}
spec = dict(faces)
res = {}
for name, order in orders.items():
    dts = [build_product(spec[n], mp) for n in order]
    outs = [torch.empty(mp.packed_size(d), dtype=torch.uint8, device=dev) for d in dts]
    tp, tu = [], []
    for it in range(12):
        flush.zero_(); torch.cuda._sleep(50000)
        a, b, c = (torch.cuda.Event(True) for _ in range(3))
        a.record(); mp.pack_multi(dts, [arr] * 12, outs); b.record()
        mp.unpack_multi(dts, outs, [dst] * 12); c.record(); torch.cuda.synchronize()
        if it >= 2:
            tp.append(a.elapsed_time(b)); tu.append(b.elapsed_time(c))
    res[name] = {"pack_us": round(1e3 * float(np.median(tp)), 1), "unpack_us": round(1e3 * float(np.median(tu)), 1)}
print(json.dumps(res))
