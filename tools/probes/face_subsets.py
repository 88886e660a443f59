"""Fused pack / unpack of subsets of the cfg2 halo faces (x faces only, y/z
faces only, all twelve): how well the access-rate-bound x-face rows overlap
the bandwidth-bound y/z rows in one launch.  Development probe."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2402_12274_b200 as mp  # noqa: E402
from golden_common import cfg2_faces, seeded_bytes  # noqa: E402
from specbuild import build_product  # noqa: E402

dev = torch.device("cuda", 0)
faces = cfg2_faces()
arr = torch.from_numpy(seeded_bytes(2, 514 ** 3 * 4)).to(dev)
dst = torch.zeros_like(arr)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
dts = {name: build_product(spec, mp) for name, spec in faces}
subsets = {
    "x": [n for n in dts if n.startswith("x")],
    "yz": [n for n in dts if not n.startswith("x")],
    "x_w1": [n for n in dts if n.startswith("x") and n.endswith("w1")],
    "x_w8": [n for n in dts if n.startswith("x") and n.endswith("w8")],
    "all": list(dts),
}
for name, sub in subsets.items():
    ds = [dts[n] for n in sub]
    outs = [torch.empty(mp.packed_size(d), dtype=torch.uint8, device=dev) for d in ds]
    tp, tu = [], []
    for it in range(12):
        flush.zero_()                 # evict, then read so no dirty flush line is written back in the timing
        flush.sum(dtype=torch.int64)
        torch.cuda._sleep(200000)
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record()
        mp.pack_multi(ds, [arr] * len(ds), outs)
        b.record()
        mp.unpack_multi(ds, outs, [dst] * len(ds))
        c.record()
        torch.cuda.synchronize()
        if it >= 2:
            tp.append(a.elapsed_time(b) * 1e3)
            tu.append(b.elapsed_time(c) * 1e3)
    print(json.dumps({"subset": name, "faces": sub, "pack_us": round(float(np.median(tp)), 1),
                      "unpack_us": round(float(np.median(tu)), 1),
                      "payload_MB": round(sum(o.numel() for o in outs) / 1e6, 2)}))
