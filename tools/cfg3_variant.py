"""cfg3 with a wider resized extent (gaps > 12 bytes between a word's bytes):
plan kind and pack/unpack time (development probe)."""
import os, sys, json
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")]
import paper_2402_12274_b200 as mp
from golden_common import cfg3_blocks, seeded_bytes
from specbuild import build_product

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
res = {}
for ext in (40, 56, 64):
    struct = ("struct", [1, 3, 1], [0, 8, 32], [("basic", 4), ("basic", 8), ("basic", 1)])
    bls, displs = cfg3_blocks(3, 2048)
    el = ("resized", 0, ext, struct)
    lb = min(d * ext for d in displs)
    ub = max((d + b - 1) * ext + ext for b, d in zip(bls, displs))
    spec = ("hvector", 64, 1, ub - lb + 4096, ("indexed", bls, displs, el))
    dt = build_product(spec, mp)
    q = dt.layout_query()
    span, n = q["max_end"], mp.packed_size(dt)
    src = torch.from_numpy(seeded_bytes(5, span)).to(dev)
    out = torch.empty(n, dtype=torch.uint8, device=dev)
    back = torch.zeros_like(src)
    r = {"plan": q["plan"], "specs": q["chain_align"]}
    for name, fn in (("pack", lambda: mp.pack_into(dt, src, out)), ("unpack", lambda: mp.unpack(dt, out, back))):
        fn(); ts = []
        for _ in range(5):
            flush.zero_(); torch.cuda._sleep(100000)
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
        r[name + "_GBs"] = round(2 * n / float(np.median(ts)) / 1e6, 1)
    res["ext%d" % ext] = r
print(json.dumps(res))
