"""cfg3 pack/unpack timing (development tool): hvector(256) of indexed(2048)
of a resized-40 struct, seeded source, L2 flushed before each launch."""
import os, sys, json
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")]
import paper_2402_12274_b200 as mp
from golden_common import cfg3_spec, seeded_bytes
from specbuild import build_product

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
dev = torch.device("cuda", 0)
dt = build_product(cfg3_spec(3), mp)
span = dt.layout_query()["max_end"]
src = torch.from_numpy(seeded_bytes(5, span)).to(dev)
dst = torch.zeros_like(src)
n = mp.packed_size(dt)
out = torch.empty(n, dtype=torch.uint8, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
res = {}
for name, fn in (("pack", lambda: mp.pack_into(dt, src, out)), ("unpack", lambda: mp.unpack(dt, out, dst))):
    fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        torch.cuda._sleep(100000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    res[name + "_us"] = round(1e3 * float(np.median(ts)), 1)
    res[name + "_GBs"] = round(2 * n / (float(np.median(ts)) / 1e3) / 1e9, 1)
print(json.dumps(res))
