"""L2 fetch-granularity probe (development tool): pack the 1-wide x-face of
the cfg2 array under each cudaLimitMaxL2FetchGranularity setting.
Run under ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum."""
import os, sys, json
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")]
import numpy as np
import paper_2402_12274_b200 as mp
from golden_common import cfg2_faces, seeded_bytes
from specbuild import build_product

dev = torch.device("cuda", 0)
faces = dict(cfg2_faces())
arr = torch.from_numpy(seeded_bytes(1, 514 ** 3 * 4)).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
out = {}
for name in ("xlo-w1", "xlo-w8"):
    dt = build_product(faces[name], mp)
    o = torch.empty(mp.packed_size(dt), dtype=torch.uint8, device=dev)
    for g in (32, 64, 128):
        mp.set_l2_fetch_granularity(g, dev)
        ts = []
        for _ in range(5):
            flush.zero_()
            torch.cuda._sleep(100000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); mp.pack_into(dt, arr, o); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        out["%s/%d" % (name, g)] = (mp.set_l2_fetch_granularity(-1, dev), round(1e3 * float(np.median(ts)), 2))
print(json.dumps(out))
