"""type_iov throughput (development tool): full device iov of cfg1, the cfg2
x-face and cfg3; L2 flushed before each launch.  Output bytes = 16 per
segment."""
import os, sys, json
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")]
import paper_2402_12274_b200 as mp
from golden_common import CFG1_SPEC, cfg2_faces, cfg3_spec
from specbuild import build_product

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
res = {}
for name, spec in (("cfg1", CFG1_SPEC), ("cfg2-xlo-w1", dict(cfg2_faces())["xlo-w1"]),
                   ("cfg2-zlo-w8", dict(cfg2_faces())["zlo-w8"]), ("cfg3", cfg3_spec(3))):
    dt = build_product(spec, mp)
    n = dt.segment_count
    out = mp.type_iov_tensor(dt)
    ts = []
    for _ in range(5):
        flush.zero_()
        torch.cuda._sleep(100000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); mp.type_iov_tensor(dt); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    res[name] = {"segments": n, "us": round(ms * 1e3, 1), "GBs_out": round(16 * n / ms / 1e6, 1),
                 "Gseg_s": round(n / ms / 1e6, 2)}
print(json.dumps(res))
