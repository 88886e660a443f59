import os, sys
sys.path[:0] = ["/root/repo", "/root/repo/tests", "/root/repo/tests/golden"]
import numpy as np, torch
import paper_2402_12274_b200 as mp
from golden_common import cfg3_spec, seeded_bytes
from specbuild import build_product
import oracle
hc = int(sys.argv[1]); which = sys.argv[2]
spec = cfg3_spec(3, hc)
dt = build_product(spec, mp)
span = dt.layout_query()["max_end"]
src_h = seeded_bytes(5, span)
src = torch.from_numpy(src_h).cuda()
out = torch.empty(mp.packed_size(dt), dtype=torch.uint8, device="cuda")
mp.pack_into(dt, src, out); torch.cuda.synchronize()
print("pack ok", hc, flush=True)
if which == "check":
    ref = oracle.OracleType(spec).pack(src_h)
    print("equal", np.array_equal(out.cpu().numpy(), ref), flush=True)
