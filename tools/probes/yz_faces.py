import os, sys
ROOT = "/root/repo"
sys.path[:0] = [ROOT, ROOT + "/tests", ROOT + "/tests/golden"]
import torch
import paper_2402_12274_b200 as mp
from golden_common import cfg2_faces, seeded_bytes
from specbuild import build_product
dev = torch.device("cuda", 0)
arr = torch.from_numpy(seeded_bytes(2, 514 ** 3 * 4)).to(dev)
dst = torch.zeros_like(arr)
ds = [build_product(s, mp) for n, s in cfg2_faces() if not n.startswith("x")]
outs = [torch.empty(mp.packed_size(d), dtype=torch.uint8, device=dev) for d in ds]
for _ in range(3):
    mp.pack_multi(ds, [arr] * len(ds), outs)
    mp.unpack_multi(ds, outs, [dst] * len(ds))
torch.cuda.synchronize()
