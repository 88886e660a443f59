"""Pack + unpack of one cfg2 face (development tool for ncu captures).
    python tools/face_one.py xlo-w8 [reps]"""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")]
import paper_2402_12274_b200 as mp
from golden_common import cfg2_faces, seeded_bytes
from specbuild import build_product

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda", 0)
dt = build_product(dict(cfg2_faces())[name], mp)
arr = torch.from_numpy(seeded_bytes(1, 514 ** 3 * 4)).to(dev)
dst = torch.zeros_like(arr)
out = torch.empty(mp.packed_size(dt), dtype=torch.uint8, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(reps):
    flush.zero_()
    mp.pack_into(dt, arr, out)
    flush.zero_()
    mp.unpack(dt, out, dst)
torch.cuda.synchronize()
