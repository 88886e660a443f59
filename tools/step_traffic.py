"""DRAM traffic of the bench step as a STEP (roofline.traffic evidence).

    ncu --replay-mode range --cache-control all \
        --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum \
        --csv --log-file gpurun_out/step_range.csv python tools/step_traffic.py

One profiled range = [fused pack of the 12 halo faces, fused unpack of them,
a READ of a 256 MiB buffer].  ncu flushes the caches before the range; the
trailing read evicts every dirty line the two kernels left in the 126 MB L2,
so the range's DRAM writes hold ALL of the step's write traffic (including
the write-back of the packed faces and of the unpacked layout), and its DRAM
reads hold the step's reads plus the 256 MiB of the flush read itself
(subtracted in tools/make_traffic.py).  Run without ncu it prints the
layout-side DRAM floor of the step (bench.step_floor) as JSON.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")]

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2402_12274_b200 as mp  # noqa: E402
from golden_common import seeded_bytes  # noqa: E402
from specbuild import build_product  # noqa: E402

FLUSH_READ = 256 << 20


def main():
    dev = torch.device("cuda", 0)
    faces = bench.face_specs()
    dts = [build_product(sp, mp) for _, sp in faces]
    arr = torch.from_numpy(seeded_bytes(2, bench.ARRAY_BYTES)).to(dev)
    dst = torch.zeros_like(arr)
    packed = [torch.empty(bench.face_bytes(sp), dtype=torch.uint8, device=dev) for _, sp in faces]
    rd = torch.zeros(FLUSH_READ // 8, dtype=torch.int64, device=dev)
    floor = bench.step_floor(dts, dev)

    def step():
        mp.pack_multi(dts, [arr] * len(dts), packed)
        mp.unpack_multi(dts, packed, [dst] * len(dts))

    for _ in range(3):      # plans built, kernels loaded
        step()
    rd.max()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    step()
    rd.max()                 # evicts the dirty lines of the step: their write-back lands in the range
    torch.cuda.cudart().cudaProfilerStop()
    torch.cuda.synchronize()
    print(json.dumps({"flush_read_bytes": FLUSH_READ, "algorithmic_bytes_per_step": bench.step_bytes(),
                      "floor": floor}))


if __name__ == "__main__":
    main()
