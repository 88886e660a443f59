"""Per-layout timing breakdown (development tool, not the driver bench).

    python tools/face_bench.py [--reps 20] [--cfg3]

Times pack and unpack of each cfg2 halo face (and optionally cfg1 / cfg3) in
isolation with CUDA events, L2 flushed before every launch, and prints one
JSON line per layout: payload GB/s and the 32 B-sector DRAM floor computed
from the iov list (bytes in distinct sectors touched on the layout side).
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import paper_2402_12274_b200 as mp  # noqa: E402
from golden_common import CFG1_SPEC, cfg2_faces, cfg3_spec, seeded_bytes  # noqa: E402
from specbuild import build_product  # noqa: E402


def sector_bytes(dt):
    iov = mp.type_iov_tensor(dt)
    o = iov[:, 0]
    e = iov[:, 0] + iov[:, 1]
    first = torch.div(o, 32, rounding_mode="floor")
    last = torch.div(e - 1, 32, rounding_mode="floor")
    return int((last - first + 1).sum().item()) * 32


def time_op(fn, reps, flush):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(reps)]
    fn()
    for a, b in evs:
        flush.zero_()
        torch.cuda._sleep(100000)   # keep the host ahead: no launch gap inside the events
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in evs]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--cfg3", action="store_true")
    ap.add_argument("--l2fetch", type=int, default=-1)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.init()
    prev = mp.set_l2_fetch_granularity(args.l2fetch, dev)
    print(json.dumps({"l2_fetch_prev": prev, "l2_fetch_now": mp.set_l2_fetch_granularity(-1, dev)}))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    cases = [("cfg1", CFG1_SPEC, 32768 * 8)]
    cases += [("cfg2-" + n, s, 514 ** 3 * 4) for n, s in cfg2_faces()]
    if args.cfg3:
        cases.append(("cfg3", cfg3_spec(3), None))
    arrays = {}
    for name, spec, span in cases:
        dt = build_product(spec, mp)
        if span is None:
            span = dt.layout_query()["max_end"]
        if span not in arrays:
            arrays[span] = (torch.from_numpy(seeded_bytes(7, span)).to(dev),
                            torch.zeros(span, dtype=torch.uint8, device=dev))
        src, dst = arrays[span]
        n = mp.packed_size(dt)
        out = torch.empty(n, dtype=torch.uint8, device=dev)
        tp = time_op(lambda: mp.pack_into(dt, src, out), args.reps, flush)
        tu = time_op(lambda: mp.unpack(dt, out, dst), args.reps, flush)
        sb = sector_bytes(dt)
        q = dt.layout_query()
        print(json.dumps({
            "layout": name, "plan": q["plan"], "segments": q["runs"], "payload": n,
            "pack_us": round(tp * 1e3, 2), "unpack_us": round(tu * 1e3, 2),
            "pack_GBs": round(2 * n / tp / 1e6, 1), "unpack_GBs": round(2 * n / tu / 1e6, 1),
            "sector_bytes": sb,
            "pack_sector_GBs": round((sb + n) / tp / 1e6, 1),
        }), flush=True)


if __name__ == "__main__":
    main()
