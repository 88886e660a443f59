"""Where the configs[0] single-call time goes (GPU box).

Times, with bench.py's own method (L2 flushed clean, a sleep kernel so the
host has enqueued the call before the first event, CUDA events around one
library call, median of 20):

* floor_4B   -- pack of one INT32 (the smallest library launch: one k_chain1
                CTA moving 4 bytes): event + launch + one DRAM round trip;
* cfg1_cold  -- pack / unpack of vector(4096,4,8,FLOAT64), L2 flushed first;
* cfg1_warm  -- the same with its 256 KiB span resident in L2 (no flush);
* cfg1_g32   -- cold, with cudaLimitMaxL2FetchGranularity = 32;
* torch_*    -- torch's own fill / copy kernels timed the same way (4 B, a
                contiguous 128 KiB copy, the cfg1 gather as a strided copy).

One JSON line; every packed result is compared with a torch gather.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import bench  # noqa: E402  (L2Flush)
import paper_2402_12274_b200 as mp  # noqa: E402
from golden_common import CFG1_SPEC, seeded_bytes  # noqa: E402
from specbuild import build_product  # noqa: E402


def timed(fn, flush, reps=20):
    fn()
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush()
        torch.cuda._sleep(100000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return round(float(np.median(ts)), 2)


def main():
    dev = torch.device("cuda", 0)
    flush = bench.L2Flush(dev)
    out = {}
    one = torch.zeros(4, dtype=torch.uint8, device=dev)
    one_out = torch.empty(4, dtype=torch.uint8, device=dev)
    out["floor_4B_pack_us"] = timed(lambda: mp.pack_into(mp.INT32, one, one_out), flush)
    out["floor_4B_pack_warm_us"] = timed(lambda: mp.pack_into(mp.INT32, one, one_out), None)
    # torch's own kernels as the frame: a 4-byte fill (no read) and copy
    out["torch_fill_4B_us"] = timed(lambda: one_out.fill_(7), flush)
    out["torch_copy_4B_us"] = timed(lambda: one_out.copy_(one), flush)

    dt = build_product(CFG1_SPEC, mp)
    src = torch.from_numpy(seeded_bytes(11, 4096 * 64)).to(dev)   # span 262,112 B, padded
    n = mp.packed_size(dt)
    packed = torch.empty(n, dtype=torch.uint8, device=dev)
    back = torch.zeros_like(src)
    ref = src[: 4096 * 64].view(4096, 64)[:, :32].reshape(-1)
    for tag, fl in (("cold", flush), ("warm", None)):
        out["cfg1_%s_pack_us" % tag] = timed(lambda: mp.pack_into(dt, src, packed), fl)
        out["cfg1_%s_unpack_us" % tag] = timed(lambda: mp.unpack(dt, packed, back), fl)
    flat = src[:n]
    out["torch_copy_128KiB_cold_us"] = timed(lambda: packed.copy_(flat), flush)
    out["torch_strided_gather_128KiB_cold_us"] = timed(
        lambda: packed.view(4096, 32).copy_(src.view(4096, 64)[:, :32]), flush)
    prev = mp.set_l2_fetch_granularity(32)
    out["cfg1_g32_pack_us"] = timed(lambda: mp.pack_into(dt, src, packed), flush)
    out["cfg1_g32_unpack_us"] = timed(lambda: mp.unpack(dt, packed, back), flush)
    mp.set_l2_fetch_granularity(prev)
    torch.cuda.synchronize()
    out["l2_fetch_default"] = prev
    out["correct"] = bool(torch.equal(packed, ref)) and bool(
        torch.equal(back[: 4096 * 64].view(4096, 64)[:, :32].reshape(-1), ref))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
