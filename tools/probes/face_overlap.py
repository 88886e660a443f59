"""Do the access-rate-bound x faces and the bandwidth-bound y/z faces overlap
when they run at the same time?  Fused pack / unpack of the x faces on one
stream and of the y/z faces on another, launched together, vs all twelve in
one fused launch (development probe; L2 flushed clean before each step)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2402_12274_b200 as mp  # noqa: E402
from golden_common import cfg2_faces, seeded_bytes  # noqa: E402
from specbuild import build_product  # noqa: E402

dev = torch.device("cuda", 0)
arr = torch.from_numpy(seeded_bytes(2, 514 ** 3 * 4)).to(dev)
dst = torch.zeros_like(arr)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
faces = [(n, build_product(s, mp)) for n, s in cfg2_faces()]
X = [d for n, d in faces if n.startswith("x")]
YZ = [d for n, d in faces if not n.startswith("x")]
ALL = [d for _, d in faces]
out = {id(d): torch.empty(mp.packed_size(d), dtype=torch.uint8, device=dev) for d in ALL}
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
main = torch.cuda.current_stream()


def fused(ds, pack):
    if pack:
        mp.pack_multi(ds, [arr] * len(ds), [out[id(d)] for d in ds])
    else:
        mp.unpack_multi(ds, [out[id(d)] for d in ds], [dst] * len(ds))


def two_streams(pack):
    ev = torch.cuda.Event()
    ev.record(main)
    for s, ds in ((s1, X), (s2, YZ)):
        s.wait_event(ev)
        with torch.cuda.stream(s):
            fused(ds, pack)
    main.wait_stream(s1)
    main.wait_stream(s2)


for name, fn in (("one launch, 12 faces", lambda p: fused(ALL, p)), ("x || y/z on two streams", two_streams)):
    res = {}
    for pack in (True, False):
        ts = []
        for it in range(12):
            flush.zero_()
            flush.sum(dtype=torch.int64)
            torch.cuda._sleep(200000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(main)
            fn(pack)
            b.record(main)
            torch.cuda.synchronize()
            if it >= 2:
                ts.append(a.elapsed_time(b) * 1e3)
        res["pack_us" if pack else "unpack_us"] = round(float(np.median(ts)), 1)
    print(json.dumps({"mode": name, **res}))
