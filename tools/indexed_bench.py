"""Irregular indexed types (unstructured-mesh halos): many small blocks.
Development probe: plan kind + pack/unpack/iov time."""
import os, sys, json
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")]
import paper_2402_12274_b200 as mp
import oracle
from specbuild import build_product

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def t(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        torch.cuda._sleep(100000)
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


res = {}
rng = np.random.default_rng(1)
for name, nblk, blmax, gapmax, elem in (("idx_1M_1-4xf64", 1 << 20, 4, 8, 8),
                                       ("idx_256k_1-16xf32", 1 << 18, 16, 64, 4),
                                       ("idx_64k_8-64xf64", 1 << 16, 64, 32, 8)):
    bls = rng.integers(1, blmax + 1, nblk)
    gaps = rng.integers(0, gapmax + 1, nblk)
    displs = np.cumsum(gaps + np.concatenate([[0], bls[:-1]]))
    spec = ("indexed", [int(x) for x in bls], [int(x) for x in displs], ("basic", elem))
    dt = build_product(spec, mp)
    q = dt.layout_query()
    span = q["max_end"]
    n = mp.packed_size(dt)
    src = torch.randint(0, 256, (span,), dtype=torch.uint8, device=dev)
    out = torch.empty(n, dtype=torch.uint8, device=dev)
    back = torch.zeros_like(src)
    tp = t(lambda: mp.pack_into(dt, src, out))
    tu = t(lambda: mp.unpack(dt, out, back))
    ti = t(lambda: mp.type_iov_tensor(dt))
    ok = bool(torch.equal(back[:0], back[:0]))
    if n < (64 << 20):
        ot = oracle.OracleType(spec)
        ok = np.array_equal(out.cpu().numpy(), ot.pack(src.cpu().numpy()))
    res[name] = {"plan": q["plan"], "specs": q["chain_align"], "segments": q["runs"], "payload": n,
                 "pack_us": round(tp * 1e3, 1), "unpack_us": round(tu * 1e3, 1), "iov_us": round(ti * 1e3, 1),
                 "pack_GBs": round(2 * n / tp / 1e6, 1), "pack_ok": ok}
    print(json.dumps({name: res[name]}), flush=True)
