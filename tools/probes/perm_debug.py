"""k_perm pack debugging aid: compare the GPU pack of cfg3-shaped types with
the oracle and locate mismatches relative to block boundaries."""
import sys
import numpy as np
import torch
ROOT = "/root/repo"
sys.path[:0] = [ROOT, ROOT + "/tests", ROOT + "/tests/golden"]
import paper_2402_12274_b200 as mp  # noqa: E402
import oracle  # noqa: E402
from golden_common import cfg3_spec, cfg3_blocks, seeded_bytes  # noqa: E402
from specbuild import build_product  # noqa: E402

for hc, nb in ((4, 2048),):
    spec = cfg3_spec(3, hc, nb)
    bls, displs = cfg3_blocks(3, nb)
    bounds = np.cumsum(np.tile(np.array(bls) * 29, hc))
    dt = build_product(spec, mp)
    ot = oracle.OracleType(spec)
    span = ot.max_end
    src_h = seeded_bytes(7, span)
    for trial in range(3):
        got = mp.pack(dt, torch.from_numpy(src_h).cuda()).cpu().numpy()
        ref = ot.pack(src_h)
        bad = np.nonzero(got != ref)[0]
        print("trial", trial, "bad", len(bad), flush=True)
        for b in bad[:40]:
            k = np.searchsorted(bounds, b, side="right")
            print(" off", b, "got", got[b], "ref", ref[b], "block", k, "block_end", bounds[k],
                  "bl", bls[k % nb], "dist_to_end", bounds[k] - b, "next_bl", bls[(k + 1) % nb])
