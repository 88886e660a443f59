"""Randomized GPU parity (in the spirit of the reference's randomized corpus,
/root/reference/pkg/tests/test_datatype.py:199-205): seeded random datatype
trees that reach every plan kind (chain, span word-gather, run table,
descriptor walk, overlapping layouts), checked against the CPU oracle for
iov, pack at count 1-3, full and short unpack, at aligned and misaligned
buffer offsets.  Plan kinds hit are asserted so a lowering change cannot
silently drop a kernel from coverage.
"""

import numpy as np
import pytest
import torch

import oracle
import paper_2402_12274_b200 as mp
from specbuild import build_product

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]
DEV = torch.device("cuda", 0)
BASICS = [("basic", 1), ("basic", 4), ("basic", 8)]


def rand_spec(rng, depth=0):
    """A random constructor tree over BYTE / INT32 / INT64 (sizes bounded)."""
    if depth >= 3 or rng.random() < 0.25:
        return BASICS[rng.integers(0, 3)]
    k = rng.integers(0, 10)
    if k >= 8:
        return struct_array(rng)
    child = rand_spec(rng, depth + 1)
    if k == 0:
        return ("contiguous", int(rng.integers(1, 6)), child)
    if k == 1:
        bl = int(rng.integers(1, 5))
        return ("vector", int(rng.integers(1, 40)), bl, int(rng.integers(-2, bl + 6)), child)
    if k == 2:
        return ("hvector", int(rng.integers(1, 30)), int(rng.integers(1, 4)), int(rng.integers(-40, 200)), child)
    if k == 3:
        n = int(rng.integers(1, 50))
        bls = rng.integers(1, 6, n)
        gaps = rng.integers(0, 5, n)
        displs = np.cumsum(gaps + np.concatenate([[0], bls[:-1]]))
        if rng.random() < 0.2:
            displs = rng.integers(0, 60, n)          # unsorted / overlapping displacements
        return ("indexed", [int(x) for x in bls], [int(x) for x in displs], child)
    if k == 4:
        n = int(rng.integers(1, 4))
        kids = [rand_spec(rng, depth + 1) for _ in range(n)]
        displs = sorted(int(x) for x in rng.integers(0, 64, n))
        return ("struct", [int(x) for x in rng.integers(1, 4, n)], displs, kids)
    if k == 5:
        return ("resized", 0, int(rng.integers(1, 80)), child)
    if k == 6:
        full = [int(x) for x in rng.integers(2, 12, 3)]
        sub = [int(rng.integers(1, f + 1)) for f in full]
        offs = [int(rng.integers(0, f - s + 1)) for f, s in zip(full, sub)]
        return ("subarray", full, sub, offs, BASICS[rng.integers(0, 3)])
    return ("indexed_block", int(rng.integers(1, 4)), [int(x) for x in sorted(rng.integers(0, 50, 6))], child)


def struct_array(rng):
    """hvector of blocks of a small resized struct (the span / word-gather
    path): 2-3 fields with gaps of 0-3 bytes, 32-64 structs per block."""
    n = int(rng.integers(2, 4))
    kids = [BASICS[rng.integers(0, 3)] for _ in range(n)]
    kids[0] = BASICS[rng.integers(1, 3)]         # >= 4-byte first field: >= 128 B per block
    bls = [int(x) for x in rng.integers(1, 3, n)]
    displs, at = [], 0
    for k, b in zip(kids, bls):
        at += int(rng.integers(0, 4))
        displs.append(at)
        at += k[1] * b
    st = ("struct", bls, displs, kids)
    ext = at + int(rng.integers(0, 4))
    bl = int(rng.integers(32, 64))
    return ("hvector", int(rng.integers(4, 40)), bl, ext * bl + int(rng.integers(0, 64)),
            ("resized", 0, ext, st))


def corpus(seed, n):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        spec = struct_array(rng) if len(out) < 12 else rand_spec(rng)
        try:
            ot = oracle.OracleType(spec)
        except Exception:
            continue
        info = ot.layout_info(3)
        if info["runs"] == 0 or info["min_off"] < 0 or info["max_end"] > (1 << 20):
            continue
        out.append(spec)
    return out


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_gpu_random_types_against_oracle(seed):
    kinds = set()
    rng = np.random.default_rng(seed + 1000)
    for spec in corpus(seed, 150):
        ot = oracle.OracleType(spec)
        dt = build_product(spec, mp)
        for count in (1, 3):
            q = dt.layout_query(count)
            kinds.add(q["plan"] if not q["overlap"] else "overlap")
            info = ot.layout_info(count)
            span, total = info["max_end"], info["nbytes"]
            off = int(rng.integers(0, 16))
            src_h = rng.integers(0, 256, span + 32, dtype=np.uint8)[:span]
            base = torch.zeros(span + 32, dtype=torch.uint8, device=DEV)
            src = base[off:off + span]
            src.copy_(torch.from_numpy(src_h))
            ref = ot.pack(src_h, count=count)
            got = mp.pack(dt, src, count=count)
            assert np.array_equal(got.cpu().numpy(), ref), (spec, count, off)
            iov = mp.type_iov_tensor(dt, count=count).cpu().numpy()
            assert np.array_equal(iov, ot.iov(count=count)), (spec, count)
            for cut in (total, total // 2):
                dst = torch.full((span,), 0xC3, dtype=torch.uint8, device=DEV)
                assert mp.unpack(dt, got[:cut], dst, count=count) == cut
                exp = np.full(span, 0xC3, np.uint8)
                ot.unpack(ref[:cut], exp, count=count)
                assert np.array_equal(dst.cpu().numpy(), exp), (spec, count, cut)
        if dt not in mp.datatypes.BUILTINS:
            mp.type_free(dt)
    oracle.reset()
    # the corpus reaches the chain, span, run-table and overlapping paths
    assert {1, 3, 4} <= kinds, kinds
