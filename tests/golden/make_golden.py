"""Generate golden vectors for the datatype hot path FROM THE REAL REFERENCE.

Run here (the dev container, where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified Python reference ``minimpi`` from
``/root/reference/pkg/src`` plus the reference's own test generator
``dt_random.gen_type`` (``/root/reference/pkg/tests/dt_random.py:58-164``),
and records, per datatype, what the reference computes: size/lb/ub/extent,
segment_count, node_count, ``type_iov_len`` at several budgets, ``type_iov``
(full list or its sha256) and windows, and sha256 digests of ``pack`` /
``unpack`` results on seeded buffers.  The fixtures are committed; the GPU box
never reads /root/reference.

Seeded buffers are regenerable anywhere with ``seeded_bytes(seed, n)``
(numpy PCG64), so the checker side rebuilds identical inputs.

Corpora:
  unit   : seeds 0xD7A0+0..5 x 40 types, cap 1500, 80% pack-safe
           (test_datatype.py:199-205)
  crit1  : seed 0x5EED, 1000 types, cap 20k (100k every 25th)
           (test_acceptance.py:58-81)
  frozen : the hand-written examples of test_datatype.py:25-139
  configs: BASELINE.json cfg1, cfg2 (12 halo faces of 514^3 f32), cfg3
           (a reduced hvector count for full pack parity; full-size counts and
           iov windows for the real cfg3)
  allreduce: reference allreduce INT64/FLOAT64 at 2 and 4 in-proc ranks
"""

import gzip
import hashlib
import json
import os
import random
import sys
import threading

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)

import minimpi as mp  # noqa: E402  (the reference, read-only)
from dt_random import gen_type  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from golden_common import (seeded_bytes, sha, iov_digest, cfg2_faces,  # noqa: E402
                           cfg3_spec, CFG1_SPEC)

INLINE_IOV = 2048     # store the full iov list up to this many segments


def build_ref(spec):
    """Build the reference Datatype for a tuple spec (indexed emulated with
    struct, as the reference has no type_indexed: SURVEY 8a a3)."""
    k = spec[0]
    if k == "basic":
        return {1: mp.BYTE, 4: mp.INT32, 8: mp.INT64}[spec[1]]
    if k == "contiguous":
        return mp.type_contiguous(spec[1], build_ref(spec[2])).commit()
    if k == "vector":
        return mp.type_vector(spec[1], spec[2], spec[3], build_ref(spec[4])).commit()
    if k == "hvector":
        return mp.type_hvector(spec[1], spec[2], spec[3], build_ref(spec[4])).commit()
    if k == "indexed_block":
        return mp.type_indexed_block(spec[1], spec[2], build_ref(spec[3])).commit()
    if k == "struct":
        return mp.type_create_struct(spec[1], spec[2],
                                     [build_ref(c) for c in spec[3]]).commit()
    if k == "subarray":
        return mp.type_create_subarray(spec[1], spec[2], spec[3],
                                       build_ref(spec[4])).commit()
    if k == "resized":
        return mp.type_create_resized(build_ref(spec[3]), spec[1], spec[2]).commit()
    if k == "indexed":
        child = build_ref(spec[3])
        ext = child.extent_bytes
        return mp.type_create_struct(list(spec[1]), [d * ext for d in spec[2]],
                                     [child] * len(spec[1])).commit()
    raise ValueError(k)


def ref_iov(dt, off=0, maxlen=-1):
    segs, n = mp.type_iov(dt, off, maxlen)
    return [(s.base_offset, s.length) for s in segs]


def record(name, spec, dt, rng, seed, pack_ok=True, max_pack_span=1 << 22,
           windows=3, full_iov=True):
    rec = {"name": name, "spec": spec, "seed": seed,
           "size": dt.size_bytes, "lb": dt.lb, "ub": dt.ub,
           "extent": dt.extent_bytes, "segments": dt.segment_count,
           "node_count": dt.node_count}
    total = dt.size_bytes
    budgets = sorted({0, 1, total, total + 7, rng.randint(0, total + 1) if total else 0,
                      total // 3})
    rec["iov_len"] = [[b, list(mp.type_iov_len(dt, b))] for b in budgets]
    rec["iov_len"].append([-1, list(mp.type_iov_len(dt, -1))])
    nseg = dt.segment_count
    if full_iov:
        runs = ref_iov(dt)
        rec["iov_sha"] = iov_digest(runs)
        if nseg <= INLINE_IOV:
            rec["iov"] = runs
        span = max((o + l for o, l in runs), default=0)
        lo = min((o for o, _ in runs), default=0)
    else:
        runs = None
        span = dt._layout.max_end if nseg else 0
        lo = dt._layout.min_off if nseg else 0
    rec["span"] = span
    rec["min_off"] = lo
    wins = []
    if nseg:
        for _ in range(windows):
            off = rng.randint(0, nseg)
            ml = rng.choice([-1, 0, 1, rng.randint(0, min(nseg, 5000) + 2)])
            w = ref_iov(dt, off, ml)
            if runs is not None:
                assert w == runs[off:off + (len(runs) if ml == -1 else ml)]
            wins.append([off, ml, len(w), iov_digest(w),
                         w if len(w) <= 64 else w[:4] + w[-4:]])
    rec["windows"] = wins
    if pack_ok and nseg and lo >= 0 and span <= max_pack_span:
        buf = seeded_bytes(seed, span)
        packed = mp.pack(dt, buf.tobytes())
        rec["pack_sha"] = sha(packed)
        data = seeded_bytes(seed + 1, total)
        out = bytearray(span)
        wrote = mp.unpack(dt, data.tobytes(), out)
        rec["unpack"] = [wrote, sha(bytes(out))]
        # partial data: prefix semantics incl. a partial last segment
        half = total // 2 + (1 if total > 2 else 0)
        out2 = bytearray(span)
        w2 = mp.unpack(dt, data.tobytes()[:half], out2)
        rec["unpack_partial"] = [half, w2, sha(bytes(out2))]
        # overflow: full write then TruncateError
        out3 = bytearray(span)
        try:
            mp.unpack(dt, data.tobytes() + b"xyz", out3)
            rec["unpack_over"] = ["no-error", sha(bytes(out3))]
        except mp.TruncateError:
            rec["unpack_over"] = ["ERR_TRUNCATE", sha(bytes(out3))]
        # count replication (pack with count 2 when the extent keeps it in range)
        if dt.extent_bytes > 0 and lo >= 0:
            span2 = span + dt.extent_bytes
            if span2 <= max_pack_span:
                buf2 = seeded_bytes(seed + 2, span2)
                try:
                    p2 = mp.pack(dt, buf2.tobytes(), count=2)
                    rec["pack_count2"] = [span2, sha(p2), len(p2)]
                except mp.ArgError:
                    rec["pack_count2"] = [span2, "ERR_ARG", 0]
    elif nseg and lo < 0:
        try:
            mp.pack(dt, bytes(max(span, 1)))
            rec["pack_neg"] = "no-error"
        except mp.ArgError:
            rec["pack_neg"] = "ERR_ARG"
    return rec


def corpus_unit():
    out = []
    for seed in range(6):
        rng = random.Random(0xD7A0 + seed)
        for i in range(40):
            pack_safe = rng.random() < 0.8
            spec, dt = gen_type(rng, depth=4, cap=1500, pack_safe=pack_safe)
            out.append(record("unit-%d-%d" % (seed, i), spec, dt, rng,
                              seed * 1000 + i, pack_ok=pack_safe))
    return out


def corpus_crit1():
    out = []
    rng = random.Random(0x5EED)
    for i in range(1000):
        cap = 100_000 if i % 25 == 24 else 20_000
        spec, dt = gen_type(rng, depth=4, cap=cap)
        out.append(record("crit1-%d" % i, spec, dt, random.Random(i), 50_000 + i,
                          max_pack_span=1 << 20, windows=2))
    return out


FROZEN = [
    ("contiguous", 10, ("basic", 1)),
    ("vector", 3, 2, 4, ("basic", 4)),
    ("vector", 5, 3, 3, ("basic", 4)),
    ("subarray", [10, 10, 10], [4, 4, 4], [3, 3, 3], ("contiguous", 2, ("basic", 8))),
    ("subarray", [4, 6], [2, 6], [1, 0], ("basic", 4)),
    ("contiguous", 0, ("basic", 4)),
    ("struct", [2, 1], [0, 8], [("basic", 4), ("basic", 4)]),
    ("indexed_block", 2, [0, 2, 7], ("basic", 4)),
    ("contiguous", 3, ("resized", 0, 12, ("contiguous", 2, ("basic", 4)))),
    ("vector", 3, 1, -2, ("basic", 4)),
    ("vector", 2, 1, 4, ("basic", 4)),
    ("subarray", [1000, 1000, 1000], [100, 100, 100], [300, 300, 300],
     ("contiguous", 2, ("basic", 8))),
    ("indexed", [3, 1, 2], [0, 5, 6], ("basic", 4)),
    ("indexed", [2, 2], [4, 0], ("basic", 8)),
    ("vector", 4, 1, 3, ("basic", 4)),
    ("vector", 50, 1, 2, ("basic", 4)),
]


def corpus_frozen():
    out = []
    for i, spec in enumerate(FROZEN):
        dt = build_ref(spec)
        big = dt.segment_count > 100_000 or (dt._layout.max_end if dt.segment_count else 0) > (1 << 24)
        out.append(record("frozen-%d" % i, spec, dt, random.Random(i), 90_000 + i,
                          pack_ok=not big, full_iov=not big, windows=4))
    return out


def corpus_configs():
    out = []
    # cfg1: vector(4096, 4, 8, FLOAT64) over 32768 doubles
    dt = build_ref(CFG1_SPEC)
    out.append(record("cfg1", CFG1_SPEC, dt, random.Random(1), 1,
                      max_pack_span=1 << 20, windows=4))
    # cfg2: 12 halo faces of the 514^3 float32 array.  Pack digests are over
    # the seeded array bytes (seeded_bytes(2, 514**3 * 4)).
    arr = seeded_bytes(2, 514 ** 3 * 4).tobytes()
    for name, spec in cfg2_faces():
        dt = build_ref(spec)
        rec = record("cfg2-" + name, spec, dt, random.Random(hash(name) & 0xffff),
                     3, pack_ok=False, windows=4)
        rec["pack_sha_array2"] = sha(mp.pack(dt, arr))
        out.append(rec)
        print("  cfg2", name, dt.segment_count, flush=True)
    # cfg3 reduced (hvector count 4) for full pack parity, seed 3
    spec_small = cfg3_spec(3, hcount=4)
    dt = build_ref(spec_small)
    out.append(record("cfg3-h4", spec_small, dt, random.Random(3), 4,
                      max_pack_span=1 << 26, windows=4))
    # cfg3 full (hvector count 256): structure, counts, iov_len and windows
    spec_full = cfg3_spec(3, hcount=256)
    dt = build_ref(spec_full)
    out.append(record("cfg3", spec_full, dt, random.Random(33), 5, pack_ok=False,
                      full_iov=False, windows=6))
    return out


def allreduce_golden():
    """Reference host allreduce (comm.py:560-595) at 2 and 4 in-proc ranks."""
    res = []
    for n in (2, 4):
        for dtype_name in ("int64", "float64"):
            count = 1000
            rng = np.random.default_rng(77 + n)
            if dtype_name == "int64":
                bufs = [rng.integers(-2 ** 20, 2 ** 20, count, dtype=np.int64) for _ in range(n)]
                dt = mp.INT64
            else:
                bufs = [rng.uniform(-1, 1, count) for _ in range(n)]
                dt = mp.FLOAT64
            outs = [None] * n
            group = "golden-ar-%d-%s" % (n, dtype_name)

            def body(rank):
                inst = mp.init(transport="inproc", rank=rank, ranks=n, group=group)
                rb = bytearray(count * 8)
                mp.allreduce(inst.world, bufs[rank].tobytes(), rb, count, dt)
                outs[rank] = bytes(rb)
                inst.finalize()

            th = [threading.Thread(target=body, args=(r,)) for r in range(n)]
            for t in th:
                t.start()
            for t in th:
                t.join()
            assert all(o == outs[0] for o in outs)
            res.append({"n": n, "dtype": dtype_name, "count": count, "seed": 77 + n,
                        "sha": sha(outs[0]),
                        "head": list(np.frombuffer(outs[0], dtype=bufs[0].dtype)[:4].tolist())})
    return res


def main():
    out = {}
    print("frozen", flush=True)
    out["frozen"] = corpus_frozen()
    print("unit", flush=True)
    out["unit"] = corpus_unit()
    print("configs", flush=True)
    out["configs"] = corpus_configs()
    print("allreduce", flush=True)
    out["allreduce"] = allreduce_golden()
    print("crit1", flush=True)
    out["crit1"] = corpus_crit1()
    for key, val in out.items():
        path = os.path.join(HERE, "%s.json.gz" % key)
        with gzip.open(path, "wt") as f:
            json.dump(val, f, separators=(",", ":"))
        print(key, len(val), os.path.getsize(path))


if __name__ == "__main__":
    main()
