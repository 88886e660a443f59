"""Pin the CPU oracle (oracle/dt_oracle.c) to the real reference.

Golden vectors were produced by the unmodified Python reference
(tests/golden/make_golden.py).  Every field recorded there must be reproduced
by the oracle: attributes, iov_len budgets, full iov digests, iov windows,
pack / unpack (full, partial, overflow) digests, count replication.
CPU only.
"""

import numpy as np
import pytest

import oracle
from conftest import load_golden, to_tuple_spec
from golden_common import iov_digest, seeded_bytes, sha


@pytest.fixture(scope="module", autouse=True)
def _fresh_oracle():
    oracle.build()
    oracle.reset()
    yield
    oracle.reset()


def check_record(rec, big_array=None):
    spec = to_tuple_spec(rec["spec"])
    t = oracle.OracleType(spec)
    name = rec["name"]
    assert (t.size_bytes, t.lb, t.ub, t.extent_bytes) == \
        (rec["size"], rec["lb"], rec["ub"], rec["extent"]), name
    assert t.segment_count == rec["segments"], name
    assert t.node_count == rec["node_count"], name
    for budget, expect in rec["iov_len"]:
        assert list(t.iov_len(budget)) == expect, (name, budget)
    if "iov_sha" in rec:
        iov = t.iov()
        assert iov_digest(iov) == rec["iov_sha"], name
        if "iov" in rec:
            assert iov.tolist() == rec["iov"], name
    for off, ml, n, dig, sample in rec["windows"]:
        w = t.iov(off, ml)
        assert len(w) == n and iov_digest(w) == dig, (name, off, ml)
    span = rec["span"]
    total = rec["size"]
    if "pack_sha" in rec:
        buf = seeded_bytes(rec["seed"], span)
        assert sha(t.pack(buf)) == rec["pack_sha"], name
        data = seeded_bytes(rec["seed"] + 1, total)
        out = np.zeros(span, np.uint8)
        wrote, tr = t.unpack(data, out)
        assert [wrote, sha(out)] == rec["unpack"] and not tr, name
        half, w2, dig2 = rec["unpack_partial"]
        out2 = np.zeros(span, np.uint8)
        got2, tr2 = t.unpack(data[:half], out2)
        assert (got2, sha(out2)) == (w2, dig2) and not tr2, name
        err, dig3 = rec["unpack_over"]
        out3 = np.zeros(span, np.uint8)
        _, tr3 = t.unpack(np.concatenate([data, np.frombuffer(b"xyz", np.uint8)]), out3)
        assert sha(out3) == dig3 and tr3 == (err == "ERR_TRUNCATE"), name
    if "pack_count2" in rec:
        span2, dig, ln = rec["pack_count2"]
        buf2 = seeded_bytes(rec["seed"] + 2, span2)
        if dig == "ERR_ARG":
            with pytest.raises(ValueError):
                t.pack(buf2, count=2)
        else:
            p2 = t.pack(buf2, count=2)
            assert len(p2) == ln and sha(p2) == dig, name
    if "pack_neg" in rec:
        assert rec["pack_neg"] == "ERR_ARG"
        with pytest.raises(ValueError):
            t.pack(np.zeros(max(span, 1), np.uint8))
    if big_array is not None and "pack_sha_array2" in rec:
        assert sha(t.pack(big_array)) == rec["pack_sha_array2"], name


@pytest.mark.parametrize("corpus", ["frozen", "unit"])
def test_oracle_matches_reference_corpus(corpus):
    for rec in load_golden(corpus):
        check_record(rec)


def test_oracle_matches_reference_crit1_corpus():
    for rec in load_golden("crit1"):
        check_record(rec)


def test_oracle_matches_reference_configs():
    recs = load_golden("configs")
    arr = seeded_bytes(2, 514 ** 3 * 4)
    for rec in recs:
        check_record(rec, big_array=arr)


def test_oracle_allreduce_matches_reference():
    for g in load_golden("allreduce"):
        rng = np.random.default_rng(g["seed"])
        n, count = g["n"], g["count"]
        if g["dtype"] == "int64":
            bufs = [rng.integers(-2 ** 20, 2 ** 20, count, dtype=np.int64) for _ in range(n)]
        else:
            bufs = [rng.uniform(-1, 1, count) for _ in range(n)]
        out = oracle.allreduce_sum(bufs)
        assert sha(out.tobytes()) == g["sha"]
