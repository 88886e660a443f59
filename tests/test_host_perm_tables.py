"""CPU check of the span lowering's word-gather tables (no GPU): the plan of
each type is dumped (mpx_plan_dump) and replayed by tests/perm_emu.py exactly
as k_perm consumes it, at every (layout, packed) address phase mod 4 and for
short unpacks, against the oracle.  Covers word-window specs (cfg3-like
structs) and per-byte specs (structs whose padding spreads a word's bytes
over more than 16 input bytes)."""

import numpy as np
import pytest

import oracle
import paper_2402_12274_b200 as mp
import perm_emu
from golden_common import cfg3_spec
from specbuild import build_product


def wide_struct_array(ext):
    st = ("struct", [1, 3, 1], [0, 8, 32], [("basic", 4), ("basic", 8), ("basic", 1)])
    return ("hvector", 3, 1, 7000, ("indexed", [5, 1, 9, 33], [0, 7, 9, 30], ("resized", 0, ext, st)))


SPECS = [
    cfg3_spec(7, hcount=2, nblocks=24),                       # word windows
    wide_struct_array(56),                                    # per-byte gathers (tail padding 23 B)
    wide_struct_array(64),
    ("indexed_block", 3, [3, 9, 14, 22, 28, 47],
     ("subarray", [8, 10, 3], [6, 7, 3], [2, 2, 0], ("basic", 1))),
    ("hvector", 5, 40, 1900, ("resized", 0, 44, ("struct", [2, 1], [0, 20], [("basic", 8), ("basic", 4)]))),
]


@pytest.mark.parametrize("spec", SPECS)
def test_perm_tables_replay_matches_oracle(spec):
    dt = build_product(spec, mp)
    plan = perm_emu.dump(mp, dt, 1)
    assert plan["kind"] == 3 and plan["specs"], "expected a span plan with word-gather specs"
    ot = oracle.OracleType(spec)
    span, total = ot.max_end, ot.size_bytes
    src = np.random.default_rng(3).integers(0, 256, span, dtype=np.uint8)
    ref = ot.pack(src)
    for la in range(4):
        for pa in range(4):
            out = np.zeros(total, np.uint8)
            perm_emu.run(plan, True, src, out, src_addr=la, dst_addr=pa)
            assert np.array_equal(out, ref), ("pack", la, pa)
            for cut in (total, total // 3 + 1):
                exp = np.full(span, 0x77, np.uint8)
                ot.unpack(ref[:cut], exp)
                got = np.full(span, 0x77, np.uint8)
                perm_emu.run(plan, False, ref, got, src_addr=pa, dst_addr=la, limit=cut)
                assert np.array_equal(got, exp), ("unpack", la, pa, cut)


def test_byte_form_used_for_wide_padding():
    plan = perm_emu.dump(mp, build_product(wide_struct_array(64), mp), 1)
    assert any(s["bytes"] for s in plan["specs"])
    plan = perm_emu.dump(mp, build_product(cfg3_spec(7, hcount=2, nblocks=24), mp), 1)
    assert not any(s["bytes"] for s in plan["specs"])
