"""Host-side logic of the product (no GPU): the C ABI loads and exports every
symbol of include/mpx.h, the C++ typerep compiler reproduces the reference's
attributes, segment counts, node counts and type_iov_len answers on every
golden type, and argument / lifecycle errors match the reference
(test_datatype.py:243-319)."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2402_12274_b200 as mp
from paper_2402_12274_b200 import ArgError, _lib
from conftest import ROOT, load_golden, to_tuple_spec
from specbuild import build_product


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "mpx.h")).read()
    declared = set(re.findall(r"\b(mpx_[a-z0-9_]+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    lib = ctypes.CDLL(_lib.SO_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), name
    # the Python binding covers the whole header
    assert declared <= set(_lib.exported_symbols()) | {"mpx_last_error"}


@pytest.mark.parametrize("corpus", ["frozen", "unit", "crit1", "configs"])
def test_host_attributes_match_reference(corpus):
    for rec in load_golden(corpus):
        dt = build_product(to_tuple_spec(rec["spec"]), mp)
        name = rec["name"]
        assert (dt.size_bytes, dt.lb, dt.ub, dt.extent_bytes) == \
            (rec["size"], rec["lb"], rec["ub"], rec["extent"]), name
        assert dt.segment_count == rec["segments"], name
        assert dt.node_count == rec["node_count"], name
        for budget, expect in rec["iov_len"]:
            assert list(mp.type_iov_len(dt, budget)) == expect, (name, budget)
        q = dt.layout_query()
        assert q["runs"] == rec["segments"]
        if rec["segments"]:
            assert q["min_off"] == rec["min_off"], name
            if rec["min_off"] >= 0 and "iov_sha" in rec:
                assert q["max_end"] == rec["span"], name
        if dt not in mp.datatypes.BUILTINS:
            mp.type_free(dt)


def test_config_plans():
    """The named BASELINE configs lower to the intended kernels."""
    from golden_common import CFG1_SPEC, cfg2_faces, cfg3_spec
    q = build_product(CFG1_SPEC, mp).layout_query()
    assert q["plan"] == 1 and q["chain_align"] == 16 and not q["overlap"]
    for name, spec in cfg2_faces():
        q = build_product(spec, mp).layout_query()
        assert q["plan"] == 1 and not q["overlap"], name
    q = build_product(cfg3_spec(3, hcount=8), mp).layout_query()
    assert q["plan"] == 3 and not q["overlap"]      # span lowering
    assert q["chain_align"] > 0                     # ... with word-gather specs (k_perm)
    # irregular indexed blocks (many short runs): the flat run table
    rng = np.random.default_rng(5)
    bls = rng.integers(1, 5, 20000)
    displs = np.cumsum(rng.integers(0, 9, 20000) + np.concatenate([[0], bls[:-1]]))
    dt = mp.type_indexed([int(x) for x in bls], [int(x) for x in displs], mp.FLOAT64).commit()
    assert dt.layout_query()["plan"] == 4


def test_frozen_examples_host():
    dt = mp.type_vector(3, 2, 4, mp.INT32).commit()
    assert (dt.size_bytes, dt.extent_bytes, dt.segment_count) == (24, 40, 3)
    elem = mp.type_contiguous(2, mp.FLOAT64).commit()
    big = mp.type_create_subarray([1000] * 3, [100] * 3, [300] * 3, elem).commit()
    assert mp.type_iov_len(big, -1) == (10000, 16_000_000)
    assert mp.type_iov_len(big, 3200) == (2, 3200)
    assert big.node_count <= 8
    e = mp.type_contiguous(0, mp.INT32).commit()
    assert mp.type_iov_len(e, 100) == (0, 0)
    ix = mp.type_indexed([3, 1, 2], [0, 5, 6], mp.INT32).commit()
    assert ix.size_bytes == 24 and ix.segment_count == 2


def test_queries_require_commit():  # test_datatype.py:243-252
    dt = mp.type_contiguous(4, mp.INT32)
    with pytest.raises(ArgError):
        mp.type_iov_len(dt, -1)
    with pytest.raises(ArgError):
        mp.packed_size(dt)
    dt.commit()
    assert mp.type_iov_len(dt, -1) == (1, 16)


def test_uncommitted_child_rejected():  # :255-258
    inner = mp.type_contiguous(2, mp.INT32)
    with pytest.raises(ArgError):
        mp.type_contiguous(3, inner)


def test_free_lifecycle():  # :261-269
    dt = mp.type_contiguous(2, mp.INT32).commit()
    mp.type_free(dt)
    with pytest.raises(ArgError):
        mp.type_iov_len(dt, -1)
    with pytest.raises(ArgError):
        mp.type_free(dt)
    with pytest.raises(ArgError):
        mp.type_free(mp.INT32)


def test_bad_bounds_rejected():  # :272-285
    with pytest.raises(ArgError):
        mp.type_contiguous(-1, mp.BYTE)
    with pytest.raises(ArgError):
        mp.type_create_subarray([4], [5], [0], mp.BYTE)
    with pytest.raises(ArgError):
        mp.type_create_subarray([4], [2], [3], mp.BYTE)
    with pytest.raises(ArgError):
        mp.type_create_resized(mp.BYTE, 0, -2)
    with pytest.raises(ArgError):
        mp.type_contiguous(True, mp.BYTE)
    dt = mp.type_vector(3, 2, 4, mp.INT32).commit()
    with pytest.raises(ArgError):
        mp.type_iov_len(dt, -2)


def test_parse_type_expr():  # :313-319
    dt = mp.parse_type_expr("vector(3, 2, 4, int32)")
    assert dt.segment_count == 3 and dt.size_bytes == 24
    with pytest.raises(ArgError):
        mp.parse_type_expr("vector(3, 2)")
    with pytest.raises(ArgError):
        mp.parse_type_expr("__import__('os')")


def test_host_magic_division_exact():
    """The device's multiply-high division (desc.cuh host_magic/fdiv),
    emulated with Python ints, is exact on edge values."""
    def magic(d):
        if d <= 1:
            return 0, 0
        l = (d - 1).bit_length()
        return -(-(1 << (63 + l)) // d), l - 1

    def fdiv(n, m, s):
        return n if m == 0 else ((n * m) >> 64) >> s

    for d in [1, 2, 3, 5, 7, 29, 40, 64, 2056, 1056784, 3015976, 2**31 - 1,
              2**32 + 1, 2**40 + 3, 2**62 - 1, 2**62]:
        m, s = magic(d)
        assert m < 2**64
        for n in [0, 1, d - 1, d, d + 1, 2 * d - 1, 12345678901, 2**62, 2**63 - 1]:
            assert fdiv(n, m, s) == n // d, (d, n)
