"""GPU parity of the datatype hot path (libmpx.so kernels) against the
reference's golden vectors and the CPU oracle.  Bit-exact everywhere.

Covers: type_iov (full list digest + windows), pack, unpack (full, partial
prefix, overflow -> TruncateError after filling), count replication, the
BASELINE configs at full size (cfg1, 12 cfg2 halo faces of a 514^3 f32
array, cfg3 = hvector(256) of indexed(2048) of a resized-40 struct), fused
multi-face pack/unpack, host-buffer staging, and the reference's error
cases (test_datatype.py:288-310).
"""

import numpy as np
import pytest
import torch

import oracle
import paper_2402_12274_b200 as mp
from paper_2402_12274_b200 import ArgError, TruncateError
from conftest import load_golden, to_tuple_spec
from golden_common import (CFG1_SPEC, cfg2_faces, cfg3_spec, iov_digest,
                           seeded_bytes, sha)
from specbuild import build_product

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def dev_bytes(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def check_record_gpu(rec):
    dt = build_product(to_tuple_spec(rec["spec"]), mp)
    name = rec["name"]
    if "iov_sha" in rec:
        iov = host(mp.type_iov_tensor(dt))
        assert iov_digest(iov) == rec["iov_sha"], name
    for off, ml, n, dig, _ in rec["windows"]:
        w = host(mp.type_iov_tensor(dt, off, ml))
        assert len(w) == n and iov_digest(w) == dig, (name, off, ml)
    span, total = rec["span"], rec["size"]
    if "pack_sha" in rec:
        buf = dev_bytes(seeded_bytes(rec["seed"], span))
        assert sha(host(mp.pack(dt, buf))) == rec["pack_sha"], name
        data = dev_bytes(seeded_bytes(rec["seed"] + 1, total))
        out = torch.zeros(max(span, 1), dtype=torch.uint8, device=DEV)[:span]
        wrote = mp.unpack(dt, data, out)
        assert [wrote, sha(host(out))] == rec["unpack"], name
        half, w2, dig2 = rec["unpack_partial"]
        out2 = torch.zeros(max(span, 1), dtype=torch.uint8, device=DEV)[:span]
        assert mp.unpack(dt, data[:half], out2) == w2, name
        assert sha(host(out2)) == dig2, name
        err, dig3 = rec["unpack_over"]
        out3 = torch.zeros(max(span, 1), dtype=torch.uint8, device=DEV)[:span]
        over = torch.cat([data, torch.tensor([120, 121, 122], dtype=torch.uint8, device=DEV)])
        with pytest.raises(TruncateError):
            mp.unpack(dt, over, out3)
        assert err == "ERR_TRUNCATE" and sha(host(out3)) == dig3, name
    if "pack_count2" in rec:
        span2, dig, ln = rec["pack_count2"]
        buf2 = dev_bytes(seeded_bytes(rec["seed"] + 2, span2))
        if dig == "ERR_ARG":
            with pytest.raises(ArgError):
                mp.pack(dt, buf2, count=2)
        else:
            p2 = host(mp.pack(dt, buf2, count=2))
            assert len(p2) == ln and sha(p2) == dig, name
    if "pack_neg" in rec:
        with pytest.raises(ArgError):
            mp.pack(dt, torch.zeros(max(span, 1), dtype=torch.uint8, device=DEV))
    if dt not in mp.datatypes.BUILTINS:
        mp.type_free(dt)


@pytest.mark.parametrize("corpus", ["frozen", "unit", "crit1"])
def test_gpu_matches_reference_corpus(corpus):
    for rec in load_golden(corpus):
        check_record_gpu(rec)


def test_gpu_configs_golden():
    for rec in load_golden("configs"):
        if rec["name"] in ("cfg3",):
            continue
        check_record_gpu(rec)


def test_gpu_cfg2_faces_full_array():
    """All 12 halo faces of the seeded 514^3 f32 array, single and fused."""
    arr_h = seeded_bytes(2, 514 ** 3 * 4)
    arr = dev_bytes(arr_h)
    recs = {r["name"]: r for r in load_golden("configs")}
    faces = cfg2_faces()
    dts = [build_product(s, mp) for _, s in faces]
    outs = []
    for (name, _), dt in zip(faces, dts):
        p = mp.pack(dt, arr)
        assert sha(host(p)) == recs["cfg2-" + name]["pack_sha_array2"], name
        outs.append(p)
    fused = [torch.empty_like(o) for o in outs]
    mp.pack_multi(dts, [arr] * len(dts), fused)
    for o, f in zip(outs, fused):
        assert torch.equal(o, f)
    # unpack every face into a zero array, then compare against the oracle
    dst = torch.zeros_like(arr)
    mp.unpack_multi(dts, outs, [dst] * len(dts))
    ref = np.zeros_like(arr_h)
    for (name, spec), o in zip(faces, outs):
        oracle.OracleType(spec).unpack(host(o), ref)
    assert sha(host(dst)) == sha(ref)


def test_gpu_cfg1_roundtrip_float64():
    rng = np.random.default_rng(1)
    src = rng.uniform(-1, 1, 32768)
    dt = build_product(CFG1_SPEC, mp)
    t = torch.from_numpy(src).to(DEV)
    packed = mp.pack(dt, t)
    assert packed.numel() == 131072
    ot = oracle.OracleType(CFG1_SPEC)
    assert sha(host(packed)) == sha(ot.pack(src.view(np.uint8)))
    back = torch.zeros_like(t)
    assert mp.unpack(dt, packed, back) == 131072
    exp = np.zeros_like(src)
    ot.unpack(host(packed), exp.view(np.uint8))
    assert np.array_equal(host(back), exp)
    iov = host(mp.type_iov_tensor(dt))
    assert iov.shape == (4096, 2) and (iov[:, 1] == 32).all()
    assert (iov[:, 0] == np.arange(4096) * 64).all()


@pytest.mark.parametrize("hcount", [8, 256])
def test_gpu_cfg3_full_size(hcount):
    """cfg3 against the oracle: iov digest, pack, unpack round trip."""
    spec = cfg3_spec(3, hcount=hcount)
    dt = build_product(spec, mp)
    ot = oracle.OracleType(spec)
    span = ot.max_end
    src_h = seeded_bytes(5, span)
    src = dev_bytes(src_h)
    packed = mp.pack(dt, src)
    ref = ot.pack(src_h)
    assert packed.numel() == ref.size
    assert sha(host(packed)) == sha(ref)
    out = torch.zeros_like(src)
    assert mp.unpack(dt, packed, out) == ref.size
    exp = np.zeros(span, np.uint8)
    ot.unpack(ref, exp)
    assert sha(host(out)) == sha(exp)
    iov = host(mp.type_iov_tensor(dt))
    assert iov_digest(iov) == iov_digest(ot.iov())
    if hcount == 256:
        rec = [r for r in load_golden("configs") if r["name"] == "cfg3"][0]
        for off, ml, n, dig, _ in rec["windows"]:
            w = host(mp.type_iov_tensor(dt, off, ml))
            assert len(w) == n and iov_digest(w) == dig


def test_gpu_host_buffers_reference_contract():  # test_datatype.py:288-310
    dt = mp.type_vector(2, 1, 4, mp.INT32).commit()
    with pytest.raises(ArgError):
        mp.pack(dt, bytes(19))
    out = mp.pack(dt, bytes(range(20)))
    assert out == bytes([0, 1, 2, 3, 16, 17, 18, 19])
    with pytest.raises(ArgError):
        mp.unpack(dt, out, bytes(20))
    c4 = mp.type_contiguous(4, mp.BYTE).commit()
    buf = bytearray(4)
    with pytest.raises(TruncateError):
        mp.unpack(c4, b"\x01\x02\x03\x04\x05", buf)
    assert bytes(buf) == b"\x01\x02\x03\x04"
    b16 = bytes(range(16))
    assert mp.pack(mp.INT32, b16, count=4) == b16
    segs, n = mp.type_iov(mp.type_vector(3, 2, 4, mp.INT32).commit(), 1, 10)
    assert n == 2 and [(s.base_offset, s.length) for s in segs] == [(16, 8), (32, 8)]
    e = mp.type_contiguous(0, mp.INT32).commit()
    assert mp.pack(e, b"") == b""
    assert mp.type_iov(e, 0, -1) == ([], 0)


def test_gpu_overlapping_unpack_last_writer_wins():
    """vector with negative stride over overlapping blocks: sequential order."""
    dt = mp.type_create_struct([4, 4], [0, 2], [mp.BYTE, mp.BYTE]).commit()
    assert dt.layout_query()["overlap"] == 1
    data = torch.arange(8, dtype=torch.uint8, device=DEV)
    out = torch.zeros(6, dtype=torch.uint8, device=DEV)
    mp.unpack(dt, data, out)
    assert host(out).tolist() == [0, 1, 4, 5, 6, 7]


def test_gpu_pinned_host_zero_copy():
    """Pinned CPU tensors are addressed by the kernels directly (UVA)."""
    specs = [("subarray", [40, 40, 40], [38, 38, 1], [1, 1, 1], ("basic", 4)),
             ("subarray", [40, 40, 40], [8, 38, 38], [31, 1, 1], ("basic", 4)),
             cfg3_spec(3, hcount=2, nblocks=64)]
    for spec in specs:
        dt = build_product(spec, mp)
        ot = oracle.OracleType(spec)
        span = ot.max_end
        src_h = seeded_bytes(9, span)
        pinned = torch.from_numpy(src_h).pin_memory()
        packed = mp.pack(dt, pinned)
        assert not packed.is_cuda and packed.is_pinned()
        ref = ot.pack(src_h)
        assert np.array_equal(packed.numpy(), ref)
        out = torch.zeros(span, dtype=torch.uint8).pin_memory()
        assert mp.unpack(dt, packed, out) == ref.size
        exp = np.zeros(span, np.uint8)
        ot.unpack(ref, exp)
        assert np.array_equal(out.numpy(), exp)
        # fused multi with mixed device / pinned operands
        outs = [torch.empty(ref.size, dtype=torch.uint8, device=DEV)]
        mp.pack_multi([dt], [pinned], outs)
        assert np.array_equal(host(outs[0]), ref)


SPAN_SPECS = [
    cfg3_spec(5, hcount=3, nblocks=48),
    ("hvector", 7, 2, 300, ("resized", 0, 36, ("struct", [2, 2, 1], [0, 5, 20],
                                                 [("basic", 1), ("basic", 4), ("basic", 1)]))),
    ("indexed", [5, 1, 9, 3], [0, 7, 9, 30], ("resized", 0, 12, ("struct", [1, 2], [0, 6],
                                                                  [("basic", 4), ("basic", 1)]))),
]


@pytest.mark.parametrize("spec", SPAN_SPECS)
@pytest.mark.parametrize("src_off", [0, 1, 2, 3, 5, 13])
def test_gpu_span_plans_every_address_phase(spec, src_off):
    """k_perm's phase tables (and the run-table kernel): layout and packed
    buffers at every offset mod 4 (and mod 16), pack + full / short unpack
    against the oracle."""
    dt = build_product(spec, mp)
    ot = oracle.OracleType(spec)
    # span plan (k_perm), or the flat run table when no word-gather form exists
    assert dt.layout_query()["plan"] in (3, 4)
    span, total = ot.max_end, ot.size_bytes
    src_h = seeded_bytes(17 + src_off, span)
    base = torch.zeros(span + 64, dtype=torch.uint8, device=DEV)
    src = base[src_off:src_off + span]
    src.copy_(torch.from_numpy(src_h))
    ref = ot.pack(src_h)
    for pk_off in (0, 1, 2, 3, 7):
        pbuf = torch.zeros(total + 16, dtype=torch.uint8, device=DEV)
        out = pbuf[pk_off:pk_off + total]
        mp.pack_into(dt, src, out)
        assert np.array_equal(host(out), ref), (src_off, pk_off)
        assert not host(pbuf[:pk_off]).any() and not host(pbuf[pk_off + total:]).any()
        dbase = torch.full((span + 64,), 0xAB, dtype=torch.uint8, device=DEV)
        dst = dbase[src_off:src_off + span]
        for cut in (total, total // 3, 1):
            dbase.fill_(0xAB)
            assert mp.unpack(dt, out[:cut], dst) == cut
            exp = np.full(span, 0xAB, np.uint8)
            ot.unpack(ref[:cut], exp)
            got = host(dbase)
            assert np.array_equal(got[src_off:src_off + span], exp), (src_off, pk_off, cut)
            assert (got[:src_off] == 0xAB).all() and (got[src_off + span:] == 0xAB).all()


def _irregular_indexed(seed, nblk, blmax, gapmax, elem):
    rng = np.random.default_rng(seed)
    bls = rng.integers(1, blmax + 1, nblk)
    gaps = rng.integers(0, gapmax + 1, nblk)
    displs = np.cumsum(gaps + np.concatenate([[0], bls[:-1]]))
    return ("indexed", [int(x) for x in bls], [int(x) for x in displs], ("basic", elem))


@pytest.mark.parametrize("spec", [
    _irregular_indexed(1, 5000, 4, 8, 8),       # thread per run
    _irregular_indexed(2, 3000, 16, 64, 4),
    _irregular_indexed(3, 800, 64, 32, 8),      # warp per run (long runs)
    _irregular_indexed(4, 4000, 3, 5, 1),       # byte runs, 1-byte words
])
@pytest.mark.parametrize("off", [0, 3])
def test_gpu_run_table_plans(spec, off):
    """Irregular indexed types (many short blocks) take the flat run table:
    pack, full / short unpack and iov windows against the oracle, at an
    aligned and a misaligned buffer offset."""
    dt = build_product(spec, mp)
    ot = oracle.OracleType(spec)
    assert dt.layout_query()["plan"] == 4
    span, total = ot.max_end, ot.size_bytes
    src_h = seeded_bytes(31 + off, span)
    base = torch.zeros(span + 32, dtype=torch.uint8, device=DEV)
    src = base[off:off + span]
    src.copy_(torch.from_numpy(src_h))
    ref = ot.pack(src_h)
    out = mp.pack(dt, src)
    assert np.array_equal(host(out), ref)
    for cut in (total, total // 2 + 3):
        dbase = torch.full((span + 32,), 7, dtype=torch.uint8, device=DEV)
        dst = dbase[off:off + span]
        assert mp.unpack(dt, out[:cut], dst) == cut
        exp = np.full(span, 7, np.uint8)
        ot.unpack(ref[:cut], exp)
        got = host(dbase)
        assert np.array_equal(got[off:off + span], exp)
        assert (got[:off] == 7).all() and (got[off + span:] == 7).all()
    iov = ot.iov()
    assert np.array_equal(host(mp.type_iov_tensor(dt)), iov)
    assert np.array_equal(host(mp.type_iov_tensor(dt, 17, 100)), iov[17:117])


def test_gpu_pack_unpack_capture_in_cuda_graph():
    """Once its plan exists, pack/unpack is stream-capture safe: a CUDA graph
    of the fused multi-face step replays to the same bytes."""
    specs = [("subarray", [40, 40, 40], [38, 38, 1], [1, 1, 1], ("basic", 4)),
             ("subarray", [40, 40, 40], [8, 38, 38], [31, 1, 1], ("basic", 4))]
    dts = [build_product(s, mp) for s in specs]
    src = dev_bytes(seeded_bytes(41, 40 ** 3 * 4))
    dst = torch.zeros_like(src)
    outs = [torch.empty(mp.packed_size(d), dtype=torch.uint8, device=DEV) for d in dts]
    cfg3 = build_product(cfg3_spec(6, hcount=2, nblocks=32), mp)
    csrc = dev_bytes(seeded_bytes(42, oracle.OracleType(cfg3_spec(6, hcount=2, nblocks=32)).max_end))
    cout = torch.empty(mp.packed_size(cfg3), dtype=torch.uint8, device=DEV)
    cback = torch.zeros_like(csrc)

    def step():
        mp.pack_multi(dts, [src] * 2, outs)
        mp.unpack_multi(dts, outs, [dst] * 2)
        mp.pack_into(cfg3, csrc, cout)
        mp.unpack(cfg3, cout, cback)

    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        step()                        # builds and uploads the plans
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
    ref = [host(o).copy() for o in outs] + [host(cout).copy()]
    for o in outs + [cout]:
        o.zero_()
    dst.zero_()
    cback.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert all(np.array_equal(host(o), r) for o, r in zip(outs + [cout], ref))
    exp = np.zeros(40 ** 3 * 4, np.uint8)
    for spec, r in zip(specs, ref):
        oracle.OracleType(spec).unpack(r, exp)
    assert np.array_equal(host(dst), exp)
    cexp = np.zeros_like(host(csrc))
    oracle.OracleType(cfg3_spec(6, hcount=2, nblocks=32)).unpack(ref[-1], cexp)
    assert np.array_equal(host(cback), cexp)


def test_gpu_layouts_beyond_32_bit_indices():
    """More than 2^31 rows / bytes: the chain kernels' 64-bit index paths and
    the iov of a > 4 GiB layout, checked against strided torch views."""
    free, _ = torch.cuda.mem_get_info()
    if free < (24 << 30):
        pytest.skip("needs 24 GiB of free device memory")
    rows = (1 << 31) + 3                                     # > 2^31 rows of 1 byte, stride 2
    dt = mp.type_vector(rows, 1, 2, mp.BYTE).commit()
    src = torch.randint(0, 256, (2 * rows,), dtype=torch.uint8, device=DEV)
    out = torch.empty(rows, dtype=torch.uint8, device=DEV)
    mp.pack_into(dt, src, out)
    assert torch.equal(out, src.view(-1, 2)[:, 0])
    back = torch.zeros_like(src)
    assert mp.unpack(dt, out, back) == rows
    assert torch.equal(back.view(-1, 2)[:, 0], out) and not back.view(-1, 2)[:, 1].any()
    iov = mp.type_iov_tensor(dt, rows - 5, 5).cpu().numpy()
    assert [tuple(x) for x in iov] == [(2 * (rows - 5 + i), 1) for i in range(5)]
    del src, out, back
    # a 4-byte-word layout whose packed offsets pass 2^32
    n = (1 << 30) + 7
    dt4 = mp.type_vector(n, 1, 3, mp.INT32).commit()        # packed 4 GiB + 28 B, span 12 GiB
    src = torch.arange(3 * n, dtype=torch.int32, device=DEV)
    out = torch.empty(n, dtype=torch.int32, device=DEV)
    mp.pack_into(dt4, src, out)
    assert torch.equal(out, src.view(-1, 3)[:, 0])
