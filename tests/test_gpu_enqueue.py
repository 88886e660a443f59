"""GPU tests of the enqueue path: device queues wrapping CUDA streams,
stream communicators, send/recv/isend/irecv_enqueue, wait(all)_enqueue,
deferred errors, rings over in-process ranks (several ranks share the one
GPU; ordering uses stream memory operations, never spinning kernels), typed
transfers, and allreduce parity with the reference's rank-ordered sum.

Mirrors /root/reference/pkg/tests/test_offload.py:41-210,
test_acceptance.py:550-636, test_p2p.py:114-132, test_comm.py:103-132.
"""

import time

import numpy as np
import pytest
import torch

import oracle
import paper_2402_12274_b200 as mp
from paper_2402_12274_b200 import ArgError, StateError
from twin import host, pair, unique_group

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(180)]
DEV = torch.device("cuda", 0)


@pytest.fixture
def inst():
    i = mp.init(group=unique_group("dev"), device=0)
    yield i
    if not i.finalized:
        i.finalize()


@pytest.fixture
def queue(inst):
    q = mp.queue_create(inst)
    yield q
    if not q.destroyed:
        mp.queue_destroy(q)


def device_comm(inst, queue):
    info = mp.info_create()
    mp.info_set(info, "type", "devstream")
    mp.info_set_hex(info, "value", bytes.fromhex(queue.handle))
    s = inst.stream_create(info)
    return mp.stream_comm_create(inst.world, s), s


def u8(data):
    return torch.tensor(list(data), dtype=torch.uint8, device=DEV)


def test_handle_is_sixteen_hex_chars(queue):
    assert len(queue.handle) == 16
    int(queue.handle, 16)
    assert queue.handle == queue.handle.lower()


def test_queue_from_hex_normalizes(queue):
    h = queue.handle
    assert mp.queue_from_hex(h.upper()) is queue
    assert mp.queue_from_hex(h.lstrip("0")) is queue
    with pytest.raises(ArgError):
        mp.queue_from_hex("zz")
    with pytest.raises(ArgError):
        mp.queue_from_hex("f" * 17)
    with pytest.raises(ArgError):
        mp.queue_from_hex("0123456789abcdef")


def test_tasks_run_in_submission_order(queue):
    log = []
    for i in range(20):
        mp.compute_enqueue(queue, log.append, i)
    mp.queue_synchronize(queue)
    assert log == list(range(20))


def test_memcpy_enqueue_bounds_checked_at_enqueue(queue):
    dst = torch.zeros(4, dtype=torch.uint8, device=DEV)
    with pytest.raises(ArgError):
        mp.memcpy_enqueue(queue, dst, u8(b"123456"), 6)
    mp.memcpy_enqueue(queue, dst, u8(b"abcd"), 4)
    mp.queue_synchronize(queue)
    assert bytes(dst.cpu().tolist()) == b"abcd"


def test_saxpy_kernel(queue):
    x = torch.ones(8, dtype=torch.float64, device=DEV)
    y = torch.full((8,), 2.0, dtype=torch.float64, device=DEV)
    mp.compute_enqueue(queue, mp.saxpy, 2.0, x, y, 8)
    mp.queue_synchronize(queue)
    assert y.cpu().tolist() == [4.0] * 8


def test_device_comm_redirects_to_enqueue(inst, queue):
    c, s = device_comm(inst, queue)
    buf = torch.zeros(4, dtype=torch.uint8, device=DEV)
    rr = mp.irecv(c, buf, 4, mp.BYTE, 0, 1)
    sr = mp.isend(c, u8(b"wxyz"), 4, mp.BYTE, 0, 1)
    assert rr.enqueued and sr.enqueued
    with pytest.raises(ArgError):
        mp.wait(sr)
    with pytest.raises(ArgError):
        mp.waitall([rr])
    mp.wait_enqueue(sr)
    mp.wait_enqueue(rr)
    mp.queue_synchronize(queue)
    assert bytes(buf.cpu().tolist()) == b"wxyz"
    assert rr.status.count == 4 and rr.status.source == 0 and rr.status.tag == 1
    mp.comm_free(c)
    mp.free_stream(s)


def test_blocking_enqueue_is_async_on_host(inst, queue):
    c, s = device_comm(inst, queue)
    with torch.cuda.stream(queue.torch_stream):
        torch.cuda._sleep(200_000_000)          # ~0.1 s of GPU time ahead of the send
    t0 = time.perf_counter()
    mp.send(c, u8(b"pipelined"), 9, mp.BYTE, 0, 5)
    host_cost = time.perf_counter() - t0
    buf = torch.zeros(9, dtype=torch.uint8, device=DEV)
    mp.recv(c, buf, 9, mp.BYTE, 0, 5)
    assert host_cost < 0.05
    mp.queue_synchronize(queue)
    assert bytes(buf.cpu().tolist()) == b"pipelined"
    mp.comm_free(c)
    mp.free_stream(s)


def test_waitall_enqueue_same_queue_only(inst, queue):
    other = mp.queue_create(inst)
    c1, s1 = device_comm(inst, queue)
    c2, s2 = device_comm(inst, other)
    b1 = torch.zeros(1, dtype=torch.uint8, device=DEV)
    b2 = torch.zeros(1, dtype=torch.uint8, device=DEV)
    ra = mp.irecv(c1, b1, 1, mp.BYTE, 0, 7)
    rb = mp.irecv(c2, b2, 1, mp.BYTE, 0, 7)
    with pytest.raises(ArgError):
        mp.waitall_enqueue([ra, rb])
    sa = mp.isend(c1, u8(b"q"), 1, mp.BYTE, 0, 7)
    sb = mp.isend(c2, u8(b"r"), 1, mp.BYTE, 0, 7)
    mp.waitall_enqueue([ra, sa])
    mp.waitall_enqueue([rb, sb])
    mp.queue_synchronize(queue)
    mp.queue_synchronize(other)
    assert b1.item() == ord("q") and b2.item() == ord("r")
    with pytest.raises(ArgError):
        mp.wait_enqueue(object())
    for c, s in ((c1, s1), (c2, s2)):
        mp.comm_free(c)
        mp.free_stream(s)
    mp.queue_destroy(other)


def test_deferred_error_surfaces_at_synchronize(inst, queue):
    c, s = device_comm(inst, queue)
    mp.send(c, u8(b"0123456789"), 10, mp.BYTE, 0, 9)
    small = torch.zeros(2, dtype=torch.uint8, device=DEV)
    mp.recv(c, small, 2, mp.BYTE, 0, 9)
    with pytest.raises(mp.TruncateError):
        mp.queue_synchronize(queue)
    mp.queue_synchronize(queue)            # error consumed, queue usable
    assert bytes(small.cpu().tolist()) == b"01"
    mp.comm_free(c)
    mp.free_stream(s)


def test_awaited_request_error_lands_on_its_status(inst, queue):
    c, s = device_comm(inst, queue)
    rr = mp.irecv(c, torch.zeros(2, dtype=torch.uint8, device=DEV), 2, mp.BYTE, 0, 11)
    sr = mp.isend(c, u8(b"0123456789"), 10, mp.BYTE, 0, 11)
    mp.wait_enqueue(rr)
    mp.wait_enqueue(sr)
    mp.queue_synchronize(queue)
    assert rr.status.error == "ERR_TRUNCATE"
    mp.comm_free(c)
    mp.free_stream(s)


def test_destroy_drains_and_invalidates(inst):
    q = mp.queue_create(inst)
    x = torch.zeros(1 << 20, device=DEV)
    mp.compute_enqueue(q, lambda: x.add_(1.0))
    mp.queue_destroy(q)
    assert float(x[0]) == 1.0
    with pytest.raises(StateError):
        mp.compute_enqueue(q, lambda: None)
    with pytest.raises(StateError):
        mp.queue_destroy(q)


def test_cross_rank_device_pipeline():
    count = 64

    def rank0(inst):
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        x = torch.ones(count, dtype=torch.float64, device=inst.device)
        mp.send(c, x, count, mp.FLOAT64, 1, 2)
        mp.queue_synchronize(q)
        mp.comm_free(c)
        mp.free_stream(s)
        mp.queue_destroy(q)

    def rank1(inst):
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        x = torch.zeros(count, dtype=torch.float64, device=inst.device)
        y = torch.full((count,), 2.0, dtype=torch.float64, device=inst.device)
        mp.recv(c, x, count, mp.FLOAT64, 0, 2)
        mp.compute_enqueue(q, mp.saxpy, 2.0, x, y, count)
        mp.queue_synchronize(q)
        assert y.cpu().tolist() == [4.0] * count
        mp.comm_free(c)
        mp.free_stream(s)
        mp.queue_destroy(q)

    pair(rank0, rank1)


def test_criterion_09a_saxpy_pipeline_without_host_sync():
    n = 4096
    out = {}

    def device_rank(inst):
        q = mp.queue_create(inst)
        dc, s = device_comm(inst, q)
        x = torch.zeros(n, dtype=torch.float64, device=inst.device)
        y = torch.full((n,), 2.0, dtype=torch.float64, device=inst.device)
        mp.recv(dc, x, n, mp.FLOAT64, 1, 11)
        mp.compute_enqueue(q, mp.saxpy, 2.0, x, y, n)
        mp.queue_synchronize(q)
        out["y"] = y.cpu()
        mp.comm_free(dc)
        mp.free_stream(s)
        mp.queue_destroy(q)

    def host_rank(inst):
        hs = inst.stream_create()
        sc = mp.stream_comm_create(inst.world, hs)
        import array
        xs = array.array("d", [1.0] * n)
        mp.send(sc, xs, n, mp.FLOAT64, 0, 11)
        mp.comm_free(sc)
        mp.free_stream(hs)

    pair(device_rank, host_rank)
    assert bool((out["y"] == 4.0).all())


def test_criterion_09b_compute_overlaps_pending_receive():
    import threading
    gate = threading.Event()
    res = {}

    def device_rank(inst):
        q = mp.queue_create(inst)
        dc, s = device_comm(inst, q)
        buf = torch.zeros(1024, dtype=torch.float64, device=inst.device)
        rreq = mp.irecv(dc, buf, 1024, mp.FLOAT64, 1, 3)
        e_compute = torch.cuda.Event(enable_timing=True)
        e_done = torch.cuda.Event(enable_timing=True)
        mp.compute_enqueue(q, lambda: e_compute.record())
        mp.wait_enqueue(rreq)
        with torch.cuda.stream(q.torch_stream):
            e_done.record()
        gate.set()
        mp.queue_synchronize(q)
        res["gap_ms"] = e_compute.elapsed_time(e_done)
        res["payload"] = bool((buf == 2.5).all())
        mp.comm_free(dc)
        mp.free_stream(s)
        mp.queue_destroy(q)

    def delayed_sender(inst):
        hs = inst.stream_create()
        sc = mp.stream_comm_create(inst.world, hs)
        gate.wait()
        time.sleep(0.3)
        data = torch.full((1024,), 2.5, dtype=torch.float64, device=inst.device)
        mp.send(sc, data, 1024, mp.FLOAT64, 0, 3)
        mp.comm_free(sc)
        mp.free_stream(hs)

    pair(device_rank, delayed_sender)
    assert res["gap_ms"] > 200.0          # compute ran while the receive was pending
    assert res["payload"]


def test_criterion_10_stream_resource_semantics():
    cap = 6
    inst = mp.init(group=unique_group("pool"), vci_pool=cap, device=0)
    try:
        streams = [inst.stream_create() for _ in range(cap)]
        with pytest.raises(mp.ExhaustedError):
            inst.stream_create()
        for s in streams:
            mp.free_stream(s)
        for _ in range(10 * cap):
            mp.free_stream(inst.stream_create())
        # the reference refuses cudaStream_t (UnsupportedError); here it works
        ts = torch.cuda.Stream(inst.device)
        info = mp.info_create()
        mp.info_set_hex(info, "value", ts.cuda_stream)
        info.set("type", "cudaStream_t")
        s = inst.stream_create(info)
        assert s.kind == mp.CUDA_STREAM and s.cuda_stream == ts.cuda_stream
        c = mp.stream_comm_create(inst.world, s)
        buf = torch.zeros(3, dtype=torch.uint8, device=inst.device)
        mp.send(c, u8(b"abc"), 3, mp.BYTE, 0, 0)
        mp.recv(c, buf, 3, mp.BYTE, 0, 0)
        ts.synchronize()
        assert bytes(buf.cpu().tolist()) == b"abc"
        mp.comm_free(c)
        mp.free_stream(s)
    finally:
        inst.finalize()


# ------------------------------------------------------------- rings


def _ring(n, nbytes, dtype_kind, blocking=False, eager_limit=None):
    """ring r -> r+1 on n in-process ranks (rank r on cuda:(r % devices):
    one GPU -> they share it; 2+ GPUs -> NVLink peer transfers), scale
    kernels before the send and after the receive on the same stream."""
    results = [None] * n

    def body(inst):
        r = inst.rank
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        g = torch.Generator(device="cpu").manual_seed(100 + r)
        if dtype_kind == "u8":
            src = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, generator=g).to(inst.device)
            dst = torch.zeros_like(src)
            dt, count = mp.BYTE, nbytes
        else:   # vector(N/32, 4, 8) of FLOAT64 over 2N bytes
            nv = nbytes // 32
            src = torch.rand(nv * 8, dtype=torch.float64, generator=g).to(inst.device)
            dst = torch.zeros_like(src)
            dt, count = mp.type_vector(nv, 4, 8, mp.FLOAT64).commit(), 1
        with torch.cuda.stream(q.torch_stream):
            if dtype_kind != "u8":
                src.mul_(2.0)                       # dependent kernel before the send
        if blocking:
            mp.send(c, src, count, dt, (r + 1) % n, 0)
            mp.recv(c, dst, count, dt, (r - 1) % n, 0)
        else:
            rr = mp.irecv(c, dst, count, dt, (r - 1) % n, 0)
            sr = mp.isend(c, src, count, dt, (r + 1) % n, 0)
            mp.waitall_enqueue([rr, sr])
        with torch.cuda.stream(q.torch_stream):
            if dtype_kind != "u8":
                dst.mul_(0.5)                       # dependent kernel after the receive
        mp.queue_synchronize(q)
        results[r] = (src.cpu(), dst.cpu())
        mp.comm_free(c)
        mp.free_stream(s)
        mp.queue_destroy(q)

    kw = {} if eager_limit is None else {"eager_limit": eager_limit}
    host([body] * n, **kw)
    for r in range(n):
        src_prev = results[(r - 1) % n][0]
        got = results[r][1]
        if dtype_kind == "u8":
            assert torch.equal(got, src_prev)
        else:
            exp = torch.zeros_like(src_prev)
            v = src_prev.view(-1, 8)
            exp.view(-1, 8)[:, :4] = v[:, :4] * 0.5
            assert torch.equal(got, exp)


@pytest.mark.parametrize("n", [2, 3, 8])
@pytest.mark.parametrize("nbytes", [8, 1 << 16, 1 << 20])
@pytest.mark.parametrize("kind", ["u8", "vector"])
def test_ring_nonblocking(n, nbytes, kind):
    if kind == "vector" and nbytes < 32:
        pytest.skip("vector type needs >= 32 bytes")
    _ring(n, nbytes, kind)


def test_ring_blocking_within_eager_limit():
    _ring(2, 1 << 16, "u8", blocking=True)


def test_ring_blocking_large_with_raised_eager_limit():
    _ring(2, 1 << 20, "vector", blocking=True, eager_limit=1 << 21)


def test_any_source_any_tag_and_fifo_order():
    def rank0(inst):
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        mp.send(c, u8(b"A"), 1, mp.BYTE, 1, 5)
        mp.send(c, u8(b"B"), 1, mp.BYTE, 1, 5)
        mp.send(c, u8(b"C"), 1, mp.BYTE, 1, 9)
        mp.queue_synchronize(q)
        mp.comm_free(c)
        mp.free_stream(s)

    def rank1(inst):
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        got = [torch.zeros(1, dtype=torch.uint8, device=inst.device) for _ in range(3)]
        r0 = mp.irecv(c, got[0], 1, mp.BYTE, mp.ANY_SOURCE, 9)
        r1 = mp.irecv(c, got[1], 1, mp.BYTE, 0, mp.ANY_TAG)
        r2 = mp.irecv(c, got[2], 1, mp.BYTE, mp.ANY_SOURCE, mp.ANY_TAG)
        mp.waitall_enqueue([r0, r1, r2])
        mp.queue_synchronize(q)
        assert [chr(int(g.item())) for g in got] == ["C", "A", "B"]
        assert (r0.status.source, r0.status.tag) == (0, 9)
        assert r1.status.tag == 5 and r2.status.tag == 5
        mp.comm_free(c)
        mp.free_stream(s)

    pair(rank0, rank1)


def test_typed_transfer_vector_to_contiguous():   # test_p2p.py:114-132
    def rank0(inst):
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        src = torch.arange(12, dtype=torch.int32, device=inst.device)
        vt = mp.type_vector(4, 1, 3, mp.INT32).commit()
        mp.send(c, src, 1, vt, 1, 0)
        back = torch.zeros(12, dtype=torch.int32, device=inst.device)
        mp.recv(c, back, 1, vt, 1, 1)
        mp.queue_synchronize(q)
        assert back.cpu().tolist() == [0, 0, 0, 3, 0, 0, 6, 0, 0, 9, 0, 0]
        mp.comm_free(c)
        mp.free_stream(s)

    def rank1(inst):
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        dst = torch.zeros(4, dtype=torch.int32, device=inst.device)
        rr = mp.irecv(c, dst, 4, mp.INT32, 0, 0)
        mp.wait_enqueue(rr)
        mp.send(c, dst, 4, mp.INT32, 0, 1)
        mp.queue_synchronize(q)
        assert dst.cpu().tolist() == [0, 3, 6, 9]
        assert rr.status.count == 4
        mp.comm_free(c)
        mp.free_stream(s)

    pair(rank0, rank1)


def test_zipper_typed_to_typed_rendezvous():
    """strided send layout into a different strided recv layout (copy_between
    semantics, datatype.py:760-797) above the eager limit."""
    import oracle
    st = ("vector", 4096, 3, 5, ("basic", 8))
    rt = ("hvector", 2048, 6, 64, ("basic", 8))

    def rank0(inst):
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        src = torch.arange(4096 * 5, dtype=torch.float64, device=inst.device)
        mp.send(c, src, 1, mp.type_vector(4096, 3, 5, mp.FLOAT64).commit(), 1, 3)
        mp.queue_synchronize(q)
        mp.comm_free(c)
        mp.free_stream(s)

    def rank1(inst):
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        dst = torch.zeros(2048 * 8, dtype=torch.float64, device=inst.device)
        mp.recv(c, dst, 1, mp.type_hvector(2048, 6, 64, mp.FLOAT64).commit(), 0, 3)
        mp.queue_synchronize(q)
        ref = np.zeros(2048 * 8, np.float64)
        src_h = np.arange(4096 * 5, dtype=np.float64)
        n = oracle.copy_between(oracle.OracleType(st), 1, src_h.view(np.uint8),
                                oracle.OracleType(rt), 1, ref.view(np.uint8))
        assert n == 4096 * 3 * 8
        assert np.array_equal(dst.cpu().numpy(), ref)
        mp.comm_free(c)
        mp.free_stream(s)

    pair(rank0, rank1, eager_limit=1024)


@pytest.mark.parametrize("st,rt,elem", [
    # 12-byte runs into 20-byte runs: 4-byte pieces
    (("vector", 1000, 3, 7, ("basic", 4)), ("vector", 700, 5, 9, ("basic", 4)), 4),
    # the cfg4 vector layout on both sides with different strides: 16-byte words
    (("vector", 2048, 4, 8, ("basic", 8)), ("vector", 1024, 8, 12, ("basic", 8)), 8),
    # odd byte runs: 1-byte words
    (("vector", 999, 3, 5, ("basic", 1)), ("vector", 1499, 2, 3, ("basic", 1)), 1),
])
def test_zipper_chain_to_chain_matches_copy_between(st, rt, elem):
    """one-pass chain -> chain transfer (k_zip) against the oracle's
    copy_between (datatype.py:760-797), rendezvous path."""
    import oracle
    from specbuild import build_product
    ot_s, ot_r = oracle.OracleType(st), oracle.OracleType(rt)
    rng = np.random.default_rng(77)
    src_h = rng.integers(0, 256, ot_s.max_end, dtype=np.uint8)

    def rank0(inst):
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        src = torch.from_numpy(src_h).to(inst.device)
        mp.send(c, src, 1, build_product(st, mp), 1, 5)
        mp.queue_synchronize(q)
        mp.comm_free(c)
        mp.free_stream(s)

    def rank1(inst):
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        dst = torch.zeros(ot_r.max_end, dtype=torch.uint8, device=inst.device)
        mp.recv(c, dst, 1, build_product(rt, mp), 0, 5)
        mp.queue_synchronize(q)
        ref = np.zeros(ot_r.max_end, np.uint8)
        n = oracle.copy_between(ot_s, 1, src_h, ot_r, 1, ref)
        assert n == min(ot_s.size_bytes, ot_r.size_bytes)
        assert np.array_equal(dst.cpu().numpy(), ref)
        mp.comm_free(c)
        mp.free_stream(s)

    pair(rank0, rank1, eager_limit=64)


# ------------------------------------------------------------- allreduce


@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("kind", ["int64", "float64", "float32"])
def test_allreduce_enqueue_native_matches_rank_ordered_oracle(n, kind):
    count = 100_003
    bufs = []
    for r in range(n):
        rng = np.random.default_rng(1000 + r)
        if kind == "int64":
            bufs.append(rng.integers(-2 ** 20, 2 ** 20, count, dtype=np.int64))
        elif kind == "float64":
            bufs.append(rng.uniform(-1, 1, count))
        else:
            bufs.append(rng.uniform(-1, 1, count).astype(np.float32))
    dtype = {"int64": mp.INT64, "float64": mp.FLOAT64, "float32": mp.FLOAT32}[kind]
    outs = [None] * n

    def body(inst):
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        sb = torch.from_numpy(bufs[inst.rank]).to(inst.device)
        rb = torch.zeros_like(sb)
        with torch.cuda.stream(q.torch_stream):
            sb.mul_(1)                                  # compute before
        mp.allreduce_enqueue(c, sb, rb, count, dtype, algo="native")
        with torch.cuda.stream(q.torch_stream):
            rb2 = rb * 1                                # compute after
        mp.queue_synchronize(q)
        outs[inst.rank] = rb2.cpu().numpy()
        mp.comm_free(c)
        mp.free_stream(s)

    host([body] * n)
    ref = oracle.allreduce_sum(bufs)
    if kind == "float32":
        ref = ref.astype(np.float32)
    for o in outs:
        assert np.array_equal(o, ref)       # bit-exact: same summation order


def test_allreduce_enqueue_nccl_single_rank():
    inst = mp.init(group=unique_group("nccl"), device=0)
    try:
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        x = torch.randn(1 << 16, device=inst.device)
        y = torch.zeros_like(x)
        mp.allreduce_enqueue(c, x, y, x.numel(), mp.FLOAT32, algo="nccl")
        mp.queue_synchronize(q)
        assert torch.equal(x, y)
        mp.comm_free(c)
        mp.free_stream(s)
    finally:
        inst.finalize()


def test_host_allreduce_reference_cases():   # test_comm.py:103-132
    def body(inst):
        r = inst.rank
        ib = torch.tensor([1 + r, 10 + 10 * r], dtype=torch.int64, device=inst.device)
        io = torch.zeros(2, dtype=torch.int64, device=inst.device)
        mp.allreduce(inst.world, ib, io, 2, mp.INT64)
        fb = torch.tensor([1.0], dtype=torch.float64, device=inst.device)
        fo = torch.zeros(1, dtype=torch.float64, device=inst.device)
        mp.allreduce(inst.world, fb, fo, 1, mp.FLOAT64)
        mp.allreduce(inst.world, fb, fo, 0, mp.FLOAT64)          # count 0: no-op
        with pytest.raises(ArgError):
            mp.allreduce(inst.world, fb, fo, 1, mp.FLOAT64, op="max")
        with pytest.raises(ArgError):
            mp.allreduce(inst.world, fb, fo, 1, mp.BYTE)
        return io.cpu().tolist(), fo.cpu().tolist()

    out = pair(body, body)
    assert out[0] == out[1] == ([3, 30], [2.0])


def test_queues_created_while_a_peer_stream_is_parked():
    """Rank 0's stream is parked in a rendezvous receive (a stream-memop
    wait) while rank 1 only then creates new queues and MPIX streams (local
    calls) before sending: creating those streams must not stall behind the
    parked stream (streams are reserved at world join)."""
    import threading
    parked = threading.Event()
    nbytes = 1 << 20
    payload = torch.arange(nbytes, dtype=torch.int64).to(torch.uint8)
    got = {}

    def rank0(inst):
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)                       # collective with rank 1
        dst = torch.zeros(nbytes, dtype=torch.uint8, device=inst.device)
        mp.recv_enqueue(c, dst, nbytes, mp.BYTE, 1, 5)    # parks the stream until delivery
        parked.set()
        mp.queue_synchronize(q)
        got["dst"] = dst.cpu()
        mp.comm_free(c)
        mp.free_stream(s)
        mp.queue_destroy(q)

    def rank1(inst):
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        assert parked.wait(60)
        time.sleep(0.05)
        extra = []
        for _ in range(3):                                # new streams while rank 0 is parked
            eq = mp.queue_create(inst)
            info = mp.info_create()
            mp.info_set(info, "type", "devstream")
            mp.info_set_hex(info, "value", bytes.fromhex(eq.handle))
            extra.append((eq, inst.stream_create(info)))
        mp.send_enqueue(c, payload.to(inst.device), nbytes, mp.BYTE, 0, 5)
        mp.queue_synchronize(q)
        for eq, es in extra:
            mp.free_stream(es)
            mp.queue_destroy(eq)
        mp.comm_free(c)
        mp.free_stream(s)
        mp.queue_destroy(q)

    pair(rank0, rank1)
    assert torch.equal(got["dst"], payload.cpu())


@pytest.mark.parametrize("nbytes", [1000, 1 << 20])
def test_receives_complete_out_of_posting_order(nbytes):
    """Rank 1 posts blocking receives for tag 2 then tag 1 before rank 0
    sends tag 1 then tag 2 (legal MPI with eager or buffered sends): the
    delivery of tag 1 must not sit in front of tag 2's on any stream."""
    import threading
    posted = threading.Event()
    got = {}

    def rank0(inst):
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        assert posted.wait(60)
        time.sleep(0.05)
        a = torch.full((nbytes,), 1, dtype=torch.uint8, device=inst.device)
        b = torch.full((nbytes,), 2, dtype=torch.uint8, device=inst.device)
        reqs = [mp.isend_enqueue(c, a, nbytes, mp.BYTE, 1, 1),
                mp.isend_enqueue(c, b, nbytes, mp.BYTE, 1, 2)]
        mp.waitall_enqueue(reqs)
        mp.queue_synchronize(q)
        mp.comm_free(c)
        mp.free_stream(s)
        mp.queue_destroy(q)

    def rank1(inst):
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        x = torch.zeros(nbytes, dtype=torch.uint8, device=inst.device)
        y = torch.zeros(nbytes, dtype=torch.uint8, device=inst.device)
        r2 = mp.irecv_enqueue(c, x, nbytes, mp.BYTE, 0, 2)
        mp.wait_enqueue(r2)                    # the stream reaches tag 1's post only after tag 2
        r1 = mp.irecv_enqueue(c, y, nbytes, mp.BYTE, 0, 1)
        mp.wait_enqueue(r1)
        posted.set()
        mp.queue_synchronize(q)
        got["x"], got["y"] = x.cpu(), y.cpu()
        mp.comm_free(c)
        mp.free_stream(s)
        mp.queue_destroy(q)

    pair(rank0, rank1)
    assert bool((got["x"] == 2).all()) and bool((got["y"] == 1).all())


# ---------------------------------------- BASELINE sizes (configs[3], [4])


@pytest.mark.timeout(600)
@pytest.mark.parametrize("n,nbytes", [(2, 64 << 20), (4, 64 << 20), (2, 1 << 30)])
@pytest.mark.parametrize("kind", ["u8", "vector"])
def test_ring_baseline_sizes(n, nbytes, kind):
    """64 MiB and 1 GiB rings (rendezvous; typed -> typed through the zipper),
    data generated and checked on the device (tests/ringkit.py)."""
    import ringkit
    ringkit.ring(n, nbytes, kind, iters=2 if nbytes < (1 << 30) else 1)


@pytest.mark.timeout(600)
@pytest.mark.parametrize("nbytes", [1 << 10, 64 << 20, 1 << 30])
@pytest.mark.parametrize("kind", ["int64", "float32"])
def test_allreduce_baseline_sizes_native(nbytes, kind):
    import ringkit
    ringkit.allreduce(2, nbytes, kind, "native")


@pytest.mark.timeout(900)
def test_eight_ranks_on_one_gpu_vector_ring_20_runs():
    """8 in-process ranks sharing one GPU, nonblocking 64 MiB vector(N/32,4,8)
    ring with the dependent scale kernels (tools/enqueue_bench.py), 20 fresh
    worlds in a row -- in a fresh process, the way a job starts: libmpx's
    first stream batch then covers the hardware queues with distinct streams
    (csrc/enqueue.cpp StreamPool::reserve).  With more streams than queues a
    stream parked in a wait parks its queue-mate (tools/stall_probe.py: 4
    ranks on 4 queues stall every run)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path[:0] = [%r, %r]\n"
            "import enqueue_bench as eb\n"
            "for k in range(20):\n"
            "    res = eb.ring(8, 64 << 20, iters=5, warmup=3, kind='vector', group='r8-%%d' %% k,\n"
            "                  device=lambda r: 0)\n"
            "    assert res['correct'], (k, res)\n"
            "print('20 ok')\n") % (root, os.path.join(root, "tools"))
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and "20 ok" in p.stdout, p.stdout[-2000:] + p.stderr[-3000:]


def test_throttled_enqueue_releases_the_gil():
    """Host run-ahead bound: with the queue's stream held up by a long kernel,
    a loop of eager self-sends soon finds 4 marks outstanding; the call then
    returns MPX_WOULD_BLOCK untouched and the binding waits in
    mpx_comm_throttle_wait WITH THE GIL RELEASED (the enqueue calls themselves
    keep it, ctypes.PyDLL) -- another Python thread keeps running meanwhile,
    and every message still arrives."""
    import threading
    inst = mp.init(group=unique_group("gil"), device=0)
    try:
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        ticks = [0]
        stop = threading.Event()

        def ticker():
            while not stop.is_set():
                ticks[0] += 1
                time.sleep(0)

        t = threading.Thread(target=ticker, daemon=True)
        t.start()
        n = 160
        src = torch.arange(n, dtype=torch.int64, device=inst.device).to(torch.uint8)
        dst = torch.zeros(n, dtype=torch.uint8, device=inst.device)
        with torch.cuda.stream(q.torch_stream):
            torch.cuda._sleep(200_000_000)          # ~0.1 s: the stream cannot pass the first mark
        before = ticks[0]
        t0 = time.perf_counter()
        for i in range(n):
            rr = mp.irecv_enqueue(c, dst[i:i + 1], 1, mp.BYTE, 0, i)
            sr = mp.isend_enqueue(c, src[i:i + 1], 1, mp.BYTE, 0, i)
            mp.waitall_enqueue([rr, sr])
        waited = time.perf_counter() - t0
        during = ticks[0] - before
        mp.queue_synchronize(q)
        stop.set()
        t.join(5)
        assert torch.equal(dst, src)
        assert waited > 0.02, waited                 # the loop really was throttled
        assert during > 100, during                  # ... and the other thread ran meanwhile
        mp.comm_free(c)
        mp.free_stream(s)
        mp.queue_destroy(q)
    finally:
        inst.finalize()
