"""Device-resident matching (csrc/dmatch.hpp): the enqueue
path's matching and point-to-point tests re-run with every world joined
with matching="device" (MINIMPI_MATCHING=device), plus the cases that only
device matching has: blocking rings beyond the eager limit (every blocking
send is buffered), rendezvous copies at match time, ANY_SOURCE races between senders resolved on the GPU, short
messages into typed receives, truncation reported from the device status.

Mirrors /root/reference/pkg/tests/test_offload.py:41-210 and test_p2p.py
(matching rules: transport.py:191-201,399-428)."""

import pytest
import torch

import paper_2402_12274_b200 as mp
from twin import host, pair

# the host-matching suites, collected again here under device matching
from test_gpu_enqueue import (  # noqa: F401
    inst, queue, device_comm, u8, _ring,
    test_deferred_error_surfaces_at_synchronize, test_awaited_request_error_lands_on_its_status,
    test_cross_rank_device_pipeline, test_criterion_09a_saxpy_pipeline_without_host_sync,
    test_criterion_09b_compute_overlaps_pending_receive, test_ring_nonblocking,
    test_ring_blocking_within_eager_limit, test_ring_blocking_large_with_raised_eager_limit,
    test_any_source_any_tag_and_fifo_order, test_typed_transfer_vector_to_contiguous,
    test_receives_complete_out_of_posting_order, test_ring_baseline_sizes)
from test_gpu_enqueue_stress import test_random_nonblocking_schedules  # noqa: F401

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]


@pytest.fixture(autouse=True)
def device_matching(monkeypatch):
    monkeypatch.setenv("MINIMPI_MATCHING", "device")


def test_mode_is_device(inst):
    assert inst.matching == "device"


@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("nbytes", [1 << 20, 16 << 20])
def test_blocking_ring_beyond_eager_limit(n, nbytes):
    """send-then-recv rings of blocking calls far above the eager limit: with
    every blocking send buffered at the sender no rank ever waits for its receiver
    (the reference guarantees this only up to its eager limit)."""
    _ring(n, nbytes, "u8", blocking=True)
    _ring(n, nbytes, "vector", blocking=True)


@pytest.mark.parametrize("n", [3, 5])
def test_any_source_race_takes_every_sender_once(n):
    """n-1 ranks send to rank 0 with one tag; rank 0 posts n-1 ANY_SOURCE
    receives before any send can have arrived: the GPU assigns each message
    to exactly one receive, in posting order of the receives."""
    got = {}

    def body(inst):
        r = inst.rank
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        if r == 0:
            bufs = [torch.zeros(64, dtype=torch.uint8, device=inst.device) for _ in range(n - 1)]
            with torch.cuda.stream(q.torch_stream):
                torch.cuda._sleep(20000)   # the posts run after the senders have started
            reqs = [mp.irecv_enqueue(c, b, 64, mp.BYTE, mp.ANY_SOURCE, 7) for b in bufs]
            mp.waitall_enqueue(reqs)
            mp.queue_synchronize(q)
            got["src"] = [rq.status.source for rq in reqs]
            got["data"] = [int(b[0].item()) for b in bufs]
            got["same"] = all(bool((b == b[0]).all()) for b in bufs)
        else:
            mp.send(c, torch.full((64,), r, dtype=torch.uint8, device=inst.device), 64, mp.BYTE, 0, 7)
            mp.queue_synchronize(q)
        mp.comm_free(c)
        mp.free_stream(s)
        mp.queue_destroy(q)

    host([body] * n)
    assert sorted(got["src"]) == list(range(1, n))
    assert got["data"] == got["src"] and got["same"]


def test_short_message_into_typed_receive_keeps_the_rest():
    """a message shorter than a typed receive fills a prefix of the layout;
    the layout's other bytes and the gaps keep their values (datatype.py:705-728
    prefix semantics)."""
    got = {}

    def rank0(inst):
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        mp.send(c, torch.arange(1, 7, dtype=torch.int32, device=inst.device), 6, mp.INT32, 1, 3)
        mp.queue_synchronize(q)
        mp.comm_free(c)
        mp.free_stream(s)
        mp.queue_destroy(q)

    def rank1(inst):
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        vt = mp.type_vector(5, 2, 3, mp.INT32).commit()          # 10 ints over 15
        dst = torch.full((15,), -1, dtype=torch.int32, device=inst.device)
        rq = mp.irecv_enqueue(c, dst, 1, vt, 0, 3)
        mp.wait_enqueue(rq)
        mp.queue_synchronize(q)
        got["dst"] = dst.cpu().tolist()
        got["count"] = rq.status.count
        got["err"] = rq.status.error
        mp.type_free(vt)
        mp.comm_free(c)
        mp.free_stream(s)
        mp.queue_destroy(q)

    pair(rank0, rank1)
    assert got["dst"] == [1, 2, -1, 3, 4, -1, 5, 6, -1, -1, -1, -1, -1, -1, -1]
    assert got["err"] is None
    assert got["count"] == 0      # 24 of 40 bytes: not a whole element of the vector type


def test_zero_byte_messages_match_in_order():
    got = {}

    def rank0(inst):
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        z = torch.zeros(1, dtype=torch.uint8, device=inst.device)
        for t in (4, 5):
            mp.send(c, z, 0, mp.BYTE, 1, t)
        mp.queue_synchronize(q)
        mp.comm_free(c)
        mp.free_stream(s)
        mp.queue_destroy(q)

    def rank1(inst):
        q = mp.queue_create(inst)
        c, s = device_comm(inst, q)
        z = torch.zeros(1, dtype=torch.uint8, device=inst.device)
        a = mp.irecv_enqueue(c, z, 0, mp.BYTE, 0, mp.ANY_TAG)
        b = mp.irecv_enqueue(c, z, 0, mp.BYTE, 0, mp.ANY_TAG)
        mp.waitall_enqueue([a, b])
        mp.queue_synchronize(q)
        got["tags"] = [a.status.tag, b.status.tag]
        got["counts"] = [a.status.count, b.status.count]
        mp.comm_free(c)
        mp.free_stream(s)
        mp.queue_destroy(q)

    pair(rank0, rank1)
    assert got["tags"] == [4, 5] and got["counts"] == [0, 0]


def test_ranks_must_agree_on_the_matching_mode():
    """a rank joining with the other mode is refused (and leaves the world
    cleanly: it can join again with the world's mode)"""
    import threading
    from twin import unique_group
    group = unique_group("mode")
    out = {}
    joined = threading.Event()

    def rank0():
        i = mp.init(rank=0, ranks=2, group=group, device=0, matching="device")
        joined.set()
        out[0] = i.matching
        i.finalize()

    def rank1():
        assert joined.wait(60)
        try:
            mp.init(rank=1, ranks=2, group=group, device=0, matching="host")
        except mp.ArgError as e:
            out["err"] = str(e)
        i = mp.init(rank=1, ranks=2, group=group, device=0, matching="device")
        out[1] = i.matching
        i.finalize()

    ts = [threading.Thread(target=f) for f in (rank0, rank1)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(120)
    assert "disagree" in out.get("err", "") and out.get(0) == out.get(1) == "device"


# ---- rendezvous (nonblocking contiguous sends above the eager limit) --------

def _comm(inst):
    q = mp.queue_create(inst)
    c, s = device_comm(inst, q)
    return q, c, s


def _close(q, c, s):
    mp.comm_free(c)
    mp.free_stream(s)
    mp.queue_destroy(q)


@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("nbytes", [(1 << 16) + 4, 4 << 20])
@pytest.mark.parametrize("order", ["recv_first", "send_first"])
def test_rendezvous_wait_send_before_recv(n, nbytes, order):
    """every rank: irecv, isend, wait(send), wait(recv) (or isend first) with
    distinct payloads per rank and iteration.  The data moves at match time
    on the stream of the side that matched second, so a send's completion
    never depends on the receiver's wait: no cycle, whatever the order."""
    got = {}

    def body(inst):
        r = inst.rank
        q, c, s = _comm(inst)
        ok = True
        for it in range(3):
            src = torch.full((nbytes,), (r * 7 + it) % 251, dtype=torch.uint8, device=inst.device)
            dst = torch.zeros(nbytes, dtype=torch.uint8, device=inst.device)
            if order == "recv_first":
                rr = mp.irecv_enqueue(c, dst, nbytes, mp.BYTE, (r - 1) % n, it)
                sr = mp.isend_enqueue(c, src, nbytes, mp.BYTE, (r + 1) % n, it)
            else:
                sr = mp.isend_enqueue(c, src, nbytes, mp.BYTE, (r + 1) % n, it)
                rr = mp.irecv_enqueue(c, dst, nbytes, mp.BYTE, (r - 1) % n, it)
            mp.wait_enqueue(sr)
            mp.wait_enqueue(rr)
            mp.queue_synchronize(q)
            want = ((r - 1) % n * 7 + it) % 251
            ok = ok and bool((dst == want).all()) and rr.status.count == nbytes and rr.status.source == (r - 1) % n
        got[r] = ok
        _close(q, c, s)

    host([body] * n)
    assert all(got[r] for r in range(n)), got


@pytest.mark.parametrize("cap", [1 << 12, 1 << 20])
def test_rendezvous_truncation_both_copy_sides(cap):
    """a 2 MiB rendezvous message into a smaller receive: the prefix lands
    (copied by k_dm_post itself for a receive within the eager limit, by the
    receiver's k_dm_xfer above it, or by the sender's k_dm_xfer when the
    receive was posted first), the status reports ERR_TRUNCATE, the sender
    completes."""
    nbytes = 2 << 20
    for first in ("recv", "send"):
        got = {}

        def rank0(inst):
            q, c, s = _comm(inst)
            src = torch.arange(nbytes, dtype=torch.int64, device=inst.device).to(torch.uint8)
            if first == "recv":
                with torch.cuda.stream(q.torch_stream):
                    torch.cuda._sleep(2000000)   # the receive is posted first
            sr = mp.isend_enqueue(c, src, nbytes, mp.BYTE, 1, 9)
            mp.wait_enqueue(sr)
            mp.queue_synchronize(q)
            got["sent"] = True
            _close(q, c, s)

        def rank1(inst):
            q, c, s = _comm(inst)
            if first == "send":
                with torch.cuda.stream(q.torch_stream):
                    torch.cuda._sleep(2000000)   # the message arrives first
            dst = torch.full((cap + 64,), 0xAB, dtype=torch.uint8, device=inst.device)
            rr = mp.irecv_enqueue(c, dst, cap, mp.BYTE, 0, 9)
            mp.wait_enqueue(rr)
            mp.queue_synchronize(q)
            h = dst.cpu()
            got["prefix"] = bool((h[:cap] == torch.arange(cap, dtype=torch.int64).to(torch.uint8)).all())
            got["rest"] = bool((h[cap:] == 0xAB).all())
            got["err"] = rr.status.error
            _close(q, c, s)

        pair(rank0, rank1)
        assert got["sent"] and got["prefix"] and got["rest"], (first, got)
        assert got["err"] == "ERR_TRUNCATE", (first, got)


def test_rendezvous_into_typed_receive():
    """a contiguous rendezvous message into a vector receive lands in the
    landing buffer prepared at the post and is unpacked at the wait."""
    n_el = 1 << 16                                    # 64 Ki doubles = 512 KiB payload
    got = {}

    def rank0(inst):
        q, c, s = _comm(inst)
        src = torch.arange(n_el, dtype=torch.float64, device=inst.device)
        sr = mp.isend_enqueue(c, src, n_el, mp.FLOAT64, 1, 2)
        mp.wait_enqueue(sr)
        mp.queue_synchronize(q)
        _close(q, c, s)

    def rank1(inst):
        q, c, s = _comm(inst)
        vt = mp.type_vector(n_el // 4, 4, 8, mp.FLOAT64).commit()
        dst = torch.full((2 * n_el,), -1.0, dtype=torch.float64, device=inst.device)
        rr = mp.irecv_enqueue(c, dst, 1, vt, 0, 2)
        mp.wait_enqueue(rr)
        mp.queue_synchronize(q)
        exp = torch.full((2 * n_el,), -1.0, dtype=torch.float64)
        exp.view(-1, 8)[:, :4] = torch.arange(n_el, dtype=torch.float64).view(-1, 4)
        got["ok"] = bool(torch.equal(dst.cpu(), exp))
        got["count"] = rr.status.count
        mp.type_free(vt)
        _close(q, c, s)

    pair(rank0, rank1)
    assert got["ok"] and got["count"] == 1


@pytest.mark.parametrize("n", [3, 5])
def test_rendezvous_any_source_takes_every_sender_once(n):
    """large isends from n-1 ranks into ANY_SOURCE receives of rank 0."""
    nbytes = 1 << 20
    got = {}

    def body(inst):
        r = inst.rank
        q, c, s = _comm(inst)
        if r == 0:
            bufs = [torch.zeros(nbytes, dtype=torch.uint8, device=inst.device) for _ in range(n - 1)]
            reqs = [mp.irecv_enqueue(c, b, nbytes, mp.BYTE, mp.ANY_SOURCE, 7) for b in bufs]
            mp.waitall_enqueue(reqs)
            mp.queue_synchronize(q)
            got["src"] = [rq.status.source for rq in reqs]
            got["data"] = [int(b[0].item()) for b in bufs]
            got["same"] = all(bool((b == b[0]).all()) for b in bufs)
        else:
            sr = mp.isend_enqueue(c, torch.full((nbytes,), r, dtype=torch.uint8, device=inst.device), nbytes,
                                  mp.BYTE, 0, 7)
            mp.wait_enqueue(sr)
            mp.queue_synchronize(q)
        _close(q, c, s)

    host([body] * n)
    assert sorted(got["src"]) == list(range(1, n))
    assert got["data"] == got["src"] and got["same"]


@pytest.mark.parametrize("nx", [16, 256])      # 16: eager (4 KiB), 256: rendezvous (1 MiB)
def test_chain_to_chain_face_into_vector(nx):
    """an x-face of a 3-D float32 array (one element per row: a chain of
    depth 2) into a vector(n/2, 2, 4) receive: one chain-to-chain copy, eager
    at the wait or rendezvous at match time (copy_between semantics,
    datatype.py:760-797); bytes outside the receive layout untouched."""
    n3 = nx + 2
    got = {}

    def rank0(inst):
        q, c, s = _comm(inst)
        # int32 payload (exact at every index) moved as 4-byte FLOAT32 elements
        a = torch.arange(n3 ** 3, dtype=torch.int32, device=inst.device)
        face = mp.type_create_subarray([n3, n3, n3], [nx, nx, 1], [1, 1, 1], mp.FLOAT32).commit()
        sr = mp.isend_enqueue(c, a, 1, face, 1, 5)
        mp.wait_enqueue(sr)
        mp.queue_synchronize(q)
        mp.type_free(face)
        _close(q, c, s)

    def rank1(inst):
        q, c, s = _comm(inst)
        n = nx * nx
        vt = mp.type_vector(n // 2, 2, 4, mp.FLOAT32).commit()
        dst = torch.full((2 * n,), -1, dtype=torch.int32, device=inst.device)
        rr = mp.irecv_enqueue(c, dst, 1, vt, 0, 5)
        mp.wait_enqueue(rr)
        mp.queue_synchronize(q)
        a = torch.arange(n3 ** 3, dtype=torch.int32).view(n3, n3, n3)
        face = a[1:nx + 1, 1:nx + 1, 1].reshape(-1)
        exp = torch.full((2 * n,), -1, dtype=torch.int32)
        exp.view(-1, 4)[:, :2] = face.view(-1, 2)
        got["ok"] = bool(torch.equal(dst.cpu(), exp))
        got["count"] = rr.status.count
        mp.type_free(vt)
        _close(q, c, s)

    pair(rank0, rank1)
    assert got["ok"] and got["count"] == 1
