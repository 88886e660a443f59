"""One rank of a multi-process job (test infrastructure for
tests/test_gpu_ipc.py): MINIMPI_TRANSPORT=ipc, rank / size / job name from
the environment.  Runs every scenario, checks bytes against the CPU oracle
and exits 0 on success (an assertion error exits non-zero)."""

import faulthandler
import os
import sys
import time

faulthandler.dump_traceback_later(int(os.environ.get("IPC_WORKER_TIMEOUT", "150")), exit=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")]

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from specbuild import build_product  # noqa: E402
import paper_2402_12274_b200 as mp  # noqa: E402


def stream_comm(inst):
    q = mp.queue_create(inst)
    info = mp.info_create()
    mp.info_set(info, "type", "devstream")
    mp.info_set_hex(info, "value", bytes.fromhex(q.handle))
    s = inst.stream_create(info)
    return q, s, mp.stream_comm_create(inst.world, s)


def data(seed, n):
    return np.random.default_rng(seed).integers(0, 256, n, dtype=np.uint8)


def ring(inst, q, c, nbytes, typed, order):
    """isend -> r+1, irecv <- r-1; `order` "recv" posts the receive first on
    every rank, "send" posts the send first and delays the receive so the
    receiving process's progress thread never runs (send matched at post)."""
    r, n = inst.rank, inst.size
    dev = inst.device
    if typed:   # vector(N/32, 4, 8) of FLOAT64 on both sides
        spec = ("vector", nbytes // 32, 4, 8, ("basic", 8))
        dt = mp.type_vector(nbytes // 32, 4, 8, mp.FLOAT64).commit()
        ot = oracle.OracleType(spec)
        span, count = ot.max_end, 1
    else:
        dt, ot, span, count = mp.BYTE, None, nbytes, nbytes
    src_h = data(1000 + r, span)
    src = torch.from_numpy(src_h).to(dev)
    dst = torch.full((span,), 0x5A, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize(dev)
    if order == "recv":
        rr = mp.irecv_enqueue(c, dst, count, dt, (r - 1) % n, 7)
        mp.barrier(inst.world)                    # every receive is posted before any send
        sr = mp.isend_enqueue(c, src, count, dt, (r + 1) % n, 7)
    else:
        sr = mp.isend_enqueue(c, src, count, dt, (r + 1) % n, 7)
        mp.barrier(inst.world)
        rr = mp.irecv_enqueue(c, dst, count, dt, (r - 1) % n, 7)
    mp.waitall_enqueue([rr, sr])
    mp.queue_synchronize(q)
    prev = data(1000 + (r - 1) % n, span)
    if typed:
        exp = np.full(span, 0x5A, np.uint8)
        ot.unpack(ot.pack(prev), exp)
    else:
        exp = prev
    assert np.array_equal(dst.cpu().numpy(), exp), ("ring", nbytes, typed, order)
    assert rr.status.source == (r - 1) % n and rr.status.tag == 7, rr.status
    if typed:
        mp.type_free(dt)
    mp.barrier(inst.world)


def tags_out_of_order(inst, q, c):
    """rank 0 sends tags 1 then 2 to rank 1, which receives 2 first (blocking
    enqueue forms; eager semantics across processes)."""
    dev = inst.device
    if inst.rank == 0:
        a = torch.full((1000,), 1, dtype=torch.uint8, device=dev)
        b = torch.full((3000,), 2, dtype=torch.uint8, device=dev)
        mp.send_enqueue(c, a, 1000, mp.BYTE, 1, 1)
        mp.send_enqueue(c, b, 3000, mp.BYTE, 1, 2)
        mp.queue_synchronize(q)
    elif inst.rank == 1:
        x = torch.zeros(3000, dtype=torch.uint8, device=dev)
        y = torch.zeros(1000, dtype=torch.uint8, device=dev)
        mp.recv_enqueue(c, x, 3000, mp.BYTE, 0, 2)
        mp.recv_enqueue(c, y, 1000, mp.BYTE, 0, 1)
        mp.queue_synchronize(q)
        assert bool((x == 2).all()) and bool((y == 1).all())
    mp.barrier(inst.world)


def any_source_and_truncation(inst, q, c):
    """every other rank sends to rank 0, which receives with ANY_SOURCE; then
    a receive smaller than its message reports ERR_TRUNCATE (nonblocking)."""
    dev, r, n = inst.device, inst.rank, inst.size
    if r == 0:
        got = set()
        for _ in range(n - 1):
            buf = torch.zeros(64, dtype=torch.uint8, device=dev)
            req = mp.irecv_enqueue(c, buf, 64, mp.BYTE, mp.ANY_SOURCE, 3)
            mp.wait_enqueue(req)
            mp.queue_synchronize(q)
            src = req.status.source
            assert bool((buf == src).all()), (src, buf[:4])
            got.add(src)
        assert got == set(range(1, n))
        small = torch.zeros(10, dtype=torch.uint8, device=dev)
        req = mp.irecv_enqueue(c, small, 10, mp.BYTE, 1, 4)
        mp.wait_enqueue(req)
        mp.queue_synchronize(q)
        assert req.status.error == "ERR_TRUNCATE", req.status
        assert bool((small == 9).all())
    else:
        mp.send_enqueue(c, torch.full((64,), r, dtype=torch.uint8, device=dev), 64, mp.BYTE, 0, 3)
        if r == 1:
            mp.send_enqueue(c, torch.full((20,), 9, dtype=torch.uint8, device=dev), 20, mp.BYTE, 0, 4)
        mp.queue_synchronize(q)
    mp.barrier(inst.world)


def allreduce(inst, q, c):
    """allreduce_enqueue across processes: rank-ordered sums (float32
    accumulated in double, comm.py:582-588) and exact int64, several calls
    back to back (the flags and handle slots are reused in stream order)."""
    dev, n = inst.device, inst.size
    for algo in algos():
        for count in (1, 1000, 1 << 20):
            xs = [np.random.default_rng(7 * count + r).uniform(-1, 1, count).astype(np.float32) for r in range(n)]
            ks = [np.random.default_rng(9 * count + r).integers(-2 ** 20, 2 ** 20, count) for r in range(n)]
            sf = torch.from_numpy(xs[inst.rank]).to(dev)
            si = torch.from_numpy(ks[inst.rank]).to(dev)
            rf, ri = torch.empty_like(sf), torch.empty_like(si)
            mp.allreduce_enqueue(c, sf, rf, count, mp.FLOAT32, algo=algo)
            mp.allreduce_enqueue(c, si, ri, count, mp.INT64, algo=algo)
            mp.queue_synchronize(q)
            acc = np.zeros(count, np.float64)
            for x in xs:
                acc += x.astype(np.float64)
            got = rf.cpu().numpy()
            if algo == "native":   # rank order, double accumulation: bit-exact
                assert np.array_equal(got, acc.astype(np.float32)), count
            else:                  # NCCL's order: |got - ref| <= 1e-6 * sum_r |x_r|
                bound = 1e-6 * np.sum([np.abs(x.astype(np.float64)) for x in xs], axis=0)
                assert np.all(np.abs(got.astype(np.float64) - acc) <= bound), count
            assert np.array_equal(ri.cpu().numpy(), np.sum(ks, axis=0)), (algo, count)
    mp.barrier(inst.world)


def algos():
    """native always; NCCL when every rank has its own GPU (one rank per device)."""
    return ["native", "nccl"] if "LOCAL_RANK" in os.environ else ["native"]


def windows(inst):
    """Passive-target reads across processes: every rank exposes a device
    tensor, reads its successor's window through a strided target type into a
    strided origin layout at a displacement (bytes checked against the
    oracle's copy_between), then a contiguous read and an out-of-bounds read
    rejected at unlock."""
    dev, r, n = inst.device, inst.rank, inst.size
    tspec = ("vector", 512, 4, 8, ("basic", 8))
    ospec = ("vector", 256, 8, 12, ("basic", 8))
    ts, os_ = oracle.OracleType(tspec), oracle.OracleType(ospec)
    disp = 3
    wbytes = ts.max_end + disp * 8 + 64
    win_t = torch.from_numpy(data(500 + r, wbytes)).to(dev)
    win = mp.win_create(inst.world, win_t, disp_unit=8)
    tgt = (r + 1) % n
    out = torch.full((os_.max_end,), 0x5A, dtype=torch.uint8, device=dev)
    tdt = mp.type_vector(512, 4, 8, mp.FLOAT64).commit()
    odt = mp.type_vector(256, 8, 12, mp.FLOAT64).commit()
    mp.win_lock(win, tgt)
    mp.win_get(win, out, 1, odt, tgt, disp, 1, tdt)
    plain = torch.zeros(64, dtype=torch.uint8, device=dev)
    mp.win_get(win, plain, 64, mp.BYTE, tgt, 1, 64, mp.BYTE)
    mp.win_unlock(win, tgt)
    src = data(500 + tgt, wbytes)
    ref = np.full(os_.max_end, 0x5A, np.uint8)
    assert oracle.copy_between(ts, 1, src[disp * 8:], os_, 1, ref) == ts.size_bytes
    assert np.array_equal(out.cpu().numpy(), ref)
    assert np.array_equal(plain.cpu().numpy(), src[8:72])
    mp.win_lock(win, tgt)
    mp.win_get(win, plain, 64, mp.BYTE, tgt, wbytes // 8, 64, mp.BYTE)     # beyond the target's region
    try:
        mp.win_unlock(win, tgt)
        raise AssertionError("out-of-bounds read was not rejected")
    except mp.ArgError:
        pass
    mp.barrier(inst.world)
    mp.win_free(win)
    mp.type_free(tdt)
    mp.type_free(odt)


def host_buffers(inst):
    """The reference's plain p2p surface on the world communicator with host
    (bytes / bytearray) buffers, across processes."""
    if inst.rank == 0:
        mp.send(inst.world, b"across processes", 16, mp.BYTE, 1, 11)
    elif inst.rank == 1:
        buf = bytearray(16)
        st = mp.recv(inst.world, buf, 16, mp.BYTE, 0, 11)
        assert bytes(buf) == b"across processes" and st.source == 0 and st.count == 16, (buf, st)
    mp.barrier(inst.world)


def posted_first_then_matched(inst, q, c):
    """rank 1: irecv A (posted first) and wait_enqueue(A), then irecv B that
    matches an already-sent message; A's send arrives only afterwards.  B's
    delivery waits (on the side stream) for rank 1's stream to pass A's wait,
    so A's delivery -- by the progress thread -- must not queue behind it."""
    dev = inst.device
    if inst.rank == 0:
        mp.send_enqueue(c, torch.full((4096,), 2, dtype=torch.uint8, device=dev), 4096, mp.BYTE, 1, 22)
        mp.queue_synchronize(q)
        mp.barrier(inst.world)          # 1: B is posted
        mp.barrier(inst.world)          # 2: rank 1 has enqueued both receives
        mp.send_enqueue(c, torch.full((4096,), 1, dtype=torch.uint8, device=dev), 4096, mp.BYTE, 1, 21)
        mp.queue_synchronize(q)
    elif inst.rank == 1:
        a = torch.zeros(4096, dtype=torch.uint8, device=dev)
        b = torch.zeros(4096, dtype=torch.uint8, device=dev)
        ra = mp.irecv_enqueue(c, a, 4096, mp.BYTE, 0, 21)
        mp.wait_enqueue(ra)
        mp.barrier(inst.world)
        rb = mp.irecv_enqueue(c, b, 4096, mp.BYTE, 0, 22)
        mp.barrier(inst.world)
        mp.wait_enqueue(rb)
        mp.queue_synchronize(q)
        assert bool((a == 1).all()) and bool((b == 2).all())
    else:
        mp.barrier(inst.world)
        mp.barrier(inst.world)
    mp.barrier(inst.world)


def rendezvous_layouts(inst, q, c):
    """Rendezvous (above the eager limit) with sender layouts the receiver must
    rebuild from their 64-byte description: a replicated vector (count > 1),
    a 3-level subarray face and an hvector of contiguous blocks, each received
    into a different layout; every byte checked against the oracle's
    copy_between (datatype.py:760-797)."""
    r, n, dev = inst.rank, inst.size, inst.device
    cases = [
        (("vector", 1024, 4, 8, ("basic", 8)), 8, ("contiguous", 32768, ("basic", 8)), 1),
        (("subarray", [40, 60, 70], [30, 50, 16], [5, 4, 3], ("basic", 4)), 1,
         ("vector", 12000, 2, 3, ("basic", 4)), 1),
        (("hvector", 300, 1, 1000, ("contiguous", 64, ("basic", 4))), 1, ("contiguous", 300 * 256, ("basic", 1)), 1),
    ]
    for k, (sspec, scount, rspec, rcount) in enumerate(cases):
        st, rt = oracle.OracleType(sspec), oracle.OracleType(rspec)
        sdt = build_product(sspec, mp)
        rdt = build_product(rspec, mp)
        sspan = st.max_end + (scount - 1) * st.extent_bytes if scount > 1 else st.max_end
        src_h = data(3000 + 10 * k + r, sspan)
        src = torch.from_numpy(src_h).to(dev)
        rspan = rt.max_end
        dst = torch.full((rspan,), 0x5A, dtype=torch.uint8, device=dev)
        torch.cuda.synchronize(dev)
        rr = mp.irecv_enqueue(c, dst, rcount, rdt, (r - 1) % n, 200 + k)
        sr = mp.isend_enqueue(c, src, scount, sdt, (r + 1) % n, 200 + k)
        mp.waitall_enqueue([rr, sr])
        mp.queue_synchronize(q)
        prev = data(3000 + 10 * k + (r - 1) % n, sspan)
        exp = np.full(rspan, 0x5A, np.uint8)
        moved = oracle.copy_between(st, scount, prev, rt, rcount, exp)
        assert moved == st.size_bytes * scount, (k, moved)
        assert np.array_equal(dst.cpu().numpy(), exp), ("rendezvous layout", k)
        assert rr.status.count == rcount, rr.status
    mp.barrier(inst.world)


def rendezvous_truncation_and_empty(inst, q, c):
    """A 1 MiB rendezvous message into a 512 KiB receive: the prefix lands,
    the receive reports ERR_TRUNCATE, the send completes (the receiver still
    writes the done flag); then a zero-byte message (count 0) both ways."""
    r, n, dev = inst.rank, inst.size, inst.device
    nb = 1 << 20
    src_h = data(4000 + r, nb)
    src = torch.from_numpy(src_h).to(dev)
    dst = torch.full((nb // 2,), 0x5A, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize(dev)
    rr = mp.irecv_enqueue(c, dst, nb // 2, mp.BYTE, (r - 1) % n, 300)
    sr = mp.isend_enqueue(c, src, nb, mp.BYTE, (r + 1) % n, 300)
    mp.waitall_enqueue([rr, sr])
    mp.queue_synchronize(q)
    prev = data(4000 + (r - 1) % n, nb)
    assert rr.status.error == "ERR_TRUNCATE", rr.status
    assert np.array_equal(dst.cpu().numpy(), prev[: nb // 2])
    empty = torch.zeros(1, dtype=torch.uint8, device=dev)
    rr = mp.irecv_enqueue(c, empty, 0, mp.BYTE, (r - 1) % n, 301)
    sr = mp.isend_enqueue(c, empty, 0, mp.BYTE, (r + 1) % n, 301)
    mp.waitall_enqueue([rr, sr])
    mp.queue_synchronize(q)
    assert rr.status.count == 0 and rr.status.error is None and rr.status.source == (r - 1) % n, rr.status
    mp.barrier(inst.world)


def stress(inst, q, c, seed=11):
    """tests/test_gpu_enqueue_stress.py's random nonblocking schedules across
    processes: eager (arena) and rendezvous (pull) messages, exact source and
    ANY_SOURCE, random posting order per rank, typed and byte sends."""
    import random
    from test_gpu_enqueue_stress import payload, schedule
    r, n, dev = inst.rank, inst.size, inst.device
    rng = random.Random(seed * 7919 + r)
    vec = {}
    for msgs in schedule(seed, n, phases=4, per_pair=2):
        ops = [("send", m) for m in msgs if m[0] == r] + [("recv", m) for m in msgs if m[1] == r]
        rng.shuffle(ops)
        reqs, checks, keep = [], [], []
        for kind, (s_, d_, tag, nb, typed, anys) in ops:
            if kind == "send":
                data_ = payload(dev, s_, tag, nb)
                if typed:
                    if nb not in vec:
                        vec[nb] = mp.type_vector(nb // 32, 4, 8, mp.FLOAT64).commit()
                    buf = torch.zeros(2 * nb, dtype=torch.uint8, device=dev)
                    buf.view(-1, 64)[:, :32] = data_.view(-1, 32)
                    reqs.append(mp.isend_enqueue(c, buf, 1, vec[nb], d_, 1000 + tag))
                else:
                    buf = data_ if nb else torch.zeros(1, dtype=torch.uint8, device=dev)
                    reqs.append(mp.isend_enqueue(c, buf, nb, mp.BYTE, d_, 1000 + tag))
                keep.append(buf)
            else:
                dst = torch.full((max(nb, 1),), 0x5A, dtype=torch.uint8, device=dev)
                rq = mp.irecv_enqueue(c, dst, nb, mp.BYTE, mp.ANY_SOURCE if anys else s_, 1000 + tag)
                reqs.append(rq)
                checks.append((rq, dst, s_, tag, nb))
        mp.waitall_enqueue(reqs)
        mp.queue_synchronize(q)
        for rq, dst, s_, tag, nb in checks:
            st = rq.status
            assert st.source == s_ and st.tag == 1000 + tag and st.count == nb and st.error is None, (s_, tag, st)
            if nb:
                assert torch.equal(dst[:nb], payload(dev, s_, tag, nb)), ("stress", s_, tag, nb)
        del keep
        mp.barrier(inst.world)
    for t in vec.values():
        mp.type_free(t)


def arena_wrap(inst, q, c, iters=40):
    """Staged (eager-path) messages wrapping the staging arena several times
    without any host synchronisation: a non-chain layout (irregular indexed
    blocks, so no rendezvous) of ~3 MiB per message through the 64 MiB arena
    of the test job, a distinct payload per iteration, every received message
    checked (an arena slot overwritten before it was consumed, or a message
    delivered to the wrong receive, shows up as a wrong payload)."""
    dev, r, n = inst.device, inst.rank, inst.size
    rng = np.random.default_rng(77)
    nblk = 1 << 16
    displs = np.cumsum(rng.integers(1, 4, nblk)).astype(np.int64) - 1
    spec = ("indexed_block", 6, [int(x) for x in displs], ("basic", 1))
    dt = mp.type_indexed_block(6, [int(x) for x in displs], mp.INT8).commit()
    ot = oracle.OracleType(spec)
    span = ot.max_end
    srcs = [torch.from_numpy(data(7000 + 97 * i + r, span)).to(dev) for i in range(iters)]
    dsts = [torch.zeros(span, dtype=torch.uint8, device=dev) for _ in range(iters)]
    torch.cuda.synchronize(dev)
    mp.barrier(inst.world)
    reqs = []
    for i in range(iters):
        reqs.append(mp.irecv_enqueue(c, dsts[i], 1, dt, (r - 1) % n, 100 + i))
        reqs.append(mp.isend_enqueue(c, srcs[i], 1, dt, (r + 1) % n, 100 + i))
    mp.waitall_enqueue(reqs)
    mp.queue_synchronize(q)
    for i in range(iters):
        exp = np.zeros(span, np.uint8)
        ot.unpack(ot.pack(data(7000 + 97 * i + (r - 1) % n, span)), exp)
        assert np.array_equal(dsts[i].cpu().numpy(), exp), ("arena wrap", i)
    mp.type_free(dt)
    mp.barrier(inst.world)


def big(inst, q, c):
    """BASELINE configs[3]/[4] at their largest size: 1 GiB messages (bytes,
    and the vector(N/32, 4, 8) FLOAT64 type over a 2 GiB span) around the
    ring through the rendezvous pull, and 1 GiB allreduce_enqueue in float32
    (rank-ordered double accumulation, bit-exact) and int64 (exact).  Data is
    generated and checked on the device (seeded torch generators)."""
    dev, r, n = inst.device, inst.rank, inst.size
    nb = 1 << 30
    prev = (r - 1) % n

    def gen(seed, numel, dtype=torch.uint8):
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        if dtype == torch.uint8:
            return torch.randint(0, 256, (numel,), generator=g, device=dev, dtype=torch.uint8)
        if dtype == torch.int64:
            return torch.randint(-2 ** 20, 2 ** 20, (numel,), generator=g, device=dev, dtype=torch.int64)
        return torch.rand(numel, generator=g, device=dev, dtype=torch.float32) * 2 - 1

    for typed in (False, True):
        span = 2 * nb - 32 if typed else nb
        src = gen(31 + r, span)
        dst = torch.full((span,), 0x5A, dtype=torch.uint8, device=dev)
        if typed:
            dt, count = mp.type_vector(nb // 32, 4, 8, mp.FLOAT64).commit(), 1
        else:
            dt, count = mp.BYTE, nb
        torch.cuda.synchronize(dev)
        mp.barrier(inst.world)
        rr = mp.irecv_enqueue(c, dst, count, dt, prev, 5)
        sr = mp.isend_enqueue(c, src, count, dt, (r + 1) % n, 5)
        mp.waitall_enqueue([rr, sr])
        mp.queue_synchronize(q)
        exp = gen(31 + prev, span)
        if typed:
            d = torch.cat([dst, torch.zeros(32, dtype=torch.uint8, device=dev)]).view(-1, 64)
            e = torch.cat([exp, torch.zeros(32, dtype=torch.uint8, device=dev)]).view(-1, 64)
            assert bool((d[:, :32] == e[:, :32]).all()), "1 GiB vector ring payload"
            assert bool((d[:-1, 32:] == 0x5A).all()), "1 GiB vector ring wrote outside the layout"
            mp.type_free(dt)
        else:
            assert bool((dst == exp).all()), "1 GiB byte ring"
        assert rr.status.count == count and rr.status.source == prev, rr.status
        del src, dst, exp
        mp.barrier(inst.world)
    for algo in algos():
        count = nb // 4
        xs = gen(51 + r, count, torch.float32)
        out = torch.empty_like(xs)
        mp.allreduce_enqueue(c, xs, out, count, mp.FLOAT32, algo=algo)
        mp.queue_synchronize(q)
        acc = torch.zeros(count, dtype=torch.float64, device=dev)
        mag = torch.zeros(count, dtype=torch.float64, device=dev)
        for k in range(n):
            x = gen(51 + k, count, torch.float32).double()
            acc += x
            mag += x.abs()
        if algo == "native":
            assert bool((out == acc.float()).all()), "1 GiB float32 allreduce (rank-ordered, double accumulation)"
        else:
            assert bool(((out.double() - acc).abs() <= 1e-6 * mag).all()), "1 GiB float32 NCCL allreduce"
        del xs, out, acc, mag
        count = nb // 8
        ks = gen(61 + r, count, torch.int64)
        out = torch.empty_like(ks)
        mp.allreduce_enqueue(c, ks, out, count, mp.INT64, algo=algo)
        mp.queue_synchronize(q)
        ref = torch.zeros_like(ks)
        for k in range(n):
            ref += gen(61 + k, count, torch.int64)
        assert bool((out == ref).all()), "1 GiB int64 allreduce (%s)" % algo
        del ks, out, ref
    mp.barrier(inst.world)


def main():
    inst = mp.init(transport="ipc")
    assert inst.transport == "ipc"
    q, s, c = stream_comm(inst)
    if os.environ.get("IPC_WORKER_MODE") == "big":
        big(inst, q, c)
        mp.comm_free(c)
        mp.free_stream(s)
        mp.queue_destroy(q)
        inst.finalize()
        print("rank %d ok" % inst.rank, flush=True)
        return
    for nbytes in (8, 1 << 16, 1 << 20, 16 << 20):
        for typed in (False, True):
            if typed and nbytes < 32:
                continue
            for order in ("recv", "send"):
                ring(inst, q, c, nbytes, typed, order)
    tags_out_of_order(inst, q, c)
    posted_first_then_matched(inst, q, c)
    allreduce(inst, q, c)
    windows(inst)
    host_buffers(inst)
    if inst.size >= 2:
        any_source_and_truncation(inst, q, c)
    arena_wrap(inst, q, c)
    rendezvous_layouts(inst, q, c)
    rendezvous_truncation_and_empty(inst, q, c)
    stress(inst, q, c)
    t0 = time.perf_counter()
    for _ in range(20):                       # arena reuse: many messages through the ring
        ring(inst, q, c, 4 << 20, False, "recv")
    mp.comm_free(c)
    mp.free_stream(s)
    mp.queue_destroy(q)
    inst.finalize()
    print("rank %d ok (%.2fs for the reuse loop)" % (inst.rank, time.perf_counter() - t0), flush=True)


if __name__ == "__main__":
    main()
