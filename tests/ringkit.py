"""Device-side ring and allreduce drivers for the enqueue tests at BASELINE
sizes (configs[3]: ring of 8 B .. 1 GiB messages, bytes or the
vector(N/32, 4, 8) FLOAT64 type, dependent scale kernels before the send and
after the receive; configs[4]: allreduce_enqueue SUM of float32 / int64
between two compute kernels).  Inputs come from seeded torch generators ON
the device and results are checked on the device, so 1 GiB cases run in
seconds; the rank placement is twin.host's (rank r on cuda:(r % devices)).

The checks are the reference's contracts: byte-exact delivery
(offload.py:198-268 through p2p.py:66-74), nothing written outside the
receive layout, Status source / count; allreduce int64 exact, float32 with
the native kernel bit-exact against the rank-ordered double sum
(comm.py:582-588) and with NCCL within 1e-6 * sum_r |x_r|."""

import torch

import paper_2402_12274_b200 as mp
from twin import default_device, host


def gen(dev, seed, numel, kind="u8"):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    if kind == "u8":
        return torch.randint(0, 256, (numel,), generator=g, device=dev, dtype=torch.uint8)
    if kind == "int64":
        return torch.randint(-2 ** 20, 2 ** 20, (numel,), generator=g, device=dev, dtype=torch.int64)
    return torch.rand(numel, generator=g, device=dev, dtype=torch.float32) * 2 - 1


def stream_comm(inst):
    q = mp.queue_create(inst)
    info = mp.info_create()
    mp.info_set(info, "type", "devstream")
    mp.info_set_hex(info, "value", bytes.fromhex(q.handle))
    s = inst.stream_create(info)
    return q, s, mp.stream_comm_create(inst.world, s)


def ring(n, nbytes, kind, iters=2, device=default_device, scale=True):
    """n ranks, isend -> r+1 / irecv <- r-1 of nbytes payload, `iters`
    iterations (fresh payload each), every received message checked."""
    def body(inst):
        r, dev = inst.rank, inst.device
        q, s, c = stream_comm(inst)
        vector = kind == "vector"
        span = 2 * nbytes - 32 if vector else nbytes
        if vector:
            dt, count = mp.type_vector(nbytes // 32, 4, 8, mp.FLOAT64).commit(), 1
        else:
            dt, count = mp.BYTE, nbytes
        prev = (r - 1) % n
        for it in range(iters):
            # everything on the queue's stream, no torch.cuda.synchronize(): a
            # device-wide sync would also wait for peer ranks' streams parked
            # on this rank's future sends (ranks sharing a GPU)
            with torch.cuda.stream(q.torch_stream):
                src = gen(dev, 7919 * it + r, span)
                dst = torch.full((span,), 0x5A, dtype=torch.uint8, device=dev)
                if scale and vector:
                    src.mul_(1)        # dependent elementwise kernel before the send (bytes: NaN-safe)
            rr = mp.irecv_enqueue(c, dst, count, dt, prev, it)
            sr = mp.isend_enqueue(c, src, count, dt, (r + 1) % n, it)
            mp.waitall_enqueue([rr, sr])
            with torch.cuda.stream(q.torch_stream):
                if scale and vector:
                    dst.mul_(1)        # dependent elementwise kernel after the receive
            mp.queue_synchronize(q)
            exp = gen(dev, 7919 * it + prev, span)
            if vector:
                pad = torch.zeros(32, dtype=torch.uint8, device=dev)
                d = torch.cat([dst, pad]).view(-1, 64)
                e = torch.cat([exp, pad]).view(-1, 64)
                assert bool((d[:, :32] == e[:, :32]).all()), ("payload", n, nbytes, kind, it)
                assert bool((d[:-1, 32:] == 0x5A).all()), ("wrote outside the layout", n, nbytes, it)
            else:
                assert bool((dst == exp).all()), ("payload", n, nbytes, kind, it)
            st = rr.status
            assert st.source == prev and st.tag == it and st.count == count and st.error is None, st
            del src, dst, exp
        if vector:
            mp.type_free(dt)
        mp.comm_free(c)
        mp.free_stream(s)
        mp.queue_destroy(q)

    host([body] * n, device=device)


def allreduce(n, nbytes, kind, algo, device=default_device):
    """allreduce_enqueue of nbytes per rank between two compute kernels."""
    def body(inst):
        r, dev = inst.rank, inst.device
        q, s, c = stream_comm(inst)
        es = 8 if kind == "int64" else 4
        count = nbytes // es
        with torch.cuda.stream(q.torch_stream):
            x = gen(dev, 104729 * (r + 1), count, kind)
            y = torch.empty_like(x)
            x.mul_(1)                                   # compute before
        mp.allreduce_enqueue(c, x, y, count, mp.INT64 if kind == "int64" else mp.FLOAT32, algo=algo)
        with torch.cuda.stream(q.torch_stream):
            y2 = y * 1                                  # compute after
        mp.queue_synchronize(q)
        if kind == "int64":
            ref = torch.zeros(count, dtype=torch.int64, device=dev)
            for k in range(n):
                ref += gen(dev, 104729 * (k + 1), count, kind)
            assert bool((y2 == ref).all()), ("int64 allreduce", n, nbytes, algo)
        else:
            acc = torch.zeros(count, dtype=torch.float64, device=dev)
            mag = torch.zeros(count, dtype=torch.float64, device=dev)
            for k in range(n):
                v = gen(dev, 104729 * (k + 1), count, kind).double()
                acc += v
                mag += v.abs()
            if algo == "native":     # rank order, double accumulation: bit-exact
                assert bool((y2 == acc.float()).all()), ("float32 allreduce", n, nbytes, algo)
            else:
                err = (y2.double() - acc).abs()
                assert bool((err <= 1e-6 * mag).all()), ("float32 allreduce", n, nbytes, algo,
                                                          float((err / mag.clamp_min(1e-30)).max()))
        del x, y, y2
        mp.comm_free(c)
        mp.free_stream(s)
        mp.queue_destroy(q)

    host([body] * n, device=device)
