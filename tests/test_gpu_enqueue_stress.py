"""Randomised enqueue stress (in-process ranks sharing the GPU): seeded
schedules of nonblocking sends and receives between every pair of ranks,
posted in a random interleaving per rank (so each message's receive comes
first on some ranks, its send on others), sizes across the eager limit
(0 B .. 1 MiB, bytes and the strided vector type), receives by exact source
or ANY_SOURCE with a unique tag, optional dependent kernels, a waitall at
the end of every phase -- an MPI-correct program, so every message must
arrive intact.  It drives the at-wait delivery, side-stream, deferral-thread,
rendezvous and throttle paths in combinations the targeted tests do not
(the reference's own randomized testing pattern, test_datatype.py:147-205,
applied to the enqueue engine)."""

import random

import pytest
import torch

import paper_2402_12274_b200 as mp
from twin import host

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]

SIZES = [0, 8, 1000, 1 << 16, (1 << 16) + 32, 1 << 20]


def payload(dev, src, tag, nbytes):
    g = torch.Generator(device=dev)
    g.manual_seed(src * 1000003 + tag)
    return torch.randint(0, 256, (nbytes,), generator=g, device=dev, dtype=torch.uint8)


def schedule(seed, n, phases, per_pair):
    """messages[phase] = list of (src, dst, tag, nbytes, typed, any_source)"""
    rng = random.Random(seed)
    out = []
    tag = 0
    for _ in range(phases):
        msgs = []
        for s in range(n):
            for d in range(n):
                for _ in range(per_pair):
                    nb = rng.choice(SIZES)
                    typed = nb >= 64 and nb % 64 == 0 and rng.random() < 0.4
                    msgs.append((s, d, tag, nb, typed, rng.random() < 0.3))
                    tag += 1
        out.append(msgs)
    return out


@pytest.mark.parametrize("seed,n", [(1, 2), (2, 3), (3, 4), (4, 2), (5, 3), (6, 4), (7, 8)])
def test_random_nonblocking_schedules(seed, n):
    plan = schedule(seed, n, phases=8 if n < 8 else 3, per_pair=3 if n < 8 else 1)

    def body(inst):
        r, dev = inst.rank, inst.device
        rng = random.Random(seed * 7919 + r)
        q = mp.queue_create(inst)
        info = mp.info_create()
        mp.info_set(info, "type", "devstream")
        mp.info_set_hex(info, "value", bytes.fromhex(q.handle))
        st = inst.stream_create(info)
        c = mp.stream_comm_create(inst.world, st)
        vec = {}

        def vtype(nb):
            if nb not in vec:
                vec[nb] = mp.type_vector(nb // 32, 4, 8, mp.FLOAT64).commit()
            return vec[nb]

        for msgs in plan:
            ops = [("send", m) for m in msgs if m[0] == r] + [("recv", m) for m in msgs if m[1] == r]
            rng.shuffle(ops)
            reqs, checks, keep = [], [], []
            with torch.cuda.stream(q.torch_stream):
                for kind, (s, d, tag, nb, typed, anys) in ops:
                    if kind == "send":
                        data = payload(dev, s, tag, nb)
                        if typed:   # the payload spread over a 2x span, blocks of 32 B every 64 B
                            buf = torch.zeros(2 * nb, dtype=torch.uint8, device=dev)
                            buf.view(-1, 64)[:, :32] = data.view(-1, 32)
                            reqs.append(mp.isend_enqueue(c, buf, 1, vtype(nb), d, tag))
                        else:
                            buf = data if nb else torch.zeros(1, dtype=torch.uint8, device=dev)
                            reqs.append(mp.isend_enqueue(c, buf, nb, mp.BYTE, d, tag))
                        keep.append(buf)
                    else:
                        src = mp.ANY_SOURCE if anys else s
                        dst = torch.full((max(nb, 1),), 0x5A, dtype=torch.uint8, device=dev)
                        rq = mp.irecv_enqueue(c, dst, nb, mp.BYTE, src, tag)   # typed sends land contiguous
                        reqs.append(rq)
                        checks.append((rq, dst, s, tag, nb))
                    if rng.random() < 0.2:
                        torch.cuda._sleep(2000)                # a dependent kernel on the queue
            mp.waitall_enqueue(reqs)
            mp.queue_synchronize(q)
            for rq, dst, s, tag, nb in checks:
                st_ = rq.status
                assert st_.source == s and st_.tag == tag and st_.count == nb and st_.error is None, \
                    (seed, r, s, tag, nb, st_)
                if nb:
                    assert torch.equal(dst[:nb], payload(dev, s, tag, nb)), (seed, r, s, tag, nb)
            del keep
        for t in vec.values():
            mp.type_free(t)
        mp.comm_free(c)
        mp.free_stream(st)
        mp.queue_destroy(q)

    host([body] * n, device=lambda r: 0)
