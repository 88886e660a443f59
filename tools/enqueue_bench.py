"""Enqueue-path measurements on the GPUs of this process (library helper used
by bench.py's "extras"; also runnable alone).

ring(n, nbytes): n in-process ranks (round-robin over the visible GPUs; with
one GPU every rank shares it, so the "link" is the device's own HBM), each
rank isend -> (r+1)%n and irecv <- (r-1)%n of nbytes contiguous uint8 on its
own CUDA stream, waitall_enqueue; time = wall clock over `iters` iterations
after warm-up, bracketed by a host barrier + stream sync on every rank.
allreduce(n, count): allreduce_enqueue of float32 on n ranks, same timing.
"""

import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _run_ranks(n, body, group, device=None):
    import paper_2402_12274_b200 as mp
    import torch
    ndev = torch.cuda.device_count()
    out, errs = [None] * n, []
    bar = threading.Barrier(n)

    def runner(r):
        inst = None
        try:
            inst = mp.init(rank=r, ranks=n, group=group, device=device(r) if device else r % ndev)
            out[r] = body(inst, bar)
        except BaseException as e:  # noqa: B902
            errs.append(e)
            bar.abort()
        finally:
            if inst is not None and not inst.finalized:
                try:
                    inst.finalize()
                except Exception:
                    pass

    th = [threading.Thread(target=runner, args=(r,), daemon=True) for r in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    if errs:
        raise errs[0]
    return out


def ring(n=2, nbytes=64 << 20, iters=20, warmup=3, group="bench-ring", kind="u8", scale=True, device=None):
    """kind "u8": contiguous bytes; "vector": vector(N/32, 4, 8) of float64
    on both sides (BASELINE configs[3]: payload N bytes over a 2N - 32 byte
    span; typed -> typed, so the rendezvous path runs the one-pass zipper),
    with the dependent scale kernel on the stream before the send and after
    the receive.  Time: CUDA events on every rank's stream, max over ranks
    (wall clock reported beside)."""
    import paper_2402_12274_b200 as mp
    import torch

    def body(inst, bar):
        q = mp.queue_create(inst)
        info = mp.info_create()
        info.set("type", "devstream")
        mp.info_set_hex(info, "value", bytes.fromhex(q.handle))
        s = inst.stream_create(info)
        c = mp.stream_comm_create(inst.world, s)
        r = inst.rank
        if kind == "u8":
            src = torch.full((nbytes,), r, dtype=torch.uint8, device=inst.device)
            dst = torch.zeros_like(src)
            count, dt = nbytes, mp.BYTE
        else:
            src = torch.full((nbytes // 4,), float(r), dtype=torch.float64, device=inst.device)
            dst = torch.zeros_like(src)
            count, dt = 1, mp.type_vector(nbytes // 32, 4, 8, mp.FLOAT64).commit()

        # the scale kernels run on the queue's stream: order it after the
        # buffers' initialisation on the current stream (a device-wide sync
        # would also wait for peer ranks' parked streams)
        q.torch_stream.wait_stream(torch.cuda.current_stream(inst.device))

        def one():
            if kind != "u8" and scale:
                with torch.cuda.stream(q.torch_stream):
                    src.mul_(1.0)                   # dependent kernel before the send
            rr = mp.irecv_enqueue(c, dst, count, dt, (r - 1) % n, 0)
            sr = mp.isend_enqueue(c, src, count, dt, (r + 1) % n, 0)
            mp.waitall_enqueue([rr, sr])
            if kind != "u8" and scale:
                with torch.cuda.stream(q.torch_stream):
                    dst.mul_(1.0)                   # dependent kernel after the receive

        for _ in range(warmup):
            one()
        mp.queue_synchronize(q)
        bar.wait()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(q.torch_stream)
        for _ in range(iters):
            one()
        e1.record(q.torch_stream)
        mp.queue_synchronize(q)
        bar.wait()
        wall = time.perf_counter() - t0
        dev_ms = e0.elapsed_time(e1)
        if kind == "u8":
            ok = bool((dst == (r - 1) % n).all())
        else:
            v = dst.view(-1, 8)
            ok = bool((v[:, :4] == float((r - 1) % n)).all())
        mp.comm_free(c)
        mp.free_stream(s)
        return dev_ms, wall, ok

    res = _run_ranks(n, body, group, device)
    ms = max(x[0] for x in res) / iters
    wall = max(x[1] for x in res)
    return {"ranks": n, "kind": kind, "scale_kernels": bool(kind != "u8" and scale), "bytes": nbytes, "iters": iters, "ms_per_iter": ms,
            "GBps_per_rank": nbytes / ms / 1e6, "wall_ms_per_iter": 1e3 * wall / iters,
            "correct": all(x[2] for x in res)}


def allreduce(n=2, count=16 << 20, iters=20, warmup=3, algo=None, group="bench-ar"):
    import paper_2402_12274_b200 as mp
    import torch

    def body(inst, bar):
        q = mp.queue_create(inst)
        info = mp.info_create()
        info.set("type", "devstream")
        mp.info_set_hex(info, "value", bytes.fromhex(q.handle))
        s = inst.stream_create(info)
        c = mp.stream_comm_create(inst.world, s)
        x = torch.full((count,), float(inst.rank + 1), device=inst.device)
        y = torch.zeros_like(x)
        for _ in range(warmup):
            mp.allreduce_enqueue(c, x, y, count, mp.FLOAT32, algo=algo)
        mp.queue_synchronize(q)
        bar.wait()
        t0 = time.perf_counter()
        for _ in range(iters):
            mp.allreduce_enqueue(c, x, y, count, mp.FLOAT32, algo=algo)
        mp.queue_synchronize(q)
        bar.wait()
        dt = time.perf_counter() - t0
        ok = bool((y == n * (n + 1) / 2).all())
        mp.comm_free(c)
        mp.free_stream(s)
        return dt, ok

    res = _run_ranks(n, body, group)
    dt = max(r[0] for r in res)
    S = 4 * count
    return {"ranks": n, "bytes": S, "algo": algo or "auto", "ms_per_iter": 1e3 * dt / iters,
            "algbw_GBps": S * iters / dt / 1e9,
            "busbw_GBps": S * iters / dt / 1e9 * (2 * (n - 1) / n if n > 1 else 1),
            "correct": all(r[1] for r in res)}


if __name__ == "__main__":
    import json
    print(json.dumps(ring(2)))
    print(json.dumps(ring(2, kind="vector", group="bench-ring-v")))
    print(json.dumps(allreduce(2, algo="native")))
    print(json.dumps(allreduce(1, algo="nccl", group="bench-ar1")))
