"""Where the time of a small-message enqueue ring goes (development probe):
n in-process ranks on this GPU, 8-byte u8 ring (irecv_enqueue, isend_enqueue,
waitall_enqueue per iteration); per-call host time of each API call on each
rank thread, host time per iteration, device time per iteration (CUDA events
on the queue stream, max over ranks).  One JSON line per n."""
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2402_12274_b200 as mp  # noqa: E402


def run(n, nbytes=8, iters=2000, warm=200):
    bar = threading.Barrier(n)
    res = [None] * n

    def body(r):
        inst = mp.init(rank=r, ranks=n, group="prof%d-%d" % (n, nbytes), device=0)
        q = mp.queue_create(inst)
        info = mp.info_create()
        info.set("type", "devstream")
        mp.info_set_hex(info, "value", bytes.fromhex(q.handle))
        s = inst.stream_create(info)
        c = mp.stream_comm_create(inst.world, s)
        src = torch.full((nbytes,), r, dtype=torch.uint8, device="cuda")
        dst = torch.zeros_like(src)
        T = [0.0, 0.0, 0.0]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for it in range(iters + warm):
            if it == warm:
                mp.queue_synchronize(q)
                bar.wait()
                w0 = time.perf_counter()
                e0.record(q.torch_stream)
            t0 = time.perf_counter()
            rr = mp.irecv_enqueue(c, dst, nbytes, mp.BYTE, (r - 1) % n, 0)
            t1 = time.perf_counter()
            sr = mp.isend_enqueue(c, src, nbytes, mp.BYTE, (r + 1) % n, 0)
            t2 = time.perf_counter()
            mp.waitall_enqueue([rr, sr])
            t3 = time.perf_counter()
            if it >= warm:
                T[0] += t1 - t0
                T[1] += t2 - t1
                T[2] += t3 - t2
        host = time.perf_counter() - w0
        e1.record(q.torch_stream)
        mp.queue_synchronize(q)
        bar.wait()
        res[r] = {"irecv_us": T[0] / iters * 1e6, "isend_us": T[1] / iters * 1e6, "waitall_us": T[2] / iters * 1e6,
                  "host_us_per_iter": host / iters * 1e6, "dev_us_per_iter": e0.elapsed_time(e1) / iters * 1e3,
                  "ok": bool((dst == (r - 1) % n).all())}
        mp.comm_free(c)
        mp.free_stream(s)
        mp.queue_destroy(q)
        inst.finalize()

    th = [threading.Thread(target=body, args=(r,)) for r in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    out = {"ranks": n, "bytes": nbytes}
    for k in res[0]:
        out[k] = round(max(x[k] for x in res), 2) if k != "ok" else all(x[k] for x in res)
    return out


if __name__ == "__main__":
    for n in (1, 2, 4):
        for nb in (8, 1 << 16):
            print(json.dumps(run(n, nb, iters=1000 if nb > 8 else 2000)), flush=True)
