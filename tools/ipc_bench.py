"""Multi-process ring (development tool): N processes, one rank
each, on the visible GPU(s) (with one GPU they share it through CUDA IPC).
Every rank isend -> r+1 / irecv <- r-1 of `bytes` per iteration on its own
stream communicator; time = CUDA events on every rank's stream, max over
ranks (gathered through the job's shared barrier and a tmp file).

    python tools/ipc_bench.py [N]     # prints one JSON line per size
"""

import json
import os
import subprocess
import sys
import tempfile
import uuid

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def worker(out_dir):
    sys.path.insert(0, ROOT)
    import torch
    import paper_2402_12274_b200 as mp
    inst = mp.init(transport="ipc")
    q = mp.queue_create(inst)
    info = mp.info_create()
    mp.info_set(info, "type", "devstream")
    mp.info_set_hex(info, "value", bytes.fromhex(q.handle))
    s = inst.stream_create(info)
    c = mp.stream_comm_create(inst.world, s)
    r, n, dev = inst.rank, inst.size, inst.device
    res = []
    sizes = [int(x) for x in os.environ.get("IPC_BENCH_LG", "12,16,20,24,26").split(",")]
    for lg in sizes:
        for kind in ("u8", "vector"):
            nb = 1 << lg
            if kind == "vector" and nb < 64:
                continue
            if kind == "u8":
                src = torch.full((nb,), r, dtype=torch.uint8, device=dev)
                dst = torch.zeros_like(src)
                dt, count = mp.BYTE, nb
            else:
                src = torch.full((nb // 4,), float(r), dtype=torch.float64, device=dev)
                dst = torch.zeros_like(src)
                dt, count = mp.type_vector(nb // 32, 4, 8, mp.FLOAT64).commit(), 1
            iters = 20 if nb <= (1 << 24) else 10
            # correctness first (untimed): distinct payloads per iteration into
            # per-iteration receive buffers, no sync until all are posted, every
            # message checked -- an overwritten staging slot or a misdelivered
            # message shows up as a wrong payload
            if nb <= (1 << 26) and (kind == "u8" or nb >= 64):
                k = 4
                srcs = [src.clone().fill_((r * 16 + i) % 256) if kind == "u8" else
                        src.clone().fill_(float(r * 16 + i)) for i in range(k)]
                dsts = [torch.zeros_like(dst) for _ in range(k)]
                reqs = []
                for i in range(k):
                    reqs.append(mp.irecv_enqueue(c, dsts[i], count, dt, (r - 1) % n, 100 + i))
                    reqs.append(mp.isend_enqueue(c, srcs[i], count, dt, (r + 1) % n, 100 + i))
                mp.waitall_enqueue(reqs)
                mp.queue_synchronize(q)
                p = (r - 1) % n
                for i in range(k):
                    if kind == "u8":
                        good = bool((dsts[i] == (p * 16 + i) % 256).all())
                    else:
                        good = bool((dsts[i].view(-1, 8)[:, :4] == float(p * 16 + i)).all())
                    assert good, ("ipc ring payload", nb, kind, i)
                del srcs, dsts
                mp.barrier(inst.world)

            def one():
                rr = mp.irecv_enqueue(c, dst, count, dt, (r - 1) % n, 0)
                sr = mp.isend_enqueue(c, src, count, dt, (r + 1) % n, 0)
                mp.waitall_enqueue([rr, sr])

            for _ in range(3):
                one()
            mp.queue_synchronize(q)
            mp.barrier(inst.world)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(q.torch_stream)
            for _ in range(iters):
                one()
            e1.record(q.torch_stream)
            mp.queue_synchronize(q)
            ms = e0.elapsed_time(e1) / iters
            ok = bool((dst.view(-1, 8)[:, :4] == float((r - 1) % n)).all()) if kind == "vector" else \
                bool((dst == (r - 1) % n).all())
            res.append({"bytes": nb, "kind": kind, "ms": ms, "ok": ok})
            mp.barrier(inst.world)
    with open(os.path.join(out_dir, "r%d.json" % r), "w") as f:
        json.dump(res, f)
    mp.comm_free(c)
    mp.free_stream(s)
    mp.queue_destroy(q)
    inst.finalize()


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    out_dir = tempfile.mkdtemp(prefix="ipcbench")
    job = "b%s" % uuid.uuid4().hex[:8]
    procs = []
    for r in range(n):
        env = dict(os.environ, MINIMPI_TRANSPORT="ipc", MINIMPI_RANK=str(r), MINIMPI_SIZE=str(n),
                   MINIMPI_GROUP=job, IPC_BENCH_OUT=out_dir)
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__), "--worker"], env=env))
    rc = [p.wait(timeout=600) for p in procs]
    if any(rc):
        print(json.dumps({"error": "worker exit codes %s" % rc}))
        sys.exit(1)
    per = [json.load(open(os.path.join(out_dir, "r%d.json" % r))) for r in range(n)]
    for i, row in enumerate(per[0]):
        ms = max(p[i]["ms"] for p in per)
        print(json.dumps({"processes": n, "kind": row["kind"], "bytes": row["bytes"], "ms_per_iter": round(ms, 4),
                          "GBps_per_rank": round(row["bytes"] / (ms / 1e3) / 1e9, 2),
                          "correct": all(p[i]["ok"] for p in per)}), flush=True)


if __name__ == "__main__":
    if "--worker" in sys.argv:
        worker(os.environ["IPC_BENCH_OUT"])
    else:
        main()
