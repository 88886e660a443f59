import sys, json
sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import enqueue_bench as eb
for nb in (8, 4096, 65536, 1 << 20, 16 << 20, 256 << 20):
    r = eb.ring(2, nb, iters=50 if nb < (16 << 20) else 10, group="sw%d" % nb)
    print(json.dumps({"bytes": nb, "us_per_iter": round(r["ms_per_iter"] * 1e3, 2), "wall_us": round(r["wall_ms_per_iter"] * 1e3, 2), "GBps": round(r["GBps_per_rank"], 1), "ok": r["correct"]}))
for nb in (4096, 1 << 20, 64 << 20):
    r = eb.ring(4, nb, iters=20, group="sw4_%d" % nb)
    print(json.dumps({"ranks": 4, "bytes": nb, "us_per_iter": round(r["ms_per_iter"] * 1e3, 2), "wall_us": round(r["wall_ms_per_iter"] * 1e3, 2), "ok": r["correct"]}))
