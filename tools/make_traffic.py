"""Write profiles/roofline_traffic.json (read by bench.py for roofline.traffic)
from two ncu captures of the bench step (both --clock-control none, metrics
dram__bytes_read.sum / dram__bytes_write.sum / gpu__time_duration.sum, --csv):

  --range R.csv  range replay of tools/step_traffic.py: [fused pack, fused
                 unpack, 256 MiB read] with caches flushed before the range,
                 so the range's DRAM bytes minus the flush read are the whole
                 step's traffic, write-backs included;
  --seq S.csv    kernel replay with --cache-control none of
                 `bench.py --no-cpu --no-extras` (the kernels in their real
                 order: L2 flush, pack, unpack): per-launch DRAM bytes of the
                 pack and unpack as the timed step sees them (the unpack also
                 absorbs write-backs of the pack's dirty output).

    python tools/make_traffic.py --range R.csv --seq S.csv [--tag r02]
"""
import argparse
import csv
import io
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}


def rows_of(path):
    text = open(path).read()
    start = text.find('"ID"')
    return list(csv.DictReader(io.StringIO(text[start:])))


def metric(r):
    return float(r["Metric Value"].replace(",", "")) * SCALE.get(r.get("Metric Unit", ""), 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--range", required=True)
    ap.add_argument("--seq", required=True)
    ap.add_argument("--tag", default="r02")
    ap.add_argument("--flush", type=int, default=256 << 20)
    a = ap.parse_args()
    rng = {}
    for r in rows_of(a.range):
        rng[r["Metric Name"]] = rng.get(r["Metric Name"], 0.0) + metric(r)
    step = {"dram_read_bytes": rng.get("dram__bytes_read.sum"), "dram_write_bytes": rng.get("dram__bytes_write.sum"),
            "flush_read_bytes": a.flush}
    step["step_bytes"] = step["dram_read_bytes"] - a.flush + step["dram_write_bytes"]
    launches = {}
    for r in rows_of(a.seq):
        name = r["Kernel Name"]
        if "k_chain" not in name:
            continue
        kind = "pack" if ("k_chain<1>" in name or "(bool)1" in name or "k_chain<true>" in name
                          or "k_chain_pack" in name) else "unpack"
        lid = (kind, r["ID"])
        grid = r.get("Grid Size", "(0")
        launches.setdefault(lid, {"grid": int(grid.strip("()").split(",")[0] or 0)})[r["Metric Name"]] = metric(r)
    # the fused 12-face launches of the timed step: the largest grid of each direction
    big = {}
    for (kind, _), m in launches.items():
        big[kind] = max(big.get(kind, 0), m["grid"])
    launches = {k: m for k, m in launches.items() if m["grid"] == big[k[0]]}
    kernels = {}
    for (kind, _), m in launches.items():
        m = dict(m)
        m.pop("grid")
        k = kernels.setdefault(kind, {"launches": 0, "dram_read_bytes": 0.0, "dram_write_bytes": 0.0,
                                      "duration_us": 0.0})
        k["launches"] += 1
        k["dram_read_bytes"] += m.get("dram__bytes_read.sum", 0.0)
        k["dram_write_bytes"] += m.get("dram__bytes_write.sum", 0.0)
        k["duration_us"] += m.get("gpu__time_duration.sum", 0.0)
    for k in kernels.values():
        n = k.pop("launches")
        for f in ("dram_read_bytes", "dram_write_bytes", "duration_us"):
            k[f] = round(k[f] / n, 1)
        k["bytes_per_launch"] = k["dram_read_bytes"] + k["dram_write_bytes"]
        k["launches_averaged"] = n
    dom = max(kernels, key=lambda x: kernels[x]["duration_us"])
    res = {"source": "profiles/%s_step_range.csv (range replay: pack + unpack + 256 MiB read, caches flushed "
                     "before) and profiles/%s_seq_launches.csv (kernel replay, --cache-control none, real order)"
                     % (a.tag, a.tag),
           "step": step, "kernels": kernels, "dominant": dom, "bytes_per_launch": kernels[dom]["bytes_per_launch"]}
    with open(os.path.join(ROOT, "profiles", "roofline_traffic.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
