"""Write profiles/roofline_traffic.json (read by bench.py for roofline.traffic)
from an `ncu --set full` capture of the fused k_chain pack + unpack launches.

    python tools/make_traffic.py profiles/r01_chain_full.ncu-rep
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    col = {k: i for i, k in enumerate(h)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}

    def val(r, k):
        return float(r[col[k]].replace(",", "")) * scale.get(units[col[k]], 1)

    kernels = {}
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        kind = "pack" if "k_chain<1>" in name or "(bool)1" in name else "unpack"
        rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
        kernels[kind] = {
            "kernel": name,
            "duration_us": val(r, "gpu__time_duration.sum"),
            "dram_read_bytes": rd,
            "dram_write_bytes": wr,
            "instructions": val(r, "smsp__inst_executed.sum"),
            "registers": val(r, "launch__registers_per_thread"),
            "bytes_per_launch": rd + wr,
        }
    dom = max(kernels, key=lambda k: kernels[k]["duration_us"])
    res = {"source": "%s (ncu --set full of the fused pack/unpack launches of bench.py)" % os.path.relpath(rep, ROOT),
           "kernels": kernels, "bytes_per_launch": kernels[dom]["bytes_per_launch"], "dominant": dom}
    with open(os.path.join(ROOT, "profiles", "roofline_traffic.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
