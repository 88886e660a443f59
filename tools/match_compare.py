"""Host vs device matching (csrc/dmatch.hpp) on the BASELINE
configs[3] ring shapes (development / evidence tool): 2 and 4 in-process
ranks on the visible GPUs, contiguous u8 and the vector(N/32,4,8) datatype,
8 B .. 64 MiB.  One JSON line per (mode, ranks, kind, bytes)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tools")]

import enqueue_bench as eb  # noqa: E402


def main():
    for mode in ("host", "device"):
        os.environ["MINIMPI_MATCHING"] = mode
        for n in (2, 4):
            for lg in (3, 16, 20, 26):
                for kind in ("u8", "vector"):
                    if kind == "vector" and lg < 5:
                        continue
                    it = 200 if lg <= 16 else 20
                    r = eb.ring(n, 1 << lg, iters=it, warmup=5, group="mc-%s-%d-%d-%s" % (mode, n, lg, kind),
                                kind=kind)
                    print(json.dumps({"matching": mode, **{k: r[k] for k in
                                      ("ranks", "kind", "bytes", "ms_per_iter", "GBps_per_rank", "correct")}}),
                          flush=True)


if __name__ == "__main__":
    main()
