"""BASELINE configs[3] / configs[4] shapes on the GPUs of this process
(development / evidence tool): nonblocking ring (contiguous u8 and the
vector(N/32,4,8) f64 datatype with the dependent scale kernels) and
allreduce_enqueue (f32, i64) over in-process ranks, sizes 8 B .. 256 MiB.
With one GPU every rank shares it: the "link" is HBM, not NVLink.
Writes one JSON object (gpurun_out/enqueue_sweep_<tag>.json, tag = argv[1], default r02)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tools")]
import torch  # noqa: E402

import enqueue_bench as eb  # noqa: E402


def main():
    out = {"gpus": torch.cuda.device_count(), "device": torch.cuda.get_device_name(0), "ring": [], "allreduce": []}
    # one GPU: ranks share it; more than ~6 ranks per device can exhaust the
    # 32 hardware queues that keep stream-memop waits from blocking peers
    for n in (2, 4):
        for lg in (3, 12, 16, 20, 24, 26, 28):
            nb = 1 << lg
            for kind in ("u8", "vector"):
                if kind == "vector" and nb < 32:
                    continue
                it = 20 if nb <= (1 << 24) else 5
                r = eb.ring(n, nb, iters=it, warmup=2, group="sw-%d-%d-%s" % (n, lg, kind), kind=kind)
                out["ring"].append({k: r[k] for k in ("ranks", "kind", "bytes", "ms_per_iter", "GBps_per_rank", "correct")})
                print(json.dumps(out["ring"][-1]), flush=True)
        for lg in (10, 16, 20, 24, 26, 28):
            nb = 1 << lg
            it = 20 if nb <= (1 << 24) else 5
            r = eb.allreduce(n, nb // 4, iters=it, warmup=2, algo="native", group="sa-%d-%d" % (n, lg))
            out["allreduce"].append({k: r[k] for k in ("ranks", "bytes", "algo", "ms_per_iter", "busbw_GBps", "correct")})
            print(json.dumps(out["allreduce"][-1]), flush=True)
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    path = os.path.join(ROOT, "gpurun_out", "enqueue_sweep_%s.json" % tag)
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
