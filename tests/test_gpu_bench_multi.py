"""The N > 1 path of bench.py (the driver's scaling run launches it under
torchrun, one process per GPU): on this box it runs with 2 processes sharing
one GPU and gloo for torch.distributed (NCCL refuses two ranks on one GPU),
which exercises every line of the multi-GPU section -- the job-name
broadcast, init(transport="ipc") from torchrun's environment, the rendezvous
ring at 64 MiB and 1 GiB (bytes and the vector type, with and without the
scale kernels), native allreduce at 64 MiB and 1 GiB, the max-over-ranks
timing and the on-device checks.  The numbers are not measurements (the two
processes time-slice one GPU); NCCL allreduce reports its refusal."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_processes_multi_gpu_section():
    env = dict(os.environ, MPX_BENCH_DIST_BACKEND="gloo", MPX_BENCH_NO_FLOOR="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29617", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu"]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=800, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    line = json.loads([x for x in p.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    mg = line["multi_gpu"]
    assert "error" not in mg, mg
    assert mg["ranks"] == 2
    assert len(mg["ring"]) == 6 and all(r["correct"] for r in mg["ring"]), mg["ring"]
    native = [a for a in mg["allreduce"] if a["algo"] == "native"]
    assert len(native) == 4 and all(a["correct"] for a in native), mg["allreduce"]
    nccl = [a for a in mg["allreduce"] if a["algo"] == "nccl"]
    assert all("error" in a for a in nccl)      # one GPU: NCCL needs a device per rank
