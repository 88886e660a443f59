"""GPU tests of multi-process worlds (csrc/ipc.hpp): 2 and 3
processes, one rank each, sharing the box's GPU through CUDA IPC.  Each rank
runs tests/ipc_worker.py (rings of bytes and strided FLOAT64 vectors with the
receive or the send posted first, tags matched out of order, ANY_SOURCE,
truncation, staging-arena reuse, allreduce_enqueue in float32 and int64,
read windows with strided types and bounds rejection)
and checks every byte against the CPU oracle / rank-ordered host sums."""

import os
import subprocess
import sys
import uuid

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]
HERE = os.path.dirname(os.path.abspath(__file__))


def run_job(n, mode="all", devices=None):
    job = "t%s" % uuid.uuid4().hex[:10]
    procs = []
    for r in range(n):
        env = dict(os.environ, MINIMPI_TRANSPORT="ipc", MINIMPI_RANK=str(r), MINIMPI_SIZE=str(n),
                   MINIMPI_GROUP=job, MPX_IPC_ARENA=str(64 << 20), IPC_WORKER_MODE=mode)
        if devices:
            env["LOCAL_RANK"] = str(r % devices)     # one rank per device (init(transport="ipc"))
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "ipc_worker.py")], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT))
    outs = []
    for p in procs:       # workers dump their stacks and exit after 150 s (faulthandler)
        try:
            out = p.communicate(timeout=200)[0].decode(errors="replace")
        except subprocess.TimeoutExpired:
            p.kill()
            out = p.communicate()[0].decode(errors="replace") + "\n[killed after 200 s]"
        outs.append((p.returncode, out))
    for r, (rc, out) in enumerate(outs):
        assert rc == 0, "rank %d failed:\n%s" % (r, out[-3000:])
        assert "rank %d ok" % r in out


@pytest.mark.parametrize("n", [2, 3])
def test_multi_process_world(n):
    run_job(n)


def test_multi_process_1gib_ring_and_allreduce():
    """1 GiB rendezvous rings (bytes and the strided vector type) and 1 GiB
    allreduce, 2 processes on this box's GPU (BASELINE configs[3]/[4] top size)."""
    run_job(2, mode="big")


def _ndev():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("n", [2, 4, 8])
def test_multi_process_one_rank_per_gpu(n):
    """The deployment shape: one process per GPU (peer mappings over NVLink,
    NCCL allreduce through ncclCommInitRank with the id shared in the job's
    segment).  Needs n devices; skipped on smaller boxes."""
    if _ndev() < n:
        pytest.skip("needs %d GPUs, %d visible" % (n, _ndev()))
    run_job(n, devices=n)
    run_job(n, mode="big", devices=n)
