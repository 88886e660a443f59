"""Enqueue path across GPUs (BASELINE configs[3] and [4]): one
in-process rank per device, so every send/recv is a peer transfer over
NVLink and allreduce_enqueue runs NCCL (ncclCommInitAll) or the native
kernel with peer loads / stores.  Needs >= 2 visible GPUs (cases with more
ranks than GPUs are skipped); the same drivers run on one GPU in
test_gpu_enqueue.py (ranks sharing the device) and, one process per GPU, in
test_gpu_ipc.py."""

import pytest
import torch

import ringkit

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]
NDEV = torch.cuda.device_count() if torch.cuda.is_available() else 0


def need(n):
    if NDEV < max(2, n):
        pytest.skip("needs %d GPUs (one rank per GPU), %d visible" % (max(2, n), NDEV))


def one_per_gpu(rank):
    return rank


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("nbytes", [8, 1 << 16, 64 << 20, 1 << 30])
@pytest.mark.parametrize("kind", ["u8", "vector"])
def test_ring_across_gpus(n, nbytes, kind):
    """8 B and 64 KiB go eager (staged), 64 MiB and 1 GiB rendezvous (one
    peer transfer; typed -> typed through the zipper)."""
    need(n)
    if kind == "vector" and nbytes < 32:
        pytest.skip("vector type needs >= 32 bytes")
    ringkit.ring(n, nbytes, kind, iters=2, device=one_per_gpu)


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("nbytes", [1 << 10, 64 << 20, 1 << 30])
@pytest.mark.parametrize("kind", ["int64", "float32"])
@pytest.mark.parametrize("algo", ["nccl", "native"])
def test_allreduce_across_gpus(n, nbytes, kind, algo):
    need(n)
    ringkit.allreduce(n, nbytes, kind, algo, device=one_per_gpu)
