"""The N > 1 host path of bench.py on CPU: two gloo ranks (torch.distributed
over 127.0.0.1) agree on the max-over-ranks time and the whole-job value, as
the driver's torchrun launch of `bench.py --gpus N` requires."""

import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import os, sys, json
sys.path.insert(0, %(root)r)
import torch.distributed as dist
dist.init_process_group("gloo", init_method="env://")
import bench
r, w, _ = bench.dist_env()
ms = 2.0 + 3.0 * r                       # rank 1 is the slow one
m = bench.max_over_ranks(ms)
v = bench.job_value(bench.step_bytes(), w, m)
print(json.dumps({"rank": r, "world": w, "max_ms": m, "value": v}), flush=True)
dist.destroy_process_group()
"""


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(120)
def test_bench_max_over_ranks_gloo_world2():
    import json
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK=str(r),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, "-c", CHILD % {"root": ROOT}],
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                      text=True))
    outs = [p.communicate(timeout=100) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e
    rows = [json.loads(o.strip().splitlines()[-1]) for o, _ in outs]
    import bench
    assert all(row["max_ms"] == 5.0 and row["world"] == 2 for row in rows)
    expect = 2 * bench.step_bytes() / 5e-3 / 1e9
    assert all(abs(row["value"] - expect) < 1e-6 * expect for row in rows)


def test_reference_arm_exits_on_nonzero_rank():
    """Under torchrun only rank 0 runs the CPU reference arm."""
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--gpus", "2", "--steps", "1", "--warmup", "0"],
                       env=env, capture_output=True, text=True, timeout=120)
    assert p.returncode == 0 and p.stdout.strip() == ""


@pytest.mark.timeout(300)
def test_reference_arm_json_contract():
    """bench.py --impl reference prints one JSON line with the contract keys
    (CPU oracle port on the host cores, no GPU needed)."""
    import json
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0"],
                       env=env, capture_output=True, text=True, timeout=280)
    assert p.returncode == 0, p.stderr
    line = json.loads(p.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_ipc_init_takes_rank_and_size_from_torchrun(monkeypatch):
    """init(transport="ipc") under torchrun: RANK / WORLD_SIZE / LOCAL_RANK /
    MASTER_PORT (no MINIMPI_* variables) give the rank, size, device and job
    name (a torchrun job of 2 once came out as size 1)."""
    import paper_2402_12274_b200 as mp
    from paper_2402_12274_b200 import runtime
    seen = {}

    class FakeInstance:
        def __init__(self, rank, size, group, device, eager, pool, transport, arena, matching="host"):
            seen.update(rank=rank, size=size, group=group, device=device, transport=transport)

    for k in ("MINIMPI_RANK", "MINIMPI_SIZE", "MINIMPI_GROUP", "MINIMPI_TRANSPORT"):
        monkeypatch.delenv(k, raising=False)
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setenv("LOCAL_RANK", "1")
    monkeypatch.setenv("MASTER_PORT", "29533")
    monkeypatch.setenv("TORCHELASTIC_RUN_ID", "none")
    monkeypatch.setattr(runtime, "Instance", FakeInstance)
    monkeypatch.setattr(runtime.torch.cuda, "device_count", lambda: 8)
    mp.init(transport="ipc")
    assert seen == {"rank": 1, "size": 2, "group": "job29533none", "device": 1, "transport": "ipc"}


def test_matching_mode_checked_before_any_device_work(monkeypatch):
    """init(matching=...): "host" (default) or "device" (csrc/dmatch.hpp),
    kwarg > MINIMPI_MATCHING > default; device matching is for in-process
    worlds only.  Checked before CUDA is touched."""
    import paper_2402_12274_b200 as mp
    from paper_2402_12274_b200 import runtime
    seen = {}

    class FakeInstance:
        def __init__(self, rank, size, group, device, eager, pool, transport, arena, matching="host"):
            seen["matching"] = matching

    monkeypatch.setattr(runtime, "Instance", FakeInstance)
    monkeypatch.setattr(runtime.torch.cuda, "device_count", lambda: 1)
    monkeypatch.delenv("MINIMPI_MATCHING", raising=False)
    with pytest.raises(mp.ArgError):
        mp.init(matching="gpu")
    with pytest.raises(mp.UnsupportedError):
        mp.init(transport="ipc", matching="device")
    mp.init()
    assert seen["matching"] == "host"
    monkeypatch.setenv("MINIMPI_MATCHING", "device")
    mp.init()
    assert seen["matching"] == "device"
    mp.init(matching="host")
    assert seen["matching"] == "host"
