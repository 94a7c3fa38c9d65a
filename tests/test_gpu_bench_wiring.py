"""bench.py's N > 1 path under torchrun, on one GPU (BP_BENCH_ONE_GPU=1:
every rank on device 0, NCCL over its socket transport, IPC over CUDA IPC
mappings): the run exits 0 and rank 0 prints one JSON line with the
contract's keys. The numbers of a time-sliced GPU mean nothing; this guards
the wiring the driver's multi-GPU runs use."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("transport", ["nccl", "ipc"])
def test_bench_two_ranks_one_gpu(transport):
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ, BP_BENCH_ONE_GPU="1", CUDA_MODULE_LOADING="EAGER")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--workload",
           "tiny", "--transport", transport, "--steps", "1", "--warmup", "3"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "e2e", "roofline", "clocks",
              "gpu_launches", "config"):
        assert k in d, k
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
