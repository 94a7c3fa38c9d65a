"""Row (e) on one GPU: the multi-process layer pipeline (one process per
stage, static per-rank programs, send/recv rings on side streams, rank 0 owning
latents and Euler updates), several processes sharing device 0, with both
transports: CUDA IPC, and NCCL (each rank given its own NCCL host id, so NCCL
treats the ranks as separate hosts and uses its socket transport; the
executor's NCCL calls, channel connection order and stream/event logic are
the ones an 8-GPU run uses). The latents must equal the single-process serial
oracle bitwise (test_engine.cpp:66-78: N-invariance), across repeated runs of
the same pipeline."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = json.load(open(os.path.join(ROOT, "tests", "golden", "goldens.json")))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run_ranks(cfg, n, tmp_path, runs=2):
    out = str(tmp_path / "mp.npz")
    env = dict(os.environ, BP_MP_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "tests", "mp_worker.py"), json.dumps(cfg), out, str(runs)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return np.load(out)


@pytest.mark.parametrize("prec,n", [("f64", 2), ("bf16", 2), ("f64", 4)])
def test_ipc_pipeline_equals_serial_bitwise(bp, tmp_path, prec, n):
    base = dict(G["mid"]["config"], precision=prec)
    if n > 2:  # four processes time-slice one GPU: a shorter schedule
        base.update(steps=3, blocks=2)
    want = bp.serial_oracle(base)
    ref = np.concatenate([b["frames"].ravel() for b in want["blocks"]])
    got = run_ranks(dict(base, devices=n, transport="ipc"), n, tmp_path)
    for r in range(2):
        assert np.array_equal(got[f"run{r}"], ref), (prec, n, r)
        assert list(got[f"ids{r}"]) == [b["block_id"] for b in want["blocks"]]
    assert int(got["boundary_bytes"]) > 0


def test_ipc_pipeline_sequential_order_uneven(bp, tmp_path):
    """Sequential order, cache off, an uneven 3-way split of 4 layers."""
    base = dict(G["mid"]["config"], precision="f64", order="sequential", cache="off")
    want = bp.serial_oracle(base)
    ref = np.concatenate([b["frames"].ravel() for b in want["blocks"]])
    got = run_ranks(dict(base, devices=3, transport="ipc", uneven_split=True), 3, tmp_path, runs=1)
    assert np.array_equal(got["run0"], ref)


@pytest.mark.parametrize("prec,n", [("f64", 2), ("bf16", 3)])
def test_nccl_pipeline_equals_serial_bitwise(bp, tmp_path, prec, n):
    """The NCCL transport, including the deadlock-free channel connection
    order (pipeline.cu: every stage receives from its predecessor before it
    sends; NCCL connects a pair lazily and blocks until both ends take part)."""
    base = dict(G["mid"]["config"], precision=prec, steps=3, blocks=2)
    want = bp.serial_oracle(base)
    ref = np.concatenate([b["frames"].ravel() for b in want["blocks"]])
    got = run_ranks(dict(base, devices=n, transport="nccl", uneven_split=n == 3), n, tmp_path)
    for r in range(2):
        assert np.array_equal(got[f"run{r}"], ref), (prec, n, r)


def run_ranks_nt(cfg, n, tmp_path, runs=2):
    """The ranks as plain processes (no torch.distributed launcher, no torch in
    the workers): file rendezvous through a fresh bootstrap directory."""
    boot = tmp_path / "boot"
    boot.mkdir()
    prefix = str(tmp_path / "nt")
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(n), LOCAL_RANK="0")
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "mp_worker_nt.py"), json.dumps(cfg),
                                       prefix, str(boot), str(runs)], cwd=ROOT, env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    logs = [p.communicate(timeout=600)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), "\n".join(l[-2000:] for l in logs)
    stats = [json.load(open(f"{prefix}.rank{r}.json")) for r in range(n)]
    return np.load(prefix + ".npz"), stats


@pytest.mark.parametrize("transport,prec,n", [("ipc", "bf16", 2), ("ipc", "bf16", 3), ("ipc", "f64", 3),
                                              ("nccl", "bf16", 2)])
def test_file_bootstrap_without_torch(bp, tmp_path, transport, prec, n):
    """No PyTorch anywhere in the ranks; stage boundaries received in place
    (zero device copies of hidden states); bitwise == the serial oracle."""
    base = dict(G["mid"]["config"], precision=prec)
    if n > 2:
        base.update(steps=3, blocks=2, layers=3)
    want = bp.serial_oracle(base)
    ref = np.concatenate([b["frames"].ravel() for b in want["blocks"]])
    got, stats = run_ranks_nt(dict(base, devices=n, transport=transport), n, tmp_path)
    for r in range(2):
        assert np.array_equal(got[f"run{r}"], ref)
    assert all(not s["torch_loaded"] for s in stats)
    assert all(s["boundary_copies"] == 0 for s in stats), stats
    # IPC + bf16: every hidden state is written into the next rank's slot by
    # the last layer's residual GEMM epilogue (the fused send), no peer copy
    fused = transport == "ipc" and prec == "bf16"
    assert [s["fused_sends"] for s in stats] == [s["passes"] if fused and r < n - 1 else 0
                                                 for r, s in enumerate(stats)], stats


def test_ipc_fused_send_equals_copy_send(bp, tmp_path, monkeypatch):
    """The fused send (epilogue stores into the peer slot) and the peer-copy
    send (BP_IPC_FUSED_SEND=0) give the same latents, bitwise, over three
    ranks with an uneven layer split (a middle rank both receives and fuses)."""
    base = dict(G["mid"]["config"], precision="bf16", steps=3, blocks=2, layers=4)
    want = bp.serial_oracle(base)
    ref = np.concatenate([b["frames"].ravel() for b in want["blocks"]])
    split = dict(base, devices=3, transport="ipc", layer_split=[1, 2, 1])
    (tmp_path / "fused").mkdir()
    (tmp_path / "copy").mkdir()
    got, stats = run_ranks_nt(split, 3, tmp_path / "fused", runs=1)
    assert np.array_equal(got["run0"], ref)
    assert stats[0]["fused_sends"] > 0 and stats[1]["fused_sends"] > 0
    monkeypatch.setenv("BP_IPC_FUSED_SEND", "0")
    got2, stats2 = run_ranks_nt(split, 3, tmp_path / "copy", runs=1)
    assert np.array_equal(got2["run0"], ref)
    assert all(s["fused_sends"] == 0 for s in stats2)


@pytest.mark.parametrize("prec", ["f64", "bf16"])
def test_ipc_pipeline_wan_block_equals_serial(bp, tmp_path, prec):
    """The optional Wan block through the multi-process executor: every
    stage, not only the first, consumes the pass's frame levels (adaLN
    modulation) and frame ids (RoPE), so ranks > 0 need the per-pass metadata;
    two IPC processes equal the single-process serial run bitwise."""
    base = dict(layers=4, hidden=256, heads=2, channels=16, height=4, width=6, context_len=16, num_b=2, num_c=4,
                steps=3, blocks=2, mode="single", precision=prec, block="wan")
    want = bp.serial_oracle(base)
    ref = np.concatenate([b["frames"].ravel() for b in want["blocks"]])
    got = run_ranks(dict(base, devices=2, transport="ipc"), 2, tmp_path, runs=1)
    assert np.array_equal(got["run0"], ref), prec


def test_ipc_fused_send_production_shape(bp, tmp_path):
    """The fused send at the benchmarked token shape (Wan2.1-1.3B width, 480p
    grid: S = 18720 rows of 1536 fp32 per hidden state, cached prefix 6240;
    4 layers on 2 ranks, 2 blocks x 2 steps): the FFN-down epilogue writes
    every tile into the peer slot; latents equal the single-process serial
    run bitwise."""
    base = dict(layers=4, hidden=1536, heads=12, ffn=8960, channels=64, height=30, width=52, context_len=512,
                num_b=8, num_c=8, steps=2, blocks=2, precision="bf16", mode="single")
    want = bp.serial_oracle(base)
    ref = np.concatenate([b["frames"].ravel() for b in want["blocks"]])
    got, stats = run_ranks_nt(dict(base, devices=2, transport="ipc"), 2, tmp_path, runs=1)
    assert np.array_equal(got["run0"], ref)
    assert stats[0]["fused_sends"] == stats[0]["passes"] > 0
