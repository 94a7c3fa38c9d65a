"""Operator surface on the GPU: `run` artifacts against the reference's own
files, `verify` (P/src/cli.cpp:133-274) and the reference's python smoke test
(P/tests/python/test_smoke.py) run unchanged against the `_blockpipe` shim."""
import json
import os
import struct

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "artifacts")


@pytest.fixture(scope="module")
def op():
    from paper_2505_21070_b200 import operator
    return operator


def parse_latents(raw: bytes):
    """latents.bin v1 (artifacts.cpp:25-45): two header lines, then per block
    'block <id> <frames>\\n' + frames*H*W*C little-endian float64."""
    lines = raw.split(b"\n", 2)
    assert lines[0] == b"blockpipe-latents v1"
    h, w, c = (int(v) for v in lines[1].split()[1:])
    rest, blocks = lines[2], []
    while rest:
        head, rest = rest.split(b"\n", 1)
        tag, bid, frames = head.split()
        assert tag == b"block"
        n = int(frames) * h * w * c
        blocks.append((int(bid), int(frames), np.frombuffer(rest[: 8 * n], dtype="<f8")))
        rest = rest[8 * n:]
    return (h, w, c), blocks


@pytest.mark.parametrize("name", sorted(os.listdir(GOLD)))
def test_run_artifacts_vs_reference(op, name, tmp_path, monkeypatch):
    monkeypatch.chdir(tmp_path)
    cfg = json.load(open(os.path.join(GOLD, name, "config.json")))
    cfg["out_dir"] = "out"
    assert op.run_and_write_artifacts(cfg) == "out/summary.json"
    for f in ("schedule.csv", "transfers.json", "summary.json"):
        assert (tmp_path / "out" / f).read_bytes() == open(os.path.join(GOLD, name, f), "rb").read(), f
    got_shape, got = parse_latents((tmp_path / "out" / "latents.bin").read_bytes())
    want_shape, want = parse_latents(open(os.path.join(GOLD, name, "latents.bin"), "rb").read())
    assert got_shape == want_shape and [b[:2] for b in got] == [b[:2] for b in want]
    for (_, _, g), (_, _, w) in zip(got, want):
        # fp64 engine: same op order except attention's exp and reductions
        assert np.max(np.abs(g - w)) <= 1e-12 * max(1.0, np.max(np.abs(w)))


def test_run_is_deterministic_and_trim_flag(op, tmp_path, monkeypatch):
    """test_cli.cpp:53-70, 157-170."""
    monkeypatch.chdir(tmp_path)
    names = ("latents.bin", "schedule.csv", "transfers.json", "summary.json")
    assert op.cli_main(["run", "--out", "a", "--mode", "single"])[0] == 0
    first = {f: (tmp_path / "a" / f).read_bytes() for f in names}
    assert op.cli_main(["run", "--out", "a", "--mode", "single"])[0] == 0
    assert first == {f: (tmp_path / "a" / f).read_bytes() for f in names}
    assert op.cli_main(["run", "--out", "t", "--mode", "single", "--trim-first-surplus"])[0] == 0
    full = (tmp_path / "a" / "latents.bin").read_bytes()
    trim = (tmp_path / "t" / "latents.bin").read_bytes()
    assert b"block 1 4\n" in full and b"block 1 2\n" in trim and len(full) > len(trim)
    _, fb = parse_latents(full)
    _, tb = parse_latents(trim)
    assert np.array_equal(fb[0][2][2 * 2 * 2 * 2:], tb[0][2])  # trimmed = the tail num_b frames


def test_seed_env_changes_latents(op, tmp_path, monkeypatch):
    monkeypatch.chdir(tmp_path)
    monkeypatch.setenv("BLOCKPIPE_SEED", "777")
    assert op.cli_main(["run", "--out", "a", "--mode", "single"])[0] == 0
    monkeypatch.setenv("BLOCKPIPE_SEED", "778")
    assert op.cli_main(["run", "--out", "b", "--mode", "single"])[0] == 0
    assert '"seed_model": 777' in (tmp_path / "a" / "summary.json").read_text()
    assert (tmp_path / "a" / "latents.bin").read_bytes() != (tmp_path / "b" / "latents.bin").read_bytes()


def test_verify_passes(op):
    code, out, err = op.cli_main(["verify"])
    assert code == 0, out + err
    assert "[FAIL]" not in out and out.count("[PASS]") == 8
    assert "[PASS] pipeline matches serial oracle" in out


def test_verify_detects_injected_cache_fault(op):
    code, out, _ = op.cli_main(["verify", "--fault-inject"])
    assert code == 1
    assert "[FAIL] feature cache matches explicit recompute" in out
    assert "cached V diverges" in out


# ---- P/tests/python/test_smoke.py, unchanged except for the module location ----------------
def test_smoke_bubble_ratio_reference_point():
    import _blockpipe as bp
    assert bp.bubble_size(4, 50, 4) == 11
    assert bp.bubble_ratio(4, 50, 4) == pytest.approx(11 / 211, abs=1e-12)
    assert bp.bubble_ratio(1, 50, 4) == 0.0
    assert bp.bubble_ratio(4, 50, 4, "sequential") == pytest.approx(15 / 215, abs=1e-12)


def test_smoke_matmul_matches_numpy():
    import _blockpipe as bp
    rng = np.random.default_rng(0)
    a = rng.normal(size=(5, 7))
    b = rng.normal(size=(7, 3))
    got = bp.matmul(a, b)
    assert np.allclose(got, a @ b, atol=1e-12)
    # and bit-identical to the reference's ascending-k unfused loop (tensor.cpp:99-107)
    want = np.zeros((5, 3))
    for i in range(5):
        for j in range(3):
            acc = 0.0
            for t in range(7):
                acc += float(a[i, t]) * float(b[t, j])
            want[i, j] = acc
    assert np.array_equal(got, want)


def test_smoke_softmax_and_layer_norm():
    import _blockpipe as bp
    x = np.array([[0.0, 0.0], [1000.0, 1000.0]])
    s = bp.softmax_rows(x)
    assert np.allclose(s, 0.5)
    y = bp.layer_norm(np.array([[5.0, 5.0, 5.0, 5.0]]))
    assert np.allclose(y, 0.0)
    z = np.random.default_rng(1).normal(size=(33, 300)) * 4
    e = np.exp(z - z.max(1, keepdims=True))
    assert np.allclose(bp.softmax_rows(z), e / e.sum(1, keepdims=True), rtol=1e-13, atol=0)
    m, v = z.mean(1, keepdims=True), z.var(1, keepdims=True)
    assert np.allclose(bp.layer_norm(z, 1e-3), (z - m) / np.sqrt(v + 1e-3), rtol=1e-12, atol=1e-12)


def test_smoke_random_source_is_deterministic(ref):
    import _blockpipe as bp
    a = bp.RandomSource(123)
    b = bp.RandomSource(123)
    xs = [a.next_normal() for _ in range(100)]
    assert xs == [b.next_normal() for _ in range(100)]
    assert np.array_equal(np.array(xs), ref.normals(123, 100))  # bit-exact vs the reference stream
    assert a.state == b.state


def test_smoke_pipeline_matches_oracle_bitwise():
    import _blockpipe as bp
    config = {"devices": 2, "steps": 4, "blocks": 4, "mode": "single"}
    got = bp.run_pipeline(config)
    want = bp.serial_oracle(config)
    assert len(got["blocks"]) == 4
    for g, w in zip(got["blocks"], want["blocks"]):
        assert g["block_id"] == w["block_id"]
        assert np.array_equal(g["frames"], w["frames"])


def test_smoke_bubble_measurements_surface():
    import _blockpipe as bp
    out = bp.run_pipeline({"devices": 1, "steps": 4, "blocks": 4, "mode": "single"})
    assert out["bubbles"]["idle_per_device"] == 0
    assert out["bubbles"]["busy_per_device"] == 16
    assert out["bubbles"]["ratio"] == 0.0


def test_smoke_traffic_report_matches_engine(op):
    """Analytics in bytes: predicted device->device bytes == engine's boundary_bytes."""
    import paper_2505_21070_b200 as bpk
    for prec in ("f64", "bf16"):
        cfg = {"devices": 2, "layers": 2, "hidden": 256, "heads": 2, "channels": 16, "height": 4, "width": 6,
               "context_len": 16, "num_b": 2, "num_c": 4, "steps": 3, "blocks": 2, "precision": prec}
        p = bpk.Pipeline(cfg)
        try:
            p.run_device()
            rep = op.traffic_report(p.schedule.ledger, prec, p.stats()["boundary_bytes"])
        finally:
            p.close()
        assert rep["match"], rep


@pytest.mark.parametrize("transport", ["ipc", "nccl"])
def test_cli_multiprocess_run_equals_single_process(tmp_path, transport):
    """The C++ host path end to end, no Python or PyTorch in the ranks: two
    `blockpipe run --transport ... --rank r --world 2` processes (file
    rendezvous in --bootstrap-dir) write latents.bin / schedule.csv /
    transfers.json byte-identical to the single-process two-stage run."""
    import subprocess
    exe = os.path.join(ROOT, "paper_2505_21070_b200", "lib", "blockpipe")
    common = ["run", "--devices", "2", "--layers", "4", "--hidden", "256", "--heads", "2", "--channels", "16",
              "--height", "4", "--width", "6", "--context-len", "16", "--steps", "3", "--blocks", "3",
              "--precision", "bf16", "--mode", "single"]
    # the config echo in schedule.csv carries out_dir (artifacts.cpp), so both
    # runs write to a relative "out" under their own working directory
    (tmp_path / "one").mkdir()
    (tmp_path / "multi").mkdir()
    single = subprocess.run([exe, *common, "--out", "out"], capture_output=True, text=True, timeout=300,
                            cwd=str(tmp_path / "one"))
    assert single.returncode == 0, single.stderr
    boot = tmp_path / "boot"
    boot.mkdir()
    procs = []
    for r in range(2):
        env = dict(os.environ, CUDA_MODULE_LOADING="EAGER")
        if transport == "nccl":  # both ranks share GPU 0: NCCL treats them as separate hosts
            env.update(NCCL_HOSTID=f"blockpipe-cli-{r}", NCCL_SOCKET_IFNAME="lo", NCCL_IB_DISABLE="1")
        procs.append(subprocess.Popen([exe, *common, "--transport", transport, "--rank", str(r), "--world", "2",
                                       "--bootstrap-dir", str(boot), "--out", "out"],
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True,
                                      cwd=str(tmp_path / "multi")))
    logs = [p.communicate(timeout=600)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), logs
    for f in ("latents.bin", "schedule.csv", "transfers.json"):
        assert (tmp_path / "multi" / "out" / f).read_bytes() == (tmp_path / "one" / "out" / f).read_bytes(), f
