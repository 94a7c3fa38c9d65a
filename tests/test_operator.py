"""Operator surface on CPU: artifacts, run config, analytics,
CLI and the host half of the `_blockpipe` compat module.

The schedule-derived artifacts (schedule.csv, transfers.json, summary.json)
depend only on the static schedule, so they are checked byte-for-byte against
files the reference itself wrote (tests/golden/artifacts/, made by
tests/golden/make_goldens.py through oracle/ref_artifacts.py). latents.bin
needs the GPU and is covered in test_gpu_operator.py. Mirrors
P/tests/test_cli.cpp and P/tests/test_analytics.cpp.
"""
import json
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "artifacts")
CASES = sorted(os.listdir(GOLD))
SCHEDULE_FILES = ("schedule.csv", "transfers.json", "summary.json")


@pytest.fixture(scope="module")
def op():
    from paper_2505_21070_b200 import operator
    return operator


def _golden_config(name):
    with open(os.path.join(GOLD, name, "config.json")) as f:
        cfg = json.load(f)
    cfg["out_dir"] = "out"  # the goldens were written with out_dir "out"
    return cfg


def _read(path):
    with open(path, "rb") as f:
        return f.read()


@pytest.mark.parametrize("name", CASES)
def test_plan_artifacts_byte_identical_to_reference(op, name, tmp_path, monkeypatch):
    monkeypatch.chdir(tmp_path)
    summary = op.plan_and_write_artifacts(_golden_config(name))
    assert summary == "out/summary.json"
    for f in SCHEDULE_FILES:
        assert _read(tmp_path / "out" / f) == _read(os.path.join(GOLD, name, f)), f
    assert not (tmp_path / "out" / "latents.bin").exists()


@pytest.mark.parametrize("name", CASES)
def test_cli_plan_with_config_file(op, name, tmp_path, monkeypatch):
    monkeypatch.chdir(tmp_path)
    (tmp_path / "c.json").write_text(json.dumps(_golden_config(name)))
    code, out, err = op.cli_main(["plan", "--config", "c.json"])
    assert (code, out, err) == (0, "wrote out/summary.json\n", "")
    for f in SCHEDULE_FILES:
        assert _read(tmp_path / "out" / f) == _read(os.path.join(GOLD, name, f)), f


def test_flags_override_config_file(op, tmp_path, monkeypatch):
    """cli.cpp:78-85: --config loads first, flags override (test_cli.cpp:83-98)."""
    monkeypatch.chdir(tmp_path)
    (tmp_path / "c.json").write_text(json.dumps({"steps": 9, "blocks": 7, "mode": "single"}))
    assert op.cli_main(["plan", "--config", "c.json", "--blocks", "4", "-T", "4", "--out", "o2"])[0] == 0
    summary = (tmp_path / "o2" / "summary.json").read_text()
    assert '"blocks": 4' in summary and '"steps": 4' in summary and '"mode": "single"' in summary


def test_order_flag_flips_the_schedule(op, tmp_path, monkeypatch):
    monkeypatch.chdir(tmp_path)
    assert op.cli_main(["plan", "--out", "rev", "--mode", "single"])[0] == 0
    assert op.cli_main(["plan", "--out", "seq", "--mode", "single", "--order", "sequential"])[0] == 0
    assert (tmp_path / "rev" / "schedule.csv").read_bytes() != (tmp_path / "seq" / "schedule.csv").read_bytes()


def test_retain_context_flag_echoed(op, tmp_path, monkeypatch):
    monkeypatch.chdir(tmp_path)
    assert op.cli_main(["plan", "--out", "off", "--no-retain-context"])[0] == 0
    assert '"retain_clean_context": false' in (tmp_path / "off" / "summary.json").read_text()


def test_config_echo_matches_reference_layout(op):
    want = json.load(open(os.path.join(GOLD, "default", "summary.json")))["config"]
    text = op.config_echo({"out_dir": "out"})
    assert json.loads(text) == want
    assert list(json.loads(text)) == list(want)  # key order
    assert text == json.dumps(want, indent=2)    # nlohmann dump(2) == python indent=2 for flat objects


def test_seed_environment_variable(op, monkeypatch):
    """run_config.cpp:57-63: BLOCKPIPE_SEED=S gives seeds S, S+1, S+2 unless set."""
    monkeypatch.setenv("BLOCKPIPE_SEED", "777")
    c = json.loads(op.config_echo({}))
    assert (c["seed_model"], c["seed_noise"], c["seed_context"]) == (777, 778, 779)
    c = json.loads(op.config_echo({"seed_noise": 5}))
    assert (c["seed_model"], c["seed_noise"], c["seed_context"]) == (777, 5, 779)


def test_config_errors(op):
    with pytest.raises(op.errors.ConfigError, match="unknown config key: bogus"):
        op.config_echo({"bogus": 1})
    with pytest.raises(op.errors.ConfigError, match="bad value for key 'devices'"):
        op.config_echo({"devices": "two"})
    with pytest.raises(op.errors.ConfigError, match="order must be reverse or sequential"):
        op.config_echo({"order": "zigzag"})
    with pytest.raises(op.errors.ConfigError, match="mode must be threaded or single"):
        op.config_echo({"mode": "async"})


def test_extension_keys_echo_only_when_set(op):
    base = json.loads(op.config_echo({}))
    assert "precision" not in base and "ffn" not in base and "uneven_split" not in base
    ext = json.loads(op.config_echo({"precision": "bf16", "ffn": 8960, "uneven_split": True}))
    assert (ext["precision"], ext["ffn"], ext["uneven_split"]) == ("bf16", 8960, True)
    assert list(ext)[: len(base)] == list(base)


# ---- analytics (P/tests/test_analytics.cpp) --------------------------------------------
def test_bubble_reference_point(op):
    assert op.bubble_size(4, 50, 4) == 11
    assert op.bubble_ratio(4, 50, 4) == pytest.approx(11 / 211, abs=1e-12)
    assert op.bubble_ratio(1, 50, 4) == 0.0
    assert op.bubble_ratio(4, 50, 4, "sequential") == pytest.approx(15 / 215, abs=1e-12)
    with pytest.raises(op.errors.ConfigError):
        op.bubble_size(0, 4, 4)


def test_bubble_grid_bitwise_vs_reference(op, ref):
    for n in (1, 2, 3, 4, 8):
        for t in (1, 2, 4, 8, 50):
            for b in (1, 2, 3, 4, 8, 100):
                for order in ("reverse", "sequential"):
                    try:
                        want = ref.bubble(n, t, b, order)
                    except ref.RefError:
                        with pytest.raises(op.errors.ConfigError):
                            op.bubble_size(n, t, b, order)
                        continue
                    assert (op.bubble_size(n, t, b, order), op.bubble_ratio(n, t, b, order)) == want


@pytest.mark.parametrize("params", [{}, dict(num_b=8, num_c=8, height=4, width=4, hidden=8),
                                    dict(frames=81, height=30, width=52, hidden=1536, channels=16, layers=30,
                                         devices=8, num_b=21, num_c=6, model_mem=2.6, kv_mem=0.3),
                                    dict(devices=3, ring_refinement=True), dict(num_c=0, devices=7)])
def test_method_costs_bitwise_vs_reference(op, ref, params):
    for m in op.METHODS:
        assert op.method_cost(m, **params) == ref.method_cost(m, **params)


def test_method_cost_row_and_bytes(op):
    row = op.method_cost("dualparal", num_b=8, num_c=8, height=4, width=4, hidden=8)
    assert row["comm_scalars"] == 2 * 12 * 4 * 4 * 8 and row["comm_overlap"] is True
    b = op.method_cost("dualparal", num_b=8, num_c=8, height=4, width=4, hidden=8, dtype="bf16")
    assert b["comm_bytes"] == 2 * row["comm_scalars"]
    with pytest.raises(ValueError):
        op.method_cost("dualparal", nonsense=1)
    with pytest.raises(op.errors.ConfigError):
        op.method_cost("gpipe")


def test_traffic_report_matches_ledger(bp, op):
    """Analytics in bytes: boundary bytes predicted from the ledger equal the
    per-pass tokens x hidden x element size the engine sends (pipeline.cu)."""
    s = bp.Schedule({"devices": 2, "steps": 4, "blocks": 4})
    rep = op.traffic_report(s.ledger, "bf16")
    tokens = sum(p["tokens"] for p in (s.pass_record(i) for i in range(s.npasses)))
    assert rep["ledger_scalars"] == tokens * 16  # hidden 16, one dev0->dev1 hop
    assert rep["predicted_bytes"] == 4 * rep["ledger_scalars"]  # fp32 residual crosses stages


# ---- CLI (P/tests/test_cli.cpp) -------------------------------------------------------------
def test_analyze_bubble_text_and_json(op):
    code, out, _ = op.cli_main(["analyze", "bubble"])
    assert code == 0 and out == "bubble N=4 T=50 blocks=4 order=reverse size=11 ratio=0.052133\n"
    code, out, _ = op.cli_main(["analyze", "bubble", "--format", "json", "--N", "2", "--order", "sequential"])
    assert code == 0 and json.loads(out) == {"N": 2, "T": 50, "blocks": 4, "order": "sequential", "size": 3,
                                             "ratio": 3 / 203}


def test_analyze_costs_table(op, ref):
    code, out, _ = op.cli_main(["analyze", "costs"])
    lines = out.splitlines()
    assert code == 0 and lines[0].split() == ["method", "comm_scalars", "overlap", "model_mem", "kv_mem"]
    assert len(lines) == 6 and "dualparal" in out and "3072" in out
    for line in lines[1:]:
        name, comm, ovl, mm, kv = line.split()
        want = ref.method_cost(name)
        assert (float(comm), ovl == "yes", float(mm), float(kv)) == pytest.approx(
            (want["comm_scalars"], want["comm_overlap"], want["model_mem"], want["kv_mem"]), abs=5e-7)
    assert len(lines[1]) == 16 + 16 + 9 + 14 + 14  # setw layout (cli.cpp:289-300)
    code, out, _ = op.cli_main(["analyze", "costs", "--format", "json", "--method", "fifo", "-N", "4"])
    assert code == 0 and json.loads(out) == [ref.method_cost("fifo", devices=4)]


def test_analyze_sweep(op):
    code, out, _ = op.cli_main(["analyze", "sweep", "--blocks", "4,8,16", "--format", "csv"])
    rows = out.splitlines()
    assert code == 0 and rows[0] == "blocks,ratio" and len(rows) == 4
    vals = [float(r.split(",")[1]) for r in rows[1:]]
    assert vals == sorted(vals, reverse=True) and vals[0] > vals[-1]
    code, out, _ = op.cli_main(["analyze", "sweep", "--devices", "2,4", "--methods", "dualparal",
                                "--format", "json"])
    assert code == 0 and [(r["axis"], r["value"]) for r in json.loads(out)] == [("N", 2), ("N", 4)]
    code, out, _ = op.cli_main(["analyze", "sweep", "--frames", "8,16", "--format", "csv"])
    assert code == 0 and out.splitlines()[0] == "axis,value,method,comm_scalars,overlap,model_mem,kv_mem"
    assert op.cli_main(["analyze", "sweep"])[0] == 2


@pytest.mark.parametrize("strategy", ["coordinated", "complete-shuffle", "subset", "fresh", "repeat"])
@pytest.mark.parametrize("num_b,num_c,seed,appends", [(4, 4, 2, 5), (8, 8, 99, 12), (3, 2, 7, 4), (2, 0, 5, 3)])
def test_noise_demo_ids_match_reference(op, ref, strategy, num_b, num_c, seed, appends):
    args = ["noise-demo", "--strategy", strategy, "--num-b", str(num_b), "--num-c", str(num_c),
            "--seed", str(seed), "--appends", str(appends)]
    code, out, err = op.cli_main(args)
    assert code == 0, err
    lines = out.splitlines()
    assert lines[0] == f"strategy={strategy} pool={num_b + num_c // 2}"
    got = [[int(v) for v in re.search(r"ids=\[([^\]]*)\]", ln).group(1).split()] for ln in lines[1:]]
    want = ref.noise_walk(strategy, appends, num_b, num_c, seed)
    assert got == want
    w = num_c // 2
    for i, ln in enumerate(lines[2:], start=1):
        window = want[i - 1][-w:] if w and len(want[i - 1]) >= w else []
        assert f"window=[{' '.join(map(str, window))}]" in ln
        assert ln.endswith(f"overlap={sum(1 for x in want[i] if x in window)}")


def test_noise_demo_overlap_signal(op):
    assert "overlap=0" in op.cli_main(["noise-demo"])[1]
    assert "overlap=0" not in op.cli_main(["noise-demo", "--strategy", "repeat"])[1]


@pytest.mark.parametrize("args,code", [
    (["bogus"], 2),
    ([], 2),
    (["run", "--devices", "3", "--layers", "4", "--mode", "single"], 2),
    (["run", "--order", "bogus"], 2),
    (["run", "--steps", "four"], 2),
    (["analyze", "costs", "--method", "gpipe"], 2),
    (["analyze", "bubble", "--format", "yaml"], 2),
    (["run", "--config", "/nonexistent/config.json"], 3),
    (["run", "--transport", "nccl", "--world", "2", "--rank", "0", "--devices", "2"], 2),  # no --bootstrap-dir
    (["run", "--rank", "1"], 2),
    (["run", "--transport", "carrier-pigeon"], 2),
    (["--help"], 0),
    (["analyze", "--help"], 0),
])
def test_cli_exit_codes(op, args, code):
    """cli.cpp:389-396, 534-543 (test_cli.cpp:147-155)."""
    got, out, err = op.cli_main(args)
    assert got == code, (out, err)
    if code == 3:
        assert err.startswith("io error: cannot open config file")


def test_cli_binary(tmp_path):
    exe = os.path.join(ROOT, "paper_2505_21070_b200", "lib", "blockpipe")
    r = subprocess.run([exe, "analyze", "bubble", "--N", "2", "--T", "8", "--blocks", "6"],
                       capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and r.stdout == "bubble N=2 T=8 blocks=6 order=reverse size=1 ratio=0.020408\n"
    r = subprocess.run([exe, "plan", "--out", str(tmp_path / "o")], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and (tmp_path / "o" / "summary.json").exists()


def test_python_module_entry_point():
    r = subprocess.run(["python", "-m", "paper_2505_21070_b200", "analyze", "bubble"], cwd=ROOT,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "size=11" in r.stdout


# ---- `_blockpipe` host surface (P/tests/python/test_smoke.py, no-GPU subset) ------------------
def test_blockpipe_compat_host_functions():
    import _blockpipe as bpc
    assert bpc.bubble_size(4, 50, 4) == 11
    assert bpc.method_cost("dualparal", num_b=8, num_c=8, height=4, width=4, hidden=8)["comm_scalars"] == 3072
    r = bpc.RandomSource(1)
    assert [r.next_u64() for _ in range(3)] == [0x910a2dec89025cc1, 0xbeeb8da1658eec67, 0xf893a2eefb32555e]
    ids = bpc.coordinated_noise_ids(num_b=8, num_c=8, appends=50)
    assert sorted(ids[0]) == list(range(12))
    for prev, nxt in zip(ids, ids[1:]):
        window = set(prev[-4:])
        assert window.isdisjoint(nxt) and window | set(nxt) == set(range(12))


def test_blockpipe_compat_permutation_vs_reference(ref):
    import _blockpipe as bpc
    for seed in (1, 7, 123456789):
        assert bpc.RandomSource(seed).permutation(17) == ref.permutation(seed, 17).tolist()
