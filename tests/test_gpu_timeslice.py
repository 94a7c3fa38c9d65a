"""Determinism while another process time-slices the GPU. Two processes run
the production-shape pipeline (Wan2.1-1.3B width, 480p grid, 4 layers, 2
blocks x 2 steps) concurrently on one device and every run must equal the
run made alone, bitwise. Time-slicing stretches the tensor pipe relative to
the warps; it exposed a parity-aliased mbarrier wait in the pair attention's
epilogue (attn_sm100.cu, o_done), which this test guards."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "tools", "dbg_timeslice.py")


def test_runs_equal_under_time_slicing(tmp_path):
    env = dict(os.environ, CUDA_MODULE_LOADING="EAGER", PYTHONPATH=ROOT)
    ref = str(tmp_path / "ref.npy")
    subprocess.run([sys.executable, TOOL, "ref", ref], cwd=ROOT, env=env, check=True, timeout=600)
    procs = [subprocess.Popen([sys.executable, TOOL, "check", ref, "4"], cwd=ROOT, env=env, stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for _ in range(2)]
    outs = [p.communicate(timeout=900)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), outs
    lines = [ln for o in outs for ln in o.splitlines() if " equal" in ln or "DIFF" in ln]
    assert len(lines) == 8 and all(ln.endswith("equal") for ln in lines), outs
