"""The reference's C++ test cases compiled against the B200 C++ mirror
(include/blockpipe/, libblockpipe_b200.so) and run on the GPU."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_cpp_cases_against_mirror():
    exe = os.path.join(ROOT, "paper_2505_21070_b200", "lib", "test_api")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "goldens.json")))
    sumsq = float(out.stdout.split("sumsq ")[1].split()[0])
    assert abs(sumsq - g["cfg1"]["sumsq"]) <= 1e-12 * g["cfg1"]["sumsq"]
