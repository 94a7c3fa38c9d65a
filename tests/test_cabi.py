"""The C-ABI library loads on a CPU-only host, exports every function the
public headers declare, and refuses compute without a GPU (no CPU fallback)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for h in ("bp_cuda.h", "bp_cuda_test.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(bp_[a-z0-9_]+)\s*\(", text):
            if not m.group(1).endswith("_fn"):
                names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol(bp):
    from paper_2505_21070_b200 import _lib
    names = declared_functions()
    assert len(names) >= 39
    for n in sorted(names):
        assert hasattr(_lib.lib, n), n
    assert set(_lib.EXPORTED) <= names


def test_compute_entry_points_fail_loudly_without_gpu(bp):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(bp.CudaError):
        bp.normals(1, 10)
    with pytest.raises(bp.CudaError):
        bp.run_pipeline({"devices": 1})
