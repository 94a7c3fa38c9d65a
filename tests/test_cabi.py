"""The C-ABI library loads on a CPU-only host, exports every function the
public headers declare, and refuses compute without a GPU (no CPU fallback)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions(headers=("bp_cuda.h",)):
    names = set()
    for h in headers:
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


def test_operator_library_exports_every_declared_symbol(bp):
    """include/bp_operator.h is served by lib/libblockpipe_b200.so."""
    import ctypes
    from paper_2505_21070_b200 import operator
    names = declared_functions(("bp_operator.h",))
    assert {"bp_cli_main", "bp_write_artifacts", "bp_bubble", "bp_method_cost"} <= names
    lib = ctypes.CDLL(operator.OP_LIB_PATH)
    for n in sorted(names):
        assert hasattr(lib, n), n


def test_only_c_abi_is_exported(bp):
    """libbp_cuda.so is built with -fvisibility=hidden: its dynamic symbol
    table holds exactly the entry points include/bp_cuda.h declares (no
    internals, no test hooks). The kernel self-test hooks of
    include/bp_cuda_test.h live in the separate libbp_cuda_test.so."""
    import subprocess
    from paper_2505_21070_b200 import _lib

    def exported(path):
        out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
        return {ln.split()[-1] for ln in out.splitlines() if " T " in ln}

    assert exported(_lib.LIB_PATH) == declared_functions()
    load_testlib = os.path.join(os.path.dirname(_lib.LIB_PATH), "libbp_cuda_test.so")
    assert exported(load_testlib) == declared_functions(("bp_cuda.h", "bp_cuda_test.h"))


def test_compute_entry_points_fail_loudly_without_gpu(bp):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(bp.CudaError):
        bp.normals(1, 10)
    with pytest.raises(bp.CudaError):
        bp.run_pipeline({"devices": 1})
    import numpy as np
    with pytest.raises(bp.CudaError):
        bp.gather_block(np.zeros((6, 1, 1, 1)), [0])
    with pytest.raises(bp.CudaError):
        bp.draw_first_block("coordinated", np.zeros((6, 1, 1, 1)), 4, 4, 1)
    import _blockpipe
    import numpy as np
    for fn in (lambda: _blockpipe.matmul(np.eye(2), np.eye(2)), lambda: _blockpipe.softmax_rows(np.eye(2)),
               lambda: _blockpipe.layer_norm(np.eye(2)), lambda: _blockpipe.RandomSource(1).next_normal()):
        with pytest.raises(bp.CudaError):
            fn()
    from paper_2505_21070_b200 import operator
    code, out, err = operator.cli_main(["run", "--out", "/tmp/bp_nogpu_run"])
    assert (code, out) == (1, "") and "no CUDA device" in err, err


def test_integration_binding_stub_matches_the_abi():
    """The ctypes stub INTEGRATION.md section 3 shows a maintainer has the
    exact field layout of bp_pipeline_desc / bp_model_desc (the full binding
    is paper_2505_21070_b200/_lib.py)."""
    import ctypes as C
    import re
    from paper_2505_21070_b200 import _lib
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = text.split("## 3.")[1].split("```python")[1].split("```")[0]
    defs = code[code.index("class ModelDesc"):code.index("EMIT =")]
    ns = {"C": C}
    exec(defs, ns)
    for stub, real in ((ns["ModelDesc"], _lib.ModelDesc), (ns["PipelineDesc"], _lib.PipelineDesc)):
        assert [f[0] for f in stub._fields_] == [f[0] for f in real._fields_]
        assert C.sizeof(stub) == C.sizeof(real)
    assert re.search(r"ModelDesc\(([^)]*)\)", code.split("EMIT =")[1]).group(1).count(",") + 1 == \
        len(_lib.ModelDesc._fields_)
