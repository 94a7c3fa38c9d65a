"""FFN-up GEMM shape with each epilogue (bf16 store, erf-GELU, fp32 store):\nthe cost of the epilogue over the mainloop.  python tools/gemm_epilogue_probe.py"""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from kernels import load_testlib
lib = load_testlib()
ms = ctypes.c_double()
for epi, tag in ((0, "store"), (1, "gelu"), (3, "f32 store")):
    assert lib.bp_bench_gemm(0, 18720, 8960, 1536, epi, 20, ctypes.byref(ms)) == 0
    print(f"ffn1 shape epi={tag:9s} ms {ms.value:.4f} TF {2*18720*8960*1536/ms.value/1e9:.1f}")
