"""cuBLAS (torch) on the pass's GEMM shapes, for comparison with
tools/bench_kernels.py gemm:  python tools/cublas_compare.py
Like for like with the stage's epilogues: QKV / cross-Q as a bf16 store,
FFN-up as a bf16 store (cuBLAS has no erf-GELU epilogue; ours pays for it),
and the residual projections (O, cross-O, FFN-down) as fp32 C += A.B
(addmm with out_dtype fp32, beta 1: the same fp32 read-modify-write of the
residual stream our TMA reduce-add epilogue does). The plain bf16-store
timing of the residual shapes is printed too."""
import torch

torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = True
shapes = [("qkv", 18720, 4608, 1536, "bf16"), ("o", 18720, 1536, 1536, "resid"), ("ffn1", 18720, 8960, 1536, "bf16"),
          ("ffn2", 18720, 1536, 8960, "resid"), ("o", 18720, 1536, 1536, "bf16"), ("ffn2", 18720, 1536, 8960, "bf16")]


def timed(fn, iters=20):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


for name, M, N, K, kind in shapes:
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16).t()  # K-major weight, like the stage's
    if kind == "resid":
        x = torch.randn(M, N, device="cuda", dtype=torch.float32)
        ms = timed(lambda: torch.addmm(x, a, b, out_dtype=torch.float32, out=x))
    else:
        c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        ms = timed(lambda: torch.matmul(a, b, out=c))
    print(f"cublas {name:5s} {kind:5s} {M}x{N}x{K} ms {ms:.4f} TF {2 * M * N * K / ms / 1e9:.1f}", flush=True)
