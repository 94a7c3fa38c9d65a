"""cuBLAS (torch.matmul, bf16) on the pass's GEMM shapes, for comparison with
tools/bench_kernels.py gemm:  python tools/cublas_compare.py"""
import torch, time
torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = True
shapes = [("qkv",18720,4608,1536),("o",18720,1536,1536),("ffn1",18720,8960,1536),("ffn2",18720,1536,8960)]
for name,M,N,K in shapes:
    a=torch.randn(M,K,device="cuda",dtype=torch.bfloat16); b=torch.randn(K,N,device="cuda",dtype=torch.bfloat16)
    c=torch.empty(M,N,device="cuda",dtype=torch.bfloat16)
    for _ in range(5): torch.matmul(a,b,out=c)
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): torch.matmul(a,b,out=c)
    e1.record(); torch.cuda.synchronize()
    ms=e0.elapsed_time(e1)/20
    print(f"cublas {name:5s} {M}x{N}x{K} ms {ms:.4f} TF {2*M*N*K/ms/1e9:.1f}")
