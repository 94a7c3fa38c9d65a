"""Per-head relative error of one attention implementation on a fixed set of
shapes (a debugging aid):  python tools/attn_probe.py IMPL"""
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
from kernels import attn, ref_attn, to_bf16_bits, from_bf16_bits, DEFAULT_GEMM_IMPL, load_testlib
lib = load_testlib()
impl = int(sys.argv[1])
for (rows, n0, n1, heads) in [(96,0,512,3),(96,0,512,1),(128,0,512,3),(256,0,512,3),(96,0,448,3),(96,0,576,3),(96,0,512,2),(300,0,512,1),(96,0,256,3),(96,0,384,3)]:
    dh=128; rng=np.random.default_rng(rows+n0*3+n1+heads); H=heads*dh
    q=to_bf16_bits(rng.standard_normal((rows,H))); k1=to_bf16_bits(rng.standard_normal((n1,H))); v1=to_bf16_bits(rng.standard_normal((n1,H)))
    want=ref_attn(from_bf16_bits(q), from_bf16_bits(k1), from_bf16_bits(v1), heads, dh, 1/np.sqrt(dh))
    lib.bp_set_kernel_impl(DEFAULT_GEMM_IMPL, impl)
    got=from_bf16_bits(attn(lib,q,None,None,k1,v1,heads,dh,1/np.sqrt(dh))).astype(np.float64)
    per=[float(np.linalg.norm(got[:,h*dh:(h+1)*dh]-want[:,h*dh:(h+1)*dh])/np.linalg.norm(want[:,h*dh:(h+1)*dh])) for h in range(heads)]
    print(rows,n0,n1,heads, ["%.3g"%x for x in per])
