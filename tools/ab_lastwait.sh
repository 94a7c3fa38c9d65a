# A/B of the pair attention's end-of-item synchronisation (lw0: the racy
# parity wait of the original build; odone: the one-phase o_done barrier)
for r in 1 2 3; do for v in lw0 odone odone2; do echo "== $v"; BP_TESTLIB_PATH=$PWD/ablib/$v/libbp_cuda_test.so python tools/bench_kernels.py attn 20 self; done; done > gpurun_out/r02y_ab_attn.txt 2>&1
tools/ab_run.sh step "lw0 odone2" 2 > gpurun_out/r02y_ab_step.txt 2>&1
