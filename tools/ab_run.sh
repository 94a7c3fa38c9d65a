#!/bin/bash
# Same-box A/B of kernel-library variants built by tools/ab_build.sh, interleaved:
#   tools/ab_run.sh gemm "pf0 pf8" [rounds]     isolated GEMMs (tools/bench_kernels.py gemm 20)
#   tools/ab_run.sh step "pf0 pf8" [rounds]     81-frame video in the step (bench.py --workload wan13-81)
ROOT=$(cd "$(dirname "$0")/.." && pwd)
what=$1; variants=$2; rounds=${3:-2}
for r in $(seq "$rounds"); do
  for v in $variants; do
    if [ "$what" = gemm ]; then
      echo "== $v"; BP_TESTLIB_PATH=$ROOT/ablib/$v/libbp_cuda_test.so python "$ROOT/tools/bench_kernels.py" gemm 20
    else
      BP_LIB_PATH=$ROOT/ablib/$v/libbp_cuda.so python "$ROOT/bench.py" --workload wan13-81 --steps 1 --warmup 3 2>/dev/null |
        python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); b=d.get('step_breakdown_s',{}); print('$v', round(d['ms_per_step'],1), {k: round(x,3) for k,x in b.items()}, d.get('clocks',{}).get('sm_mhz'))"
    fi
  done
done
