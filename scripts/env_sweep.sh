#!/bin/bash
# c2 bench step under tuning-switch settings (each setting twice, interleaved).  Usage: bash scripts/env_sweep.sh TAG "VAR=a VAR=b ..."
TAG=${1:-env}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for rep in 1 2; do
  for S in $2; do
    env $S timeout 300 python bench.py --no-cpu-baseline --no-vcycle --no-smoothers 2>/dev/null |
      python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('$S', round(d['value'],1), round(d['ms_per_step'],4), round(d['roofline']['frac'],4), round(d['roofline']['kernel_ms']*1e3,2), round(d['residual_kernel']['ms']*1e3,2))"
  done
done 2>&1 | tee $OUT/env_sweep.txt
