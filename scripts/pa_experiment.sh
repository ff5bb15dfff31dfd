#!/bin/bash
# Pre-aggregated scatter (RAV_SCHUR_PA) against the default: sweep kernel alone (c2, c3), the c2
# bench step, and the oracle parity tests with the variant on.  Usage: bash scripts/pa_experiment.sh TAG
TAG=${1:-pa}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for rep in 1 2; do
  for PA in 0 1; do
    for C in c2 c3; do
      echo "PA=$PA $C: $(RAV_SCHUR_PA=$PA python scripts/sweep_variants.py $C | tail -1)"
    done
  done
done 2>&1 | tee $OUT/sweep.txt
for PA in 0 1 0 1; do
  RAV_SCHUR_PA=$PA timeout 300 python bench.py --no-cpu-baseline --no-vcycle --no-smoothers 2>/dev/null |
    python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('PA=$PA', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'])"
done 2>&1 | tee $OUT/bench.txt
RAV_SCHUR_PA=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schur.py tests/test_gpu_batch.py tests/test_gpu_residual_table.py -m gpu -q -x > $OUT/pytest_pa1.log 2>&1; echo "pytest PA=1 rc=$?"; tail -3 $OUT/pytest_pa1.log
