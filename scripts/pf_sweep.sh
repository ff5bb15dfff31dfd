#!/bin/bash
# RAV_SCHUR_PF (rectangular blocks bulk-prefetched ahead in the thread sweep) re-tuned after the
# pre-aggregated scatter: sweep kernel alone at c2 / c3, then the c2 bench step.
OUT=gpurun_out/${1:-pf}
mkdir -p $OUT
for rep in 1 2; do
  for PF in 0 1 2; do
    for C in c2 c3; do
      echo "PF=$PF $C: $(RAV_SCHUR_PF=$PF python scripts/sweep_variants.py $C | tail -1)"
    done
  done
done 2>&1 | tee $OUT/pf_sweep.txt
bash scripts/env_sweep.sh ${1:-pf} "RAV_SCHUR_PF=0 RAV_SCHUR_PF=1 RAV_SCHUR_PF=2"
