# Residual kernel register cap / block size re-check with the B-value table (DESIGN 5.1b)
for cfg in c2 c3 c4; do
  for env in "RAV_NB_MINB=6" "RAV_NB_MINB=5" "RAV_NB_MINB=8" "RAV_NB_MINB=1" "RAV_NB_BS=256" "RAV_NB_MINB=5 RAV_NB_BS=256"; do
    echo -n "$cfg $env: "; env $env python scripts/resid_variants.py $cfg 2>&1 | grep residual
  done
done
