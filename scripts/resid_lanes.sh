# Residual lanes-per-row re-check with the B-value table (2D: G = 1 default at large levels)
for cfg in c2 c3; do
  for env in "RAV_NB_LANES=0" "RAV_NB_LANES=2" "RAV_NB_LANES=4" "RAV_NB_LANES=2 RAV_NB_BS=256"; do
    echo -n "$cfg $env: "; env $env python scripts/resid_variants.py $cfg 2>&1 | grep residual
  done
done
