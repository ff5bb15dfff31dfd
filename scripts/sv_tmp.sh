for cfg in c2 c5; do
for m in 0 1 2 3 4; do RAV_SCHUR_SPLIT=$m python scripts/sweep_variants.py $cfg; done
done
