python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { echo "$1"; env $1 timeout 300 python scripts/sweep_variants.py c2 2>&1 | tail -1; }
run "RAV_SCHUR_NRB=0 RAV_SCHUR_MINB=4"
run "RAV_SCHUR_NRB=1 RAV_SCHUR_MINB=4"
run "RAV_SCHUR_NRB=1 RAV_SCHUR_MINB=3"
run "RAV_SCHUR_NRB=1 RAV_SCHUR_MINB=5"
