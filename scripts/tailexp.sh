python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for t in 0 1; do echo "NDC=$t"; RAV_SCHUR_NDC=$t timeout 120 python scripts/sweep_variants.py c2 | tail -1; RAV_SCHUR_NDC=$t timeout 120 python scripts/sweep_variants.py c3 | tail -1; RAV_SCHUR_NDC=$t timeout 300 python bench.py --steps 10 --warmup 3 --no-vcycle --no-smoothers --no-paper --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline'])"; done
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
