#!/bin/bash
# One GPU session: build, gpu tests, smoke, bench, ncu launch list + full captures.
# Usage (from repo root, under gpurun): bash scripts/gpu_round.sh TAG [skip-tests]
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
(nproc; lscpu | grep "Model name"; free -g) > $OUT/host.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > $OUT/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build.log; exit 1; }
if [ "$2" != "skip-tests" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -x --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 $OUT/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log
fi
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; tail -c 3000 $OUT/bench.json
if [ "$NCU" != "0" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/launches.csv \
     python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-vcycle --no-smoothers > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
  for K in ${NCU_KERNELS:-schur_sweep_thread_kernel nb_residual_kernel}; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 5 -c 1 -o $OUT/prof_$K \
       python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-vcycle --no-smoothers > $OUT/ncu_$K.log 2>&1; echo "ncu $K rc=$?"
  done
fi
