#!/bin/bash
# Round evidence: full GPU tests, smoke, bench lines (C3 default, C4, C5), launch lists.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
for c in ${CONFIGS:-C3 C4 C5}; do
  extra=""; [ "$c" != "C3" ] && extra="--no-cpu-baseline"
  timeout 600 python bench.py --config $c $extra > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
if [ -n "$LAUNCHES" ]; then
  for c in $LAUNCHES; do
    timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
      --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
      > gpurun_out/launches_$c.log 2>&1
  done
fi
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log; for c in ${CONFIGS:-C3 C4 C5}; do cut -c1-400 gpurun_out/bench_$c.json; done
