#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
bash scripts/sweep_bulk.sh
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 250 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
  > gpurun_out/launches_bench.log 2>&1
