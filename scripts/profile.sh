#!/bin/bash
# ncu evidence: the launch list of the bench (per-launch device times,
# cold-cache, serialised) and one --set full capture of each relax kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 450 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
  > gpurun_out/launches_bench.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_bulk -s 3 -c 1 \
  -o gpurun_out/prof_bulk -f python scripts/ab_relax.py --n 16384 --reps 5 > gpurun_out/prof_bulk.log 2>&1
PROTOX_KERNEL=ldg timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_stream -s 3 -c 1 \
  -o gpurun_out/prof_ldg -f python scripts/ab_relax.py --n 16384 --reps 5 > gpurun_out/prof_ldg.log 2>&1
