#!/bin/bash
# Final ncu evidence of the kernels bench.py times (round summary -> profiles/).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 250 --csv \
  --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 120 --csv \
  --log-file gpurun_out/launches_c4.csv python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_bulk -s 3 -c 1 \
  -o gpurun_out/prof_bulk_c3 -f python scripts/ab_relax.py --n 16384 --reps 5 > /dev/null 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_bulk -s 3 -c 1 \
  -o gpurun_out/prof_bulk_c5 -f python scripts/ab_relax.py --n 8192 --reps 5 --stencil 1 > /dev/null 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_tb -c 1 \
  -o gpurun_out/prof_tb_c4 -f python scripts/ab_solve.py --n 32768 --tk 4 --sweeps 4 --reps 1 --every 4 > /dev/null 2>&1
