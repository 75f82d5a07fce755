#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 250 --csv \
  --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_bulk -s 3 -c 1 \
  -o gpurun_out/prof_bulk_final -f python scripts/ab_relax.py --n 16384 --reps 5 > /dev/null 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_tb -c 1 \
  -o gpurun_out/prof_tb_final -f python scripts/ab_solve.py --n 16384 --tk 4 --sweeps 4 --reps 1 > /dev/null 2>&1
PROTOX_KERNEL=ldg timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_stream -s 3 -c 1 \
  -o gpurun_out/prof_ldg_final -f python scripts/ab_relax.py --n 16384 --reps 5 > /dev/null 2>&1
