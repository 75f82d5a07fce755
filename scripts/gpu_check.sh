#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/ab.jsonl
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.sw_power_cap --format=csv -lms 100 > gpurun_out/clocks_ab.csv &
SMI=$!
for sw in 20 100 400; do
  timeout 300 python scripts/ab_solve.py --n 16384 --tk 1 --sweeps $sw --reps 3 >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
done
timeout 300 python scripts/ab_relax.py --n 16384 --reps 200 >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
kill $SMI
timeout 900 python scripts/order_ladder.py > gpurun_out/ladder.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_tb -c 1 \
  -o gpurun_out/prof_tb_c4 -f python scripts/ab_solve.py --n 32768 --tk 4 --sweeps 4 --reps 1 > /dev/null 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
