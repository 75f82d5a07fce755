#!/bin/bash
# ncu --set full of one temporal-blocking pass (wide and narrow kernels), 16384^2, k=4.
# The reports are summarised on the box (raw metrics, details, SASS source page).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for impl in ${TB_IMPLS:-wide narrow}; do
  R=/tmp/prof_tb_$impl
  PROTOX_TB_IMPL=$impl timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_tb -s 1 -c 1 \
    -o $R -f python scripts/ab_solve.py --n ${TB_N:-16384} --tk 4 --sweeps 8 --every 4 --reps 1 --nograph \
    > gpurun_out/prof_tb_$impl.log 2>&1
  $NCU -i $R.ncu-rep --page raw --csv > gpurun_out/prof_tb_${impl}_raw.csv 2>&1
  $NCU -i $R.ncu-rep --page details > gpurun_out/prof_tb_${impl}_details.txt 2>&1
  $NCU -i $R.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_tb_${impl}_sass.csv 2>&1
  gzip -f gpurun_out/prof_tb_${impl}_sass.csv
done
ls -la gpurun_out
