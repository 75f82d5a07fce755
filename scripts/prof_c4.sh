#!/bin/bash
# ncu --set full of the C4 temporal-blocking pass (32768^2, k=4), summarised on the box
# into gpurun_out/profiles/ (profiles/*.json + relax_traffic.json C4 entry).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/profiles
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_tb -s 1 -c 1 \
  -o /tmp/prof_tb_c4 -f python scripts/ab_solve.py --n 32768 --tk 4 --sweeps 8 --every 4 --reps 1 --nograph \
  > gpurun_out/prof_c4.log 2>&1
python scripts/summarize_ncu.py ${NAME:-round1_ncu_k_tbw_k4_32768_C4} /tmp/prof_tb_c4.ncu-rep C4 25769803776 > gpurun_out/prof_c4_summary.log 2>&1
cp profiles/${NAME:-round1_ncu_k_tbw_k4_32768_C4}.json profiles/relax_traffic.json gpurun_out/profiles/
