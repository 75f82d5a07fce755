#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/ab.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "temporal or relax_block" > gpurun_out/pytest_tb.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_tb.log
timeout 600 python scripts/diag_tb2.py > gpurun_out/diag_tb2.log 2>&1
for nw in 7 15; do
  for ev in 1 4; do
    echo -n "{\"nw\": $nw, \"r\": " >> gpurun_out/ab.jsonl
    PROTOX_TB_NW=$nw timeout 200 python scripts/ab_solve.py --n 16384 --tk 4 --every $ev >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err || echo null >> gpurun_out/ab.jsonl
    sed -i '$ s/$/}/' gpurun_out/ab.jsonl
  done
done
echo -n "{\"nw\": 152, \"r\": " >> gpurun_out/ab.jsonl; timeout 200 python scripts/ab_solve.py --n 16384 --tk 2 --every 4 >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err; sed -i '$ s/$/}/' gpurun_out/ab.jsonl
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_tb -c 1 \
  -o gpurun_out/prof_tb_v3 -f python scripts/ab_solve.py --n 16384 --tk 4 --sweeps 4 --reps 1 --every 4 > /dev/null 2>&1
