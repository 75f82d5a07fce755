#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/ab.jsonl
for nw in 8 16; do
  for ev in 1 4; do
    echo -n "{\"nw\": $nw, \"r\": " >> gpurun_out/ab.jsonl
    PROTOX_TB_NW=$nw timeout 200 python scripts/ab_solve.py --n 16384 --tk 4 --every $ev >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err || echo null >> gpurun_out/ab.jsonl
    sed -i '$ s/$/}/' gpurun_out/ab.jsonl
  done
done
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
