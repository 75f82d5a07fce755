#!/bin/bash
# A/B sweep of the TMA relax kernel knobs at 16384^2 (results: gpurun_out/sweep.jsonl)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/sweep.jsonl
for nst in 3 5 7; do for st in 0 1; do for ch in 64 256 1024; do
  echo -n "{\"nst\": $nst, \"store\": $st, \"chunk\": $ch, \"r\": " >> gpurun_out/sweep.jsonl
  PROTOX_BULK_NST=$nst PROTOX_BULK_STORE=$st PROTOX_BULK_CHUNK=$ch timeout 120 python scripts/ab_relax.py --n 16384 --reps 25 >> gpurun_out/sweep.jsonl 2>>gpurun_out/sweep.err || echo "null" >> gpurun_out/sweep.jsonl
  sed -i '$ s/$/}/' gpurun_out/sweep.jsonl
done; done; done
PROTOX_CEILING=1 timeout 200 python scripts/ab_relax.py --n 16384 > gpurun_out/ceiling.jsonl 2>>gpurun_out/sweep.err
