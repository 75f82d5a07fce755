#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/ab.jsonl
for c in 0 1 2 3; do echo -n "{\"cfg\": $c, \"r\": " >> gpurun_out/ab.jsonl; PROTOX_BULK_CFG=$c timeout 200 python scripts/ab_relax.py --n 16384 --reps 40 >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err || echo null >> gpurun_out/ab.jsonl; sed -i '$ s/$/}/' gpurun_out/ab.jsonl; done
for c in 0 1 2; do echo -n "{\"cfg9_8192\": $c, \"r\": " >> gpurun_out/ab.jsonl; PROTOX_BULK_CFG=$c timeout 200 python scripts/ab_relax.py --n 8192 --reps 40 --stencil 1 >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err || echo null >> gpurun_out/ab.jsonl; sed -i '$ s/$/}/' gpurun_out/ab.jsonl; done
for c in 0 1 2; do echo -n "{\"cfg_solve\": $c, \"r\": " >> gpurun_out/ab.jsonl; PROTOX_BULK_CFG=$c timeout 200 python scripts/ab_solve.py --n 16384 --tk 1 --reps 5 >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err || echo null >> gpurun_out/ab.jsonl; sed -i '$ s/$/}/' gpurun_out/ab.jsonl; done
