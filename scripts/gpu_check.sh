#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool racecheck --print-limit 10 python scripts/sanitize_cases.py bulk_relax > gpurun_out/sanitize_racecheck_bulk.log 2>&1
timeout 200 python scripts/ab_relax.py --n 16384 --reps 25 > gpurun_out/ab_fence.jsonl 2>&1
