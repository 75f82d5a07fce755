#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/ab.jsonl
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
PROTOX_BULK_NST=5 timeout 200 python scripts/ab_relax.py --n 16384 >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
PROTOX_KERNEL=ldg timeout 200 python scripts/ab_relax.py --n 16384 >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
timeout 200 python scripts/ab_relax.py --n 16384 >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
