#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/ab.jsonl
timeout 200 python scripts/ab_relax.py --n 8192 --reps 25 --stencil 1 >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
timeout 200 python scripts/ab_relax.py --n 8192 --reps 25 --stencil 0 >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
timeout 200 python scripts/ab_relax.py --n 16384 --reps 25 --stencil 0 >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
timeout 200 python scripts/ab_solve.py --n 16384 --tk 4 --every 4 >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
timeout 200 python scripts/ab_solve.py --n 32768 --tk 4 --every 4 >> gpurun_out/ab.jsonl 2>>gpurun_out/ab.err
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
