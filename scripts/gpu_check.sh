#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mg.py -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_mg.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_mg.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "resident or config2 or ragged" > gpurun_out/pytest_res.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_res.log
timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
