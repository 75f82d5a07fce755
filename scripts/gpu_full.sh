#!/bin/bash
# Full GPU check: pytest -m gpu, smoke(), bench lines for C3 (default) and C4.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
timeout 600 python bench.py --config C4 --no-cpu-baseline > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log gpurun_out/bench_C3.json gpurun_out/bench_C4.json
