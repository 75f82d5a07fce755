#!/bin/bash
# Full GPU validation after this session's changes + the host CPU-fusion ratio on the GPU box.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
timeout 600 python scripts/cpu_fusion_ratio.py gpurun_out/cpu_fusion_ratio_gpubox.json > gpurun_out/cpu_ratio.log 2>&1
nproc > gpurun_out/host.txt; lscpu | head -20 >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log; cut -c1-300 gpurun_out/bench_C3.json; tail -4 gpurun_out/cpu_ratio.log
