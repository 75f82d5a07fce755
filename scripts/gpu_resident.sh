#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "resident or config2 or config1 or ragged or norm_every or host" > gpurun_out/pytest_res.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_res.log
for k in 1 2 3; do PROTOX_RESIDENT_K=$k timeout 300 python bench.py --config C2 --no-cpu-baseline --no-e2e > gpurun_out/bench_C2_k$k.json 2> gpurun_out/bench_C2_k$k.err; done
tail -3 gpurun_out/pytest_res.log
for k in 1 2 3; do python -c "import json; d=json.load(open('gpurun_out/bench_C2_k$k.json')); print('K=$k', d['value'], d['ms_per_step'])"; done
