cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mg.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"
for v in 1 2 0; do PROTOX_SMALLBOX=$v timeout 300 python bench.py --config C1 --no-cpu-baseline --no-e2e > gpurun_out/bench_C1_$v.json 2>gpurun_out/bench_C1_$v.err; python -c "import json; d=json.load(open('gpurun_out/bench_C1_$v.json')); print('variant $v', d['value'], d['ms_per_step'])"; done
