cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_nan.py -m gpu -q -p no:cacheprovider 2>&1 | tail -2
for i in 1 2 3; do
for v in base cur; do
L=paper_2307_07931_b200/libprotox.so; [ $v = base ] && L=paper_2307_07931_b200/libprotox_base.so
PROTOX_LIB=$L timeout 400 python bench.py --no-cpu-baseline --no-e2e --no-halo-proxy 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', round(d['value'],2), 'kernel_ms', round(r['kernel_ms'],4), 'step_ms', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['gpu_launches'])"
done
done
