cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nan.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "temporal or tb or tbw or C4 or config4" 2>&1 | tail -2
for v in base swz base swz; do
L=paper_2307_07931_b200/libprotox.so; [ $v = swz ] && L=paper_2307_07931_b200/libprotox_swz.so
PROTOX_LIB=$L timeout 400 python bench.py --config C4 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', round(d['value'],1), 'kernel_ms', round(r['kernel_ms'],3), 'step_ms', round(d['ms_per_step'],1), d['clocks']['sm_mhz'])"
done
