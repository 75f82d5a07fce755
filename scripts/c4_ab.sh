# BJ.C4 A/B: the default k_tbw against a variant build (scripts/build_variant.py NAME px_tb.cu FLAGS)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
V=${VARIANT:-noidle}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nan.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "temporal or tb or tbw or C4 or config4" 2>&1 | tail -2
for v in base $V base $V; do
L=paper_2307_07931_b200/libprotox.so; [ $v != base ] && L=paper_2307_07931_b200/libprotox_$v.so
PROTOX_LIB=$L timeout 400 python bench.py --config C4 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; c=d['clocks']; print('$v', round(d['value'],1), 'kernel_ms', round(r['kernel_ms'],3), 'step_ms', round(d['ms_per_step'],1), c['sm_mhz'], c.get('power_w'), c.get('power_limit_w'))"
done
