# BJ.C3 A/B: periodic images read in place by k_bulk (PROTOX_WRAP=1) vs per-sweep ghost fill (0),
# with and without programmatic dependent launches (PROTOX_PDL)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for v in "1 1" "0 1" "1 0" "0 0" "1 1" "0 1" "1 0" "0 0"; do
set -- $v
PROTOX_WRAP=$1 PROTOX_PDL=$2 timeout 400 python bench.py --config C3 --no-cpu-baseline --no-e2e --no-halo-proxy 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; c=d['clocks']; print('wrap$1 pdl$2', round(d['value'],2), 'step_ms', round(d['ms_per_step'],3), 'kernel_ms', round(r['kernel_ms'],4), c['sm_mhz'], c.get('power_w'), d['gpu_launches'])"
done
