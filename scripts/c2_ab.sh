# BJ.C2 A/B of the resident solve: k_resident_reg (iterate in registers, default) vs
# k_resident (shared-memory row walk, PROTOX_RESIDENT_REG=0)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for u in 1 0 1 0; do
PROTOX_RESIDENT_REG=$u timeout 300 python bench.py --config C2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('reg$u', round(d['value'],1), round(d['roofline']['solve_kernel']['us_per_sweep'],3), d['roofline']['solve_kernel'].get('kernel'))"
done
