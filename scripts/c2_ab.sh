cd "${GRAFT_REPO_ROOT:-/root/repo}"
for v in 0 32 100 300 0 100; do
PROTOX_LIB=paper_2307_07931_b200/libprotox_ll$v.so timeout 300 python bench.py --config C2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('ll$v', round(d['value'],1), round(d['roofline']['solve_kernel']['us_per_sweep'],3))"
done
