# BJ.C2 per-sweep time of diagnostic builds of k_resident (scripts/build_variant.py):
# rsd1 = no tag wait (compute + barrier floor), rsd2 = no row compute (handshake floor)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for v in ${VARIANTS:-default rsd1 rsd2 default rsd1 rsd2}; do
  lib=""; [ "$v" != default ] && lib=paper_2307_07931_b200/libprotox_$v.so
  PROTOX_LIB=$lib timeout 300 python bench.py --config C2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), round(d['roofline']['solve_kernel']['us_per_sweep'],3))"
done
