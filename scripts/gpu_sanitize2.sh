#!/bin/bash
# compute-sanitizer over the kernels added this session (k_tbw, k3_*), then the full case list under memcheck.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
rm -f gpurun_out/sanitize2_*.log
for tool in memcheck racecheck synccheck initcheck; do
  for c in tb_solve tb_dirichlet9_solve tb_fixed_k2_solve relax3_solve relax3_27_solve; do
    timeout 600 $CS --tool $tool --print-limit 10 python scripts/sanitize_cases.py $c >> gpurun_out/sanitize2_$tool.log 2>&1
    echo "$c exit $?" >> gpurun_out/sanitize2_$tool.log
  done
done
grep -h -E "ERROR SUMMARY|exit|Hazard|error" gpurun_out/sanitize2_*.log | sort | uniq -c | head -40
