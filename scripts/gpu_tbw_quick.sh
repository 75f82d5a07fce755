#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/tbwq.log; : > $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "temporal or relax_block" >> $O 2>&1; echo "pytest exit $?" >> $O
for n in 16384 32768; do timeout 300 python scripts/ab_solve.py --n $n --tk 4 --sweeps 100 --every 4 >> $O 2>&1; done
TB_IMPLS=wide bash scripts/prof_tb.sh > /dev/null 2>&1
cat $O | tail -4
