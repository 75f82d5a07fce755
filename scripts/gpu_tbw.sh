#!/bin/bash
# Temporal blocking: wide vs narrow kernel A/B + parity tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/tbw.log; : > $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "temporal or relax_block or self_exchange" >> $O 2>&1; echo "pytest exit $?" >> $O
for impl in wide narrow; do
  for n in 16384 32768; do
    PROTOX_TB_IMPL=$impl timeout 300 python scripts/ab_solve.py --n $n --tk 4 --sweeps 100 --every 4 >> $O 2>&1
  done
done
timeout 300 python scripts/ab_solve.py --n 8192 --tk 4 --sweeps 100 --every 1 --stencil 1 --bc 1 >> $O 2>&1
timeout 300 python scripts/ab_solve.py --n 8192 --tk 1 --sweeps 100 --every 1 --stencil 1 --bc 1 >> $O 2>&1
timeout 300 python scripts/ab_solve.py --n 8192 --tk 4 --sweeps 100 --every 4 --stencil 1 --bc 1 >> $O 2>&1
cat $O | tail -20
