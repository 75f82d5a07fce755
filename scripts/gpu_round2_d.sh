#!/bin/bash
# PDL A/B (slab overhead), parity subset, C3 bench line (halo proxy, full-size oracle baseline)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_p2p_ipc.py tests/test_gpu_parity.py tests/test_gpu_nan.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_pdl.log 2>&1
tail -3 gpurun_out/pytest_pdl.log
PROTOX_PDL=0 timeout 300 python scripts/slab_overhead.py 8 1 2>&1 | grep '{' | sed 's/^/nopdl /'
timeout 300 python scripts/slab_overhead.py 8 4 2 1 2>&1 | grep '{' | sed 's/^/pdl /'
s=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; echo "bench wall $(( $(date +%s) - s )) s"
tail -c 2500 gpurun_out/bench_C3.json
