#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_p2p_ipc.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "p2p or self_exchange or nccl" > gpurun_out/pytest_p2p.log 2>&1
tail -3 gpurun_out/pytest_p2p.log
timeout 300 python scripts/slab_overhead.py 8 4 2 1 2>&1 | grep '{'
