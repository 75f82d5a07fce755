#!/bin/bash
# round-2 validation pass: smoke, GPU parity suite, slab overhead, C3 bench
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/host.txt; nproc >> gpurun_out/host.txt; lscpu | grep "Model name" >> gpurun_out/host.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -30 gpurun_out/pytest_gpu.log
timeout 600 python scripts/slab_overhead.py > gpurun_out/slab_overhead.jsonl 2>&1
cat gpurun_out/slab_overhead.jsonl
timeout 600 python bench.py > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
cat gpurun_out/bench_C3.json
