#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/ab_comm.jsonl
for n in 16384 4096 2048; do timeout 300 python scripts/ab_comm.py $n >> gpurun_out/ab_comm.jsonl 2>> gpurun_out/ab_comm.err; done
