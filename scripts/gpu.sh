#!/bin/bash
# GPU-box driver for gpurun (one GPU).  Writes under gpurun_out/.
#   bash scripts/gpu.sh check            build + smoke + the whole -m gpu suite
#   bash scripts/gpu.sh bench [CFG...]   bench.py lines (default C3 C4 C2 C1 C5 C3D)
#   bash scripts/gpu.sh overhead [P...]  per-sweep halo-path overheads at the P-rank slab shapes
#   bash scripts/gpu.sh launches [CFG]   ncu launch list of a short bench run (per-launch device times)
#   bash scripts/gpu.sh full KREGEX SKIP SCRIPT ARGS...   one ncu --set full capture of a kernel
#   bash scripts/gpu.sh sanitize [CASE...]                compute-sanitizer over scripts/sanitize_cases.py
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
cmd=${1:-check}; shift || true
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
case "$cmd" in
  check)
    nvidia-smi -L > gpurun_out/host.txt; nproc >> gpurun_out/host.txt
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
    timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
    tail -15 gpurun_out/pytest_gpu.log ;;
  bench)
    cfgs=${*:-C3 C4 C2 C1 C5 C3D}
    for c in $cfgs; do
      extra=""; [ "$c" != "C3" ] && extra="--no-cpu-baseline"
      timeout 900 python bench.py --config $c $extra > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
      echo "$c: $(tail -c 300 gpurun_out/bench_$c.json)"
    done ;;
  overhead)
    timeout 900 python scripts/slab_overhead.py ${*:-8 4 2 1} 2>&1 | grep '{' | tee gpurun_out/slab_overhead.jsonl ;;
  launches)
    c=${1:-C3}
    timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
      --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline \
      --no-e2e --no-halo-proxy > gpurun_out/launches_$c.log 2>&1
    python scripts/summarize_ncu.py --launches gpurun_out/launches_$c.csv round2_launches_$c | tail -20
    mkdir -p gpurun_out/profiles; cp profiles/round2_launches_$c.json gpurun_out/profiles/ ;;
  full)
    k=$1; skip=$2; shift 2
    timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 \
      -o gpurun_out/full_$k -f python "$@" > gpurun_out/full_$k.log 2>&1
    tail -3 gpurun_out/full_$k.log ;;
  sanitize)
    CS=/usr/local/cuda/bin/compute-sanitizer
    cases=${*:-all}
    for tool in memcheck racecheck synccheck initcheck; do
      for c in $cases; do
        timeout 900 $CS --tool $tool --print-limit 10 python scripts/sanitize_cases.py $c > gpurun_out/sanitize_${tool}_$c.log 2>&1
        echo "$tool $c exit $? $(grep -h 'ERROR SUMMARY' gpurun_out/sanitize_${tool}_$c.log | tail -1)"
      done
    done ;;
  *) echo "unknown command $cmd"; exit 2 ;;
esac
