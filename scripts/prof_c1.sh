cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_cluster_box -c 1 -o /tmp/c1 -f python bench.py --config C1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/c1prof.log 2>&1
/usr/local/cuda/bin/ncu -i /tmp/c1.ncu-rep --page raw --csv > gpurun_out/c1_raw.csv 2>&1
/usr/local/cuda/bin/ncu -i /tmp/c1.ncu-rep --page source --csv --print-source sass > gpurun_out/c1_sass.csv 2>&1; gzip -f gpurun_out/c1_sass.csv
/usr/local/cuda/bin/ncu -i /tmp/c1.ncu-rep --page details > gpurun_out/c1_details.txt 2>&1
