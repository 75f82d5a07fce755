#!/bin/bash
# ncu --set full captures summarised on the box: the 27-point 3D kernel, the cluster small-box kernel (C1),
# and five repeated C3 bench lines (run-to-run spread).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/profiles
NCU=/usr/local/cuda/bin/ncu
cat > /tmp/k27.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2307_07931_b200 import protox as P
n = 512
g = P.Grid3((n, n, n), 1)
a, b, r = g.alloc(), g.alloc(), g.alloc()
P.init_field3(g, r, 1, 20230714)
prm = P.relax_params(1 / n, (1 / n) ** 2 / 12, P.PX_MEHRSTELLEN_27PT_3D)
nb = P.norm_buffer3()
for i in range(3):
    P.fill_ghosts3(g, 1, a)
    P.relax_step3(prm, g, a, b, r, nb)
torch.cuda.synchronize()
PY
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k3_relax -s 1 -c 1 -o /tmp/p27 -f python /tmp/k27.py > gpurun_out/p27.log 2>&1
python scripts/summarize_ncu.py round1_ncu_k3_relax27_512 /tmp/p27.ncu-rep C3D27 3221225472 > gpurun_out/p27_sum.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_cluster_box -c 1 -o /tmp/pc1 -f python bench.py --config C1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/pc1.log 2>&1
python scripts/summarize_ncu.py round1_ncu_k_cluster_box_c1 /tmp/pc1.ncu-rep > gpurun_out/pc1_sum.log 2>&1
cp profiles/round1_ncu_k3_relax27_512.json profiles/round1_ncu_k_cluster_box_c1.json profiles/relax_traffic.json gpurun_out/profiles/
for i in 1 2 3 4 5; do timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/c3_rep_$i.json 2>/dev/null; done
for i in 1 2 3 4 5; do python -c "import json; d=json.load(open('gpurun_out/c3_rep_$i.json')); print(d['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"; done
