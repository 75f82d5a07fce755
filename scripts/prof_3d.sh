#!/bin/bash
# 3D: bench line (C3D) + ncu --set full of one k3_relax launch at 512^3, summarised on the box.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/profiles
timeout 600 python bench.py --config C3D > gpurun_out/bench_C3D.json 2> gpurun_out/bench_C3D.err
NCU=/usr/local/cuda/bin/ncu
cat > /tmp/k3one.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2307_07931_b200 import protox as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = P.Grid3((n, n, n), 1)
a, b, r = g.alloc(), g.alloc(), g.alloc()
P.init_field3(g, r, 1, 20230714)
prm = P.relax_params(1 / n, (1 / n) ** 2 / 12, P.PX_LAPLACE_7PT_3D)
nb = P.norm_buffer3()
for i in range(3):
    P.fill_ghosts3(g, 0, a)
    P.relax_step3(prm, g, a, b, r, nb)
torch.cuda.synchronize()
PY
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k3_relax -s 1 -c 1 \
  -o /tmp/prof_k3 -f python /tmp/k3one.py 512 > gpurun_out/prof_k3.log 2>&1
python scripts/summarize_ncu.py ${NAME:-round1_ncu_k3_relax_512} /tmp/prof_k3.ncu-rep C3D 3221225472 > gpurun_out/prof_k3_summary.log 2>&1
$NCU -i /tmp/prof_k3.ncu-rep --page details > gpurun_out/prof_k3_details.txt 2>&1
cp profiles/${NAME:-round1_ncu_k3_relax_512}.json profiles/relax_traffic.json gpurun_out/profiles/
cut -c1-1500 gpurun_out/bench_C3D.json; tail -3 gpurun_out/bench_C3D.err
