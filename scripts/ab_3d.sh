#!/bin/bash
# A/B of the 3D relax kernel: L2 policy knob, kernel time via CUDA events (px3_relax_step).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
cat > /tmp/k3ab.py <<'PY'
import sys, json, torch, os
sys.path.insert(0, ".")
from paper_2307_07931_b200 import protox as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = P.Grid3((n, n, n), 1)
a, b, r = g.alloc(), g.alloc(), g.alloc()
P.init_field3(g, r, 1, 20230714)
prm = P.relax_params(1 / n, (1 / n) ** 2 / 12, P.PX_LAPLACE_7PT_3D)
nb = P.norm_buffer3()
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(30)]
for i in range(30):
    src, dst = (a, b) if i % 2 == 0 else (b, a)
    P.fill_ghosts3(g, 0, src, stream=s)
    evs[i][0].record(s); P.relax_step3(prm, g, src, dst, r, nb, stream=s); evs[i][1].record(s)
s.synchronize()
ms = sorted(x.elapsed_time(y) for x, y in evs[5:])
med = ms[len(ms) // 2]
print(json.dumps({"n": n, "policy": os.environ.get("PROTOX_K3_POLICY", "0"), "nst": os.environ.get("PROTOX_K3_NST", "4"), "promo": os.environ.get("PROTOX_K3_PROMO", "3"), "ms_median": med, "GBps": 24 * n**3 / med / 1e6}))
PY
for nst in 3 4; do for it in 1 2; do PROTOX_K3_NST=$nst timeout 120 python /tmp/k3ab.py 512 >> gpurun_out/ab3d.log 2>&1; done; done
cat gpurun_out/ab3d.log
