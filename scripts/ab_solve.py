"""Time px_solve (CUDA graph, norms every E sweeps) on one GPU: plain
(temporal_k=1) vs temporal blocking.  Prints Gcell-updates/s per config.

    python scripts/ab_solve.py --n 16384 --tk 4 --sweeps 100 --every 1
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2307_07931_b200 import inputs
from paper_2307_07931_b200 import protox as P

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--tk", type=int, default=1)
ap.add_argument("--sweeps", type=int, default=100)
ap.add_argument("--every", type=int, default=1)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--stencil", type=int, default=0)
ap.add_argument("--nograph", action="store_true", help="launch kernels directly (for ncu)")
ap.add_argument("--bc", type=int, default=0, help="0 periodic, 1 Dirichlet-CC, 2 fixed ghosts")
args = ap.parse_args()
n = args.n
g = max(1, args.tk)
lay = P.Layout(P.box(0, 0, n - 1, n - 1), (256, 256), g, args.bc, 1)
a, b, r = lay.alloc(0), lay.alloc(0), lay.alloc(0)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
P.init_field(lay, 0, lay.patch(0, r), P.PX_FIELD_HASH, inputs.DEFAULT_SEED, stream=s)
P.fill_ghosts(lay, 0, lay.patch(0, r), stream=s)
prm = P.relax_params(1.0 / n, (1.0 / n) ** 2 / 8, args.stencil)
run = lambda: P.solve(lay, None, 0, prm, args.sweeps, args.every, lay.patch(0, a), lay.patch(0, b),
                      lay.patch(0, r), use_graph=not args.nograph, stream=s, temporal_k=args.tk)
run()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(args.reps):
    res = run()
e1.record(s)
s.synchronize()
ms = e0.elapsed_time(e1) / args.reps
rate = n * n * args.sweeps / (ms * 1e-3) / 1e9
print(json.dumps({"n": n, "tk": args.tk, "sweeps": args.sweeps, "every": args.every, "stencil": args.stencil, "bc": args.bc, "tb_impl": os.environ.get("PROTOX_TB_IMPL", "wide"),
                  "ms_per_solve": ms, "Gcell_s": rate, "GBps_at_24B": rate * 24, "last_norm": res.norms[-1].tolist()}))
