"""Where does a C4 step's time go?  32768^2 periodic, ghost 4, k = 4: time
px_solve (graph) for N = 4, 8, 40, 100 sweeps (norms every 4) and one
px_relax_block pass alone, CUDA events on the stream."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2307_07931_b200 import inputs
from paper_2307_07931_b200 import protox as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
h = 1.0 / n
lay = P.Layout(P.box(0, 0, n - 1, n - 1), (256, 256), 4, P.PX_BC_PERIODIC, 1)
li = lay.local(0)
a, b, r = lay.alloc(0), lay.alloc(0), lay.alloc(0)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
P.init_field(lay, 0, lay.patch(0, r), P.PX_FIELD_HASH, inputs.DEFAULT_SEED, stream=s)
P.fill_ghosts(lay, 0, lay.patch(0, r), stream=s)
prm = P.relax_params(h, h * h / 8)
pa, pb, pr = lay.patch(0, a), lay.patch(0, b), lay.patch(0, r)
out = {}


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    s.synchronize()
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    s.synchronize()
    return e0.elapsed_time(e1) / reps


nb = P.norm_buffer(li.owned)
s.wait_stream(torch.cuda.current_stream())
out["relax_block_ms"] = timed(lambda: P.relax_block(prm, 4, pa, pb, pr, li.owned, nb, stream=s), 10)
for N in (4, 8, 40, 100):
    out[f"solve_{N}_ms"] = timed(lambda: P.solve(lay, None, 0, prm, N, 4, pa, pb, pr, use_graph=True, stream=s,
                                                 temporal_k=4), 3)
    out[f"solve_{N}_kernels"] = P.last_solve_kernels()
out["per_pass_slope_ms"] = (out["solve_100_ms"] - out["solve_40_ms"]) / 15
print(json.dumps(out))
