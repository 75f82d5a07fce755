"""Where does the C3 step spend the time the sweep kernel alone does not
account for?  16384² periodic, 100 sweeps, norms every sweep:
  step_graph     px_solve from a CUDA graph (the bench's step)
  step_nograph   the same enqueued launch by launch
  relax_events   100 px_relax_step launches, CUDA events around each (kernel_ms)
  relax_stream   100 px_relax_step launches back to back, events around all
ms per sweep; each measured three times, interleaved."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2307_07931_b200 import inputs
from paper_2307_07931_b200 import protox as P

n, N = 16384, 100
h = 1.0 / n
lay = P.Layout(P.box(0, 0, n - 1, n - 1), (256, 256), 1, P.PX_BC_PERIODIC, 1)
li = lay.local(0)
a, b, r = lay.alloc(0), lay.alloc(0), lay.alloc(0)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
P.init_field(lay, 0, lay.patch(0, r), P.PX_FIELD_HASH, inputs.DEFAULT_SEED, stream=s)
prm = P.relax_params(h, h * h / 8)
pa, pb, pr = lay.patch(0, a), lay.patch(0, b), lay.patch(0, r)
nb = P.norm_buffer(li.owned)
s.wait_stream(torch.cuda.current_stream())


def ev():
    return torch.cuda.Event(enable_timing=True)


def step(graph):
    e0, e1 = ev(), ev()
    e0.record(s)
    P.solve(lay, None, 0, prm, N, 1, pa, pb, pr, use_graph=graph, stream=s)
    e1.record(s)
    s.synchronize()
    return e0.elapsed_time(e1) / N


def relax_events():
    evs = [(ev(), ev()) for _ in range(N)]
    for i in range(N):
        src, dst = (pa, pb) if i % 2 == 0 else (pb, pa)
        evs[i][0].record(s)
        P.relax_step(prm, src, dst, pr, li.owned, nb, stream=s)
        evs[i][1].record(s)
    s.synchronize()
    return sum(x.elapsed_time(y) for x, y in evs) / N


def relax_stream():
    e0, e1 = ev(), ev()
    e0.record(s)
    for i in range(N):
        src, dst = (pa, pb) if i % 2 == 0 else (pb, pa)
        P.relax_step(prm, src, dst, pr, li.owned, nb, stream=s)
    e1.record(s)
    s.synchronize()
    return e0.elapsed_time(e1) / N


out = {k: [] for k in ("step_graph", "step_nograph", "relax_events", "relax_stream")}
step(True)
for _ in range(3):
    out["step_graph"].append(step(True))
    out["step_nograph"].append(step(False))
    out["relax_events"].append(relax_events())
    out["relax_stream"].append(relax_stream())
print(json.dumps({k: [round(v, 4) for v in vs] for k, vs in out.items()}))
