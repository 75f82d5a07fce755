"""Dirichlet temporal blocking vs plain sweeps on the GPU (same layout), and vs
the oracle at a mid size: bitwise comparison of phi^N."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2307_07931_b200 import inputs
from paper_2307_07931_b200 import protox as P

def run(n, tk, st, bc, N, every, g=4, nx=None):
    nx = nx or n
    lay = P.Layout(P.box(0, 0, nx - 1, n - 1), (256, 256), g, bc, 1)
    a, b, r = lay.alloc(0), lay.alloc(0), lay.alloc(0)
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    P.init_field(lay, 0, lay.patch(0, r), P.PX_FIELD_HASH, inputs.DEFAULT_SEED, stream=s)
    P.fill_ghosts(lay, 0, lay.patch(0, r), stream=s)
    prm = P.relax_params(1.0 / n, (1.0 / n) ** 2 / 8, st)
    res = P.solve(lay, None, 0, prm, N, every, lay.patch(0, a), lay.patch(0, b), lay.patch(0, r),
                  use_graph=False, stream=s, temporal_k=tk)
    s.synchronize()
    out = lay.view(0, b if res.in_scratch else a).cpu().numpy()
    return out, res.norms

for (n, nx) in [(8192, 8192), (4096, 4096), (2048, 8192), (8192, 2048), (1024, 8192)]:
    for st in (0, 1):
        for bc in (0, 1):
            o1, n1 = run(n, 1, st, bc, 8, 1, nx=nx)
            o4, n4 = run(n, 4, st, bc, 8, 1, nx=nx)
            d = np.argwhere(o1.view(np.uint64) != o4.view(np.uint64))
            print(f"ny={n} nx={nx} st={st} bc={bc}: ndiff={len(d)} first={d[:5].tolist()} "
                  f"norm1={n1[-1].tolist()} norm4={n4[-1].tolist()}", flush=True)
