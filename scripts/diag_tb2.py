"""Temporal blocking vs plain sweeps on the same layout (bitwise), big sizes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_2307_07931_b200 import inputs
from paper_2307_07931_b200 import protox as P

for (n0, n1, K, N) in [(16384, 16384, 4, 4), (16384, 2048, 4, 4), (4096, 4096, 4, 4), (16384, 16384, 2, 2),
                       (16384, 1024, 4, 4), (8192, 8192, 4, 4)]:
    g = 4
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (256, 256), g, P.PX_BC_PERIODIC, 1)
    r = lay.alloc(0)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    P.init_field(lay, 0, lay.patch(0, r), P.PX_FIELD_HASH, inputs.DEFAULT_SEED, stream=s)
    P.fill_ghosts(lay, 0, lay.patch(0, r), stream=s)
    outs = []
    for tk in (1, K):
        a, b = lay.alloc(0), lay.alloc(0)
        s.wait_stream(torch.cuda.current_stream())
        res = P.solve(lay, None, 0, P.relax_params(1.0 / n0, (1.0 / n0) ** 2 / 8), N, 1, lay.patch(0, a),
                      lay.patch(0, b), lay.patch(0, r), stream=s, temporal_k=tk)
        outs.append((lay.view(0, b if res.in_scratch else a).cpu().numpy(), res.norms))
    d = outs[0][0] != outs[1][0]
    bad = np.argwhere(d)
    print(f"{n0}x{n1} K={K} N={N}: {len(bad)} mismatches; norms equal: {np.array_equal(outs[0][1][:,0], outs[1][1][:,0])}", end=" ")
    if len(bad):
        print("rows", np.unique(bad[:, 0])[:12], "cols", np.unique(bad[:, 1])[:24], "ncols", len(np.unique(bad[:, 1])),
              "nrows", len(np.unique(bad[:, 0])))
    else:
        print()
    sys.stdout.flush()
