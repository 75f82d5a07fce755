"""Diagnose temporal blocking mismatches: one pass of K sweeps vs the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch

import oracle
from helpers import BC_MAP, owned_to_host, to_device_ghosted
from paper_2307_07931_b200 import protox as P

for K, N, n0, n1, bc in [(2, 2, 1000, 300, 0), (2, 2, 448, 64, 0), (2, 4, 1000, 300, 0), (4, 4, 1000, 300, 0),
                         (2, 1, 1000, 300, 0)]:
    g = 4
    h = 1.0 / 1024
    lam = h * h / 8
    rng = np.random.default_rng(1)
    phi0 = rng.uniform(-1, 1, (n1 + 2 * g, n0 + 2 * g))
    rho = rng.uniform(-1, 1, (n1 + 2 * g, n0 + 2 * g))
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (n0, n1), g, bc, 1)
    a = to_device_ghosted(lay, 0, phi0, g)
    b = lay.alloc(0)
    r = to_device_ghosted(lay, 0, rho, g)
    P.fill_ghosts(lay, 0, lay.patch(0, r))
    torch.cuda.synchronize()
    res = P.solve(lay, None, 0, P.relax_params(h, lam), N, -1, lay.patch(0, a), lay.patch(0, b), lay.patch(0, r),
                  temporal_k=K)
    out = owned_to_host(lay, 0, b if res.in_scratch else a)
    p = oracle.Problem(n0, n1, h, lam, ghost=g, bc=BC_MAP[bc], nsweeps=N, norm_every=-1)
    ref, _ = oracle.solve(p, phi0, rho)
    ref = ref[g:-g, g:-g]
    bad = np.argwhere(out != ref)
    print(f"K={K} N={N} {n0}x{n1}: {len(bad)} mismatches", end=" ")
    if len(bad):
        ys, xs = bad[:, 0], bad[:, 1]
        print("rows", np.unique(ys)[:20], "cols", np.unique(xs)[:40], "max", np.max(np.abs(out - ref)))
    else:
        print()
