"""BASELINE config 5 companion: convergence-order ladders h -> h/2 on the GPU
(libprotox kernels), written to profiles/round1_c5_order_ladder.json.

* truncation: τ_h = max|Δ_h φ* − f_h| for φ* = cos(πx) sin(πy) e^y on a vertex
  grid with FIXED ghosts = φ* (one px_residual_norm), 5-point with f = Δφ*,
  Mehrstellen with f = Δφ* + S5(Δφ*)/12 (px_mehrstellen_rhs); 1/h = 16..8192.
* discrete: Jacobi to convergence on Dirichlet-CC with ρ = sin πx sin πy,
  error vs φ* = −ρ/(2π²); 1/h = 16..512.
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_2307_07931_b200 import inputs
from paper_2307_07931_b200 import protox as P


def truncation(n, st):
    h = 1.0 / (n + 1)
    xi = np.arange(-1, n + 1) * h + h
    X, Y = np.meshgrid(xi, xi, indexing="xy")
    phi = np.cos(np.pi * X) * np.sin(np.pi * Y) * np.exp(Y)
    lap = -np.pi**2 * phi + np.cos(np.pi * X) * ((1 - np.pi**2) * np.sin(np.pi * Y) * np.exp(Y)
                                                + 2 * np.pi * np.cos(np.pi * Y) * np.exp(Y))
    lay = P.Layout(P.box(0, 0, n - 1, n - 1), (n, n), 1, P.PX_BC_FIXED_GHOSTS, 1)
    a, r = lay.alloc(0), lay.alloc(0)
    lay.view(0, a, ghosts=True).copy_(torch.from_numpy(phi))
    lay.view(0, r, ghosts=True).copy_(torch.from_numpy(lap))
    rhs = r
    if st == 1:
        f = lay.alloc(0)
        P.mehrstellen_rhs(lay.patch(0, r), lay.patch(0, f), lay.local(0).owned)
        rhs = f
    nb = P.norm_buffer(lay.local(0).owned)
    P.residual_norm(P.relax_params(h, 0.0, st), lay.patch(0, a), lay.patch(0, rhs), lay.local(0).owned, nb)
    torch.cuda.synchronize()
    return nb[0].item()


def discrete(n, st):
    h = 1.0 / n
    lay = P.Layout(P.box(0, 0, n - 1, n - 1), (n, n), 1, P.PX_BC_DIRICHLET_CC, 1)
    a, b, r = lay.alloc(0), lay.alloc(0), lay.alloc(0)
    rho = inputs.sine_field(n, n)
    lay.view(0, r).copy_(torch.from_numpy(rho))
    rhs = r
    if st == 1:
        P.fill_ghosts(lay, 0, lay.patch(0, r))
        f = lay.alloc(0)
        P.mehrstellen_rhs(lay.patch(0, r), lay.patch(0, f), lay.local(0).owned)
        rhs = f
        lam = 3 * h * h / 10
        rate = lam * 2 * math.pi**2
    else:
        lam = h * h / 4
        rate = 1 - math.cos(math.pi * h)
    nsw = int(36 / rate) + 10
    nsw += nsw % 2
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    res = P.solve(lay, None, 0, P.relax_params(h, lam, st), nsw, 0, lay.patch(0, a), lay.patch(0, b),
                  lay.patch(0, rhs), use_graph=nsw <= 20000, stream=s)
    out = lay.view(0, b if res.in_scratch else a).cpu().numpy()
    return float(np.max(np.abs(out + rho / (2 * math.pi**2)))), nsw


def ladder(vals):
    return [vals[i] / vals[i + 1] for i in range(len(vals) - 1)]


def main():
    out = {}
    ns = [16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192]
    for st, name in ((0, "5pt"), (1, "mehrstellen")):
        t = [truncation(n - 1, st) for n in ns]
        out[f"truncation_{name}"] = {"inv_h": ns, "tau": t, "ratio": ladder(t)}
    nd = [16, 32, 64, 128, 256, 512]
    for st, name in ((0, "5pt"), (1, "mehrstellen")):
        e = [discrete(n, st) for n in nd]
        out[f"discrete_{name}"] = {"inv_h": nd, "error": [x[0] for x in e], "sweeps": [x[1] for x in e],
                                   "ratio": ladder([x[0] for x in e])}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "round1_c5_order_ladder.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
