#!/usr/bin/env python
"""Multigrid V-cycle timing on one B200 (px_mg_solve).

    python scripts/bench_mg.py [--n 16384] [--levels 11] [--cycles 6] [--bc 0|1] [--stencil 0|1]

Prints one JSON line: ms per V(nu1,nu2)-cycle (CUDA events around the graph
replay of the whole solve, warm-up first), the residual max-norm after every
cycle and the per-cycle reduction factor, and the level-0 relax sweep time
for scale (a V(2,2)-cycle costs about 4 level-0 sweeps + the transfers).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--levels", type=int, default=11)
    ap.add_argument("--cycles", type=int, default=6)
    ap.add_argument("--nu1", type=int, default=2)
    ap.add_argument("--nu2", type=int, default=2)
    ap.add_argument("--nuc", type=int, default=16)
    ap.add_argument("--bc", type=int, default=0)
    ap.add_argument("--stencil", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch

    from paper_2307_07931_b200 import inputs
    from paper_2307_07931_b200 import protox as P

    n = a.n
    h = 1.0 / n
    lam = h * h / 8 if a.stencil == 0 else 3 * h * h / 16
    lay = P.Layout(P.box(0, 0, n - 1, n - 1), (256, 256), 1, a.bc, 1)
    phi, scr, rho = lay.alloc(0), lay.alloc(0), lay.alloc(0)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    P.init_field(lay, 0, lay.patch(0, rho), P.PX_FIELD_HASH, inputs.DEFAULT_SEED, 1, 1, stream=s)
    if a.bc == 0:  # periodic: a solvable (zero-mean) right-hand side
        s.synchronize()
        v = lay.view(0, rho)
        v -= v.mean()
        torch.cuda.synchronize()
    prm = P.relax_params(h, lam, a.stencil)

    def run():
        with torch.cuda.stream(s):
            lay.view(0, phi).zero_()
        return P.mg_solve(lay, prm, a.levels, a.cycles, lay.patch(0, phi), lay.patch(0, scr), lay.patch(0, rho),
                          nu1=a.nu1, nu2=a.nu2, nu_coarse=a.nuc, use_graph=True, stream=s)

    norms = run()  # builds the plan and the graph
    times = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            lay.view(0, phi).zero_()
        e0.record(s)
        norms = P.mg_solve(lay, prm, a.levels, a.cycles, lay.patch(0, phi), lay.patch(0, scr), lay.patch(0, rho),
                           nu1=a.nu1, nu2=a.nu2, nu_coarse=a.nuc, use_graph=True, stream=s)
        e1.record(s)
        s.synchronize()
        times.append(e0.elapsed_time(e1))
    t = min(times)
    # one level-0 relax sweep for scale
    nb = P.norm_buffer(lay.local(0).owned, torch.device("cuda"))
    s.wait_stream(torch.cuda.current_stream())
    evs = []
    for i in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        P.relax_step(prm, lay.patch(0, phi), lay.patch(0, scr), lay.patch(0, rho), lay.local(0).owned, nb, stream=s)
        e1.record(s)
        evs.append((e0, e1))
    s.synchronize()
    sweep_ms = min(x.elapsed_time(y) for x, y in evs[1:])
    r = [float(x) for x in norms[:, 0]]
    print(json.dumps({
        "what": f"px_mg_solve V({a.nu1},{a.nu2}) cycles, nu_coarse {a.nuc}, {a.levels} levels, {n}^2, "
                f"bc {a.bc}, stencil {a.stencil}, graph replay, CUDA events",
        "ms_per_cycle": t / a.cycles, "cycles": a.cycles, "level0_relax_sweep_ms": sweep_ms,
        "cycle_in_level0_sweeps": t / a.cycles / sweep_ms,
        "residual_max": r, "reduction_per_cycle": [r[i + 1] / r[i] for i in range(len(r) - 1)],
        "finest_cell_updates_per_s_equiv": n * n * (a.nu1 + a.nu2) * a.cycles / (t * 1e-3),
    }))


if __name__ == "__main__":
    main()
