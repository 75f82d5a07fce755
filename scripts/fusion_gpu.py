"""The paper's experiment (ProtoX fused vs Proto unfused, PAPER.md:212,
figure `runtime`) re-run on the B200: per sweep, Proto's separate
abstractions -- exchange, laplace(φ, wgt) into a temporary
(px_stencil_apply), forallInPlace update (px_pointwise_update), exchange +
computeMaxResidualAcrossProcs (px_residual_norm) -- against the fused sweep
(px_relax_step with its fused ghost images and norms).  Same inputs, bitwise
equal results; CUDA events on the launching stream.

    python scripts/fusion_gpu.py [n] [sweeps] [out.json]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2307_07931_b200 import inputs
from paper_2307_07931_b200 import protox as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
N = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out_path = sys.argv[3] if len(sys.argv) > 3 else None
h = 1.0 / n
lam = h * h / 8
lay = P.Layout(P.box(0, 0, n - 1, n - 1), (256, 256), 1, P.PX_BC_PERIODIC, 1)
li = lay.local(0)
s = torch.cuda.Stream()
rho = lay.alloc(0)
s.wait_stream(torch.cuda.current_stream())
P.init_field(lay, 0, lay.patch(0, rho), P.PX_FIELD_HASH, inputs.DEFAULT_SEED, stream=s)
prm = P.relax_params(h, lam)
pr = lay.patch(0, rho)


def unfused():
    phi, temp = lay.alloc(0), lay.alloc(0)
    nb = P.norm_buffer(li.owned)
    s.wait_stream(torch.cuda.current_stream())
    pp, pt = lay.patch(0, phi), lay.patch(0, temp)

    def sweep():
        P.fill_ghosts(lay, 0, pp, stream=s)                                   # exchange
        P.stencil_apply(0, 1.0 / (h * h), pp, pt, li.owned, stream=s)           # temp = laplace(phi, wgt)
        P.pointwise_update(pp, pt, pr, lam, li.owned, stream=s)                 # forallInPlace(jacobiUpdate)
        P.fill_ghosts(lay, 0, pp, stream=s)                                   # computeMaxResidualAcrossProcs
        P.residual_norm(prm, pp, pr, li.owned, nb, stream=s)

    for _ in range(2):  # warm-up, then restart from φ0 = 0
        sweep()
    s.synchronize()
    phi.zero_()
    s.wait_stream(torch.cuda.current_stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(N):
        sweep()
    e1.record(s)
    s.synchronize()
    return phi, e0.elapsed_time(e1) / N


def fused():
    """The product path: px_solve (fused sweeps with fused ghost images and
    norms every sweep), N sweeps replayed from a CUDA graph."""
    a, b = lay.alloc(0), lay.alloc(0)
    s.wait_stream(torch.cuda.current_stream())
    pa, pb = lay.patch(0, a), lay.patch(0, b)
    c, d = lay.alloc(0), lay.alloc(0)
    s.wait_stream(torch.cuda.current_stream())
    P.solve(lay, None, 0, prm, N, 1, lay.patch(0, c), lay.patch(0, d), pr, use_graph=True, stream=s)  # warm-up
    res = P.solve(lay, None, 0, prm, N, 1, pa, pb, pr, use_graph=True, stream=s)  # build the graph
    a.zero_(), b.zero_()
    s.wait_stream(torch.cuda.current_stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    res = P.solve(lay, None, 0, prm, N, 1, pa, pb, pr, use_graph=True, stream=s)
    e1.record(s)
    s.synchronize()
    return (b if res.in_scratch else a), e0.elapsed_time(e1) / N


phi_u, t_u = unfused()
phi_f, t_f = fused()
same = bool(torch.equal(lay.view(0, phi_u), lay.view(0, phi_f)))
res = {"what": "Proto unfused (exchange, laplace pass, update pass, exchange + residual pass per sweep) vs "
               "the fused sweep on one B200, periodic %dx%d, %d timed sweeps (CUDA events)" % (n, n, N),
       "unfused_ms_per_sweep": t_u, "fused_ms_per_sweep": t_f, "speedup_fused": t_u / t_f,
       "unfused_Gcell_s": n * n / (t_u * 1e-3) / 1e9, "fused_Gcell_s": n * n / (t_f * 1e-3) / 1e9,
       "algorithmic_bytes_per_cell": {"unfused": 64, "fused": 24},
       "phi_bitwise_equal": same,
       "fused_path": "px_solve, N sweeps, norms every sweep, CUDA graph (the bench's C3 path)",
       "paper": "ProtoX up to 2x faster than Proto on a 2.3 GHz quad-core i7 (PAPER.md:212)"}
print(json.dumps(res))
if out_path:
    json.dump(res, open(out_path, "w"), indent=1)
