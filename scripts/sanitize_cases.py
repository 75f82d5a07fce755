"""Small invocations of every libprotox kernel, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_2307_07931_b200 import inputs
from paper_2307_07931_b200 import protox as P


def fields(lay, rank=0):
    a, b, r = lay.alloc(rank), lay.alloc(rank), lay.alloc(rank)
    P.init_field(lay, rank, lay.patch(rank, r), P.PX_FIELD_HASH, 1)
    P.init_field(lay, rank, lay.patch(rank, a), P.PX_FIELD_HASH, 2)
    return a, b, r


def case(name, fn):
    fn()
    torch.cuda.synchronize()
    print("ok", name, flush=True)


def relax(n0, n1, g=1, st=0, bc=P.PX_BC_PERIODIC, k=1):
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (n0, n1), g, bc, 1)
    a, b, r = fields(lay)
    P.fill_ghosts(lay, 0, lay.patch(0, a))
    P.fill_ghosts(lay, 0, lay.patch(0, r))
    nb = P.norm_buffer(lay.local(0).owned)
    prm = P.relax_params(1.0 / n0, (1.0 / n0) ** 2 / 8, st)
    if k == 1:
        P.relax_step(prm, lay.patch(0, a), lay.patch(0, b), lay.patch(0, r), lay.local(0).owned, nb)
        P.residual_norm(prm, lay.patch(0, a), lay.patch(0, r), lay.local(0).owned, nb)
    else:
        P.relax_block(prm, k, lay.patch(0, a), lay.patch(0, b), lay.patch(0, r), lay.local(0).owned, nb)


def solve(n0, n1, nranks=1, g=1, st=0, bc=P.PX_BC_PERIODIC, N=5, E=2, tk=1, graph=False):
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (n0, n1 // nranks), g, bc, nranks)
    parts = [fields(lay, r) for r in range(nranks)]
    if tk > 1:
        P.exchange_ghosts_local(lay, [lay.patch(r, parts[r][2]) for r in range(nranks)])
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    P.solve(lay, None, 0, P.relax_params(1.0 / n0, (1.0 / n0) ** 2 / 8, st), N, E,
            [lay.patch(r, p[0]) for r, p in enumerate(parts)], [lay.patch(r, p[1]) for r, p in enumerate(parts)],
            [lay.patch(r, p[2]) for r, p in enumerate(parts)], temporal_k=tk, use_graph=graph, stream=s)


def solve3(n, st=P.PX_LAPLACE_7PT_3D, bc=P.PX_BC_PERIODIC, N=3, E=1):
    g = P.Grid3(n, 1)
    a, b, r = g.alloc(), g.alloc(), g.alloc()
    P.init_field3(g, r, 1, 1)
    P.init_field3(g, a, 1, 2)
    if st == P.PX_MEHRSTELLEN_27PT_3D:
        P.fill_ghosts3(g, bc, r)
        f = g.alloc()
        P.mehrstellen_rhs3(g, r, f)
        r = f
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    P.solve3(g, bc, P.relax_params(1.0 / n[0], (1.0 / n[0]) ** 2 / 12, st), N, E, a, b, r, stream=s)


def push_solve(n0, n1, N=5, E=1, st=0):
    """Fused peer-memory push (self-exchange, peer communicator): push_init,
    the PUSH k_bulk sweeps as programmatic dependent launches, k_wait."""
    import os
    os.environ["PROTOX_NCCL_SELF_EXCHANGE"] = "1"
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (n0, n1), 1, P.PX_BC_PERIODIC, 1)
    a, b, r = fields(lay)
    pa, pb, pr = lay.patch(0, a), lay.patch(0, b), lay.patch(0, r)
    comm = P.Comm(None, 1, 0, torch.cuda.current_device())
    P.comm_p2p_import(comm, lay, [P.comm_p2p_export(comm, lay, 0, pa, pb)])
    P.solve(lay, comm, 0, P.relax_params(1.0 / n0, 1.0 / (8.0 * n0 * n0), st), N, E, pa, pb, pr)
    torch.cuda.synchronize()
    comm.close()


def reg2_solve():
    os.environ["PROTOX_RESIDENT_REG"] = "2"  # read once per process: this case runs alone
    solve(1024, 1024, N=5, E=2)


def async_solve(n0, n1, N=6, E=2):
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (n0, n1), 1, P.PX_BC_PERIODIC, 1)
    a, b, r = fields(lay)
    d = torch.zeros(2 * (N // E + 2), dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    P.solve_async(lay, None, 0, P.relax_params(1.0 / n0, (1.0 / n0) ** 2 / 8), N, E, lay.patch(0, a),
                  lay.patch(0, b), lay.patch(0, r), d, use_graph=True, stream=s)
    s.synchronize()


def other():
    lay = P.Layout(P.box(0, 0, 199, 99), (200, 100), 1, P.PX_BC_DIRICHLET_CC, 1)
    a, b, r = fields(lay)
    P.fill_ghosts(lay, 0, lay.patch(0, a))
    P.mehrstellen_rhs(lay.patch(0, a), lay.patch(0, b), lay.local(0).owned)
    P.stencil_apply(1, 2.0, lay.patch(0, a), lay.patch(0, b), lay.local(0).owned)
    x = torch.rand(4096, dtype=torch.float64, device="cuda")
    y = torch.rand(4096, dtype=torch.float64, device="cuda")
    z = torch.empty(4096, dtype=torch.float64, device="cuda")
    P.stream_ceiling(x, y, z, 0)
    P.stream_ceiling(x, None, z, 1)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    cases = {
        "ldg_relax": lambda: relax(300, 70, st=0),
        "ldg_relax9": lambda: relax(130, 41, st=1, bc=P.PX_BC_DIRICHLET_CC),
        "bulk_relax": lambda: relax(2048, 2048),
        "bulk_relax9": lambda: relax(2050, 2048, st=1),
        "tb_relax_block": lambda: relax(1000, 300, g=4, k=4),
        "smallbox_solve": lambda: solve(64, 64, bc=P.PX_BC_DIRICHLET_CC),
        "boxw_fixed9_solve": lambda: solve(62, 52, st=1, bc=P.PX_BC_FIXED_GHOSTS),
        "resident_reg_solve": lambda: solve(1024, 1024, N=5, E=2),
        "resident_reg_dirichlet_solve": lambda: solve(1000, 700, N=5, E=2, bc=P.PX_BC_DIRICHLET_CC),
        "resident_reg2_solve": reg2_solve,
        "async_solve": lambda: async_solve(1024, 1024),
        "persist_solve": lambda: solve(600, 90, st=1),
        "local_multipart_solve": lambda: solve(256, 150, nranks=3, bc=P.PX_BC_FIXED_GHOSTS),
        "tb_solve": lambda: solve(1000, 300, nranks=3, g=4, tk=4, N=9, E=3),
        "graph_solve": lambda: solve(600, 90, N=4, E=1, graph=True),
        "pdl_bulk_solve": lambda: solve(2048, 2050, N=4, E=1),
        "push_solve": lambda: push_solve(1100, 70, N=5, E=1),
        "push_solve9": lambda: push_solve(640, 300, N=4, E=2, st=1),
        "tb_dirichlet9_solve": lambda: solve(1000, 300, g=4, tk=4, N=8, E=4, st=1, bc=P.PX_BC_DIRICHLET_CC),
        "tb_fixed_k2_solve": lambda: solve(500, 120, g=2, tk=2, N=4, E=1, bc=P.PX_BC_FIXED_GHOSTS),
        "relax3_solve": lambda: solve3((70, 37, 13)),
        "relax3_27_solve": lambda: solve3((66, 34, 9), st=P.PX_MEHRSTELLEN_27PT_3D, bc=P.PX_BC_DIRICHLET_CC),
        "other_kernels": other,
    }
    for name, fn in cases.items():
        if which in ("all", name):
            case(name, fn)
