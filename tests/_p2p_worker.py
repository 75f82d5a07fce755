"""Worker of tests/test_gpu_p2p_ipc.py: one rank of a slab-decomposed solve
in the fused peer-memory push mode (px_comm_create_peer + px_comm_p2p_export
/ px_comm_p2p_import).  Every rank runs on cuda:0 in its own process, so the
CUDA IPC mappings, the cross-process release/acquire arrival counters and the
peer-memory norm all-reduce all run for real ("information is
exchanged between the boxes", :173 computeMaxResidualAcrossProcs).  The
records travel over a gloo process group.

    python tests/_p2p_worker.py OUT_DIR BC N0 N1 N1SWEEPS N2SWEEPS E SEED STENCIL GRAPH [INF_AT_ROW]
(env: RANK, WORLD_SIZE, MASTER_ADDR, MASTER_PORT)
Writes OUT_DIR/rank{r}.npz: the owned slab of φ^(N1+N2) and both norm lists.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch
import torch.distributed as dist

from paper_2307_07931_b200 import protox as P


def main():
    out, bc, n0, n1, na, nb, E, seed, st, graph = sys.argv[1:11]
    bc, n0, n1, na, nb, E, seed, st, graph = (int(bc), int(n0), int(n1), int(na), int(nb), int(E), int(seed),
                                             int(st), int(graph))
    inf_row = int(sys.argv[11]) if len(sys.argv) > 11 else -1
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    g = 1
    rng = np.random.default_rng(seed)
    phi0 = rng.uniform(-1, 1, (n1 + 2 * g, n0 + 2 * g))
    rho = rng.uniform(-1, 1, (n1 + 2 * g, n0 + 2 * g))
    if inf_row >= 0:  # ρ = +inf at one cell of interior row inf_row (one rank's slab)
        rho[g + inf_row, g + n0 // 3] = np.inf
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (n0, n1 // (2 * world)), g, bc, world)
    li = lay.local(rank)

    def ghosted(glob):
        t = lay.alloc(rank)
        v = lay.view(rank, t, ghosts=True)
        y0, x0 = li.alloc.lo.c[1] + g, li.alloc.lo.c[0] + g
        v.copy_(torch.from_numpy(np.ascontiguousarray(glob[y0:y0 + v.shape[0], x0:x0 + v.shape[1]])))
        return t

    a, r = ghosted(phi0), ghosted(rho)
    b = lay.alloc(rank)
    if bc == P.PX_BC_FIXED_GHOSTS:
        b.copy_(a)  # fixed ghost cells belong to every iterate
    pa, pb, pr = lay.patch(rank, a), lay.patch(rank, b), lay.patch(rank, r)
    comm = P.Comm(None, world, rank, 0)
    rec = P.comm_p2p_export(comm, lay, rank, pa, pb)
    recs = [None] * world
    dist.all_gather_object(recs, rec)
    P.comm_p2p_import(comm, lay, recs)
    prm = P.relax_params(1.0 / n0, 1.0 / (8.0 * n0 * n0), stencil=st)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    torch.cuda.synchronize()
    if os.environ.get("PROTOX_TEST_LOST_PEER") == "1":
        # rank 1 never solves: rank 0's waits for its pushes must give up
        # (px_spin_until) and px_solve report PX_ERR_STATE instead of hanging
        import time
        msg, t0 = "", time.time()
        if rank == 0:
            try:
                P.solve(lay, comm, rank, prm, na, E, pa, pb, pr, use_graph=bool(graph), stream=s)
            except P.PxError as e:
                msg = str(e)
        np.savez(os.path.join(out, f"rank{rank}.npz"), msg=np.array(msg), secs=time.time() - t0)
        dist.barrier()
        dist.destroy_process_group()
        return
    r1 = P.solve(lay, comm, rank, prm, na, E, pa, pb, pr, use_graph=bool(graph), stream=s)
    k1 = P.last_solve_kernels()
    # continue from φ^na wherever it is (the registered pair in swapped order)
    (cur, ct), (oth, ot) = ((pb, b), (pa, a)) if r1.in_scratch else ((pa, a), (pb, b))
    r2 = P.solve(lay, comm, rank, prm, nb, E, cur, oth, pr, use_graph=bool(graph), stream=s)
    res = ot if r2.in_scratch else ct
    owned = lay.view(rank, res).cpu().numpy()
    np.savez(os.path.join(out, f"rank{rank}.npz"), phi=owned, n1=r1.norms, n2=r2.norms,
             y0=li.owned.lo.c[1], kernels=np.array(k1))
    dist.barrier()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
