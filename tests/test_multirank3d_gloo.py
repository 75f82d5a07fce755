"""The 3D z-slab path on CPU: world_size 2 and 3 processes over
torch.distributed gloo (127.0.0.1).  Each rank owns the planes px3_slab gives
it, fills its x / y ghosts by the boundary rule, exchanges its z ghost planes
with exactly the posting order px3_solve_comm uses over NCCL (send up, send
down, recv down, recv up; NCCL's in-order matching per peer pair emulated
with per-peer sequence tags), advances its slab one sweep with the 3D oracle
(fixed ghosts = the exchanged / filled ones), and all-reduces the residual
norms.  The gathered result must be bit-identical to the undecomposed 3D
oracle: this checks the partitioner, the neighbour ranks, the periodic ring
and the plane pairing of the GPU path."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, bc, q):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    from paper_2307_07931_b200 import protox as P
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        n = (10, 7, 12)
        N, E = 5, 2
        h = 1.0 / 12
        lam = h * h / 12
        rng = np.random.default_rng(17)
        phi0 = rng.uniform(-1, 1, (n[2] + 2, n[1] + 2, n[0] + 2))
        rho = rng.uniform(-1, 1, (n[2] + 2, n[1] + 2, n[0] + 2))
        z0, z1 = P.slab3(n[2], world, rank)
        nz = z1 - z0
        per = bc == oracle.BC_PERIODIC
        lo = rank - 1 if rank > 0 else (world - 1 if per else -1)
        hi = rank + 1 if rank < world - 1 else (0 if per else -1)
        a = phi0[z0:z1 + 2].copy()  # planes z0-1 .. z1 (ghosted)
        f = rho[z0:z1 + 2].copy()
        sent = {}

        def tag(peer, kind):  # per ordered pair sequence number: NCCL's in-order matching
            key = (kind, peer)
            sent[key] = sent.get(key, 0) + 1
            return sent[key]

        def fill_xy(u):
            for k in range(1, nz + 1):
                pl = u[k]
                if per:
                    pl[:, 0], pl[:, -1] = pl[:, -2], pl[:, 1]
                    pl[0, :], pl[-1, :] = pl[-2, :], pl[1, :]
                else:
                    pl[:, 0], pl[:, -1] = -pl[:, 1], -pl[:, -2]
                    pl[0, :], pl[-1, :] = -pl[1, :], -pl[-2, :]

        def exchange(u):
            fill_xy(u)
            reqs = []
            # posting order of px3_solve_comm: send up, send down, recv down, recv up
            if hi >= 0:
                reqs.append(dist.isend(torch.from_numpy(u[nz].copy()), hi, tag=1000 * rank + tag(hi, "s")))
            if lo >= 0:
                reqs.append(dist.isend(torch.from_numpy(u[1].copy()), lo, tag=1000 * rank + tag(lo, "s")))
            bufs = {}
            if lo >= 0:
                bufs["lo"] = torch.empty(u[0].shape, dtype=torch.float64)
                reqs.append(dist.irecv(bufs["lo"], lo, tag=1000 * lo + tag(lo, "r")))
            if hi >= 0:
                bufs["hi"] = torch.empty(u[0].shape, dtype=torch.float64)
                reqs.append(dist.irecv(bufs["hi"], hi, tag=1000 * hi + tag(hi, "r")))
            for r_ in reqs:
                r_.wait()
            if lo >= 0:
                u[0] = bufs["lo"].numpy()
            else:
                u[0] = -u[1]
            if hi >= 0:
                u[nz + 1] = bufs["hi"].numpy()
            else:
                u[nz + 1] = -u[nz]

        norms = []
        for it in range(N + 1):
            exchange(a)
            p = oracle.Problem3((n[0], n[1], nz), h, lam, bc=oracle.BC_FIXED, nsweeps=1 if it < N else 0,
                                norm_every=1 if (it < N and it % E == 0) or it == N else -1)
            out, nm = oracle.solve3(p, a, f)
            if len(nm):
                # max over the bit patterns of |r| as integers, as px3d.cu does (ncclUint64)
                mx = torch.from_numpy(np.array([nm[0, 0]], dtype=np.float64).view(np.int64).copy())
                sm = torch.tensor([nm[0, 1]], dtype=torch.float64)
                dist.all_reduce(mx, op=dist.ReduceOp.MAX)
                dist.all_reduce(sm, op=dist.ReduceOp.SUM)
                norms.append((float(mx.numpy().view(np.float64)[0]), sm.item()))
            if it < N:
                a[1:nz + 1] = out[1:nz + 1]
        parts = [None] * world
        dist.all_gather_object(parts, (z0, a[1:nz + 1, 1:-1, 1:-1].copy(), norms))
        if rank == 0:
            q.put(("ok", parts))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback
        q.put(("err", traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("bc", [0, 1])
def test_z_slabs_over_gloo_match_undecomposed_oracle(world, bc):
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, bc, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    status, payload = q.get(timeout=300)
    for p_ in procs:
        p_.join(timeout=60)
    assert status == "ok", payload
    n = (10, 7, 12)
    h = 1.0 / 12
    rng = np.random.default_rng(17)
    phi0 = rng.uniform(-1, 1, (n[2] + 2, n[1] + 2, n[0] + 2))
    rho = rng.uniform(-1, 1, (n[2] + 2, n[1] + 2, n[0] + 2))
    p = oracle.Problem3(n, h, h * h / 12, bc=bc, nsweeps=5, norm_every=2)
    ref, rn = oracle.solve3(p, phi0, rho)
    got = np.concatenate([part[1] for part in sorted(payload, key=lambda t: t[0])], axis=0)
    assert np.array_equal(got.view(np.uint64), ref[1:-1, 1:-1, 1:-1].view(np.uint64))
    norms = np.array(payload[0][2])
    assert np.array_equal(norms[:, 0], rn[:, 0])
    np.testing.assert_allclose(norms[:, 1], rn[:, 1], rtol=1e-12)
