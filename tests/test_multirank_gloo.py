"""The N>1 path on CPU: world_size 2 and 3 processes over torch.distributed
`gloo` (127.0.0.1).  Each rank holds its slab in libprotox's layout
(px_layout_local geometry), exchanges y-ghost rows with exactly the transfers
of px_layout_halo_plan (NCCL's in-order send/recv matching emulated with
per-peer tags), all-reduces the residual norms (max / sum), and advances its
slab with the oracle.  The gathered result must be bit-identical to the
undecomposed oracle run: this checks the partitioner, neighbour ranks, span
offsets/counts and posting order the GPU path uses over NCCL.

The max-norm all-reduce is emulated exactly as libprotox performs it
(px_solve.cu, px_comm_allreduce_norms): a max over the IEEE-754 bit patterns
of the non-negative |r| values as integers (ncclUint64 / ncclMax there,
int64 MAX here -- identical for patterns below 2^63), which keeps a NaN of any
rank (reading R7).  `test_nan_norm_allreduce_over_gloo` puts a NaN in one
rank's slab only and checks that every rank's reduced norms are NaN exactly
where the undecomposed oracle's are."""
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


def _worker(rank, world, port, bc, g, st, q, nan_cell=None):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle
    from helpers import BC_MAP
    from paper_2307_07931_b200 import protox as P
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        n0, n1, N, E = 48, 60, 7, 2
        h = 1.0 / 48
        lam = h * h / 8
        rng = np.random.default_rng(42)
        phi0 = rng.uniform(-1, 1, (n1 + 2 * g, n0 + 2 * g))
        rho = rng.uniform(-1, 1, (n1 + 2 * g, n0 + 2 * g))
        if nan_cell is not None:  # (y, x) of an interior cell of phi0 (ghosted indexing)
            phi0[nan_cell] = np.nan
        lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (12, 10), g, bc, world)
        li = lay.local(rank)
        ld, off = li.ld, li.patch_offset
        y0, y1 = li.owned.lo.c[1], li.owned.hi.c[1]
        ny = y1 - y0 + 1
        flat = np.zeros(li.alloc_elems)
        rhs_flat = np.zeros(li.alloc_elems)

        def win(a):  # (ny+2g, n0+2g) ghosted window of a flat slab array
            return a.reshape(-1, ld)[:, off:off + n0 + 2 * g]

        win(flat)[:] = phi0[y0:y0 + ny + 2 * g]
        win(rhs_flat)[:] = rho[y0:y0 + ny + 2 * g]
        fixed_ghosts = win(flat).copy()

        def local_fill(a):
            w = win(a)
            rows = slice(g, g + ny)
            for t in range(1, g + 1):
                if bc == P.PX_BC_PERIODIC:
                    w[rows, g - t] = w[rows, g + n0 - t]
                    w[rows, g + n0 - 1 + t] = w[rows, g + t - 1]
                elif bc == P.PX_BC_DIRICHLET_CC:
                    w[rows, g - t] = -w[rows, g + t - 1]
                    w[rows, g + n0 - 1 + t] = -w[rows, g + n0 - t]
                else:
                    w[rows, g - t] = fixed_ghosts[rows, g - t]
                    w[rows, g + n0 - 1 + t] = fixed_ghosts[rows, g + n0 - 1 + t]
            for t in range(1, g + 1):
                if li.nbr_lo < 0:
                    w[g - t] = -w[g + t - 1] if bc == P.PX_BC_DIRICHLET_CC else fixed_ghosts[g - t]
                if li.nbr_hi < 0:
                    w[g + ny - 1 + t] = -w[g + ny - t] if bc == P.PX_BC_DIRICHLET_CC else fixed_ghosts[g + ny - 1 + t]

        def exchange(a):
            local_fill(a)
            reqs, seen = [], {}
            for op in lay.halo_plan(rank):
                key = (op.peer, op.is_recv)
                tag = seen.get(key, 0)
                seen[key] = tag + 1
                # op.offset counts from patch.data = allocation + patch_offset
                sl = slice(off + op.offset, off + op.offset + op.count)
                buf = torch.from_numpy(a[sl]) if op.is_recv else torch.from_numpy(a[sl].copy())
                if op.is_recv:
                    reqs.append((dist.irecv(buf, src=op.peer, tag=tag), sl, buf))
                else:
                    reqs.append((dist.isend(buf, dst=op.peer, tag=tag), None, buf))
            for rq, sl, buf in reqs:
                rq.wait()
                if sl is not None:
                    a[sl] = buf.numpy()

        local = oracle.Problem(n0, ny, h, lam, b0=n0, b1=ny, ghost=g, bc=oracle.BC_FIXED, stencil=st,
                               nsweeps=1, norm_every=-1)

        def residual_allreduce():
            exchange(flat)
            m, s = oracle.residual(local, win(flat), win(rhs_flat))
            # the library's max: over the bit patterns of |r| >= 0 as integers
            t = torch.from_numpy(np.array([m], dtype=np.float64).view(np.int64).copy())
            u = torch.tensor([s], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dist.all_reduce(u, op=dist.ReduceOp.SUM)
            return float(t.numpy().view(np.float64)[0]), u.item(), bool(np.isnan(m))

        norms = []
        for it in range(N):
            if it % E == 0:
                norms.append(residual_allreduce())
            exchange(flat)
            out, _ = oracle.solve(local, win(flat), win(rhs_flat))
            win(flat)[g:g + ny, g:g + n0] = out[g:g + ny, g:g + n0]
        norms.append(residual_allreduce())
        got = [None] * world if rank == 0 else None
        dist.gather_object(win(flat)[g:g + ny, g:g + n0].copy(), got, dst=0)
        if rank == 0:
            full = np.ascontiguousarray(np.concatenate(got, 0))
            p = oracle.Problem(n0, n1, h, lam, b0=12, b1=10, ghost=g, bc=BC_MAP[bc], stencil=st,
                               nsweeps=N, norm_every=E)
            ref, rn = oracle.solve(p, phi0, rho)
            refi = np.ascontiguousarray(ref[g:g + n1, g:g + n0])
            ok = np.array_equal(full.view(np.uint64), refi.view(np.uint64))  # NaN-aware, bitwise
            nm = np.array([x[:2] for x in norms])
            local_nan = [x[2] for x in norms]
            ok_max = (np.array_equal(np.isnan(nm[:, 0]), np.isnan(rn[:, 0])) and
                      np.array_equal(nm[:, 0].view(np.uint64), rn[:, 0].view(np.uint64)))
            ok_sum = np.allclose(nm[:, 1], rn[:, 1], rtol=1e-12, atol=0, equal_nan=True)
            q.put((ok, ok_max, ok_sum, float(np.nanmax(np.abs(full - refi))), int(np.isnan(rn[:, 0]).sum()),
                   int(sum(local_nan))))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # report instead of hanging the parent
        import traceback
        q.put(("error", rank, traceback.format_exc()))
        raise


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("bc", [0, 1, 2])
@pytest.mark.parametrize("g,st", [(1, 0), (2, 1)])
def test_slab_exchange_over_gloo(world, bc, g, st):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, bc, g, st, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert res[0] != "error", res
    ok, ok_max, ok_sum, d = res[:4]
    assert ok, d
    assert ok_max and ok_sum


@pytest.mark.parametrize("world", [2, 3])
def test_nan_norm_allreduce_over_gloo(world):
    """A NaN in the LAST rank's slab only: rank 0's own residuals stay finite
    for the first recorded iterates (the NaN needs sweeps to cross slabs), yet
    the reduced max must be NaN in every entry where the undecomposed oracle's
    is (all of them here), and the field bit-identical (NaN payloads included)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n1 = 60
    cell = (n1 - 3, 20)  # ghosted (y, x): interior row n1-4, inside the last slab for world 2 and 3
    procs = [ctx.Process(target=_worker, args=(r, world, port, 0, 1, 0, q, cell)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert res[0] != "error", res
    ok, ok_max, ok_sum, _, n_nan_ref, n_nan_rank0 = res
    assert n_nan_ref == 5  # N = 7, E = 2: entries for phi^0, ^2, ^4, ^6 and phi^7 -- all NaN
    assert n_nan_rank0 < n_nan_ref  # rank 0 alone saw finite maxima: the reduction carried the NaN
    assert ok and ok_max and ok_sum
