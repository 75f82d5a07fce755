"""The fused peer-memory push path across PROCESSES:
2 or 3 ranks, each its own process on cuda:0, peer-memory communicator (no
NCCL), IPC records all-gathered over gloo.  Exercises the CUDA IPC mappings,
the cross-process release/acquire arrival counters of the single-launch
sweep kernel, the push of φ^0, and the peer-memory norm all-reduce.  φ must be
bit-identical to the oracle's N1+N2 sweeps, max-norms bit-identical, Σr²
within 1e-12.  The two solves have different lengths and the
second starts from whichever buffer holds φ^N1 (registered pair swapped)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle
from paper_2307_07931_b200 import protox as P

from helpers import BC_MAP, bits_equal, ulp_diff

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUM_RTOL = 1e-12


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(tmp_path, world, bc, n0, n1, na, nb, E, seed, st, graph, inf_row=-1, extra_env=None):
    port = _port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   **(extra_env or {}))
        args = [sys.executable, os.path.join(ROOT, "tests", "_p2p_worker.py"), str(tmp_path), *map(str, (
            bc, n0, n1, na, nb, E, seed, st, graph, inf_row))]
        procs.append(subprocess.Popen(args, env=env, cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                      text=True, start_new_session=True))
    outs = []
    try:
        for p in procs:
            outs.append(p.communicate(timeout=300)[0])
    finally:
        for p in procs:
            if p.poll() is None:
                os.killpg(p.pid, 9)
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-4000:]
    return [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]


@pytest.mark.parametrize("world,bc,st,graph,sep", [
    (2, P.PX_BC_PERIODIC, 0, 1, 0),
    (3, P.PX_BC_PERIODIC, 1, 0, 0),
    (2, P.PX_BC_DIRICHLET_CC, 0, 0, 0),
    (3, P.PX_BC_FIXED_GHOSTS, 1, 1, 0),
    (3, P.PX_BC_PERIODIC, 1, 1, 1),
    (2, P.PX_BC_DIRICHLET_CC, 1, 0, 1),
])
def test_p2p_push_across_processes(tmp_path, world, bc, st, graph, sep):
    """sep = 1: the ghost ring by a fill kernel per sweep (the path of slabs
    >= 64 M cells, forced here by PROTOX_SEP_FILL_CELLS=0); the pushed rows
    then carry their corner images themselves (9-point needs them)."""
    n0, n1, na, nb, E, seed = 384, 96 * world, 7, 6, 1, 4100 + world + 10 * bc
    res = _run(tmp_path, world, bc, n0, n1, na, nb, E, seed, st, graph,
               extra_env={"PROTOX_SEP_FILL_CELLS": "0"} if sep else None)
    for r in res:
        assert str(r["kernels"]) == "k_bulk", str(r["kernels"])  # one sweep kernel: the push is fused
    g = 1
    rng = np.random.default_rng(seed)
    phi0 = rng.uniform(-1, 1, (n1 + 2 * g, n0 + 2 * g))
    rho = rng.uniform(-1, 1, (n1 + 2 * g, n0 + 2 * g))
    prob = oracle.Problem(n0, n1, 1.0 / n0, 1.0 / (8.0 * n0 * n0), b0=n0, b1=n1 // (2 * world), ghost=g,
                          bc=BC_MAP[bc], stencil=st, nsweeps=na + nb, norm_every=E)
    ref, rn = oracle.solve(prob, phi0, rho)
    got = np.concatenate([r["phi"] for r in sorted(res, key=lambda r: int(r["y0"]))], axis=0)
    assert bits_equal(got, ref[1:-1, 1:-1]), ulp_diff(got, ref[1:-1, 1:-1])
    # every rank holds the same all-reduced norms (same bits: rank-order sum)
    for r in res[1:]:
        assert bits_equal(r["n1"], res[0]["n1"]) and bits_equal(r["n2"], res[0]["n2"])
    n1s, n2s = res[0]["n1"], res[0]["n2"]
    # solve 1's final entry is the residual of φ^na, which solve 2 records first
    assert n1s.shape[0] == na // E + 1 and n2s.shape[0] == nb // E + 1
    bad = [j for j in range(na // E + 1) if n1s[j, 0] != rn[j, 0]]
    assert not bad, ("solve 1", bad, n1s[bad, 0], rn[bad, 0])
    bad = [j for j in range(nb // E + 1) if n2s[j, 0] != rn[na // E + j, 0]]
    assert not bad, ("solve 2", bad, n2s[bad, 0], rn[[na // E + j for j in bad], 0])
    gpu = np.concatenate([n1s[:-1], n2s])
    assert gpu.shape == rn.shape
    assert bits_equal(gpu[:, 0], rn[:, 0]), np.max(np.abs(gpu[:, 0] - rn[:, 0]))
    np.testing.assert_allclose(gpu[:, 1], rn[:, 1], rtol=SUM_RTOL, atol=0)


def test_p2p_inf_nan_through_peer_allreduce(tmp_path):
    """ρ = +inf at one cell of the LAST rank's slab (3 processes): r(φ⁰) is
    inf only there, so the peer-memory all-reduce must give max = inf on
    every rank at entry 0, then NaN (inf - inf) from entry 1 on (reading R7,
    P:173); the field's NaN region spreads across the slab boundaries through
    the pushed ghost rows and must match the oracle's NaN mask exactly, every
    other cell bit for bit."""
    world, bc, n0, n1, na, nb, E, seed = 3, P.PX_BC_PERIODIC, 256, 288, 3, 4, 1, 77
    inf_row = n1 - 3
    res = _run(tmp_path, world, bc, n0, n1, na, nb, E, seed, 0, 1, inf_row)
    g = 1
    rng = np.random.default_rng(seed)
    phi0 = rng.uniform(-1, 1, (n1 + 2 * g, n0 + 2 * g))
    rho = rng.uniform(-1, 1, (n1 + 2 * g, n0 + 2 * g))
    rho[g + inf_row, g + n0 // 3] = np.inf
    prob = oracle.Problem(n0, n1, 1.0 / n0, 1.0 / (8.0 * n0 * n0), b0=n0, b1=n1 // (2 * world), ghost=g,
                          bc=BC_MAP[bc], stencil=0, nsweeps=na + nb, norm_every=E)
    ref, rn = oracle.solve(prob, phi0, rho)
    got = np.concatenate([r["phi"] for r in sorted(res, key=lambda r: int(r["y0"]))], axis=0)
    ref = np.ascontiguousarray(ref[1:-1, 1:-1])
    mg, mr = np.isnan(got), np.isnan(ref)
    assert mr.any() and np.array_equal(mg, mr), (mg.sum(), mr.sum())
    assert bits_equal(got[~mg], ref[~mr])
    for r in res[1:]:
        assert bits_equal(r["n1"], res[0]["n1"]) and bits_equal(r["n2"], res[0]["n2"])
    gn = np.concatenate([res[0]["n1"][:-1], res[0]["n2"]])
    assert gn[0, 0] == np.inf and rn[0, 0] == np.inf
    assert np.array_equal(np.isnan(gn[:, 0]), np.isnan(rn[:, 0])), (gn[:, 0], rn[:, 0])
    assert np.isnan(gn[1:, 0]).all()
    assert np.array_equal(np.isnan(gn[:, 1]), np.isnan(rn[:, 1]))


def test_p2p_lost_peer_reports_instead_of_hanging(tmp_path):
    """A rank whose neighbour never runs its solve: the bounded peer waits
    (px_spin_until, %globaltimer) give up after PX_SPIN_TIMEOUT_NS and
    px_solve returns PX_ERR_STATE ('timed out') within seconds -- a lost or
    stalled peer ends the solve with an error, not a GPU hang."""
    res = _run(tmp_path, 2, P.PX_BC_PERIODIC, 384, 192, 4, 1, 1, 5, 0, 0,
               extra_env={"PROTOX_TEST_LOST_PEER": "1"})
    assert "timed out" in str(res[0]["msg"]), str(res[0]["msg"])
    assert float(res[0]["secs"]) < 60.0

