"""GPU parity of the 3D relaxation (px3_*) against
the 3D oracle (oracle/protox_oracle3d.cpp, pinned in tests/test_oracle_pins3d.py)
on the same seeded inputs: φ bit-identical, max-norms bit-identical, Σr²
within 1e-12 relative (different summation order, R16).  Shapes
span several 64 x 32 tiles with ragged tails in every dimension, several z
chunks, all three boundary rules and the norm schedules; the full-size case
(512³, the bench's launch configuration) is checked on sampled cells by
oracle windows around them."""
import math

import numpy as np
import pytest

import oracle
from paper_2307_07931_b200 import inputs
from paper_2307_07931_b200 import protox as P

from helpers import BC_MAP, bits_equal, ulp_diff

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SUM_RTOL = 1e-12
BCS = [P.PX_BC_PERIODIC, P.PX_BC_DIRICHLET_CC, P.PX_BC_FIXED_GHOSTS]


def _upload(grid, glob):
    t = grid.alloc()
    grid.view(t, ghosts=True).copy_(torch.from_numpy(np.ascontiguousarray(glob)))
    return t


def _fields(n, g, seed):
    rng = np.random.default_rng(seed)
    shape = (n[2] + 2 * g, n[1] + 2 * g, n[0] + 2 * g)
    return rng.uniform(-1, 1, shape), rng.uniform(-1, 1, shape)


def _check_norms(gpu, orc):
    assert gpu.shape == orc.shape, (gpu.shape, orc.shape)
    assert bits_equal(gpu[:, 0], orc[:, 0]), (gpu[:, 0], orc[:, 0])
    np.testing.assert_allclose(gpu[:, 1], orc[:, 1], rtol=SUM_RTOL, atol=0)


def run3(n, bc, N, E, seed=1, graph=True, g=1, h=None, lam=None, phi0=None, rho=None):
    h = h or 1.0 / max(n)
    lam = lam if lam is not None else h * h / 12  # λ = h²/(4D), D = 3
    if phi0 is None:
        phi0, rho = _fields(n, g, seed)
    grid = P.Grid3(n, g)
    a, b, r = _upload(grid, phi0), grid.alloc(), _upload(grid, rho)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    res = P.solve3(grid, bc, P.relax_params(h, lam, P.PX_LAPLACE_7PT_3D), N, E, a, b, r, use_graph=graph,
                   stream=s)
    out = grid.view(b if res.in_scratch else a).cpu().numpy()
    p = oracle.Problem3(n, h, lam, ghost=g, bc=BC_MAP[bc], nsweeps=N, norm_every=E)
    ref, rn = oracle.solve3(p, phi0, rho)
    return out, res.norms, ref[g:-g, g:-g, g:-g], rn


@pytest.mark.parametrize("bc", BCS)
@pytest.mark.parametrize("n", [(64, 32, 6), (70, 37, 13), (130, 65, 9), (5, 3, 2), (1, 1, 1)])
def test_solve3_bitwise(bc, n):
    out, norms, ref, rn = run3(n, bc, 7, 2, seed=sum(n) + bc)
    assert bits_equal(out, ref), ulp_diff(out, ref)
    _check_norms(norms, rn)


@pytest.mark.parametrize("E", [-1, 0, 1, 3])
@pytest.mark.parametrize("graph", [True, False])
def test_solve3_norm_schedules_and_graph(E, graph):
    n = (96, 40, 11)
    out, norms, ref, rn = run3(n, P.PX_BC_PERIODIC, 6, E, seed=7 + E, graph=graph)
    assert bits_equal(out, ref)
    if E >= 0:
        _check_norms(norms, rn)
    else:
        assert norms.shape[0] == 0


@pytest.mark.parametrize("N,E", [(0, 1), (0, 0), (3, 5), (4, 4), (1, 1)])
def test_solve3_zero_sweeps_and_sparse_norms(N, E):
    """N = 0 returns φ⁰ untouched in φ (and the norm of φ⁰ when E >= 0); norm
    periods longer than the solve report only the final sweep's norm."""
    n = (40, 24, 5)
    out, norms, ref, rn = run3(n, P.PX_BC_DIRICHLET_CC, N, E, seed=40 + N + E)
    assert bits_equal(out, ref)
    _check_norms(norms, rn)


@pytest.mark.parametrize("N,E", [(0, 0), (4, 3), (6, -1)])
def test_solve3_mehrstellen27_norm_schedules(N, E):
    n = (48, 20, 6)
    h = 1.0 / 48
    lam = h * h / 12
    phi0, rho = _fields(n, 1, 77 + N)
    grid = P.Grid3(n, 1)
    a, b, r = _upload(grid, phi0), grid.alloc(), _upload(grid, rho)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    res = P.solve3(grid, P.PX_BC_PERIODIC, P.relax_params(h, lam, P.PX_MEHRSTELLEN_27PT_3D), N, E, a, b, r,
                   use_graph=False, stream=s)
    out = grid.view(b if res.in_scratch else a).cpu().numpy()
    ref, rn = oracle.solve3(oracle.Problem3(n, h, lam, nsweeps=N, norm_every=E, stencil=1), phi0, rho)
    assert bits_equal(out, ref[1:-1, 1:-1, 1:-1])
    if E < 0:
        assert res.norms.shape[0] == 0
    else:
        _check_norms(res.norms, rn)


def test_solve3_many_z_chunks_and_ghost2():
    """z extent large enough that the planner splits columns into several z
    chunks (each re-reads its first plane); ghost width 2; non-pow2 h."""
    n = (64, 64, 150)
    out, norms, ref, rn = run3(n, P.PX_BC_DIRICHLET_CC, 5, 1, seed=3, g=2, h=1.0 / 150)
    assert bits_equal(out, ref), ulp_diff(out, ref)
    _check_norms(norms, rn)


def test_solve3_repeat_replays_cached_graph():
    n = (66, 34, 8)
    phi0, rho = _fields(n, 1, 5)
    grid = P.Grid3(n, 1)
    a, b, r = _upload(grid, phi0), grid.alloc(), _upload(grid, rho)
    prm = P.relax_params(1 / 66, (1 / 66) ** 2 / 12, P.PX_LAPLACE_7PT_3D)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    r1 = P.solve3(grid, P.PX_BC_PERIODIC, prm, 4, 1, a, b, r, use_graph=True, stream=s)
    r2 = P.solve3(grid, P.PX_BC_PERIODIC, prm, 4, 1, a, b, r, use_graph=True, stream=s)  # continues from φ^4
    p = oracle.Problem3(n, 1 / 66, (1 / 66) ** 2 / 12, nsweeps=8, norm_every=1)
    ref, rn = oracle.solve3(p, phi0, rho)
    out = grid.view(b if r2.in_scratch else a).cpu().numpy()
    assert bits_equal(out, ref[1:-1, 1:-1, 1:-1])
    assert bits_equal(np.concatenate([r1.norms[:4, 0], r2.norms[:, 0]]), rn[:, 0])


def test_relax_step3_and_residual_vs_oracle():
    n = (100, 50, 7)
    h = 1 / 100
    lam = h * h / 12
    phi0, rho = _fields(n, 1, 9)
    grid = P.Grid3(n, 1)
    a, b, r = _upload(grid, phi0), grid.alloc(), _upload(grid, rho)
    prm = P.relax_params(h, lam, P.PX_LAPLACE_7PT_3D)
    nb, nb2 = P.norm_buffer3(), P.norm_buffer3()
    P.fill_ghosts3(grid, P.PX_BC_PERIODIC, a)
    P.relax_step3(prm, grid, a, b, r, nb)
    P.fill_ghosts3(grid, P.PX_BC_PERIODIC, b)
    P.residual_norm3(prm, grid, b, r, nb2)
    torch.cuda.synchronize()
    p = oracle.Problem3(n, h, lam, nsweeps=1, norm_every=1)
    ref, rn = oracle.solve3(p, phi0, rho)
    assert bits_equal(grid.view(b).cpu().numpy(), ref[1:-1, 1:-1, 1:-1])
    got = np.array([nb[:2].cpu().numpy(), nb2[:2].cpu().numpy()])
    _check_norms(got, rn)


@pytest.mark.parametrize("bc", [P.PX_BC_PERIODIC, P.PX_BC_DIRICHLET_CC])
@pytest.mark.parametrize("g", [1, 2])
def test_fill_ghosts3_matches_oracle_exchange(bc, g):
    n = (9, 6, 5)
    rng = np.random.default_rng(4)
    glob = rng.uniform(-1, 1, (n[2] + 2 * g, n[1] + 2 * g, n[0] + 2 * g))
    grid = P.Grid3(n, g)
    t = _upload(grid, glob)
    P.fill_ghosts3(grid, bc, t)
    torch.cuda.synchronize()
    want = oracle.exchange3(oracle.Problem3(n, 1.0, 0.0, ghost=g, bc=BC_MAP[bc]), glob)
    assert bits_equal(grid.view(t, ghosts=True).cpu().numpy(), want)


def test_init_field3_hash_bitwise():
    n = (37, 20, 11)
    grid = P.Grid3(n, 1)
    t = grid.alloc()
    P.init_field3(grid, t, 1, inputs.DEFAULT_SEED)
    torch.cuda.synchronize()
    assert bits_equal(grid.view(t).cpu().numpy(), inputs.hash_field3(*n))


def test_nan_propagates3():
    n = (64, 32, 4)
    phi0, rho = _fields(n, 1, 2)
    phi0[2, 5, 9] = np.nan
    out, norms, ref, rn = run3(n, P.PX_BC_PERIODIC, 1, 1, phi0=phi0, rho=rho)
    assert math.isnan(norms[0, 0]) and math.isnan(rn[0, 0])


def test_errors3():
    grid = P.Grid3((16, 8, 4), 1)
    a, b, r = grid.alloc(), grid.alloc(), grid.alloc()
    with pytest.raises(P.PxError, match="PX_LAPLACE_7PT_3D"):
        P.solve3(grid, 0, P.relax_params(1 / 16, 1e-4, P.PX_LAPLACE_5PT), 2, 1, a, b, r)
    with pytest.raises(P.PxError, match="differ"):
        P.solve3(grid, 0, P.relax_params(1 / 16, 1e-4, P.PX_LAPLACE_7PT_3D), 2, 1, a, a, r)
    g2 = P.Grid3((16, 8, 5), 1)
    c = g2.alloc()
    pa, pc = grid.patch(a), g2.patch(c)
    import ctypes
    nb = P.norm_buffer3()
    st = P.lib().px3_relax_step(ctypes.byref(P.relax_params(1 / 16, 1e-4, P.PX_LAPLACE_7PT_3D)), ctypes.byref(pa),
                                ctypes.byref(pc), ctypes.byref(pa), ctypes.c_void_p(nb.data_ptr()), None)
    assert st == P.PX_ERR_SHAPE
    bad = grid.patch(a)
    bad.data += 8  # misaligned cell (0,0,0)
    st = P.lib().px3_fill_ghosts(0, ctypes.byref(bad), None)
    assert st == P.PX_ERR_ALIGN


# ------------------------------------------------------------ full size (512³)
def test_full_size_512_sampled_windows():
    """512³ periodic, hash ρ (device generator), φ⁰ = 0, N = 12 sweeps in the
    bench's launch configuration: each sampled cell is recomputed by the
    oracle on the (2N+1)³ window around it (FIXED ghosts one layer further
    out cannot reach the centre in N sweeps) -- bit-identical; the recorded
    norm of φ⁰ equals the closed form r(0) = −ρ."""
    n = (512, 512, 512)
    N = 12
    h = 1 / 512
    lam = h * h / 12
    grid = P.Grid3(n, 1)
    a, b, r = grid.alloc(), grid.alloc(), grid.alloc()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    P.init_field3(grid, r, 1, inputs.DEFAULT_SEED, stream=s)
    res = P.solve3(grid, P.PX_BC_PERIODIC, P.relax_params(h, lam, P.PX_LAPLACE_7PT_3D), N, 1, a, b, r,
                   use_graph=True, stream=s)
    out_t = b if res.in_scratch else a
    vw = grid.view(out_t)
    assert res.norms[0, 0] == float(grid.view(r).abs().max().item())  # r(φ⁰ = 0) = −ρ
    rng = np.random.default_rng(12)
    samples = [(0, 0, 0), (511, 511, 511), (255, 3, 509)] + [tuple(int(v) for v in rng.integers(0, 512, 3))
                                                             for _ in range(3)]
    w = N  # window half-width
    m = 2 * w + 1
    for (x, y, z) in samples:
        idx = [(np.arange(c - w - 1, c + w + 2) % 512) for c in (x, y, z)]
        iz, iy, ix = np.meshgrid(idx[2], idx[1], idx[0], indexing="ij")
        rho_g = inputs.hash_values3(ix, iy, iz, n[0], n[1])
        p = oracle.Problem3((m, m, m), h, lam, bc=oracle.BC_FIXED, nsweeps=N, norm_every=-1)
        ref, _ = oracle.solve3(p, np.zeros(p.gshape), np.ascontiguousarray(rho_g))
        got = float(vw[z, y, x].item())
        want = ref[w + 1, w + 1, w + 1]
        assert np.float64(got).view(np.uint64) == np.float64(want).view(np.uint64), ((x, y, z), got, want)


# ------------------------------------------------------- 27-point Mehrstellen (R-3D4)
@pytest.mark.parametrize("bc", BCS)
@pytest.mark.parametrize("n", [(64, 32, 5), (70, 37, 9), (3, 2, 2)])
def test_solve3_mehrstellen27_bitwise(bc, n):
    h = 1.0 / max(n)
    lam = h * h / 12
    phi0, rho = _fields(n, 1, 100 + sum(n) + bc)
    grid = P.Grid3(n, 1)
    a, b, r = _upload(grid, phi0), grid.alloc(), _upload(grid, rho)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    res = P.solve3(grid, bc, P.relax_params(h, lam, P.PX_MEHRSTELLEN_27PT_3D), 5, 2, a, b, r, use_graph=True,
                   stream=s)
    out = grid.view(b if res.in_scratch else a).cpu().numpy()
    p = oracle.Problem3(n, h, lam, bc=BC_MAP[bc], nsweeps=5, norm_every=2, stencil=1)
    ref, rn = oracle.solve3(p, phi0, rho)
    assert bits_equal(out, ref[1:-1, 1:-1, 1:-1]), ulp_diff(out, ref[1:-1, 1:-1, 1:-1])
    _check_norms(res.norms, rn)


@pytest.mark.parametrize("bc", [P.PX_BC_PERIODIC, P.PX_BC_DIRICHLET_CC])
def test_mehrstellen27_corrected_rhs_and_solve(bc):
    """px3_mehrstellen_rhs (ρ ghosts by the BC rule) then the 27-point solve ==
    the oracle with rhs_correction, bit for bit; several z chunks."""
    n = (66, 40, 70)
    h = 1.0 / 70
    lam = h * h / 12
    phi0, rho = _fields(n, 1, 55 + bc)
    grid = P.Grid3(n, 1)
    a, b, r = _upload(grid, phi0), grid.alloc(), _upload(grid, rho)
    f = grid.alloc()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    P.fill_ghosts3(grid, bc, r, stream=s)
    P.mehrstellen_rhs3(grid, r, f, stream=s)
    s.synchronize()
    p = oracle.Problem3(n, h, lam, bc=BC_MAP[bc], nsweeps=6, norm_every=1, stencil=1, rhs_correction=True)
    assert bits_equal(grid.view(f).cpu().numpy(), oracle.rhs3(p, rho))
    res = P.solve3(grid, bc, P.relax_params(h, lam, P.PX_MEHRSTELLEN_27PT_3D), 6, 1, a, b, f, use_graph=False,
                   stream=s)
    out = grid.view(b if res.in_scratch else a).cpu().numpy()
    ref, rn = oracle.solve3(p, phi0, rho)
    assert bits_equal(out, ref[1:-1, 1:-1, 1:-1]), ulp_diff(out, ref[1:-1, 1:-1, 1:-1])
    _check_norms(res.norms, rn)


# ------------------------------------------------------- z slabs over NCCL
@pytest.mark.parametrize("st,bc,graph", [(P.PX_LAPLACE_7PT_3D, P.PX_BC_PERIODIC, True),
                                         (P.PX_LAPLACE_7PT_3D, P.PX_BC_PERIODIC, False),
                                         (P.PX_MEHRSTELLEN_27PT_3D, P.PX_BC_PERIODIC, True),
                                         (P.PX_LAPLACE_7PT_3D, P.PX_BC_DIRICHLET_CC, True)])
def test_solve3_comm_nccl_self_exchange(st, bc, graph, monkeypatch):
    """px3_solve_comm with a one-rank NCCL communicator: in self-exchange mode
    (periodic) the z ghost planes travel through ncclSend/ncclRecv to the rank
    itself with the slab plan's posting order, inside the CUDA graph, and the
    norms are all-reduced -- bit-identical to the oracle; Dirichlet: local faces."""
    monkeypatch.setenv("PROTOX_NCCL_SELF_EXCHANGE", "1")
    n = (70, 37, 13)
    h = 1.0 / 70
    lam = h * h / 12
    phi0, rho = _fields(n, 1, 300 + st + bc)
    grid = P.Grid3(n, 1)
    a, b, r = _upload(grid, phi0), grid.alloc(), _upload(grid, rho)
    comm = P.Comm(P.comm_unique_id(), 1, 0, torch.cuda.current_device())
    try:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        res = P.solve3_comm(comm, grid, bc, P.relax_params(h, lam, st), 6, 2, a, b, r, use_graph=graph, stream=s)
        out = grid.view(b if res.in_scratch else a).cpu().numpy()
    finally:
        P.release3()
        comm.close()
    p = oracle.Problem3(n, h, lam, bc=BC_MAP[bc], nsweeps=6, norm_every=2,
                        stencil=0 if st == P.PX_LAPLACE_7PT_3D else 1)
    ref, rn = oracle.solve3(p, phi0, rho)
    assert bits_equal(out, ref[1:-1, 1:-1, 1:-1]), ulp_diff(out, ref[1:-1, 1:-1, 1:-1])
    _check_norms(res.norms, rn)


def test_init_field3_hash_slab_offset():
    """A z-slab's hash field (z0 = its first global plane) is the matching
    planes of the whole-domain field: every decomposition sees one ρ."""
    n = (20, 9, 12)
    full = inputs.hash_field3(*n)
    for z0, z1 in (P.slab3(12, 3, r) for r in range(3)):
        g = P.Grid3((n[0], n[1], z1 - z0), 1)
        t = g.alloc()
        P.init_field3(g, t, 1, inputs.DEFAULT_SEED, z0=z0)
        torch.cuda.synchronize()
        assert bits_equal(g.view(t).cpu().numpy(), full[z0:z1])


@pytest.mark.parametrize("st,bc,graph", [(P.PX_LAPLACE_7PT_3D, P.PX_BC_PERIODIC, True),
                                         (P.PX_LAPLACE_7PT_3D, P.PX_BC_DIRICHLET_CC, False),
                                         (P.PX_MEHRSTELLEN_27PT_3D, P.PX_BC_DIRICHLET_CC, True)])
def test_solve3_host_batch_bitwise(st, bc, graph):
    """px3_solve_host_batch: five problems (two with φ⁰ from the host, three from
    zero) through the three rotating buffer sets, each bit-identical to its
    own oracle solve; odd N (result in the scratch field)."""
    n, N, E = (70, 37, 9), 5, 2
    h = 1.0 / 70
    lam = h * h / 12
    probs = []
    for i in range(5):
        phi0, rho = _fields(n, 1, 500 + i)
        if i % 2:
            phi0 = np.zeros_like(phi0)
        probs.append((phi0, rho))
    outs = [torch.empty((n[2], n[1], n[0]), dtype=torch.float64).pin_memory().numpy() for _ in probs]
    rhos = [np.ascontiguousarray(r[1:-1, 1:-1, 1:-1]) for _, r in probs]
    phi0s = [None if i % 2 else np.ascontiguousarray(f[1:-1, 1:-1, 1:-1]) for i, (f, _) in enumerate(probs)]
    torch.cuda.synchronize()
    norms = P.solve3_host_batch(n, 1, bc, P.relax_params(h, lam, st), N, E, rhos, outs, phi0s, use_graph=graph,
                                stream=torch.cuda.Stream())
    for i, (phi0, rho) in enumerate(probs):
        # the oracle starts from the same owned cells (its ghosts are refilled every sweep)
        p = oracle.Problem3(n, h, lam, bc=BC_MAP[bc], nsweeps=N, norm_every=E,
                            stencil=0 if st == P.PX_LAPLACE_7PT_3D else 1)
        ref, rn = oracle.solve3(p, phi0, rho)
        assert bits_equal(outs[i], ref[1:-1, 1:-1, 1:-1]), (i, ulp_diff(outs[i], ref[1:-1, 1:-1, 1:-1]))
        _check_norms(norms[i], rn)


def test_solve3_host_batch_rejects_fixed_ghosts_and_bad_shapes():
    n = (8, 8, 4)
    z = np.zeros((4, 8, 8))
    prm = P.relax_params(1 / 8, 1 / 768, P.PX_LAPLACE_7PT_3D)
    with pytest.raises(P.PxError):
        P.solve3_host_batch(n, 1, P.PX_BC_FIXED_GHOSTS, prm, 2, 1, [z], [z.copy()], stream=torch.cuda.Stream())
    with pytest.raises(ValueError):
        P.solve3_host_batch(n, 1, P.PX_BC_PERIODIC, prm, 2, 1, [np.zeros((8, 8, 4))], [z.copy()],
                            stream=torch.cuda.Stream())
