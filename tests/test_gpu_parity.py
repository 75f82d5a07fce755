"""GPU parity: libprotox (through its C ABI) against the CPU oracle on the
same seeded inputs.  Bar: φ bit-identical to the oracle
(canonical expression tree, every * and + rounded separately), max-norms
bit-identical (max is order-independent), Σr² within 1e-12 relative
(different summation order; BASELINE north star tolerance 1e-12)."""
import math

import numpy as np
import pytest

import oracle
from paper_2307_07931_b200 import inputs
from paper_2307_07931_b200 import protox as P

from helpers import BC_MAP, bits_equal, owned_to_host, rel_max, to_device_ghosted, ulp_diff

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SUM_RTOL = 1e-12


def _orc_problem(n0, n1, h, lam, bc, st, nsweeps, E, b0=None, b1=None, g=1, corr=False):
    return oracle.Problem(n0, n1, h, lam, b0=b0 or n0, b1=b1 or n1, ghost=g, bc=BC_MAP[bc],
                          stencil=st, rhs_correction=corr, nsweeps=nsweeps, norm_every=E)


def _fields(n0, n1, g, seed, bc, kind="random"):
    rng = np.random.default_rng(seed)
    if kind == "random":
        phi0 = rng.uniform(-1, 1, (n1 + 2 * g, n0 + 2 * g))
        rho = rng.uniform(-1, 1, (n1 + 2 * g, n0 + 2 * g))
    else:
        phi0 = np.zeros((n1 + 2 * g, n0 + 2 * g))
        rho = np.zeros_like(phi0)
        rho[g:g + n1, g:g + n0] = inputs.sine_field(n0, n1)
    return phi0, rho


def _check_norms(gpu, orc):
    assert gpu.shape == orc.shape, (gpu.shape, orc.shape)
    assert bits_equal(gpu[:, 0], orc[:, 0]), np.max(np.abs(gpu[:, 0] - orc[:, 0]))
    np.testing.assert_allclose(gpu[:, 1], orc[:, 1], rtol=SUM_RTOL, atol=0)


def run_gpu_solve(n0, n1, h, lam, bc, st, N, E, phi0_g, rho_g, g=1, box=None, nranks=1,
                  graph=True, corr=False, tk=1, async_=False):
    """Solve on the GPU; nranks > 1 runs all slabs on this device (local
    transport); async_: through px_solve_async (norms in device memory)."""
    dom = P.box(0, 0, n0 - 1, n1 - 1)
    lay = P.Layout(dom, box or (n0, n1 // nranks), g, bc, nranks)
    phis, scrs, rhss, fs = [], [], [], []
    for r in range(nranks):
        phis.append(to_device_ghosted(lay, r, phi0_g, g))
        scrs.append(lay.alloc(r))
        rhss.append(to_device_ghosted(lay, r, rho_g, g))
    if corr:
        # Mehrstellen right-hand side f = ρ + S5(ρ)/12 (ρ ghosts by the BC rule)
        parts = [lay.patch(r, rhss[r]) for r in range(nranks)]
        P.exchange_ghosts_local(lay, parts)
        for r in range(nranks):
            f = lay.alloc(r)
            P.mehrstellen_rhs(lay.patch(r, rhss[r]), lay.patch(r, f), lay.local(r).owned)
            fs.append(f)
        rhss = fs
    if tk > 1:
        # temporal blocking advances ghost cells too: ρ needs its ghosts (depth >= k)
        P.exchange_ghosts_local(lay, [lay.patch(r, t) for r, t in enumerate(rhss)])
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())  # allocations/copies ran on the current stream
    parts = ([lay.patch(r, t) for r, t in enumerate(phis)], [lay.patch(r, t) for r, t in enumerate(scrs)],
             [lay.patch(r, t) for r, t in enumerate(rhss)])
    if async_:
        ne = 0 if E < 0 else ((N + E - 1) // E if E > 0 else 0) + 1
        d = torch.full((2 * max(ne, 1),), -1.0, dtype=torch.float64, device="cuda")
        nw, ins = P.solve_async(lay, None, 0, P.relax_params(h, lam, st), N, E, *parts, d, use_graph=graph,
                                stream=stream, temporal_k=tk)
        stream.synchronize()
        norms = d.view(-1, 2)[:nw].cpu().numpy()
    else:
        res = P.solve(lay, None, 0, P.relax_params(h, lam, st), N, E, *parts, use_graph=graph, stream=stream,
                      temporal_k=tk)
        norms, ins = res.norms, res.in_scratch
    out_t = scrs if ins else phis
    out = np.concatenate([owned_to_host(lay, r, out_t[r]) for r in range(nranks)], axis=0)
    return out, norms, lay


# --------------------------------------------------------- single sweep
@pytest.mark.parametrize("bc", [P.PX_BC_PERIODIC, P.PX_BC_DIRICHLET_CC, P.PX_BC_FIXED_GHOSTS])
@pytest.mark.parametrize("st", [P.PX_LAPLACE_5PT, P.PX_MEHRSTELLEN_9PT])
@pytest.mark.parametrize("shape", [(64, 64), (1000, 77), (3, 5), (513, 70)])
def test_relax_step_bitwise(bc, st, shape):
    n0, n1 = shape
    h = 1.0 / max(n0, n1)
    lam = h * h / 8 if st == P.PX_LAPLACE_5PT else 3 * h * h / 16
    phi0, rho = _fields(n0, n1, 1, 7 + n0, bc)
    p = _orc_problem(n0, n1, h, lam, bc, st, 1, 1)
    ref, rnorm = oracle.solve(p, phi0, rho)
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (n0, n1), 1, bc, 1)
    a = to_device_ghosted(lay, 0, phi0, 1)
    b = lay.alloc(0)
    r = to_device_ghosted(lay, 0, rho, 1)
    P.fill_ghosts(lay, 0, lay.patch(0, a))
    nb = P.norm_buffer(lay.local(0).owned)
    P.relax_step(P.relax_params(h, lam, st), lay.patch(0, a), lay.patch(0, b), lay.patch(0, r),
                 lay.local(0).owned, nb)
    torch.cuda.synchronize()
    out = owned_to_host(lay, 0, b)
    assert bits_equal(out, ref[1:-1, 1:-1]), ulp_diff(out, ref[1:-1, 1:-1])
    nrm = nb[:2].cpu().numpy()
    assert nrm[0] == rnorm[0, 0]
    assert abs(nrm[1] - rnorm[0, 1]) <= SUM_RTOL * rnorm[0, 1]
    # the scratch of the norm buffer is left zeroed for the next call
    assert torch.count_nonzero(nb[2:4]).item() == 0


def test_relax_step_unaligned_region_and_phase():
    """A region starting at an odd column (pairs start at column -1) and
    a sub-region of the patch."""
    n0, n1 = 130, 40
    h = 1.0 / 128
    lam = h * h / 8
    phi0, rho = _fields(n0, n1, 1, 3, P.PX_BC_PERIODIC)
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (n0, n1), 1, P.PX_BC_PERIODIC, 1)
    a = to_device_ghosted(lay, 0, phi0, 1)
    b = lay.alloc(0)
    r = to_device_ghosted(lay, 0, rho, 1)
    P.fill_ghosts(lay, 0, lay.patch(0, a))
    region = P.box(7, 3, 100, 30)
    nb = P.norm_buffer(region)
    P.relax_step(P.relax_params(h, lam), lay.patch(0, a), lay.patch(0, b), lay.patch(0, r), region, nb)
    torch.cuda.synchronize()
    p = _orc_problem(n0, n1, h, lam, P.PX_BC_PERIODIC, 0, 1, 1)
    ref, _ = oracle.solve(p, phi0, rho)
    out = owned_to_host(lay, 0, b)
    assert bits_equal(out[3:31, 7:101], ref[1:-1, 1:-1][3:31, 7:101])
    # cells outside the region are untouched (zero)
    assert np.all(out[:3] == 0) and np.all(out[:, :7] == 0) and np.all(out[:, 101:] == 0)
    # residual of φ^0 restricted to the region
    lapl = oracle.apply_laplacian(p, phi0)
    rr = (lapl - rho[1:-1, 1:-1])[3:31, 7:101]
    assert nb[0].item() == np.max(np.abs(rr))


# ------------------------------------------------------------ full solves
def test_config1_full_bitwise_and_closed_form():
    """BASELINE config 1: 64x64 box, 1 ghost layer, Dirichlet-CC, 100 sweeps,
    ρ = sin πx sin πy, λ = 2^-15, norms every sweep."""
    n, N = 64, 100
    h, lam = 1.0 / 64, 2.0**-15
    phi0, rho = _fields(n, n, 1, 0, P.PX_BC_DIRICHLET_CC, kind="sine")
    out, norms, _ = run_gpu_solve(n, n, h, lam, P.PX_BC_DIRICHLET_CC, 0, N, 1, phi0, rho)
    ref, rn = oracle.solve(_orc_problem(n, n, h, lam, P.PX_BC_DIRICHLET_CC, 0, N, 1), phi0, rho)
    assert bits_equal(out, ref[1:-1, 1:-1])
    _check_norms(norms, rn)
    g = math.cos(math.pi / 128) ** 2
    np.testing.assert_allclose(norms[:, 0], g ** (np.arange(101) + 1), rtol=2e-13)


@pytest.mark.parametrize("kind", ["sine", "hash"])
def test_config2_full_bitwise(kind):
    """BASELINE config 2: 1024² single box, periodic, 1000 sweeps, max-norm every 10."""
    n, N, E = 1024, 1000, 10
    h, lam = 1.0 / n, 2.0**-23
    phi0 = np.zeros((n + 2, n + 2))
    rho = np.zeros_like(phi0)
    rho[1:-1, 1:-1] = inputs.sine_field(n, n, 2, 2) if kind == "sine" else inputs.hash_field(n, n)
    out, norms, _ = run_gpu_solve(n, n, h, lam, P.PX_BC_PERIODIC, 0, N, E, phi0, rho)
    ref, rn = oracle.solve(_orc_problem(n, n, h, lam, P.PX_BC_PERIODIC, 0, N, E), phi0, rho)
    assert norms.shape == (101, 2)
    assert bits_equal(out, ref[1:-1, 1:-1]), ulp_diff(out, ref[1:-1, 1:-1])
    _check_norms(norms, rn)
    if kind == "sine":
        g = math.cos(math.pi / n) ** 2
        m = np.arange(0, 1001, 10)
        np.testing.assert_allclose(norms[:, 0], g**m * np.max(np.abs(rho)), rtol=1e-12)


@pytest.mark.parametrize("bc", [P.PX_BC_PERIODIC, P.PX_BC_DIRICHLET_CC, P.PX_BC_FIXED_GHOSTS])
@pytest.mark.parametrize("st", [P.PX_LAPLACE_5PT, P.PX_MEHRSTELLEN_9PT])
@pytest.mark.parametrize("graph", [True, False])
def test_solve_ragged_multibox(bc, st, graph):
    """Non-power-of-two, ragged shapes (last warp strip and row chunk partial),
    several boxes, odd sweep count (result in scratch), norms every 3."""
    n0, n1, N, E = 600, 90, 17, 3
    h = 1.0 / 600
    lam = h * h / 8 if st == 0 else 3 * h * h / 16
    phi0, rho = _fields(n0, n1, 1, 11, bc)
    out, norms, _ = run_gpu_solve(n0, n1, h, lam, bc, st, N, E, phi0, rho, box=(200, 30), graph=graph)
    ref, rn = oracle.solve(_orc_problem(n0, n1, h, lam, bc, st, N, E, b0=200, b1=30), phi0, rho)
    assert bits_equal(out, ref[1:-1, 1:-1]), ulp_diff(out, ref[1:-1, 1:-1])
    _check_norms(norms, rn)


@pytest.mark.parametrize("shape", [(64, 64), (3, 5), (1, 40), (40, 1), (127, 129), (100, 40), (62, 52), (18, 7),
                                   (2, 64), (6, 30)])
@pytest.mark.parametrize("bc", [P.PX_BC_PERIODIC, P.PX_BC_DIRICHLET_CC, P.PX_BC_FIXED_GHOSTS])
@pytest.mark.parametrize("st", [P.PX_LAPLACE_5PT, P.PX_MEHRSTELLEN_9PT])
def test_solve_whole_box_shapes(shape, bc, st):
    """Whole-box solves in one launch: k_boxw (one warp per row group, the box
    in registers) with four rows per warp (64 x 64, 62 x 52: a partial warp,
    2 x 64: one column pair), two (6 x 30) and one (40 x 1, 18 x 7), k_box1 with up to 4
    and up to 16 cells per thread (127 x 129 = 16383 cells), one-cell-wide
    boxes (a cell is then its own image on both sides), every BC and stencil; odd and even
    sweep counts and norm periods 1, 3 and 0 (final entry only)."""
    n0, n1 = shape
    h = 1.0 / 128
    lam = h * h / 8 if st == 0 else 3 * h * h / 16
    phi0, rho = _fields(n0, n1, 1, 29 + n0, bc)
    for N, E in ((9, 1), (10, 3), (7, 0)):
        out, norms, _ = run_gpu_solve(n0, n1, h, lam, bc, st, N, E, phi0, rho)
        ref, rn = oracle.solve(_orc_problem(n0, n1, h, lam, bc, st, N, E), phi0, rho)
        assert bits_equal(out, ref[1:-1, 1:-1]), (N, E, ulp_diff(out, ref[1:-1, 1:-1]))
        _check_norms(norms, rn)


@pytest.mark.parametrize("shape", [(130, 400), (1022, 149), (4, 5000), (1024, 101), (2048, 9), (1100, 900),
                                   (66, 1036), (1000, 700), (2, 600)])
@pytest.mark.parametrize("bc", [P.PX_BC_PERIODIC, P.PX_BC_DIRICHLET_CC, P.PX_BC_FIXED_GHOSTS])
@pytest.mark.parametrize("st", [P.PX_LAPLACE_5PT, P.PX_MEHRSTELLEN_9PT])
def test_solve_resident_shapes(shape, bc, st):
    """Shared-memory-resident solve (k_resident, LL row mailbox): uneven rows
    per CTA, one row per CTA, 34 rows x 2 column pairs per CTA (the rolled
    column walk), an odd CTA count (101, 9: the mailbox alignment), 9 CTAs of
    one row, 6-7 rows with more column pairs than threads (1100 x 900) and
    exactly 7 rows per CTA (the unrolled walk's limit); the register-resident
    kernel (k_resident_reg: nx/2 <= 512 pairs, <= 7 rows) with a partial last
    warp (1000 x 700) and a single pair (2 x 600); even and odd sweep counts
    (k_resident_reg2 ends an odd count with a one-level pass); norms every 4."""
    n0, n1 = shape
    h = 1.0 / 1024
    lam = h * h / 8 if st == 0 else 3 * h * h / 16
    phi0, rho = _fields(n0, n1, 1, 17, bc)
    for N in (10, 13):
        out, norms, _ = run_gpu_solve(n0, n1, h, lam, bc, st, N, 4, phi0, rho)
        ref, rn = oracle.solve(_orc_problem(n0, n1, h, lam, bc, st, N, 4), phi0, rho)
        assert bits_equal(out, ref[1:-1, 1:-1]), ulp_diff(out, ref[1:-1, 1:-1])
        _check_norms(norms, rn)


@pytest.mark.parametrize("bc", [P.PX_BC_PERIODIC, P.PX_BC_DIRICHLET_CC, P.PX_BC_FIXED_GHOSTS])
def test_solve_persistent_path(bc):
    """2500 x 300 does not fit the SMs' shared memory and is below the TMA
    kernel's size: the L2 persistent cooperative kernel (k_persist) runs."""
    n0, n1, N, E = 2500, 300, 9, 2
    h = 1.0 / 2048
    lam = h * h / 8
    phi0, rho = _fields(n0, n1, 1, 23, bc)
    out, norms, _ = run_gpu_solve(n0, n1, h, lam, bc, 0, N, E, phi0, rho, box=(500, 100))
    ref, rn = oracle.solve(_orc_problem(n0, n1, h, lam, bc, 0, N, E, b0=500, b1=100), phi0, rho)
    assert bits_equal(out, ref[1:-1, 1:-1]), ulp_diff(out, ref[1:-1, 1:-1])
    _check_norms(norms, rn)


@pytest.mark.parametrize("nranks", [2, 3, 4, 5, 8])
@pytest.mark.parametrize("bc", [P.PX_BC_PERIODIC, P.PX_BC_DIRICHLET_CC, P.PX_BC_FIXED_GHOSTS])
@pytest.mark.parametrize("st", [P.PX_LAPLACE_5PT, P.PX_MEHRSTELLEN_9PT])
def test_slab_decomposition_local_transport(nranks, bc, st):
    """Slabs of box-rows on one device exchanging by D2D copies: identical
    to the undecomposed oracle (decomposition invariance, P12), P = 2..8."""
    n0, n1, N, E = 256, 160, 12, 4
    h = 1.0 / 256
    lam = h * h / 8 if st == 0 else 3 * h * h / 16
    phi0, rho = _fields(n0, n1, 1, 5 + nranks, bc)
    out, norms, _ = run_gpu_solve(n0, n1, h, lam, bc, st, N, E, phi0, rho, box=(64, 10), nranks=nranks)
    ref, rn = oracle.solve(_orc_problem(n0, n1, h, lam, bc, st, N, E), phi0, rho)
    assert bits_equal(out, ref[1:-1, 1:-1]), ulp_diff(out, ref[1:-1, 1:-1])
    _check_norms(norms, rn)


@pytest.mark.parametrize("g", [2, 4])
def test_wider_ghosts_k1(g):
    n0, n1, N = 128, 96, 9
    h = 1.0 / 128
    lam = h * h / 8
    for bc in (P.PX_BC_PERIODIC, P.PX_BC_DIRICHLET_CC):
        phi0, rho = _fields(n0, n1, g, 2 + g, bc)
        out, norms, _ = run_gpu_solve(n0, n1, h, lam, bc, 0, N, 2, phi0, rho, g=g, box=(32, 32), nranks=3)
        ref, rn = oracle.solve(_orc_problem(n0, n1, h, lam, bc, 0, N, 2, g=g), phi0, rho)
        assert bits_equal(out, ref[g:-g, g:-g])
        _check_norms(norms, rn)


def test_mehrstellen_corrected_rhs_solve():
    """BASELINE config 5 shape at reduced size: Dirichlet-CC, Mehrstellen with
    f = ρ + S5(ρ)/12 computed on the device (px_mehrstellen_rhs)."""
    n, N = 256, 50
    h = 1.0 / n
    lam = 2.0**-19  # h²/8
    phi0, rho = _fields(n, n, 1, 0, P.PX_BC_DIRICHLET_CC, kind="sine")
    out, norms, _ = run_gpu_solve(n, n, h, lam, P.PX_BC_DIRICHLET_CC, 1, N, 5, phi0, rho,
                                  box=(64, 64), nranks=2, corr=True)
    p = _orc_problem(n, n, h, lam, P.PX_BC_DIRICHLET_CC, 1, N, 5, corr=True)
    ref, rn = oracle.solve(p, phi0, rho)
    assert bits_equal(out, ref[1:-1, 1:-1])
    _check_norms(norms, rn)


def test_norm_every_variants_and_zero_sweeps():
    n0, n1 = 96, 64
    h = 1.0 / 96
    lam = h * h / 8
    phi0, rho = _fields(n0, n1, 1, 1, P.PX_BC_PERIODIC)
    for N, E in [(0, 1), (0, 0), (5, 0), (5, -1), (6, 7), (8, 1)]:
        out, norms, _ = run_gpu_solve(n0, n1, h, lam, P.PX_BC_PERIODIC, 0, N, E, phi0, rho)
        ref, rn = oracle.solve(_orc_problem(n0, n1, h, lam, P.PX_BC_PERIODIC, 0, N, E), phi0, rho)
        assert bits_equal(out, ref[1:-1, 1:-1])
        if E < 0:
            assert norms.shape[0] == 0
        else:
            _check_norms(norms, rn)


def test_solve_host_e2e_matches_oracle():
    n0, n1, N = 256, 128, 20
    h = 1.0 / 256
    lam = h * h / 8
    phi0, rho = _fields(n0, n1, 1, 21, P.PX_BC_PERIODIC)
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (n0, n1), 1, P.PX_BC_PERIODIC, 1)
    torch.cuda.synchronize()
    out, norms = P.solve_host(lay, P.relax_params(h, lam), N, 5, phi0[1:-1, 1:-1], rho[1:-1, 1:-1],
                              stream=torch.cuda.Stream())
    ref, rn = oracle.solve(_orc_problem(n0, n1, h, lam, P.PX_BC_PERIODIC, 0, N, 5), phi0, rho)
    assert bits_equal(out, ref[1:-1, 1:-1])
    _check_norms(norms, rn)


@pytest.mark.parametrize("tk", [1, 4])
def test_solve_host_batch_matches_oracle(tk):
    """Pipelined host-buffer batch: each problem bit-identical to its own
    oracle solve; φ0 = NULL means zero; an odd sweep count leaves φ^N in the
    scratch buffer (the D2H must pick it)."""
    n0, n1, N, E = 256, 96, 19, 4
    g = 4 if tk > 1 else 1
    h = 1.0 / 256
    lam = h * h / 8
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (64, 32), g, P.PX_BC_PERIODIC, 1)
    probs = [_fields(n0, n1, g, 40 + i, P.PX_BC_PERIODIC) for i in range(5)]
    phi0s = [None if i % 2 == 0 else probs[i][0] for i in range(5)]
    rhos = [torch.from_numpy(np.ascontiguousarray(pr[1][g:g + n1, g:g + n0])).pin_memory() for pr in probs]
    outs = [torch.empty((n1, n0), dtype=torch.float64).pin_memory() for _ in probs]
    p0 = [None if q is None else np.ascontiguousarray(q[g:g + n1, g:g + n0]) for q in phi0s]
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    for rep in range(2):  # second call replays the cached plans / buffers
        norms = P.solve_host_batch(lay, P.relax_params(h, lam), N, E, [r.numpy() for r in rhos],
                                   [o.numpy() for o in outs], p0, stream=s, temporal_k=tk)
        for i, (phi0, rho) in enumerate(probs):
            if phi0s[i] is None:
                phi0 = np.zeros_like(phi0)
            ref, rn = oracle.solve(_orc_problem(n0, n1, h, lam, P.PX_BC_PERIODIC, 0, N, E, b0=64, b1=32, g=g),
                                   phi0, rho)
            assert bits_equal(outs[i].numpy(), ref[g:g + n1, g:g + n0]), (rep, i)
            _check_norms(norms[i], rn)


def test_solve_host_batch_errors():
    lay = P.Layout(P.box(0, 0, 63, 63), (64, 64), 1, P.PX_BC_PERIODIC, 1)
    a = np.zeros((64, 64))
    with pytest.raises(P.PxError):
        P.solve_host_batch(lay, P.relax_params(1 / 64, 1 / 64 ** 2 / 8), 4, 1, [a], [a.copy()], stream=0)
    assert P.solve_host_batch(lay, P.relax_params(1 / 64, 1 / 64 ** 2 / 8), 4, 1, [], [],
                              stream=torch.cuda.Stream()) == []


# ------------------------------------------------------------ other ops
@pytest.mark.parametrize("st", [P.PX_LAPLACE_5PT, P.PX_MEHRSTELLEN_9PT])
def test_stencil_apply_vs_oracle(st):
    n0, n1 = 200, 50
    rng = np.random.default_rng(8)
    src = rng.uniform(-1, 1, (n1 + 2, n0 + 2))
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (n0, n1), 1, P.PX_BC_FIXED_GHOSTS, 1)
    a = to_device_ghosted(lay, 0, src, 1)
    b = lay.alloc(0)
    scale = 3.0
    P.stencil_apply(st, scale, lay.patch(0, a), lay.patch(0, b), lay.local(0).owned)
    torch.cuda.synchronize()
    offs, alpha, _ = oracle.stencil_taps(st, 1.0)
    ref = oracle.apply_taps(offs, alpha, scale, src, (-1, -1), (0, 0), (n0 - 1, n1 - 1))
    assert bits_equal(owned_to_host(lay, 0, b), ref)


def test_stencil_apply_domain_violation():
    lay = P.Layout(P.box(0, 0, 63, 63), (64, 64), 1, P.PX_BC_PERIODIC, 1)
    a, b = lay.alloc(0), lay.alloc(0)
    with pytest.raises(P.PxError, match=r"i=\(-1,0\) tap=\(-1,0\)"):
        P.stencil_apply(0, 1.0, lay.patch(0, a), lay.patch(0, b), P.box(-1, 0, 10, 10))


def test_mehrstellen_rhs_vs_oracle():
    n = 128
    rng = np.random.default_rng(4)
    rho = rng.uniform(-1, 1, (n + 2, n + 2))
    lay = P.Layout(P.box(0, 0, n - 1, n - 1), (n, n), 1, P.PX_BC_DIRICHLET_CC, 1)
    r = to_device_ghosted(lay, 0, rho, 1)
    P.fill_ghosts(lay, 0, lay.patch(0, r))
    f = lay.alloc(0)
    P.mehrstellen_rhs(lay.patch(0, r), lay.patch(0, f), lay.local(0).owned)
    torch.cuda.synchronize()
    p = _orc_problem(n, n, 1.0 / n, 0.0, P.PX_BC_DIRICHLET_CC, 1, 0, 0, corr=True)
    assert bits_equal(owned_to_host(lay, 0, f), oracle.rhs(p, rho))


def test_residual_norm_vs_oracle():
    n0, n1 = 300, 200
    h = 1.0 / 300
    phi0, rho = _fields(n0, n1, 1, 9, P.PX_BC_DIRICHLET_CC)
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (n0, n1), 1, P.PX_BC_DIRICHLET_CC, 1)
    a = to_device_ghosted(lay, 0, phi0, 1)
    r = to_device_ghosted(lay, 0, rho, 1)
    P.fill_ghosts(lay, 0, lay.patch(0, a))
    nb = P.norm_buffer(lay.local(0).owned)
    for _ in range(3):  # repeated use of one buffer (scratch restored)
        P.residual_norm(P.relax_params(h, 0.0), lay.patch(0, a), lay.patch(0, r), lay.local(0).owned, nb)
    torch.cuda.synchronize()
    ref = oracle.residual(_orc_problem(n0, n1, h, 0.0, P.PX_BC_DIRICHLET_CC, 0, 0, 0), phi0, rho)
    assert nb[0].item() == ref[0]
    assert abs(nb[1].item() - ref[1]) <= SUM_RTOL * ref[1]


def test_nan_propagates_to_max_norm():
    n = 64
    phi0, rho = _fields(n, n, 1, 1, P.PX_BC_PERIODIC)
    phi0[20, 30] = np.nan
    lay = P.Layout(P.box(0, 0, n - 1, n - 1), (n, n), 1, P.PX_BC_PERIODIC, 1)
    a = to_device_ghosted(lay, 0, phi0, 1)
    r = to_device_ghosted(lay, 0, rho, 1)
    nb = P.norm_buffer(lay.local(0).owned)
    P.residual_norm(P.relax_params(1.0 / n, 0.0), lay.patch(0, a), lay.patch(0, r), lay.local(0).owned, nb)
    assert math.isnan(nb[0].item())


def test_init_field_hash_bitwise():
    n0, n1 = 1000, 300
    lay = P.Layout(P.box(5, -7, 5 + n0 - 1, -7 + n1 - 1), (n0, 100), 1, P.PX_BC_PERIODIC, 3)
    parts = []
    for r in range(3):
        t = lay.alloc(r)
        P.init_field(lay, r, lay.patch(r, t), P.PX_FIELD_HASH, inputs.DEFAULT_SEED)
        parts.append(owned_to_host(lay, r, t))
    assert bits_equal(np.concatenate(parts, 0), inputs.hash_field(n0, n1))


def test_fill_ghosts_matches_oracle_exchange():
    n0, n1, g = 40, 24, 3
    for bc in (P.PX_BC_PERIODIC, P.PX_BC_DIRICHLET_CC):
        rng = np.random.default_rng(bc)
        glob = rng.uniform(-1, 1, (n1 + 2 * g, n0 + 2 * g))
        lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (8, 8), g, bc, 1)
        t = to_device_ghosted(lay, 0, glob, g)
        P.fill_ghosts(lay, 0, lay.patch(0, t))
        ex = oracle.exchange(_orc_problem(n0, n1, 1.0, 0.0, bc, 0, 0, 0, b0=8, b1=8, g=g), glob)
        assert bits_equal(lay.view(0, t, ghosts=True).cpu().numpy(), ex)


def test_error_paths_on_device():
    lay = P.Layout(P.box(0, 0, 63, 63), (64, 64), 1, P.PX_BC_PERIODIC, 1)
    a, b, r = lay.alloc(0), lay.alloc(0), lay.alloc(0)
    pa, pb, pr = lay.patch(0, a), lay.patch(0, b), lay.patch(0, r)
    prm = P.relax_params(1.0 / 64, 1e-5)
    # overlapping input/output
    with pytest.raises(P.PxError, match="overlap"):
        P.relax_step(prm, pa, pa, pr, lay.local(0).owned)
    # different 16-byte phases
    pr2 = P.px_patch(pr.data + 8, pr.box, pr.ld)
    with pytest.raises(P.PxError, match="PX_ERR_ALIGN"):
        P.relax_step(prm, pa, pb, pr2, lay.local(0).owned)
    # wrong layout patch for solve
    bad = P.px_patch(pa.data, P.box(0, 0, 63, 63), pa.ld)
    with pytest.raises(P.PxError, match="PX_ERR_SHAPE"):
        P.solve(lay, None, 0, prm, 2, 1, bad, pb, pr)
    with pytest.raises(P.PxError, match="non-default stream"):
        P.solve(lay, None, 0, prm, 2, 1, pa, pb, pr, use_graph=True, stream=0)


def test_kernels_are_counted():
    before = P.kernel_launch_count()
    test_relax_step_bitwise(P.PX_BC_PERIODIC, 0, (64, 64))
    assert P.kernel_launch_count() > before


# ----------------------------------------------- TMA bulk-copy kernel path
@pytest.mark.parametrize("shape", [(2048, 2048), (2050, 2100), (2560, 1700)])
@pytest.mark.parametrize("st", [P.PX_LAPLACE_5PT, P.PX_MEHRSTELLEN_9PT])
@pytest.mark.parametrize("bc", [P.PX_BC_PERIODIC, P.PX_BC_DIRICHLET_CC])
def test_relax_step_bulk_kernel_bitwise(shape, st, bc):
    """Large enough (>= 4M cells, even width) for the TMA pipeline; ragged
    last strip (2050 -> a 2-column strip) and ragged last row chunk."""
    n0, n1 = shape
    h = 1.0 / 2048
    lam = h * h / 8
    phi0, rho = _fields(n0, n1, 1, n0 + st, bc)
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (n0, n1), 1, bc, 1)
    a = to_device_ghosted(lay, 0, phi0, 1)
    b = lay.alloc(0)
    r = to_device_ghosted(lay, 0, rho, 1)
    P.fill_ghosts(lay, 0, lay.patch(0, a))
    assert P.relax_variant(lay.patch(0, a), lay.patch(0, b), lay.patch(0, r), lay.local(0).owned) == 1
    nb = P.norm_buffer(lay.local(0).owned)
    for _ in range(2):  # the norm buffer is reusable
        P.relax_step(P.relax_params(h, lam, st), lay.patch(0, a), lay.patch(0, b), lay.patch(0, r),
                     lay.local(0).owned, nb)
    torch.cuda.synchronize()
    ref, rn = oracle.solve(_orc_problem(n0, n1, h, lam, bc, st, 1, 1), phi0, rho)
    out = owned_to_host(lay, 0, b)
    assert bits_equal(out, ref[1:-1, 1:-1]), ulp_diff(out, ref[1:-1, 1:-1])
    nrm = nb[:2].cpu().numpy()
    assert nrm[0] == rn[0, 0]
    assert abs(nrm[1] - rn[0, 1]) <= SUM_RTOL * rn[0, 1]


@pytest.mark.parametrize("nranks", [1, 3])
@pytest.mark.parametrize("bc", [P.PX_BC_PERIODIC, P.PX_BC_DIRICHLET_CC, P.PX_BC_FIXED_GHOSTS])
@pytest.mark.parametrize("st", [P.PX_LAPLACE_5PT, P.PX_MEHRSTELLEN_9PT])
def test_solve_bulk_kernel_bitwise(nranks, bc, st):
    """Multi-sweep solves through the TMA kernel with fused ghost images."""
    n0, n1, N, E = 2048, 6144, 5, 2
    h = 1.0 / 2048
    lam = h * h / 8
    phi0, rho = _fields(n0, n1, 1, 31 + bc, bc)
    out, norms, lay = run_gpu_solve(n0, n1, h, lam, bc, st, N, E, phi0, rho, box=(256, 256), nranks=nranks)
    ref, rn = oracle.solve(_orc_problem(n0, n1, h, lam, bc, st, N, E), phi0, rho)
    assert bits_equal(out, ref[1:-1, 1:-1]), ulp_diff(out, ref[1:-1, 1:-1])
    _check_norms(norms, rn)


# ------------------------------------------------- temporal blocking (a7)
@pytest.mark.parametrize("tk", [2, 4])
@pytest.mark.parametrize("bc", [P.PX_BC_PERIODIC, P.PX_BC_FIXED_GHOSTS, P.PX_BC_DIRICHLET_CC])
@pytest.mark.parametrize("st", [P.PX_LAPLACE_5PT, P.PX_MEHRSTELLEN_9PT])
@pytest.mark.parametrize("nranks,hinv", [(1, 1024), (3, 1000)])
def test_solve_temporal_blocking_bitwise(tk, bc, st, nranks, hinv):
    """k sweeps per pass (ghost width 4) == k plain sweeps, bit for bit: ragged
    strips (1000 columns = one full CTA strip + a ragged one), several row chunks, 3 slabs with
    local transport, an odd sweep count (2 or 4-blocks + plain sweeps),
    power-of-two h (fused multiply-add path) and h = 1/1000 (separate ops).
    DIRICHLET_CC: every level re-derives its first ghost column / row by odd
    reflection (corners by the product rule), as the oracle's exchange does
    between sweeps."""
    n0, n1, N, E = 1000, 300, 11, 3
    h = 1.0 / hinv
    lam = h * h / 8 if st == 0 else 3 * h * h / 16
    g = 4
    phi0, rho = _fields(n0, n1, g, 40 + tk + bc + st, bc)
    out, norms, _ = run_gpu_solve(n0, n1, h, lam, bc, st, N, E, phi0, rho, g=g, box=(50, 50),
                                  nranks=nranks, tk=tk)
    ref, rn = oracle.solve(_orc_problem(n0, n1, h, lam, bc, st, N, E, g=g), phi0, rho)
    assert bits_equal(out, ref[g:-g, g:-g]), ulp_diff(out, ref[g:-g, g:-g])
    _check_norms(norms, rn)


@pytest.mark.parametrize("bc,st", [(P.PX_BC_PERIODIC, P.PX_LAPLACE_5PT), (P.PX_BC_DIRICHLET_CC, P.PX_LAPLACE_5PT),
                                   (P.PX_BC_DIRICHLET_CC, P.PX_MEHRSTELLEN_9PT)])
def test_temporal_blocking_large_tall(bc, st):
    """Bulk-sized temporal blocking (many chunks per strip, several strips), k = 4."""
    n0, n1, N, E = 2048, 2560, 8, 1
    h = 1.0 / 2048
    lam = h * h / 8 if st == 0 else 3 * h * h / 16
    g = 4
    phi0, rho = _fields(n0, n1, g, 77, bc)
    out, norms, _ = run_gpu_solve(n0, n1, h, lam, bc, st, N, E, phi0, rho, g=g, box=(256, 256),
                                  tk=4)
    ref, rn = oracle.solve(_orc_problem(n0, n1, h, lam, bc, st, N, E, g=g), phi0, rho)
    assert bits_equal(out, ref[g:-g, g:-g]), ulp_diff(out, ref[g:-g, g:-g])
    _check_norms(norms, rn)


def test_temporal_blocking_unsupported_cases():
    lay = P.Layout(P.box(0, 0, 127, 127), (64, 64), 2, P.PX_BC_DIRICHLET_CC, 1)
    a, b, r = lay.alloc(0), lay.alloc(0), lay.alloc(0)
    with pytest.raises(P.PxError, match="not built"):
        P.solve(lay, None, 0, P.relax_params(1 / 128, 1e-6), 4, 1, lay.patch(0, a), lay.patch(0, b),
                lay.patch(0, r), temporal_k=3)
    with pytest.raises(P.PxError, match="exceeds the ghost width"):
        P.solve(lay, None, 0, P.relax_params(1 / 128, 1e-6), 4, 1, lay.patch(0, a), lay.patch(0, b),
                lay.patch(0, r), temporal_k=4)


@pytest.mark.parametrize("k", [2, 4])
@pytest.mark.parametrize("st", [P.PX_LAPLACE_5PT, P.PX_MEHRSTELLEN_9PT])
def test_relax_block_bitwise(k, st):
    """px_relax_block: k sweeps in one pass == k plain sweeps (periodic ghosts
    filled to depth 4 for φ and ρ); norms = residual of φ_in."""
    n0, n1, g = 1500, 700, 4
    h = 1.0 / 2048
    lam = h * h / 8 if st == 0 else 3 * h * h / 16
    phi0, rho = _fields(n0, n1, g, 91 + k + st, P.PX_BC_PERIODIC)
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (n0, n1), g, P.PX_BC_PERIODIC, 1)
    a = to_device_ghosted(lay, 0, phi0, g)
    b = lay.alloc(0)
    r = to_device_ghosted(lay, 0, rho, g)
    P.fill_ghosts(lay, 0, lay.patch(0, a))
    P.fill_ghosts(lay, 0, lay.patch(0, r))
    nb = P.norm_buffer(lay.local(0).owned)
    P.relax_block(P.relax_params(h, lam, st), k, lay.patch(0, a), lay.patch(0, b), lay.patch(0, r),
                  lay.local(0).owned, nb)
    torch.cuda.synchronize()
    ref, rn = oracle.solve(_orc_problem(n0, n1, h, lam, P.PX_BC_PERIODIC, st, k, k, g=g), phi0, rho)
    out = owned_to_host(lay, 0, b)
    assert bits_equal(out, ref[g:-g, g:-g]), ulp_diff(out, ref[g:-g, g:-g])
    assert nb[0].item() == rn[0, 0]
    assert abs(nb[1].item() - rn[0, 1]) <= SUM_RTOL * rn[0, 1]


@pytest.mark.parametrize("st", [P.PX_LAPLACE_5PT, P.PX_MEHRSTELLEN_9PT])
def test_truncation_ladder_matches_oracle(st):
    """BASELINE config 5 ladder at oracle-feasible sizes: τ_h from the GPU
    residual kernel equals the oracle's (max-norm bit for bit), ratio 4 / 16."""
    taus = []
    for n in (15, 31, 63, 127):
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
            rhs = lay.alloc(0)
            P.mehrstellen_rhs(lay.patch(0, r), lay.patch(0, rhs), lay.local(0).owned)
        nb = P.norm_buffer(lay.local(0).owned)
        P.residual_norm(P.relax_params(h, 0.0, st), lay.patch(0, a), lay.patch(0, rhs), lay.local(0).owned, nb)
        torch.cuda.synchronize()
        ref = oracle.residual(oracle.Problem(n, n, h, 0.0, bc=oracle.BC_FIXED, stencil=st, rhs_correction=(st == 1)),
                              phi, lap)
        assert nb[0].item() == ref[0]
        taus.append(ref[0])
    ratios = [taus[i] / taus[i + 1] for i in range(3)]
    lo, hi = (3.8, 4.2) if st == 0 else (14.0, 17.5)
    assert all(lo < q < hi for q in ratios), ratios


# ------------------------------------------ NCCL path on one GPU (self-exchange)
@pytest.mark.parametrize("tk,graph", [(1, True), (1, False), (4, True)])
def test_nccl_self_exchange_solve(tk, graph, monkeypatch):
    """The multi-GPU code path on one GPU: a one-rank NCCL communicator in
    self-exchange mode sends the periodic ghost rows to itself with the
    library's grouped send/recv (halo plan), on the comm stream, overlapped
    with the interior kernel, captured in a CUDA graph; the norm ring goes
    through ncclAllReduce.  Bit-identical to the oracle."""
    monkeypatch.setenv("PROTOX_NCCL_SELF_EXCHANGE", "1")
    n0, n1, N, E, g = 2048, 2304, 9, 2, max(1, tk)
    h = 1.0 / 2048
    lam = h * h / 8
    phi0, rho = _fields(n0, n1, g, 300 + tk, P.PX_BC_PERIODIC)
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (256, 256), g, P.PX_BC_PERIODIC, 1)
    comm = P.Comm(P.comm_unique_id(), 1, 0, torch.cuda.current_device())
    try:
        a = to_device_ghosted(lay, 0, phi0, g)
        b = lay.alloc(0)
        r = to_device_ghosted(lay, 0, rho, g)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        if tk > 1:
            P.exchange_ghosts(lay, comm, 0, lay.patch(0, r), stream=s)
        before = P.kernel_launch_count()
        res = P.solve(lay, comm, 0, P.relax_params(h, lam), N, E, lay.patch(0, a), lay.patch(0, b),
                      lay.patch(0, r), use_graph=graph, stream=s, temporal_k=tk)
        assert P.kernel_launch_count() - before >= (3 * N if tk == 1 else 2)  # boundary + interior launches
        out = owned_to_host(lay, 0, b if res.in_scratch else a)
    finally:
        comm.close()
    ref, rn = oracle.solve(_orc_problem(n0, n1, h, lam, P.PX_BC_PERIODIC, 0, N, E, g=g), phi0, rho)
    assert bits_equal(out, ref[g:-g, g:-g]), ulp_diff(out, ref[g:-g, g:-g])
    _check_norms(res.norms, rn)


def test_nccl_allreduce_norms_single_rank():
    comm = P.Comm(P.comm_unique_id(), 1, 0, torch.cuda.current_device())
    try:
        m = torch.tensor([1.0, 3.0, float("nan")], dtype=torch.float64, device="cuda")
        s2 = torch.tensor([2.0, 4.0, 5.0], dtype=torch.float64, device="cuda")
        P.comm_allreduce_norms(comm, m, s2, 3)
        torch.cuda.synchronize()
        assert s2.tolist() == [2.0, 4.0, 5.0]
        assert m[:2].tolist() == [1.0, 3.0]
    finally:
        comm.close()


@pytest.mark.parametrize("graph,kind,n0,n1,N2,st", [
    (True, "nccl", 1536, 2304, 8, 0),
    (False, "nccl", 1536, 2304, 5, 1),
    (True, "peer", 640, 300, 3, 0),
    (False, "peer", 2048, 2048, 7, 1),
])
def test_p2p_halo_push_self_exchange(graph, kind, n0, n1, N2, st, monkeypatch):
    """Fused halo push over peer memory, self-exchange mode on one GPU (the
    one-rank periodic layout is its own neighbour): ONE k_bulk launch per
    sweep stores the slab's boundary rows (and x images) into the
    'neighbour's' ghost rows and counts arrivals; its boundary items wait for
    them.  NCCL communicator (px_comm_enable_p2p) or peer-memory one
    (px_comm_create_peer + export/import, no NCCL at all).  Two consecutive
    solves of different lengths (epoch counters); the second starts from
    whichever buffer holds the first's result (registered pair swapped).
    Bit-identical to the oracle's N1+N2 sweeps."""
    monkeypatch.setenv("PROTOX_NCCL_SELF_EXCHANGE", "1")
    N, E = 8, 2
    h = 1.0 / 2048
    lam = h * h / 8
    phi0, rho = _fields(n0, n1, 1, 404, P.PX_BC_PERIODIC)
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (128, 100 if n1 == 300 else 256), 1, P.PX_BC_PERIODIC, 1)
    uid = P.comm_unique_id() if kind == "nccl" else None
    comm = P.Comm(uid, 1, 0, torch.cuda.current_device())
    try:
        a = to_device_ghosted(lay, 0, phi0, 1)
        b = lay.alloc(0)
        r = to_device_ghosted(lay, 0, rho, 1)
        pa, pb, pr = lay.patch(0, a), lay.patch(0, b), lay.patch(0, r)
        if kind == "nccl":
            P.comm_enable_p2p(comm, lay, 0, pa, pb)
        else:
            P.comm_p2p_import(comm, lay, [P.comm_p2p_export(comm, lay, 0, pa, pb)])
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        prm = P.relax_params(h, lam, st)
        r1 = P.solve(lay, comm, 0, prm, N, E, pa, pb, pr, use_graph=graph, stream=s)
        assert P.last_solve_kernels() == "k_bulk"
        assert not r1.in_scratch
        r2 = P.solve(lay, comm, 0, prm, N2, E, pa, pb, pr, use_graph=graph, stream=s)
        out = owned_to_host(lay, 0, b if r2.in_scratch else a)
        if N2 % 2:  # continue from the scratch buffer: the registered pair in swapped order
            r3 = P.solve(lay, comm, 0, prm, 2, E, pb, pa, pr, use_graph=graph, stream=s)
            assert P.last_solve_kernels() == "k_bulk"
            out = owned_to_host(lay, 0, a if r3.in_scratch else b)
    finally:
        comm.close()
    total = N + N2 + (2 if N2 % 2 else 0)
    ref, rn = oracle.solve(_orc_problem(n0, n1, h, lam, P.PX_BC_PERIODIC, st, total, E), phi0, rho)
    assert bits_equal(out, ref[1:-1, 1:-1]), ulp_diff(out, ref[1:-1, 1:-1])
    # norms: first solve's entries are φ^0..φ^6, final φ^8; second continues from φ^8
    _check_norms(r1.norms, rn[: N // E + 1])
    if N2 % 2 == 0:
        _check_norms(r2.norms, rn[N // E:])
    else:
        assert r2.norms[0, 0] == rn[N // E, 0]


def test_p2p_registration_invalidates_cached_graph(monkeypatch):
    """A solve captured as a CUDA graph in NCCL mode, then px_comm_enable_p2p
    on the same communicator and buffers: the next identical solve must run
    the push path (the plan key carries the peer registration), and the
    three solves together stay bit-identical to the oracle."""
    monkeypatch.setenv("PROTOX_NCCL_SELF_EXCHANGE", "1")
    n0, n1, N, E = 1024, 4200, 4, 1  # interior rows x columns > 4M: the TMA kernel
    h = 1.0 / 2048
    lam = h * h / 8
    phi0, rho = _fields(n0, n1, 1, 909, P.PX_BC_PERIODIC)
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (256, 200), 1, P.PX_BC_PERIODIC, 1)
    comm = P.Comm(P.comm_unique_id(), 1, 0, torch.cuda.current_device())
    try:
        a = to_device_ghosted(lay, 0, phi0, 1)
        b = lay.alloc(0)
        r = to_device_ghosted(lay, 0, rho, 1)
        pa, pb, pr = lay.patch(0, a), lay.patch(0, b), lay.patch(0, r)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        prm = P.relax_params(h, lam)
        P.solve(lay, comm, 0, prm, N, E, pa, pb, pr, use_graph=True, stream=s)
        assert P.last_solve_kernels() == "k_stream+k_bulk"
        P.comm_enable_p2p(comm, lay, 0, pa, pb)
        P.solve(lay, comm, 0, prm, N, E, pa, pb, pr, use_graph=True, stream=s)
        assert P.last_solve_kernels() == "k_bulk"
        P.solve(lay, comm, 0, prm, N, E, pa, pb, pr, use_graph=True, stream=s)
        out = owned_to_host(lay, 0, a)
    finally:
        comm.close()
    ref, _ = oracle.solve(_orc_problem(n0, n1, h, lam, P.PX_BC_PERIODIC, 0, 3 * N, E), phi0, rho)
    assert bits_equal(out, ref[1:-1, 1:-1]), ulp_diff(out, ref[1:-1, 1:-1])


@pytest.mark.gpu
def test_temporal_blocking_narrow_kernel_subprocess():
    """The narrow temporal-blocking kernel (2 columns per lane, A/B baseline,
    PROTOX_TB_IMPL=narrow is read once per process) stays bit-identical:
    periodic and FIXED_GHOSTS cases re-run in a child process."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    ids = [f"tests/test_gpu_parity.py::test_solve_temporal_blocking_bitwise[{c}]"
           for c in ("1-1024-0-0-4", "1-1024-1-2-2", "3-1000-0-2-4", "3-1000-1-0-2")]
    ids.append("tests/test_gpu_parity.py::test_temporal_blocking_large_tall[0-0]")
    env = dict(os.environ, PROTOX_TB_IMPL="narrow")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-m", "gpu", *ids],
                       cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_separate_ghost_fill_subprocess():
    """The ghost ring by fill kernels after each sweep instead of fused images
    (the path of single-rank slabs >= 64 M cells; PROTOX_SEP_FILL_CELLS=0,
    read once per process, forces it at test sizes): the single-rank bulk
    solves of every BC and stencil, the ragged multi-box solves and the
    self-exchange push re-run in a child process, bit-identical."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PROTOX_SEP_FILL_CELLS="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-m", "gpu",
                        "tests/test_gpu_parity.py", "-k",
                        "(test_solve_bulk_kernel_bitwise and 1-) or test_solve_ragged_multibox or "
                        "test_p2p_halo_push_self_exchange or test_wider_ghosts_k1"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("case", [(64, 64, P.PX_BC_DIRICHLET_CC, 1, 1), (1024, 1024, P.PX_BC_PERIODIC, 10, 1),
                                  (2048, 1536, P.PX_BC_PERIODIC, 1, 1), (1024, 768, P.PX_BC_DIRICHLET_CC, 4, 4)])
def test_solve_async_bitwise(case):
    """px_solve_async (no host round trip, norms to device memory) runs the
    same solves: φ^N bit-identical to the oracle and the norms as px_solve's,
    for the whole-box, resident, streaming and temporally blocked paths."""
    n0, n1, bc, E, tk = case
    h = 1.0 / max(n0, n1)
    lam = h * h / 8
    phi0, rho = _fields(n0, n1, tk, 31, bc)
    N = 12
    out, norms, _ = run_gpu_solve(n0, n1, h, lam, bc, 0, N, E, phi0, rho, g=tk, tk=tk, async_=True)
    ref, rn = oracle.solve(_orc_problem(n0, n1, h, lam, bc, 0, N, E, g=tk), phi0, rho)
    assert bits_equal(out, ref[tk:-tk, tk:-tk]), ulp_diff(out, ref[tk:-tk, tk:-tk])
    _check_norms(norms, rn)
    out2, norms2, _ = run_gpu_solve(n0, n1, h, lam, bc, 0, N, E, phi0, rho, g=tk, tk=tk)
    assert bits_equal(out, out2) and bits_equal(norms, norms2)


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(1000, 700), (66, 1036), (1024, 1024)])
@pytest.mark.parametrize("bc", [P.PX_BC_PERIODIC, P.PX_BC_DIRICHLET_CC, P.PX_BC_FIXED_GHOSTS])
def test_solve_resident_reg_general_h_lambda(shape, bc):
    """k_resident_reg with h and λ that are not powers of two (its rounded
    multiply-then-add path; power-of-two h, λ take the exact fused
    multiply-adds): bit-identical to the oracle."""
    n0, n1 = shape
    h = 1.0 / (n1 - 1)
    lam = 0.9 * h * h / 8
    phi0, rho = _fields(n0, n1, 1, 23, bc)
    for N, E in ((11, 3), (6, 0)):
        out, norms, _ = run_gpu_solve(n0, n1, h, lam, bc, 0, N, E, phi0, rho)
        ref, rn = oracle.solve(_orc_problem(n0, n1, h, lam, bc, 0, N, E), phi0, rho)
        assert bits_equal(out, ref[1:-1, 1:-1]), ulp_diff(out, ref[1:-1, 1:-1])
        _check_norms(norms, rn)


@pytest.mark.gpu
@pytest.mark.parametrize("var", [("PROTOX_RESIDENT_K", "2"), ("PROTOX_RESIDENT_K", "3"),
                                 ("PROTOX_RESIDENT_REG", "0"), ("PROTOX_RESIDENT_REG", "2"),
                                 ("PROTOX_WRAP", "1")])
def test_resident_temporal_blocking_variant_subprocess(var):
    """The resident-solve variants (read once per process) stay bit-identical:
    the shared-memory temporally blocked kernel (PROTOX_RESIDENT_K=2,3), the
    shared-memory row walk (PROTOX_RESIDENT_REG=0) and the register kernel with
    two sweeps per mailbox hop (PROTOX_RESIDENT_REG=2); the resident-path
    tests re-run in child processes."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for k in (var[1],):
        env = dict(os.environ, **{var[0]: k})
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-m", "gpu",
                            "tests/test_gpu_parity.py", "-k",
                            "resident_shapes or config2_full or resident_reg_general or solve_async or "
                            "solve_bulk_kernel"],
                           cwd=root, env=env, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, (k, r.stdout[-3000:] + r.stderr[-2000:])


@pytest.mark.gpu
def test_unfused_proto_sequence_bitwise():
    """Proto's unfused sequence (px_stencil_apply -> px_pointwise_update, then
    px_residual_norm of the updated iterate) equals the oracle bit
    for bit -- the baseline of the fused-vs-unfused measurement."""
    n0, n1, N = 300, 170, 5
    h = 1.0 / 256
    lam = h * h / 8
    phi0, rho = _fields(n0, n1, 1, 5, P.PX_BC_PERIODIC)
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (n0, n1), 1, P.PX_BC_PERIODIC, 1)
    li = lay.local(0)
    a, t, r = to_device_ghosted(lay, 0, phi0, 1), lay.alloc(0), to_device_ghosted(lay, 0, rho, 1)
    pa, pt, pr = lay.patch(0, a), lay.patch(0, t), lay.patch(0, r)
    nb = P.norm_buffer(li.owned)
    got = []
    for _ in range(N):
        P.fill_ghosts(lay, 0, pa)
        P.stencil_apply(0, 1.0 / (h * h), pa, pt, li.owned)
        P.pointwise_update(pa, pt, pr, lam, li.owned)
        P.fill_ghosts(lay, 0, pa)
        P.residual_norm(P.relax_params(h, lam), pa, pr, li.owned, nb)
        got.append(nb[:2].cpu().numpy())
    ref, rn = oracle.solve(_orc_problem(n0, n1, h, lam, P.PX_BC_PERIODIC, 0, N, 1), phi0, rho)
    assert bits_equal(owned_to_host(lay, 0, a), ref[1:-1, 1:-1])
    _check_norms(np.array(got), rn[1:])
