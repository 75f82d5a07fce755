"""Full-size parity at BASELINE sizes, in the launch configuration bench.py
times (px_solve, 100 sweeps, norms every sweep, CUDA graph, 256² boxes).

The oracle cannot run 16384² x 100 sweeps in test time, so sampled cells are
recomputed by the oracle one by one: after N sweeps a cell depends only on
the initial data within Chebyshev distance N, so an oracle run on the
(2N+1)² window around it (window border = FIXED ghosts, which cannot reach
the centre in N sweeps) gives the exact value -- compared bit for bit.
The recorded norms are checked against properties that hold at any size:
r(φ⁰) = −ρ for φ⁰ = 0, and the closed-form trajectory of an eigenmode."""
import math

import numpy as np
import pytest

import oracle
from paper_2307_07931_b200 import inputs
from paper_2307_07931_b200 import protox as P

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _window_value(rho_window, n_sweeps, h, lam, st=0, corr=False):
    """Centre value after N sweeps of φ⁰ = 0 on a ghosted window of ρ."""
    m = rho_window.shape[0] - 2
    p = oracle.Problem(m, m, h, lam, bc=oracle.BC_FIXED, stencil=st, rhs_correction=corr,
                       nsweeps=n_sweeps, norm_every=-1)
    out, _ = oracle.solve(p, np.zeros_like(rho_window), rho_window)
    c = m // 2 + 1
    return out[c, c]


def _samples(n, k, seed):
    rng = np.random.default_rng(seed)
    pts = [(0, 0), (n - 1, n - 1), (0, n - 1), (n - 1, 0), (255, 256), (n // 2, 1)]
    pts += [tuple(int(v) for v in rng.integers(0, n, 2)) for _ in range(k)]
    return pts


def test_config3_fullsize_sampled_bitwise():
    n, N = 16384, 100
    h = 1.0 / n
    lam = h * h / 8
    lay = P.Layout(P.box(0, 0, n - 1, n - 1), (256, 256), 1, P.PX_BC_PERIODIC, 1)
    phi, scr, rho = lay.alloc(0), lay.alloc(0), lay.alloc(0)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())  # zero-fills ran on the current stream
    P.init_field(lay, 0, lay.patch(0, rho), P.PX_FIELD_HASH, inputs.DEFAULT_SEED, stream=s)
    s.synchronize()
    pa, pb, pr = lay.patch(0, phi), lay.patch(0, scr), lay.patch(0, rho)
    assert P.relax_variant(pa, pb, pr, lay.local(0).owned) == 1  # the TMA kernel the bench times
    res = P.solve(lay, None, 0, P.relax_params(h, lam), N, 1, pa, pb, pr, use_graph=True, stream=s)
    out = lay.view(0, scr if res.in_scratch else phi)
    R = N
    for (x, y) in _samples(n, 10, 3):
        win = inputs.hash_window(n, n, x - R - 1, y - R - 1, 2 * R + 3, 2 * R + 3)
        want = _window_value(win, N, h, lam)
        got = out[y, x].item()
        assert np.float64(got).view(np.uint64) == np.float64(want).view(np.uint64), (x, y, got, want)
    # r(φ⁰) = −ρ: max|ρ| exactly, Σρ² to 1e-12
    rv = lay.view(0, rho)
    assert res.norms.shape == (N + 1, 2)
    assert res.norms[0, 0] == torch.max(torch.abs(rv)).item()
    ss = torch.sum(rv * rv).item()
    assert abs(res.norms[0, 1] - ss) <= 1e-12 * ss


def test_config3_fullsize_sine_closed_form_norms():
    """Periodic ρ = sin 2πx sin 2πy (an eigenmode, μ = −(8/h²)sin²(πh)):
    ‖r(φᵐ)‖∞ = gᵐ·max|ρ| with g = cos²(π/n)."""
    n, N = 16384, 100
    h = 1.0 / n
    lam = h * h / 8
    lay = P.Layout(P.box(0, 0, n - 1, n - 1), (256, 256), 1, P.PX_BC_PERIODIC, 1)
    phi, scr, rho = lay.alloc(0), lay.alloc(0), lay.alloc(0)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())  # zero-fills ran on the current stream
    P.init_field(lay, 0, lay.patch(0, rho), P.PX_FIELD_SINE, 0, 2, 2, stream=s)
    res = P.solve(lay, None, 0, P.relax_params(h, lam), N, 1, lay.patch(0, phi), lay.patch(0, scr),
                  lay.patch(0, rho), use_graph=True, stream=s)
    g = math.cos(math.pi / n) ** 2
    rmax = torch.max(torch.abs(lay.view(0, rho))).item()
    m = np.arange(N + 1)
    np.testing.assert_allclose(res.norms[:, 0], g**m * rmax, rtol=1e-12)


def test_config5_fullsize_mehrstellen_sampled_bitwise():
    """BASELINE config 5: 8192² Dirichlet-CC, Mehrstellen with the corrected
    right-hand side computed on the device; interior samples bit-identical,
    norms on the closed-form trajectory of the sine mode."""
    n, N = 8192, 100
    h = 1.0 / n
    lam = h * h / 8
    lay = P.Layout(P.box(0, 0, n - 1, n - 1), (256, 256), 1, P.PX_BC_DIRICHLET_CC, 1)
    phi, scr, rho, f = lay.alloc(0), lay.alloc(0), lay.alloc(0), lay.alloc(0)
    rho_h = inputs.sine_field(n, n)
    lay.view(0, rho).copy_(torch.from_numpy(rho_h))
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())  # zero-fills ran on the current stream
    P.fill_ghosts(lay, 0, lay.patch(0, rho), stream=s)
    P.mehrstellen_rhs(lay.patch(0, rho), lay.patch(0, f), lay.local(0).owned, stream=s)
    res = P.solve(lay, None, 0, P.relax_params(h, lam, P.PX_MEHRSTELLEN_9PT), N, 1, lay.patch(0, phi),
                  lay.patch(0, scr), lay.patch(0, f), use_graph=True, stream=s)
    out = lay.view(0, scr if res.in_scratch else phi)
    R = N
    xc = inputs.cell_centres(n)
    for (x, y) in [(R + 2, R + 2), (n // 2, n // 3), (n - R - 3, 4000), (1234, n - R - 3)]:
        xs, ys = xc[x - R - 1:x + R + 2], xc[y - R - 1:y + R + 2]
        win = np.outer(np.sin(np.pi * ys), np.sin(np.pi * xs))
        # the window's ghost ring carries the true ρ (used by the RHS correction)
        want = _window_value(win, N, h, lam, st=1, corr=True)
        got = out[y, x].item()
        assert np.float64(got).view(np.uint64) == np.float64(want).view(np.uint64), (x, y, got, want)
    a = -4 * math.sin(math.pi * h / 2) ** 2
    mu9 = (2 * a + a * a / 6) / (h * h)
    g = 1 + lam * mu9
    fmax = torch.max(torch.abs(lay.view(0, f))).item()
    np.testing.assert_allclose(res.norms[:, 0], g ** np.arange(N + 1) * fmax, rtol=1e-12)


def test_config4_fullsize_temporal_blocking_sampled_bitwise():
    """BASELINE config 4 in the bench's launch configuration: 32768², 256²
    boxes, ghost width 4, temporal blocking k = 4, norm every exchange,
    CUDA graph; sampled cells bit-identical to the oracle's window runs."""
    n, N, E, K = 32768, 100, 4, 4
    h = 1.0 / n
    lam = h * h / 8
    lay = P.Layout(P.box(0, 0, n - 1, n - 1), (256, 256), K, P.PX_BC_PERIODIC, 1)
    phi, scr, rho = lay.alloc(0), lay.alloc(0), lay.alloc(0)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    P.init_field(lay, 0, lay.patch(0, rho), P.PX_FIELD_HASH, inputs.DEFAULT_SEED, stream=s)
    P.fill_ghosts(lay, 0, lay.patch(0, rho), stream=s)
    res = P.solve(lay, None, 0, P.relax_params(h, lam), N, E, lay.patch(0, phi), lay.patch(0, scr),
                  lay.patch(0, rho), use_graph=True, stream=s, temporal_k=K)
    out = lay.view(0, scr if res.in_scratch else phi)
    R = N
    for (x, y) in _samples(n, 6, 11):
        win = inputs.hash_window(n, n, x - R - 1, y - R - 1, 2 * R + 3, 2 * R + 3)
        want = _window_value(win, N, h, lam)
        got = out[y, x].item()
        assert np.float64(got).view(np.uint64) == np.float64(want).view(np.uint64), (x, y, got, want)
    rv = lay.view(0, rho)
    assert res.norms.shape == (N // E + 1, 2)
    assert res.norms[0, 0] == torch.max(torch.abs(rv)).item()
    ss = torch.sum(rv * rv).item()
    assert abs(res.norms[0, 1] - ss) <= 1e-12 * ss
    del phi, scr, rho
    torch.cuda.empty_cache()


@pytest.mark.parametrize("k", [1, 4])
def test_beyond_2_31_elements_sampled_bitwise(k):
    """Maximum-size edge case: a 65536 x 33000 periodic domain is 2.16e9 cells
    (> 2^31; 17.3 GB per array with its ghosts and padding, 52 GB in all), so
    every element offset of the last ~350 rows overflows 32 bits.  k = 1 (the
    TMA sweep kernel) and k = 4 (temporal blocking, ghost 4), 4 sweeps, norms
    every sweep / pass: cells sampled in the first and last rows (the largest
    offsets) bit-identical to oracle window runs; the first recorded max-norm
    equals max|ρ| (r(φ⁰) = −ρ for φ⁰ = 0) computed by torch over the whole
    field."""
    n0, n1, N = 65536, 33000, 4
    h = 1.0 / n0
    lam = h * h / 8
    g = 4 if k == 4 else 1
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (256, 200), g, P.PX_BC_PERIODIC, 1)
    li = lay.local(0)
    assert li.alloc_elems > 2 ** 31
    phi, scr, rho = lay.alloc(0), lay.alloc(0), lay.alloc(0)
    try:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        P.init_field(lay, 0, lay.patch(0, rho), P.PX_FIELD_HASH, inputs.DEFAULT_SEED, stream=s)
        P.fill_ghosts(lay, 0, lay.patch(0, rho), stream=s)
        res = P.solve(lay, None, 0, P.relax_params(h, lam), N, k, lay.patch(0, phi), lay.patch(0, scr),
                      lay.patch(0, rho), use_graph=True, stream=s, temporal_k=k)
        assert ("k_tbw" if k == 4 else "k_bulk") in P.last_solve_kernels()
        out = lay.view(0, scr if res.in_scratch else phi)
        R = N
        rng = np.random.default_rng(31)
        pts = [(0, 0), (n0 - 1, n1 - 1), (0, n1 - 1), (n0 - 1, n1 - 2), (12345, n1 - 1), (n0 // 2, n1 - 3)]
        pts += [(int(rng.integers(0, n0)), int(rng.integers(n1 - 400, n1))) for _ in range(6)]
        for (x, y) in pts:
            win = inputs.hash_window(n0, n1, x - R - 1, y - R - 1, 2 * R + 3, 2 * R + 3)
            want = _window_value(win, N, h, lam)
            got = out[y, x].item()
            assert np.float64(got).view(np.uint64) == np.float64(want).view(np.uint64), (x, y, got, want)
        assert res.norms[0, 0] == torch.max(torch.abs(lay.view(0, rho))).item()
    finally:
        del phi, scr, rho
        P.release_cached()
        torch.cuda.empty_cache()
