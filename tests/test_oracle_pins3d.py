"""Pins of the 3D CPU oracle (oracle/protox_oracle3d.cpp, SURVEY §8(f) NEXT
rank 3) to what the paper and the mathematics fix -- none re-types the
oracle's tap loop:

* the 7-point operator is exact on integer quadratics and kills constants and
  linears (the 3D form of Eq.1 / PAPER.md:27-29, 133);
* its eigenvalues on periodic and cell-centred Dirichlet modes are the
  closed-form sums of the 1D ones;
* a dense brute force: the operator assembled as a Kronecker sum of 1D
  second-difference matrices (independent construction), iterated densely;
* the N-sweep result for arbitrary φ⁰, ρ equals the spectral closed form
  φ̂ᴺ = gᴺ φ̂⁰ + (1 − gᴺ)/μ · ρ̂ (FFT periodic, DST-II Dirichlet);
* the sine mode trajectory and the manufactured-solution error ratio 4 as h
  halves (second order, BJ.ns) with λ = h²/(4D), D = 3;
* exchange == numpy wrap / odd-reflection padding; box decomposition
  invariance (bitwise); NaN propagation.
"""
import math

import numpy as np
import pytest

import oracle
from oracle import BC_DIRICHLET_CC, BC_FIXED, BC_PERIODIC

sfft = pytest.importorskip("scipy.fft")


def _rand(p, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, p.gshape), rng.uniform(-1, 1, p.gshape)


def _interior(p, a):
    g = p.ghost
    return a[g:g + p.n[2], g:g + p.n[1], g:g + p.n[0]]


def _centres(n, h):
    return (np.arange(n) + 0.5) * h


# ------------------------------------------------------------ exactness
def test_laplacian_exact_on_integer_quadratics():
    n = (6, 5, 7)
    p = oracle.Problem3(n, 1.0, 0.0, bc=BC_FIXED, ghost=1)
    g = 1
    z, y, x = np.meshgrid(np.arange(-g, n[2] + g), np.arange(-g, n[1] + g), np.arange(-g, n[0] + g),
                          indexing="ij")
    x, y, z = x.astype(float), y.astype(float), z.astype(float)
    for (a, b, c, d, e, f) in [(1, 0, 0, 0, 0, 0), (0, 2, 0, 0, 0, 0), (0, 0, -3, 0, 0, 0),
                               (2, -1, 5, 3, -7, 4)]:
        phi = a * x * x + b * y * y + c * z * z + d * x * y + e * y * z + f * z * x + 3 * x - 2 * y + z + 11
        lap = oracle.apply_laplacian3(p, phi)
        assert np.all(lap == 2 * a + 2 * b + 2 * c)
    for phi in (np.full(p.gshape, 7.25), 2 * x - 3 * y + 5 * z + 1):
        assert np.all(oracle.apply_laplacian3(p, phi) == 0.0)


# ------------------------------------------------------------ spectra
@pytest.mark.parametrize("k", [(1, 0, 0), (1, 2, 3), (3, 1, 2)])
def test_periodic_eigenvalues(k):
    n = (8, 12, 16)
    h = 1.0 / 8
    p = oracle.Problem3(n, h, 0.0, bc=BC_PERIODIC)
    cells = [np.arange(m) for m in n]
    Z, Y, X = np.meshgrid(*cells[::-1], indexing="ij")
    v = np.cos(2 * np.pi * (k[0] * X / n[0] + k[1] * Y / n[1] + k[2] * Z / n[2]))
    mu = -(4 / h**2) * sum(math.sin(math.pi * k[d] / n[d]) ** 2 for d in range(3))
    lap = oracle.apply_laplacian3(p, oracle.ghosted3(p, v))
    np.testing.assert_allclose(lap, mu * v, rtol=0, atol=1e-11 * abs(mu))


@pytest.mark.parametrize("k", [(1, 1, 1), (2, 1, 3), (4, 3, 1)])
def test_dirichlet_cc_eigenvalues(k):
    n = (8, 6, 10)
    h = 1.0 / 8
    p = oracle.Problem3(n, h, 0.0, bc=BC_DIRICHLET_CC)
    xs = [np.sin(k[d] * np.pi * (np.arange(n[d]) + 0.5) / n[d]) for d in range(3)]
    v = xs[2][:, None, None] * xs[1][None, :, None] * xs[0][None, None, :]
    mu = -(4 / h**2) * sum(math.sin(k[d] * math.pi / (2 * n[d])) ** 2 for d in range(3))
    lap = oracle.apply_laplacian3(p, oracle.ghosted3(p, v))
    np.testing.assert_allclose(lap, mu * v, rtol=0, atol=1e-11 * abs(mu))


# ------------------------------------------------------------ dense brute force
def _t1(m, bc):
    """1D undivided second difference on m cells with the boundary rule folded in."""
    T = -2 * np.eye(m) + np.eye(m, k=1) + np.eye(m, k=-1)
    if bc == BC_PERIODIC:
        T[0, -1] += 1
        T[-1, 0] += 1
    elif bc == BC_DIRICHLET_CC:  # ghost = -mirror
        T[0, 0] -= 1
        T[-1, -1] -= 1
    return T


def _dense_op(n, h, bc):
    I = [np.eye(m) for m in n]
    A = (np.kron(I[2], np.kron(I[1], _t1(n[0], bc))) + np.kron(I[2], np.kron(_t1(n[1], bc), I[0]))
         + np.kron(_t1(n[2], bc), np.kron(I[1], I[0])))
    return A / (h * h)


@pytest.mark.parametrize("bc", [BC_PERIODIC, BC_DIRICHLET_CC])
@pytest.mark.parametrize("box", [None, (2, 2, 3)])
def test_dense_bruteforce_trajectory_and_norms(bc, box):
    n = (4, 4, 6)
    h = 1.0 / 4
    lam = h * h / 12
    N = 7
    p = oracle.Problem3(n, h, lam, b=box, bc=bc, nsweeps=N, norm_every=2)
    phi0, rho = _rand(p, 5 + bc)
    out, norms = oracle.solve3(p, phi0, rho)
    A = _dense_op(n, h, bc)
    x = _interior(p, phi0).reshape(-1).copy()
    f = _interior(p, rho).reshape(-1)
    want = []
    for it in range(N):
        if it % 2 == 0:
            r = A @ x - f
            want.append((np.max(np.abs(r)), np.sum(r * r)))
        x = x + lam * (A @ x - f)
    r = A @ x - f
    want.append((np.max(np.abs(r)), np.sum(r * r)))
    scale = np.max(np.abs(x))
    np.testing.assert_allclose(_interior(p, out).reshape(-1), x, rtol=0, atol=1e-13 * scale)
    np.testing.assert_allclose(norms, np.array(want), rtol=1e-12)


# ------------------------------------------------------------ spectral closed form
def _spectral(phi0, rho, mu, lam, N):
    g = 1 + lam * mu
    with np.errstate(divide="ignore"):
        gN = np.sign(g) ** N * np.exp(N * np.log(np.abs(g)))
    with np.errstate(divide="ignore", invalid="ignore"):
        out = gN * phi0 + np.where(mu != 0, (1 - gN) / np.where(mu != 0, mu, 1), 0.0) * rho
    zero = mu == 0
    out[zero] = phi0[zero] - N * lam * rho[zero]
    return out


@pytest.mark.parametrize("bc", [BC_PERIODIC, BC_DIRICHLET_CC])
def test_n_sweeps_equal_spectral_closed_form(bc):
    n = (16, 8, 12)
    h = 1.0 / 16
    lam = h * h / 12
    N = 60
    p = oracle.Problem3(n, h, lam, bc=bc, nsweeps=N, norm_every=-1)
    phi0, rho = _rand(p, 11 + bc)
    out, _ = oracle.solve3(p, phi0, rho)
    a0, r0 = _interior(p, phi0), _interior(p, rho)
    if bc == BC_PERIODIC:
        ks = [np.fft.fftfreq(m) * m for m in n]
        s = [np.sin(np.pi * k / m) ** 2 for k, m in zip(ks, n)]
        mu = -(4 / h**2) * (s[2][:, None, None] + s[1][None, :, None] + s[0][None, None, :])
        want = np.real(np.fft.ifftn(_spectral(np.fft.fftn(a0), np.fft.fftn(r0), mu, lam, N)))
    else:
        s = [np.sin(np.pi * np.arange(1, m + 1) / (2 * m)) ** 2 for m in n]
        mu = -(4 / h**2) * (s[2][:, None, None] + s[1][None, :, None] + s[0][None, None, :])
        want = sfft.idstn(_spectral(sfft.dstn(a0, type=2), sfft.dstn(r0, type=2), mu, lam, N), type=2)
    got = _interior(p, out)
    assert np.max(np.abs(got - want)) <= 1e-13 * np.max(np.abs(want))


# ------------------------------------------------------------ sine mode, order
def _sine_mode(n, h):
    xs = np.sin(np.pi * _centres(n, h))
    return xs[:, None, None] * xs[None, :, None] * xs[None, None, :]


def test_sine_mode_trajectory_closed_form():
    n = 8
    h = 1.0 / n
    lam = h * h / 12  # λ = h²/(4D), D = 3
    N = 40
    p = oracle.Problem3((n, n, n), h, lam, bc=BC_DIRICHLET_CC, nsweeps=N, norm_every=1)
    rho = _sine_mode(n, h)
    out, norms = oracle.solve3(p, np.zeros(p.gshape), oracle.ghosted3(p, rho))
    mu = -(12 / h**2) * math.sin(math.pi * h / 2) ** 2
    g = 1 + lam * mu  # = cos²(πh/2)
    assert abs(g - math.cos(math.pi * h / 2) ** 2) < 1e-15
    want = (1 - g**N) / mu * rho
    np.testing.assert_allclose(_interior(p, out), want, rtol=0, atol=1e-15)
    # r(φ^k) = −g^k ρ: max-norm g^k max|ρ|
    gm = np.max(np.abs(rho))
    ks = np.arange(N + 1)
    np.testing.assert_allclose(norms[:, 0], g**ks * gm, rtol=1e-12)


def test_manufactured_solution_second_order():
    """Δφ = sin πx sin πy sin πz, homogeneous Dirichlet: φ* = −ρ/(3π²).  The
    oracle iterated to convergence reaches the discrete solution ρ/μ (closed
    form), and its error against φ* falls towards a factor 4 per halving of h
    (second order, BJ.ns; pre-asymptotic at these tiny grids: 3.42, 3.85)."""
    errs, want = [], []
    for n, N in [(4, 400), (8, 1500), (16, 5500)]:
        h = 1.0 / n
        lam = h * h / 12
        p = oracle.Problem3((n, n, n), h, lam, b=(n, n, min(n, 8)), bc=BC_DIRICHLET_CC, nsweeps=N,
                            norm_every=-1)
        rho = _sine_mode(n, h)
        out, _ = oracle.solve3(p, np.zeros(p.gshape), oracle.ghosted3(p, rho))
        errs.append(np.max(np.abs(_interior(p, out) + rho / (3 * np.pi**2))))
        mu = -(12 / h**2) * math.sin(math.pi * h / 2) ** 2
        want.append(np.max(np.abs(rho)) * abs(1 / mu + 1 / (3 * np.pi**2)))
    np.testing.assert_allclose(errs, want, rtol=1e-9)
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 3.3 < r1 < r2 < 4.05, (errs, r1, r2)


# ------------------------------------------------------------ exchange / invariance
def test_exchange_equals_numpy_padding():
    n = (5, 4, 3)
    rng = np.random.default_rng(2)
    a = rng.uniform(-1, 1, (n[2], n[1], n[0]))
    for g in (1, 2):
        p = oracle.Problem3(n, 1.0, 0.0, ghost=g, bc=BC_PERIODIC)
        got = oracle.exchange3(p, oracle.ghosted3(p, a, np.nan))
        assert np.array_equal(got, np.pad(a, g, mode="wrap"))
        p = oracle.Problem3(n, 1.0, 0.0, ghost=g, bc=BC_DIRICHLET_CC)
        got = oracle.exchange3(p, oracle.ghosted3(p, a, np.nan))
        sym = np.pad(a, g, mode="symmetric")
        outside = sum(((np.arange(-g, m + g) < 0) | (np.arange(-g, m + g) >= m)).astype(int)[sh]
                      for m, sh in zip(n[::-1], [(slice(None), None, None), (None, slice(None), None),
                                                 (None, None, slice(None))]))
        assert np.array_equal(got, sym * (-1.0) ** outside)
        p = oracle.Problem3(n, 1.0, 0.0, ghost=g, bc=BC_FIXED)
        ring = oracle.ghosted3(p, a, 3.5)
        assert np.array_equal(oracle.exchange3(p, ring), ring)


@pytest.mark.parametrize("bc", [BC_PERIODIC, BC_DIRICHLET_CC, BC_FIXED])
def test_box_decomposition_invariance(bc):
    n = (8, 6, 9)
    h = 1.0 / 8
    base = dict(h=h, lam=h * h / 12, bc=bc, nsweeps=9, norm_every=3)
    p1 = oracle.Problem3(n, **base)
    p2 = oracle.Problem3(n, b=(4, 3, 3), **base)
    phi0, rho = _rand(p1, 21 + bc)
    o1, n1 = oracle.solve3(p1, phi0, rho)
    o2, n2 = oracle.solve3(p2, phi0, rho)
    assert np.array_equal(o1, o2)
    assert np.array_equal(n1[:, 0], n2[:, 0])
    np.testing.assert_allclose(n1[:, 1], n2[:, 1], rtol=1e-13)


def test_nan_propagates():
    n = (4, 4, 4)
    p = oracle.Problem3(n, 0.25, 0.25**2 / 12, nsweeps=1, norm_every=1)
    phi0, rho = _rand(p, 3)
    phi0[2, 2, 2] = np.nan
    _, norms = oracle.solve3(p, phi0, rho)
    assert math.isnan(norms[0, 0]) and math.isnan(norms[-1, 0])


def test_infinite_residual_sum_is_inf():
    """Reading R6: Σr² is the plain sum of squares -- +inf with one infinite
    residual (not the NaN an inf - inf compensation term would give)."""
    n = (4, 4, 4)
    p = oracle.Problem3(n, 0.25, 0.25**2 / 12, nsweeps=0, norm_every=1)
    phi0, rho = _rand(p, 3)
    rho[2, 2, 2] = np.inf
    _, norms = oracle.solve3(p, phi0, rho)
    assert norms[0, 0] == np.inf and norms[0, 1] == np.inf


# ------------------------------------------------------- 27-point Mehrstellen (R-3D4)
def test_mehrstellen27_exact_on_integer_quadratics():
    n = (6, 5, 7)
    p = oracle.Problem3(n, 1.0, 0.0, bc=BC_FIXED, ghost=1, stencil=1)
    z, y, x = np.meshgrid(np.arange(-1, n[2] + 1), np.arange(-1, n[1] + 1), np.arange(-1, n[0] + 1),
                          indexing="ij")
    x, y, z = x.astype(float), y.astype(float), z.astype(float)
    for (a, b, c, d, e, f) in [(1, 0, 0, 0, 0, 0), (0, 0, 1, 0, 0, 0), (2, -1, 5, 3, -7, 4), (0, 0, 0, 1, 1, 1)]:
        phi = a * x * x + b * y * y + c * z * z + d * x * y + e * y * z + f * z * x + 3 * x - 2 * y + z + 11
        lap = oracle.apply_laplacian3(p, phi)  # = fl(1/30) * (60 (a+b+c)) exactly up to that one rounding
        np.testing.assert_allclose(lap, 2 * (a + b + c), rtol=2e-16, atol=0)
    assert np.all(oracle.apply_laplacian3(p, np.full(p.gshape, 3.5)) == 0.0)


def _mu27(c, h):
    """Eigenvalue of the 27-point operator on a separable cosine/sine mode with
    per-dimension factors c_d = cos(θ_d)."""
    cx, cy, cz = c
    return (-128 + 28 * (cx + cy + cz) + 12 * (cx * cy + cy * cz + cz * cx) + 8 * cx * cy * cz) / (30 * h * h)


@pytest.mark.parametrize("k", [(1, 0, 0), (1, 2, 3), (3, 1, 2)])
def test_mehrstellen27_periodic_eigenvalues(k):
    n = (8, 12, 16)
    h = 1.0 / 8
    p = oracle.Problem3(n, h, 0.0, bc=BC_PERIODIC, stencil=1)
    Z, Y, X = np.meshgrid(*[np.arange(m) for m in n[::-1]], indexing="ij")
    v = np.cos(2 * np.pi * (k[0] * X / n[0] + k[1] * Y / n[1] + k[2] * Z / n[2]))
    mu = _mu27([math.cos(2 * math.pi * k[d] / n[d]) for d in range(3)], h)
    lap = oracle.apply_laplacian3(p, oracle.ghosted3(p, v))
    np.testing.assert_allclose(lap, mu * v, rtol=0, atol=1e-11 * abs(mu))


@pytest.mark.parametrize("k", [(1, 1, 1), (2, 1, 3)])
def test_mehrstellen27_dirichlet_eigenvalues(k):
    n = (8, 6, 10)
    h = 1.0 / 8
    p = oracle.Problem3(n, h, 0.0, bc=BC_DIRICHLET_CC, stencil=1)
    xs = [np.sin(k[d] * np.pi * (np.arange(n[d]) + 0.5) / n[d]) for d in range(3)]
    v = xs[2][:, None, None] * xs[1][None, :, None] * xs[0][None, None, :]
    mu = _mu27([math.cos(k[d] * math.pi / n[d]) for d in range(3)], h)
    lap = oracle.apply_laplacian3(p, oracle.ghosted3(p, v))
    np.testing.assert_allclose(lap, mu * v, rtol=0, atol=1e-11 * abs(mu))


def _shift(m, s, bc):
    """1D shift (u_{i+s}) with the boundary rule folded in (s = -1, 0, 1)."""
    if s == 0:
        return np.eye(m)
    S = np.eye(m, k=s)
    if bc == BC_PERIODIC:
        S[(0 if s < 0 else m - 1), (m - 1 if s < 0 else 0)] = 1.0
    elif bc == BC_DIRICHLET_CC:
        i = 0 if s < 0 else m - 1
        S[i, i] = -1.0
    return S


def _dense27(n, h, bc):
    w = {0: -128.0, 1: 14.0, 2: 3.0, 3: 1.0}
    A = np.zeros((n[0] * n[1] * n[2],) * 2)
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                A += w[abs(dx) + abs(dy) + abs(dz)] * np.kron(_shift(n[2], dz, bc),
                                                            np.kron(_shift(n[1], dy, bc), _shift(n[0], dx, bc)))
    return A / (30 * h * h)


@pytest.mark.parametrize("bc", [BC_PERIODIC, BC_DIRICHLET_CC])
def test_mehrstellen27_dense_bruteforce(bc):
    n = (4, 4, 5)
    h = 1.0 / 4
    lam = h * h / 12
    N = 6
    p = oracle.Problem3(n, h, lam, b=(2, 2, 5), bc=bc, nsweeps=N, norm_every=1, stencil=1)
    phi0, rho = _rand(p, 31 + bc)
    out, norms = oracle.solve3(p, phi0, rho)
    A = _dense27(n, h, bc)
    x = _interior(p, phi0).reshape(-1).copy()
    f = _interior(p, rho).reshape(-1)
    want = []
    for _ in range(N):
        r = A @ x - f
        want.append((np.max(np.abs(r)), np.sum(r * r)))
        x = x + lam * r
    r = A @ x - f
    want.append((np.max(np.abs(r)), np.sum(r * r)))
    np.testing.assert_allclose(_interior(p, out).reshape(-1), x, rtol=0, atol=1e-13 * np.max(np.abs(x)))
    np.testing.assert_allclose(norms, np.array(want), rtol=1e-12)


def test_mehrstellen27_rhs_correction_is_rho_plus_s7_over_12():
    n = (6, 5, 4)
    p = oracle.Problem3(n, 0.1, 0.0, bc=BC_PERIODIC, stencil=1, rhs_correction=True)
    rng = np.random.default_rng(8)
    rho = rng.uniform(-1, 1, (n[2], n[1], n[0]))
    pad = np.pad(rho, 1, mode="wrap")
    s7 = (pad[1:-1, 1:-1, :-2] + pad[1:-1, 1:-1, 2:] + pad[1:-1, :-2, 1:-1] + pad[1:-1, 2:, 1:-1]
          + pad[:-2, 1:-1, 1:-1] + pad[2:, 1:-1, 1:-1] - 6 * rho)
    np.testing.assert_allclose(oracle.rhs3(p, oracle.ghosted3(p, rho)), rho + s7 / 12, rtol=0, atol=1e-15)


def _truncation(n, stencil, corr):
    """max |Δ_h φ*(cells) − f_h| with φ* = sin πx sin πy sin πz, ρ = Δφ* = −3π²φ*
    and FIXED ghosts holding φ*, ρ sampled (cell centres, h = 1/n)."""
    h = 1.0 / n
    c = (np.arange(-1, n + 1) + 0.5) * h
    s = np.sin(np.pi * c)
    phi = s[:, None, None] * s[None, :, None] * s[None, None, :]
    rho = -3 * np.pi**2 * phi
    p = oracle.Problem3((n, n, n), h, 0.0, bc=BC_FIXED, stencil=stencil, rhs_correction=corr, nsweeps=0,
                        norm_every=0)
    _, norms = oracle.solve3(p, phi, rho)
    return norms[0, 0]


def test_truncation_order_ladder():
    """7-point: τ_h ratio 4 as h halves (second order); 27-point Mehrstellen
    with f = ρ + S7(ρ)/12: ratio 16 (fourth order); without the correction it
    drops back to 4."""
    t7 = [_truncation(n, 0, False) for n in (16, 32, 64)]
    t27 = [_truncation(n, 1, True) for n in (16, 32, 64)]
    t27n = [_truncation(n, 1, False) for n in (16, 32, 64)]
    for t, lo, hi in ((t7, 3.9, 4.1), (t27, 15.5, 16.5), (t27n, 3.9, 4.1)):
        r = [t[i] / t[i + 1] for i in range(2)]
        assert all(lo < q < hi for q in r), (t, r)
