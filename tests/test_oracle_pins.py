"""Pins of the CPU oracle against what the paper and the mathematics fix.

No GPU, no libprotox: these tests check ``oracle/`` against
  * constants printed in the paper (Fig. ProtoX index arithmetic, PAPER.md:216-243,
    Fig. ProtoXgpu launch shape PAPER.md:284-318; tests/golden/fig_protox_constants.json),
  * a transcription of the paper's fused loop body (Fig. ProtoX),
  * closed forms: stencil exactness on polynomials, Laplacian eigenvalues,
    Jacobi damping factor, spectral N-sweep solution, exact trajectories,
  * dense 8x8 brute force built from Eq.1 by matrix assembly,
  * invariants (exchange == flat periodic / reflected array, idempotence,
    linearity, translation equivariance, constants, decomposition invariance),
  * order ladders (second order for the 5-point Laplacian as h halves, fourth
    for Mehrstellen with the corrected right-hand side).
Each pin is chosen so that a dropped term, wrong sign, wrong index or swapped
operand in the oracle fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.fft as sfft

import oracle
from oracle import BC_DIRICHLET_CC, BC_FIXED, BC_PERIODIC, ST_LAPLACE5, ST_MEHRSTELLEN9, Problem
from paper_2307_07931_b200 import inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rel_max(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


# ---------------------------------------------------------------- P1 layout
def test_fig_protox_layout_constants():
    """Fig. ProtoX and Fig. ProtoXgpu:
    a 64x64 box stored with one ghost layer as 66x66, dim-0 fastest."""
    with open(os.path.join(GOLDEN, "fig_protox_constants.json")) as f:
        G = json.load(f)
    n, m = G["box_n"], G["box_m"]
    lo, hi = (-1, -1), (n, n)
    assert m == n + 2
    assert oracle.box_ordinal(lo, hi, (0, 0)) == G["center_offset"]
    assert oracle.box_ordinal(lo, hi, (1, 0)) == G["center_offset"] + 1
    assert oracle.box_ordinal(lo, hi, (0, 1)) == G["center_offset"] + m
    for i1 in range(G["loop_last"] + 1):
        b = m * (i1 // n) + (i1 % n)  # reading of the garbled line PAPER.md:224
        x, y = i1 % n, i1 // n
        assert oracle.box_ordinal(lo, hi, (x, y)) == b + G["center_offset"]
        assert oracle.box_ordinal(lo, hi, (x, y - 1)) == b + G["south_offset"]
        assert oracle.box_ordinal(lo, hi, (x - 1, y)) == b + G["west_offset"]
        assert oracle.box_ordinal(lo, hi, (x + 1, y)) == b + G["east_offset"]
        assert oracle.box_ordinal(lo, hi, (x, y + 1)) == b + G["north_offset"]
    assert G["rho_offset"] == m * m
    # the HIP launch covers the box with one spare block; the guard '< 4096' masks it
    assert G["gpu_blocks"] * G["gpu_threads"] >= n * n == (G["gpu_blocks"] - 1) * G["gpu_threads"]
    assert oracle.box_ordinal(lo, hi, (n + 1, 0)) == -1  # outside the box


def test_fig_protox_transcription_matches_oracle():
    """Transcribe the loop body of Fig. ProtoX literally --
    Y[b+67] = (s20 + weight1*s21) - lambda1*s22 with weight1 = λ/h², and
    retval = max |s21/a_h1² - s22| -- and compare with one oracle iteration
    on a periodic 64x64 box.  Different expression trees: agree to rounding."""
    n, m = 64, 66
    h = 1.0 / 256  # 64x64 box of the 256x256 domain of the paper's example
    lam = h * h / 8
    rng = np.random.default_rng(5)
    phi = rng.uniform(-1, 1, (n, n))
    rho = rng.uniform(-1, 1, (n, n))
    X = np.pad(phi, 1, mode="wrap").reshape(-1)  # ghosted φ, m*m, dim-0 fastest
    Y = X.copy()
    weight1, lambda1, a_h1 = lam / (h * h), lam, h
    rhs = rho.reshape(-1)
    retval = 0.0
    for i1 in range(4096):
        b15 = m * (i1 // n) + (i1 % n)
        a48 = b15 + 67
        s20 = X[a48]
        s21 = (X[b15 + 1] - 4.0 * s20) + X[b15 + 66] + X[b15 + 68] + X[b15 + 133]
        s22 = rhs[i1]
        Y[a48] = (s20 + weight1 * s21) - lambda1 * s22
        retval = max(retval, abs((1.0 / (a_h1 * a_h1)) * s21 - s22))
    y_fig = Y.reshape(m, m)[1:-1, 1:-1]

    p = Problem(n, n, h, lam, bc=BC_PERIODIC, nsweeps=1, norm_every=1)
    out, norms = oracle.solve(p, oracle.ghosted(p, phi), oracle.ghosted(p, rho))
    assert rel_max(out[1:-1, 1:-1], y_fig) < 1e-14
    # the fused code reports the residual of the PRE-update iterate (reading R4)
    assert abs(norms[0, 0] - retval) <= 1e-14 * retval


# ------------------------------------------------------ P2 polynomial exactness
@pytest.mark.parametrize("kind,factor", [(ST_LAPLACE5, 1), (ST_MEHRSTELLEN9, 6)])
def test_stencil_exact_on_quadratics(kind, factor):
    """Undivided S on integer-valued polynomials is exact in fp64: constants
    and linears -> 0, a x² + b xy + c y² -> factor·(2a + 2c)."""
    offs, alpha, _ = oracle.stencil_taps(kind, 1.0)
    assert alpha.sum() == 0.0
    ys, xs = np.meshgrid(np.arange(-1, 11), np.arange(-1, 13), indexing="ij")
    xs = xs.astype(np.float64)
    ys = ys.astype(np.float64)
    for (a, b, c, d, e, f) in [(0, 0, 0, 0, 0, 7), (0, 0, 0, 3, -5, 2), (1, 0, 1, 0, 0, 0),
                               (3, -2, 5, 7, 1, -4), (-6, 11, 2, 0, 9, 1)]:
        src = a * xs**2 + b * xs * ys + c * ys**2 + d * xs + e * ys + f
        out = oracle.apply_taps(offs, alpha, 1.0, src, (-1, -1), (0, 0), (11, 9))
        assert np.all(out == factor * (2 * a + 2 * c)), (a, b, c, d, e, f)


def test_laplacian_on_x2_plus_y2_is_4_and_scaled():
    """S5(x²+y²) = 4; sampled at spacing h = 2^-3, Δ_h = S5/h² gives 4 exactly."""
    h = 0.125
    offs, alpha, scale = oracle.stencil_taps(ST_LAPLACE5, h)
    assert scale == 1.0 / (h * h)
    ys, xs = np.meshgrid(np.arange(0, 8), np.arange(0, 8), indexing="ij")
    src = (xs * h) ** 2 + (ys * h) ** 2  # x² + y² sampled at spacing h: Δ = 4 exactly
    out = oracle.apply_taps(offs, alpha, scale, src.astype(np.float64), (0, 0), (1, 1), (6, 6))
    assert np.all(out == 4.0)


def test_stencil_domain_violation_names_point_and_tap():
    offs, alpha, _ = oracle.stencil_taps(ST_LAPLACE5, 1.0)
    src = np.zeros((6, 6))
    with pytest.raises(oracle.OracleError, match=r"i=\(0,0\) tap=\(-1,0\)"):
        oracle.apply_taps(offs, alpha, 1.0, src, (0, 0), (0, 0), (3, 3))


def test_linearity_and_translation_equivariance():
    offs, alpha, _ = oracle.stencil_taps(ST_MEHRSTELLEN9, 1.0)
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, (10, 12))
    y = rng.uniform(-1, 1, (10, 12))
    a, b = 0.75, -2.5
    L = lambda s, lo=(0, 0): oracle.apply_taps(offs, alpha, 1.0, s, lo, (lo[0] + 1, lo[1] + 1),
                                               (lo[0] + 10, lo[1] + 8))
    lhs = L(a * x + b * y)
    rhs = a * L(x) + b * L(y)
    assert rel_max(lhs, rhs) < 1e-13
    assert np.array_equal(L(x), L(x, lo=(37, -5)))


# ------------------------------------------------ P3 closed-form eigenvalues
def _mu5(ax, ay, h):
    return (ax + ay) / (h * h)


def _mu9(ax, ay, h):
    return (ax + ay + ax * ay / 6.0) / (h * h)


@pytest.mark.parametrize("kind", [ST_LAPLACE5, ST_MEHRSTELLEN9])
def test_eigenvalues_periodic(kind):
    """Periodic: cos/sin(2πk x) modes, a_k = -4 sin²(πk h), Δ_h v = μ v."""
    n = 16
    h = 1.0 / n
    p = Problem(n, n, h, 0.0, bc=BC_PERIODIC, stencil=kind)
    x = inputs.cell_centres(n)
    for k, l in [(1, 1), (2, 5), (7, 3), (8, 8), (0, 4)]:
        v = np.outer(np.sin(2 * np.pi * l * x + 0.3), np.cos(2 * np.pi * k * x))
        ax, ay = -4 * math.sin(math.pi * k * h) ** 2, -4 * math.sin(math.pi * l * h) ** 2
        mu = (_mu5 if kind == ST_LAPLACE5 else _mu9)(ax, ay, h)
        out = oracle.apply_laplacian(p, oracle.ghosted(p, v))
        assert np.max(np.abs(out - mu * v)) < 1e-11 * max(abs(mu), 1.0), (k, l)


@pytest.mark.parametrize("kind", [ST_LAPLACE5, ST_MEHRSTELLEN9])
def test_eigenvalues_dirichlet_cc(kind):
    """Cell-centred Dirichlet by odd reflection: sin(kπ(i+½)h), a_k = -4 sin²(kπh/2)."""
    n = 16
    h = 1.0 / n
    p = Problem(n, n, h, 0.0, bc=BC_DIRICHLET_CC, stencil=kind)
    x = inputs.cell_centres(n)
    for k, l in [(1, 1), (2, 5), (16, 3), (9, 16)]:
        v = np.outer(np.sin(l * np.pi * x), np.sin(k * np.pi * x))
        ax, ay = -4 * math.sin(k * math.pi * h / 2) ** 2, -4 * math.sin(l * math.pi * h / 2) ** 2
        mu = (_mu5 if kind == ST_LAPLACE5 else _mu9)(ax, ay, h)
        out = oracle.apply_laplacian(p, oracle.ghosted(p, v))
        assert np.max(np.abs(out - mu * v)) < 1e-11 * abs(mu), (k, l)


def test_eigenvalues_vertex_fixed_ghosts():
    """Vertex-centred Dirichlet (FIXED ghosts = 0): sin(kπ i h), h = 1/(n+1)."""
    n = 15
    h = 1.0 / (n + 1)
    p = Problem(n, n, h, 0.0, bc=BC_FIXED)
    xi = (np.arange(n) + 1) * h
    for k, l in [(1, 1), (3, 14), (15, 15)]:
        v = np.outer(np.sin(l * np.pi * xi), np.sin(k * np.pi * xi))
        mu = _mu5(-4 * math.sin(k * math.pi * h / 2) ** 2, -4 * math.sin(l * math.pi * h / 2) ** 2, h)
        out = oracle.apply_laplacian(p, oracle.ghosted(p, v, 0.0))
        assert np.max(np.abs(out - mu * v)) < 1e-11 * abs(mu)


# --------------------------------------------------------- P4 dense brute force
def _dense_matrix(n, bc, h, kind):
    """Assemble the n²xn² matrix of Δ_h with the BC folded in, directly from
    Eq.1 and the tap list given here (not the oracle's)."""
    if kind == ST_LAPLACE5:
        taps = {(0, 0): -4.0, (1, 0): 1.0, (-1, 0): 1.0, (0, 1): 1.0, (0, -1): 1.0}
        sc = 1.0 / (h * h)
    else:
        taps = {(0, 0): -20.0}
        for o in [(1, 0), (-1, 0), (0, 1), (0, -1)]:
            taps[o] = 4.0
        for o in [(1, 1), (-1, 1), (1, -1), (-1, -1)]:
            taps[o] = 1.0
        sc = 1.0 / (6.0 * h * h)
    A = np.zeros((n * n, n * n))
    for y in range(n):
        for x in range(n):
            for (dx, dy), a in taps.items():
                qx, qy, s = x + dx, y + dy, 1.0
                if bc == BC_PERIODIC:
                    qx, qy = qx % n, qy % n
                else:
                    if qx < 0 or qx >= n:
                        qx, s = (-qx - 1 if qx < 0 else 2 * n - 1 - qx), -s
                    if qy < 0 or qy >= n:
                        qy, s = (-qy - 1 if qy < 0 else 2 * n - 1 - qy), -s
                A[x + y * n, qx + qy * n] += s * a * sc
    return A


@pytest.mark.parametrize("bc", [BC_PERIODIC, BC_DIRICHLET_CC])
@pytest.mark.parametrize("kind", [ST_LAPLACE5, ST_MEHRSTELLEN9])
def test_dense_8x8_bruteforce(bc, kind):
    n, nsw = 8, 37
    h = 1.0 / n
    lam = h * h / 8
    A = _dense_matrix(n, bc, h, kind)
    rng = np.random.default_rng(11 + bc + 2 * kind)
    phi0 = rng.uniform(-1, 1, (n, n))
    rho = rng.uniform(-1, 1, (n, n))
    v = phi0.reshape(-1).copy()
    f = rho.reshape(-1)
    res = []
    for it in range(nsw):
        if it % 5 == 0:
            r = A @ v - f
            res.append((np.max(np.abs(r)), np.sum(r * r)))
        v = v + lam * (A @ v - f)
    r = A @ v - f
    res.append((np.max(np.abs(r)), np.sum(r * r)))
    p = Problem(n, n, h, lam, bc=bc, stencil=kind, nsweeps=nsw, norm_every=5, b0=4, b1=4)
    out, norms = oracle.solve(p, oracle.ghosted(p, phi0), oracle.ghosted(p, rho))
    assert rel_max(out[1:-1, 1:-1].reshape(-1), v) < 1e-13
    assert norms.shape == (len(res), 2)
    np.testing.assert_allclose(norms, np.array(res), rtol=1e-12)


# --------------------------------------------- P5 Jacobi damping per sweep
@pytest.mark.parametrize("omega_lam", ["h2/8", "h2/4"])
def test_jacobi_damping_factor(omega_lam):
    """ρ = 0, φ0 = one mode: one sweep multiplies it by g = 1 + λμ."""
    n = 32
    h = 1.0 / n
    lam = h * h / 8 if omega_lam == "h2/8" else h * h / 4
    x = inputs.cell_centres(n)
    for k, l in [(1, 1), (3, 7), (32, 32)]:
        v = np.outer(np.sin(l * np.pi * x), np.sin(k * np.pi * x))
        sk, sl = math.sin(k * math.pi * h / 2) ** 2, math.sin(l * math.pi * h / 2) ** 2
        g = 1 - 0.5 * (sk + sl) if lam == h * h / 8 else 0.5 * (math.cos(k * math.pi * h) + math.cos(l * math.pi * h))
        p = Problem(n, n, h, lam, bc=BC_DIRICHLET_CC, nsweeps=3, norm_every=-1)
        out, _ = oracle.solve(p, oracle.ghosted(p, v), oracle.ghosted(p, np.zeros_like(v)))
        assert np.max(np.abs(out[1:-1, 1:-1] - g**3 * v)) < 1e-14


# ----------------------------------------- P6 spectral N-sweep closed form
def _spectral_periodic(phi0, f, h, lam, N, kind):
    n = phi0.shape[0]
    k = np.arange(n)
    a = -4 * np.sin(np.pi * k / n) ** 2
    ay, ax = np.meshgrid(a, a, indexing="ij")
    mu = (_mu5 if kind == ST_LAPLACE5 else _mu9)(ax, ay, h)
    P, F = np.fft.fft2(phi0), np.fft.fft2(f)
    g = 1 + lam * mu
    gN = g**N
    with np.errstate(divide="ignore", invalid="ignore"):
        src = np.where(mu == 0, -N * lam, (1 - gN) / np.where(mu == 0, 1, mu))
    out = gN * P + src * F
    return np.real(np.fft.ifft2(out)), mu


def _spectral_dirichlet_cc(phi0, f, h, lam, N, kind):
    n = phi0.shape[0]
    m = np.arange(1, n + 1)
    a = -4 * np.sin(m * np.pi * h / 2) ** 2
    ay, ax = np.meshgrid(a, a, indexing="ij")
    mu = (_mu5 if kind == ST_LAPLACE5 else _mu9)(ax, ay, h)
    P = sfft.dstn(phi0, type=2)
    F = sfft.dstn(f, type=2)
    g = 1 + lam * mu
    # g may be negative (the ω=1 checkerboard): g**N handles the sign exactly
    gN = g**N
    out = gN * P + (1 - gN) / mu * F
    return sfft.idstn(out, type=2), mu


@pytest.mark.parametrize("kind", [ST_LAPLACE5, ST_MEHRSTELLEN9])
@pytest.mark.parametrize("bc", [BC_PERIODIC, BC_DIRICHLET_CC])
@pytest.mark.parametrize("lam_div", [8, 4])
def test_spectral_closed_form_nsweeps(kind, bc, lam_div):
    """φ̂^N = g^N φ̂⁰ + (1 - g^N)/μ · f̂ per mode (FFT periodic, DST-II cell-centred)."""
    n, N = 32, 100
    h = 1.0 / n
    lam = h * h / lam_div if kind == ST_LAPLACE5 else 3 * h * h / (10 if lam_div == 4 else 16)
    rng = np.random.default_rng(100 + kind + 3 * bc + lam_div)
    phi0 = rng.uniform(-1, 1, (n, n))
    rho = rng.uniform(-1, 1, (n, n))
    p = Problem(n, n, h, lam, bc=bc, stencil=kind, nsweeps=N, norm_every=-1, b0=8, b1=16)
    out, _ = oracle.solve(p, oracle.ghosted(p, phi0), oracle.ghosted(p, rho))
    fn = _spectral_periodic if bc == BC_PERIODIC else _spectral_dirichlet_cc
    ref, _ = fn(phi0, rho, h, lam, N, kind)
    assert rel_max(out[1:-1, 1:-1], ref) < 1e-12


def test_spectral_residual_norms():
    """Residual of φ^m, r̂ = μ φ̂^m − ρ̂: max and Σr² of the oracle's record."""
    n, N, E = 32, 40, 10
    h = 1.0 / n
    lam = h * h / 8
    rng = np.random.default_rng(7)
    phi0 = rng.uniform(-1, 1, (n, n))
    rho = rng.uniform(-1, 1, (n, n))
    p = Problem(n, n, h, lam, bc=BC_DIRICHLET_CC, nsweeps=N, norm_every=E)
    _, norms = oracle.solve(p, oracle.ghosted(p, phi0), oracle.ghosted(p, rho))
    for j, m in enumerate([0, 10, 20, 30, 40]):
        phim, mu = _spectral_dirichlet_cc(phi0, rho, h, lam, m, ST_LAPLACE5)
        R = mu * sfft.dstn(phim, type=2) - sfft.dstn(rho, type=2)
        r = sfft.idstn(R, type=2)
        assert abs(norms[j, 0] - np.max(np.abs(r))) < 1e-9 * np.max(np.abs(r))
        assert abs(norms[j, 1] - np.sum(r * r)) < 1e-9 * np.sum(r * r)


# --------------------------------------------- P7/P8 exact trajectories
def test_config1_exact_trajectory():
    """BASELINE config 1: Dirichlet-CC 64², h = 1/64, λ = h²/8 = 2^-15, φ0 = 0,
    ρ = sin πx sin πy (an eigenvector): r(φ^k) = -g^k ρ with g = cos²(π/128);
    ‖r‖∞ = g^(k+1) (max|ρ| = g) and ‖r‖₂,h = g^k/2.  Values in
    tests/golden/config1_closed_form.json (written by tests/golden/make_closed_form.py)."""
    with open(os.path.join(GOLDEN, "config1_closed_form.json")) as f:
        G = json.load(f)
    n = 64
    h = 1.0 / n
    lam = 2.0**-15
    rho = inputs.sine_field(n, n)
    p = Problem(n, n, h, lam, bc=BC_DIRICHLET_CC, nsweeps=100, norm_every=1)
    out, norms = oracle.solve(p, oracle.ghosted(p, np.zeros_like(rho)), oracle.ghosted(p, rho))
    g = G["g"]
    assert abs(g - math.cos(math.pi / 128) ** 2) < 1e-16
    assert norms.shape == (101, 2)
    k = np.arange(101)
    np.testing.assert_allclose(norms[:, 0], g ** (k + 1), rtol=2e-13)
    np.testing.assert_allclose(np.sqrt(h * h * norms[:, 1]), g**k / 2, rtol=2e-13)
    assert abs(norms[99, 0] - G["resmax_phi99"]) < 2e-13
    assert abs(norms[100, 0] - G["resmax_phi100"]) < 2e-13
    assert abs(np.abs(out[1:-1, 1:-1]).max() - G["max_phi100"]) < 1e-16 * 10
    # ω = 1 variant (λ = 2^-14)
    p2 = Problem(n, n, h, 2.0**-14, bc=BC_DIRICHLET_CC, nsweeps=100, norm_every=-1)
    out2, _ = oracle.solve(p2, oracle.ghosted(p2, np.zeros_like(rho)), oracle.ghosted(p2, rho))
    assert abs(np.abs(out2[1:-1, 1:-1]).max() - G["max_phi100_omega1"]) < 1e-16 * 10


def test_config2_periodic_sine_closed_form():
    """Config 2 shape (periodic sine, wavenumber 2), reduced to 128²: the
    residual max-norm of φ^m is g^m·max|ρ| with g = cos²(π/n)."""
    n, N, E = 128, 60, 10
    h = 1.0 / n
    lam = h * h / 8
    rho = inputs.sine_field(n, n, 2, 2)
    p = Problem(n, n, h, lam, bc=BC_PERIODIC, nsweeps=N, norm_every=E, b0=32, b1=64)
    _, norms = oracle.solve(p, oracle.ghosted(p, np.zeros_like(rho)), oracle.ghosted(p, rho))
    g = math.cos(math.pi / n) ** 2
    m = np.array([0, 10, 20, 30, 40, 50, 60])
    np.testing.assert_allclose(norms[:, 0], g**m * np.max(np.abs(rho)), rtol=1e-12)


# ------------------------------------------------ P9/P10 order ladders
def _truncation(n, kind, corrected):
    """τ_h = max|Δ_h φ*_sampled − f_h| on a vertex grid, ghosts = φ* (FIXED)."""
    h = 1.0 / (n + 1)
    xi = np.arange(-1, n + 1) * h + h  # ghost + interior + ghost vertices
    # φ* = cos(πx) sin(πy) e^y;  Δφ* = -π²φ* + cos(πx) e^y [(1-π²) sin(πy) + 2π cos(πy)]
    X, Y = np.meshgrid(xi, xi, indexing="xy")
    phi = np.cos(np.pi * X) * np.sin(np.pi * Y) * np.exp(Y)
    lap = -np.pi**2 * phi + np.cos(np.pi * X) * (
        (1 - np.pi**2) * np.sin(np.pi * Y) * np.exp(Y) + 2 * np.pi * np.cos(np.pi * Y) * np.exp(Y))
    p = Problem(n, n, h, 0.0, bc=BC_FIXED, stencil=kind, rhs_correction=corrected)
    r = oracle.residual(p, phi, lap)
    return r[0]


def test_truncation_order_ladder():
    t5 = [_truncation(n - 1, ST_LAPLACE5, False) for n in (16, 32, 64, 128)]
    r5 = [t5[i] / t5[i + 1] for i in range(3)]
    assert all(3.8 < r < 4.2 for r in r5), r5
    t9 = [_truncation(n - 1, ST_MEHRSTELLEN9, True) for n in (8, 16, 32, 64)]
    r9 = [t9[i] / t9[i + 1] for i in range(3)]
    assert all(14.5 < r < 17.5 for r in r9), r9
    # without the RHS correction Mehrstellen is only second order
    t9u = [_truncation(n - 1, ST_MEHRSTELLEN9, False) for n in (16, 32, 64)]
    assert all(3.5 < t9u[i] / t9u[i + 1] < 4.5 for i in range(2))


def _converged_error(n, kind):
    """Jacobi to convergence on Dirichlet-CC, ρ = sin πx sin πy; error against
    φ* = −ρ/(2π²) at cell centres (Δφ* = ρ, Eq.2)."""
    h = 1.0 / n
    rho = inputs.sine_field(n, n)
    if kind == ST_LAPLACE5:
        lam, rate = h * h / 4, 1 - math.cos(math.pi * h)
    else:
        lam = 3 * h * h / 10
        rate = lam * 2 * math.pi**2
    nsw = int(32 / rate) + 10
    p = Problem(n, n, h, lam, bc=BC_DIRICHLET_CC, stencil=kind, rhs_correction=(kind == ST_MEHRSTELLEN9),
                nsweeps=nsw, norm_every=-1)
    out, _ = oracle.solve(p, oracle.ghosted(p, np.zeros_like(rho)), oracle.ghosted(p, rho))
    exact = -rho / (2 * math.pi**2)
    return np.max(np.abs(out[1:-1, 1:-1] - exact))


def test_manufactured_solution_second_order():
    """BASELINE north star: the manufactured-solution solve converges at second
    order as h halves (5-point); fourth order for corrected Mehrstellen."""
    e5 = [_converged_error(n, ST_LAPLACE5) for n in (8, 16, 32, 64)]
    r5 = [e5[i] / e5[i + 1] for i in range(3)]
    assert all(3.9 < r < 4.1 for r in r5), r5
    # closed form of the discrete error for the eigen-mode (P10)
    for n, e in zip((8, 16, 32, 64), e5):
        h = 1.0 / n
        mu = -8 * math.sin(math.pi * h / 2) ** 2 / (h * h)
        emax = math.cos(math.pi / (2 * n)) ** 2 * abs(1 / mu + 1 / (2 * math.pi**2))
        assert abs(e - emax) < 1e-9 * emax + 1e-14
    e9 = [_converged_error(n, ST_MEHRSTELLEN9) for n in (8, 16, 32)]
    r9 = [e9[i] / e9[i + 1] for i in range(2)]
    assert all(15.0 < r < 17.0 for r in r9), r9


# ---------------------------------------------------------- P11 invariants
def test_exchange_equals_flat_periodic_array():
    """SPEC grid example: ghosts equal the flat periodic array."""
    n0, n1, g = 12, 8, 2
    p = Problem(n0, n1, 1.0, 0.0, b0=4, b1=4, ghost=g, bc=BC_PERIODIC)
    ys, xs = np.meshgrid(np.arange(n1), np.arange(n0), indexing="ij")
    field = (xs + 10.0 * ys).astype(np.float64)
    glob = oracle.ghosted(p, field, np.nan)
    ex = oracle.exchange(p, glob)
    assert np.array_equal(ex, np.pad(field, g, mode="wrap"))
    assert np.array_equal(oracle.exchange(p, ex), ex)  # idempotent
    # every box's own ghost ring also equals the wrapped global field
    flat = np.pad(field, 4 + g, mode="wrap")
    for ib in range((n0 // 4) * (n1 // 4)):
        bx, by = ib % 3, ib // 3
        want = flat[4 + by * 4: 4 + by * 4 + 4 + 2 * g, 4 + bx * 4: 4 + bx * 4 + 4 + 2 * g]
        assert np.array_equal(oracle.exchange_box(p, glob, ib), want)


def test_exchange_dirichlet_cc_odd_reflection():
    n, g = 8, 2
    p = Problem(n, n, 1.0, 0.0, b0=4, b1=4, ghost=g, bc=BC_DIRICHLET_CC)
    rng = np.random.default_rng(3)
    field = rng.uniform(-1, 1, (n, n))
    ex = oracle.exchange(p, oracle.ghosted(p, field, np.nan))
    want = np.pad(field, g, mode="symmetric")
    sign = np.ones((n + 2 * g, n + 2 * g))
    sign[:g, :] *= -1
    sign[-g:, :] *= -1
    sign[:, :g] *= -1
    sign[:, -g:] *= -1
    assert np.array_equal(ex, want * sign)


def test_exchange_fixed_keeps_domain_ghosts():
    n = 6
    p = Problem(n, n, 1.0, 0.0, b0=3, b1=3, bc=BC_FIXED)
    field = np.arange(n * n, dtype=np.float64).reshape(n, n)
    glob = oracle.ghosted(p, field, -7.0)
    ex = oracle.exchange(p, glob)
    assert np.array_equal(ex, glob)


def test_constants_preserved_and_mean_invariant():
    n = 16
    h = 1.0 / n
    p = Problem(n, n, h, h * h / 8, bc=BC_PERIODIC, nsweeps=25, norm_every=-1)
    c = np.full((n, n), 0.625)
    out, _ = oracle.solve(p, oracle.ghosted(p, c), oracle.ghosted(p, np.zeros_like(c)))
    assert np.all(out == 0.625)
    rho = inputs.sine_field(n, n, 2, 4)
    rng = np.random.default_rng(2)
    phi0 = rng.uniform(-1, 1, (n, n))
    out, _ = oracle.solve(p, oracle.ghosted(p, phi0), oracle.ghosted(p, rho))
    assert abs(out[1:-1, 1:-1].mean() - phi0.mean()) < 1e-14


# ------------------------------------------- P12 decomposition invariance
@pytest.mark.parametrize("bc", [BC_PERIODIC, BC_DIRICHLET_CC])
@pytest.mark.parametrize("kind", [ST_LAPLACE5, ST_MEHRSTELLEN9])
def test_box_decomposition_invariance_bitwise(bc, kind):
    n0, n1 = 24, 16
    h = 1.0 / 16
    rng = np.random.default_rng(9)
    phi0 = rng.uniform(-1, 1, (n1, n0))
    rho = rng.uniform(-1, 1, (n1, n0))
    outs = []
    for b0, b1 in [(24, 16), (8, 8), (12, 4), (4, 16)]:
        p = Problem(n0, n1, h, h * h / 8, b0=b0, b1=b1, bc=bc, stencil=kind, nsweeps=13, norm_every=4)
        outs.append(oracle.solve(p, oracle.ghosted(p, phi0), oracle.ghosted(p, rho)))
    for o, nrm in outs[1:]:
        assert np.array_equal(o, outs[0][0])
        assert np.array_equal(nrm[:, 0], outs[0][1][:, 0])
        np.testing.assert_allclose(nrm[:, 1], outs[0][1][:, 1], rtol=1e-15)


# --------------------------------------------------------- norms details
def test_neumaier_sum_exact_cases():
    assert oracle.neumaier_sum(np.array([1e16, 1.0, -1e16])) == 1.0
    assert oracle.neumaier_sum(np.array([1.0, 1e100, 1.0, -1e100])) == 2.0
    x = np.random.default_rng(0).uniform(0, 1, 100000)
    assert oracle.neumaier_sum(x) == math.fsum(x)


def test_max_norm_propagates_nan():
    n = 8
    p = Problem(n, n, 1.0 / n, 0.0, bc=BC_PERIODIC)
    phi = np.zeros((n, n))
    phi[3, 4] = np.nan
    r = oracle.residual(p, oracle.ghosted(p, phi), oracle.ghosted(p, np.ones((n, n))))
    assert math.isnan(r[0])


def test_norms_of_infinite_residual():
    """Σr² is the plain sum of the squares (reading R6): one r = ±inf makes it
    +inf (every term is >= 0), not the NaN a compensation term (inf - inf)
    would produce; max|r| is inf.  A NaN term makes both NaN.  The rest of the
    field is finite, so only the definition fixes these values."""
    n = 8
    p = Problem(n, n, 1.0 / n, 0.0, bc=BC_PERIODIC)
    phi = np.random.default_rng(3).uniform(-1, 1, (n, n))
    rho = np.ones((n, n))
    rho[2, 5] = np.inf
    m, s = oracle.residual(p, oracle.ghosted(p, phi), oracle.ghosted(p, rho))
    assert m == np.inf and s == np.inf
    rho[6, 1] = np.nan
    m, s = oracle.residual(p, oracle.ghosted(p, phi), oracle.ghosted(p, rho))
    assert math.isnan(m) and math.isnan(s)
    assert oracle.neumaier_sum(np.array([1.0, np.inf, 2.0])) == np.inf
    assert math.isnan(oracle.neumaier_sum(np.array([1.0, np.inf, np.nan])))


def test_fault_injection_sign_flip_breaks_spectral_pin():
    """SPEC S:447 idea: a flipped λ sign must fail the closed-form check."""
    n, N = 16, 20
    h = 1.0 / n
    lam = h * h / 8
    rng = np.random.default_rng(4)
    phi0, rho = rng.uniform(-1, 1, (n, n)), rng.uniform(-1, 1, (n, n))
    ref, _ = _spectral_periodic(phi0, rho, h, lam, N, ST_LAPLACE5)
    p = Problem(n, n, h, -lam, bc=BC_PERIODIC, nsweeps=N, norm_every=-1)
    out, _ = oracle.solve(p, oracle.ghosted(p, phi0), oracle.ghosted(p, rho))
    assert rel_max(out[1:-1, 1:-1], ref) > 1e-3


# ------------------------------------------------ multigrid V-cycle (R-MG)
# The paper names multigrid but defines none; the V-cycle
# is DESIGN.md readings R-MG1..R-MG6.  Pins: exactness of the transfer
# operators on polynomials, an 8x8 dense brute-force V-cycle built here from
# matrices, and the fixed point = the discrete solution (spectral closed form).
def test_mg_restrict_linear_exact():
    """-R of a linear cell-centred field is minus the field at the coarse
    centres, exactly (dyadic coefficients)."""
    n = 16
    x = (np.arange(n) + 0.5) / n
    d = 0.75 + 0.5 * x[None, :] - 0.25 * x[:, None]
    X = (np.arange(n // 2) + 0.5) / (n // 2)
    want = -(0.75 + 0.5 * X[None, :] - 0.25 * X[:, None])
    assert np.array_equal(oracle.mg_restrict(d), want)
    # and it is minus the 2x2 average for arbitrary data
    rng = np.random.default_rng(3)
    r = rng.uniform(-1, 1, (6, 10))
    np.testing.assert_allclose(oracle.mg_restrict(r), -0.25 * (r[0::2, 0::2] + r[0::2, 1::2] + r[1::2, 0::2] + r[1::2, 1::2]),
                               rtol=0, atol=4e-16)


def test_mg_prolong_linear_and_walls():
    """Bilinear cell-centred prolongation reproduces a linear field at every
    fine cell away from the walls; periodic constants everywhere; with odd
    reflection a constant c gives c/2 in the fine cells next to a wall and
    c/4 in the corner cells (the interpolant vanishes on the wall)."""
    nc = 8
    X = (np.arange(nc) + 0.5) / nc
    e = 0.5 + 0.25 * X[None, :] + 0.125 * X[:, None]
    out = oracle.mg_prolong(e, np.zeros((2 * nc, 2 * nc)), BC_DIRICHLET_CC)
    x = (np.arange(2 * nc) + 0.5) / (2 * nc)
    want = 0.5 + 0.25 * x[None, :] + 0.125 * x[:, None]
    assert np.array_equal(out[1:-1, 1:-1], want[1:-1, 1:-1])
    c = 0.75
    per = oracle.mg_prolong(np.full((nc, nc), c), np.ones((2 * nc, 2 * nc)), BC_PERIODIC)
    assert np.array_equal(per, np.full((2 * nc, 2 * nc), 1.0 + c))
    dc = oracle.mg_prolong(np.full((nc, nc), c), np.zeros((2 * nc, 2 * nc)), BC_DIRICHLET_CC)
    assert np.array_equal(dc[1:-1, 1:-1], np.full((2 * nc - 2, 2 * nc - 2), c))
    assert np.array_equal(dc[0, 1:-1], np.full(2 * nc - 2, c / 2))
    assert np.array_equal(dc[1:-1, -1], np.full(2 * nc - 2, c / 2))
    assert dc[0, 0] == c / 4 and dc[-1, -1] == c / 4


def _dense_prolong(nc, bc):
    """(2nc)² x nc² bilinear prolongation with the boundary rule folded in."""
    nf = 2 * nc
    Pm = np.zeros((nf * nf, nc * nc))
    for y in range(nf):
        for x in range(nf):
            I, J = x // 2, y // 2
            xn = I + 1 if x % 2 else I - 1
            yn = J + 1 if y % 2 else J - 1
            for (qx, qy, w) in [(I, J, 9), (xn, J, 3), (I, yn, 3), (xn, yn, 1)]:
                s = 1.0
                if bc == BC_PERIODIC:
                    qx, qy = qx % nc, qy % nc
                else:
                    if qx < 0 or qx >= nc:
                        qx, s = (-qx - 1 if qx < 0 else 2 * nc - 1 - qx), -s
                    if qy < 0 or qy >= nc:
                        qy, s = (-qy - 1 if qy < 0 else 2 * nc - 1 - qy), -s
                Pm[x + y * nf, qx + qy * nc] += s * w / 16.0
    return Pm


def _dense_restrict(nc):
    nf = 2 * nc
    Rm = np.zeros((nc * nc, nf * nf))
    for J in range(nc):
        for I in range(nc):
            for a in (0, 1):
                for b in (0, 1):
                    Rm[I + J * nc, (2 * I + a) + (2 * J + b) * nf] = 0.25
    return Rm


@pytest.mark.parametrize("bc", [BC_PERIODIC, BC_DIRICHLET_CC])
@pytest.mark.parametrize("kind", [ST_LAPLACE5, ST_MEHRSTELLEN9])
def test_mg_dense_8x8_vcycle_bruteforce(bc, kind):
    """Two V(2,2)-cycles, 3 levels (8, 4, 2), 3 coarse sweeps: dense matrices
    A_l (Eq.1 with the BC), R (2x2 average), P (bilinear), the recursion
    written with them; the oracle agrees to rounding."""
    n, levels, nu1, nu2, nuc, cyc = 8, 3, 2, 2, 3, 2
    h = 1.0 / n
    lam = h * h / 8 if kind == ST_LAPLACE5 else 3 * h * h / 16
    A = [_dense_matrix(n >> l, bc, h * 2**l, kind) for l in range(levels)]
    lamv = [lam * 4**l for l in range(levels)]
    Rm = [_dense_restrict(n >> (l + 1)) for l in range(levels - 1)]
    Pm = [_dense_prolong(n >> (l + 1), bc) for l in range(levels - 1)]

    def V(l, v, f):
        if l == levels - 1:
            for _ in range(nuc):
                v = v + lamv[l] * (A[l] @ v - f)
            return v
        for _ in range(nu1):
            v = v + lamv[l] * (A[l] @ v - f)
        fc = Rm[l] @ (f - A[l] @ v)
        e = V(l + 1, np.zeros(fc.size), fc)
        v = v + Pm[l] @ e
        for _ in range(nu2):
            v = v + lamv[l] * (A[l] @ v - f)
        return v

    rng = np.random.default_rng(5 + bc + 2 * kind)
    phi0, rho = rng.uniform(-1, 1, (n, n)), rng.uniform(-1, 1, (n, n))
    v, f = phi0.reshape(-1).copy(), rho.reshape(-1)
    res = []
    r = A[0] @ v - f
    res.append((np.max(np.abs(r)), np.sum(r * r)))
    for _ in range(cyc):
        v = V(0, v, f)
        r = A[0] @ v - f
        res.append((np.max(np.abs(r)), np.sum(r * r)))
    p = Problem(n, n, h, lam, bc=bc, stencil=kind, b0=4, b1=8)
    out, norms = oracle.mg_solve(p, oracle.MG(levels, nu1, nu2, nuc, cyc), oracle.ghosted(p, phi0),
                                 oracle.ghosted(p, rho))
    assert rel_max(out[1:-1, 1:-1].reshape(-1), v) < 1e-13
    np.testing.assert_allclose(norms, np.array(res), rtol=1e-12)


@pytest.mark.parametrize("kind", [ST_LAPLACE5, ST_MEHRSTELLEN9])
def test_mg_converges_to_discrete_solution(kind):
    """Fixed point: V-cycles drive φ to A⁻¹ρ.  Dirichlet-CC sine mode: φ* =
    ρ/μ₁₁ in closed form; periodic random zero-mean ρ: the FFT solve.  Per
    cycle the residual drops by < 0.35 (V(2,2), ω = 1/2 Jacobi smoother)."""
    n = 32
    h = 1.0 / n
    lam = h * h / 8 if kind == ST_LAPLACE5 else 3 * h * h / 16
    x = (np.arange(n) + 0.5) * h
    rho = np.outer(np.sin(np.pi * x), np.sin(np.pi * x))
    a = -4 * math.sin(math.pi * h / 2) ** 2
    mu = (_mu5 if kind == ST_LAPLACE5 else _mu9)(a, a, h)
    p = Problem(n, n, h, lam, bc=BC_DIRICHLET_CC, stencil=kind)
    out, norms = oracle.mg_solve(p, oracle.MG(5, 2, 2, 8, 30), np.zeros(p.gshape), oracle.ghosted(p, rho))
    assert rel_max(out[1:-1, 1:-1], rho / mu) < 1e-12
    ratios = norms[1:12, 0] / norms[:11, 0]
    assert np.all(ratios < 0.35), ratios
    # periodic, random zero-mean right-hand side
    rng = np.random.default_rng(9)
    f = rng.uniform(-1, 1, (n, n))
    f -= f.mean()
    pp = Problem(n, n, h, lam, bc=BC_PERIODIC, stencil=kind, b0=8, b1=16)
    out, norms = oracle.mg_solve(pp, oracle.MG(5, 2, 2, 8, 40), np.zeros(pp.gshape), oracle.ghosted(pp, f))
    k = np.arange(n)
    ak = -4 * np.sin(np.pi * k / n) ** 2
    ay, ax = np.meshgrid(ak, ak, indexing="ij")
    muk = (_mu5 if kind == ST_LAPLACE5 else _mu9)(ax, ay, h)
    F = np.fft.fft2(f)
    S = np.where(muk == 0, 0, F / np.where(muk == 0, 1, muk))
    want = np.real(np.fft.ifft2(S))
    assert rel_max(out[1:-1, 1:-1] - out[1:-1, 1:-1].mean(), want) < 1e-10
    assert norms[-1, 0] < 1e-11 * norms[0, 0]
