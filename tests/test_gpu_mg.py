"""GPU parity of the multigrid V-cycle (px_mg_solve)
against the oracle's orc_mg_solve (readings R-MG1..R-MG6) on the
same seeded inputs: φ bit-identical, max-norms bit-identical, Σr² within
1e-12 relative (different summation order)."""
import numpy as np
import pytest

import oracle
from paper_2307_07931_b200 import protox as P

from helpers import BC_MAP, bits_equal, to_device_ghosted, ulp_diff

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SUM_RTOL = 1e-12


def _fields(n0, n1, g, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, (n1 + 2 * g, n0 + 2 * g)), rng.uniform(-1, 1, (n1 + 2 * g, n0 + 2 * g))


def run_mg(n0, n1, bc, st, levels, ncyc, nu1, nu2, nuc, box=None, g=1, graph=True, seed=1, reps=1):
    h = 1.0 / max(n0, n1)
    lam = h * h / 8 if st == 0 else 3 * h * h / 16
    phi0, rho = _fields(n0, n1, g, seed)
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), box or (n0, n1), g, bc, 1)
    phi, scr, f = to_device_ghosted(lay, 0, phi0, g), lay.alloc(0), to_device_ghosted(lay, 0, rho, g)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    for _ in range(reps):  # reps > 1: the cached plan / graph replays on the same φ^0
        lay.view(0, phi, ghosts=True).copy_(torch.from_numpy(phi0))
        s.wait_stream(torch.cuda.current_stream())
        norms = P.mg_solve(lay, P.relax_params(h, lam, st), levels, ncyc, lay.patch(0, phi), lay.patch(0, scr),
                           lay.patch(0, f), nu1=nu1, nu2=nu2, nu_coarse=nuc, use_graph=graph, stream=s)
    out = lay.view(0, phi, ghosts=True).cpu().numpy()
    p = oracle.Problem(n0, n1, h, lam, b0=(box or (n0, n1))[0], b1=(box or (n0, n1))[1], ghost=g,
                       bc=BC_MAP[bc], stencil=st)
    ref, rn = oracle.mg_solve(p, oracle.MG(levels, nu1, nu2, nuc, ncyc), phi0, rho)
    return out, norms, ref, rn


def _check(out, norms, ref, rn, g):
    assert bits_equal(out[g:-g, g:-g], ref[g:-g, g:-g]), ulp_diff(out[g:-g, g:-g], ref[g:-g, g:-g])
    assert bits_equal(out, ref), "ghost ring differs"
    assert norms.shape == rn.shape
    assert bits_equal(norms[:, 0], rn[:, 0])
    np.testing.assert_allclose(norms[:, 1], rn[:, 1], rtol=SUM_RTOL, atol=0)


@pytest.mark.parametrize("bc", [P.PX_BC_PERIODIC, P.PX_BC_DIRICHLET_CC])
@pytest.mark.parametrize("st", [P.PX_LAPLACE_5PT, P.PX_MEHRSTELLEN_9PT])
@pytest.mark.parametrize("graph", [True, False])
def test_mg_vcycles_bitwise(bc, st, graph):
    """V(2,2), 4 levels (96x160 -> 12x20), coarse level in one CTA, 3 cycles."""
    out, norms, ref, rn = run_mg(96, 160, bc, st, 4, 3, 2, 2, 8, box=(32, 40), graph=graph)
    _check(out, norms, ref, rn, 1)
    assert rn[-1, 0] < 0.1 * rn[0, 0]  # it converges


@pytest.mark.parametrize("nu", [(1, 0, 3), (0, 1, 0), (3, 2, 1), (0, 0, 5)])
def test_mg_cycle_shapes_and_parity_of_swaps(nu):
    """Odd sweep counts (result in the scratch buffer, copied back), ν = 0
    (restriction straight after prolongation), no coarse sweeps."""
    nu1, nu2, nuc = nu
    out, norms, ref, rn = run_mg(64, 64, P.PX_BC_DIRICHLET_CC, 0, 3, 2, nu1, nu2, nuc, seed=4)
    _check(out, norms, ref, rn, 1)


def test_mg_deep_hierarchy_and_replay():
    """256² down to 2x2 (8 levels), ghost width 2 on level 0, the cached
    plan replayed twice."""
    out, norms, ref, rn = run_mg(256, 256, P.PX_BC_PERIODIC, 0, 8, 2, 2, 2, 4, g=2, reps=2, seed=7)
    _check(out, norms, ref, rn, 2)


def test_mg_single_level_is_jacobi():
    """levels = 1: one cycle = nu_coarse Jacobi sweeps = px_solve's result."""
    out, norms, ref, rn = run_mg(128, 64, P.PX_BC_PERIODIC, 1, 1, 2, 0, 0, 5, seed=9)
    _check(out, norms, ref, rn, 1)


def test_mg_large_level0_on_bulk_kernel():
    """2048² (level 0 on the TMA relax kernel, >= 4M cells) down to 16², 2 cycles."""
    out, norms, ref, rn = run_mg(2048, 2048, P.PX_BC_DIRICHLET_CC, 0, 8, 2, 2, 2, 8, box=(512, 512), seed=11)
    _check(out, norms, ref, rn, 1)


def test_mg_errors():
    lay = P.Layout(P.box(0, 0, 63, 63), (64, 64), 1, P.PX_BC_FIXED_GHOSTS, 1)
    a, b, c = lay.alloc(0), lay.alloc(0), lay.alloc(0)
    s = torch.cuda.Stream()
    with pytest.raises(P.PxError, match="PERIODIC or DIRICHLET_CC"):
        P.mg_solve(lay, P.relax_params(1 / 64, 1 / 64**2 / 8), 3, 1, lay.patch(0, a), lay.patch(0, b),
                   lay.patch(0, c), stream=s)
    lay2 = P.Layout(P.box(0, 0, 47, 47), (48, 48), 1, P.PX_BC_PERIODIC, 1)
    a, b, c = lay2.alloc(0), lay2.alloc(0), lay2.alloc(0)
    with pytest.raises(P.PxError, match="divisible"):
        P.mg_solve(lay2, P.relax_params(1 / 48, 1 / 48**2 / 8), 6, 1, lay2.patch(0, a), lay2.patch(0, b),
                   lay2.patch(0, c), stream=s)
