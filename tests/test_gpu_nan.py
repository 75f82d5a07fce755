"""NaN / inf propagation through every solve-kernel family (reading R7, SURVEY
§8(c) A7): Fig. ProtoX's `(ret >= |x|) ? ret : |x|` silently drops
a NaN; libprotox must instead report max|r| = NaN exactly where the oracle's
NaN-propagating max (oracle/protox_oracle.cpp, `residual`) does, for the
batched cross-rank max too (computeMaxResidualAcrossProcs).

Two injections, each through every kernel family px_solve can choose:
  nan_phi  a NaN in φ⁰ at a face-adjacent cell: every recorded max is NaN;
  inf_rho  ρ = +inf at one cell: r(φ⁰) has |r| = inf there (entry 0 is inf,
           not NaN), φ¹ = -inf there, and r(φ¹) = inf - inf = NaN -- so the
           norm sequence is (inf, NaN, NaN, ...) and a kernel that confuses
           inf with NaN, or drops NaN after an inf, fails.
The field is compared NaN-aware (same NaN mask; every other cell bit for bit:
GPU and CPU NaN payloads differ by design), max-norms by NaN mask and bits,
Σr² by NaN mask and 1e-12 relative.  Each case asserts which kernel the solve
actually ran (px_last_solve_kernels)."""
import os

import numpy as np
import pytest

import oracle
from paper_2307_07931_b200 import protox as P

from helpers import BC_MAP, bits_equal, owned_to_host, to_device_ghosted
from test_gpu_parity import run_gpu_solve

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

KINDS = ["nan_phi", "inf_rho"]


def _fields(n0, n1, g, seed, kind):
    rng = np.random.default_rng(seed)
    phi0 = rng.uniform(-1, 1, (n1 + 2 * g, n0 + 2 * g))
    rho = rng.uniform(-1, 1, (n1 + 2 * g, n0 + 2 * g))
    if kind == "nan_phi":
        phi0[g, g + 5] = np.nan                     # interior row 0: images at the y face
    else:
        rho[g + n1 // 2, g + n0 // 3] = np.inf      # interior cell in the middle
    return phi0, rho


def _orc(n0, n1, h, lam, bc, N, E, phi0, rho, g=1, b=None, st=0):
    p = oracle.Problem(n0, n1, h, lam, b0=(b or (n0, n1))[0], b1=(b or (n0, n1))[1], ghost=g,
                       bc=BC_MAP[bc], stencil=st, nsweeps=N, norm_every=E)
    return oracle.solve(p, phi0, rho)


def check_nan_parity(out, ref, gn, rn, kind):
    out, ref = np.ascontiguousarray(out), np.ascontiguousarray(ref)
    mo, mr = np.isnan(out), np.isnan(ref)
    assert mr.any(), "injection did not reach the field"
    assert np.array_equal(mo, mr), f"NaN masks differ: gpu {mo.sum()} oracle {mr.sum()}"
    assert bits_equal(out[~mo], ref[~mr])
    assert gn.shape == rn.shape, (gn.shape, rn.shape)
    nm_g, nm_r = np.isnan(gn[:, 0]), np.isnan(rn[:, 0])
    assert np.array_equal(nm_g, nm_r), (gn[:, 0], rn[:, 0])
    assert bits_equal(gn[~nm_r, 0], rn[~nm_r, 0])
    assert np.array_equal(np.isnan(gn[:, 1]), np.isnan(rn[:, 1]))
    fin = np.isfinite(rn[:, 1])
    assert np.array_equal(gn[~fin & ~np.isnan(rn[:, 1]), 1], rn[~fin & ~np.isnan(rn[:, 1]), 1])
    np.testing.assert_allclose(gn[fin, 1], rn[fin, 1], rtol=1e-12, atol=0)
    # what the oracle fixes for the two injections (not a GPU property)
    if kind == "nan_phi":
        assert nm_r.all()
    else:
        assert rn[0, 0] == np.inf and nm_r[1:].all()


def _solve_case(n0, n1, bc, N, E, kind, seed, nranks=1, tk=1, box=None, graph=True):
    g = max(1, tk)
    h = 1.0 / max(n0, n1)
    lam = h * h / 8
    phi0, rho = _fields(n0, n1, g, seed, kind)
    out, norms, _ = run_gpu_solve(n0, n1, h, lam, bc, 0, N, E, phi0, rho, g=g, box=box, nranks=nranks,
                                  graph=graph, tk=tk)
    kern = P.last_solve_kernels()
    ref, rn = _orc(n0, n1, h, lam, bc, N, E, phi0, rho, g=g, b=box)
    check_nan_parity(out, ref[g:-g, g:-g], norms, rn, kind)
    return kern


def _box_kernel(cols, rows):
    """The whole-box kernel px_solve picks (PROTOX_SMALLBOX, read once per
    process: default k_boxw for even widths <= 64 and <= 16 rows (any), <= 32
    (even) or <= 64 (multiple of 4), else the 8-CTA cluster kernel from 16 rows, else k_box1;
    'cluster' skips k_boxw; 'box1' / 'old' force k_box1 / the round-1 one-CTA
    k_smallbox)."""
    mode = os.environ.get("PROTOX_SMALLBOX", "")
    if mode.startswith("b"):
        return "k_box1"
    if mode.startswith("o"):
        return "k_smallbox"
    cl = int(os.environ.get("PROTOX_BOXW_CL", "8"))
    cl = cl if cl in (1, 2, 4, 8) else 8
    fits = lambda r: any(r <= 16 * rw and r % rw == 0 for rw in (1, 2, 4))  # noqa: E731
    while cl > 1 and (rows % cl or not fits(rows // cl)):
        cl //= 2
    boxw = cols % 2 == 0 and cols <= 64 and fits(rows // cl)
    if boxw and not mode.startswith("c"):
        return "k_boxw"
    return "k_cluster_box" if rows >= 16 else "k_box1"


@pytest.mark.parametrize("kind", KINDS)
def test_nan_box_c1(kind):
    """BJ.C1 shape (64², Dirichlet-CC): the whole solve in one launch."""
    assert _box_kernel(64, 64) in _solve_case(64, 64, P.PX_BC_DIRICHLET_CC, 30, 1, kind, 11)


@pytest.mark.parametrize("kind", KINDS)
def test_nan_box_short(kind):
    """A box of < 16 rows, periodic."""
    assert _box_kernel(64, 12) in _solve_case(64, 12, P.PX_BC_PERIODIC, 20, 1, kind, 12)


@pytest.mark.parametrize("mode", ["box1", "old", "cluster", "boxw_cl1", "boxw_cl2", "boxw_cl4", "boxw_nomb"])
def test_box_kernel_variants_subprocess(mode):
    """The other whole-box kernels (k_box1 for every box it fits; the round-1
    one-CTA k_smallbox; the 8-CTA cluster kernel where k_boxw would run;
    k_boxw on one CTA or over a cluster of 2 or 4 CTAs instead of 8, and with
    plain DSMEM stores + a cluster barrier per sweep instead of st.async
    counted on mbarriers) stay
    bit-identical: the small-box parity and NaN tests
    re-run in a child process with PROTOX_SMALLBOX=<mode>."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    extra = {"PROTOX_SMALLBOX": mode}
    if mode.startswith("boxw_cl"):
        extra = {"PROTOX_BOXW_CL": mode[-1]}
    elif mode == "boxw_nomb":
        extra = {"PROTOX_BOXW_MB": "0"}
    env = dict(os.environ, **extra)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-m", "gpu",
                        "tests/test_gpu_nan.py", "tests/test_gpu_parity.py", "-k",
                        "nan_box_c1 or nan_box_short or config1 or test_solve_ragged_multibox or "
                        "norm_every_variants or whole_box"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


@pytest.mark.parametrize("kind", KINDS)
def test_nan_resident(kind):
    """BJ.C2 shape (1024², norm every 10): k_resident (iterate in shared memory)."""
    assert "k_resident" in _solve_case(1024, 1024, P.PX_BC_PERIODIC, 40, 10, kind, 13)


@pytest.mark.parametrize("kind", KINDS)
def test_nan_persist(kind):
    """3.1M cells (too big for shared memory, below the 4M-cell TMA threshold): k_persist."""
    assert "k_persist" in _solve_case(2048, 1536, P.PX_BC_PERIODIC, 6, 1, kind, 14)


@pytest.mark.parametrize("kind", KINDS)
def test_nan_bulk(kind):
    """4M cells, one sweep kernel per sweep: k_bulk (TMA bulk-copy pipeline)."""
    assert "k_bulk" in _solve_case(2048, 2048, P.PX_BC_PERIODIC, 4, 1, kind, 15, box=(256, 256))


@pytest.mark.parametrize("kind", KINDS)
def test_nan_stream_slabs(kind):
    """Three slabs on one device (local transport): k_stream per slab."""
    assert "k_stream" in _solve_case(1000, 300, P.PX_BC_DIRICHLET_CC, 6, 2, kind, 16, nranks=3,
                                     box=(1000, 100))


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("tk", [2, 4])
def test_nan_temporal_blocking(kind, tk):
    """k_tbw (k sweeps per pass): its max uses fmax and recovers NaN from Σr²."""
    assert "k_tb" in _solve_case(1024, 1000, P.PX_BC_PERIODIC, 8, 2, kind, 17 + tk, tk=tk, box=(256, 200))


@pytest.mark.parametrize("kind", KINDS)
def test_nan_temporal_blocking_dirichlet_two_slabs(kind):
    """k_tbw with Dirichlet faces over two slabs on one device (norm slot over two launches)."""
    assert "k_tb" in _solve_case(512, 400, P.PX_BC_DIRICHLET_CC, 8, 4, kind, 21, tk=4, nranks=2,
                                 box=(512, 200))


@pytest.mark.parametrize("kind", KINDS)
def test_nan_nccl_self_exchange(kind, monkeypatch):
    """The multi-GPU code path on one GPU (NCCL self-exchange): boundary rows,
    grouped send/recv, interior, and the batched norm all-reduce -- max as u64
    bit patterns (ncclUint64/ncclMax) -- must keep NaN."""
    monkeypatch.setenv("PROTOX_NCCL_SELF_EXCHANGE", "1")
    n0, n1, N, E = 1024, 768, 6, 1
    h = 1.0 / 1024
    lam = h * h / 8
    phi0, rho = _fields(n0, n1, 1, 23, kind)
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (256, 256), 1, P.PX_BC_PERIODIC, 1)
    comm = P.Comm(P.comm_unique_id(), 1, 0, torch.cuda.current_device())
    try:
        a, b, r = to_device_ghosted(lay, 0, phi0, 1), lay.alloc(0), to_device_ghosted(lay, 0, rho, 1)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        res = P.solve(lay, comm, 0, P.relax_params(h, lam), N, E, lay.patch(0, a), lay.patch(0, b),
                      lay.patch(0, r), use_graph=True, stream=s)
        out = owned_to_host(lay, 0, b if res.in_scratch else a)
    finally:
        comm.close()
    ref, rn = _orc(n0, n1, h, lam, P.PX_BC_PERIODIC, N, E, phi0, rho, b=(256, 256))
    check_nan_parity(out, ref[1:-1, 1:-1], res.norms, rn, kind)


def test_nan_allreduce_norms_single_rank():
    """px_comm_allreduce_norms on one rank keeps NaN and inf in the max ring
    (u64 bit-pattern max) and in the sum ring."""
    comm = P.Comm(P.comm_unique_id(), 1, 0, torch.cuda.current_device())
    try:
        m = torch.tensor([1.0, float("inf"), float("nan"), 0.0], dtype=torch.float64, device="cuda")
        s2 = torch.tensor([2.0, float("inf"), float("nan"), 0.0], dtype=torch.float64, device="cuda")
        P.comm_allreduce_norms(comm, m, s2, 4)
        torch.cuda.synchronize()
        mm, ss = m.cpu().numpy(), s2.cpu().numpy()
        assert mm[0] == 1.0 and mm[1] == np.inf and np.isnan(mm[2]) and mm[3] == 0.0
        assert ss[0] == 2.0 and ss[1] == np.inf and np.isnan(ss[2]) and ss[3] == 0.0
    finally:
        comm.close()


@pytest.mark.parametrize("kind", KINDS)
def test_nan_multigrid(kind):
    """px_mg_solve (relax smoother, restriction, prolongation, coarse K9 solve)."""
    n0 = n1 = 128
    h = 1.0 / 128
    lam = h * h / 8
    phi0, rho = _fields(n0, n1, 1, 25, kind)
    lay = P.Layout(P.box(0, 0, n0 - 1, n1 - 1), (32, 32), 1, P.PX_BC_PERIODIC, 1)
    phi, scr, f = to_device_ghosted(lay, 0, phi0, 1), lay.alloc(0), to_device_ghosted(lay, 0, rho, 1)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    norms = P.mg_solve(lay, P.relax_params(h, lam), 4, 2, lay.patch(0, phi), lay.patch(0, scr), lay.patch(0, f),
                       nu1=2, nu2=2, nu_coarse=8, use_graph=True, stream=s)
    out = lay.view(0, phi).cpu().numpy()
    p = oracle.Problem(n0, n1, h, lam, b0=32, b1=32, ghost=1, bc=BC_MAP[P.PX_BC_PERIODIC], stencil=0)
    ref, rn = oracle.mg_solve(p, oracle.MG(4, 2, 2, 8, 2), phi0, rho)
    out, ref = np.ascontiguousarray(out), np.ascontiguousarray(ref[1:-1, 1:-1])
    mo, mr = np.isnan(out), np.isnan(ref)
    assert mr.any() and np.array_equal(mo, mr)
    assert bits_equal(out[~mo], ref[~mr])
    assert np.array_equal(np.isnan(norms[:, 0]), np.isnan(rn[:, 0])) and np.isnan(rn[-1, 0])
    fin = ~np.isnan(rn[:, 0])
    assert bits_equal(norms[fin, 0], rn[fin, 0])
