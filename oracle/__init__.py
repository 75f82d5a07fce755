"""CPU oracle for the ProtoX 2D Poisson point-Jacobi relaxation.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this package.  The product library (``paper_2307_07931_b200``) never imports
it, and the two share no code: this wrapper marshals numpy arrays into the
single-threaded C++ oracle ``protox_oracle.cpp`` (see its header for the
paper passages each function follows).

Array convention: a *global ghosted array* of a problem with domain n0 x n1 and
ghost width g is a numpy float64 array of shape (n1 + 2g, n0 + 2g); element
[y + g, x + g] is cell (x, y) (x = dimension 0, fastest in memory, as fixed by
the index arithmetic of Fig. ProtoX).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "protox_oracle.cpp")
_SRC3 = os.path.join(_HERE, "protox_oracle3d.cpp")
_LIB = os.path.join(_HERE, "liborc.so")

BC_PERIODIC, BC_DIRICHLET_CC, BC_FIXED = 0, 1, 2
ST_LAPLACE5, ST_MEHRSTELLEN9 = 0, 1

_CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c++17", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the oracle with g++ (plain -O2, -ffp-contract=off)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(os.path.getmtime(_SRC),
                                                                          os.path.getmtime(_SRC3)):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", *_CFLAGS, _SRC, _SRC3, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


class _Problem(ctypes.Structure):
    _fields_ = [
        ("n0", ctypes.c_int64), ("n1", ctypes.c_int64),
        ("b0", ctypes.c_int64), ("b1", ctypes.c_int64),
        ("ghost", ctypes.c_int32), ("bc", ctypes.c_int32),
        ("stencil", ctypes.c_int32), ("rhs_correction", ctypes.c_int32),
        ("h", ctypes.c_double), ("lam", ctypes.c_double),
        ("nsweeps", ctypes.c_int64), ("norm_every", ctypes.c_int64),
    ]


class _Problem3(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64 * 3), ("b", ctypes.c_int64 * 3),
        ("ghost", ctypes.c_int32), ("bc", ctypes.c_int32),
        ("stencil", ctypes.c_int32), ("rhs_correction", ctypes.c_int32),
        ("h", ctypes.c_double), ("lam", ctypes.c_double),
        ("nsweeps", ctypes.c_int64), ("norm_every", ctypes.c_int64),
    ]


class _MG(ctypes.Structure):
    _fields_ = [("levels", ctypes.c_int64), ("nu1", ctypes.c_int64), ("nu2", ctypes.c_int64),
                ("nu_coarse", ctypes.c_int64), ("ncycles", ctypes.c_int64)]


_lib = None


def _L():
    global _lib
    if _lib is None:
        # PROTOX_ORACLE_LIB: a mutated build for scripts/oracle_mutation_check.py
        _lib = ctypes.CDLL(os.environ.get("PROTOX_ORACLE_LIB") or build())
        d = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        P = ctypes.POINTER(_Problem)
        _lib.orc_last_error.restype = ctypes.c_char_p
        _lib.orc_solve.argtypes = [P, d, d, d, d, i64, ctypes.POINTER(i64)]
        _lib.orc_apply_laplacian.argtypes = [P, d, d]
        _lib.orc_residual.argtypes = [P, d, d, d]
        _lib.orc_rhs.argtypes = [P, d, d]
        _lib.orc_exchange.argtypes = [P, d]
        _lib.orc_exchange_box.argtypes = [P, d, i64, d]
        _lib.orc_apply_taps.argtypes = [i64, ctypes.POINTER(i64), d, ctypes.c_double, d,
                                        i64, i64, i64, i64, i64, i64, i64, i64, d]
        _lib.orc_stencil_taps.argtypes = [ctypes.c_int32, ctypes.c_double,
                                          ctypes.POINTER(i64), d, d]
        _lib.orc_stencil_taps.restype = i64
        _lib.orc_box_ordinal.argtypes = [i64] * 6
        _lib.orc_box_ordinal.restype = i64
        _lib.orc_mg_solve.argtypes = [P, ctypes.POINTER(_MG), d, d, d, d, i64, ctypes.POINTER(i64)]
        _lib.orc_mg_restrict.argtypes = [i64, i64, d, d]
        _lib.orc_mg_prolong.argtypes = [i64, i64, ctypes.c_int32, d, d]
        _lib.orc_neumaier_sum.argtypes = [d, i64]
        _lib.orc_neumaier_sum.restype = ctypes.c_double
        P3 = ctypes.POINTER(_Problem3)
        _lib.orc3_last_error.restype = ctypes.c_char_p
        _lib.orc3_solve.argtypes = [P3, d, d, d, d, i64, ctypes.POINTER(i64)]
        _lib.orc3_apply_laplacian.argtypes = [P3, d, d]
        _lib.orc3_exchange.argtypes = [P3, d]
        _lib.orc3_rhs.argtypes = [P3, d, d]
    return _lib


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class OracleError(RuntimeError):
    pass


def _check(rc: int):
    if rc != 0:
        raise OracleError(_L().orc_last_error().decode())


@dataclass
class Problem:
    """A relaxation problem (domain n0 x n1 split into b0 x b1 boxes)."""
    n0: int
    n1: int
    h: float
    lam: float
    b0: int | None = None
    b1: int | None = None
    ghost: int = 1
    bc: int = BC_PERIODIC
    stencil: int = ST_LAPLACE5
    rhs_correction: bool = False
    nsweeps: int = 0
    norm_every: int = 0

    def c(self) -> _Problem:
        return _Problem(self.n0, self.n1, self.b0 or self.n0, self.b1 or self.n1,
                        self.ghost, self.bc, self.stencil, int(self.rhs_correction),
                        self.h, self.lam, self.nsweeps, self.norm_every)

    @property
    def gshape(self):
        return (self.n1 + 2 * self.ghost, self.n0 + 2 * self.ghost)

    def n_norms(self) -> int:
        if self.norm_every < 0:
            return 0
        k = 0
        if self.norm_every > 0:
            k = (self.nsweeps + self.norm_every - 1) // self.norm_every
        return k + 1


def ghosted(p: Problem, interior: np.ndarray, ghost_values: float | np.ndarray = 0.0) -> np.ndarray:
    """Embed an (n1, n0) interior array into a global ghosted array."""
    g = p.ghost
    out = np.empty(p.gshape, dtype=np.float64)
    out[...] = ghost_values
    out[g:g + p.n1, g:g + p.n0] = interior
    return out


def solve(p: Problem, phi0_g: np.ndarray, rho_g: np.ndarray):
    """Run p.nsweeps iterations of figure `Proto`.  Returns (phi_g, norms)
    where norms[j] = (max|r|, sum r^2) of phi^(j*E) for j*E < N, then of phi^N."""
    phi0_g = np.ascontiguousarray(phi0_g, dtype=np.float64)
    rho_g = np.ascontiguousarray(rho_g, dtype=np.float64)
    assert phi0_g.shape == p.gshape and rho_g.shape == p.gshape
    out = np.zeros(p.gshape, dtype=np.float64)
    cap = max(p.n_norms(), 1)
    norms = np.zeros((cap, 2), dtype=np.float64)
    nw = ctypes.c_int64(0)
    pc = p.c()
    _check(_L().orc_solve(ctypes.byref(pc), _dp(phi0_g), _dp(rho_g), _dp(out), _dp(norms), cap,
                          ctypes.byref(nw)))
    return out, norms[: nw.value]


def apply_laplacian(p: Problem, phi_g: np.ndarray) -> np.ndarray:
    """Δ_h φ on the interior (after the boundary exchange)."""
    phi_g = np.ascontiguousarray(phi_g, dtype=np.float64)
    out = np.zeros((p.n1, p.n0), dtype=np.float64)
    pc = p.c()
    _check(_L().orc_apply_laplacian(ctypes.byref(pc), _dp(phi_g), _dp(out)))
    return out


def residual(p: Problem, phi_g: np.ndarray, rho_g: np.ndarray) -> tuple[float, float]:
    phi_g = np.ascontiguousarray(phi_g, dtype=np.float64)
    rho_g = np.ascontiguousarray(rho_g, dtype=np.float64)
    out = np.zeros(2, dtype=np.float64)
    pc = p.c()
    _check(_L().orc_residual(ctypes.byref(pc), _dp(phi_g), _dp(rho_g), _dp(out)))
    return float(out[0]), float(out[1])


def rhs(p: Problem, rho_g: np.ndarray) -> np.ndarray:
    rho_g = np.ascontiguousarray(rho_g, dtype=np.float64)
    out = np.zeros((p.n1, p.n0), dtype=np.float64)
    pc = p.c()
    _check(_L().orc_rhs(ctypes.byref(pc), _dp(rho_g), _dp(out)))
    return out


def exchange(p: Problem, glob: np.ndarray) -> np.ndarray:
    g = np.array(glob, dtype=np.float64, order="C", copy=True)
    pc = p.c()
    _check(_L().orc_exchange(ctypes.byref(pc), _dp(g)))
    return g


def exchange_box(p: Problem, glob: np.ndarray, ib: int) -> np.ndarray:
    glob = np.ascontiguousarray(glob, dtype=np.float64)
    b0, b1, g = p.b0 or p.n0, p.b1 or p.n1, p.ghost
    out = np.zeros((b1 + 2 * g, b0 + 2 * g), dtype=np.float64)
    pc = p.c()
    _check(_L().orc_exchange_box(ctypes.byref(pc), _dp(glob), ib, _dp(out)))
    return out


def apply_taps(offs, alpha, scale, src: np.ndarray, src_lo, dest_lo, dest_hi) -> np.ndarray:
    """Eq.1 on one box: src has shape (ny, nx) over box [src_lo, src_lo+(nx-1,ny-1)]."""
    src = np.ascontiguousarray(src, dtype=np.float64)
    offs_a = np.ascontiguousarray(np.asarray(offs, dtype=np.int64).reshape(-1))
    alpha_a = np.ascontiguousarray(np.asarray(alpha, dtype=np.float64))
    ny, nx = src.shape
    dny, dnx = dest_hi[1] - dest_lo[1] + 1, dest_hi[0] - dest_lo[0] + 1
    out = np.zeros((dny, dnx), dtype=np.float64)
    _check(_L().orc_apply_taps(len(alpha_a), offs_a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                               _dp(alpha_a), scale, _dp(src), src_lo[0], src_lo[1],
                               src_lo[0] + nx - 1, src_lo[1] + ny - 1, dest_lo[0], dest_lo[1],
                               dest_hi[0], dest_hi[1], _dp(out)))
    return out


def stencil_taps(kind: int, h: float):
    offs = np.zeros(32, dtype=np.int64)
    alpha = np.zeros(16, dtype=np.float64)
    scale = ctypes.c_double(0)
    n = _L().orc_stencil_taps(kind, h, offs.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                              _dp(alpha), ctypes.byref(scale))
    return offs[: 2 * n].reshape(n, 2).copy(), alpha[:n].copy(), scale.value


def box_ordinal(lo, hi, p) -> int:
    return int(_L().orc_box_ordinal(lo[0], lo[1], hi[0], hi[1], p[0], p[1]))


def neumaier_sum(x: np.ndarray) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
    return float(_L().orc_neumaier_sum(_dp(x), x.size))


# --------------------------------------------------------------- multigrid
@dataclass
class MG:
    """V(nu1, nu2)-cycle options (readings R-MG1..R-MG6)."""
    levels: int
    nu1: int = 2
    nu2: int = 2
    nu_coarse: int = 4
    ncycles: int = 1


def mg_solve(p: Problem, m: MG, phi0_g: np.ndarray, rho_g: np.ndarray):
    """m.ncycles V-cycles.  Returns (phi_g, norms) with norms[k] = (max|r|,
    sum r^2) of the finest iterate after k cycles, k = 0..ncycles."""
    phi0_g = np.ascontiguousarray(phi0_g, dtype=np.float64)
    rho_g = np.ascontiguousarray(rho_g, dtype=np.float64)
    assert phi0_g.shape == p.gshape and rho_g.shape == p.gshape
    out = np.zeros(p.gshape, dtype=np.float64)
    norms = np.zeros((m.ncycles + 1, 2), dtype=np.float64)
    nw = ctypes.c_int64(0)
    pc, mc = p.c(), _MG(m.levels, m.nu1, m.nu2, m.nu_coarse, m.ncycles)
    _check(_L().orc_mg_solve(ctypes.byref(pc), ctypes.byref(mc), _dp(phi0_g), _dp(rho_g), _dp(out),
                             _dp(norms), m.ncycles + 1, ctypes.byref(nw)))
    return out, norms[: nw.value]


def mg_restrict(d: np.ndarray) -> np.ndarray:
    """-R d: minus the 2x2 average of a fine (n1, n0) array."""
    d = np.ascontiguousarray(d, dtype=np.float64)
    n1, n0 = d.shape
    out = np.zeros((n1 // 2, n0 // 2), dtype=np.float64)
    _check(_L().orc_mg_restrict(n0, n1, _dp(d), _dp(out)))
    return out


def mg_prolong(e: np.ndarray, fine: np.ndarray, bc: int) -> np.ndarray:
    """fine + P e (cell-centred bilinear, coarse ghosts by the rule bc)."""
    e = np.ascontiguousarray(e, dtype=np.float64)
    f = np.array(fine, dtype=np.float64, order="C", copy=True)
    nc1, nc0 = e.shape
    assert f.shape == (2 * nc1, 2 * nc0)
    _check(_L().orc_mg_prolong(nc0, nc1, bc, _dp(e), _dp(f)))
    return f


# ------------------------------------------------------------------------ 3D
# (protox_oracle3d.cpp, readings R-3D1..R-3D3)
# A global ghosted 3D array has shape (n2 + 2g, n1 + 2g, n0 + 2g); element
# [z + g, y + g, x + g] is cell (x, y, z) (dimension 0 fastest in memory).

def _check3(rc: int):
    if rc != 0:
        raise OracleError(_L().orc3_last_error().decode())


@dataclass
class Problem3:
    """3D relaxation problem: domain n = (n0, n1, n2) split into boxes b."""
    n: tuple
    h: float
    lam: float
    b: tuple | None = None
    ghost: int = 1
    bc: int = BC_PERIODIC
    nsweeps: int = 0
    norm_every: int = 0
    stencil: int = 0            # 0 = 7-point, 1 = 27-point Mehrstellen
    rhs_correction: bool = False

    def c(self) -> _Problem3:
        b = self.b or self.n
        return _Problem3((ctypes.c_int64 * 3)(*self.n), (ctypes.c_int64 * 3)(*b), self.ghost, self.bc,
                         self.stencil, int(self.rhs_correction), self.h, self.lam, self.nsweeps,
                         self.norm_every)

    @property
    def gshape(self):
        g = self.ghost
        return (self.n[2] + 2 * g, self.n[1] + 2 * g, self.n[0] + 2 * g)

    def n_norms(self) -> int:
        if self.norm_every < 0:
            return 0
        k = (self.nsweeps + self.norm_every - 1) // self.norm_every if self.norm_every > 0 else 0
        return k + 1


def ghosted3(p: Problem3, interior: np.ndarray, ghost_values: float | np.ndarray = 0.0) -> np.ndarray:
    g = p.ghost
    out = np.empty(p.gshape, dtype=np.float64)
    out[...] = ghost_values
    out[g:g + p.n[2], g:g + p.n[1], g:g + p.n[0]] = interior
    return out


def solve3(p: Problem3, phi0_g: np.ndarray, rho_g: np.ndarray):
    """p.nsweeps iterations of figure `Proto` in 3D.  Returns (phi_g, norms)."""
    phi0_g = np.ascontiguousarray(phi0_g, dtype=np.float64)
    rho_g = np.ascontiguousarray(rho_g, dtype=np.float64)
    assert phi0_g.shape == p.gshape and rho_g.shape == p.gshape
    out = np.zeros(p.gshape, dtype=np.float64)
    cap = max(p.n_norms(), 1)
    norms = np.zeros((cap, 2), dtype=np.float64)
    nw = ctypes.c_int64(0)
    pc = p.c()
    _check3(_L().orc3_solve(ctypes.byref(pc), _dp(phi0_g), _dp(rho_g), _dp(out), _dp(norms), cap,
                            ctypes.byref(nw)))
    return out, norms[: nw.value]


def apply_laplacian3(p: Problem3, phi_g: np.ndarray) -> np.ndarray:
    phi_g = np.ascontiguousarray(phi_g, dtype=np.float64)
    out = np.zeros((p.n[2], p.n[1], p.n[0]), dtype=np.float64)
    pc = p.c()
    _check3(_L().orc3_apply_laplacian(ctypes.byref(pc), _dp(phi_g), _dp(out)))
    return out


def exchange3(p: Problem3, glob: np.ndarray) -> np.ndarray:
    g = np.array(glob, dtype=np.float64, order="C", copy=True)
    pc = p.c()
    _check3(_L().orc3_exchange(ctypes.byref(pc), _dp(g)))
    return g


def rhs3(p: Problem3, rho_g: np.ndarray) -> np.ndarray:
    """The right-hand side the 3D solve uses: ρ, or ρ + S7(ρ)/12 (27-point with correction)."""
    rho_g = np.ascontiguousarray(rho_g, dtype=np.float64)
    out = np.zeros((p.n[2], p.n[1], p.n[0]), dtype=np.float64)
    pc = p.c()
    _check3(_L().orc3_rhs(ctypes.byref(pc), _dp(rho_g), _dp(out)))
    return out
