"""Shared test helpers: move host fields into libprotox patches and back,
and run the oracle on the same seeded inputs."""
from __future__ import annotations

import numpy as np

import oracle
from paper_2307_07931_b200 import protox as P

BC_MAP = {P.PX_BC_PERIODIC: oracle.BC_PERIODIC, P.PX_BC_DIRICHLET_CC: oracle.BC_DIRICHLET_CC,
          P.PX_BC_FIXED_GHOSTS: oracle.BC_FIXED}


def to_device_ghosted(layout: "P.Layout", rank: int, glob: np.ndarray, g: int, device="cuda"):
    """Copy the rank's ghosted window of a global ghosted host array
    (shape (n1+2g, n0+2g)) into a fresh layout tensor."""
    import torch
    t = layout.alloc(rank, device)
    li = layout.local(rank)
    v = layout.view(rank, t, ghosts=True)
    d = layout.domain
    y0 = li.alloc.lo.c[1] - d.lo.c[1] + g
    x0 = li.alloc.lo.c[0] - d.lo.c[0] + g
    win = glob[y0:y0 + v.shape[0], x0:x0 + v.shape[1]]
    v.copy_(torch.from_numpy(np.ascontiguousarray(win)))
    return t


def owned_to_host(layout, rank, t) -> np.ndarray:
    return layout.view(rank, t).cpu().numpy()


def bits_equal(a: np.ndarray, b: np.ndarray) -> bool:
    return np.array_equal(np.ascontiguousarray(a).view(np.uint64), np.ascontiguousarray(b).view(np.uint64))


def ulp_diff(a: np.ndarray, b: np.ndarray) -> int:
    ia = np.ascontiguousarray(a).view(np.int64)
    ib = np.ascontiguousarray(b).view(np.int64)
    return int(np.max(np.abs(ia - ib))) if ia.size else 0


def rel_max(a, b) -> float:
    den = max(float(np.max(np.abs(b))), 1e-300)
    return float(np.max(np.abs(a - b))) / den
