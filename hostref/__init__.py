"""The paper's CPU experiment re-run on this host as CONTEXT (SURVEY §8(f)
NEXT rank 4): Proto's unfused abstractions vs the ProtoX fused loop
(figures `Proto`, `ProtoX`, `ProtoXomp`).

Not the product (the CUDA library) and not the oracle; used by
tests/test_hostref_cpu.py and scripts/cpu_fusion_ratio.py only.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "protox_cpu.cpp")
_LIB = os.path.join(_HERE, "libprotox_cpu.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O3", "-march=native", "-fopenmp", "-ffp-contract=off", "-std=c++17",
                               "-fPIC", "-shared", _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


def _L():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        d = ctypes.POINTER(ctypes.c_double)
        i = ctypes.c_int
        _lib.cpu_run.argtypes = [i, i, i, i, i, ctypes.c_double, ctypes.c_double, d, d, d, d]
    return _lib


def run(variant: int, box: int, nboxes: int, iters: int, h: float, lam: float, rho: np.ndarray,
        threads: int = 1):
    """variant 0 = Proto (unfused), 1 = ProtoX (fused).  rho: (n, n), n = nboxes*box.
    Returns (phi, seconds, maxnorm history)."""
    n = nboxes * box
    rho = np.ascontiguousarray(rho, dtype=np.float64)
    assert rho.shape == (n, n)
    out = np.zeros((n, n))
    hist = np.zeros(max(iters, 1))
    sec = ctypes.c_double(0)
    dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    rc = _L().cpu_run(variant, box, nboxes, iters, threads, h, lam, dp(rho), dp(out), ctypes.byref(sec), dp(hist))
    if rc != 0:
        raise ValueError("bad arguments")
    return out, sec.value, hist[:iters]
