"""libprotox: B200-native fused 2D Poisson point-Jacobi relaxation (ProtoX,
arXiv 2307.07931).  The C-ABI library is ``libprotox.so`` (header
``include/protox.h``); ``paper_2307_07931_b200.protox`` is the thin ctypes
binding with the same names.  Import the binding explicitly:

    from paper_2307_07931_b200 import protox
"""
__all__ = ["protox", "inputs"]
