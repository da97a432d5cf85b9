"""paper_1604_02153_b200 — B200-native (sm_100a) GN Hessian-matvec path of the veloreg
registration solver (arXiv 1604.02153), behind the reference's operator/solver API.

libvrg.so (CUDA kernels + C ABI, include/vrg.h) is the product; `api` is the Python host
mirror of the reference API over it.  There is no CPU fallback.
"""
from . import _capi  # noqa: F401

__all__ = ["_capi"]
