"""B200-native MPM hot path of CRESSim-MPM (arxiv 2502.18437).

The product is ``libmpm_b200.so`` (sm_100a kernels + C++ engine behind the C-ABI of
``include/mpm_b200.h``).  This package holds its ctypes mirror (``capi``), the Python
mirror of the reference's solver / scene API (``api``) and the benchmark / parity scene
specifications (``scenes``).  Nothing here computes physics on the CPU.
"""
from . import capi  # noqa: F401

__all__ = ["capi", "api", "scenes"]
