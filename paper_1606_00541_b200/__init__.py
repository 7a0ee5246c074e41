"""hecsolve-b200: the level-scheduled HEC triangular solve of arXiv 1606.00541
rebuilt for NVIDIA B200 (sm_100a).

The product is ``libhecsolve_b200.so`` (C++ host setup + CUDA kernels + the
C-ABI of ``include/hecsolve_c.h``); this package is its Python face, mirroring
the reference's API names (see ``api``).
"""
from .api import *  # noqa: F401,F403
from .api import (CsrMatrix, DevicePrecond, DeviceSpmv, DeviceTri, HecError, ZeroPivotError,  # noqa: F401
                  apply, build_preconditioner, gmres, prepare_lower, prepare_upper, solve)
from ._lib import LIB_PATH, STRATEGY_AUTO, STRATEGY_LEVELS, STRATEGY_PIPELINE  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
