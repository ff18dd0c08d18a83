"""B200-native dual-gradient hot path for ridge-regularised dual ascent on matching LPs.

The compute lives in ``lib/libdualip.so`` (C ABI in ``include/dualip.h``, CUDA for
sm_100a).  ``_lib`` is the ctypes binding (same names as the C entry points) and
``problem.MatchingProblem`` a small owner of one ``dl_problem`` handle built
from torch CUDA tensors.  Importing this package loads the library; if it is not
built the import fails (no CPU fallback).
"""
from . import _lib  # noqa: F401  (loads libdualip.so or raises)
from ._lib import (DL_GRAD_PARTIAL, DL_PROJ_BOX, DL_PROJ_BOXCUT, DL_PROJ_SIMPLEX,  # noqa: F401
                   DualipError, HISTORY_DTYPE)
from .problem import MatchingProblem  # noqa: F401

__all__ = ["MatchingProblem", "DualipError", "DL_PROJ_SIMPLEX", "DL_PROJ_BOXCUT", "DL_PROJ_BOX",
           "DL_GRAD_PARTIAL", "HISTORY_DTYPE"]
