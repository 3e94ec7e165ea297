"""B200-native (sm_100a, fp64) additive-Vanka monolithic multigrid for Q2-Q1
Taylor-Hood Stokes, after Spies, Olson & MacLachlan (arXiv 2401.06277).

The compute path is the C-ABI library ``libsvk.so`` (include/svk.h, sources in
``csrc/``); ``svk.Solver`` is a thin ctypes binding over it.
"""
from .svk import Solver, SvkError, load_library, LIB_PATH  # noqa: F401

__all__ = ["Solver", "SvkError", "load_library", "LIB_PATH"]
