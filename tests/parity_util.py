"""Parity measure shared by the GPU parity tests (test infrastructure only)."""
import numpy as np


def rel(a, b):
    """Relative difference of `a` from the oracle value `b`, the LARGER of
    ||a - b||_2 / ||b||_2 and max|a - b| / max|b|.  The elementwise term keeps a
    single wrong entry from hiding in the 2-norm of a large vector (at N = 256 an
    isolated error can be ~800x the RMS-relative tolerance and still pass the
    2-norm alone)."""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    d = a - b
    two = np.linalg.norm(d) / max(np.linalg.norm(b), 1e-300)
    mx = np.abs(d).max() / max(np.abs(b).max(), 1e-300) if d.size else 0.0
    return float(max(two, mx))
