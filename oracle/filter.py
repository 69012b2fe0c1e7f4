"""Oracle for Alg. 1, "Chebyshev Filter" — TEST INFRASTRUCTURE ONLY.

Followed line by line with a uniform degree for every column (R8;
the staggered `Y_{i+1,1:m-1} = Y_{i,1:m-1}` of l. 5 is the per-vector-degree
variant, not built):

  l. 1  A~ = (A - c I)/e,  sigma_1 = e / (lambda - c)
  l. 2  Y_1 = sigma_1 A~ Y_0
  l. 3  for i = 1 .. m-1:
  l. 4     sigma_{i+1} = 1 / (2/sigma_1 - sigma_i)
  l. 5     Y_{i+1} = 2 sigma_{i+1} A~ Y_i - sigma_{i+1} sigma_i Y_{i-1}

Pinned (tests/test_oracle_filter.py) by the closed form on exact eigenvectors:
Y_m = rho_m(t) v with rho_m(t) = C_m((t-c)/e) / C_m((lambda-c)/e).
"""
from __future__ import annotations

import numpy as np


def cheb_filter(A, Y0: np.ndarray, m: int, lam: float, c: float, e: float) -> np.ndarray:
    """A: anything supporting A @ Y (sparse/dense n x n); Y0: n x k."""
    def At(Y):                       # A~ Y = (A Y - c Y) / e
        return (A @ Y - c * Y) / e
    sigma1 = e / (lam - c)
    Y_prev = Y0
    Y = sigma1 * At(Y0)
    sigma = sigma1
    for _ in range(1, m):
        sigma_next = 1.0 / (2.0 / sigma1 - sigma)
        Y_next = 2.0 * sigma_next * At(Y) - sigma_next * sigma * Y_prev
        Y_prev, Y = Y, Y_next
        sigma = sigma_next
    return Y


def cheb_T(m: int, x: np.ndarray) -> np.ndarray:
    """Chebyshev polynomial of the first kind C_m(x) = cos(m arccos x) extended to |x| > 1."""
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    a = np.abs(x) <= 1
    out[a] = np.cos(m * np.arccos(x[a]))
    hi = x > 1
    out[hi] = np.cosh(m * np.arccosh(x[hi]))
    lo = x < -1
    out[lo] = (-1) ** m * np.cosh(m * np.arccosh(-x[lo]))
    return out
