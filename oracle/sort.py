"""Oracle for Alg. 2, "The Truncated FFT Sorting Algorithm".

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Step by step, in the paper's order:
  l. 3-5  P_low^(i) = Trunc_p0(FFT(P^(i)))  for every problem i
          -> `trunc_dft`: the DFT written as its defining sum, evaluated only
             at the kept modes (no FFT), reading R1/R2 of DESIGN.md:
             S[k] = sum_x P[x] exp(-2 pi i <k, x> / p),  k in [-p0/2, p0/2-1]^d,
             x in {0..p-1}^d the integer node index, angle reduced exactly as
             (k_d * x_d mod p).  The sum over x factorises per axis, so it is
             evaluated one axis at a time (same sum, different bracketing).
  l. 6-12 greedy: start at problem 0 (PAPER.md:235, 0-based), repeatedly take
          the unvisited j with the smallest Frobenius distance to the current
          problem, scanning j ascending with strict `<`
          -> `greedy_order`.  Readings: R3 (dis = 1000 read as +inf), R4
             (strict `<` = lowest index wins ties), R5 (compare squared
             distances), R6 (several fields: concatenate the signatures).
"""
from __future__ import annotations

import math
import numpy as np


def dft_matrix(p: int, p0: int) -> np.ndarray:
    """E[k, x] = exp(-2 pi i ((k x) mod p) / p) for k = -p0/2 .. p0/2-1, x = 0..p-1."""
    k = np.arange(-(p0 // 2), p0 - p0 // 2, dtype=np.int64)
    x = np.arange(p, dtype=np.int64)
    r = np.mod(np.outer(k, x), p)                      # exact integer angle reduction
    ang = 2.0 * math.pi * r.astype(np.float64) / p
    return np.cos(ang) - 1j * np.sin(ang)


def trunc_dft(P: np.ndarray, dim: int, p: int, p0: int) -> np.ndarray:
    """Truncated, unnormalised DFT of one field P (x fastest, p^dim values).

    Returns the p0^dim kept coefficients in C order [k_z][k_y][k_x] (complex128).
    """
    if p0 > p or p0 % 2:
        raise ValueError("p0 must be even and <= p")
    E = dft_matrix(p, p0)
    if dim == 2:
        G = P.reshape(p, p)                              # G[y, x]
        S = E @ G @ E.T                                  # S[ky, kx] = sum_y sum_x E[ky,y] G[y,x] E[kx,x]
    elif dim == 3:
        G = P.reshape(p, p, p)                           # G[z, y, x]
        T = G @ E.T                                      # T[z, y, kx]  = sum_x G[z,y,x] E[kx,x]
        T = np.einsum("by,zya->zba", E, T)               # T[z, ky, kx] = sum_y E[ky,y] T[z,y,kx]
        S = np.einsum("cz,zba->cba", E, T)               # S[kz,ky,kx]  = sum_z E[kz,z] T[z,ky,kx]
    else:
        raise ValueError("dim must be 2 or 3")
    return S.reshape(-1)


def signatures(params: np.ndarray, dim: int, p: int, p0: int) -> np.ndarray:
    """params [N, F, p^dim] -> sig [N, F * p0^dim]: fields concatenated (reading R6)."""
    N, F = params.shape[:2]
    out = np.empty((N, F * p0 ** dim), dtype=np.complex128)
    m = p0 ** dim
    for i in range(N):
        for f in range(F):
            out[i, f * m:(f + 1) * m] = trunc_dft(params[i, f], dim, p, p0)
    return out


def pair_d2(sig: np.ndarray) -> np.ndarray:
    """D2[i, j] = ||S_i - S_j||_F^2 as a sum of |differences|^2 (never via ||a||^2+||b||^2-2<a,b>)."""
    N = sig.shape[0]
    D2 = np.empty((N, N))
    for i in range(N):
        d = sig - sig[i]
        D2[i] = (d.real * d.real + d.imag * d.imag).sum(axis=1)
    return D2


def greedy_order(D2: np.ndarray, start: int = 0):
    """Alg. 2 ll. 6-12 on a distance matrix.  Returns (order, best, second).

    best[t] / second[t] are the smallest and runner-up squared distances seen at
    greedy step t+1 (second = inf when only one candidate was left).
    """
    N = D2.shape[0]
    visited = [False] * N
    order = [start]
    visited[start] = True
    cur = start
    best_l, second_l = [], []
    for _ in range(N - 1):
        dis = math.inf                                   # reading R3: "dis = 1000" -> +inf
        second = math.inf
        jmin = -1
        for j in range(N):                               # seq_0 scanned in ascending index
            if visited[j]:
                continue
            dj = D2[cur, j]
            if dj < dis:                                 # strict <
                second = dis
                dis = dj
                jmin = j
            elif dj < second:
                second = dj
        order.append(jmin)
        visited[jmin] = True
        cur = jmin
        best_l.append(dis)
        second_l.append(second)
    return np.array(order, dtype=np.int32), np.array(best_l), np.array(second_l)


def rel_gaps(best: np.ndarray, second: np.ndarray) -> np.ndarray:
    """(second - best) / best per step (0 for exact ties, inf when best == 0 < second)."""
    with np.errstate(divide="ignore", invalid="ignore"):
        g = (second - best) / best
    g = np.where(second == best, 0.0, g)
    return g


def sort_problems(params: np.ndarray, dim: int, p: int, p0: int, start: int = 0):
    """Whole Alg. 2: (order, best_d2, rel_gap, near_tie_steps)."""
    sig = signatures(params, dim, p, p0)
    D2 = pair_d2(sig)
    order, best, second = greedy_order(D2, start)
    gap = rel_gaps(best, second)
    near = np.nonzero(gap < 1e-12)[0]
    return order, best, gap, near
