"""Oracle for the result of the solve: the L eigenpairs of smallest |lambda|.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

SCSF "is purely an acceleration technique and does not alter the solution
results"; the problem is A^(i) v_j = lambda_j v_j, j = 1..L,
|lambda_1| <= ... <= |lambda_L|.  So the oracle computes
that plain definition for each operator independently of sort order, chain
and warm start.  Every configuration is SPD (R20), so "smallest
|lambda|" = algebraically smallest.

  jacobi_eigh        cyclic Jacobi (textbook two-sided, row-cyclic order,
                     Rutishauser's stable 2x2 rotation), for tiny dense A.
  smallest_eigpairs  shift-invert block Lanczos: A = U^T U by banded Cholesky
                     (LAPACK dpbtrf through scipy, a library primitive), block
                     Lanczos with full reorthogonalisation on A^{-1}, block
                     size 8 so (near-)degenerate eigenvalues are captured;
                     the small projected matrix is diagonalised by numpy.eigh
                     (library primitive); Ritz pairs are accepted on the TRUE
                     residual ||A v - lambda v|| computed with A itself, and
                     the function RAISES (OracleNotConverged) rather than
                     return a pair above that bound.
"""
from __future__ import annotations

import math
import numpy as np
import scipy.linalg as sla

from . import operator as op


def jacobi_eigh(A: np.ndarray, tol: float = 1e-15, max_sweeps: int = 100):
    """Cyclic Jacobi: returns (ascending eigenvalues, eigenvectors as columns, sweeps)."""
    A = np.array(A, dtype=np.float64, copy=True)
    n = A.shape[0]
    V = np.eye(n)
    normF = np.linalg.norm(A)
    sweeps = 0
    for sweeps in range(1, max_sweeps + 1):
        off = float(np.linalg.norm(A - np.diag(np.diag(A))))   # direct, no cancellation
        if off <= tol * normF:
            sweeps -= 1
            break
        for p in range(n - 1):
            for q in range(p + 1, n):
                apq = A[p, q]
                if apq == 0.0:
                    continue
                theta = (A[q, q] - A[p, p]) / (2.0 * apq)
                t = math.copysign(1.0, theta) / (abs(theta) + math.sqrt(1.0 + theta * theta))
                c = 1.0 / math.sqrt(1.0 + t * t)
                s = t * c
                # A <- J^T A J with J = rotation in the (p, q) plane
                ap = A[:, p].copy()
                aq = A[:, q].copy()
                A[:, p] = c * ap - s * aq
                A[:, q] = s * ap + c * aq
                ap = A[p, :].copy()
                aq = A[q, :].copy()
                A[p, :] = c * ap - s * aq
                A[q, :] = s * ap + c * aq
                A[p, q] = A[q, p] = 0.0
                vp = V[:, p].copy()
                vq = V[:, q].copy()
                V[:, p] = c * vp - s * vq
                V[:, q] = s * vp + c * vq
    w = np.diag(A).copy()
    idx = np.argsort(w, kind="stable")
    return w[idx], V[:, idx], sweeps


class OracleNotConverged(RuntimeError):
    """smallest_eigpairs hit its Krylov cap before every wanted pair met its residual bound."""


class SolveResult:
    def __init__(self, lam, V, resid, krylov_dim, normA):
        self.lam = lam              # ascending
        self.V = V                  # n x k orthonormal
        self.resid = resid          # ||A v - lam v||_2 per pair
        self.krylov_dim = krylov_dim
        self.normA = normA          # ||A||_inf


def smallest_eigpairs(fields, i, k: int, block: int = 8, seed: int = 7,
                      rtol: float = 1e-12, floor_rel: float = 2e-14, max_dim: int | None = None):
    """k smallest eigenpairs of SPD A^(i) by shift-invert block Lanczos.

    A pair is accepted when ||A v - lam v|| <= max(rtol*|lam|, floor_rel*||A||_inf);
    the floor is the fp64 limit of forming A v (about eps*||A||).
    """
    A = op.assemble_csr(fields, i)
    n = A.shape[0]
    normA = float(np.abs(A).sum(axis=1).max())
    if n <= 64 or k >= n // 2:
        lam, V, _ = jacobi_eigh(A.toarray())
        V = V[:, :k]
        lam = lam[:k]
        R = A @ V - V * lam
        return SolveResult(lam, V, np.linalg.norm(R, axis=0), n, normA)
    ab, _ = op.banded_upper(fields, i)
    U = sla.cholesky_banded(ab, lower=False)

    def solve(X):
        return sla.cho_solve_banded((U, False), X)

    max_dim = max_dim or min(n, 12 * k + 8 * block)
    rng = np.random.default_rng(seed)
    X, _ = np.linalg.qr(rng.standard_normal((n, block)))
    Qbuf = np.empty((n, max_dim + block))     # orthonormal Krylov blocks of A^{-1}, side by side
    Qbuf[:, :block] = X
    Q = lambda jj: Qbuf[:, jj * block:(jj + 1) * block]
    Tblocks = {}                              # (j, j) diagonal and (j+1, j) subdiagonal blocks
    Bprev = None
    check_every = max(1, (k // block) // 4)
    j = 0
    while True:
        W = solve(Q(j))
        if j > 0:
            W = W - Q(j - 1) @ Bprev.T
        Aj = Q(j).T @ W
        Aj = 0.5 * (Aj + Aj.T)
        Tblocks[(j, j)] = Aj
        W = W - Q(j) @ Aj
        Qall = Qbuf[:, :(j + 1) * block]
        for _ in range(2):                    # full reorthogonalisation, twice
            W = W - Qall @ (Qall.T @ W)
        Xn, Bj = np.linalg.qr(W)
        Tblocks[(j + 1, j)] = Bj
        Bprev = Bj
        m = (j + 1) * block
        done = m + block > max_dim
        if (m >= k + block and (j % check_every == 0)) or done:
            T = np.zeros((m, m))
            for jj in range(j + 1):
                T[jj * block:(jj + 1) * block, jj * block:(jj + 1) * block] = Tblocks[(jj, jj)]
                if jj > 0:
                    Bt = Tblocks[(jj, jj - 1)]
                    T[jj * block:(jj + 1) * block, (jj - 1) * block:jj * block] = Bt
                    T[(jj - 1) * block:jj * block, jj * block:(jj + 1) * block] = Bt.T
            mu, S = np.linalg.eigh(T)         # eigenvalues of A^{-1} on the Krylov space
            order = np.argsort(-mu)[:k]       # largest mu <-> smallest lambda = 1/mu
            Vk = Qall @ S[:, order]
            # Rayleigh quotients with A itself (more accurate than 1/mu)
            AV = A @ Vk
            lam = np.einsum("ij,ij->j", Vk, AV)
            R = AV - Vk * lam
            res = np.linalg.norm(R, axis=0)
            tol = np.maximum(rtol * np.abs(lam), floor_rel * normA)
            if np.all(res <= tol):
                idx = np.argsort(lam, kind="stable")
                return SolveResult(lam[idx], Vk[:, idx], res[idx], m, normA)
            if done:
                # never hand back unconverged pairs as the reference
                bad = int(np.sum(res > tol))
                raise OracleNotConverged(
                    f"operator {i}: {bad} of {k} pairs above max({rtol:g} |lam|, {floor_rel:g} ||A||) "
                    f"at Krylov dimension {m} (worst ||r|| / bound = {float(np.max(res / tol)):.3e})")
        Qbuf[:, (j + 1) * block:(j + 2) * block] = Xn
        j += 1
