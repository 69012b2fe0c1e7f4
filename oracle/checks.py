"""Checks applied to any returned eigenpairs (GPU or oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

  rel_residual      the paper's metric ||A v - lam v||_2 / ||A v||_2
  resid_over_normA  the north-star metric ||A v - lam v||_2 / ||A||_inf (BASELINE.json)
  orth_error        max |V^T V - I|
  clusters          maximal runs of eigenvalues with relative gap < rel (R21)
  subspace_sine     ||(I - U U^T) V||_2  (direct sine, not sqrt(1 - cos^2))
  inertia_below     Sylvester inertia: #eigenvalues of A below sigma, counted as
                    the negative pivots of a no-pivot banded LDL^T of A - sigma I
  inertia_blocks    the same count by block Gaussian elimination over the grid's
                    block-tridiagonal structure (blocks of u = largest stencil
                    stride unknowns): inertia(A - sigma I) = sum_i inertia(S_i),
                    S_0 = D_0 - sigma I, S_i = D_i - sigma I - E_i S_{i-1}^{-1} E_i^T
                    (Haynsworth inertia additivity of the Schur complement); each
                    S_i's count from a Bunch-Kaufman LDL^T (scipy.linalg.ldl, a
                    library primitive).  Used for O8 at C3-C5 sizes.
  loewner_bounds    a_min lam_j(L0) + c_min <= lam_j(A) <= a_max lam_j(L0) + c_max
                    (Courant-Fischer; flux form is monotone in the face coefficients)
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from . import operator as op


def rel_residual(A, lam, V):
    AV = A @ V
    R = AV - V * lam
    return np.linalg.norm(R, axis=0) / np.linalg.norm(AV, axis=0)


def resid_over_normA(A, lam, V, normA):
    R = A @ V - V * lam
    return np.linalg.norm(R, axis=0) / normA


def orth_error(V):
    G = V.T @ V
    return float(np.abs(G - np.eye(G.shape[0])).max())


def clusters(lam, rel: float = 1e-3):
    """List of (start, stop) index ranges; consecutive lam closer than rel*|lam| share a cluster."""
    lam = np.asarray(lam)
    out = []
    s = 0
    for j in range(1, len(lam) + 1):
        if j == len(lam) or (lam[j] - lam[j - 1]) > rel * max(abs(lam[j]), abs(lam[j - 1])):
            out.append((s, j))
            s = j
    return out


def subspace_sine(U, V):
    """Largest principal-angle sine of span(V) against span(U) (U orthonormal)."""
    R = V - U @ (U.T @ V)
    return float(np.linalg.norm(R, 2))


def compare_pairs(lam_ref, U_ref, lam, V, L, rel_cluster: float = 1e-3):
    """Compare L returned pairs against a reference with >= L (+guard) pairs.

    Returns (max relative eigenvalue error, max cluster subspace sine).  A cluster
    that straddles index L is checked one-sided: the returned part must lie in the
    span of the reference's whole cluster.
    """
    lam_ref = np.asarray(lam_ref)
    ev_err = float(np.max(np.abs(lam[:L] - lam_ref[:L]) / np.abs(lam_ref[:L])))
    worst = 0.0
    for (s, e) in clusters(lam_ref, rel_cluster):
        if s >= L:
            break
        # one-sided when the cluster straddles L: V's part must lie in the whole reference cluster
        worst = max(worst, subspace_sine(U_ref[:, s:e], V[:, s:min(e, L)]))
    return ev_err, worst


def inertia_below(fields, i, sigma: float) -> int:
    """Number of eigenvalues of A^(i) below sigma (negative pivots of LDL^T of A - sigma I).

    No pivoting.  The (u+1)x(u+1) window W holds rows/cols k..k+u of the partially
    eliminated matrix: row r = k+u+1 enters untouched, because every earlier pivot
    p <= k only updates rows p+1..p+u.  The matrix is padded past n with unit pivots.
    """
    ab, u = op.banded_upper(fields, i)               # ab[u + r - c, c] = A[r, c], r <= c
    n = ab.shape[1]
    assert n > u
    W = np.zeros((u + 1, u + 1))
    for c in range(u + 1):
        col = ab[u - c:, c]                          # A[0..c, c]
        W[:c + 1, c] = col
        W[c, :c + 1] = col
    W[np.arange(u + 1), np.arange(u + 1)] -= sigma
    neg = 0
    for k in range(n):
        d = W[0, 0]
        if d == 0.0:
            raise ZeroDivisionError("zero pivot; perturb sigma")
        if d < 0.0:
            neg += 1
        l = W[0, 1:].copy()
        W[:u, :u] = W[1:, 1:] - np.outer(l, l) / d
        r = k + u + 1
        if r < n:
            vals = ab[:, r].copy()                   # A[k+1 .. r, r]
            vals[u] -= sigma
        else:
            vals = np.zeros(u + 1)
            vals[u] = 1.0
        W[u, :] = vals
        W[:, u] = vals
    return neg


def _negative_count(S: np.ndarray) -> int:
    """#negative eigenvalues of dense symmetric S from its LDL^T (Sylvester: inertia(S) = inertia(D))."""
    _, d, _ = sla.ldl(S, lower=True)
    # D is block diagonal with 1x1 and 2x2 blocks: a symmetric tridiagonal matrix
    w = sla.eigvalsh_tridiagonal(np.diag(d).copy(), np.diag(d, -1).copy())
    return int(np.sum(w < 0.0))


def inertia_blocks(fields, i, sigma: float) -> int:
    """Number of eigenvalues of A^(i) below sigma by block LDL^T of A - sigma I.

    With u = the largest stencil stride, A couples unknowns at most u apart, so in
    consecutive blocks of u unknowns A is block tridiagonal (diagonal blocks D_i,
    sub-diagonal blocks E_i = A[block i, block i-1]).  Block elimination without
    block pivoting gives A - sigma I = L diag(S_0, S_1, ...) L^T, so by Sylvester's
    law of inertia the count is the sum of the negative counts of the S_i.
    """
    A = op.assemble_csr(fields, i)
    n = A.shape[0]
    u = op.strides(fields)[-1]
    S_prev = None
    neg = 0
    for r0 in range(0, n, u):
        r1 = min(n, r0 + u)
        S = A[r0:r1, r0:r1].toarray() - sigma * np.eye(r1 - r0)
        if S_prev is not None:
            E = A[r0:r1, r0 - u:r0].toarray()           # rows of this block, columns of the previous one
            S = S - E @ np.linalg.solve(S_prev, E.T)
            S = 0.5 * (S + S.T)
        neg += _negative_count(S)
        S_prev = S
    return neg


def laplacian_eigs(dim: int, nx: int, count: int | None = None):
    """Closed form: lam = 4/h^2 sum_d sin^2(i_d pi h / 2), i_d = 1..nx (ascending)."""
    h = 1.0 / (nx + 1)
    s = 4.0 / h ** 2 * np.sin(np.arange(1, nx + 1) * np.pi * h / 2.0) ** 2
    if dim == 2:
        lam = (s[:, None] + s[None, :]).ravel()
    else:
        lam = (s[:, None, None] + s[None, :, None] + s[None, None, :]).ravel()
    lam = np.sort(lam)
    return lam if count is None else lam[:count]


def loewner_bounds(fields, i, count: int):
    """Courant-Fischer bounds on the `count` smallest eigenvalues of A^(i)."""
    a_min = min(float(f[i].min()) for f in fields.faces)
    a_max = max(float(f[i].max()) for f in fields.faces)
    c_min = float(fields.c[i].min())
    c_max = float(fields.c[i].max())
    l0 = laplacian_eigs(fields.dim, fields.nx, count)
    return a_min * l0 + c_min, a_max * l0 + c_max
