"""Oracle-side FD assembly of A^(i) from the coefficient fields.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper discretises with central finite differences on a regular grid with
unknowns in row-major order (Eq. 2; Appendix B PAPER.md:651-710,
A = tridiag(1, -2, 1)/dx^2).  Its Eq. 2 form k * Lap is not symmetric for a
variable k, while the problem statement needs Hermitian A,
so DESIGN.md reading R20 adopts the divergence (flux) form -div(a grad u) + c u
with face-midpoint coefficients, the sign making A positive definite:

  node (i, j[, l]), unknown k = i + nx*j (+ nx*ny*l), h = 1/(nx+1)
  A[k,k]      = (sum of the 2*dim face coefficients around the node) / h^2 + c[k]
  A[k,k+1]    = -a(x-face between i and i+1) / h^2          (i < nx-1)
  A[k,k+nx]   = -a(y-face between j and j+1) / h^2          (j < ny-1)
  A[k,k+nx*ny]= -a(z-face between l and l+1) / h^2          (l < nz-1, 3-D)

For a == 1, c == 0 this is -(Kronecker sum of App. B's tridiag(1,-2,1)/h^2),
i.e. h^2 A = -M_Eq2 on the paper's 2x2 example (pinned in tests).

Vibration family (thin plate  Lap(D Lap u) = lambda rho u;
SPEC discretize "vibration"; reading R25): with Lh the 5-point Dirichlet
Laplacian  (Lh u)_k = (4 u_k - sum of the 4 neighbours) / h^2  (= -Lap_h, SPD),
  A_bih = Lh diag(D) Lh      (13-point, symmetric: Lh is symmetric),
  B     = diag(rho)^(-1/2) A_bih diag(rho)^(-1/2),
the standard form of the pencil (A_bih, diag(rho)): same eigenvalues, eigenvectors
y = diag(rho)^(1/2) u.  Both products are formed literally with scipy.sparse, then
(B + B^T)/2 removes the last-ulp asymmetry of the products' summation order.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def _is_vib(fields) -> bool:
    return getattr(fields, "family", "flux") == "vib"


def laplacian_csr(nx: int, h: float) -> sp.csr_matrix:
    """Lh = -Lap_h on the nx x nx interior grid, Dirichlet, x fastest: kron sum of tridiag(-1, 2, -1)/h^2
    (App. B P:651-710's 1-D matrix, negated)."""
    T = sp.diags([-np.ones(nx - 1), 2.0 * np.ones(nx), -np.ones(nx - 1)], [-1, 0, 1]) / (h * h)
    I = sp.identity(nx)
    return (sp.kron(I, T) + sp.kron(T, I)).tocsr()


def vibration_csr(fields, i) -> sp.csr_matrix:
    """B = diag(rho)^-1/2 Lh diag(D) Lh diag(rho)^-1/2 of operator i (D = params[i,0], rho = params[i,1])."""
    D = np.asarray(fields.params[i, 0], dtype=np.float64)
    rho = np.asarray(fields.params[i, 1], dtype=np.float64)
    Lh = laplacian_csr(fields.nx, fields.h)
    A = Lh @ sp.diags(D) @ Lh
    S = sp.diags(1.0 / np.sqrt(rho))
    B = (S @ A @ S).tocsr()
    # symmetric in exact arithmetic; the sparse products sum the two paths of an (i, i+nx+-1)
    # entry in either order, so average with the transpose for exact symmetry (SPEC invariant)
    return ((B + B.T) * 0.5).tocsr()


def _face_arrays(fields, i):
    return [np.asarray(f[i], dtype=np.float64) for f in fields.faces]


def stencil(fields, i):
    """Per-node stencil values (diag, [off_x, off_y(, off_z)]) of operator i, x fastest.

    off_d[k] = A[k, k + stride_d] (zero where the neighbour is outside the grid).
    """
    if _is_vib(fields):
        B = vibration_csr(fields, i)
        n = B.shape[0]
        offs = []
        for st in strides(fields):
            o = np.zeros(n)
            o[:n - st] = B.diagonal(st)
            offs.append(o)
        return B.diagonal(0).copy(), offs
    dim, nx, h = fields.dim, fields.nx, fields.h
    inv_h2 = 1.0 / (h * h)
    faces = _face_arrays(fields, i)
    c = np.asarray(fields.c[i], dtype=np.float64)
    if dim == 2:
        ax, ay = faces                                   # ax[j, 0..nx], ay[0..ny, i]
        diag = (ax[:, :-1] + ax[:, 1:] + ay[:-1, :] + ay[1:, :]) * inv_h2 + c.reshape(nx, nx)
        offx = -ax[:, 1:] * inv_h2                       # face between i and i+1
        offx[:, -1] = 0.0                                # i = nx-1: neighbour is the boundary
        offy = -ay[1:, :] * inv_h2
        offy[-1, :] = 0.0
        return diag.reshape(-1), [offx.reshape(-1), offy.reshape(-1)]
    ax, ay, az = faces                                   # ax[l, j, 0..nx], ay[l, 0..ny, i], az[0..nz, j, i]
    cc = c.reshape(nx, nx, nx)
    diag = (ax[:, :, :-1] + ax[:, :, 1:] + ay[:, :-1, :] + ay[:, 1:, :]
            + az[:-1, :, :] + az[1:, :, :]) * inv_h2 + cc
    offx = -ax[:, :, 1:] * inv_h2
    offx[:, :, -1] = 0.0
    offy = -ay[:, 1:, :] * inv_h2
    offy[:, -1, :] = 0.0
    offz = -az[1:, :, :] * inv_h2
    offz[-1, :, :] = 0.0
    return diag.reshape(-1), [offx.reshape(-1), offy.reshape(-1), offz.reshape(-1)]


def strides(fields):
    nx = fields.nx
    if _is_vib(fields):
        return [1, 2, nx - 1, nx, nx + 1, 2 * nx]
    return [1, nx] if fields.dim == 2 else [1, nx, nx * nx]


def assemble_csr(fields, i) -> sp.csr_matrix:
    """Explicit sparse symmetric A^(i)."""
    if _is_vib(fields):
        return vibration_csr(fields, i)
    n = fields.n
    diag, offs = stencil(fields, i)
    rows, cols, vals = [np.arange(n)], [np.arange(n)], [diag]
    for off, st in zip(offs, strides(fields)):
        k = np.arange(n - st)
        v = off[:n - st]
        keep = v != 0.0
        for r, c in ((k[keep], k[keep] + st), (k[keep] + st, k[keep])):
            rows.append(r)
            cols.append(c)
            vals.append(v[keep])
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n))
    return A.tocsr()


def assemble_dense(fields, i) -> np.ndarray:
    return assemble_csr(fields, i).toarray()


def banded_upper(fields, i):
    """A^(i) in LAPACK upper banded storage ab[u + r - c, c] = A[r, c] (r <= c); u = largest stride."""
    n = fields.n
    diag, offs = stencil(fields, i)
    st = strides(fields)
    u = st[-1]
    ab = np.zeros((u + 1, n))
    ab[u] = diag
    for off, s in zip(offs, st):
        ab[u - s, s:] = off[:n - s]                      # A[c-s, c] = off[c-s]
    return ab, u


def norm_inf(fields, i) -> float:
    """||A||_inf = max row sum of |A| (Gershgorin bound on lambda_max for SPD A)."""
    A = assemble_csr(fields, i)
    return float(np.abs(A).sum(axis=1).max())
