"""Pins of the oracle's vibration operator (R25) — CPU.

B = diag(rho)^-1/2 Lh diag(D) Lh diag(rho)^-1/2 is pinned against things other than itself:
  - D = rho = 1: B = Lh^2, eigenvalues = squares of the closed-form Dirichlet Laplacian spectrum;
  - the energy u^T A_bih u = sum_k D_k ((Lh u)_k)^2 with Lh u written as explicit point loops;
  - the pencil (A_bih, diag(rho)) solved by scipy's generalized eigh has B's eigenvalues;
  - scaling laws D -> c D, rho -> c rho;  13-point pattern and exact symmetry;
  - the 4*pi^4 continuum limit of the simply supported unit plate.
"""
import numpy as np
import pytest
import scipy.linalg as sla

import synth
from oracle import checks, eig as oeig, operator as oop


def vib_fields(nx, D, rho):
    n = nx * nx
    params = np.stack([np.broadcast_to(D, (n,)), np.broadcast_to(rho, (n,))])[None].astype(np.float64)
    return synth.OperatorFields(2, nx, 1.0 / (nx + 1), [], np.zeros((1, n)), params.copy(), "vib")


def test_unit_coefficients_square_the_laplacian_spectrum():
    nx = 7
    f = vib_fields(nx, 1.0, 1.0)
    lam = np.linalg.eigvalsh(oop.assemble_dense(f, 0))
    ref = np.sort(checks.laplacian_eigs(2, nx) ** 2)
    assert np.max(np.abs(lam - ref) / ref) <= 1e-12


def test_energy_matches_pointwise_laplacian_loops():
    nx = 6
    h = 1.0 / (nx + 1)
    rng = np.random.default_rng(3)
    D = rng.uniform(0.5, 2.0, nx * nx)
    rho = rng.uniform(0.5, 2.0, nx * nx)
    f = vib_fields(nx, D, rho)
    B = oop.assemble_dense(f, 0)
    for _ in range(3):
        y = rng.standard_normal(nx * nx)
        u = y / np.sqrt(rho)                     # B = S A S with S = rho^-1/2: y^T B y = u^T A u
        E = 0.0
        for j in range(nx):
            for i in range(nx):
                k = i + nx * j
                lap = 4.0 * u[k]
                if i > 0:
                    lap -= u[k - 1]
                if i < nx - 1:
                    lap -= u[k + 1]
                if j > 0:
                    lap -= u[k - nx]
                if j < nx - 1:
                    lap -= u[k + nx]
                E += D[k] * (lap / h ** 2) ** 2
        assert abs(y @ B @ y - E) <= 1e-12 * abs(E)


def test_pencil_eigenvalues_equal_standard_form():
    nx = 5
    rng = np.random.default_rng(11)
    D = rng.uniform(0.3, 3.0, nx * nx)
    rho = rng.uniform(0.3, 3.0, nx * nx)
    f = vib_fields(nx, D, rho)
    Lh = oop.laplacian_csr(nx, f.h).toarray()
    A = Lh @ np.diag(D) @ Lh
    lam_pencil = sla.eigh(A, np.diag(rho), eigvals_only=True)
    lam_std = np.linalg.eigvalsh(oop.assemble_dense(f, 0))
    assert np.max(np.abs(lam_pencil - lam_std) / lam_std) <= 1e-10


def test_scaling_laws():
    nx = 5
    rng = np.random.default_rng(2)
    D = rng.uniform(0.5, 2.0, nx * nx)
    rho = rng.uniform(0.5, 2.0, nx * nx)
    base = np.linalg.eigvalsh(oop.assemble_dense(vib_fields(nx, D, rho), 0))
    l2 = np.linalg.eigvalsh(oop.assemble_dense(vib_fields(nx, 3.0 * D, rho), 0))
    l3 = np.linalg.eigvalsh(oop.assemble_dense(vib_fields(nx, D, 4.0 * rho), 0))
    assert np.allclose(l2, 3.0 * base, rtol=1e-12)
    assert np.allclose(l3, base / 4.0, rtol=1e-12)


def test_thirteen_point_pattern_and_symmetry():
    nx = 6
    rng = np.random.default_rng(4)
    f = vib_fields(nx, rng.uniform(0.5, 2.0, nx * nx), rng.uniform(0.5, 2.0, nx * nx))
    B = oop.assemble_dense(f, 0)
    assert np.array_equal(B, B.T)
    allowed = {0, 1, 2, nx - 1, nx, nx + 1, 2 * nx}
    r, c = np.nonzero(B)
    assert set(np.abs(r - c).tolist()) <= allowed
    assert max(np.count_nonzero(B[k]) for k in range(nx * nx)) == 13
    # the stencil()/banded form used by the banded solvers reproduces B exactly
    diag, offs = oop.stencil(f, 0)
    R = np.diag(diag)
    for o, s in zip(offs, oop.strides(f)):
        R += np.diag(o[:nx * nx - s], s) + np.diag(o[:nx * nx - s], -s)
    assert np.array_equal(R, B)


def test_continuum_limit_simply_supported_plate():
    lam = []
    for nx in (8, 16, 32):
        f = vib_fields(nx, 1.0, 1.0)
        r = oeig.smallest_eigpairs(f, 0, 1)
        lam.append(r.lam[0])
    err = np.abs(np.array(lam) - 4.0 * np.pi ** 4)
    assert err[2] < err[1] < err[0]
    assert err[2] / (4.0 * np.pi ** 4) < 5e-3


@pytest.mark.parametrize("N", [2])
def test_v1_fields_spd_and_oracle_pairs(N):
    cfg = synth.get_config("V1").with_(nx=12)
    f = synth.make_batch(cfg, N)
    for i in range(N):
        r = oeig.smallest_eigpairs(f, i, 10)
        A = oop.assemble_csr(f, i)
        assert np.all(r.lam > 0)
        assert np.max(checks.resid_over_normA(A, r.lam, r.V, r.normA)) <= 1e-12
        dense = np.linalg.eigvalsh(A.toarray())[:10]
        assert np.max(np.abs(dense - r.lam) / dense) <= 1e-10
