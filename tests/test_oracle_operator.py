"""Pins for oracle/operator.py (FD assembly) — CPU only."""
import numpy as np
import pytest

import synth
from oracle import operator as op
from tests.conftest import load_golden


def test_eq2_worked_example():
    # h^2 A = -M_Eq2 for k == 1 on the 2x2 grid (exact integers)
    M = np.array(load_golden("eq2_matrix.txt"))
    f = synth.constant_fields(2, 2)
    A = op.assemble_dense(f, 0)
    assert np.array_equal(np.round(A * f.h ** 2, 12), -M)


def _appB_T(nx):
    pat = np.array(load_golden("appB_tridiag.txt"))
    sub, dia, sup = pat[1, 0], pat[1, 1], pat[1, 2]
    T = np.diag(np.full(nx, dia)) + np.diag(np.full(nx - 1, sup), 1) + np.diag(np.full(nx - 1, sub), -1)
    return T


@pytest.mark.parametrize("nx", [3, 5, 8])
def test_kronecker_sum_of_appB_2d(nx):
    # a == 1 -> A = -(I (x) T + T (x) I) / h^2, x fastest
    f = synth.constant_fields(2, nx)
    T = _appB_T(nx) / f.h ** 2
    I = np.eye(nx)
    K = -(np.kron(I, T) + np.kron(T, I))
    assert np.allclose(op.assemble_dense(f, 0), K, rtol=1e-14, atol=0)


def test_kronecker_sum_of_appB_3d():
    nx = 4
    f = synth.constant_fields(3, nx, c=2.5)
    T = _appB_T(nx) / f.h ** 2
    I = np.eye(nx)
    K = -(np.kron(np.kron(I, I), T) + np.kron(np.kron(I, T), I) + np.kron(np.kron(T, I), I))
    assert np.allclose(op.assemble_dense(f, 0), K + 2.5 * np.eye(nx ** 3), rtol=1e-14, atol=0)


def _energy(fields, i, u):
    """Flux-form energy u^T A u = sum_faces a_f (u_left - u_right)^2 / h^2 + sum c u^2,
    with u = 0 outside the grid (Dirichlet).  Written independently of assembly."""
    dim, nx, h = fields.dim, fields.nx, fields.h
    U = u.reshape((nx,) * dim)
    E = float(np.sum(fields.c[i] * u * u))
    for ax in range(dim):
        npax = dim - 1 - ax                                  # numpy axis of grid axis ax
        pad = [(0, 0)] * dim
        pad[npax] = (1, 1)
        Up = np.pad(U, pad)
        d = np.diff(Up, axis=npax)                           # one difference per face
        E += float(np.sum(fields.faces[ax][i] * d * d)) / h ** 2
    return E


@pytest.mark.parametrize("cfg", ["C1", "C3", "C4"])
def test_energy_identity_variable_coefficients(cfg):
    c = synth.get_config(cfg)
    small = c.with_(nx=6)
    f = synth.make_batch(small, 2)
    rng = np.random.default_rng(0)
    for i in range(2):
        A = op.assemble_csr(f, i)
        for _ in range(3):
            u = rng.standard_normal(f.n)
            assert abs(u @ (A @ u) - _energy(f, i, u)) <= 1e-12 * abs(_energy(f, i, u))
        # symmetric positive definite
        D = A.toarray()
        assert np.array_equal(D, D.T)
        assert np.linalg.eigvalsh(D)[0] > 0


def test_banded_storage_round_trip():
    f = synth.make_batch(synth.get_config("C4").with_(nx=5), 1)
    ab, u = op.banded_upper(f, 0)
    D = op.assemble_dense(f, 0)
    n = f.n
    R = np.zeros((n, n))
    for c in range(n):
        for r in range(max(0, c - u), c + 1):
            R[r, c] = R[c, r] = ab[u + r - c, c]
    assert np.array_equal(R, D)


def test_norm_inf_is_gershgorin_bound():
    f = synth.make_batch(synth.get_config("C1"), 1)
    D = op.assemble_dense(f, 0)
    assert op.norm_inf(f, 0) >= np.linalg.eigvalsh(D)[-1]
