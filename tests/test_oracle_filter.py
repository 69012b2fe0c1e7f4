"""Pins for oracle/filter.py (Alg. 1) — CPU only."""
import numpy as np
import pytest

import synth
from oracle import filter as ofilt, operator as op, checks


def _lap_eigvec(nx, i, j):
    h = 1.0 / (nx + 1)
    x = np.arange(1, nx + 1) * h
    v = np.outer(np.sin(j * np.pi * x), np.sin(i * np.pi * x)).reshape(-1)   # v[y, x]
    lam = 4 / h ** 2 * (np.sin(i * np.pi * h / 2) ** 2 + np.sin(j * np.pi * h / 2) ** 2)
    return v / np.linalg.norm(v), lam


@pytest.mark.parametrize("m", [1, 2, 7, 20])
def test_closed_form_on_laplacian_eigenvectors(m):
    # C_m(A~) acts on an eigenvector as the scalar C_m((t-c)/e); Alg. 1's sigma
    # scaling divides by C_m((lambda-c)/e)
    nx = 12
    f = synth.constant_fields(2, nx)
    A = op.assemble_csr(f, 0)
    modes = [(1, 1), (2, 1), (3, 4), (7, 9), (12, 12)]
    V = np.stack([_lap_eigvec(nx, i, j)[0] for i, j in modes], axis=1)
    t = np.array([_lap_eigvec(nx, i, j)[1] for i, j in modes])
    alpha, beta = 600.0, 1.02 * t.max()
    c, e = (alpha + beta) / 2, (beta - alpha) / 2
    lam = t[0]
    Y = ofilt.cheb_filter(A, V, m, lam, c, e)
    rho = ofilt.cheb_T(m, (t - c) / e) / ofilt.cheb_T(m, np.array([(lam - c) / e]))[0]
    assert np.allclose(Y, V * rho, rtol=0, atol=1e-12 * np.abs(rho).max())
    # normalisation at the scale point: rho_m(lambda) = 1
    assert abs(rho[0] - 1.0) < 1e-12


def test_m1_formula():
    # m = 1 -> Y_1 = (A - cI) Y_0 / (lambda - c)
    rng = np.random.default_rng(0)
    f = synth.make_batch(synth.get_config("C1").with_(nx=6), 1)
    A = op.assemble_dense(f, 0)
    Y0 = rng.standard_normal((36, 3))
    lam, c, e = 30.0, 500.0, 400.0
    Y = ofilt.cheb_filter(A, Y0, 1, lam, c, e)
    assert np.allclose(Y, (A @ Y0 - c * Y0) / (lam - c), rtol=1e-14, atol=0)


def test_similarity_invariance_and_damping():
    # filtering commutes with an orthogonal similarity; components inside
    # [alpha, beta] are damped below 1 while the scale point keeps weight 1
    rng = np.random.default_rng(1)
    n = 20
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    d = np.linspace(1, 100, n)
    A = Q @ np.diag(d) @ Q.T
    Y0 = rng.standard_normal((n, 4))
    lam, alpha, beta = 1.0, 30.0, 100.0
    c, e = (alpha + beta) / 2, (beta - alpha) / 2
    Y = ofilt.cheb_filter(A, Y0, 10, lam, c, e)
    Yd = ofilt.cheb_filter(np.diag(d), Q.T @ Y0, 10, lam, c, e)
    assert np.allclose(Q.T @ Y, Yd, rtol=0, atol=1e-10 * np.abs(Yd).max())
    rho = ofilt.cheb_T(10, (d - c) / e) / ofilt.cheb_T(10, np.array([(lam - c) / e]))[0]
    assert np.all(np.abs(rho[d >= alpha]) < 1e-3) and abs(rho[0] - 1) < 1e-12
