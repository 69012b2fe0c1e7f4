"""Pins for oracle/eig.py and oracle/checks.py — CPU only."""
import numpy as np
import pytest

import synth
from oracle import eig, checks, operator as op


def test_jacobi_matches_library_eigh():
    # special case reducing to a library routine (LAPACK syevd via numpy)
    rng = np.random.default_rng(0)
    B = rng.standard_normal((30, 30))
    A = B + B.T
    w, V, sweeps = eig.jacobi_eigh(A)
    wr = np.linalg.eigvalsh(A)
    assert np.abs(w - wr).max() < 1e-13 * np.abs(wr).max()
    assert checks.orth_error(V) < 1e-13
    assert np.abs(A @ V - V * w).max() < 1e-12 * np.abs(wr).max()
    assert abs(np.sum(w) - np.trace(A)) < 1e-12 * np.abs(A).sum()   # trace identity
    assert 3 <= sweeps <= 15


def test_jacobi_closed_form_laplacian():
    nx = 6
    f = synth.constant_fields(2, nx)
    w, V, _ = eig.jacobi_eigh(op.assemble_dense(f, 0))
    ex = checks.laplacian_eigs(2, nx)
    assert np.abs(w - ex).max() < 1e-13 * ex.max()


@pytest.mark.parametrize("dim,nx,k,c", [(2, 32, 16, 0.0), (2, 40, 60, 3.0), (3, 10, 30, 0.0)])
def test_lanczos_closed_form_laplacian(dim, nx, k, c):
    # closed form lam = 4/h^2 sum sin^2(i pi h/2) + c (north_star)
    f = synth.constant_fields(dim, nx, c=c)
    r = eig.smallest_eigpairs(f, 0, k)
    ex = checks.laplacian_eigs(dim, nx, k) + c
    assert np.abs(r.lam - ex).max() < 1e-12 * ex.max()
    A = op.assemble_csr(f, 0)
    assert checks.rel_residual(A, r.lam, r.V).max() < 1e-11
    assert checks.orth_error(r.V) < 1e-12


def test_lanczos_vs_jacobi_tiny_variable_grid():
    # two independent algorithms on a tiny variable-coefficient grid
    cfg = synth.get_config("C3").with_(nx=12)
    f = synth.make_batch(cfg, 1)
    r = eig.smallest_eigpairs(f, 0, 20)
    w, V, _ = eig.jacobi_eigh(op.assemble_dense(f, 0))
    assert np.abs(r.lam - w[:20]).max() < 1e-12 * w[19]
    ev, sine = checks.compare_pairs(w, V, r.lam, r.V, 20)
    assert ev < 1e-12 and sine < 1e-9


def test_lanczos_vs_library_dense_c1():
    cfg = synth.get_config("C1")
    f = synth.make_batch(cfg, 1)
    k = cfg.L + 8
    r = eig.smallest_eigpairs(f, 0, k)
    D = op.assemble_dense(f, 0)
    w, V = np.linalg.eigh(D)
    ev, sine = checks.compare_pairs(w, V, r.lam, r.V, cfg.L)
    assert ev < 1e-12 and sine < 1e-9


@pytest.mark.parametrize("cfg_name", ["C1", "C2"])
def test_loewner_and_inertia(cfg_name):
    cfg = synth.get_config(cfg_name)
    f = synth.make_batch(cfg, 1, start=3)
    r = eig.smallest_eigpairs(f, 0, cfg.L + 8)
    lo, hi = checks.loewner_bounds(f, 0, cfg.L)
    assert np.all(lo <= r.lam[:cfg.L] * (1 + 1e-12)) and np.all(r.lam[:cfg.L] <= hi * (1 + 1e-12))
    lamL = r.lam[cfg.L - 1]
    eta = 1e-9
    below = int(np.sum(r.lam < lamL * (1 - eta)))
    assert checks.inertia_below(f, 0, lamL * (1 - eta)) == below      # nothing missed below lam_L
    assert checks.inertia_below(f, 0, lamL * (1 + eta)) >= cfg.L


def test_residual_metrics_on_exact_pairs():
    nx = 8
    f = synth.constant_fields(2, nx)
    A = op.assemble_csr(f, 0)
    h = f.h
    x = np.arange(1, nx + 1) * h
    v = np.outer(np.sin(np.pi * x), np.sin(2 * np.pi * x)).reshape(-1)   # v[y, x] mode (i=2 in x, j=1 in y)
    v /= np.linalg.norm(v)
    lam = 4 / h ** 2 * (np.sin(np.pi * h / 2) ** 2 + np.sin(2 * np.pi * h / 2) ** 2)
    assert checks.rel_residual(A, np.array([lam]), v[:, None])[0] < 1e-14
    assert checks.rel_residual(A, np.array([lam * 1.01]), v[:, None])[0] == pytest.approx(0.01, rel=1e-9)


def test_clusters_and_subspace_sine():
    lam = np.array([1.0, 1.0 + 1e-7, 2.0, 3.0, 3.0001])
    assert checks.clusters(lam) == [(0, 2), (2, 3), (3, 5)]
    U = np.eye(4)[:, :2]
    th = 1e-3
    V = np.array([[1, 0], [0, np.cos(th)], [0, np.sin(th)], [0, 0]])
    assert checks.subspace_sine(U, V) == pytest.approx(np.sin(th), rel=1e-9)


@pytest.mark.parametrize("cfg_name,nx", [("C3", 12), ("C4", 6), ("C1", 10), ("V1", 8)])
def test_inertia_counts_match_dense_eigvalsh(cfg_name, nx):
    """O8's two counting routines (no-pivot banded LDL^T; block Schur complements + Haynsworth)
    against counting the eigenvalues of the dense matrix (LAPACK via numpy) below each shift,
    including shifts 1e-9 relative either side of an eigenvalue and between a close pair."""
    cfg = synth.get_config(cfg_name).with_(nx=nx)
    f = synth.make_batch(cfg, 1)
    w = np.linalg.eigvalsh(op.assemble_dense(f, 0))
    gaps = np.diff(w) / w[1:]
    j = int(np.argmin(gaps[:40]))                      # closest pair among the low eigenvalues
    shifts = [0.5 * w[0], w[3] * (1 - 1e-9), w[3] * (1 + 1e-9), w[10] * (1 - 1e-9), 0.5 * (w[j] + w[j + 1]),
              0.5 * (w[25] + w[26]), 1.5 * w[-1]]
    for sigma in shifts:
        want = int(np.sum(w < sigma))
        assert checks.inertia_blocks(f, 0, sigma) == want, sigma
        if not getattr(f, "is_vib", False):
            assert checks.inertia_below(f, 0, sigma) == want, sigma


def test_smallest_eigpairs_raises_instead_of_returning_unconverged():
    cfg = synth.get_config("C2").with_(nx=30, L=20)
    f = synth.make_batch(cfg, 1)
    with pytest.raises(eig.OracleNotConverged):
        eig.smallest_eigpairs(f, 0, 20, max_dim=24)      # Krylov space capped far too small
