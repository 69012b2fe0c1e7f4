"""Thin-plate vibration family on the device (R25) — GPU.

scsf_assemble_vibration's 13-point standard form B, the 13-point filter step and the full
SCSF solve against the oracle (oracle/operator.py vibration_csr, oracle/eig.py), plus the
closed form of unit coefficients (B = Lh^2).  Acceptance as for the other families.
"""
import numpy as np
import pytest

import synth
from oracle import checks, filter as ofilt, operator as oop
from tests.helpers import PAPER_TOL_SLACK, check_pairs, device_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2510_23215_b200 import scsf
    scsf.load_library()
    return scsf


def _np_block(t, n):
    return t[:, :n].cpu().numpy().T


def _unit_fields(nx, D=1.0, rho=1.0):
    n = nx * nx
    params = np.empty((1, 2, n))
    params[0, 0] = D
    params[0, 1] = rho
    return synth.OperatorFields(2, nx, 1.0 / (nx + 1), [], np.zeros((1, n)), params, "vib")


@pytest.mark.parametrize("nx", [3, 7, 24, 100])
def test_assemble_vibration_matches_oracle(lib, nx):
    cfg = synth.get_config("V1").with_(nx=nx)
    f = synth.make_batch(cfg, 3)
    ops, _ = device_problem(f)
    assert ops.stencil == lib.STENCIL_VIB13
    coef = ops.coef.cpu().numpy()
    n = f.n
    offsets = [1, 2, nx - 1, nx, nx + 1, 2 * nx]
    for i in range(3):
        assert np.all(coef[i, :, n:] == 0.0)
        if nx <= 24:                  # rebuild the device's B densely (nx = 3: offsets 2 and nx-1 coincide)
            Bd = np.diag(coef[i, 0, :n])
            for d, o in enumerate(offsets):
                Bd += np.diag(coef[i, 1 + d, :n - o], o) + np.diag(coef[i, 1 + d, :n - o], -o)
            B = oop.assemble_dense(f, i)
            assert np.max(np.abs(Bd - B)) <= 1e-14 * np.abs(B).max()
            if nx == 3:
                continue
        diag, offs = oop.stencil(f, i)
        scale = np.abs(diag).max()
        assert np.max(np.abs(coef[i, 0, :n] - diag)) <= 1e-14 * scale
        for d, off in enumerate(offs):
            assert np.max(np.abs(coef[i, 1 + d, :n] - off)) <= 1e-14 * scale
            assert np.all((coef[i, 1 + d, :n] == 0) == (off == 0))     # same zero pattern


@pytest.mark.parametrize("nx,k,m", [(24, 5, 20), (100, 3, 20), (13, 7, 3), (3, 2, 4)])
def test_vibration_filter_matches_oracle(lib, nx, k, m):
    import torch
    cfg = synth.get_config("V1").with_(nx=nx)
    f = synth.make_batch(cfg, 2)
    ops, _ = device_problem(f)
    assert lib.filter_kind(ops) == 0                      # per-step streaming 13-point kernel
    n, ld = f.n, ops.ld
    rng = np.random.default_rng(8)
    Y0 = rng.standard_normal((n, k))
    A = oop.assemble_csr(f, 1)
    normA = float(np.abs(A).sum(axis=1).max())
    lam, alpha = 1e-4 * normA, 0.01 * normA
    c, e = (alpha + normA) / 2, (normA - alpha) / 2
    Yd = torch.zeros((k, ld), dtype=torch.float64, device="cuda")
    Yd[:, :n] = torch.from_numpy(Y0.T.copy())
    Ym = _np_block(lib.cheb_filter(ops, 1, Yd, m, lam, c, e), n)
    ref = ofilt.cheb_filter(A, Y0, m, lam, c, e)
    scale = np.abs(ref).max(axis=0)
    assert np.all(np.abs(Ym - ref).max(axis=0) <= 1e-12 * scale)


def test_unit_plate_closed_form(lib):
    """D = rho = 1: B = Lh^2, eigenvalues = squared Dirichlet Laplacian eigenvalues."""
    nx, L, nex = 32, 16, 4
    f = _unit_fields(nx)
    ops, _ = device_problem(f)
    evals, evecs, st = lib.solve_one(ops, 0, L, nex, 20, 1e-8, 400, seed=1)
    ex = checks.laplacian_eigs(2, nx, L) ** 2
    assert np.all(np.abs(evals.cpu().numpy()[:L] - ex) <= 1e-9 * ex)
    V = _np_block(evecs, f.n)
    assert checks.orth_error(V[:, :L]) <= 1e-12
    A = oop.assemble_csr(f, 0)
    assert checks.rel_residual(A, evals.cpu().numpy()[:L], V[:, :L]).max() <= 1e-8 * 10


def test_v1_full_size_chain_sample(lib):
    """configs V1 at full size (n = 1e4, L = 200): the head of the sorted queue as one warm chain."""
    cfg = synth.get_config("V1")
    f = synth.make_batch(cfg, 24)
    ops, params = device_problem(f)
    perm, _, _ = lib.sort(params, cfg.dim, cfg.nx, cfg.p0)
    chain = perm[:3]
    evals, evecs, stats = lib.solve_queue(ops, chain, cfg.L, cfg.nex, cfg.degree, cfg.tol, cfg.max_iter, seed=3)
    ev = evals.cpu().numpy()
    for k, i in enumerate(chain):
        assert stats[k]["status"] == 0, stats[k]
        V = evecs[k, :, :f.n].cpu().numpy().T
        check_pairs(f, int(i), ev[k], V, cfg.L, paper_tol=PAPER_TOL_SLACK * cfg.tol, lock_floor=True)
    assert stats[1]["iterations"] < stats[0]["iterations"]          # the warm start pays


def test_v1_small_chains_every_operator(lib):
    cfg = synth.get_config("V1").with_(nx=24, L=40)
    f = synth.make_batch(cfg, 16)
    ops, params = device_problem(f)
    perm, _, _ = lib.sort(params, cfg.dim, cfg.nx, cfg.p0)
    evals, evecs, stats = lib.solve_chains(ops, perm, 4, cfg.L, cfg.nex, cfg.degree, cfg.tol, cfg.max_iter, seed=5)
    ev = evals.cpu().numpy()
    for k, i in enumerate(perm):
        assert stats[k]["status"] == 0, stats[k]
        check_pairs(f, int(i), ev[k], evecs[k, :, :f.n].cpu().numpy().T, cfg.L, paper_tol=PAPER_TOL_SLACK * cfg.tol, lock_floor=True)


def test_grf_vib_family_matches_host(lib):
    import torch
    cfg = synth.get_config("V1")
    f = synth.make_batch(cfg, 3, start=5)
    xi = torch.from_numpy(synth.draw_xi(cfg, 3, start=5)).cuda()
    faces, c, params = lib.grf_fields(cfg.dim, cfg.nx, cfg.K, cfg.s, cfg.sigma, cfg.vscale, cfg.family, xi)
    assert faces == [] and c is None
    got = params.cpu().numpy()
    assert float(np.max(np.abs(got - f.params) / f.params)) <= 1e-12
    ops = lib.assemble_vibration(cfg.nx, cfg.h, params)
    ops_h, _ = device_problem(f)
    a, b = ops.coef.cpu().numpy(), ops_h.coef.cpu().numpy()
    assert float(np.max(np.abs(a - b))) <= 1e-12 * float(np.max(np.abs(b)))


def test_vibration_rejected_where_unsupported(lib):
    import torch
    cfg = synth.get_config("V1").with_(nx=8)
    f = synth.make_batch(cfg, 1)
    ops, _ = device_problem(f)
    comms = lib.comm_create_loopback(1)
    try:
        with pytest.raises(lib.ScsfError):
            lib.solve_queue_dist(ops, [0], 4, 1, comms[0], 20, 1e-8, seed=1)
    finally:
        comms[0].close()
    faces = [torch.ones((1, 8, 9), dtype=torch.float64, device="cuda"),
             torch.ones((1, 9, 8), dtype=torch.float64, device="cuda")]
    bad = lib.Operators(2, 8, 8, 1, 1, ops.ld, torch.empty((1, 3, ops.ld), dtype=torch.float64, device="cuda"),
                        lib.STENCIL_VIB13)
    with pytest.raises(lib.ScsfError):                       # scsf_assemble builds flux stencils only
        lib._check(lib.load_library().scsf_assemble(lib.ctypes.byref(bad.c_struct()), 0.1,
                                                    lib._ptr(faces[0]), lib._ptr(faces[1]), None, None,
                                                    lib._ptr(bad.coef), None))
