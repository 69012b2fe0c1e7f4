"""Parity of scsf_assemble / scsf_cheb_filter / scsf_solve_* against the oracle — GPU.

Acceptance (BASELINE.json north_star): eigenvalues within 1e-9 relative,
||Ax - lx|| / ||A||_inf <= 1e-8 per pair, subspace sines <= 1e-6 (per
cluster, R21), orthonormality 1e-12; the paper metric
||Ax - lx|| / ||Ax|| is checked against tol with the rounding slack of
tests/helpers.PAPER_TOL_SLACK.
"""
import numpy as np
import pytest

import synth
from oracle import checks, eig as oeig, filter as ofilt, operator as oop
from oracle import sort as osort
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
    """device block [k, ld] -> numpy n x k (column-major view)."""
    return t[:, :n].cpu().numpy().T


# ------------------------------------------------------------------ assembly ----
@pytest.mark.parametrize("cfg_name,nx", [("C1", 32), ("C2", 17), ("C3", 23), ("C4", 9), ("C5", 31)])
def test_assemble_matches_oracle_stencil(lib, cfg_name, nx):
    cfg = synth.get_config(cfg_name).with_(nx=nx)
    f = synth.make_batch(cfg, 3)
    ops, _ = device_problem(f)
    coef = ops.coef.cpu().numpy()
    eps = np.finfo(np.float64).eps
    for i in range(3):
        diag, offs = oop.stencil(f, i)
        n = f.n
        # diag = (sum of the 2d face coefficients) / h^2 + c: the two sides add the 2d + 1 positive
        # terms in different orders, so they may differ by up to 2d rounding steps (2d eps relative);
        # an off-diagonal is one product -a / h^2 on both sides (1 rounding step each: 2 eps)
        assert np.allclose(coef[i, 0, :n], diag, rtol=2 * cfg.dim * eps, atol=0)
        for d, off in enumerate(offs):
            assert np.allclose(coef[i, 1 + d, :n], off, rtol=2 * eps, atol=0)
        assert np.all(coef[i, :, n:] == 0.0)


# -------------------------------------------------------------------- filter ----
@pytest.mark.parametrize("streaming", [False, True])
@pytest.mark.parametrize("cfg_name,nx,k,m", [("C1", 32, 20, 20), ("C3", 29, 9, 7), ("C4", 11, 13, 20),
                                             ("C2", 40, 1, 1), ("C2", 100, 6, 20), ("C5", 110, 3, 5),
                                             ("C2", 92, 5, 20), ("C1", 132, 3, 20), ("C3", 76, 4, 9),
                                             ("C2", 124, 2, 3), ("C1", 30, 5, 20), ("C3", 34, 3, 7),
                                             ("C3", 200, 5, 20), ("C3", 190, 3, 9), ("C4", 12, 5, 20),
                                             ("C4", 40, 3, 7), ("C4", 20, 6, 9), ("C3", 200, 3, 150),
                                             ("C2", 100, 4, 256), ("C4", 20, 2, 201)])
def test_filter_matches_oracle(lib, cfg_name, nx, k, m, streaming, monkeypatch):
    """Both filter paths: resident (2-D: the register-patch kernel k_filter_rp when one CTA holds a
    column -- nx 30/32/34/40; 30 and 34 leave a 2-row top patch -- the cluster kernel with DSMEM
    halos when a column fits 16 CTAs -- nx 92/100/132 give ragged row splits over 8 CTAs, nx 200/190
    over 16 (a non-portable cluster) --
    else the single-CTA kernel for n <= 12288) and streaming (per-step launches, vectorised when
    nx % 4 == 0, scalar otherwise); SCSF_FILTER_STREAMING=1 forces streaming."""
    import torch
    if streaming:
        monkeypatch.setenv("SCSF_FILTER_STREAMING", "1")
    else:
        monkeypatch.delenv("SCSF_FILTER_STREAMING", raising=False)
    cfg = synth.get_config(cfg_name).with_(nx=nx)
    f = synth.make_batch(cfg, 2)
    ops, _ = device_problem(f)
    n, ld = f.n, ops.ld
    rng = np.random.default_rng(5)
    Y0 = rng.standard_normal((n, k))
    A = oop.assemble_csr(f, 1)
    normA = float(np.abs(A).sum(axis=1).max())
    lam, alpha = 0.002 * normA, 0.1 * normA
    c, e = (alpha + normA) / 2, (normA - alpha) / 2
    Yd = torch.zeros((k, ld), dtype=torch.float64, device="cuda")
    Yd[:, :n] = torch.from_numpy(Y0.T.copy())
    Ym = _np_block(lib.cheb_filter(ops, 1, Yd, m, lam, c, e), n)
    ref = ofilt.cheb_filter(A, Y0, m, lam, c, e)
    scale = np.abs(ref).max(axis=0)
    assert np.all(np.abs(Ym - ref).max(axis=0) <= 1e-12 * scale)


@pytest.mark.parametrize("cfg_name,nx,k,m", [("C3", 200, 5, 20), ("C3", 190, 3, 9), ("C2", 100, 6, 20),
                                             ("C2", 92, 5, 21), ("C3", 76, 4, 9), ("C1", 132, 3, 20)])
@pytest.mark.parametrize("split,tmem", [("0", "1"), ("1", "1"), ("1", "0"), ("2", "1"), ("2", "0")])
def test_filter_tmem_variant(lib, cfg_name, nx, k, m, split, tmem, monkeypatch):
    """k_filter_cl with the patch rows of Y_s / Y_{s-1} in tensor memory (SCSF_FILTER_TMEM=1: tcgen05
    alloc / st / ld / dealloc) against the oracle, on 16-CTA (nx 190/200) and 8-CTA clusters with ragged
    slabs and odd / even degrees (the two TMEM slots swap roles every step); SCSF_FILTER_SPLIT=1 is the
    split arrive / wait step synchronisation (interior warps ahead of the cluster barrier), with and
    without TMEM."""
    import torch
    monkeypatch.setenv("SCSF_FILTER_TMEM", tmem)
    monkeypatch.setenv("SCSF_FILTER_SPLIT", split)
    monkeypatch.delenv("SCSF_FILTER_STREAMING", raising=False)
    cfg = synth.get_config(cfg_name).with_(nx=nx)
    f = synth.make_batch(cfg, 1)
    ops, _ = device_problem(f)
    n, ld = f.n, ops.ld
    Y0 = np.random.default_rng(13).standard_normal((n, k))
    A = oop.assemble_csr(f, 0)
    normA = float(np.abs(A).sum(axis=1).max())
    lam, alpha = 0.002 * normA, 0.1 * normA
    c, e = (alpha + normA) / 2, (normA - alpha) / 2
    Yd = torch.zeros((k, ld), dtype=torch.float64, device="cuda")
    Yd[:, :n] = torch.from_numpy(Y0.T.copy())
    Ym = _np_block(lib.cheb_filter(ops, 0, Yd, m, lam, c, e), n)
    ref = ofilt.cheb_filter(A, Y0, m, lam, c, e)
    assert np.all(np.abs(Ym - ref).max(axis=0) <= 1e-12 * np.abs(ref).max(axis=0))


def test_filter_closed_form_laplacian(lib):
    import torch
    nx = 24
    f = synth.constant_fields(2, nx)
    ops, _ = device_problem(f)
    h = f.h
    x = np.arange(1, nx + 1) * h
    modes = [(1, 1), (1, 2), (5, 3), (24, 24)]
    V = np.stack([np.outer(np.sin(j * np.pi * x), np.sin(i * np.pi * x)).reshape(-1) for i, j in modes], 1)
    t = np.array([4 / h ** 2 * (np.sin(i * np.pi * h / 2) ** 2 + np.sin(j * np.pi * h / 2) ** 2) for i, j in modes])
    beta = 8 / h ** 2
    alpha = 2000.0
    c, e = (alpha + beta) / 2, (beta - alpha) / 2
    Yd = torch.zeros((4, ops.ld), dtype=torch.float64, device="cuda")
    Yd[:, :f.n] = torch.from_numpy(V.T.copy())
    Y = _np_block(lib.cheb_filter(ops, 0, Yd, 20, t[0], c, e), f.n)
    rho = ofilt.cheb_T(20, (t - c) / e) / ofilt.cheb_T(20, np.array([(t[0] - c) / e]))[0]
    assert np.allclose(Y, V * rho, rtol=0, atol=1e-12 * np.abs(V).max())


# --------------------------------------------------------------------- solve ----
def test_closed_form_laplacian_solve(lib):
    # O4: constant coefficients; the L cut splits a degenerate pair, so eigenvalues only
    nx, L, nex = 32, 16, 4
    f = synth.constant_fields(2, nx, c=1.5)
    ops, _ = device_problem(f)
    evals, evecs, st = lib.solve_one(ops, 0, L, nex, 20, 1e-8, 200, seed=1)
    ex = checks.laplacian_eigs(2, nx, L) + 1.5
    assert np.all(np.abs(evals.cpu().numpy()[:L] - ex) <= 1e-9 * ex)
    V = _np_block(evecs, f.n)
    assert checks.orth_error(V[:, :L]) <= 1e-12
    A = oop.assemble_csr(f, 0)
    assert checks.rel_residual(A, evals.cpu().numpy()[:L], V[:, :L]).max() <= 1e-8 * 10


def test_c1_full_chain_parity(lib):
    """configs[0] at full size: all 64 operators along the sorted queue, every one vs the oracle."""
    cfg = synth.get_config("C1")
    f = synth.make_batch(cfg)
    ops, params = device_problem(f)
    perm, _, _ = lib.sort(params, cfg.dim, cfg.nx, cfg.p0)
    evals, evecs, stats = lib.solve_queue(ops, perm, cfg.L, cfg.nex, cfg.degree, cfg.tol, cfg.max_iter, seed=7)
    ev = evals.cpu().numpy()
    vecs = evecs.cpu().numpy()
    for k, i in enumerate(perm):
        assert stats[k]["status"] == 0, stats[k]
        check_pairs(f, int(i), ev[k], vecs[k, :, :f.n].T, cfg.L, paper_tol=PAPER_TOL_SLACK * cfg.tol)
    assert all(s["warm"] == (k > 0) for k, s in enumerate(stats))


@pytest.mark.parametrize("cfg_name,count", [("C2", 5), ("C3", 2), ("C4", 2)])
def test_full_size_chain_sample(lib, cfg_name, count):
    """Full-size operators from the head of the sorted queue, solved as one warm chain."""
    cfg = synth.get_config(cfg_name)
    f = synth.make_batch(cfg, 24)
    ops, params = device_problem(f)
    perm, _, _ = lib.sort(params, cfg.dim, cfg.nx, cfg.p0)
    chain = perm[:count]
    evals, evecs, stats = lib.solve_queue(ops, chain, cfg.L, cfg.nex, cfg.degree, cfg.tol, cfg.max_iter, seed=3)
    ev = evals.cpu().numpy()
    for k, i in enumerate(chain):
        assert stats[k]["status"] == 0, stats[k]
        V = evecs[k, :, :f.n].cpu().numpy().T
        check_pairs(f, int(i), ev[k], V, cfg.L, paper_tol=PAPER_TOL_SLACK * cfg.tol)


def test_c5_full_size_properties(lib):
    """configs[4] (b = 360, global-memory small kernels): residual, orthonormality, Loewner bounds."""
    cfg = synth.get_config("C5")
    f = synth.make_batch(cfg, 1)
    ops, _ = device_problem(f)
    evals, evecs, st = lib.solve_one(ops, 0, cfg.L, cfg.nex, cfg.degree, cfg.tol, cfg.max_iter, seed=5)
    lam = evals.cpu().numpy()[:cfg.L]
    V = _np_block(evecs, f.n)[:, :cfg.L]
    A = oop.assemble_csr(f, 0)
    normA = float(np.abs(A).sum(axis=1).max())
    assert checks.resid_over_normA(A, lam, V, normA).max() <= 1e-8
    assert checks.rel_residual(A, lam, V).max() <= PAPER_TOL_SLACK * cfg.tol
    assert checks.orth_error(V) <= 1e-12
    lo, hi = checks.loewner_bounds(f, 0, cfg.L)
    assert np.all(lo <= lam * (1 + 1e-12)) and np.all(lam <= hi * (1 + 1e-12))
    assert np.all(np.diff(lam) >= 0)


# ----------------------------------------------------------------- edge cases ----
def test_exact_warm_start_converges_without_filtering(lib):
    # warm start from the exact eigenvectors of the same operator locks at once
    cfg = synth.get_config("C1")
    f = synth.make_batch(cfg, 1)
    ops, _ = device_problem(f)
    ev, vecs, st = lib.solve_one(ops, 0, cfg.L, cfg.nex, 20, 1e-8, 200, seed=2)
    ev2, vecs2, st2 = lib.solve_one(ops, 0, cfg.L, cfg.nex, 20, 1e-8, 200, warm=vecs, seed=2)
    assert st2["iterations"] <= 1
    assert np.abs(ev2.cpu().numpy()[:cfg.L] - ev.cpu().numpy()[:cfg.L]).max() <= 1e-12 * ev.cpu().numpy()[cfg.L - 1]


def test_identical_operators_chain(lib):
    # N = 2 identical problems -> the second solve needs (almost) no iteration
    cfg = synth.get_config("C1")
    f = synth.make_batch(cfg, 1)
    f2 = f.subset([0, 0])
    ops, _ = device_problem(f2)
    evals, evecs, stats = lib.solve_queue(ops, [0, 1], cfg.L, cfg.nex, 20, 1e-8, 200, seed=4)
    assert stats[1]["iterations"] <= 1 < stats[0]["iterations"]


def test_tiny_full_block_and_odd_sizes(lib):
    # b = n (whole spectrum), odd b, L = 1, degree 1.  nex = 0 with b < n is not a case the
    # method converges on (lambda_L sits at the edge of the damped interval [alpha, beta]).
    f = synth.make_batch(synth.get_config("C1").with_(nx=5), 1)
    ops, _ = device_problem(f)
    D = oop.assemble_dense(f, 0)
    w = np.linalg.eigvalsh(D)
    for L, nex, m in [(25, 0, 8), (7, 2, 1), (1, 1, 20), (1, 3, 5), (24, 1, 3)]:
        ev, vecs, st = lib.solve_one(ops, 0, L, nex, m, 1e-10, 500, seed=9)
        assert np.abs(ev.cpu().numpy()[:L] - w[:L]).max() <= 1e-9 * w[:L].max(), (L, nex, m)


def test_no_extra_columns_is_reported_not_garbage(lib):
    """nex = 0 with b = L < n: the damped interval [alpha, beta] starts at the L-th Ritz value itself
    (reading R9), so that pair gains nothing per filter and the method need not converge.  The solve
    must then end cleanly: SCSF_ERR_NUMERICAL or OK, finite outputs, and correct values when OK."""
    f = synth.make_batch(synth.get_config("C1").with_(nx=12), 1)
    ops, _ = device_problem(f)
    w = np.linalg.eigvalsh(oop.assemble_dense(f, 0))
    ev, vecs, st = lib.solve_one(ops, 0, 8, 0, 20, 1e-8, 60, seed=3, raise_on_fail=False)
    e = ev.cpu().numpy()[:8]
    assert st["status"] in (lib.SCSF_OK, lib.SCSF_ERR_NUMERICAL)
    assert np.all(np.isfinite(e)) and bool(torch_isfinite(vecs))
    if st["status"] == lib.SCSF_OK:
        assert np.abs(e - w[:8]).max() <= 1e-9 * w[7]
    else:
        assert st["n_locked"] < 8 and st["iterations"] == 60


def torch_isfinite(t):
    import torch
    return torch.isfinite(t).all()


def test_max_iter_zero_reports_not_converged(lib):
    cfg = synth.get_config("C1")
    f = synth.make_batch(cfg, 1)
    ops, _ = device_problem(f)
    with pytest.raises(lib.NotConverged):
        lib.solve_one(ops, 0, cfg.L, cfg.nex, 20, 1e-8, 0, seed=1)
    ev, vecs, st = lib.solve_one(ops, 0, cfg.L, cfg.nex, 20, 1e-8, 0, seed=1, raise_on_fail=False)
    assert st["status"] == lib.SCSF_ERR_NUMERICAL and st["max_rel_resid"] > 1e-8


def test_bad_arguments(lib):
    import torch
    f = synth.make_batch(synth.get_config("C1").with_(nx=6), 1)
    ops, _ = device_problem(f)
    for L, nex, m, tol in [(0, 1, 20, 1e-8), (30, 10, 20, 1e-8), (4, 1, 0, 1e-8), (4, 1, 20, 0.0), (4, 1, -3, 1e-8),
                           (4, 1, 257, 1e-8), (4, 1, -257, 1e-8)]:
        with pytest.raises(lib.ScsfError) as ei:
            lib.solve_one(ops, 0, L, nex, m, tol, 10)
        assert ei.value.code == lib.SCSF_ERR_ARG
    with pytest.raises(lib.ScsfError) as ei:
        lib.solve_one(ops, 0, 4, 1, 20, 1e-8, 10, ws=torch.empty(1024, dtype=torch.uint8, device="cuda"))
    assert ei.value.code == lib.SCSF_ERR_WORKSPACE
    with pytest.raises(lib.ScsfError):
        lib.solve_queue(ops, [0, 3], 4, 1)


def test_empty_chain(lib):
    f = synth.make_batch(synth.get_config("C1").with_(nx=6), 1)
    ops, _ = device_problem(f)
    evals, evecs, stats = lib.solve_queue(ops, [], 4, 1)
    assert evals.shape[0] == 0 and stats == []


def test_launch_count_increases(lib):
    f = synth.make_batch(synth.get_config("C1").with_(nx=6), 1)
    ops, _ = device_problem(f)
    before = lib.launch_count()
    lib.solve_one(ops, 0, 4, 1, 8, 1e-8, 100)
    assert lib.launch_count() > before


def test_solve_chains_matches_single_chains_bitwise(lib):
    """scsf_solve_chains runs contiguous slices concurrently; each slice must equal scsf_solve_queue
    on the same slice bit for bit (deterministic kernels, no cross-chain state)."""
    import torch
    cfg = synth.get_config("C1")
    f = synth.make_batch(cfg, 24)
    ops, params = device_problem(f)
    perm, _, _ = lib.sort(params, cfg.dim, cfg.nx, cfg.p0)
    starts = lib.split_chains(len(perm), 3)
    ev, vec, st = lib.solve_chains(ops, perm, 3, cfg.L, cfg.nex, cfg.degree, cfg.tol, cfg.max_iter, seed=11)
    for c in range(3):
        a, b = starts[c], starts[c + 1]
        ev1, vec1, st1 = lib.solve_queue(ops, perm[a:b], cfg.L, cfg.nex, cfg.degree, cfg.tol, cfg.max_iter, seed=11)
        assert torch.equal(ev[a:b], ev1) and torch.equal(vec[a:b], vec1)
        assert [s["iterations"] for s in st[a:b]] == [s["iterations"] for s in st1]
        assert st[a]["warm"] == 0 and all(s["warm"] == 1 for s in st[a + 1:b])
    for k in (0, 7, 8, 23):
        check_pairs(f, int(perm[k]), ev[k].cpu().numpy(), vec[k, :, :f.n].cpu().numpy().T, cfg.L,
                    paper_tol=PAPER_TOL_SLACK * cfg.tol)


def test_solve_chains_more_chains_than_operators(lib):
    cfg = synth.get_config("C1")
    f = synth.make_batch(cfg, 3)
    ops, _ = device_problem(f)
    ev, vec, st = lib.solve_chains(ops, [2, 0, 1], 8, cfg.L, cfg.nex, seed=1)
    assert all(s["status"] == 0 and s["warm"] == 0 for s in st)


def test_solve_chains_host_streams_identical_results(lib):
    """scsf_solve_chains_host (pairs streamed to pinned host memory while the chains run) returns
    exactly what scsf_solve_chains leaves on the device."""
    import torch
    cfg = synth.get_config("C1")
    f = synth.make_batch(cfg, 24)
    ops, params = device_problem(f)
    perm, _, _ = lib.sort(params, cfg.dim, cfg.nx, cfg.p0)
    ev, vec, st = lib.solve_chains(ops, perm, 5, cfg.L, cfg.nex, cfg.degree, cfg.tol, cfg.max_iter, seed=21)
    he = torch.empty((len(perm), cfg.L), dtype=torch.float64).pin_memory()
    hv = torch.zeros((len(perm), cfg.L, f.n + 3), dtype=torch.float64).pin_memory()
    st2 = lib.solve_chains_host(ops, perm, 5, cfg.L, cfg.nex, he, hv, cfg.degree, cfg.tol, cfg.max_iter, seed=21)
    assert [s["iterations"] for s in st2] == [s["iterations"] for s in st]
    assert torch.equal(he, ev.cpu())
    assert torch.equal(hv[:, :, :f.n], vec[:, :, :f.n].cpu())
    he2 = torch.empty((len(perm), cfg.L), dtype=torch.float64).pin_memory()
    lib.solve_chains_host(ops, perm, 5, cfg.L, cfg.nex, he2, None, cfg.degree, cfg.tol, cfg.max_iter, seed=21)
    assert torch.equal(he2, ev.cpu())


# --------------------------------------------------- adaptive degree ----
@pytest.mark.parametrize("cfg_name,nx,L,n_ops,cap", [("C1", 32, 16, 6, 20),     # register-patch resident filter
                                                      ("C2", 100, 40, 4, 40),    # cluster-resident filter
                                                      ("C4", 20, 24, 4, 40),     # 3-D streaming step (k_stencil_v4)
                                                      ("C5", 500, 20, 2, 60)])   # 2-D streaming step
def test_adaptive_degree_matches_oracle(lib, cfg_name, nx, L, n_ops, cap):
    """degree < 0 (Alg. 1 l. 5's per-column degrees, capped at |degree|) reaches the same
    eigenpairs as the uniform degree, with fewer filtered column-steps."""
    cfg = synth.get_config(cfg_name).with_(nx=nx, L=L)
    f = synth.make_batch(cfg, n_ops)
    ops, params = device_problem(f)
    perm, _, _ = lib.sort(params, cfg.dim, cfg.nx, cfg.p0)
    ev_u, _, st_u = lib.solve_queue(ops, perm, cfg.L, cfg.nex, cap, cfg.tol, 400, seed=4, want_vecs=False)
    ev, vec, st = lib.solve_queue(ops, perm, cfg.L, cfg.nex, -cap, cfg.tol, 400, seed=4)
    e = ev.cpu().numpy()
    for k, i in enumerate(perm):
        assert st[k]["status"] == 0, st[k]
        check_pairs(f, int(i), e[k], vec[k, :, :f.n].cpu().numpy().T, cfg.L, paper_tol=PAPER_TOL_SLACK * cfg.tol)
    assert np.abs(e - ev_u.cpu().numpy()).max() <= 1e-9 * np.abs(e).max()
    # work: column-steps of the adaptive filter never exceed the uniform degree's per iteration
    steps_a = sum(s["spmm_columns"] for s in st) / max(1, sum(s["iterations"] for s in st))
    steps_u = sum(s["spmm_columns"] for s in st_u) / max(1, sum(s["iterations"] for s in st_u))
    assert steps_a <= steps_u * (1 + 1e-12), (steps_a, steps_u)


@pytest.mark.parametrize("degree", [40, -40])
def test_filter_split_sync_bitwise(lib, degree, monkeypatch):
    """The step synchronisation of k_filter_cl changes no arithmetic: a C3-shaped chain (200 x 200, the
    16-CTA cluster kernel, an empty top CTA) solved with the split arrive / wait (SCSF_FILTER_SPLIT=1) or
    the mbarrier neighbour sync with st.async ghost pushes (=2) returns bitwise the eigenpairs of the
    per-step cluster barrier (=0), uniform and per-column degrees."""
    import torch
    monkeypatch.delenv("SCSF_FILTER_STREAMING", raising=False)
    cfg = synth.get_config("C3").with_(L=24)
    f = synth.make_batch(cfg, 2)
    ops, params = device_problem(f)
    perm, _, _ = lib.sort(params, cfg.dim, cfg.nx, cfg.p0)
    out = []
    for split in ("0", "1", "2"):
        monkeypatch.setenv("SCSF_FILTER_SPLIT", split)
        ev, vec, st = lib.solve_queue(ops, perm, cfg.L, cfg.nex, degree, cfg.tol, 400, seed=9)
        assert all(s["status"] == 0 for s in st), st
        out.append((ev.cpu(), vec.cpu()))
    for k in (1, 2):
        assert torch.equal(out[0][0], out[k][0]) and torch.equal(out[0][1], out[k][1]), k


@pytest.mark.parametrize("nx", [200, 198, 164, 92])
def test_filter_trimmed_cluster_bitwise(lib, nx, monkeypatch):
    """Launching only the CTAs whose slab holds rows (SCSF_FILTER_TRIM=1: 15 of 16 on 200 x 200 and
    198 x 198, whose 14-row slabs cover 210 rows; 14 of 16 on 164 x 164; 92 x 92 fills its 8) changes
    no arithmetic: the filtered block, including its zeroed ld padding (written by the last CTA
    launched), is bitwise that of the full cluster, and both match the oracle (Alg. 1)."""
    import torch
    monkeypatch.delenv("SCSF_FILTER_STREAMING", raising=False)
    cfg = synth.get_config("C3").with_(nx=nx)
    f = synth.make_batch(cfg, 1)
    ops, _ = device_problem(f)
    n, ld, k, m = f.n, ops.ld, 7, 11
    Y0 = np.random.default_rng(21).standard_normal((n, k))
    A = oop.assemble_csr(f, 0)
    normA = float(np.abs(A).sum(axis=1).max())
    lam, alpha = 0.002 * normA, 0.1 * normA
    c, e = (alpha + normA) / 2, (normA - alpha) / 2
    outs = []
    for trim in ("0", "1"):
        monkeypatch.setenv("SCSF_FILTER_TRIM", trim)
        Yd = torch.full((k, ld), 7.0, dtype=torch.float64, device="cuda")
        Yd[:, :n] = torch.from_numpy(Y0.T.copy())
        outs.append(lib.cheb_filter(ops, 0, Yd, m, lam, c, e).cpu())
    assert torch.equal(outs[0], outs[1])
    ref = ofilt.cheb_filter(A, Y0, m, lam, c, e)
    Ym = _np_block(outs[1].cuda(), n)
    assert np.all(np.abs(Ym - ref).max(axis=0) <= 1e-12 * np.abs(ref).max(axis=0))
