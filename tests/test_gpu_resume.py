"""Resumable chains on the GPU (scsf_solve_chains_resume, pipeline.run_resumable).

A queue solved in checkpointed segments, with the process state thrown away between
calls (new workspace, states round-tripped through .npy files), must give bit-identical
pairs to one scsf_solve_chains pass: the warm start of a resumed operator reads exactly
the block and Ritz values the uninterrupted chain would have handed it.
"""
import numpy as np
import pytest

import synth
from tests.helpers import device_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2510_23215_b200 import scsf
    scsf.load_library()
    return scsf


@pytest.fixture(scope="module")
def c1(lib):
    cfg = synth.get_config("C1")
    f = synth.make_batch(cfg, 24)
    ops, params = device_problem(f)
    perm, _, _ = lib.sort(params, cfg.dim, cfg.nx, cfg.p0)
    return cfg, ops, perm


def test_resume_api_cold_equals_solve_chains(lib, c1):
    import torch
    cfg, ops, perm = c1
    starts = lib.split_chains(len(perm), 4)
    ev0, V0, st0 = lib.solve_chains(ops, perm, 4, cfg.L, cfg.nex, cfg.degree, cfg.tol, cfg.max_iter, seed=7)
    sd = lib.chain_state_doubles(ops, cfg.L, cfg.nex)
    assert sd == (cfg.L + cfg.nex) * (cfg.n + 1)
    out = torch.empty((4, sd), dtype=torch.float64, device="cuda")
    ev1, V1, st1 = lib.solve_chains_resume(ops, perm, starts, cfg.L, cfg.nex, None, out, cfg.degree, cfg.tol,
                                           cfg.max_iter, seed=7, want_vecs=True)
    torch.cuda.synchronize()
    assert torch.equal(ev0, ev1)
    assert torch.equal(V0[:, :, :cfg.n], V1[:, :, :cfg.n])
    b = cfg.L + cfg.nex
    for c in range(4):                        # state = [theta_b | V_b] of the chain's last operator
        last = int(starts[c + 1]) - 1
        assert torch.equal(out[c, :cfg.L], ev0[last])
        Vs = out[c, b:].view(b, cfg.n)
        assert torch.equal(Vs[:cfg.L], V0[last, :, :cfg.n])


def test_segmented_resume_is_bit_identical(lib, c1, tmp_path):
    import torch
    from paper_2510_23215_b200.pipeline import SolveParams, run_resumable
    cfg, ops, perm = c1
    ev0, V0, st0 = lib.solve_chains(ops, perm, 4, cfg.L, cfg.nex, cfg.degree, cfg.tol, cfg.max_iter, seed=7)
    sp = SolveParams(L=cfg.L, nex=cfg.nex, degree=cfg.degree, tol=cfg.tol, max_iter=cfg.max_iter, seed=7)
    done, total = run_resumable(ops, perm, 4, sp, str(tmp_path), segment=2, want_vecs=True, max_segments=1)
    assert (done, total) == (1, 3)
    done, total = run_resumable(ops, perm, 4, sp, str(tmp_path), segment=2, want_vecs=True, max_segments=1)
    assert (done, total) == (2, 3)
    done, total = run_resumable(ops, perm, 4, sp, str(tmp_path), segment=2, want_vecs=True)
    assert (done, total) == (3, 3)
    ev = np.load(tmp_path / "evals.npy")
    V = np.load(tmp_path / "evecs.npy")
    stats = np.load(tmp_path / "stats.npy")
    assert np.array_equal(ev, ev0.cpu().numpy())
    assert np.array_equal(V, V0[:, :, :cfg.n].cpu().numpy())
    assert np.all(stats[:, 0] == 0)
    assert np.array_equal(stats[:, 1], [s["iterations"] for s in st0])


def test_resume_rejects_aliasing(lib, c1):
    import torch
    cfg, ops, perm = c1
    sd = lib.chain_state_doubles(ops, cfg.L, cfg.nex)
    buf = torch.zeros((2, sd), dtype=torch.float64, device="cuda")
    with pytest.raises(lib.ScsfError):
        lib.solve_chains_resume(ops, perm[:4], [0, 2, 4], cfg.L, cfg.nex, buf, buf)
