"""Row-partitioned solve (BASELINE.json configs[4]) — GPU.

One GPU is available to this run, so the multi-rank path is exercised with the
in-process loopback communicator: `world` virtual ranks on one device, each on
its own host thread and CUDA stream, exchanging halos / all-reduces through
host barriers (no kernel waits on another rank).  The NCCL backend runs with
world = 1 (the same slab kernels; every collective is the identity).  Every
result is compared with the oracle (and with the one-GPU solve), at the same
acceptance as tests/test_gpu_solve.py.
"""
import threading

import numpy as np
import pytest

import synth
from oracle import checks, eig as oeig, operator as oop
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


def _run_loopback(lib, ops, chain, L, nex, world, degree=20, tol=1e-8, seed=11):
    import torch
    comms = lib.comm_create_loopback(world)
    out = [None] * world
    err = [None] * world

    def work(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                res = lib.solve_queue_dist(ops, chain, L, nex, comms[r], degree, tol, seed=seed, stream=st)
            st.synchronize()
            out[r] = res
        except Exception as e:        # surfaced below
            err[r] = e

    th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for c in comms:
        c.close()
    for e in err:
        if e is not None:
            raise e
    return out


def _assemble_slabs(out, nx, n):
    """Stack the ranks' slab rows into global [n_chain, L, n] (numpy)."""
    parts = []
    for ev, vec, st, (y0, y1) in out:
        parts.append(vec[:, :, :nx * (y1 - y0)].cpu().numpy())
    full = np.concatenate(parts, axis=2)
    assert full.shape[2] == n
    return full


@pytest.mark.parametrize("world,nx", [(2, 40), (3, 40), (4, 36)])
def test_loopback_row_partition_matches_oracle(lib, world, nx):
    """configs[4]-family operator (-Lap u + V u) split over 2, 3 (ragged rows) and 4 slabs."""
    cfg = synth.get_config("C5").with_(nx=nx, L=12)
    f = synth.make_batch(cfg, 3)
    ops, _ = device_problem(f)
    chain = np.array([2, 0, 1], dtype=np.int32)
    out = _run_loopback(lib, ops, chain, cfg.L, cfg.nex, world)
    ev0 = out[0][0].cpu().numpy()
    for r in range(1, world):                      # replicated b x b work: identical on every rank
        assert np.array_equal(out[r][0].cpu().numpy(), ev0)
        assert [s["iterations"] for s in out[r][2]] == [s["iterations"] for s in out[0][2]]
    V = _assemble_slabs(out, nx, f.n)
    for k, i in enumerate(chain):
        assert out[0][2][k]["status"] == 0, out[0][2][k]
        check_pairs(f, int(i), ev0[k], V[k].T, cfg.L, paper_tol=PAPER_TOL_SLACK * cfg.tol)
    # same answer as the one-GPU solve (different reduction order: not bitwise)
    ev1, vec1, st1 = lib.solve_queue(ops, chain, cfg.L, cfg.nex, cfg.degree, cfg.tol, cfg.max_iter, seed=11)
    e1 = ev1.cpu().numpy()
    assert np.abs(ev0 - e1).max() <= 1e-10 * np.abs(e1).max()


@pytest.mark.parametrize("world,nx", [(1, 40), (2, 40), (3, 36)])
def test_loopback_row_partition_adaptive_degree(lib, world, nx):
    """Per-column degrees (degree < 0, Alg. 1 l. 5's staggered update P:175) through the
    row partition's slab step: every rank picks the same degrees (k_lock on all-reduced residuals),
    finished columns are skipped, and the pairs match the oracle and the one-GPU adaptive solve."""
    cfg = synth.get_config("C5").with_(nx=nx, L=12)
    f = synth.make_batch(cfg, 3)
    ops, _ = device_problem(f)
    chain = np.array([1, 2, 0], dtype=np.int32)
    out = _run_loopback(lib, ops, chain, cfg.L, cfg.nex, world, degree=-40)
    ev0 = out[0][0].cpu().numpy()
    for r in range(1, world):
        assert np.array_equal(out[r][0].cpu().numpy(), ev0)
    V = _assemble_slabs(out, nx, f.n)
    for k, i in enumerate(chain):
        assert out[0][2][k]["status"] == 0, out[0][2][k]
        check_pairs(f, int(i), ev0[k], V[k].T, cfg.L, paper_tol=PAPER_TOL_SLACK * cfg.tol)
    ev1, _, st1 = lib.solve_queue(ops, chain, cfg.L, cfg.nex, -40, cfg.tol, cfg.max_iter, seed=11)
    e1 = ev1.cpu().numpy()
    assert np.abs(ev0 - e1).max() <= 1e-10 * np.abs(e1).max()
    # fewer filtered column-steps than the uniform degree 40 would apply
    it = sum(s["iterations"] for s in out[0][2])
    assert sum(s["spmm_columns"] for s in out[0][2]) < it * (40 + 2) * (cfg.L + cfg.nex)


def test_loopback_chain_head_random_block_is_partition_independent(lib):
    """The cold start draws the same global random block on any partition (global row hash):
    the 1-slab and 2-slab loopback solves of a chain head agree to rounding."""
    cfg = synth.get_config("C5").with_(nx=32, L=8)
    f = synth.make_batch(cfg, 1)
    ops, _ = device_problem(f)
    chain = np.array([0], dtype=np.int32)
    a = _run_loopback(lib, ops, chain, cfg.L, cfg.nex, 1)
    b = _run_loopback(lib, ops, chain, cfg.L, cfg.nex, 2)
    ea, eb = a[0][0].cpu().numpy(), b[0][0].cpu().numpy()
    assert np.abs(ea - eb).max() <= 1e-10 * np.abs(ea).max()
    assert a[0][2][0]["iterations"] == b[0][2][0]["iterations"]


def test_nccl_world1_matches_oracle(lib):
    """The NCCL backend (libnccl resolved from the process) on one rank: the slab kernels with
    identity collectives, compared with the oracle."""
    import torch
    uid = lib.comm_unique_id()
    comm = lib.comm_create(0, 1, uid)
    cfg = synth.get_config("C5").with_(nx=48, L=16)
    f = synth.make_batch(cfg, 2)
    ops, _ = device_problem(f)
    chain = np.array([1, 0], dtype=np.int32)
    ev, vec, st, rows = lib.solve_queue_dist(ops, chain, cfg.L, cfg.nex, comm, seed=2)
    torch.cuda.synchronize()
    comm.close()
    assert rows == (0, cfg.nx)
    e = ev.cpu().numpy()
    for k, i in enumerate(chain):
        assert st[k]["status"] == 0
        check_pairs(f, int(i), e[k], vec[k, :, :f.n].cpu().numpy().T, cfg.L, paper_tol=PAPER_TOL_SLACK * cfg.tol)


def test_dist_bad_arguments(lib):
    import torch
    comms = lib.comm_create_loopback(1)
    try:
        f3 = synth.make_batch(synth.get_config("C4").with_(nx=8, L=4), 1)
        ops3, _ = device_problem(f3)
        with pytest.raises(lib.ScsfError):                     # 3-D: not row-partitioned
            lib.solve_queue_dist(ops3, [0], 4, 1, comms[0])
        f2 = synth.make_batch(synth.get_config("C5").with_(nx=30, L=4), 1)
        ops2, _ = device_problem(f2)
        with pytest.raises(lib.ScsfError):                     # nx % 4 != 0
            lib.solve_queue_dist(ops2, [0], 4, 1, comms[0])
    finally:
        for c in comms:
            c.close()
    torch.cuda.synchronize()
