"""Host logic of the multi-GPU chain split — CPU, gloo world size 2."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_23215_b200.pipeline import chain_bounds, gather_evals


@pytest.mark.parametrize("N,world", [(64, 8), (1000, 8), (7, 3), (3, 8), (0, 2), (200, 1)])
def test_chain_bounds_partition(N, world):
    spans = [chain_bounds(N, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == N
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c and a <= b
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1


def test_chain_bounds_bad_args():
    with pytest.raises(ValueError):
        chain_bounds(10, 0, 0)
    with pytest.raises(ValueError):
        chain_bounds(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N, L, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    perm = np.random.default_rng(0).permutation(N).astype(np.int32)   # same on every rank
    lo, hi = chain_bounds(N, world, rank)
    chain = perm[lo:hi]
    evals = torch.from_numpy(np.stack([np.arange(L) + 1000.0 * i for i in chain]).astype(np.float64)
                             if len(chain) else np.zeros((0, L)))
    full = gather_evals(evals, chain, N, L)
    if rank == 0:
        out_q.put(full.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("N", [9, 2, 1])
def test_gather_evals_gloo_world2(N):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    L = 3
    procs = [ctx.Process(target=_worker, args=(r, 2, port, N, L, q)) for r in range(2)]
    for p in procs:
        p.start()
    full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    expect = np.stack([np.arange(L) + 1000.0 * i for i in range(N)])
    assert np.array_equal(full, expect)


# ------------------------------------------------ row partition (configs[4]) ----
@pytest.mark.parametrize("ny,world", [(500, 8), (10, 3), (7, 7), (100, 1), (63, 4)])
def test_slab_rows_partition_matches_library(ny, world):
    """scsf_slab_rows (host-only C function) == pipeline.slab_partition; contiguous cover, sizes +-1."""
    from paper_2510_23215_b200 import scsf
    from paper_2510_23215_b200.pipeline import slab_partition
    parts = slab_partition(ny, world)
    assert parts == [scsf.slab_rows(ny, world, r) for r in range(world)]
    assert parts[0][0] == 0 and parts[-1][1] == ny
    assert all(b == c for (_, b), (c, _) in zip(parts, parts[1:]))
    sizes = [b - a for a, b in parts]
    assert min(sizes) >= 1 and max(sizes) - min(sizes) <= 1


def _comm_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_23215_b200.pipeline import make_comm
    made = []
    got = make_comm(rank, world, uid_fn=lambda: bytes(range(128)),
                    create_fn=lambda r, w, uid: made.append((r, w, uid)) or (r, w, uid))
    out_q.put((rank, got[0], got[1], got[2] == bytes(range(128))))
    dist.barrier()
    dist.destroy_process_group()


def test_make_comm_broadcasts_rank0_id_gloo_world2():
    """The NCCL bootstrap: rank 0's unique id reaches every rank through torch.distributed."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_comm_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res == [(0, 0, 2, True), (1, 1, 2, True)]


def _slab_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_23215_b200.pipeline import gather_slabs, slab_partition
    nx, ny, nc, L = 4, 7, 2, 3
    full = torch.arange(nc * L * nx * ny, dtype=torch.float64).reshape(nc, L, nx * ny)
    y0, y1 = slab_partition(ny, world)[rank]
    local = torch.zeros((nc, L, 32), dtype=torch.float64)
    local[:, :, :nx * (y1 - y0)] = full[:, :, nx * y0:nx * y1]
    out = gather_slabs(local, nx, (y0, y1), ny)
    if rank == 0:
        out_q.put(bool(torch.equal(out, full)))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_slabs_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok
