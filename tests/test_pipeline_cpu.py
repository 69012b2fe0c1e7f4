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
