"""SCSF end to end on one GPU per process (Fig. 1 / Fig. 2 c-e).

    host fields --H2D--> scsf_assemble --> scsf_sort (Alg. 2) --> this rank's
    contiguous chain of the sorted queue ("M independent chunks")
    --> scsf_solve_queue (Alg. 3, warm-started along the chain) --D2H--> results

Multi-GPU: one process per GPU (torchrun).  Every rank computes the same
permutation (the sort is deterministic), solves its own contiguous slice and
nothing crosses GPUs until the final gather of eigenvalues and stats — the
path has no data-path collective; eigenvectors stay on their
rank.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import scsf


def chain_bounds(N: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of the sorted queue owned by `rank` (floor split)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    return (rank * N) // world, ((rank + 1) * N) // world


@dataclass
class SolveParams:
    L: int
    nex: int
    degree: int = 20
    tol: float = 1e-8
    max_iter: int = 200
    p0: int = 20
    seed: int = 0


@dataclass
class DeviceProblem:
    """Inputs resident on one device."""
    dim: int
    nx: int
    h: float
    params: torch.Tensor          # [N, F, n]
    faces: list                   # dim tensors
    c: torch.Tensor               # [N, n]
    ops: scsf.Operators | None = None

    @property
    def n_ops(self) -> int:
        return self.params.shape[0]


def to_device(dim: int, nx: int, h: float, params: np.ndarray, faces, c: np.ndarray, device,
              pinned: bool = True, non_blocking: bool = True) -> DeviceProblem:
    """H2D copy of host arrays (pinned staging so the copies are DMA transfers)."""
    def up(a):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
        if pinned:
            t = t.pin_memory()
        return t.to(device, non_blocking=non_blocking)
    return DeviceProblem(dim, nx, h, up(params), [up(f) for f in faces], up(c))


def host_bytes(params, faces, c) -> int:
    return int(params.nbytes + sum(f.nbytes for f in faces) + c.nbytes)


@dataclass
class RankResult:
    order: np.ndarray             # full sorted queue (perm)
    chain: np.ndarray             # this rank's operator indices, in solve order
    evals: torch.Tensor           # [len(chain), L] (device)
    evecs: torch.Tensor | None    # [len(chain), L, ld] (device) or None
    stats: list = field(default_factory=list)
    d2_best: np.ndarray | None = None


def run_device(prob: DeviceProblem, sp: SolveParams, rank: int = 0, world: int = 1,
               want_vecs: bool = True, ws: torch.Tensor | None = None) -> RankResult:
    """Assemble, sort and solve this rank's chain; everything stays on the device."""
    if prob.ops is None:
        prob.ops = scsf.assemble(prob.dim, prob.nx, prob.h, prob.faces, prob.c)
    p = prob.nx
    perm, best, _ = scsf.sort(prob.params, prob.dim, p, sp.p0)
    lo, hi = chain_bounds(len(perm), world, rank)
    chain = perm[lo:hi]
    evals, evecs, stats = scsf.solve_queue(prob.ops, chain, sp.L, sp.nex, sp.degree, sp.tol, sp.max_iter,
                                           sp.seed, want_vecs=want_vecs, raise_on_fail=False, ws=ws)
    return RankResult(perm, chain, evals, evecs, stats, best)


def generate(dim: int, nx: int, h: float, params: np.ndarray, faces, c: np.ndarray, sp: SolveParams,
             device=None, rank: int = 0, world: int = 1, want_vecs: bool = True):
    """Public end-to-end call on host arrays: returns numpy (chain, evals, evecs, stats).

    evecs is [len(chain), L, n] (host) when want_vecs, else None.
    """
    device = device or torch.device("cuda", torch.cuda.current_device())
    prob = to_device(dim, nx, h, params, faces, c, device)
    res = run_device(prob, sp, rank, world, want_vecs)
    n = nx ** dim
    evals = res.evals.cpu().numpy()
    evecs = None
    if want_vecs and res.evecs is not None:
        evecs = res.evecs[:, :, :n].cpu().numpy()
    return res.chain, evals, evecs, res.stats


def gather_evals(evals: torch.Tensor, chain: np.ndarray, N: int, L: int):
    """All-gather every rank's (chain, evals) into full [N, L] by operator index (rank order).

    Works on any torch.distributed backend (gloo on CPU, nccl on GPUs); the
    only cross-rank exchange of the path, done once at the end.
    """
    import torch.distributed as dist
    world = dist.get_world_size()
    dev = evals.device
    idx = torch.as_tensor(np.asarray(chain, dtype=np.int64), device=dev)
    counts = [None] * world
    dist.all_gather_object(counts, int(idx.numel()))
    maxc = max(counts)
    pad_e = torch.zeros((maxc, L), dtype=torch.float64, device=dev)
    pad_i = torch.full((maxc,), -1, dtype=torch.int64, device=dev)
    pad_e[:idx.numel()] = evals
    pad_i[:idx.numel()] = idx
    ge = [torch.empty_like(pad_e) for _ in range(world)]
    gi = [torch.empty_like(pad_i) for _ in range(world)]
    dist.all_gather(ge, pad_e)
    dist.all_gather(gi, pad_i)
    out = torch.full((N, L), float("nan"), dtype=torch.float64)
    for e, i, cnt in zip(ge, gi, counts):
        out[i[:cnt].cpu()] = e[:cnt].cpu()
    return out


# ------------------------------------------------- row-partitioned operator ----
# configs[4] / SURVEY §8(a) a11: one operator's grid rows split over the ranks
# (scsf_solve_queue_dist); the NCCL communicator is bootstrapped here.
def make_comm(rank: int, world: int, uid_fn=None, create_fn=None):
    """NCCL communicator of this rank: rank 0 makes the 128-byte unique id, torch.distributed
    broadcasts it (any backend), every rank builds its communicator from it."""
    import torch.distributed as dist
    uid_fn = uid_fn or scsf.comm_unique_id
    create_fn = create_fn or scsf.comm_create
    box = [uid_fn() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(box, src=0)
    return create_fn(rank, world, box[0])


def slab_partition(ny: int, world: int) -> list[tuple[int, int]]:
    """Rows [y0, y1) of every rank (scsf_slab_rows; contiguous, sizes differ by at most 1)."""
    return [((r * ny) // world, ((r + 1) * ny) // world) for r in range(world)]


def gather_slabs(evecs_local: torch.Tensor, nx: int, rows: tuple[int, int], ny: int):
    """All-gather every rank's slab rows of [n_chain, L, ld_loc] eigenvectors into [n_chain, L, nx ny]."""
    import torch.distributed as dist
    world = dist.get_world_size()
    y0, y1 = rows
    n_loc = nx * (y1 - y0)
    parts = slab_partition(ny, world)
    maxrows = max(b - a for a, b in parts)
    nc, L = evecs_local.shape[0], evecs_local.shape[1]
    pad = torch.zeros((nc, L, nx * maxrows), dtype=evecs_local.dtype, device=evecs_local.device)
    pad[:, :, :n_loc] = evecs_local[:, :, :n_loc]
    got = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(got, pad)
    return torch.cat([g[:, :, :nx * (b - a)] for g, (a, b) in zip(got, parts)], dim=2)
