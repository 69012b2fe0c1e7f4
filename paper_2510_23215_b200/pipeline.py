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


# ------------------------------------------------------------ resumable run ----
# SURVEY f4 / §3 "checkpoint / resume": per-chain cursor plus the last Ritz block persisted, so
# an interrupted dataset run resumes from each chain's last solved operator as a warm start
# (P:270-277).  Every chain's slice of the sorted queue is cut into segments of `segment`
# operators; one call of scsf_solve_chains_resume advances every chain by one segment.  After a
# segment the pairs land in memory-mapped .npy files (by queue position), then the chain states
# go to state_<j>.npy and finally manifest.json's cursor moves to j (each file written to a
# temporary name and renamed), so a crash at any point leaves a consistent checkpoint.
def segment_plan(chain_start, segment: int):
    """[(queue positions of segment j, chain_start of segment j)] for contiguous chains."""
    cs = np.asarray(chain_start, dtype=np.int64)
    if segment < 1:
        raise ValueError("segment must be >= 1")
    nc = len(cs) - 1
    n_seg = int(max(((cs[c + 1] - cs[c] + segment - 1) // segment for c in range(nc)), default=0))
    plan = []
    for j in range(n_seg):
        pos, starts = [], [0]
        for c in range(nc):
            lo = min(int(cs[c]) + j * segment, int(cs[c + 1]))
            hi = min(lo + segment, int(cs[c + 1]))
            pos.extend(range(lo, hi))
            starts.append(starts[-1] + hi - lo)
        plan.append((np.asarray(pos, dtype=np.int64), np.asarray(starts, dtype=np.int32)))
    return plan


def _atomic_write(path, write):
    """write(file object) to path.tmp, fsync, then rename over path."""
    import os
    tmp = f"{path}.tmp"
    with open(tmp, "wb") as fh:
        write(fh)
        fh.flush()
        os.fsync(fh.fileno())
    os.replace(tmp, path)


def run_resumable(ops, queue, n_chains: int, sp: SolveParams, out_dir: str, segment: int = 8,
                  want_vecs: bool = False, max_segments: int | None = None, solve_fn=None,
                  state_doubles: int | None = None, n: int | None = None, device=None):
    """Solve the sorted `queue` as n_chains warm-start chains, checkpointing to `out_dir` after
    every segment; a later call with the same arguments continues where the last one stopped.

    Output files (queue position order): evals.npy [N, L], stats.npy [N, 3] (status,
    iterations, max_rel_resid), evecs.npy [N, L, n] when want_vecs, state_<j>.npy, manifest.json.
    max_segments: stop after that many segments in this call (an interruption, for tests).
    solve_fn / state_doubles / n / device: injection points for host-only tests; default is
    scsf.solve_chains_resume on ops' device.
    Returns (segments done, total segments)."""
    import json
    import os
    queue = np.asarray(queue, dtype=np.int32)
    N = int(queue.shape[0])
    starts = scsf.split_chains(N, n_chains)
    nc = len(starts) - 1
    plan = segment_plan(starts, segment)
    solve_fn = solve_fn or scsf.solve_chains_resume
    if device is None:
        device = ops.coef.device
    n = ops.nx * ops.ny * ops.nz if n is None else n
    sd = scsf.chain_state_doubles(ops, sp.L, sp.nex) if state_doubles is None else state_doubles
    os.makedirs(out_dir, exist_ok=True)
    man_path = os.path.join(out_dir, "manifest.json")
    key = {"N": N, "L": sp.L, "nex": sp.nex, "n": int(n), "n_chains": nc, "segment": int(segment),
           "degree": sp.degree, "tol": sp.tol, "max_iter": sp.max_iter, "seed": sp.seed, "want_vecs": bool(want_vecs),
           "queue_crc": int(np.bitwise_xor.reduce(queue.astype(np.int64) * (1 + np.arange(N, dtype=np.int64))))
           if N else 0}
    fmm = np.lib.format.open_memmap
    if os.path.exists(man_path):
        man = json.load(open(man_path))
        if man["key"] != key:
            raise ValueError(f"{out_dir} holds a checkpoint of a different run: {man['key']} != {key}")
        cursor = int(man["cursor"])
        ev = fmm(os.path.join(out_dir, "evals.npy"), mode="r+")
        sts = fmm(os.path.join(out_dir, "stats.npy"), mode="r+")
        vec = fmm(os.path.join(out_dir, "evecs.npy"), mode="r+") if want_vecs else None
    else:
        cursor = 0
        ev = fmm(os.path.join(out_dir, "evals.npy"), mode="w+", dtype=np.float64, shape=(N, sp.L))
        sts = fmm(os.path.join(out_dir, "stats.npy"), mode="w+", dtype=np.float64, shape=(N, 3))
        vec = (fmm(os.path.join(out_dir, "evecs.npy"), mode="w+", dtype=np.float64, shape=(N, sp.L, n))
               if want_vecs else None)
    state = None
    if cursor > 0:
        state = torch.from_numpy(np.load(os.path.join(out_dir, f"state_{cursor}.npy"))).to(device)
    done_now = 0
    for j in range(cursor, len(plan)):
        if max_segments is not None and done_now >= max_segments:
            break
        pos, seg_starts = plan[j]
        state_out = torch.empty((nc, sd), dtype=torch.float64, device=device)
        evals, evecs, stats = solve_fn(ops, queue[pos], seg_starts, sp.L, sp.nex, state, state_out,
                                       degree=sp.degree, tol=sp.tol, max_iter=sp.max_iter, seed=sp.seed,
                                       want_vecs=want_vecs, raise_on_fail=False)
        ev[pos] = evals.cpu().numpy()
        sts[pos] = np.array([[s["status"], s["iterations"], s["max_rel_resid"]] for s in stats]).reshape(-1, 3)
        if want_vecs:
            vec[pos] = evecs[:, :, :n].cpu().numpy()
            vec.flush()
        ev.flush()
        sts.flush()
        host_state = state_out.cpu().numpy()
        _atomic_write(os.path.join(out_dir, f"state_{j + 1}.npy"),
                      lambda fh: np.save(fh, host_state))
        _atomic_write(man_path, lambda fh: fh.write(json.dumps({"key": key, "cursor": j + 1,
                                                                "segments": len(plan)}).encode()))
        if j > 0 and os.path.exists(os.path.join(out_dir, f"state_{j}.npy")):
            os.remove(os.path.join(out_dir, f"state_{j}.npy"))
        state = state_out
        cursor = j + 1
        done_now += 1
    return cursor, len(plan)
