"""Checkpoint / resume host logic (pipeline.run_resumable) — CPU.

The solver is replaced by a stand-in whose outputs depend on the whole warm-start history
of a chain (every value folds in the chain state it received), so a resumed run matches an
uninterrupted one only if segments, positions and chain states are carried exactly.
"""
import json
import os

import numpy as np
import pytest
import torch

from paper_2510_23215_b200 import scsf
from paper_2510_23215_b200.pipeline import SolveParams, run_resumable, segment_plan

SD = 5          # state doubles of the stand-in


def fake_solve(ops, queue, starts, L, nex, state_in, state_out, calls=None, fail_at=None, **kw):
    if calls is not None:
        calls.append(len(queue))
        if fail_at is not None and len(calls) == fail_at:
            raise RuntimeError("simulated crash")
    nq = len(queue)
    evals = torch.empty((nq, L), dtype=torch.float64)
    stats = []
    for c in range(len(starts) - 1):
        acc = float(state_in[c, 0]) if state_in is not None else 0.0
        for k in range(starts[c], starts[c + 1]):
            acc = acc * 1.5 + float(queue[k]) + 1.0
            evals[k] = acc + torch.arange(L, dtype=torch.float64)
            stats.append({"status": 0, "iterations": int(queue[k]) % 7, "max_rel_resid": 1e-9 * (k + 1)})
        state_out[c] = acc
    return evals, None, stats


def direct(queue, n_chains, L):
    """What one pass over every chain gives (no segments)."""
    starts = scsf.split_chains(len(queue), n_chains)
    out = np.empty((len(queue), L))
    for c in range(len(starts) - 1):
        acc = 0.0
        for k in range(starts[c], starts[c + 1]):
            acc = acc * 1.5 + float(queue[k]) + 1.0
            out[k] = acc + np.arange(L)
    return out


def run(tmp, queue, n_chains, segment, **kw):
    sp = SolveParams(L=3, nex=1)
    return run_resumable(None, queue, n_chains, sp, str(tmp), segment=segment, state_doubles=SD, n=4,
                         device=torch.device("cpu"), **kw)


@pytest.mark.parametrize("N,chains,segment", [(23, 4, 2), (10, 3, 4), (8, 8, 1), (5, 2, 9), (40, 6, 3)])
def test_segment_plan_covers_queue_in_chain_order(N, chains, segment):
    starts = scsf.split_chains(N, chains)
    plan = segment_plan(starts, segment)
    seen = np.concatenate([p for p, _ in plan]) if plan else np.array([], dtype=np.int64)
    assert sorted(seen.tolist()) == list(range(N))
    for c in range(len(starts) - 1):               # each chain's positions in increasing order, segment-sized
        mine = [p[s[c]:s[c + 1]] for p, s in plan]
        flat = np.concatenate(mine)
        assert flat.tolist() == list(range(starts[c], starts[c + 1]))
        assert all(len(m) <= segment for m in mine)


@pytest.mark.parametrize("stops", [[1], [2, 1], [1, 1, 1, 1]])
def test_interrupted_run_matches_uninterrupted(tmp_path, stops):
    rng = np.random.default_rng(5)
    queue = rng.permutation(23).astype(np.int32)
    fn = lambda *a, **k: fake_solve(*a, **k)                        # noqa: E731
    done, total = run(tmp_path / "full", queue, 4, 2, solve_fn=fn)
    assert done == total == 3
    for s in stops:                                                  # stop-and-restart several times
        run(tmp_path / "cut", queue, 4, 2, solve_fn=fn, max_segments=s)
    done, total = run(tmp_path / "cut", queue, 4, 2, solve_fn=fn)
    assert done == total
    a = np.load(tmp_path / "full" / "evals.npy")
    b = np.load(tmp_path / "cut" / "evals.npy")
    assert np.array_equal(a, b)
    assert np.array_equal(a, direct(queue, 4, 3))
    assert np.array_equal(np.load(tmp_path / "full" / "stats.npy"), np.load(tmp_path / "cut" / "stats.npy"))
    assert sorted(os.listdir(tmp_path / "cut")) == sorted(os.listdir(tmp_path / "full"))


def test_crash_inside_a_segment_resumes_from_last_checkpoint(tmp_path):
    queue = np.arange(17, dtype=np.int32)[::-1].copy()
    calls = []
    with pytest.raises(RuntimeError):
        run(tmp_path, queue, 3, 2, solve_fn=lambda *a, **k: fake_solve(*a, calls=calls, fail_at=3, **k))
    man = json.load(open(tmp_path / "manifest.json"))
    assert man["cursor"] == 2                                        # segments 0 and 1 were committed
    assert [f for f in os.listdir(tmp_path) if f.startswith("state_")] == ["state_2.npy"]
    calls2 = []
    done, total = run(tmp_path, queue, 3, 2, solve_fn=lambda *a, **k: fake_solve(*a, calls=calls2, **k))
    assert done == total == 3 and len(calls2) == 1                   # only the missing segment re-ran
    assert np.array_equal(np.load(tmp_path / "evals.npy"), direct(queue, 3, 3))


def test_checkpoint_of_another_run_is_refused(tmp_path):
    queue = np.arange(9, dtype=np.int32)
    run(tmp_path, queue, 2, 2, solve_fn=fake_solve, max_segments=1)
    with pytest.raises(ValueError):
        run(tmp_path, queue[::-1].copy(), 2, 2, solve_fn=fake_solve)
    with pytest.raises(ValueError):
        run(tmp_path, queue, 3, 2, solve_fn=fake_solve)


def test_bad_segment():
    with pytest.raises(ValueError):
        segment_plan([0, 4], 0)
