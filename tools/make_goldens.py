"""Write the oracle goldens of the full-size parity tests (tests/golden/*.npz).

Calls ONLY oracle/ (and the seeded input generator synth/, which holds none of the
method's arithmetic): nothing here comes from the CUDA path.  Each file holds, for a
stated sample of operators of one BASELINE.json config at full size,

  lam     [k, L + 8]  the oracle's smallest eigenvalues (oracle.eig.smallest_eigpairs,
                      shift-invert block Lanczos; it raises rather than return an
                      unconverged pair), the definition of the result
  resid   [k, L + 8]  their true residuals ||A v - lam v||_2
  sig_lo, sig_hi [k]  lam_L (1 -/+ eta), eta = 1e-9
  n_lo, n_hi     [k]  Sylvester inertia counts of A - sigma I at those shifts
                      (oracle.checks.inertia_blocks): the number of eigenvalues of A
                      below sigma, so "no eigenvalue below lam_L was missed"
  ops, pos       [k]  operator index and its position in the sorted queue
  perm           [N]  the oracle's truncated-FFT greedy order (oracle.sort, Alg. 2)

Samples (positions in the sorted queue cut into CHAINS contiguous chains, the way
tests/test_gpu_bench_config.py and bench.py run it):
  C3  every chain's head and tail (32 + 32) + 8 seeded picks
  C4  the heads and tails of chains 0, 8, 16, 24 + 8 seeded picks (a C4 operator
      costs ~2 min of oracle time here: banded Cholesky of half-bandwidth 1600)
  C5  operators 0 and 1 (the 2-operator chain of tests/test_gpu_c5.py)

  python tools/make_goldens.py C5 C3 C4
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from oracle import checks, eig, sort as osort  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
CHAINS = 32
ETA = 1e-9
GUARD = 8


def queue_sample(N, chains, chain_ids, picks, seed=0):
    starts = [(c * N) // chains for c in range(chains + 1)]
    pos = set()
    for c in chain_ids:
        pos.add(starts[c])
        pos.add(starts[c + 1] - 1)
    rng = np.random.default_rng(seed)
    pos |= set(int(x) for x in rng.choice(N, picks, replace=False))
    return sorted(pos)


def run(name):
    cfg = synth.get_config(name)
    f = synth.make_batch(cfg)
    perm = np.arange(cfg.n_ops, dtype=np.int32)
    if name == "C5":
        pos = [0, 1]
        ops = [0, 1]
    else:
        perm, _, _, _ = osort.sort_problems(f.params, cfg.dim, cfg.nx, cfg.p0)
        perm = np.asarray(perm, dtype=np.int32)
        ids = range(CHAINS) if name == "C3" else range(0, CHAINS, 8)
        pos = queue_sample(cfg.n_ops, CHAINS, ids, 8)
        ops = [int(perm[k]) for k in pos]
    k = cfg.L + GUARD
    out = {key: [] for key in ("lam", "resid", "sig_lo", "sig_hi", "n_lo", "n_hi", "krylov")}
    for j, op in enumerate(ops):
        t0 = time.time()
        r = eig.smallest_eigpairs(f, op, k)
        lamL = float(r.lam[cfg.L - 1])
        lo, hi = lamL * (1 - ETA), lamL * (1 + ETA)
        n_lo = checks.inertia_blocks(f, op, lo)
        n_hi = checks.inertia_blocks(f, op, hi)
        assert n_lo == int(np.sum(r.lam < lo)) and n_hi >= cfg.L, (op, n_lo, n_hi)
        for key, v in (("lam", r.lam), ("resid", r.resid), ("sig_lo", lo), ("sig_hi", hi), ("n_lo", n_lo),
                       ("n_hi", n_hi), ("krylov", r.krylov_dim)):
            out[key].append(v)
        print(f"{name} {j + 1}/{len(ops)} op {op}: lam_L {lamL:.10g} counts {n_lo}/{n_hi} "
              f"krylov {r.krylov_dim} {time.time() - t0:.1f}s", flush=True)
    path = os.path.join(GOLDEN, f"{name.lower()}_oracle.npz")
    np.savez(path, pos=np.array(pos, dtype=np.int32), ops=np.array(ops, dtype=np.int32), perm=perm,
             lam=np.array(out["lam"]), resid=np.array(out["resid"]), sig_lo=np.array(out["sig_lo"]),
             sig_hi=np.array(out["sig_hi"]), n_lo=np.array(out["n_lo"], dtype=np.int64),
             n_hi=np.array(out["n_hi"], dtype=np.int64), krylov=np.array(out["krylov"], dtype=np.int64),
             L=cfg.L, eta=ETA, chains=CHAINS, tool="tools/make_goldens.py")
    print("wrote", path, flush=True)


if __name__ == "__main__":
    for name in sys.argv[1:] or ["C5", "C3", "C4"]:
        run(name)
