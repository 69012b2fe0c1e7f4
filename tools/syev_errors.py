"""Accuracy of scsf_syev_small (eigenvalues, orthogonality, residual) for b around the block-Jacobi switch."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2510_23215_b200 import scsf

rng = np.random.default_rng(0)
for b in (120, 129, 133, 160, 240, 360):
    for kind in ("dense", "warm"):
        if kind == "dense":
            B = rng.standard_normal((b, b)); G = B + B.T
        else:
            d = np.sort(rng.uniform(10, 2000, b)); E = rng.standard_normal((b, b)) * 1e-6 * d.max(); G = np.diag(d) + E + E.T
        th, Z, sw = scsf.syev_small(torch.from_numpy(G.T.copy()).cuda(), return_sweeps=True)
        th = th.cpu().numpy(); Zn = Z.cpu().numpy().T
        w = np.linalg.eigvalsh(G); sc = np.abs(w).max()
        print(f"b={b} {kind}: sweeps {sw} ev {np.abs(th - w).max() / sc:.2e} orth {np.abs(Zn.T @ Zn - np.eye(b)).max():.2e} "
              f"res {np.abs(G @ Zn - Zn * th).max() / sc:.2e} sorted {bool(np.all(np.diff(th) >= 0))}")
