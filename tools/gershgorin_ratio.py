"""How far the Gershgorin bound (the filter's beta, reading R10) sits above lambda_max, per config.

CPU only: the oracle's own assembly (oracle/operator.py) and ARPACK (scipy eigsh) for lambda_max.
  python tools/gershgorin_ratio.py > profiles/r02_gershgorin_ratio.json
"""
import json
import sys

import numpy as np
import scipy.sparse.linalg as spl

sys.path.insert(0, ".")
import synth  # noqa: E402
from oracle import operator as op  # noqa: E402

out = {}
for name in ["C1", "C2", "C3", "C4", "C5", "V1"]:
    cfg = synth.get_config(name)
    f = synth.make_batch(cfg, 3)
    r = []
    for i in range(3):
        A = op.assemble_csr(f, i)
        g = float(np.abs(A).sum(axis=1).max())
        lm = float(spl.eigsh(A, k=1, which="LA", return_eigenvectors=False, tol=1e-10)[0])
        r.append(g / lm)
    out[name] = {"gershgorin_over_lambda_max": r, "operators": [0, 1, 2]}
print(json.dumps(out, indent=1))
