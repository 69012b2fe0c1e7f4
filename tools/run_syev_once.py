import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2510_23215_b200 import scsf
b = int(sys.argv[1]) if len(sys.argv) > 1 else 120
rng = np.random.default_rng(0)
B = rng.standard_normal((b, b))
G = torch.from_numpy(B + B.T).cuda()
for _ in range(2):
    th, Z, sw = scsf.syev_small(G, return_sweeps=True)
torch.cuda.synchronize()
print("sweeps", sw)
