import sys, time, torch
sys.path.insert(0, ".")
import synth
from paper_2510_23215_b200 import scsf
cfg = synth.get_config("C2")
f = synth.make_batch(cfg, 1000)
dev = torch.device("cuda", 0)
faces = [torch.from_numpy(x).to(dev) for x in f.faces]
ops = scsf.assemble(cfg.dim, cfg.nx, cfg.h, faces, torch.from_numpy(f.c).to(dev))
params = torch.from_numpy(f.params).to(dev)
perm, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.p0)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _, _, st = scsf.solve_chains(ops, perm, 32, cfg.L, cfg.nex, cfg.degree, 1e-300, 7, seed=1, want_vecs=False, raise_on_fail=False)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
print(sys.argv[1] if len(sys.argv) > 1 else "", f"{dt*1e3:.1f} ms", "iters", sum(s["iterations"] for s in st), "fallbacks", sum(s["cholqr_fallbacks"] for s in st))
