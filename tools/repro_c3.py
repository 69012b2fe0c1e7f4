import sys; sys.path.insert(0,'.')
import synth, numpy as np, torch
from tests.helpers import device_problem
from paper_2510_23215_b200 import scsf
cfg = synth.get_config("C3").with_(nx=int(sys.argv[1]) if len(sys.argv) > 1 else 40)
f = synth.make_batch(cfg, 2)
ops, params = device_problem(f)
try:
    ev, vec, st = scsf.solve_one(ops, 0, 200, 40, 20, 1e-8, 200, seed=1)
    print("ok", st)
except Exception as e:
    print("ERR", e)
