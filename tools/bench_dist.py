"""configs[4] (C5: 500 x 500, L = 300, b = 360) on one B200: the row-partitioned path
(`scsf_solve_queue_dist`) with one NCCL rank beside the one-GPU chain solve, and the
loopback communicator with 2 virtual ranks (its host-barrier exchanges make it a correctness
vehicle, not a timing one).  Prints one JSON object.

  python tools/bench_dist.py [N_OPS] [DEGREE]

Each path runs twice and the second pass is timed (the first fills the CUDA-graph cache).
"""
import json
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2510_23215_b200 import scsf  # noqa: E402


def main():
    nops = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    cfg = synth.get_config("C5")
    m = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.degree
    f = synth.make_batch(cfg, nops)
    dev = torch.device("cuda", 0)
    faces = [torch.from_numpy(x).to(dev) for x in f.faces]
    ops = scsf.assemble(cfg.dim, cfg.nx, cfg.h, faces, torch.from_numpy(f.c).to(dev))
    params = torch.from_numpy(f.params).to(dev)
    perm, _, _ = scsf.sort(params, cfg.dim, cfg.nx, cfg.p0)
    out = {"config": "C5", "n": cfg.n, "L": cfg.L, "b": cfg.b, "operators": nops, "degree": m}

    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev1, _, st1 = scsf.solve_queue(ops, perm, cfg.L, cfg.nex, m, cfg.tol, cfg.max_iter, seed=9,
                                       want_vecs=False, raise_on_fail=False)
    torch.cuda.synchronize()
    t1 = time.perf_counter() - t0
    out["one_gpu_chain"] = {"s_per_operator": t1 / nops, "iterations": [s["iterations"] for s in st1],
                            "status": [s["status"] for s in st1]}

    comm = scsf.comm_create(0, 1, scsf.comm_unique_id())
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev2, _, st2, rows = scsf.solve_queue_dist(ops, perm, cfg.L, cfg.nex, comm, m, cfg.tol, seed=9,
                                                  want_vecs=False, raise_on_fail=False)
    torch.cuda.synchronize()
    t2 = time.perf_counter() - t0
    comm.close()
    out["row_partitioned_nccl_world1"] = {"s_per_operator": t2 / nops, "iterations": [s["iterations"] for s in st2],
                                          "status": [s["status"] for s in st2],
                                          "max_rel_eval_diff_vs_one_gpu": float(
                                              (ev2 - ev1).abs().max() / ev1.abs().max())}

    comms = scsf.comm_create_loopback(2)
    res = [None, None]

    def work(r):
        torch.cuda.set_device(0)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            res[r] = scsf.solve_queue_dist(ops, perm[:1], cfg.L, cfg.nex, comms[r], m, cfg.tol, seed=9,
                                           want_vecs=False, raise_on_fail=False, stream=st)
        st.synchronize()

    t0 = time.perf_counter()
    th = [threading.Thread(target=work, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    t3 = time.perf_counter() - t0
    for c in comms:
        c.close()
    out["row_partitioned_loopback_2slabs_first_op"] = {
        "s": t3, "iterations": res[0][2][0]["iterations"], "status": res[0][2][0]["status"],
        "max_rel_eval_diff_vs_one_gpu": float((res[0][0][0] - ev1[0]).abs().max() / ev1[0].abs().max())}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
