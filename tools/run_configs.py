"""Run BASELINE configs end to end on one GPU and report s/SIMP iteration,
N_cg per iteration and the compliance history (for BASELINE.md).
   python tools/run_configs.py 0 1 2 3 [precond=jacobi|mg|auto]   (config 4: use bench.py)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from workloads import make_problem  # noqa: E402
from paper_2504_05604_b200 import topo  # noqa: E402

out = []
over = dict(a.split("=") for a in sys.argv[1:] if "=" in a)
for cfg in [int(a) for a in sys.argv[1:] if "=" not in a] or [0, 1, 2, 3]:
    p, f, fx, pas = make_problem(cfg, **over)
    n_iter = p["n_iter"]
    with topo.Problem(p, f, fx, pas) as pr:
        s = torch.cuda.Stream()
        pr.set_stream(s.cuda_stream)
        ncg, ms, c = [], [], []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for it in range(n_iter):
            ch, _, _ = pr.optimize(1)
            t = pr.timings()
            ncg.append(t["cg_iters"])
            ms.append(t["ms_total"])
            c.append(float(ch[0]))
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        t = pr.timings()
    rec = dict(config=cfg, precond=over.get("precond", "auto"), grid=[p["nelx"], p["nely"], p["nelz"]], n_iter=n_iter,
               s_per_iter_median=float(np.median(ms[2:] if len(ms) > 2 else ms)) / 1e3,
               s_per_iter_mean=float(np.mean(ms)) / 1e3, wall_s=wall, ncg=ncg, c=c,
               volume=t["volume"], launches=t["kernel_launches"])
    out.append(rec)
    print(json.dumps(rec), flush=True)
