"""MG-PCG vs Jacobi-PCG on one config: iterations, solve time per SIMP iteration.
python tools/mg_probe.py CFG N_ITER [precond ...]"""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2504_05604_b200 import topo
from workloads import make_problem

cfg = int(sys.argv[1]); n_iter = int(sys.argv[2])
pcs = sys.argv[3:] or ["mg", "jacobi"]
out = {}
for pc in pcs:
    p, f, fx, pas = make_problem(cfg, precond=pc)
    t0 = time.time()
    with topo.Problem(p, f, fx, pas) as pr:
        t_init = time.time() - t0
        rows = []
        for it in range(n_iter):
            c, _, _ = pr.optimize(1)
            t = pr.timings()
            rows.append(dict(c=float(c[0]), cg=t["cg_iters"], ms_solve=t["ms_solve"], ms_total=t["ms_total"],
                             ms_sens=t["ms_sens"], ms_filter=t["ms_filter"], ms_oc=t["ms_oc"]))
            print(pc, it, rows[-1], flush=True)
        out[pc] = dict(levels=pr.mg_levels(), rows=rows, init_s=t_init)
print(json.dumps(out))
