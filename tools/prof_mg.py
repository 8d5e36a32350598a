"""One SIMP iteration of a config with the default (multigrid) solver, after one
warm-up iteration -- for ncu launch lists.  python tools/prof_mg.py CFG [precond]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_05604_b200 import topo
from workloads import make_problem

cfg = int(sys.argv[1])
pc = sys.argv[2] if len(sys.argv) > 2 else "auto"
p, f, fx, pas = make_problem(cfg, precond=pc)
with topo.Problem(p, f, fx, pas) as pr:
    pr.optimize(1)
    c, _, _ = pr.optimize(1)
    t = pr.timings()
    print("levels", pr.mg_levels(), "cg", t["cg_iters"], "ms_solve", t["ms_solve"], "c", c)
