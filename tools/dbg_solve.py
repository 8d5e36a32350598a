"""Diagnostics: two solves of a config, printing solve info and MG fallbacks.
python tools/dbg_solve.py CFG [key=value ...]  (TOPO_MG_VERBOSE=1 prints smoother weights)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_05604_b200 import topo
from workloads import make_problem
cfg = int(sys.argv[1])
over = {k: (int(v) if v.lstrip("-").isdigit() else v) for k, v in (a.split("=") for a in sys.argv[2:])}
p, f, fx, pas = make_problem(cfg, **over)
with topo.Problem(p, f, fx, pas) as pr:
    for it in range(2):
        u, info = pr.solve(want_u=False)
        print(it, info, "fallbacks", pr.timings()["mg_fallbacks"], flush=True)
