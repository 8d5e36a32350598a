"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck):
multigrid single slab (configs 0-1, an obstacle case, mg_nu 2), loopback
x-slabs, Jacobi; OC compaction, symmetric-sweep coarse inverse and the fp32 z
path all execute.   compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_05604_b200 import topo
from workloads import make_problem

runs = [(0, {}, None), (1, {}, None), (2, dict(nelx=40, nely=16, nelz=8, obstacle=(20.0, 8.0, 3.0)), None),
        (1, dict(mg_nu=2), None), (1, dict(precond="jacobi"), None),
        (1, {}, dict(mode=topo.TOPO_DIST_LOOPBACK, rank=0, world=3, device=0))]
for cfg, over, dist in runs:
    p, f, fx, pas = make_problem(cfg, **over)
    kw = {"dist": dist} if dist else {}
    with topo.Problem(p, f, fx, pas, **kw) as pr:
        c, _, nd = pr.optimize(3, want_x=False)
        t = pr.timings()
    print("cfg", cfg, over, "W", dist["world"] if dist else 1, "c", [round(v, 6) for v in c],
          "fallbacks", t["mg_fallbacks"], flush=True)
print("sanitize run done")
