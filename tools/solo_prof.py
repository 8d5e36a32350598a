"""One SIMP iteration of rank W//2's slab of a W-slab config-4 run alone on the GPU
(TOPO_DIST_SOLO, 20 PCG iterations per solve), after one warm-up iteration --
for ncu launch lists of the per-rank kernel sequence.
   python tools/solo_prof.py W [cfg=4]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_05604_b200 import topo  # noqa: E402
from workloads import make_problem  # noqa: E402

W = int(sys.argv[1])
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 4
p, f, fx, pas = make_problem(cfg)
dist = dict(mode=topo.TOPO_DIST_SOLO, rank=W // 2, world=W, device=0) if W > 1 else None
kw = {"dist": dist} if dist else {}
with topo.Problem(dict(p, cg_max_iter=20) if W > 1 else p, f, fx, pas, **kw) as pr:
    pr.optimize(1, want_x=False)
    pr.optimize(1, want_x=False)
    t = pr.timings()
    print("W", W, "cg", t["cg_iters"], "ms_solve", t["ms_solve"], "ms_mg_setup", t["ms_mg_setup"])
