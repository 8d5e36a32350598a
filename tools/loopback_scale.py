"""Multi-slab multigrid at scale on ONE GPU (in-process loopback transport):
config 3 (12.8 M DOF), W = 1 vs W = 2 / 4 slabs, 3 SIMP iterations; the c
histories must agree (same partition logic as NCCL x-slabs).  Timing is NOT a
multi-GPU number (the slabs run one after another on one GPU).
   python tools/loopback_scale.py [cfg] [W list, default 1,2,4 (cfg 4: 1,2)] [SIMP iterations=3]"""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2504_05604_b200 import topo
from workloads import make_problem

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
Ws = [int(w) for w in sys.argv[2].split(",")] if len(sys.argv) > 2 else ([1, 2, 4] if cfg != 4 else [1, 2])
n_it = int(sys.argv[3]) if len(sys.argv) > 3 else 3
p, f, fx, pas = make_problem(cfg)
res = {}
for W in Ws:
    dist = None if W == 1 else dict(mode=topo.TOPO_DIST_LOOPBACK, rank=0, world=W, device=0)
    kw = {"dist": dist} if dist else {}
    with topo.Problem(p, f, fx, pas, **kw) as pr:
        t0 = time.perf_counter()
        c, _, _ = pr.optimize(n_it, want_x=False)
        wall = time.perf_counter() - t0
        t = pr.timings()
        res[W] = dict(c=[float(v) for v in c], ncg=t["cg_iters_total"], wall=wall, levels=pr.mg_levels(),
                      fallbacks=t["mg_fallbacks"], mg_dist_levels=pr.count("mg_dist") if W > 1 else 0)
    print(W, json.dumps(res[W]), file=sys.stderr, flush=True)
for W in Ws[1:]:
    rel = max(abs(a - b) / abs(b) for a, b in zip(res[W]["c"], res[1]["c"]))
    res[W]["max_rel_c_vs_W1"] = rel
print(json.dumps(res))
