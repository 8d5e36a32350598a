"""Per-rank compute time of a W-GPU x-slab run, measured on ONE GPU
(TOPO_DIST_SOLO: rank r's slab alone, every exchange / allreduce / all-gather
omitted; include/topo.h).  The kernel sequence and sizes are rank r's of the
NCCL run; the PCG iteration COUNT is not (the coupling is dropped), so the
per-iteration costs are the numbers to read:
  ms_per_cg  = (ms_solve - ms_mg_setup) / cg_iters   (one MG-PCG iteration)
  ms_setup   = per-design multigrid setup
  ms_rest    = E, sensitivities, filter, OC
W = 1 is the single-GPU run (TOPO_DIST_SINGLE) of the same workload.  This is
the compute side of a strong-scaling projection: halo / allreduce time over
NVLink is NOT in it (one GPU per gpurun call; DESIGN.md §6 states the bytes).
In SOLO mode the PCG runs exactly cg_max_iter = 20 iterations per solve (no
convergence or breakdown exit: the decoupled slab is not the problem).

   python tools/solo_scale.py [cfg=4] [W list=1,2,4,8] [iters=3] [--weak]
--weak: SURVEY config 4w, 128 x W element planes (128 x 256 x 256 per rank).
"""
import json
import os
import statistics as st
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_05604_b200 import topo  # noqa: E402
from workloads import make_problem  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
Ws = [int(w) for w in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8").split(",")]
iters = int(sys.argv[3]) if len(sys.argv) > 3 and not sys.argv[3].startswith("-") else 3
weak = "--weak" in sys.argv
out = {"cfg": f"{cfg}w" if weak else cfg, "scaling": "weak" if weak else "strong",
       "what": "rank W//2's slab alone on one B200 (TOPO_DIST_SOLO), SIMP iterations 3.. of the run", "runs": {}}
p, f, fx, pas = make_problem(cfg)
for W in Ws:
    if weak:
        p, f, fx, pas = make_problem(cfg, nelx=128 * W)
    r = W // 2
    dist = None if W == 1 else dict(mode=topo.TOPO_DIST_SOLO, rank=r, world=W, device=0)
    kw = {"dist": dist} if dist else {}
    pw = p if W == 1 else dict(p, cg_max_iter=20)
    rows = []
    with topo.Problem(pw, f, fx, pas, **kw) as pr:
        nd = pr.count("mg_dist") if W > 1 else 0
        lv = pr.mg_levels()
        pr.optimize(2, want_x=False)                  # warm-up: graphs captured, design moves off uniform
        for _ in range(iters):
            pr.optimize(1, want_x=False)
            t = pr.timings()
            rows.append(t)
        fb = t["mg_fallbacks"]
        lo, hi = pr.owned_range()
    med = lambda k: st.median(float(x[k]) for x in rows)  # noqa: E731
    cg = [int(x["cg_iters"]) for x in rows]
    per = [(x["ms_solve"] - x["ms_mg_setup"]) / max(1, x["cg_iters"]) for x in rows]
    out["runs"][W] = dict(rank=r, owned_elem_planes=[lo, hi], mg_levels=lv, mg_dist_levels=nd,
                          ms_per_cg=st.median(per), cg_iters=cg, ms_setup=med("ms_mg_setup"),
                          ms_rest=st.median(x["ms_efield"] + x["ms_sens"] + x["ms_filter"] + x["ms_oc"] for x in rows),
                          ms_total=med("ms_total"), mg_fallbacks=fb)
    print(W, json.dumps(out["runs"][W]), file=sys.stderr, flush=True)
b = out["runs"].get(1)
if b:
    for W, d in out["runs"].items():
        d["cg_speedup_vs_1"] = b["ms_per_cg"] / d["ms_per_cg"]
        d["setup_speedup_vs_1"] = b["ms_setup"] / d["ms_setup"]
        d["rest_speedup_vs_1"] = b["ms_rest"] / d["ms_rest"]
print(json.dumps(out))
