"""Multigrid robustness over a whole optimisation: per SIMP iteration the PCG
iteration count, the preconditioner actually used and the fallback count.
python tools/mg_robust.py CFG [key=value ...]"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_05604_b200 import topo
from workloads import make_problem
cfg = sys.argv[1]
cfg = "paper" if cfg == "paper" else int(cfg)
over = {k: (int(v) if v.lstrip("-").isdigit() else float(v) if "." in v else v)
        for k, v in (a.split("=") for a in sys.argv[2:])}
p, f, fx, pas = make_problem(cfg, **over)
rows = []
with topo.Problem(p, f, fx, pas) as pr:
    for it in range(p["n_iter"]):
        pr.optimize(1)
        t = pr.timings()
        rows.append((t["cg_iters"], t["mg_fallbacks"], t["mg_promotions"]))
print(json.dumps(dict(cfg=str(cfg), over=over, ncg=[r[0] for r in rows], fallbacks=rows[-1][1], promotions=rows[-1][2],
                      first_fallback_it=next((i for i, r in enumerate(rows) if r[1] > 0), None))))
