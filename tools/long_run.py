"""Long, void-heavy SIMP runs at the large BASELINE configs on one GPU: the
MG-PCG iteration count, the true residual and the safety-net counters (theta
cuts, fp64 promotions, Jacobi fallbacks) of every SIMP iteration, well past the
configs' own n_iter (robustness of the fp32 K-cycle
preconditioner as voids form).  One JSON line per config.
   python tools/long_run.py 3:100 4:60        (config:iterations)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from workloads import make_problem  # noqa: E402
from paper_2504_05604_b200 import topo  # noqa: E402

for spec in sys.argv[1:] or ["3:100"]:
    cfg, n_iter = (int(v) for v in spec.split(":"))
    p, f, fx, pas = make_problem(cfg)
    with topo.Problem(p, f, fx, pas) as pr:
        s = torch.cuda.Stream()
        pr.set_stream(s.cuda_stream)
        ncg, ms, ms_solve, c, change, vol = [], [], [], [], [], []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for it in range(n_iter):
            ch, _, _ = pr.optimize(1, want_x=False)
            t = pr.timings()
            ncg.append(int(t["cg_iters"]))
            ms.append(t["ms_total"])
            ms_solve.append(t["ms_solve"])
            c.append(float(ch[0]))
            change.append(t["change"])
            vol.append(t["volume"])
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        t = pr.timings()
        # the last design's solve again, for its true residual (f - K u in fp64)
        _, info = pr.solve(want_u=False)
        x = pr.get("xphys")
    grey = float(np.mean((x > 0.05) & (x < 0.95)))
    rec = dict(config=cfg, grid=[p["nelx"], p["nely"], p["nelz"]], n_iter=n_iter, wall_s=wall,
               s_per_iter_mean=float(np.mean(ms)) / 1e3, s_per_iter_last10=float(np.mean(ms[-10:])) / 1e3,
               ncg=ncg, ncg_max=int(max(ncg)), ms_solve=[round(v, 2) for v in ms_solve],
               c=c, change=[round(v, 4) for v in change], volume_last=vol[-1],
               void_fraction_last=float(np.mean(x < 0.05)), solid_fraction_last=float(np.mean(x > 0.95)),
               grey_fraction_last=grey, true_rel_res_last=info["true_rel_res"], ncg_resolve=int(info["iters"]),
               mg_theta_cuts=int(t["mg_theta_cuts"]), mg_promotions=int(t["mg_promotions"]),
               mg_fallbacks=int(t["mg_fallbacks"]))
    print(json.dumps(rec), flush=True)
