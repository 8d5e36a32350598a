"""Diagnostics: device time of one SIMP iteration (events around optimize(1))
vs the library's own phase timers, with and without profile mode.
python tools/step_gap.py [cfg]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from workloads import make_problem
from paper_2504_05604_b200 import topo

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
p, f, fx, pas = make_problem(cfg)
stream = torch.cuda.Stream()
with topo.Problem(p, f, fx, pas) as pr:
    pr.set_stream(stream.cuda_stream)
    for _ in range(3):
        pr.optimize(1)
    pr.snapshot()
    for prof in (False, True, False, True):
        pr.restore()
        pr.profile(prof)
        torch.cuda.synchronize()
        rows = []
        for _ in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pr.optimize(1)
            e1.record(stream)
            torch.cuda.synchronize()
            t = pr.timings()
            ph = sum(t[k] for k in ("ms_efield", "ms_solve", "ms_sens", "ms_filter", "ms_oc"))
            rows.append((round(e0.elapsed_time(e1), 2), round(t["ms_total"], 2), round(ph, 2), t["cg_iters"]))
        print(json.dumps(dict(profile=prof, steps=rows)), flush=True)
