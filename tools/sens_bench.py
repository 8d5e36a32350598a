"""Time the A5 sensitivity step (k_sens_x / k_sens + f.u) at a BASELINE config
after one solve, CUDA events on the bound stream.  TOPO_SENS_X=0 selects the
per-element gather kernel k_sens (A/B).   python tools/sens_bench.py [cfg]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_05604_b200 import topo  # noqa: E402
from workloads import make_problem, random_density  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = 20
p, f, fx, pas = make_problem(cfg)
s = torch.cuda.Stream()
with topo.Problem(p, f, fx, pas) as pr:
    pr.set_stream(s.cuda_stream)
    pr.set_xphys(random_density(pr.n_el, seed=3))
    pr.solve(want_u=False)
    c0 = pr.sensitivity(want=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        pr.sensitivity(want=False)
    e1.record(s)
    torch.cuda.synchronize()
    print(f"cfg {cfg} sensitivity: {e0.elapsed_time(e1) / reps:.3f} ms per step (TOPO_SENS_X="
          f"{os.environ.get('TOPO_SENS_X', '1')}), c = {c0}")
