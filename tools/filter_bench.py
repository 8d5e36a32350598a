"""Time the A6 filter (x -> xPhys, density filter: k_filt_prep + apply) and the
dc filter at a BASELINE config, CUDA events on the bound stream.
TOPO_FILT25=0 selects the per-output gather kernel (A/B)."""
import os
import sys

import numpy as np
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
    pr.set_density(random_density(pr.n_el, seed=3))
    for what in ("x", "dc"):
        inp = None if what == "x" else -random_density(pr.n_el, seed=4)
        pr.filter(what, inp, want=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            pr.filter(what, None, want=False)
        e1.record(s)
        e1.synchronize()
        print(f"cfg {cfg} filter {what}: {e0.elapsed_time(e1) / reps:.3f} ms per application "
              f"(TOPO_FILT25={os.environ.get('TOPO_FILT25', '1')})")
