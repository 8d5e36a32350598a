"""Short PCG run for ncu captures: config N, x = volfrac, `iters` PCG iterations
(the solve stops with ENOCONV, which is expected here)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from workloads import make_problem
from paper_2504_05604_b200 import topo

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 40
p, f, fx, pas = make_problem(cfg, cg_max_iter=iters, cg_check_every=8)
with topo.Problem(p, f, fx, pas) as pr:
    try:
        pr.solve(want_u=False)
    except topo.TopoError as e:
        assert e.code == topo.TOPO_ENOCONV, e
    pr.matvec_load(np.ones(3 * pr.n_nd))
    pr.matvec_run(4)
    print("ok", pr.timings()["kernel_launches"])
