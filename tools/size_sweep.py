"""Find the smallest grid where the solve fails (debug aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import config_params, cantilever_load, cantilever_fixed
from paper_2504_05604_b200 import topo
sizes = [(16, 8, 8), (32, 16, 16), (40, 40, 8), (64, 32, 32), (64, 64, 8), (64, 8, 64), (128, 64, 64), (256, 128, 128)]
for dims in sizes:
    p = config_params(dict(nelx=dims[0], nely=dims[1], nelz=dims[2], volfrac=0.15, rmin=3.0, n_iter=1,
                           cg_rtol=1e-8, obstacle=None), cg_max_iter=24, cg_check_every=8)
    try:
        with topo.Problem(p, cantilever_load(*dims), cantilever_fixed(*dims)) as pr:
            try:
                pr.solve(want_u=False)
            except topo.TopoError as e:
                if e.code != topo.TOPO_ENOCONV:
                    raise
        print(dims, "ok", flush=True)
    except Exception as e:
        print(dims, "FAIL", e, flush=True)
        break
