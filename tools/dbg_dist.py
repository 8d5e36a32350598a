"""Debug: distributed multigrid levels (loopback W) vs one slab: V-cycle and solve."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2504_05604_b200 import topo
from workloads import config_params, cantilever_load, cantilever_fixed, random_density, random_vector

dims = (128, 32, 16)
for fp32 in (0, 1):
    p = config_params(dict(nelx=dims[0], nely=dims[1], nelz=dims[2], volfrac=0.2, rmin=1.5, n_iter=4, cg_rtol=1e-10,
                           obstacle=None), precond="mg", mg_fp32=fp32, mg_cycle=sys.argv[1] if len(sys.argv) > 1 else "K")
    f, fx = cantilever_load(*dims), cantilever_fixed(*dims)
    x = random_density(int(np.prod(dims)), seed=3)
    b = np.where(fx == 0, random_vector(fx.size, seed=9), 0.0)
    res = {}
    for key, mode, W, env in (("single", topo.TOPO_DIST_SINGLE, 1, {}), ("force1", topo.TOPO_DIST_SINGLE, 1, {"TOPO_DIST_FORCE1": "1"}),
                              ("force1l1", topo.TOPO_DIST_SINGLE, 1, {"TOPO_DIST_FORCE1": "1", "TOPO_DIST_LEVELS": "1"}),("rep2", topo.TOPO_DIST_LOOPBACK, 2, {"TOPO_DIST_LEVELS": "0"}),
                              ("d1_2", topo.TOPO_DIST_LOOPBACK, 2, {"TOPO_DIST_LEVELS": "1"}),
                              ("d2_2", topo.TOPO_DIST_LOOPBACK, 2, {}), ("d2_4", topo.TOPO_DIST_LOOPBACK, 4, {})):
        os.environ["TOPO_DIST_MIN_NODES"] = "0"
        os.environ.pop("TOPO_DIST_LEVELS", None)
        os.environ.pop("TOPO_DIST_FORCE1", None)
        os.environ.update(env)
        with topo.Problem(p, f, fx, None, dist=dict(mode=mode, rank=0, world=W, device=0)) as pr:
            nd = pr.count("mg_dist")
            pr.set_xphys(x)
            z = pr.mg_vcycle(b)
            try:
                if key.startswith("force"):
                    raise RuntimeError("skipped")
                u, info = pr.solve()
            except Exception as e:
                u, info = None, {"err": str(e)}
            t = pr.timings()
        res[key] = z
        z1 = res["single"]
        print(f"fp32={fp32} {key:7s} dist={nd} relz={np.linalg.norm(z - z1) / np.linalg.norm(z1):.3e} "
              f"precond={info.get('precond')} iters={info.get('iters')} fb={t['mg_fallbacks']} prom={t['mg_promotions']} {info.get('err', '')}")
