"""Diagnostics: single slab vs W loopback slabs, multigrid pieces."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
os.environ["TOPO_MG_VERBOSE"] = "1"
import numpy as np
from paper_2504_05604_b200 import topo
from workloads import config_params, cantilever_load, cantilever_fixed, cylinder_passive, random_density, random_vector

W = int(sys.argv[1]) if len(sys.argv) > 1 else 2
fp32 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
dims, obst = (37, 13, 5), (18.0, 6.0, 3.0)
p = config_params(dict(nelx=dims[0], nely=dims[1], nelz=dims[2], volfrac=0.3, rmin=1.5, n_iter=5, cg_rtol=1e-10,
                       obstacle=obst), precond="mg", mg_fp32=fp32)
f, fx = cantilever_load(*dims), cantilever_fixed(*dims)
pas = cylinder_passive(*dims, *obst)
x = random_density(int(np.prod(dims)), seed=4)
x[pas != 0] = 0
b = np.where(fx == 0, random_vector(len(f), seed=7), 0.0)
res = {}
for mode, world in ((topo.TOPO_DIST_SINGLE, 1), (topo.TOPO_DIST_LOOPBACK, W)):
    with topo.Problem(p, f, fx, pas, dist=dict(mode=mode, rank=0, world=world, device=0)) as pr:
        pr.set_xphys(x)
        lv = pr.mg_levels()
        r = {}
        for l in range(len(lv)):
            n = 3 * (lv[l][0] + 1) * (lv[l][1] + 1) * (lv[l][2] + 1)
            r[f"A{l}"] = pr.mg_apply(l, random_vector(n, seed=20 + l))
        r["z"] = pr.mg_vcycle(b)
        res[world] = r
        print("world", world, "levels", lv, flush=True)
for k in res[1]:
    a, c = res[1][k], res[W][k]
    d = np.abs(a - c)
    print(k, "relL2 %.3e" % (np.linalg.norm(a - c) / max(1e-300, np.linalg.norm(a))), "argmax", int(np.argmax(d)),
          flush=True)
a, c = res[1]["z"], res[W]["z"]
d = np.abs(a - c).reshape(dims[2] + 1, dims[0] + 1, dims[1] + 1, 3).max(axis=(0, 2, 3))
print("per-x-plane max |dz|:", np.array2string(d, precision=2, max_line_width=200))
