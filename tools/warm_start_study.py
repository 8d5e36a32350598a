"""Offline (CPU, oracle only) study of PCG initial guesses over a SIMP run: the
relative residual and the energy-norm error of
  prev   u_{k-1}                       (what the product uses, cg_warm_start)
  lin    2 u_{k-1} - u_{k-2}
  scal   alpha u_{k-1},  alpha = f.u / u.K u      (1-D Galerkin projection)
  gal2/3 the Galerkin projection onto the last 2 / 3 solutions
for the design of every iteration k.  Study tool, not the oracle and not the
product.  Usage: python tools/warm_start_study.py [nelx nely nelz n_iter]
Result (48x24x24, volfrac 0.12, rmin 1.5, 26 iterations; DESIGN.md "Open
items"): gal2 lowers the energy error 2-3x and the residual ~1.5x below prev;
at ~0.47 decades per MG-PCG iteration that is less than one iteration of ~17
for two more fine matvecs and one more 813 MB vector at config 4 -- not built."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import oracle  # noqa: E402
from oracle.fem import assemble  # noqa: E402
from oracle.ke import element_stiffness  # noqa: E402
from oracle.mesh import edof_matrix  # noqa: E402
from workloads import config_params, cantilever_load, cantilever_fixed  # noqa: E402

a = [int(v) for v in sys.argv[1:5]]
nx, ny, nz, n_iter = a if len(a) == 4 else (48, 24, 24, 26)
p = config_params(dict(nelx=nx, nely=ny, nelz=nz, volfrac=0.12, rmin=1.5, n_iter=n_iter, cg_rtol=1e-8,
                       obstacle=None))
f = cantilever_load(nx, ny, nz)
fx = np.asarray(cantilever_fixed(nx, ny, nz), bool)
t = time.time()
recs = oracle.run_optimization(p, f, fx.astype(np.uint8), None, n_iter=n_iter, record=True)["records"]
print("oracle loop %.0f s" % (time.time() - t))
KE = element_stiffness(p["nu"])
edof = edof_matrix(nx, ny, nz)
nf = np.linalg.norm(f)
for k in range(2, len(recs)):
    E = p["Emin"] + recs[k]["xPhys"] ** p["penal"] * (p["E0"] - p["Emin"])
    K = assemble(nx, ny, nz, KE, E, edof)
    ut = recs[k]["u"]

    def res(u):
        r = f - K @ u
        r[fx] = 0
        return np.linalg.norm(r) / nf

    def eerr(u):
        e = u - ut
        return np.sqrt(e @ (K @ e) / (ut @ (K @ ut)))

    def galerkin(us):
        B = np.stack(us, 1)
        return B @ np.linalg.solve(B.T @ (K @ B), B.T @ f)

    u1, u2 = recs[k - 1]["u"], recs[k - 2]["u"]
    guesses = [("prev", u1), ("lin", 2 * u1 - u2), ("scal", (f @ u1) / (u1 @ (K @ u1)) * u1),
               ("gal2", galerkin([u1, u2])),
               ("gal3", galerkin([u1, u2, recs[k - 3]["u"]]) if k >= 3 else galerkin([u1, u2]))]
    print(k, " | ".join("%s res %.2e eerr %.2e" % (n, res(g), eerr(g)) for n, g in guesses), flush=True)
