"""Write tests/golden/cfg2_oracle_history.npz: BASELINE config 2 (120x40x20,
cylinder obstacle, rmin 2.5, volfrac 0.2) run through the ORACLE's SIMP loop
(oracle.run_optimization: CSR assembly, Jacobi-CG to a true relative residual of
1e-12 -- the oracle's solver at this size -- brute-force filter, literal OC
bisection).

Calls only oracle/ and workloads/ (no CUDA path).  Stores c, fu, change,
lambda, volume per iteration and xPhys after iterations 10 and n_iter.
Usage: python tools/make_golden_cfg2.py [n_iter] (default 30 = the config's
BASELINE iteration count).  Takes ~1 h on one core (SciPy sparse kernels are
single-threaded)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from workloads import make_problem  # noqa: E402


def main(n_iter=30, out=None, dump_dir=None):
    p, f, fixed, passive = make_problem(2)
    t0 = time.time()
    r = oracle.run_optimization(p, f, fixed, passive, n_iter=n_iter, record=True)
    print(f"oracle config 2, {n_iter} iterations: {time.time() - t0:.0f} s", flush=True)
    recs = r.pop("records")
    snaps = {}
    for it, rec in enumerate(recs):
        if dump_dir:
            np.save(os.path.join(dump_dir, f"cfg2_xphys_{it:02d}.npy"), rec["xPhys"])
        if it + 1 in (10, n_iter):       # design after iteration it (x) and its filtered xPhys
            snaps[f"x_{it + 1}"] = rec["xnew"]
    for k in (10, n_iter):
        if k < n_iter:
            snaps[f"xphys_{k}"] = recs[k]["xPhys"]
    snaps[f"xphys_{n_iter}"] = r["xPhys"]
    out = out or os.path.join(ROOT, "tests", "golden", "cfg2_oracle_history.npz")
    keep = {k: np.asarray(r[k]) for k in ("c", "fu", "change", "lam", "vol", "n_oc")}
    np.savez_compressed(out, **keep, **snaps)
    print("c =", keep["c"].tolist())
    print("wrote", out)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 30, dump_dir=os.environ.get("DUMP_DIR"))
