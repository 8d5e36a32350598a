"""Run a BASELINE config on the GPU and dump xPhys at chosen SIMP iterations
(npy, external numbering) plus the per-iteration PCG counts -- inputs for
offline (CPU) preconditioner studies with oracle/mg.py.
Usage: python tools/dump_designs.py CFG OUTDIR it1,it2,...  [key=value params]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_05604_b200 import topo  # noqa: E402
from workloads import make_problem  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if sys.argv[1].isdigit() else sys.argv[1]
    out = sys.argv[2]
    its = sorted(int(v) for v in sys.argv[3].split(","))
    over = {}
    for kv in sys.argv[4:]:
        k, v = kv.split("=")
        over[k] = float(v) if "." in v or "e" in v else int(v) if v.lstrip("-").isdigit() else v
    os.makedirs(out, exist_ok=True)
    p, f, fx, pas = make_problem(cfg, **over)
    ncg, c = [], []
    with topo.Problem(p, f, fx, pas) as pr:
        for it in range(max(its) + 1):
            if it in its:
                np.save(os.path.join(out, f"cfg{cfg}_xphys_{it:03d}.npy"), pr.get("xphys"))
            ch, _, _ = pr.optimize(1, want_x=False)
            t = pr.timings()
            ncg.append(int(t["cg_iters"]))
            c.append(float(ch[0]))
    json.dump(dict(cfg=cfg, its=its, ncg=ncg, c=c, params={k: v for k, v in p.items() if k != "obstacle"}),
              open(os.path.join(out, f"cfg{cfg}_run.json"), "w"))
    print("ncg", ncg)


if __name__ == "__main__":
    main()
