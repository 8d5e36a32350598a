"""The paper's own benchmark protocol (§4.2, Table 1; SURVEY
§8(f) NEXT f1) on one B200: 32x16x16 cantilever, volfrac 0.2, penal 3, rmin 4,
200 iterations, point load, sensitivity filter.  Prints a Table-1-style phase
report (JSON) next to the paper's laptop numbers (context only).

   python tools/paper_protocol.py [--iters 200] [--oracle-iters 0] [--variant plain|obstacle|both]

variant obstacle: the section-3 example WITH its cylinder obstacle (P:59
"A cylindrical obstacle region is defined within the domain"; the shape of
SPEC's example S:376, workloads.paper_obstacle: 576 passive-void elements).
--oracle-iters k: the oracle timed beside the GPU on this host (same run), its
c history compared with the GPU's over those k iterations.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

PAPER_TABLE1 = {"assembly": 33.9, "solve": 99.8, "filter": 0.7, "update": 10.8, "total": 147.3,
                "hardware": "Intel Core Ultra 7 155U laptop (PAPER P:88)", "matlab_total": 274.3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--oracle-iters", type=int, default=0)
    ap.add_argument("--set", nargs="*", default=[], help="parameter overrides key=value")
    ap.add_argument("--variant", default="plain", choices=["plain", "obstacle", "both"])
    args = ap.parse_args()
    for v in (["plain", "obstacle"] if args.variant == "both" else [args.variant]):
        run(args, v)


def run(args, variant):
    over = {k: (int(v) if v.lstrip("-").isdigit() else float(v) if "." in v else v)
            for k, v in (a.split("=") for a in args.set)}
    import torch
    from workloads import make_problem
    from paper_2504_05604_b200 import topo
    p, f, fx, pas = make_problem("paper" if variant == "plain" else "paper_obstacle", **over)
    ph = dict(assembly=0.0, solve=0.0, filter=0.0, update=0.0)
    ncg, c = [], []
    with topo.Problem(p, f, fx, pas) as pr:
        s = torch.cuda.Stream()
        pr.set_stream(s.cuda_stream)
        pr.optimize(1)                      # warm-up (graph capture, module load)
        pr.set_density(None)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.iters):
            ch, _, _ = pr.optimize(1, want_x=False)
            t = pr.timings()
            ph["assembly"] += t["ms_efield"] / 1e3
            ph["solve"] += t["ms_solve"] / 1e3
            ph["filter"] += t["ms_filter"] / 1e3
            ph["update"] += (t["ms_sens"] + t["ms_oc"]) / 1e3
            ncg.append(t["cg_iters"])
            c.append(float(ch[0]))
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        vol = pr.timings()["volume"]
        tt = pr.timings()
        mgc = dict(levels=pr.mg_levels(), fallbacks=tt["mg_fallbacks"], promotions=tt["mg_promotions"])
    tot = sum(ph.values())
    rec = {"workload": "paper protocol 32x16x16, volfrac 0.2, penal 3, rmin 4, point load, "
                       "sensitivity filter, PCG rtol 1e-10" + (", cylinder obstacle (576 passive-void elements)"
                                                               if variant == "obstacle" else ""),
           "variant": variant, "passive_elements": int(0 if pas is None else (pas != 0).sum()),
           "iterations": args.iters, "gpu_wall_s": wall, "gpu_phase_s": ph,
           "gpu_phase_pct": {k: 100 * v / tot for k, v in ph.items()},
           "cg_iters_mean": float(np.mean(ncg)), "cg_iters": ncg, "multigrid": mgc,
           "c_first": c[0], "c_last": c[-1], "volume": vol,
           "paper_table1_s": PAPER_TABLE1,
           "speedup_vs_paper_total": PAPER_TABLE1["total"] / wall}
    if args.oracle_iters > 0:
        import oracle
        t0 = time.perf_counter()
        r = oracle.run_optimization(p, f, fx, pas, n_iter=args.oracle_iters)
        to = time.perf_counter() - t0
        rec["oracle_s_per_iter"] = to / args.oracle_iters
        rec["gpu_s_per_iter"] = wall / args.iters
        rec["oracle_over_gpu_per_iter"] = (to / args.oracle_iters) / (wall / args.iters)
        rec["oracle_cores"] = os.cpu_count()
        rec["oracle_note"] = "oracle as it stands: CSR assembly, SuperLU direct solve, brute-force filter, literal OC"
        rec["oracle_c_rel_err_vs_gpu"] = float(np.max(np.abs(np.array(c[:args.oracle_iters]) - r["c"]) / r["c"]))
    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
