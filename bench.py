#!/usr/bin/env python
"""Benchmark of the matrix-free SIMP hot path (BASELINE.json metric: seconds per
SIMP iteration; PCG matvec GDOF/s; % of HBM roofline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

A "step" is one SIMP iteration (modulus, PCG solve,
sensitivities, filter, OC) of BASELINE config --config (default 4: the
512x256x256 cantilever, 101.6 M DOF, fp64) with all inputs resident in HBM.
Steps continue the optimisation (x evolves), so W warm-up + K timed steps of
config 4 are its 5 BASELINE iterations.  The solve is PCG in fp64 to rtol 1e-8
with the library's default preconditioner: geometric multigrid (SURVEY §8(f)
f2, coarse levels in fp32 = f3); --precond jacobi times the north_star's
Jacobi-PCG instead.  N > 1: launched by torchrun, one rank per GPU, x-slab
decomposition with NCCL (strong scaling): the fine level is slab-local with
halo exchanges, the coarse multigrid levels are replicated on every rank.  Prints ONE JSON line on rank 0.  See DESIGN.md "Measurement" for
every number's definition.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = dict(hbm_gbs=6650.0)   # B200_PROFILING.md fallback (only if MEASURED_PEAKS.json is absent)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region: ONE
    `nvidia-smi -lms 50` process (the profiling recipe's clocks line at 50 ms), started
    before the timed region and stopped after it.  (Spawning nvidia-smi per sample
    stalls the library's host-side batch polling and costs ~15 % at config 4.)"""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device, enabled=True):
        self.device = device
        self.enabled = enabled
        self.samples = []
        self._p = None
        self._t = None
        self._first = threading.Event()

    def _read(self):
        for line in self._p.stdout:
            line = line.strip()
            if line and line[0].isdigit():
                self.samples.append([v.strip() for v in line.split(",")])
                self._first.set()

    def __enter__(self):
        if not self.enabled:
            return self
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.Q,
                                        "--format=csv,noheader,nounits", "-lms", "50"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self._p = None
            return self
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()
        self._first.wait(5.0)          # nvidia-smi is up and sampling before timing starts
        self.samples.clear()           # keep only samples taken during the timed region
        return self

    def __exit__(self, *a):
        if self._p is not None:
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except Exception:
                self._p.kill()
            self._t.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if len(s) > 2 + k and s[2 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def ncu_traffic(cfg, world, keys):
    """sum over `keys` of dram__bytes_read.sum + dram__bytes_write.sum (one launch
    each) from the newest committed ncu --set full capture that has them
    (profiles/r*_ncu_cfg<cfg>*.json), or None."""
    import glob
    if world != 1:
        return None
    for fn in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_cfg%d*.json" % cfg)), reverse=True):
        try:
            d = json.load(open(fn))
            return sum((d[k]["dram_read_GB"] + d[k]["dram_write_GB"]) * 1e9 for k in keys), os.path.basename(fn)
        except Exception:
            continue
    return None


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# CPU baseline: the oracle as it stands, on a bounded x-slab sample of the
# same workload, extrapolated to one full SIMP iteration.
# ---------------------------------------------------------------------------
def oracle_sample(p, n_cg, slab=8):
    import oracle
    from workloads import cantilever_fixed, random_vector
    nelx, nely, nelz = p["nelx"], p["nely"], p["nelz"]
    sx = min(slab, nelx)
    n_el_s = sx * nely * nelz
    KE = oracle.element_stiffness(p["nu"])
    x = np.full(n_el_s, p["volfrac"])
    E = p["Emin"] + x ** p["penal"] * (p["E0"] - p["Emin"])
    fx = cantilever_fixed(sx, nely, nelz)
    pv = random_vector(3 * (sx + 1) * (nely + 1) * (nelz + 1), seed=1)
    t0 = time.perf_counter()
    q = oracle.matvec_elementwise(sx, nely, nelz, KE, E, pv, fx)
    t_mv = time.perf_counter() - t0
    # one Jacobi-PCG iteration = matvec + 3 axpy + 2 dots + 1 scaling (numpy)
    t0 = time.perf_counter()
    r = pv.copy(); z = r * 0.5; pp = z.copy(); uu = np.zeros_like(r)
    a = (r @ z) / (pp @ q); uu += a * pp; r -= a * q; z = 0.5 * r; pp = z + 0.3 * pp
    t_vec = time.perf_counter() - t0
    t0 = time.perf_counter()
    edof = oracle.edof_matrix(sx, nely, nelz)
    ce = oracle.element_energies(q, KE, edof)
    _, c, dc, dv = oracle.sensitivities(x, ce, p["penal"], p["E0"], p["Emin"])
    t_sens = time.perf_counter() - t0
    t0 = time.perf_counter()
    H, Hs = oracle.filter_matrix(sx, nely, nelz, p["rmin"])
    dcf = oracle.apply_filter(H, Hs, 0, "dc", dc)
    dvf = oracle.apply_filter(H, Hs, 0, "dv", dv)
    t_filt = time.perf_counter() - t0
    t0 = time.perf_counter()
    xn, lam, V, npass = oracle.oc_update(x, dcf, dvf, p["volfrac"], p["move"], p["oc_tol"],
                                         p["oc_lmax"], 0, H, Hs)
    oracle.apply_filter(H, Hs, 0, "x", xn)
    t_oc = time.perf_counter() - t0
    scale = (nelx * nely * nelz) / n_el_s
    est = n_cg * (t_mv + t_vec) * scale + (t_sens + t_filt + t_oc) * scale
    _ORACLE_REST[0] = (t_sens + t_filt + t_oc) * scale
    sample = (f"oracle on an x-slab of {sx}x{nely}x{nelz} elements ({n_el_s} el): element-loop "
              f"matvec {t_mv:.2f}s + PCG vector ops {t_vec:.2f}s, ce/dc {t_sens:.2f}s, filter "
              f"{t_filt:.2f}s, OC ({npass} passes) {t_oc:.2f}s; scaled x{scale:.0f} to the full "
              f"grid with N_cg={n_cg} PCG iterations per SIMP iteration")
    return est, sample, (t_mv + t_vec + t_sens + t_filt + t_oc)


def oracle_sample_mg(p, n_cg, cycle="K", div=None):
    """Algorithm-matched CPU baseline: the oracle's own MG-PCG (oracle.mg:
    Galerkin hierarchy, damped-Jacobi V/K-cycle, flexible PCG -- the GPU arm's
    algorithm) on the same cantilever scaled down by `div` per axis (x = volfrac),
    timed per PCG iteration and for the per-design setup (assembly + Galerkin
    hierarchy + coarsest Cholesky); the sensitivities, filter and OC on an
    8-plane x-slab (oracle_sample); both extrapolated by the DOF / element counts
    to the full grid with the GPU arm's N_cg per SIMP iteration."""
    import oracle
    from oracle import mg
    from workloads import cantilever_fixed, cantilever_load
    if div is None:   # a sample of ~2e5 DOF (config 4: 1/8 per axis; config 2: the full grid)
        ndof_full = 3 * (p["nelx"] + 1) * (p["nely"] + 1) * (p["nelz"] + 1)
        div = max(1, int(round((ndof_full / 2.0e5) ** (1.0 / 3.0))))
    dims = tuple(max(2, n // div) for n in (p["nelx"], p["nely"], p["nelz"]))
    x = np.full(int(np.prod(dims)), p["volfrac"])
    E = p["Emin"] + x ** p["penal"] * (p["E0"] - p["Emin"])
    KE = oracle.element_stiffness(p["nu"])
    f, fx = cantilever_load(*dims), cantilever_fixed(*dims)
    t0 = time.perf_counter()
    K = oracle.assemble(*dims, KE, E)
    _, it0 = mg.solve_mgcg(K, f, fx, dims, rtol=1e-30, max_iter=0, cycle=cycle)   # setup only
    t_setup = time.perf_counter() - t0
    k = 4                                    # k PCG iterations minus the (rebuilt) setup
    t0 = time.perf_counter()
    _, itk = mg.solve_mgcg(K, f, fx, dims, rtol=1e-30, max_iter=k, cycle=cycle)
    t_it = time.perf_counter() - t0
    t0 = time.perf_counter()
    mg.solve_mgcg(K, f, fx, dims, rtol=1e-30, max_iter=0, cycle=cycle)
    t_h = time.perf_counter() - t0
    t_iter = max(0.0, t_it - t_h) / max(1, itk)
    ndof_s = 3 * (dims[0] + 1) * (dims[1] + 1) * (dims[2] + 1)
    ndof = 3 * (p["nelx"] + 1) * (p["nely"] + 1) * (p["nelz"] + 1)
    sc = ndof / ndof_s
    _, sample_rest, wall_rest = oracle_sample(p, 0)
    est_rest = _ORACLE_REST[0]
    est = (t_setup + n_cg * t_iter) * sc + est_rest
    sample = (f"oracle MG-PCG ({cycle}-cycle, flexible PCG: the GPU arm's algorithm) on the cantilever "
              f"scaled to {dims[0]}x{dims[1]}x{dims[2]} ({ndof_s} DOF): setup {t_setup:.2f}s, "
              f"{t_iter:.3f}s per PCG iteration; scaled x{sc:.0f} by DOF with N_cg={n_cg} (the GPU arm's "
              f"count); plus {sample_rest.split('; scaled')[0].replace('oracle on', 'ce/dc, filter, OC on')} "
              f"scaled by elements -- extrapolated")
    return est, sample, t_setup + t_it + t_h + wall_rest


_ORACLE_REST = [0.0]


def cores_used():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


# ---------------------------------------------------------------------------
def run_reference(args, cfg_p, world, rank):
    """--impl reference: the oracle as it stands."""
    if rank != 0:
        return
    n_cg = args.ref_ncg
    if n_cg is None:   # the GPU arm's MG-PCG count at this config (profiles/ncg_cfg<cfg>_mg.json)
        try:
            with open(os.path.join(ROOT, "profiles", f"ncg_cfg{args.config}_mg.json")) as fh:
                n_cg = int(json.load(fh)["cg_iters_per_simp_iteration"])
        except Exception:
            n_cg = 30
    vals, sample = [], ""
    # each step is one bounded sample (~30 s); warm-up samples are skipped beyond one
    for i in range(min(args.warmup, 1) + args.steps):
        est, sample, wall = oracle_sample_mg(cfg_p, n_cg)
        if i >= min(args.warmup, 1):
            vals.append(est)
    v = float(np.mean(vals))
    line = {"impl": "reference", "metric": "s per SIMP iteration", "value": v,
            "unit": "s/iteration", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "weak" if args.weak else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, cfg_p, world),
            "cpu_baseline": {"value": v, "unit": "s/iteration", "cores": cores_used(),
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "s/iteration", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(args, p, world):
    n_nd = (p["nelx"] + 1) * (p["nely"] + 1) * (p["nelz"] + 1)
    tag = f"{args.config}w (weak, 128 element planes per GPU)" if getattr(args, "weak", False) else f"{args.config}"
    return {"workload": f"BASELINE config {tag}: cantilever {p['nelx']}x{p['nely']}x{p['nelz']} "
                        f"Hex8, fp64, volfrac {p['volfrac']}, rmin {p['rmin']}, PCG rtol {p['cg_rtol']}",
            "nelx": p["nelx"], "nely": p["nely"], "nelz": p["nelz"], "n_dof": 3 * n_nd,
            "filter": "density (mode 0)", "parallelism": f"x-slab{world}",
            "l2": "inputs larger than L2 (one DOF vector = %.0f MB)" % (3 * n_nd * 8 / 1e6)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=None, help="default: --steps")
    ap.add_argument("--matvec-reps", type=int, default=50)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-ncg", type=int, default=None)
    ap.add_argument("--ref-slab", type=int, default=8)
    ap.add_argument("--precond", default="auto", choices=["auto", "mg", "jacobi"],
                    help="PCG preconditioner (auto: geometric multigrid where the hierarchy can be built)")
    ap.add_argument("--mg-coarse-max", type=int, default=0, help="coarsest MG level DOF bound (0 = library auto)")
    ap.add_argument("--no-clocks", action="store_true", help="diagnostics: no nvidia-smi sampling")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling (SURVEY §8(d) config 4w): 128 x N element planes, 128x256x256 per GPU")
    ap.add_argument("--mg-nu", type=int, default=1, help="MG smoothing sweeps per level and side")
    ap.add_argument("--mg-omega", type=float, default=None, help="MG smoother theta (default: the library's)")
    ap.add_argument("--mg-nu-deep", type=int, default=0, help="MG sweeps on the small coarse levels (0 = library auto)")
    ap.add_argument("--cg-check-every", type=int, default=0, help="PCG iterations per CUDA-graph batch (0 = library auto)")
    args = ap.parse_args()

    from workloads import make_problem
    if args.e2e_steps is None:
        args.e2e_steps = args.steps
    world, rank, local = dist_env()
    weak_over = {"nelx": 128 * world} if args.weak else {}
    p, f, fx, pas = make_problem(args.config, precond=args.precond, mg_coarse_max=args.mg_coarse_max, **weak_over,
                                 mg_nu=args.mg_nu, mg_nu_deep=args.mg_nu_deep, cg_check_every=args.cg_check_every,
                                 **({} if args.mg_omega is None else {"mg_omega": args.mg_omega}))

    if args.impl == "reference":
        run_reference(args, p, world, rank)
        return

    import torch
    torch.cuda.set_device(local)
    dist = None
    pg = None
    if world > 1:
        import torch.distributed as td
        td.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = td
    from paper_2504_05604_b200 import topo
    if world > 1:
        obj = [topo.nccl_unique_id() if rank == 0 else None]
        pg.broadcast_object_list(obj, src=0)
        dist = dict(mode=topo.TOPO_DIST_NCCL, rank=rank, world=world, device=local, nccl_id=obj[0])

    stream = torch.cuda.Stream()
    pr = topo.Problem(p, f, fx, pas, dist=dist)
    pr.set_stream(stream.cuda_stream)
    n_dof = pr.count("ndof")
    n_el = pr.count("nel")
    n_nd = pr.count("nodes")

    def barrier():
        if pg is not None:
            pg.barrier()

    def max_over_ranks(v):
        if pg is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up SIMP iterations (untimed) ----
    cg_warm = []
    for _ in range(args.warmup):
        pr.optimize(1, want_x=False)
        cg_warm.append(pr.timings()["cg_iters"])

    # ---- timed SIMP iterations (device-resident inputs) ----
    pr.snapshot()          # the e2e leg below replays exactly these iterations
    pr.profile(True)
    l0 = pr.timings()["kernel_launches"]
    cg_timed, phase = [], []
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local, not args.no_clocks) as clk:
        with torch.cuda.stream(stream):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                c_hist, _, _ = pr.optimize(1, want_x=False)   # device-resident: the design stays in HBM
                t = pr.timings()
                cg_timed.append(t["cg_iters"])
                phase.append({k: t[k] for k in ("ms_efield", "ms_solve", "ms_mg_setup", "ms_sens", "ms_filter", "ms_oc")})
            e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms_total = max_over_ranks(e0.elapsed_time(e1))
    launches = pr.timings()["kernel_launches"] - l0
    mv_ms, mv_samples = pr.kernel_time()
    kt = [pr.kernel_time_k(k) for k in range(3)]
    mg_levels = pr.mg_levels()
    use_mg = bool(mg_levels) and pr.timings()["mg_fallbacks"] == 0
    pr.profile(False)
    clocks = clk.summary()
    s_per_iter = ms_total / 1e3 / args.steps

    # ---- standalone matvec GDOF/s (device-resident, CUDA events on the stream) ----
    from workloads import random_vector
    pr.matvec_load(random_vector(3 * n_nd, seed=1))
    pr.matvec_run(3)
    torch.cuda.synchronize()
    barrier()
    with torch.cuda.stream(stream):
        m0 = torch.cuda.Event(enable_timing=True)
        m1 = torch.cuda.Event(enable_timing=True)
        m0.record(stream)
        pr.matvec_run(args.matvec_reps)
        m1.record(stream)
    torch.cuda.synchronize()
    mv_standalone_ms = max_over_ranks(m0.elapsed_time(m1) / args.matvec_reps)
    gdofs = n_dof / (mv_standalone_ms * 1e-3) / 1e9

    # ---- end-to-end through the C ABI with pinned host buffers ----
    e2e = None
    if args.e2e_steps > 0:
        pr.restore()       # same design and warm start as the first timed step
        # two pinned host buffers used in turn: step k reads the design step k-1 wrote
        # back (no host-side copy in the timed loop)
        xbuf = [torch.empty(n_el, dtype=torch.float64, pin_memory=True).numpy() for _ in range(2)]
        xbuf[0][:] = pr.get("x")
        torch.cuda.synchronize()
        barrier()
        w0 = time.perf_counter()
        for k in range(args.e2e_steps):
            x_in, x_out = xbuf[k % 2], xbuf[(k + 1) % 2]
            pr.filter("x", x_in, want=False)            # H2D design variables, xPhys = H x / Hs
            c_e2e, _, _ = pr.optimize(1, x_out=x_out)    # one SIMP iteration, D2H x and c
        torch.cuda.synchronize()
        w1 = time.perf_counter()
        e2e_s = max_over_ranks((w1 - w0) / args.e2e_steps)
        e2e = {"value": e2e_s, "unit": "s/iteration", "h2d_bytes_per_step": 8 * n_el,
               "d2h_bytes_per_step": 8 * n_el + 8}

    peaks, peaks_src = load_peaks()
    hbm = float(peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
    own_el = n_el // world
    own_nd = n_nd // world
    if use_mg:
        # dominant kernel: the TMA-fed WHT matvec k_mv_wht, three variants per
        # MG-PCG iteration, algorithmic bytes per launch:
        #   <2,1,0> PCG   p = V(r) + beta p, q = K p, p.q : read V(r) 24 + p_old 24, write p 24 + q 24 B/node
        #   <3,0,2> pre   z = w D^-1 r, res = r - K z    : read r 24 + D^-1 8 + mask 1, write res
        #                                                  12 (fp32 hierarchy) / 24 B/node (the
        #                                                  epilogue's second r read hits L2; z is not
        #                                                  stored: k_mg_prolong0 recomputes it)
        #   <0,0,1> post  w = z + w D^-1 (r - K z), r.w  : read z 12 (fp32 hierarchy: z stored in fp32) /
        #                                                  24 + r 24 + D^-1 8 + mask 1, write w 24 B/node
        # each + E (8 B/el)
        #   (round 2: with the fp32 hierarchy on one slab the V-cycle output w is stored in
        #   fp32 -- PCG reads w 12 B/node, post writes it 12 B/node -- and the K-cycle's
        #   flexible beta reads q (24 B/node) in the post-smoothing epilogue)
        f32 = int(p.get("mg_fp32", 1)) != 0
        w32 = f32 and world == 1
        kc = int(p.get("mg_cycle", 1)) != 0
        var = [("k_mv_wht<8,2,1,0>", 84 if w32 else 96, kt[0]), ("k_mv_wht<8,3,0,2>", 45 if f32 else 57, kt[1]),
               ("k_mv_wht<8,0,0,1>", (57 if w32 else 69 if f32 else 81) + (24 if kc else 0), kt[2])]
        per = [{"kernel": n, "bytes_per_launch": b * own_nd + 8 * own_el, "mean_ms": t[0], "samples": t[1],
                "achieved": (b * own_nd + 8 * own_el) / (t[0] * 1e-3) / 1e9 if t[0] > 0 else None}
               for n, b, t in var]
        tot_b = sum(v["bytes_per_launch"] for v in per)
        tot_ms = sum(v["mean_ms"] for v in per)
        achieved = tot_b / (tot_ms * 1e-3) / 1e9 if tot_ms > 0 else None
        tr = None if args.weak else ncu_traffic(args.config, world, [v["kernel"] for v in per])
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": (achieved / hbm) if achieved else None, "traffic": tr[0] if tr else None,
                "traffic_source": (f"profiles/{tr[1]} (ncu --set full, one launch of each variant)" if tr else None),
                "kernel": "k_mv_wht (3 variants per MG-PCG iteration; bytes and time summed)",
                "bytes_per_launch": tot_b, "mean_ms": tot_ms, "variants": per, "peak_source": peaks_src}
    else:
        # dominant kernel: the fused PCG matvec k_mv_wht<8,1,1,0>; algorithmic bytes per
        # launch = read r (24 B/node), M^-1 (8 B/node), p_old (24 B/node), fixed mask (1 B/node),
        # E (8 B/el); write p_new (24 B/node), q (24 B/node)  -> 105 B/node + 8 B/el
        mv_bytes = 105 * own_nd + 8 * own_el
        achieved = mv_bytes / (mv_ms * 1e-3) / 1e9 if mv_ms > 0 else None
        tr = None if args.weak else ncu_traffic(args.config, world, ["k_mv_wht<8,1,1>"])
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": (achieved / hbm) if achieved else None, "traffic": tr[0] if tr else None,
                "traffic_source": f"profiles/{tr[1]} (ncu --set full, one launch)" if tr else None,
                "kernel": "k_mv_wht<8,1,1,0> (p = M^-1 r + beta p; q = K p; p.q)", "samples": mv_samples,
                "mean_ms": mv_ms, "bytes_per_launch": mv_bytes, "peak_source": peaks_src}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # algorithm-matched: the oracle's own MG-PCG with this arm's cycle, at this
        # arm's mean PCG iteration count (Jacobi arm: the oracle's slab sample with
        # the Jacobi-PCG count)
        n_cg = int(round(np.mean(cg_timed)))
        if use_mg:
            est, sample, wall = oracle_sample_mg(p, n_cg, cycle="K" if int(p.get("mg_cycle", 1)) else "V")
        else:
            est, sample, wall = oracle_sample(p, n_cg)
        cpu = {"value": est, "unit": "s/iteration", "cores": cores_used(), "kind": "oracle",
               "sample": sample + f" (wall {wall:.1f}s; SciPy sparse kernels single-threaded)"}
        try:
            os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
            with open(os.path.join(ROOT, "gpurun_out", f"ncg_cfg{args.config}{'_mg' if use_mg else ''}.json"),
                      "w") as fh:
                json.dump({"cg_iters_per_simp_iteration": n_cg, "per_step": cg_timed}, fh)
        except Exception:
            pass

    if rank == 0:
        line = {"metric": "s per SIMP iteration", "value": s_per_iter, "unit": "s/iteration",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms_total / args.steps, "higher_is_better": False,
                "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                # config = the workload only (identical to the reference arm's); the
                # solver this arm used is reported beside it
                "config": workload_config(args, p, world),
                "solver": {"precond": "multigrid" if use_mg else "jacobi",
                           "mg_levels": [list(d) for d in mg_levels] if use_mg else None},
                "matvec_gdofs": gdofs, "matvec_ms": mv_standalone_ms,
                "cg_iters_per_step": cg_timed, "cg_iters_warmup": cg_warm,
                "ms_per_cg_iter": [ph["ms_solve"] / max(1, n) for ph, n in zip(phase, cg_timed)],
                "phase_ms": phase, "c_last": float(c_hist[-1]),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(launches), "clocks": clocks}
        print(json.dumps(line), flush=True)
    pr.close()
    if pg is not None:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
