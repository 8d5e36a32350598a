"""Offline (CPU) study of multigrid smoothers on GPU-dumped designs: how many
MG-PCG iterations a smoother variant needs on a void-rich late-iteration
design.  Uses oracle/mg.py's hierarchy (Galerkin, trilinear P, M1-M4) and
level operators; the smoothers are written out here (study tool, not the
oracle).  Usage:
  python tools/mg_smoother_study.py gpurun_out/designs/cfg2_xphys_029.npy 2 [variants...]
Variants: jac (damped Jacobi, theta/lam, nu sweeps), cheb (Chebyshev on
D^-1 A over [lam/alpha, 1.1 lam], degree k), mixed (Jacobi on the fine level,
Chebyshev below)."""
import sys
import os
import time

import numpy as np
import scipy.linalg as sla

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from oracle import mg  # noqa: E402
from workloads import make_problem  # noqa: E402


def lam_max_est(A, d, v0, k):
    v = v0.copy()
    for _ in range(k):
        v = (A @ v) / d
        v /= np.linalg.norm(v)
    return float((v @ (A @ v)) / (v @ (d * v)))


def smooth(A, d, b, x, kind, lam, nu, theta, alpha, deg):
    if kind == "jac":
        w = theta / lam
        for _ in range(nu):
            x = x + w * (b - A @ x) / d
        return x
    # Chebyshev on D^-1 A over [lo, hi]
    hi = 1.1 * lam
    lo = hi / alpha
    th, de = 0.5 * (hi + lo), 0.5 * (hi - lo)
    sig = th / de
    for _ in range(nu):
        r = b - A @ x
        dd = (r / d) / th
        rho = 1.0 / sig
        x = x + dd
        for _ in range(deg - 1):
            r = r - A @ dd
            rho_n = 1.0 / (2.0 * sig - rho)
            dd = rho_n * rho * dd + (2.0 * rho_n / de) * (r / d)
            x = x + dd
            rho = rho_n
    return x


CYCLE = os.environ.get("CYCLE", "V")
KTHR = float(os.environ.get("KTHR", "0"))   # Notay's threshold: skip the second FCG step when ||r2|| <= t ||r||
SKIPS, CALLS = {}, {}        # V, W (gamma = 2 below level 0), K (Notay K-cycle), K1 (K at level 1 only)


def make_vcycle(levels, ops, lams, spec):
    L = len(levels)

    def coarse(rc, l):
        """approximate A_{l}^{-1} rc for a coarse level l >= 1 (full-length vector)."""
        A, d, free = ops[l]
        kmin, kmax = 1, 99
        if CYCLE.startswith("K") and "-" in CYCLE:
            kmin, kmax = (int(v) for v in CYCLE[1:].split("-"))
        elif CYCLE.startswith("K") and len(CYCLE) > 1:
            kmax = int(CYCLE[1:])
        if l == L - 1 or CYCLE == "V" or l > kmax or l < kmin:
            return V(rc, l)
        if CYCLE == "W":
            x = V(rc, l)
            r2 = rc.copy()
            r2[free] = rc[free] - A @ x[free]
            return x + V(r2, l)
        # K-cycle: two flexible-CG steps preconditioned by the level-l cycle (Notay 2008)
        x1 = V(rc, l)
        v1 = np.zeros_like(rc)
        v1[free] = A @ x1[free]
        rho1, a1 = x1 @ v1, x1 @ rc
        r2 = rc - (a1 / rho1) * v1
        if KTHR > 0 and np.linalg.norm(r2) <= KTHR * np.linalg.norm(rc):
            SKIPS[l] = SKIPS.get(l, 0) + 1
            return (a1 / rho1) * x1
        CALLS[l] = CALLS.get(l, 0) + 1
        x2 = V(r2, l)
        v2 = np.zeros_like(rc)
        v2[free] = A @ x2[free]
        gam, bet, a2 = x2 @ v1, x2 @ v2, x2 @ r2
        rho2 = bet - gam * gam / rho1
        return (a1 / rho1 - gam * a2 / (rho1 * rho2)) * x1 + (a2 / rho2) * x2

    def V(b, l=0):
        A, d, free = ops[l]
        bf = b[free]
        if l == L - 1:
            x = np.zeros_like(b)
            x[free] = sla.cho_solve(levels[-1]["chol"], bf)
            return x
        kind, nu, deg = spec(l)
        xf = smooth(A, d, bf, np.zeros_like(bf), kind, lams[l], nu, 1.6, 30.0 if kind == "cheb" else 0, deg)
        r = np.zeros_like(b)
        r[free] = bf - A @ xf
        rc = levels[l]["P"].T @ r
        rc[levels[l + 1]["fixed"] != 0] = 0.0
        ec = coarse(rc, l + 1)
        xf = xf + (levels[l]["P"] @ ec)[free]
        xf = smooth(A, d, bf, xf, kind, lams[l], nu, 1.6, 30.0 if kind == "cheb" else 0, deg)
        x = np.zeros_like(b)
        x[free] = xf
        return x
    return V


def pcg(A, f, M, free, rtol, maxit=2000):
    nb = np.linalg.norm(f[free])
    u = np.zeros_like(f)
    r = f.copy()
    r[~free] = 0
    z = M(r)
    p = z.copy()
    rz = r @ z
    for it in range(maxit):
        q = np.zeros_like(p)
        q[free] = A @ p[free]
        a = rz / (p @ q)
        u += a * p
        r -= a * q
        if np.linalg.norm(r) <= rtol * nb:
            return it + 1
        zn = M(r)
        rzn = r @ zn
        beta = -a * (q @ zn) / rz if FLEX else rzn / rz   # Polak-Ribiere: (r_new - r_old) . z_new = -a q . z_new
        z = zn
        p = z + beta * p
        rz = rzn
    return maxit


FLEX = os.environ.get("FLEX", "0") == "1"


def main():
    xfile, cfg = sys.argv[1], int(sys.argv[2])
    variants = sys.argv[3:] or ["jac:1:1", "jac:2:1", "cheb:1:2", "cheb:1:3", "mixed:1:2", "mixed:1:3"]
    p, f, fx, pas = make_problem(cfg)
    dims = (p["nelx"], p["nely"], p["nelz"])
    xp = np.load(xfile)
    E = p["Emin"] + xp ** p["penal"] * (p["E0"] - p["Emin"])
    KE = oracle.element_stiffness(p["nu"])
    K = oracle.assemble(*dims, KE, E)
    nlev = int(os.environ.get("NLEV", "0")) or None
    levels = mg.hierarchy(K, fx, dims, n_lev=nlev, coarse_max=1000)
    ops = [mg.level_operator(lv) for lv in levels]
    if ops[-1][0].shape[0] > 40000:
        import scipy.sparse.linalg as spla
        lu = spla.splu(ops[-1][0].tocsc())
        levels[-1]["chol"] = None
        sla_cho_solve = sla.cho_solve
        sla.cho_solve = lambda c, b: lu.solve(b) if c is None else sla_cho_solve(c, b)
    else:
        levels[-1]["chol"] = sla.cho_factor(ops[-1][0].toarray())
    lams = []
    for l, lv in enumerate(levels[:-1]):
        A, d, free = ops[l]
        v0 = mg.start_vector(lv["K"].shape[0], lv["fixed"])[free]
        lams.append(lam_max_est(A, d, v0, 30))
    print("levels", [lv["dims"] for lv in levels], "lam", np.round(lams, 3))
    free = fx == 0
    A0 = ops[0][0]
    for v in variants:
        if "/" in v:      # per level: J<nu> (Jacobi) or C<deg>[x<nu>] (Chebyshev); the last entry repeats
            toks = v.split("/")

            def spec(l, toks=toks):
                t = toks[min(l, len(toks) - 1)]
                nu = int(t.split("x")[1]) if "x" in t else 1
                base = t.split("x")[0]
                return ("jac", int(base[1:]), 1) if base[0] == "J" else ("cheb", nu, int(base[1:]))
            V = make_vcycle(levels, ops, lams, spec)
            t0 = time.time()
            it = pcg(A0, f, V, free, p["cg_rtol"])
            k0, n0, d0 = spec(0)
            print(f"{v:16s} iters {it:4d}  fine matvecs/iter {2 * n0 * d0 + 1}  ({time.time() - t0:.1f} s)"
                  f"  skips {SKIPS} second steps {CALLS}", flush=True)
            SKIPS.clear()
            CALLS.clear()
            continue
        kind, nu, deg = v.split(":")
        nu, deg = int(nu), int(deg)
        if kind == "mixed":
            spec = lambda l, nu=nu, deg=deg: ("jac", 1, 1) if l == 0 else ("cheb", nu, deg)  # noqa: E731
        else:
            spec = lambda l, kind=kind, nu=nu, deg=deg: (kind, nu, deg)  # noqa: E731
        V = make_vcycle(levels, ops, lams, spec)
        t0 = time.time()
        it = pcg(A0, f, V, free, p["cg_rtol"])
        fine_mv = (2 * nu * deg if kind != "mixed" else 2) + 1
        print(f"{v:12s} iters {it:4d}  fine matvecs/iter {fine_mv}  fine-matvec total {it * fine_mv:5d}  "
              f"({time.time() - t0:.1f} s)", flush=True)


if __name__ == "__main__":
    main()
