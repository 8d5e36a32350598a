"""Geometric multigrid preconditioner for the K(x)u = f solve (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Why: SURVEY §8(f) NEXT f2 -- "matrix-free geometric multigrid preconditioner on
the hex-grid hierarchy, replacing Jacobi"; the paper names the solve as the
dominant cost (Table 1 "Solve" 67.8 %) and scalability of
the solver as future work (§4.3).  The paper gives no multigrid
algorithm, so this module writes out the textbook one (DESIGN.md readings
M1-M6), each step in plain NumPy/SciPy, no blocking or fusion:

  M1 hierarchy   nested Hex8 grids, coarse element = 2x2x2 fine elements,
                 n_c = ceil(n/2) per axis (an odd axis gets a half-empty last
                 coarse element; its outer node is a plain coarse node)
  M2 transfer    P = trilinear interpolation (per axis: even fine node 2j <- coarse
                 j; odd fine node 2j+1 <- (j, j+1) with weights 1/2, 1/2),
                 restriction = P^T
  M3 operators   Galerkin: K_{l+1} = P^T K_l P (unmasked); the level operator
                 acts on free DOFs only (A_l = K_l[free, free])
  M4 coarse BCs  coarse DOF (j, c) fixed iff the fine node at min(2j, n) (per
                 axis: the coarse node's position, clamped into the fine grid) has
                 DOF c fixed.  The hierarchy is only built while property Q holds:
                 every fixed fine DOF interpolates from fixed coarse DOFs only.
                 Under Q, P^T K P restricted to free coarse DOFs IS the Galerkin
                 operator of the free-DOF problem (pinned in tests)
  M5 smoother    damped Jacobi x <- x + w_l D^-1 (b - A x), nu pre- and nu
                 post-smoothing steps (symmetric V-cycle -> SPD preconditioner)
                 with w_l = theta / lam_l, lam_l = Rayleigh quotient of D^-1 A_l
                 after k power steps from a fixed hash-generated start vector
                 (lam_l <= lam_max: a fixed w would diverge where lam_max(D^-1 A)
                 exceeds 2/w, which random densities reach: lam_max ~ 4.7).  8 steps
                 estimate 0.80-0.95 of lam_max, so theta = 1.4 keeps w lam_max <= 1.75
  M6 coarsest    exact solve (dense Cholesky) on the coarsest level; coarsening
                 stops at the first level with <= coarse_max DOFs
  M8 cycle       V-cycle (one recursive call per coarse level), or the K-cycle of
                 Notay & Vassilevski ("Recursive Krylov-based multigrid cycles",
                 2008): every coarse level above the coarsest is solved by TWO
                 flexible-CG steps preconditioned by that level's cycle (always two;
                 no residual-ratio threshold), written out in coarse_correction
  M9 outer       PCG with z = V(r); with a K-cycle (a nonlinear preconditioner) the
                 flexible (Polak-Ribiere) beta = z_new.(r_new - r_old) / (z_old.r_old)
                 = -alpha (z_new.q) / rz, q = A p (Notay's FCG(1))
The outer Krylov method is the same PCG as solve_jacobi_cg (stopping on the
true residual), with z = V(r) instead of z = D^-1 r.
The smoother parameters (theta, sweeps per level) and the cycle are INPUTS of
this module (reading M5/M8: the paper gives no multigrid, the values used are
chosen by measurement on the GPU and passed in by the tests); nothing here is
tuned to the GPU implementation.
"""
import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp


def coarse_dims(nelx, nely, nelz):
    """M1: coarse grid of ceil(n/2) elements per axis."""
    return (nelx + 1) // 2, (nely + 1) // 2, (nelz + 1) // 2


def prolongation_1d(n):
    """M2 along one axis: (n+1) fine nodes x (ceil(n/2)+1) coarse nodes."""
    nc = (n + 1) // 2
    P = np.zeros((n + 1, nc + 1))
    for i in range(n + 1):
        if i % 2 == 0:
            P[i, i // 2] = 1.0
        else:
            P[i, (i - 1) // 2] = 0.5
            P[i, (i + 1) // 2] = 0.5
    return P


def prolongation(nelx, nely, nelz):
    """M2: DOF-level trilinear interpolation P [3 n_nd_fine, 3 n_nd_coarse] in the
    SPEC S:45 numbering (node = iz (nx+1)(ny+1) + ix (ny+1) + iy, DOF 3n + c):
    node-level P = Pz (x) Px (x) Py, DOF-level = P_node (x) I_3."""
    Px, Py, Pz = (sp.csr_matrix(prolongation_1d(n)) for n in (nelx, nely, nelz))
    Pn = sp.kron(Pz, sp.kron(Px, Py))
    P = sp.kron(Pn, sp.identity(3)).tocsr()
    P.eliminate_zeros()                 # kron keeps explicit zeros; the sparsity pattern is used (Q)
    return P


def prolongation_loops(nelx, nely, nelz):
    """Same matrix by explicit enumeration of fine nodes (brute-force check)."""
    cx, cy, cz = coarse_dims(nelx, nely, nelz)
    w1 = [prolongation_1d(n) for n in (nelx, nely, nelz)]
    rows, cols, vals = [], [], []
    for iz in range(nelz + 1):
        for ix in range(nelx + 1):
            for iy in range(nely + 1):
                n = iz * (nelx + 1) * (nely + 1) + ix * (nely + 1) + iy
                for jz in range(cz + 1):
                    for jx in range(cx + 1):
                        for jy in range(cy + 1):
                            w = w1[0][ix, jx] * w1[1][iy, jy] * w1[2][iz, jz]
                            if w == 0.0:
                                continue
                            m = jz * (cx + 1) * (cy + 1) + jx * (cy + 1) + jy
                            for c in range(3):
                                rows.append(3 * n + c)
                                cols.append(3 * m + c)
                                vals.append(w)
    nf = 3 * (nelx + 1) * (nely + 1) * (nelz + 1)
    nc = 3 * (cx + 1) * (cy + 1) * (cz + 1)
    return sp.csr_matrix((vals, (rows, cols)), shape=(nf, nc))


def coarse_fixed(nelx, nely, nelz, fixed):
    """M4: coarse DOF (j, c) fixed iff fine node min(2j, n) (per axis) has DOF c fixed."""
    cx, cy, cz = coarse_dims(nelx, nely, nelz)
    fixed = np.asarray(fixed)
    out = np.zeros(3 * (cx + 1) * (cy + 1) * (cz + 1), dtype=np.uint8)
    for jz in range(cz + 1):
        for jx in range(cx + 1):
            for jy in range(cy + 1):
                ix, iy, iz = min(2 * jx, nelx), min(2 * jy, nely), min(2 * jz, nelz)
                n = iz * (nelx + 1) * (nely + 1) + ix * (nely + 1) + iy
                m = jz * (cx + 1) * (cy + 1) + jx * (cy + 1) + jy
                out[3 * m:3 * m + 3] = fixed[3 * n:3 * n + 3]
    return out


def property_q(P, fixed_f, fixed_c):
    """M4: True iff every fixed fine DOF receives interpolation weight only from
    fixed coarse DOFs (then masking commutes with the Galerkin product)."""
    rows = np.flatnonzero(np.asarray(fixed_f) != 0)
    sub = P[rows].tocoo()
    return not np.any(np.asarray(fixed_c)[sub.col] == 0)


def n_levels(nelx, nely, nelz, coarse_max=1000):
    """M6: number of levels: coarsen until a level has <= coarse_max DOFs (or
    the grid cannot shrink any more)."""
    dims, L = (nelx, nely, nelz), 1
    while 3 * (dims[0] + 1) * (dims[1] + 1) * (dims[2] + 1) > coarse_max:
        nd = coarse_dims(*dims)
        if nd == dims:
            break
        dims, L = nd, L + 1
    return L


def hierarchy(K, fixed, dims, n_lev=None, coarse_max=1000):
    """Levels [dict(dims, K, fixed, P (to the next-coarser level))], fine first (M1-M4)."""
    if n_lev is None:
        n_lev = n_levels(*dims, coarse_max=coarse_max)
    levels = [dict(dims=tuple(dims), K=K.tocsr(), fixed=np.asarray(fixed, dtype=np.uint8))]
    for _ in range(n_lev - 1):
        lv = levels[-1]
        P = prolongation(*lv["dims"])
        fc = coarse_fixed(*lv["dims"], lv["fixed"])
        if not property_q(P, lv["fixed"], fc):
            break                       # M4: stop coarsening where Q fails
        lv["P"] = P
        Kc = (P.T @ lv["K"] @ P).tocsr()
        levels.append(dict(dims=coarse_dims(*lv["dims"]), K=Kc, fixed=fc))
    return levels


def level_operator(lv):
    """A_l on the free DOFs, its diagonal and the free index set (M3)."""
    free = np.flatnonzero(lv["fixed"] == 0)
    A = lv["K"][free][:, free].tocsr()
    return A, A.diagonal(), free


def start_vector(n_dof, fixed):
    """M5: deterministic start vector of the power steps: DOF k (external
    numbering of its level) gets 2 u - 1, u = (splitmix64(k) >> 11) / 2^53;
    0 on fixed DOFs.  Integer arithmetic, so any implementation reproduces it."""
    M = (1 << 64) - 1
    v = np.zeros(n_dof)
    for k in range(n_dof):
        z = (k + 0x9E3779B97F4A7C15) & M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        z = z ^ (z >> 31)
        v[k] = 2.0 * ((z >> 11) * 2.0 ** -53) - 1.0
    v[np.asarray(fixed) != 0] = 0.0
    return v


def lambda_estimate(lv, k=8):
    """M5: lam = (v^T A v) / (v^T D v) after v <- D^-1 A v applied k times
    (power method on D^-1 A, no normalisation needed for k this small)."""
    A, d, free = level_operator(lv)
    v = start_vector(lv["K"].shape[0], lv["fixed"])[free]
    for _ in range(k):
        v = (A @ v) / d
    return float((v @ (A @ v)) / (v @ (d * v)))


def jacobi_bound(KE):
    """lam_bar = lam_max(KE) / KE_ii >= lam_max(D^-1 K) for every modulus field
    E > 0 and every Dirichlet set (reading M5): x^T K x = sum_e E_e x_e^T KE x_e
    <= lam_max(KE) sum_e E_e |x_e|^2 = (lam_max(KE) / KE_ii) x^T D x, because
    KE's diagonal is constant (App. A)."""
    KE = np.asarray(KE)
    return float(np.linalg.eigvalsh(KE).max() / KE[0, 0])


def smoother_weights(levels, theta=1.6, k=8):
    """w_l = theta / lam_l on every level but the coarsest (M5)."""
    for lv in levels[:-1]:
        lv["lam"] = lambda_estimate(lv, k)
        lv["omega"] = theta / lv["lam"]
    return levels


def level_sweeps(levels, nu=1, nu_deep=0, deep_nodes=150000):
    """Sweeps per level (M5): nu on the fine level and on coarse levels with more
    than deep_nodes nodes; nu_deep (0 -> nu) on the smaller coarse levels.  Both
    are inputs (the GPU's choice is passed in by the tests)."""
    def nodes(d):
        return (d[0] + 1) * (d[1] + 1) * (d[2] + 1)
    out = []
    for l, lv in enumerate(levels):
        if l == 0 or nodes(lv["dims"]) > deep_nodes or nu_deep <= 0:
            out.append(nu)
        else:
            out.append(nu_deep)
    return out


def coarse_correction(levels, rc, omega, nu, l, ops, cycle="V", kmax=None):
    """Approximate A_l^{-1} rc on coarse level l (full-length vector, 0 on fixed
    DOFs) -- reading M8.  cycle "V": one cycle B_l(rc).  cycle "K" (Notay &
    Vassilevski 2008, K-cycle = two steps of flexible CG preconditioned by B_l):
        x1 = B_l(rc);  v1 = A x1;  rho1 = x1.v1;  a1 = x1.rc;  r2 = rc - (a1/rho1) v1
        x2 = B_l(r2);  v2 = A x2;  g = x2.v1;  b = x2.v2;  a2 = x2.r2;  rho2 = b - g^2/rho1
        e  = (a1/rho1 - g a2/(rho1 rho2)) x1 + (a2/rho2) x2     (rho2 <= 0: second step dropped)
    i.e. e is the A-orthogonal (Galerkin) projection of A^-1 rc onto span{x1, x2}.
    The coarsest level is solved exactly (never K'd); kmax (None = every level
    above the coarsest) limits the K-cycle to levels l <= kmax (an input: the
    GPU keeps a single cycle on the level above the coarsest of 6+ level
    hierarchies, reading M8)."""
    if cycle == "V" or l == len(levels) - 1 or (kmax is not None and l > kmax):
        return vcycle(levels, rc, omega, nu, l, ops, cycle, kmax)
    A, _, free = ops[l]

    def Ax(x):
        y = np.zeros_like(x)
        y[free] = A @ x[free]
        return y
    x1 = vcycle(levels, rc, omega, nu, l, ops, cycle, kmax)
    v1 = Ax(x1)
    rho1, a1 = float(x1 @ v1), float(x1 @ rc)
    r2 = rc - (a1 / rho1) * v1
    x2 = vcycle(levels, r2, omega, nu, l, ops, cycle, kmax)
    v2 = Ax(x2)
    g, bb, a2 = float(x2 @ v1), float(x2 @ v2), float(x2 @ r2)
    rho2 = bb - g * g / rho1
    if not rho2 > 0.0:
        return (a1 / rho1) * x1
    return (a1 / rho1 - g * a2 / (rho1 * rho2)) * x1 + (a2 / rho2) * x2


def vcycle(levels, b, omega=None, nu=1, _l=0, _ops=None, cycle="V", kmax=None):
    """One V-cycle z = V(b) for a full-length level-_l vector b (0 on fixed DOFs).
    M5/M6; textbook recursion (Briggs, Henson, McCormick, "A Multigrid Tutorial",
    V-cycle scheme), written out without fusion.  omega None -> each level's
    lv["omega"] (smoother_weights), else one fixed weight on every level.
    nu: sweeps per side, one int for every level or a per-level sequence (M5)."""
    if _ops is None:
        _ops = [level_operator(lv) for lv in levels]
        for k, lv in enumerate(levels):
            if k == len(levels) - 1:
                lv["chol"] = sla.cho_factor(_ops[k][0].toarray())
    A, d, free = _ops[_l]
    lv = levels[_l]
    bf = b[free]
    w = lv.get("omega") if omega is None else omega
    if _l == len(levels) - 1:
        xf = sla.cho_solve(lv["chol"], bf)
    else:
        nl = nu[_l] if hasattr(nu, "__len__") else nu
        xf = np.zeros_like(bf)
        for _ in range(nl):
            xf = xf + w * (bf - A @ xf) / d
        r = np.zeros_like(b)
        r[free] = bf - A @ xf
        rc = lv["P"].T @ r
        rc[levels[_l + 1]["fixed"] != 0] = 0.0
        ec = coarse_correction(levels, rc, omega, nu, _l + 1, _ops, cycle, kmax)
        xf = xf + (lv["P"] @ ec)[free]
        for _ in range(nl):
            xf = xf + w * (bf - A @ xf) / d
    x = np.zeros_like(b)
    x[free] = xf
    return x


def solve_mgcg(K, f, fixed, dims, rtol=1e-10, theta=1.6, nu=1, coarse_max=1000,
               max_iter=10000, u0=None, power_steps=8, nu_deep=0, cycle="V", flexible=None, kmax=None):
    """PCG with the multigrid preconditioner (cycle "V" or "K", M8) on K_ff u_f =
    f_f, stopping on the TRUE relative residual (same loop as solve_jacobi_cg).
    flexible (default: True for the K-cycle) -> Polak-Ribiere beta (M9).
    Returns (u, iters)."""
    if flexible is None:
        flexible = cycle == "K"
    levels = smoother_weights(hierarchy(K, fixed, dims, coarse_max=coarse_max), theta, power_steps)
    nu = level_sweeps(levels, nu, nu_deep)
    ops = [level_operator(lv) for lv in levels]
    levels[-1]["chol"] = sla.cho_factor(ops[-1][0].toarray())
    A, _, free = ops[0]
    fx = np.asarray(fixed) != 0
    nb = np.linalg.norm(f[~fx])
    u = np.zeros(K.shape[0]) if u0 is None else np.where(fx, 0.0, u0)
    if nb == 0.0:
        return np.zeros(K.shape[0]), 0

    def M(r):
        return vcycle(levels, r, None, nu, 0, ops, cycle, kmax)

    def res(u):
        r = np.zeros_like(u)
        r[free] = f[free] - A @ u[free]
        return r
    r = res(u)
    z = M(r)
    p = z.copy()
    rz = r @ z
    it = 0
    while it < max_iter:
        if np.linalg.norm(r) <= rtol * nb:
            rt = res(u)
            if np.linalg.norm(rt) <= rtol * nb:
                break
            r = rt
            z = M(r)
            p = z.copy()
            rz = r @ z
        q = np.zeros_like(p)
        q[free] = A @ p[free]
        alpha = rz / (p @ q)
        u = u + alpha * p
        r = r - alpha * q
        z = M(r)
        rz_new = r @ z
        beta = -alpha * (z @ q) / rz if flexible else rz_new / rz     # M9: z.(r_new - r_old) = -alpha z.q
        p = z + beta * p
        rz = rz_new
        it += 1
    return u, it
