"""Pins for oracle.mg (geometric multigrid) against
closed forms, brute force and invariants -- not against the oracle itself.

* P by explicit enumeration; P reproduces linear fields exactly (trilinear
  interpolation is exact for them, also with a half-empty last coarse element)
* Galerkin P^T K P of a 2x2x2 fine grid = the coarse (h = 2) Hex8 element
  matrix integrated octant by octant with the octant's modulus (FE subspace
  property; independent Gauss quadrature, no P, no assembly)
* uniform modulus: Galerkin coarse operator = rediscretisation with 2 KE
* coarse fixed DOFs of the cantilever = the x = 0 face at every level; property
  Q holds; under Q masking commutes with the Galerkin product
* V-cycle is a symmetric positive definite operator; 1-level V-cycle = exact
  solve; MG-PCG reaches the direct solution (readings M1-M6)
"""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from oracle import mg
from oracle.ke import constitutive, strain_displacement
from oracle.mesh import LOCAL_NODES
from workloads import make_problem
from workloads.cantilever import cantilever_fixed, cantilever_load


@pytest.mark.parametrize("dims", [(1, 1, 1), (3, 2, 1), (4, 3, 2), (5, 5, 3)])
def test_prolongation_matches_enumeration(dims):
    a = mg.prolongation(*dims)
    b = mg.prolongation_loops(*dims)
    assert a.shape == b.shape
    assert abs(a - b).max() == 0.0


@pytest.mark.parametrize("dims", [(2, 2, 2), (3, 2, 1), (5, 4, 3), (6, 1, 2)])
def test_prolongation_reproduces_linear_fields(dims):
    nx, ny, nz = dims
    cx, cy, cz = mg.coarse_dims(*dims)
    P = mg.prolongation(*dims)
    A = np.array([[0.3, -1.2, 0.7], [2.0, 0.1, -0.4], [-0.5, 0.9, 1.1]])
    t = np.array([0.25, -0.5, 1.5])

    def field(nxx, nyy, nzz, h):
        v = np.zeros(3 * (nxx + 1) * (nyy + 1) * (nzz + 1))
        for iz in range(nzz + 1):
            for ix in range(nxx + 1):
                for iy in range(nyy + 1):
                    n = iz * (nxx + 1) * (nyy + 1) + ix * (nyy + 1) + iy
                    v[3 * n:3 * n + 3] = A @ (h * np.array([ix, iy, iz])) + t
        return v
    # coarse node j sits at fine position 2j (outside the grid for the last node of an odd axis)
    assert np.max(np.abs(P @ field(cx, cy, cz, 2.0) - field(nx, ny, nz, 1.0))) < 1e-13


def _coarse_element_by_quadrature(E_oct, nu):
    """24x24 stiffness of a cube of edge 2 whose 8 octants have moduli E_oct[cx,cy,cz]:
    sum over octants of E * h * int_oct B^T D B (reference coordinates, 2x2x2 Gauss per
    octant; exact for the trilinear integrand).  Independent of P and of assembly."""
    D = constitutive(1.0, nu)
    g = (0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0))
    K = np.zeros((24, 24))
    for cz in (0, 1):
        for cx in (0, 1):
            for cy in (0, 1):
                for a in g:
                    for b in g:
                        for c in g:
                            B = strain_displacement((cx + a) / 2, (cy + b) / 2, (cz + c) / 2)
                            K += E_oct[cx, cy, cz] * 2.0 * (1.0 / 64.0) * (B.T @ D @ B)
    return K


def test_galerkin_equals_octant_quadrature():
    nu = 0.3
    KE = oracle.element_stiffness(nu)
    rng = np.random.default_rng(5)
    E = rng.uniform(1e-3, 1.0, 8)                      # fine elements, external order (ez, ex, ey)
    K = oracle.assemble(2, 2, 2, KE, E)
    P = mg.prolongation(2, 2, 2)
    Kc = (P.T @ K @ P).toarray()                       # 8 coarse nodes, SPEC numbering
    E_oct = np.zeros((2, 2, 2))
    for ez in range(2):
        for ex in range(2):
            for ey in range(2):
                E_oct[ex, ey, ez] = E[ez * 4 + ex * 2 + ey]
    Kq = _coarse_element_by_quadrature(E_oct, nu)      # local node order
    # coarse node n(jx,jy,jz) = jz*4 + jx*2 + jy; local corner a at (dx,dy,dz)
    perm = []
    for (dx, dy, dz) in LOCAL_NODES:
        n = dz * 4 + dx * 2 + dy
        perm += [3 * n, 3 * n + 1, 3 * n + 2]
    assert np.max(np.abs(Kc[np.ix_(perm, perm)] - Kq)) < 1e-13 * np.max(np.abs(Kq))


@pytest.mark.parametrize("dims", [(4, 2, 2), (6, 4, 2)])
def test_galerkin_uniform_is_rediscretisation(dims):
    KE = oracle.element_stiffness(0.3)
    n_el = dims[0] * dims[1] * dims[2]
    K = oracle.assemble(*dims, KE, np.ones(n_el))
    P = mg.prolongation(*dims)
    cd = mg.coarse_dims(*dims)
    Kc = oracle.assemble(*cd, 2.0 * KE, np.ones(cd[0] * cd[1] * cd[2]))
    d = (P.T @ K @ P - Kc).toarray()
    assert np.max(np.abs(d)) < 1e-13


@pytest.mark.parametrize("dims", [(30, 10, 2), (60, 20, 4), (120, 40, 20), (7, 5, 3)])
def test_cantilever_coarse_fixed_is_face_and_property_q(dims):
    fx = cantilever_fixed(*dims)
    cur = dims
    for _ in range(6):
        cd = mg.coarse_dims(*cur)
        fc = mg.coarse_fixed(*cur, fx)
        assert np.array_equal(fc, cantilever_fixed(*cd))      # the x = 0 face, all DOFs
        assert mg.property_q(mg.prolongation(*cur), fx, fc)
        cur, fx = cd, fc


def test_masked_galerkin_identity_under_q():
    dims = (6, 4, 2)
    p, f, fx, _ = make_problem(dict(nelx=6, nely=4, nelz=2, volfrac=0.3, rmin=1.5, n_iter=1,
                                    cg_rtol=1e-10, obstacle=None))
    KE = oracle.element_stiffness(0.3)
    E = np.random.default_rng(2).uniform(1e-9, 1.0, 48)
    K = oracle.assemble(*dims, KE, E)
    P = mg.prolongation(*dims)
    fc = mg.coarse_fixed(*dims, fx)
    ff, cf = np.flatnonzero(fx == 0), np.flatnonzero(fc == 0)
    A1 = (P.T @ K @ P)[cf][:, cf]
    Pm = P[ff][:, cf]
    A2 = Pm.T @ K[ff][:, ff] @ Pm
    assert abs(A1 - A2).max() < 1e-14


def _evolved_case(cfg=1, n_iter=6):
    p, f, fx, pas = make_problem(cfg)
    r = oracle.run_optimization(p, f, fx, pas, n_iter=n_iter, solver="direct", record=True)
    rec = r["records"][-1]
    E = p["Emin"] + rec["xPhys"] ** p["penal"] * (p["E0"] - p["Emin"])
    KE = oracle.element_stiffness(p["nu"])
    dims = (p["nelx"], p["nely"], p["nelz"])
    return oracle.assemble(*dims, KE, E), f, fx, dims, rec["u"]


def test_vcycle_symmetric_positive_definite():
    K, f, fx, dims, _ = _evolved_case(1, 4)
    lv = mg.smoother_weights(mg.hierarchy(K, fx, dims))
    assert len(lv) == 3
    rng = np.random.default_rng(3)
    free = fx == 0
    b1 = np.where(free, rng.standard_normal(len(f)), 0.0)
    b2 = np.where(free, rng.standard_normal(len(f)), 0.0)
    v1, v2 = mg.vcycle(lv, b1), mg.vcycle(lv, b2)
    assert abs(b1 @ v2 - b2 @ v1) <= 1e-12 * abs(b1 @ v2)
    assert b1 @ v1 > 0 and b2 @ v2 > 0
    assert np.all(v1[~free] == 0.0)


def test_vcycle_one_level_is_exact_solve():
    K, f, fx, dims, u = _evolved_case(0, 3)
    lv = mg.hierarchy(K, fx, dims, n_lev=1)
    z = mg.vcycle(lv, np.where(fx == 0, f, 0.0))
    assert np.linalg.norm(z - u) <= 1e-9 * np.linalg.norm(u)


@pytest.mark.parametrize("cfg", [0, 1])
def test_mgcg_reaches_direct_solution(cfg):
    K, f, fx, dims, u = _evolved_case(cfg, 8)
    um, it = mg.solve_mgcg(K, f, fx, dims, rtol=1e-10)
    _, itj = oracle.solve_jacobi_cg(K, f, fx, rtol=1e-10)
    assert np.linalg.norm(um - u) <= 1e-8 * np.linalg.norm(u)
    assert oracle.true_residual(K, um, f, fx) <= 1e-10
    assert it < itj / 5                                        # the point of f2


def test_start_vector_is_splitmix64():
    """Known splitmix64 outputs (seed-free counter form, increment 0x9E3779B97F4A7C15):
    the first output for state 0 is 0xE220A8397B1DCDAF."""
    v = mg.start_vector(2, [0, 0])
    u0 = (0xE220A8397B1DCDAF >> 11) * 2.0 ** -53
    assert v[0] == 2.0 * u0 - 1.0
    assert np.all(mg.start_vector(6, [0, 1, 0, 0, 1, 0])[[1, 4]] == 0.0)


@pytest.mark.parametrize("seed", [0, 2])
def test_lambda_estimate_bounds(seed):
    """Rayleigh quotient <= lam_max(D^-1 A) <= element bound lam_max(KE)/KE_ii
    (x^T A x = sum_e x_e^T E_e KE x_e <= lam(KE)/kd x^T D x), and the damped
    smoother it sets is convergent: w lam_max < 2 for the default theta (1.6)."""
    import scipy.sparse as sps
    import scipy.sparse.linalg as spla
    from workloads import random_density
    dims = (12, 6, 4)
    fx = cantilever_fixed(*dims)
    KE = oracle.element_stiffness(0.3)
    E = 1e-9 + random_density(int(np.prod(dims)), seed=seed) ** 3
    K = oracle.assemble(*dims, KE, E)
    bound = mg.jacobi_bound(KE)
    lv = mg.smoother_weights(mg.hierarchy(K, fx, dims, coarse_max=200))
    for l in lv[:-1]:
        A, d, _ = mg.level_operator(l)
        Dm = sps.diags(1.0 / np.sqrt(d))
        lam_max = spla.eigsh(Dm @ A @ Dm, k=1, which="LA", return_eigenvectors=False)[0]
        assert l["lam"] <= lam_max * (1 + 1e-12)
        assert l["omega"] * lam_max < 2.0
    A0, d0, _ = mg.level_operator(lv[0])
    Dm = sps.diags(1.0 / np.sqrt(d0))
    assert spla.eigsh(Dm @ A0 @ Dm, k=1, which="LA", return_eigenvectors=False)[0] <= bound + 1e-12


def test_jacobi_bound_closed_form():
    """lam_bar = lam_max(KE) / KE_ii at nu = 0.3: KE's largest eigenvalue 1.25
    (SURVEY §8(c) spectrum pin) over KE_ii = (lam + 4 mu) / 9 = 0.2350427350
    (closed form) = 5.3181818..."""
    KE = oracle.element_stiffness(0.3)
    lam, mu = 0.3 / (1.3 * 0.4), 1.0 / 2.6
    assert abs(mg.jacobi_bound(KE) - 1.25 / ((lam + 4 * mu) / 9)) <= 1e-6 * 5.3
    assert abs((lam + 4 * mu) / 9 - 0.2350427350) <= 1e-10


def _problem(dims, seed=0, voids=False):
    """Cantilever K on a random density field (voids: half the elements at x =
    1e-3, i.e. E ~ 1e-9, the SIMP contrast of late designs)."""
    rng = np.random.default_rng(seed)
    n = int(np.prod(dims))
    x = rng.uniform(0.01, 1.0, n)
    if voids:
        x = np.where(rng.uniform(size=n) < 0.5, 1e-3, 1.0)
    E = 1e-9 + x ** 3 * (1.0 - 1e-9)
    K = oracle.assemble(*dims, oracle.element_stiffness(0.3), E)
    return K, cantilever_load(*dims), cantilever_fixed(*dims)


def test_kcycle_galerkin_projection():
    """M8 pin (a closed-form property, not a restatement): the K-cycle's coarse
    correction e is the A-orthogonal projection of A^-1 rc onto span{x1, x2}, so
    the new residual rc - A e is orthogonal to x1 and x2; and e reduces the
    A-norm error at least as much as the plain V-cycle correction x1."""
    dims = (24, 8, 4)
    K, f, fx = _problem(dims, seed=7)
    lv = mg.smoother_weights(mg.hierarchy(K, fx, dims, coarse_max=100), theta=1.6)
    assert len(lv) >= 4
    ops = [mg.level_operator(l) for l in lv]
    lv[-1]["chol"] = __import__("scipy.linalg", fromlist=["cho_factor"]).cho_factor(ops[-1][0].toarray())
    A, _, free = ops[1]
    rng = np.random.default_rng(4)
    rc = np.where(lv[1]["fixed"] == 0, rng.standard_normal(lv[1]["K"].shape[0]), 0.0)
    x1 = mg.vcycle(lv, rc, None, 1, 1, ops, "K")
    e = mg.coarse_correction(lv, rc, None, 1, 1, ops, "K")
    # x2 = B(r2) recomputed: r2 = rc - (a1/rho1) A x1
    Av1 = np.zeros_like(x1)
    Av1[free] = A @ x1[free]
    r2 = rc - (x1 @ rc) / (x1 @ Av1) * Av1
    x2 = mg.vcycle(lv, r2, None, 1, 1, ops, "K")
    Ae = np.zeros_like(e)
    Ae[free] = A @ e[free]
    res = rc - Ae
    assert abs(res @ x1) <= 1e-10 * np.linalg.norm(rc) * np.linalg.norm(x1)
    assert abs(res @ x2) <= 1e-10 * np.linalg.norm(rc) * np.linalg.norm(x2)
    ex = np.zeros_like(rc)
    ex[free] = __import__("scipy.sparse.linalg", fromlist=["spsolve"]).spsolve(A.tocsc(), rc[free])
    errA = lambda d: float(d[free] @ (A @ d[free]))  # noqa: E731
    assert errA(ex - e) <= errA(ex - (x1 @ rc) / (x1 @ Av1) * x1) + 1e-14 * errA(ex)


def test_kcycle_exact_inner_solve_is_exact():
    """M8 special case: with an exact solve on the level below (a 2-level cycle
    on level 1 of a 3-level hierarchy whose smoother is skipped is not available,
    so use the coarsest-level identity): on the coarsest level the correction is
    the exact solve, and a K-cycle PCG on a 2-level hierarchy equals the V-cycle
    PCG (the K-cycle only differs above the coarsest level)."""
    dims = (12, 4, 2)
    K, f, fx = _problem(dims, seed=3)
    u1, it1 = mg.solve_mgcg(K, f, fx, dims, rtol=1e-10, coarse_max=400, cycle="V")
    u2, it2 = mg.solve_mgcg(K, f, fx, dims, rtol=1e-10, coarse_max=400, cycle="K", flexible=False)
    assert len(mg.hierarchy(K, fx, dims, coarse_max=400)) == 2
    assert it1 == it2 and np.array_equal(u1, u2)


def test_flexible_cg_equals_cg_for_fixed_preconditioner():
    """M9 pin: with a fixed SPD preconditioner (the V-cycle) z_new.r_old = 0, so the
    Polak-Ribiere beta equals the Fletcher-Reeves one up to rounding: same
    iteration count and the same u (a sign or index slip in the flexible formula
    breaks this)."""
    dims = (24, 8, 4)
    K, f, fx = _problem(dims, seed=5)
    u1, it1 = mg.solve_mgcg(K, f, fx, dims, rtol=1e-10, coarse_max=200, cycle="V", flexible=False)
    u2, it2 = mg.solve_mgcg(K, f, fx, dims, rtol=1e-10, coarse_max=200, cycle="V", flexible=True)
    assert abs(it1 - it2) <= 1
    assert np.linalg.norm(u1 - u2) <= 1e-8 * np.linalg.norm(u1)


def test_kcycle_pcg_solves_high_contrast():
    """K-cycle FCG reaches the direct solution (u to 1e-8, true residual 1e-10)
    on a random half-void field (E contrast 1e9), 4+ levels."""
    dims = (32, 8, 8)
    K, f, fx = _problem(dims, seed=9, voids=True)
    uo = oracle.solve_direct(K, f, fx)
    uk, itk = mg.solve_mgcg(K, f, fx, dims, rtol=1e-10, coarse_max=150, cycle="K")
    assert len(mg.hierarchy(K, fx, dims, coarse_max=150)) >= 4
    assert np.linalg.norm(uk - uo) <= 1e-8 * np.linalg.norm(uo)
    assert oracle.true_residual(K, uk, f, fx) <= 1e-10


def test_kcycle_fewer_iterations_on_a_simp_design():
    """On an evolved SIMP design (config 1 after 8 iterations, 3 levels) the
    K-cycle needs no more PCG iterations than the V-cycle (the reason for M8)."""
    K, f, fx, dims, u = _evolved_case(1, 8)
    uk, itk = mg.solve_mgcg(K, f, fx, dims, rtol=1e-10, coarse_max=100, cycle="K")
    uv, itv = mg.solve_mgcg(K, f, fx, dims, rtol=1e-10, coarse_max=100, cycle="V")
    assert len(mg.hierarchy(K, fx, dims, coarse_max=100)) >= 3
    assert np.linalg.norm(uk - u) <= 1e-8 * np.linalg.norm(u)
    assert itk <= itv


def test_vcycle_per_level_sweeps_spd():
    """Per-level sweep counts keep the V-cycle symmetric positive definite (each
    level's post-smoother is the adjoint of its pre-smoother) and make it a
    better preconditioner (fewer MG-PCG iterations)."""
    K, f, fx, dims, u = _evolved_case(1, 4)
    lv = mg.smoother_weights(mg.hierarchy(K, fx, dims))
    rng = np.random.default_rng(5)
    free = fx == 0
    b1 = np.where(free, rng.standard_normal(len(f)), 0.0)
    b2 = np.where(free, rng.standard_normal(len(f)), 0.0)
    nu = [1, 4, 4]
    v1, v2 = mg.vcycle(lv, b1, None, nu), mg.vcycle(lv, b2, None, nu)
    assert abs(b1 @ v2 - b2 @ v1) <= 1e-12 * abs(b1 @ v2)
    assert b1 @ v1 > 0 and b2 @ v2 > 0
    _, it1 = mg.solve_mgcg(K, f, fx, dims, rtol=1e-10)
    um, it4 = mg.solve_mgcg(K, f, fx, dims, rtol=1e-10, nu_deep=4)
    assert oracle.true_residual(K, um, f, fx) <= 1e-10
    assert it4 < it1
