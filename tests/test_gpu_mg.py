"""GPU parity of the geometric multigrid preconditioner (
DESIGN.md readings M1-M6) against oracle/mg.py, step by step:

  hierarchy          level grids equal the oracle's (coarse_max rule, property Q)
  A_l (Galerkin)     y = A_l x on every level vs the oracle's P^T K P, rel 1e-12
                     (mg_fp32 = 1: levels >= 1 in fp32, rel 1e-5 in L2: unit
                     roundoff 6e-8 times the ~30-term sums of each row)
  V-cycle            z = V(b) vs the oracle's textbook recursion, rel 1e-9
                     (fp32 levels: 1e-4)
  MG-PCG solve       true residual <= 1e-10, u within 1e-8 of the direct solve,
                     far fewer iterations than Jacobi-PCG
  SIMP loop          c history within 1e-6 of the oracle (MG preconditioning
                     changes only how u is reached)
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from workloads import (make_problem, config_params, cantilever_load, cantilever_fixed,  # noqa: E402
                       cylinder_passive, random_density, random_vector)
import oracle  # noqa: E402
from oracle import mg  # noqa: E402


@pytest.fixture(scope="module")
def topo():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_05604_b200 import topo as t
    return t


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.linalg.norm(a - b) / np.linalg.norm(b), np.max(np.abs(a - b)) / np.max(np.abs(b))


def assert_rel(a, b, tol, what=""):
    r2, rm = rel(a, b)
    assert r2 <= tol and rm <= tol, f"{what}: relL2={r2:.3e} relmax={rm:.3e} tol={tol:g}"


# (dims, obstacle): even/odd sizes, 2..5 levels, an obstacle, one-element-thick axes
CASES = [
    ((30, 10, 2), None),                 # config 0 grid: 2 levels (level 1 stored = coarsest)
    ((60, 20, 4), None),                 # config 1 grid: 3 levels
    ((37, 13, 5), (18.0, 6.0, 3.0)),     # odd sizes, obstacle
    ((48, 16, 8), (24.0, 8.0, 3.2)),     # scaled config 2: 4 levels
    ((25, 7, 3), None),                  # odd, thin
]


def _case(dims, obst, seed=0, **over):
    p = config_params(dict(nelx=dims[0], nely=dims[1], nelz=dims[2], volfrac=0.3, rmin=1.5,
                           n_iter=5, cg_rtol=1e-10, obstacle=obst), precond="mg", **over)
    f, fx = cantilever_load(*dims), cantilever_fixed(*dims)
    pas = cylinder_passive(*dims, *obst) if obst else None
    x = random_density(int(np.prod(dims)), seed=seed)
    if pas is not None:
        x[pas != 0] = 0.0
    E = p["Emin"] + x ** p["penal"] * (p["E0"] - p["Emin"])
    K = oracle.assemble(*dims, oracle.element_stiffness(p["nu"]), E)
    return p, f, fx, pas, x, K


@pytest.mark.parametrize("dims,obst", CASES)
@pytest.mark.parametrize("fp32", [0, 1])
def test_mg_hierarchy_and_galerkin_operators(topo, dims, obst, fp32):
    p, f, fx, pas, x, K = _case(dims, obst, mg_fp32=fp32)
    lv = mg.hierarchy(K, fx, dims, coarse_max=1000)
    with topo.Problem(p, f, fx, pas) as pr:
        pr.set_xphys(x)
        assert pr.mg_levels() == [l["dims"] for l in lv]
        for l, L in enumerate(lv):
            xv = random_vector(L["K"].shape[0], seed=10 + l)
            y = pr.mg_apply(l, xv)
            yo = oracle.matvec_free(L["K"], xv, L["fixed"])
            if fp32 and l >= 1:
                r2, _ = rel(y, yo)
                assert r2 <= 1e-5, f"A_{l} fp32 relL2 {r2:.2e}"
            else:
                assert_rel(y, yo, 1e-12, f"A_{l} {L['dims']}")


@pytest.mark.parametrize("dims,obst", CASES)
@pytest.mark.parametrize("nu,fp32,deep,cycle", [(1, 0, 0, "V"), (2, 0, 0, "V"), (1, 1, 0, "V"), (2, 1, 0, "V"),
                                                (1, 0, 4, "V"), (1, 1, 6, "V"), (1, 0, 0, "K"), (1, 1, 0, "K"),
                                                (1, 0, 3, "K")])
def test_mg_vcycle_parity(topo, dims, obst, nu, fp32, deep, cycle):
    """z = B(b) for the V-cycle and the K-cycle (M8) vs the oracle's recursion."""
    p, f, fx, pas, x, K = _case(dims, obst, seed=1, mg_nu=nu, mg_omega=1.5, mg_fp32=fp32, mg_nu_deep=deep,
                                mg_cycle=cycle)
    lv = mg.smoother_weights(mg.hierarchy(K, fx, dims, coarse_max=1000), theta=1.5)
    b = np.where(fx == 0, random_vector(K.shape[0], seed=3), 0.0)
    zo = mg.vcycle(lv, b, None, nu=mg.level_sweeps(lv, nu, deep), cycle=cycle)
    with topo.Problem(p, f, fx, pas) as pr:
        pr.set_xphys(x)
        z = pr.mg_vcycle(b)
    assert_rel(z, zo, 1e-4 if fp32 else 1e-9, f"{cycle}-cycle {dims} nu={nu} fp32={fp32} deep={deep}")
    assert np.all(z[fx != 0] == 0)


@pytest.mark.parametrize("dims,obst", CASES)
@pytest.mark.parametrize("nu,fp32,deep,cycle", [(1, 0, 0, "V"), (1, 1, 0, "V"), (2, 1, 0, "V"), (1, 1, 8, "V"),
                                                (1, 0, 0, "K"), (1, 1, 0, "K")])
def test_mg_solve_parity(topo, dims, obst, nu, fp32, deep, cycle):
    """MG-PCG (V: standard PCG; K: flexible PCG, M9) solves to the direct
    solution, in the oracle's number of iterations (same algorithm, same
    parameters) and far fewer than Jacobi-PCG."""
    p, f, fx, pas, x, K = _case(dims, obst, seed=2, mg_fp32=fp32, mg_nu=nu, mg_nu_deep=deep, mg_cycle=cycle)
    uo = oracle.solve_direct(K, f, fx)
    _, it_o = mg.solve_mgcg(K, f, fx, dims, rtol=1e-10, theta=1.6, nu=nu, nu_deep=deep, cycle=cycle)
    its = {}
    for pc in ("jacobi", "mg"):
        with topo.Problem(dict(p, precond=pc), f, fx, pas) as pr:
            pr.set_xphys(x)
            u, info = pr.solve()
        assert info["precond"] == pc
        assert info["true_rel_res"] <= 1e-10
        assert oracle.true_residual(K, u, f, fx) <= 1e-10
        assert np.linalg.norm(u - uo) <= 1e-8 * np.linalg.norm(uo)
        its[pc] = info["iters"]
    assert abs(its["mg"] - it_o) <= (3 if fp32 else 2)   # same algorithm as the oracle's MG-PCG
    assert its["mg"] * 5 < its["jacobi"]


@pytest.mark.parametrize("cfg,n_iter", [(0, 20), (1, 10)])
def test_mg_loop_parity_configs(topo, cfg, n_iter):
    p, f, fx, pas = make_problem(cfg, precond="mg")
    ro = oracle.run_optimization(p, f, fx, pas, n_iter=n_iter)
    with topo.Problem(p, f, fx, pas) as pr:
        c, xo, nd = pr.optimize(n_iter)
        xphys = pr.get("xphys")
        _, info = pr.solve()
        assert pr.timings()["mg_fallbacks"] == 0
    assert info["precond"] == "mg" and info["mg_levels"] >= 2
    assert_rel(c, ro["c"], 1e-6, "c history (MG)")
    assert_rel(xphys, ro["xPhys"], 1e-6, "xPhys (MG)")


def test_mg_loop_parity_obstacle(topo):
    dims, obst = (48, 16, 8), (24.0, 8.0, 3.2)
    p = config_params(dict(nelx=48, nely=16, nelz=8, volfrac=0.2, rmin=2.5, n_iter=10,
                           cg_rtol=1e-10, obstacle=obst), precond="mg")
    f, fx = cantilever_load(*dims), cantilever_fixed(*dims)
    pas = cylinder_passive(*dims, *obst)
    ro = oracle.run_optimization(p, f, fx, pas, n_iter=10)
    with topo.Problem(p, f, fx, pas) as pr:
        c, x, nd = pr.optimize(10)
        xphys = pr.get("xphys")
    assert_rel(c, ro["c"], 1e-6, "c history (MG, obstacle)")
    assert_rel(xphys, ro["xPhys"], 1e-6, "xPhys (MG, obstacle)")


def test_mg_selection_rules(topo):
    """AUTO picks MG on one slab and on x-slabs (nu = 1), Jacobi on x-slabs with
    nu > 1 or when the grid is too small; explicit MG where the hierarchy cannot
    be built is EINVAL."""
    p, f, fx, pas = make_problem(0)
    lb = dict(mode=topo.TOPO_DIST_LOOPBACK, rank=0, world=2, device=0)
    with topo.Problem(p, f, fx, pas) as pr:
        assert len(pr.mg_levels()) == 2
    with topo.Problem(p, f, fx, pas, dist=lb) as pr:
        assert len(pr.mg_levels()) == 2
        _, info = pr.solve()
        assert info["precond"] == "mg"
    with topo.Problem(dict(p, mg_nu=2), f, fx, pas, dist=lb) as pr:
        assert pr.mg_levels() == []
        _, info = pr.solve()
        assert info["precond"] == "jacobi"
    with pytest.raises(topo.TopoError) as e:
        topo.Problem(dict(p, mg_nu=2, precond="mg"), f, fx, pas, dist=lb)
    assert e.value.code == topo.TOPO_EINVAL
    tiny = config_params(dict(nelx=3, nely=2, nelz=2, volfrac=0.3, rmin=1.5, n_iter=1,
                              cg_rtol=1e-10, obstacle=None))
    ft, fxt = cantilever_load(3, 2, 2), cantilever_fixed(3, 2, 2)
    with topo.Problem(tiny, ft, fxt) as pr:
        assert pr.mg_levels() == []
    with pytest.raises(topo.TopoError) as e:
        topo.Problem(dict(tiny, precond="mg"), ft, fxt)
    assert e.value.code == topo.TOPO_EINVAL
    # a single fixed odd node cannot be represented on the coarse grid (property Q)
    fx1 = np.zeros_like(fx)
    n = 1 * 11 * 31 + 1 * 11 + 1                     # node (ix, iy, iz) = (1, 1, 1)
    fx1[3 * n:3 * n + 3] = 1
    fx1[:3 * 11] = 1                                  # and the ix = 0, iz = 0 row
    with pytest.raises(topo.TopoError) as e:
        topo.Problem(dict(p, precond="mg"), f, fx1)
    assert e.value.code == topo.TOPO_EINVAL


def test_mg_long_run_no_jacobi_fallback(topo):
    """Config 1's full 50 iterations with the default (fp32-level) hierarchy: the
    warm-started smoother-weight estimate stays finite (normalised power vectors),
    so the hierarchy is never promoted to fp64, the solve never falls back to
    Jacobi and the c history matches the oracle."""
    p, f, fx, pas = make_problem(1)
    ro = oracle.run_optimization(p, f, fx, pas, n_iter=50)
    with topo.Problem(p, f, fx, pas) as pr:
        c, x, nd = pr.optimize(50)
        t = pr.timings()
    assert t["mg_fallbacks"] == 0
    assert t["mg_promotions"] == 0
    assert_rel(c, ro["c"], 1e-6, "c history (50 iterations, MG)")


@pytest.mark.gpu
def test_mg_paper_protocol_200_iterations(topo):
    """The paper's 200-iteration benchmark protocol (NEXT f1) on the
    default hierarchy: 400+ warm power steps per level over the run must neither
    overflow the smoother-weight estimate (promotion) nor break the V-cycle
    (Jacobi fallback); iteration counts stay multigrid-like throughout."""
    p, f, fx, pas = make_problem("paper")
    with topo.Problem(p, f, fx, pas) as pr:
        ncg = []
        for _ in range(200):
            pr.optimize(1)
            ncg.append(pr.timings()["cg_iters"])
        t = pr.timings()
    assert t["mg_fallbacks"] == 0 and t["mg_promotions"] == 0
    assert max(ncg) <= 40, ncg


@pytest.mark.parametrize("W", [2, 3, 4])
@pytest.mark.parametrize("fp32", [0, 1])
def test_mg_loopback_slabs_match_single(topo, W, fp32):
    """Multigrid on W x-slabs (in-process halo copies on one GPU; the coarse
    levels replicated, the level-1 restriction summed over slabs): the smoother
    weights, one V-cycle, a solve and a 5-iteration optimisation equal the single
    slab up to rounding (slab-boundary partial sums), and the oracle."""
    dims, obst = (37, 13, 5), (18.0, 6.0, 3.0)
    p, f, fx, pas, x, K = _case(dims, obst, seed=4, mg_fp32=fp32)
    b = np.where(fx == 0, random_vector(K.shape[0], seed=7), 0.0)
    outs = []
    for mode, world in ((topo.TOPO_DIST_SINGLE, 1), (topo.TOPO_DIST_LOOPBACK, W)):
        with topo.Problem(p, f, fx, pas, dist=dict(mode=mode, rank=0, world=world, device=0)) as pr:
            pr.set_xphys(x)
            z = pr.mg_vcycle(b)
            u, info = pr.solve()
            assert info["precond"] == "mg"
            pr.set_density(None)
            c, _, _ = pr.optimize(5)
            t = pr.timings()
            assert t["mg_fallbacks"] == 0 and t["mg_promotions"] == 0
            outs.append((z, u, info["iters"], c))
    (z1, u1, it1, c1), (zW, uW, itW, cW) = outs
    assert_rel(zW, z1, 1e-5 if fp32 else 1e-11, f"V-cycle W={W}")
    assert abs(itW - it1) <= 1
    assert oracle.true_residual(K, uW, f, fx) <= 1e-10
    assert_rel(uW, u1, 1e-7, f"u W={W}")
    assert_rel(cW, c1, 1e-9, f"c history W={W}")
    ro = oracle.run_optimization(p, f, fx, pas, n_iter=5)
    assert_rel(cW, ro["c"], 1e-6, "c history vs oracle")


@pytest.mark.gpu
def test_mg_theta_cut_recovers(topo):
    """An over-aggressive smoother theta (1.99: coarse-level weights beyond the
    convergent range) makes the V-cycle indefinite; the solve lowers theta
    (mg_theta_cuts) and still converges with multigrid, not Jacobi."""
    p, f, fx, pas, x, K = _case((60, 20, 4), None, seed=9, mg_omega=1.99)
    with topo.Problem(p, f, fx, pas) as pr:
        pr.set_xphys(x)
        u, info = pr.solve()
        t = pr.timings()
    assert oracle.true_residual(K, u, f, fx) <= 1e-10
    assert t["mg_fallbacks"] == 0
    assert info["precond"] == "mg"
    print("theta cuts", t["mg_theta_cuts"], "promotions", t["mg_promotions"], "iters", info["iters"])


def test_kcycle_iterations_config2(topo):
    """Config 2 (obstacle, 312k DOF, 5 levels), 14 SIMP iterations: the K-cycle
    (M8, flexible PCG M9) gives the same designs as the V-cycle (c history to
    1e-6: only the way u is reached differs) with far fewer PCG iterations once
    voids have formed (the V-cycle's count grows ~5x over the run)."""
    p, f, fx, pas = make_problem(2)
    out = {}
    for cyc in ("V", "K"):
        with topo.Problem(dict(p, mg_cycle=cyc), f, fx, pas) as pr:
            ncg, cs = [], []
            for _ in range(14):
                c, _, _ = pr.optimize(1, want_x=False)
                cs.append(c[0])
                ncg.append(pr.timings()["cg_iters"])
            out[cyc] = (np.array(cs), np.array(ncg))
    assert_rel(out["K"][0], out["V"][0], 1e-6, "c history K vs V")
    print("ncg V", out["V"][1].tolist(), "K", out["K"][1].tolist())
    assert out["K"][1][-4:].max() * 2 < out["V"][1][-4:].min()


@pytest.mark.parametrize("dims,obst", CASES[:4])
def test_krylov_fp32_refinement(topo, dims, obst):
    """SURVEY f3 as scoped (topo_params.krylov_fp32): the MG-PCG keeps r and q in
    fp32 inside fp64 iterative refinement (the fp64 true residual decides, with
    residual replacement): the solve still reaches the direct solution (u to
    1e-8, true residual 1e-10) -- only the route differs."""
    p, f, fx, pas, x, K = _case(dims, obst, seed=2, krylov_fp32=1)
    uo = oracle.solve_direct(K, f, fx)
    with topo.Problem(p, f, fx, pas) as pr:
        pr.set_xphys(x)
        u, info = pr.solve()
        r = pr.get("r")
    assert info["precond"] == "mg"
    assert info["true_rel_res"] <= 1e-10
    assert oracle.true_residual(K, u, f, fx) <= 1e-10
    assert np.linalg.norm(u - uo) <= 1e-8 * np.linalg.norm(uo)
    rt = np.where(fx != 0, 0.0, f - oracle.matvec_free(K, u, fx))
    assert np.linalg.norm(r - rt) <= 1e-6 * np.linalg.norm(f)    # the fp32 recursion tracks the true residual


@pytest.mark.parametrize("dims,obst", [((48, 16, 8), (24.0, 8.0, 3.2)), ((37, 13, 5), (18.0, 6.0, 3.0)),
                                       ((60, 20, 4), None)])
@pytest.mark.parametrize("fp32", [0, 1])
def test_l1_face_layout_matches_oracle(topo, monkeypatch, dims, obst, fp32):
    """The face-accumulating level-1 operator (k_mg_l1_face: x-complete face sums
    per node plane and element column, gathered from 4 faces; the default on
    grids with >= 1 M level-1 elements) forced on small grids: A_1 x against the
    oracle's Galerkin operator, and the V-cycle and K-cycle PCG solve against
    the element-corner layout (same sums, another order)."""
    p, f, fx, pas, x, K = _case(dims, obst, seed=4, mg_fp32=fp32)
    lv = mg.hierarchy(K, fx, dims, coarse_max=1000)
    assert len(lv) >= 3
    xv = random_vector(lv[1]["K"].shape[0], seed=11)
    yo = oracle.matvec_free(lv[1]["K"], xv, lv[1]["fixed"])
    b = np.where(fx == 0, random_vector(K.shape[0], seed=12), 0.0)
    out = {}
    for face in ("1", "0"):
        monkeypatch.setenv("TOPO_L1_FACE", face)
        with topo.Problem(p, f, fx, pas) as pr:
            pr.set_xphys(x)
            y = pr.mg_apply(1, xv)
            if fp32:
                assert rel(y, yo)[0] <= 1e-5, f"A_1 fp32 face={face}"
            else:
                assert_rel(y, yo, 1e-12, f"A_1 face={face}")
            z = pr.mg_vcycle(b)
            u, info = pr.solve()
            assert info["true_rel_res"] <= 1e-10
            out[face] = (z, u, info["iters"])
    assert_rel(out["1"][0], out["0"][0], 1e-5 if fp32 else 1e-11, "V-cycle face vs corners")
    assert_rel(out["1"][1], out["0"][1], 1e-8, "u face vs corners")
    assert abs(out["1"][2] - out["0"][2]) <= 1
