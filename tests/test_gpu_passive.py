"""GPU parity with passive regions (reading R27): passive
void (mask 1, the paper's obstacles P:47) and passive SOLID (mask 2,
S:252) elements, the OC's BisectionFailure (S:283 -> TOPO_EBISECT), and the
paper's section-3 protocol with its cylinder obstacle.
Tolerances as in test_gpu_parity.py (north_star)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from workloads import (config_params, cantilever_load, cantilever_fixed, solid_block_passive,  # noqa: E402
                       random_density, make_problem)
import oracle  # noqa: E402


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


def assert_rel(a, b, tol, what):
    r2, rm = rel(a, b)
    assert r2 <= tol and rm <= tol, f"{what}: relL2={r2:.3e} relmax={rm:.3e}"


# (dims, rmin, solid box (x range, y range, z range), void cylinder (cx, cy, r) or None)
CASES = [
    ((30, 10, 4), 1.5, ((20, 24), (0, 3), (0, 4)), (12.0, 5.0, 2.0)),
    ((37, 13, 5), 2.5, ((25, 30), (0, 4), (1, 4)), (15.0, 6.0, 3.0)),
    ((23, 9, 7), 3.0, ((0, 4), (5, 9), (0, 7)), None),
]


def _problem(case, **over):
    dims, rmin, box, cyl = case
    p = config_params(dict(nelx=dims[0], nely=dims[1], nelz=dims[2], volfrac=0.25, rmin=rmin,
                           n_iter=8, cg_rtol=1e-10, obstacle=None), **over)
    f, fx = cantilever_load(*dims), cantilever_fixed(*dims)
    pas = solid_block_passive(*dims, *box, base=cyl)
    return p, f, fx, pas


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_step_parity_solid_void(topo, case, mode):
    """One SIMP step on identical inputs with solid and void regions."""
    p, f, fx, pas = _problem(case, filter_mode=mode)
    dims = (p["nelx"], p["nely"], p["nelz"])
    n_el = int(np.prod(dims))
    KE = oracle.element_stiffness(p["nu"])
    edof = oracle.edof_matrix(*dims)
    H, Hs = oracle.filter_matrix(*dims, p["rmin"])
    x = random_density(n_el, seed=4, lo=0.05, hi=0.45)
    x[pas == 1] = 0.0
    x[pas == 2] = 1.0
    with topo.Problem(p, f, fx, pas) as pr:
        pr.set_density(x)
        assert np.array_equal(pr.get("x"), x)
        u, info = pr.solve()
        E = pr.get("E")
        c, ce, dc = pr.sensitivity()
        dcf = pr.filter("dc")
        dvf = pr.get("dvf")
        xnew, lam, chg, vol = pr.oc_step()
        xphys = pr.get("xphys")
    assert np.all(E[pas == 2] == p["E0"])
    K = oracle.assemble(*dims, KE, E)
    assert oracle.true_residual(K, u, f, fx) <= 1e-10
    ce_o = oracle.element_energies(u, KE, edof)
    _, c_o, dc_o, dv_o = oracle.sensitivities(x, ce_o, p["penal"], p["E0"], p["Emin"], pas)
    assert_rel(ce, ce_o, 1e-9, "ce")
    assert_rel(dc, dc_o, 1e-9, "dc")
    assert c == pytest.approx(c_o, rel=1e-9)
    dcf_o = oracle.apply_filter(H, Hs, mode, "dc", dc, x=x, passive=pas)
    dvf_o = oracle.apply_filter(H, Hs, mode, "dv", dv_o, x=x, passive=pas)
    assert_rel(dcf, dcf_o, 1e-9, "dc~")
    assert_rel(dvf, dvf_o, 1e-13, "dv~")
    xn_o, lam_o, V_o, _ = oracle.oc_update(x, dcf_o, dvf_o, p["volfrac"], p["move"], p["oc_tol"],
                                           p["oc_lmax"], mode, H, Hs, pas)
    assert lam == pytest.approx(lam_o, rel=1e-8)
    assert_rel(xnew, xn_o, 1e-9, "xnew")
    D = pas == 0
    assert chg == pytest.approx(np.max(np.abs(xn_o - x)[D]), rel=1e-9, abs=1e-12)
    xp_o = oracle.apply_filter(H, Hs, mode, "x", xn_o, passive=pas)
    assert_rel(xphys, xp_o, 1e-9, "xPhys")
    assert abs(vol - p["volfrac"]) <= 1e-6
    assert np.all(xnew[pas == 2] == 1.0) and np.all(xphys[pas == 2] == 1.0)
    assert np.all(xnew[pas == 1] == 0.0) and np.all(xphys[pas == 1] == 0.0)


@pytest.mark.parametrize("precond", ["jacobi", "mg"])
@pytest.mark.parametrize("mode", [0, 1])
def test_loop_parity_solid_void(topo, precond, mode):
    """8 SIMP iterations with a solid block and a void cylinder: c history to
    1e-6, final xPhys to 1e-6, passive values held."""
    case = ((48, 16, 8), 2.5, ((36, 44), (0, 5), (0, 8)), (20.0, 8.0, 3.2))
    p, f, fx, pas = _problem(case, filter_mode=mode, precond=precond)
    ro = oracle.run_optimization(p, f, fx, pas, n_iter=8)
    with topo.Problem(p, f, fx, pas) as pr:
        c, x, nd = pr.optimize(8)
        xphys = pr.get("xphys")
        t = pr.timings()
    assert nd == 8
    assert_rel(c, ro["c"], 1e-6, "c history")
    assert_rel(xphys, ro["xPhys"], 1e-6, "xPhys")
    assert abs(t["volume"] - p["volfrac"]) <= 1e-6
    assert np.all(xphys[pas == 2] == 1.0) and np.all(xphys[pas == 1] == 0.0)
    assert np.all(x[pas == 2] == 1.0) and np.all(x[pas == 1] == 0.0)


@pytest.mark.parametrize("W", [2, 3])
def test_loopback_slabs_solid(topo, W):
    """x-slabs (loopback) with a solid block straddling a slab boundary."""
    case = ((36, 12, 6), 2.5, ((14, 22), (0, 4), (0, 6)), (9.0, 6.0, 2.5))
    p, f, fx, pas = _problem(case, precond="jacobi")
    outs = []
    for mode, world in ((topo.TOPO_DIST_SINGLE, 1), (topo.TOPO_DIST_LOOPBACK, W)):
        with topo.Problem(p, f, fx, pas, dist=dict(mode=mode, rank=0, world=world, device=0)) as pr:
            c, x, nd = pr.optimize(5)
            outs.append((c, pr.get("xphys")))
    assert_rel(outs[1][0], outs[0][0], 1e-9, "c W")
    assert_rel(outs[1][1], outs[0][1], 1e-8, "xPhys W")
    ro = oracle.run_optimization(p, f, fx, pas, n_iter=5)
    assert_rel(outs[1][0], ro["c"], 1e-6, "c vs oracle")


def test_solid_volume_infeasible_ebisect(topo):
    """the filtered solid spill alone exceeds the design volume target
    -> TOPO_EBISECT from topo_oc_step (the oracle raises BisectionFailure), and
    the design is left unchanged; a feasible target on the same mask passes."""
    dims = (12, 6, 6)
    n = int(np.prod(dims))
    pas = solid_block_passive(*dims, (0, 6), (0, 6), (0, 6))
    f, fx = cantilever_load(*dims), cantilever_fixed(*dims)
    H, Hs = oracle.filter_matrix(*dims, 2.5)
    D = pas == 0
    for volfrac, ok in ((0.03, False), (0.4, True)):
        p = config_params(dict(nelx=dims[0], nely=dims[1], nelz=dims[2], volfrac=volfrac, rmin=2.5,
                               n_iter=1, cg_rtol=1e-10, obstacle=None))
        x = np.where(D, volfrac, 0.0)
        x[pas == 2] = 1.0
        dv = oracle.apply_filter(H, Hs, 0, "dv", D.astype(float))
        with topo.Problem(p, f, fx, pas) as pr:
            pr.solve(want_u=False)
            _, _, dc = pr.sensitivity()
            dcf = pr.filter("dc")
            if ok:
                xnew, lam, chg, vol = pr.oc_step()
                xn_o, lam_o, _, _ = oracle.oc_update(x, dcf, dv, volfrac, p["move"], p["oc_tol"],
                                                     p["oc_lmax"], 0, H, Hs, pas)
                assert lam == pytest.approx(lam_o, rel=1e-8)
                assert abs(vol - volfrac) <= 1e-6
            else:
                with pytest.raises(oracle.BisectionFailure):
                    oracle.oc_update(x, dcf, dv, volfrac, p["move"], p["oc_tol"], p["oc_lmax"], 0, H, Hs,
                                     pas)
                with pytest.raises(topo.TopoError) as e:
                    pr.oc_step()
                assert e.value.code == topo.TOPO_EBISECT
                assert np.array_equal(pr.get("x"), x)


def test_bad_passive_value_einval(topo):
    p, f, fx, _ = make_problem(0)
    pas = np.zeros(600, dtype=np.uint8)
    pas[7] = 3
    with pytest.raises(topo.TopoError) as e:
        topo.Problem(p, f, fx, pas)
    assert e.value.code == topo.TOPO_EINVAL


@pytest.mark.parametrize("precond", ["jacobi", "mg"])
def test_paper_protocol_obstacle_parity(topo, precond):
    """The paper's section-3 example (32x16x16, point load, rmin 4, sensitivity
    filter) WITH its cylinder obstacle: first 5 iterations vs oracle."""
    p, f, fx, pas = make_problem("paper_obstacle", precond=precond)
    assert pas.sum() == 576
    ro = oracle.run_optimization(p, f, fx, pas, n_iter=5)
    with topo.Problem(p, f, fx, pas) as pr:
        c, x, nd = pr.optimize(5)
        xphys = pr.get("xphys")
    assert_rel(c, ro["c"], 1e-6, "c history (paper protocol, obstacle)")
    assert_rel(xphys, ro["xPhys"], 1e-6, "xPhys (paper protocol, obstacle)")
    assert np.all(xphys[pas != 0] == 0)
