"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by
element on identical seeded inputs.  Tolerances (north_star):
  matvec                      rel L2 <= 1e-13 (reordered fp64 sums)
  solve                       true rel. residual <= 1e-10, u rel L2 <= 1e-8 vs direct
  ce, dc, dc~, dv~, xPhys, xnew   <= 1e-9 relative (rel L2 AND max|d|/max|ref|, R#25)
  10-iteration c history      <= 1e-6 relative
  volume                      <= 1e-6 absolute on the mean design density
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from workloads import (make_problem, config_params, cantilever_load, cantilever_fixed,  # noqa: E402
                       cylinder_passive, random_density, random_vector)
import oracle  # noqa: E402


@pytest.fixture(scope="module")
def topo():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_05604_b200 import topo as t
    return t


def rel(a, b):
    """(rel L2, max|a-b|/max|b|) -- reading R#25."""
    a, b = np.asarray(a, float), np.asarray(b, float)
    nb = np.linalg.norm(b)
    mb = np.max(np.abs(b)) if b.size else 0.0
    return (np.linalg.norm(a - b) / nb if nb else np.linalg.norm(a)), \
           (np.max(np.abs(a - b)) / mb if mb else np.max(np.abs(a), initial=0.0))


def assert_rel(a, b, tol, what=""):
    r2, rm = rel(a, b)
    assert r2 <= tol and rm <= tol, f"{what}: relL2={r2:.3e} relmax={rm:.3e} tol={tol:g}"


# small grids that span several CUDA blocks and ragged tails; (dims, rmin, obstacle)
SMALL = [
    ((30, 10, 2), 1.5, None),            # config 0 grid
    ((60, 20, 4), 1.5, None),            # config 1 grid
    ((37, 13, 5), 2.5, (18.0, 6.0, 3.0)),  # ragged, obstacle, R = 2
    ((23, 9, 7), 3.0, None),             # R = 2, 93-point stencil, odd sizes
    ((9, 3, 2), 4.0, None),              # R = 3 wider than parts of the grid
    ((10, 45, 9), 1.5, None),            # 2 x 2 y-z matvec tiles (odd tile origins), ragged
    ((7, 66, 15), 2.5, (3.0, 30.0, 5.0)),  # 3 x 3 tiles, obstacle
]


def _problem(dims, rmin, obstacle, **over):
    p = config_params(dict(nelx=dims[0], nely=dims[1], nelz=dims[2], volfrac=0.3, rmin=rmin,
                           n_iter=10, cg_rtol=1e-10, obstacle=obstacle), **over)
    f, fx = cantilever_load(*dims), cantilever_fixed(*dims)
    pas = cylinder_passive(*dims, *obstacle) if obstacle else None
    return p, f, fx, pas


def _xfield(n_el, pas, seed=0, hi=1.0):
    x = random_density(n_el, seed=seed, hi=hi)
    if pas is not None:
        x[pas != 0] = 0.0
    return x


@pytest.mark.parametrize("case", SMALL)
def test_matvec_parity(topo, case):
    p, f, fx, pas = _problem(*case)
    dims = (p["nelx"], p["nely"], p["nelz"])
    n_el = np.prod(dims)
    KE = oracle.element_stiffness(p["nu"])
    x = _xfield(n_el, pas)
    E = p["Emin"] + x ** p["penal"] * (p["E0"] - p["Emin"])
    K = oracle.assemble(*dims, KE, E)
    pv = random_vector(K.shape[0], seed=1)
    qo = oracle.matvec_free(K, pv, fx)
    with topo.Problem(p, f, fx, pas) as pr:
        pr.set_xphys(x)
        pr.update_modulus()
        q = pr.apply_K(pv)
        assert_rel(pr.get("E"), E, 1e-15, "E")
        d = pr.get("invdiag")
        free = fx == 0
        dK = K.diagonal()
        assert np.all(d[~free] == 0)
        assert_rel(d[free], 1.0 / dK[free], 1e-14, "invdiag")
    assert_rel(q, qo, 1e-13, "matvec")


@pytest.mark.parametrize("case", SMALL[:3])
@pytest.mark.parametrize("precond", ["jacobi", "mg"])
def test_solve_parity_random_density(topo, case, precond):
    """Config 1's standalone solve on x ~ U[0.01, 1] (seed 0), plus others."""
    p, f, fx, pas = _problem(*case, precond=precond)
    dims = (p["nelx"], p["nely"], p["nelz"])
    x = _xfield(np.prod(dims), pas, seed=0)
    KE = oracle.element_stiffness(p["nu"])
    E = p["Emin"] + x ** p["penal"] * (p["E0"] - p["Emin"])
    K = oracle.assemble(*dims, KE, E)
    uo = oracle.solve_direct(K, f, fx)
    with topo.Problem(p, f, fx, pas) as pr:
        pr.set_xphys(x)
        u, info = pr.solve()
    assert info["true_rel_res"] <= 1e-10
    assert oracle.true_residual(K, u, f, fx) <= 1e-10
    assert np.linalg.norm(u - uo) <= 1e-8 * np.linalg.norm(uo)
    assert np.all(u[fx != 0] == 0)


@pytest.mark.parametrize("case", SMALL)
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_sens_filter_oc_parity(topo, case, mode):
    """One SIMP step on identical inputs: ce/dc on the GPU's own u (oracle
    recomputes from the same u), dc~/dv~ on identical dc, xnew on identical
    x, and the GPU's OC against the oracle's literal bisection."""
    p, f, fx, pas = _problem(*case, filter_mode=mode)
    dims = (p["nelx"], p["nely"], p["nelz"])
    n_el = int(np.prod(dims))
    KE = oracle.element_stiffness(p["nu"])
    edof = oracle.edof_matrix(*dims)
    H, Hs = oracle.filter_matrix(*dims, p["rmin"])
    x = _xfield(n_el, pas, seed=3, hi=0.6)      # mean ~0.3: the volume target is reachable
    with topo.Problem(p, f, fx, pas) as pr:
        pr.set_density(x)
        u, info = pr.solve()
        c, ce, dc = pr.sensitivity()
        dcf = pr.filter("dc")
        dvf = pr.get("dvf")
        hs = pr.get("hs")
        xnew, lam, chg, vol = pr.oc_step()
        xphys = pr.get("xphys")
    xphys0 = x
    ce_o = oracle.element_energies(u, KE, edof)
    E_o, c_o, dc_o, dv_o = oracle.sensitivities(xphys0, ce_o, p["penal"], p["E0"], p["Emin"], pas)
    assert_rel(ce, ce_o, 1e-9, "ce")
    assert_rel(dc, dc_o, 1e-9, "dc")
    assert c == pytest.approx(c_o, rel=1e-9)     # north_star 1e-9 (ce); WHT vs dense quadratic form
    assert_rel(hs, Hs, 1e-14, "Hs")
    dcf_o = oracle.apply_filter(H, Hs, mode, "dc", dc, x=x, passive=pas)
    dvf_o = oracle.apply_filter(H, Hs, mode, "dv", dv_o, x=x, passive=pas)
    assert_rel(dcf, dcf_o, 1e-9, "dc~")
    assert_rel(dvf, dvf_o, 1e-13, "dv~")
    trace = []
    xn_o, lam_o, V_o, npass = oracle.oc_update(x, dcf_o, dvf_o, p["volfrac"], p["move"], p["oc_tol"],
                                               p["oc_lmax"], mode, H, Hs, pas, trace=trace)
    assert lam == pytest.approx(lam_o, rel=1e-8)
    assert_rel(xnew, xn_o, 1e-9, "xnew")
    D = np.ones(n_el, bool) if pas is None else pas == 0
    assert chg == pytest.approx(np.max(np.abs(xn_o - x)[D]), rel=1e-9, abs=1e-12)
    xp_o = oracle.apply_filter(H, Hs, mode, "x", xn_o, passive=pas)
    assert_rel(xphys, xp_o, 1e-9, "xPhys")
    assert abs(vol - np.mean(xp_o[D])) <= 1e-9
    assert abs(vol - p["volfrac"]) <= 1e-6
    if pas is not None:
        assert np.all(xnew[pas != 0] == 0) and np.all(xphys[pas != 0] == 0)


@pytest.mark.parametrize("cfg,n_iter", [(0, 20), (1, 10)])
@pytest.mark.parametrize("mode", [0, 1])
def test_loop_parity_configs(topo, cfg, n_iter, mode):
    """BASELINE configs 0/1 with the north_star Jacobi-PCG: c history (fixed
    n_iter) within 1e-6 relative, volume within 1e-6, final design within 1e-6.
    (The multigrid variant: tests/test_gpu_mg.py.)"""
    p, f, fx, pas = make_problem(cfg, filter_mode=mode, precond="jacobi")
    ro = oracle.run_optimization(p, f, fx, pas, n_iter=n_iter)
    with topo.Problem(p, f, fx, pas) as pr:
        c, x, nd = pr.optimize(n_iter)
        xphys = pr.get("xphys")
        t = pr.timings()
    assert nd == n_iter
    assert_rel(c, ro["c"], 1e-6, "c history")
    assert_rel(xphys, ro["xPhys"], 1e-6, "final xPhys")
    assert abs(t["volume"] - p["volfrac"]) <= 1e-6
    assert t["kernel_launches"] > 0


def test_loop_parity_obstacle(topo):
    """Scaled config 2 (cylinder obstacle, rmin 2.5, volfrac 0.2): 10 iterations."""
    dims, obst = (48, 16, 8), (24.0, 8.0, 3.2)
    p = config_params(dict(nelx=48, nely=16, nelz=8, volfrac=0.2, rmin=2.5, n_iter=10,
                           cg_rtol=1e-10, obstacle=obst))
    f, fx = cantilever_load(*dims), cantilever_fixed(*dims)
    pas = cylinder_passive(*dims, *obst)
    ro = oracle.run_optimization(p, f, fx, pas, n_iter=10)
    with topo.Problem(p, f, fx, pas) as pr:
        c, x, nd = pr.optimize(10)
        xphys = pr.get("xphys")
    assert_rel(c, ro["c"], 1e-6, "c history")
    assert_rel(xphys, ro["xPhys"], 1e-6, "xPhys")
    assert np.all(xphys[pas != 0] == 0)


@pytest.mark.parametrize("W", [2, 3, 4])
def test_loopback_slabs_match_single(topo, W):
    """x-slab decomposition (W slabs on one GPU, in-process halo copies):
    identical problem, results equal W = 1 to rounding, and the oracle."""
    dims, obst = (37, 13, 5), (18.0, 6.0, 3.0)
    p, f, fx, pas = _problem(dims, 2.5, obst, precond="jacobi")
    x0 = _xfield(int(np.prod(dims)), pas, seed=5)
    pv = random_vector(3 * 38 * 14 * 6, seed=1)
    outs = []
    for mode, world in ((topo.TOPO_DIST_SINGLE, 1), (topo.TOPO_DIST_LOOPBACK, W)):
        with topo.Problem(p, f, fx, pas, dist=dict(mode=mode, rank=0, world=world, device=0)) as pr:
            pr.set_xphys(x0)
            pr.update_modulus()
            q = pr.apply_K(pv)
            pr.set_density(x0)
            c, x, nd = pr.optimize(5)
            outs.append((q, c, x, pr.get("xphys"), pr.get("u")))
    (q1, c1, x1, xp1, u1), (qW, cW, xW, xpW, uW) = outs
    assert_rel(qW, q1, 1e-14, "matvec W")
    assert_rel(cW, c1, 1e-9, "c hist W")
    assert_rel(xpW, xp1, 1e-8, "xPhys W")
    assert_rel(uW, u1, 1e-7, "u W")
    ro = oracle.run_optimization(p, f, fx, pas, n_iter=5, x0=x0)
    assert_rel(cW, ro["c"], 1e-6, "c hist vs oracle")


def test_zero_load_and_errors(topo):
    p, f, fx, pas = make_problem(0)
    with topo.Problem(p, 0 * f, fx) as pr:
        u, info = pr.solve()
        assert not np.any(u)
        assert info["iters"] == 0
    with topo.Problem(p, f, fx) as pr:
        with pytest.raises(topo.TopoError) as e:
            pr.oc_step()
        assert e.value.code == topo.TOPO_ESTATE
        with pytest.raises(topo.TopoError) as e:
            pr.sensitivity()
        assert e.value.code == topo.TOPO_ESTATE
    for pc, mx in (("jacobi", 5), ("mg", 1)):
        with topo.Problem(dict(p, cg_max_iter=mx, precond=pc), f, fx) as pr:
            with pytest.raises(topo.TopoError) as e:
                pr.solve()
            assert e.value.code == topo.TOPO_ENOCONV


def test_single_element_and_tiny(topo):
    """Degenerate grids: 1x1x1 (one element) and 2x1x1."""
    for dims in ((1, 1, 1), (2, 1, 1), (3, 1, 1)):
        p = config_params(dict(nelx=dims[0], nely=dims[1], nelz=dims[2], volfrac=0.5, rmin=1.5,
                               n_iter=3, cg_rtol=1e-10, obstacle=None))
        f, fx = cantilever_load(*dims), cantilever_fixed(*dims)
        ro = oracle.run_optimization(p, f, fx, None, n_iter=3)
        with topo.Problem(p, f, fx) as pr:
            c, x, nd = pr.optimize(3)
        assert_rel(c, ro["c"], 1e-6, f"c {dims}")


def test_snapshot_restore_bitwise_determinism(topo):
    """S:446 determinism: replaying the same SIMP iterations from a device
    snapshot gives bit-identical compliance histories and designs (all
    reductions are fixed-order)."""
    p, f, fx, pas = make_problem(1)
    with topo.Problem(p, f, fx, pas) as pr:
        pr.optimize(3)
        pr.snapshot()
        c1, x1, _ = pr.optimize(4)
        pr.restore()
        c2, x2, _ = pr.optimize(4)
    assert np.array_equal(c1, c2) and np.array_equal(x1, x2)


def test_paper_protocol_parity(topo):
    """The paper's own benchmark protocol (32x16x16, rmin 4 -> 251-point
    stencil, point load, sensitivity filter): first 5 iterations vs oracle."""
    p, f, fx, pas = make_problem("paper")
    ro = oracle.run_optimization(p, f, fx, pas, n_iter=5)
    with topo.Problem(p, f, fx, pas) as pr:
        c, x, nd = pr.optimize(5)
        xphys = pr.get("xphys")
        assert pr.count("stencil") == 251
    assert_rel(c, ro["c"], 1e-6, "c history (paper protocol)")
    assert_rel(xphys, ro["xPhys"], 1e-6, "xPhys (paper protocol)")
