"""GPU parity at BASELINE.json's full sizes (configs 2, 3, 4), in the launch
configuration bench.py times (same library, same kernels, same grids).  The
oracle computes sampled outputs one by one (matvec rows, residual rows, ce,
filter rows, OC xnew at the GPU's lambda) on the GPU's own inputs, plus
properties that hold at any size (true residual, energy identity, volume).
Config 2 is small enough for the oracle's full per-component pipeline."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from workloads import make_problem, random_vector  # noqa: E402
import oracle  # noqa: E402
from oracle.mesh import LOCAL_NODES  # noqa: E402


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


def sample_nodes(nelx, nely, nelz, n, seed=0):
    rng = np.random.default_rng(seed)
    ix = np.concatenate([rng.integers(0, nelx + 1, n), [0, 1, nelx - 1, nelx, nelx, nelx // 2]])
    iy = np.concatenate([rng.integers(0, nely + 1, n), [0, nely, 0, nely, 0, nely]])
    iz = np.concatenate([rng.integers(0, nelz + 1, n), [0, nelz, nelz, 0, nelz // 2, nelz]])
    return iz * (nelx + 1) * (nely + 1) + ix * (nely + 1) + iy


def sample_elems(nelx, nely, nelz, n, seed=0):
    rng = np.random.default_rng(seed)
    ex = np.concatenate([rng.integers(0, nelx, n), [0, nelx - 1, 0, nelx - 1, nelx // 2]])
    ey = np.concatenate([rng.integers(0, nely, n), [0, nely - 1, nely - 1, 0, 0]])
    ez = np.concatenate([rng.integers(0, nelz, n), [0, nelz - 1, 0, nelz - 1, nelz - 1]])
    return ez * nelx * nely + ex * nely + ey


def edof_rows(nelx, nely, nelz, elems):
    nxy = (nelx + 1) * (nely + 1)
    ez, rem = np.divmod(elems, nelx * nely)
    ex, ey = np.divmod(rem, nely)
    cols = []
    for (dx, dy, dz) in LOCAL_NODES:
        n = (ez + dz) * nxy + (ex + dx) * (nely + 1) + (ey + dy)
        cols += [3 * n, 3 * n + 1, 3 * n + 2]
    return np.stack(cols, axis=1)


@pytest.mark.parametrize("cfg", [3, 4])
def test_fullsize_sampled(topo, cfg):
    p, f, fx, pas = make_problem(cfg)
    nelx, nely, nelz = p["nelx"], p["nely"], p["nelz"]
    n_el = nelx * nely * nelz
    n_nd = (nelx + 1) * (nely + 1) * (nelz + 1)
    KE = oracle.element_stiffness(p["nu"])
    nodes = sample_nodes(nelx, nely, nelz, 400)
    elems = sample_elems(nelx, nely, nelz, 300)
    with topo.Problem(p, f, fx, pas) as pr:
        # --- A1/A2: modulus and matvec rows on a random p (x = volfrac) ---
        pr.update_modulus()
        E = pr.get("E")
        x0 = np.full(n_el, p["volfrac"])
        assert_rel(E, p["Emin"] + x0 ** p["penal"] * (p["E0"] - p["Emin"]), 1e-15, "E")
        pv = random_vector(3 * n_nd, seed=1)
        q = pr.apply_K(pv)
        qo = oracle.matvec_rows(nelx, nely, nelz, KE, E, pv, fx, nodes)
        assert_rel(q.reshape(-1, 3)[nodes], qo, 1e-13, "matvec rows")
        del q
        # --- A4: solve; true residual (GPU) and sampled residual rows (oracle) ---
        u, info = pr.solve()
        tol = p["cg_rtol"]
        assert info["true_rel_res"] <= tol
        r_rows = f.reshape(-1, 3)[nodes] - oracle.matvec_rows(nelx, nely, nelz, KE, E, u, fx, nodes)
        assert np.linalg.norm(r_rows) <= tol * np.linalg.norm(f)
        # --- A5: ce, dc on the GPU's u; energy identity ---
        c, ce, dc = pr.sensitivity()
        ue = u[edof_rows(nelx, nely, nelz, elems)]
        ce_o = np.einsum("ei,ij,ej->e", ue, KE, ue)
        assert_rel(ce[elems], ce_o, 1e-9, "ce sampled")
        dc_o = -p["penal"] * x0[elems] ** (p["penal"] - 1) * (p["E0"] - p["Emin"]) * ce_o
        assert_rel(dc[elems], dc_o, 1e-9, "dc sampled")
        fu = float(f @ u)
        assert abs(c - fu) <= np.linalg.norm(u) * tol * np.linalg.norm(f) * 1.01 + 1e-12 * abs(fu)
        # --- A6: filter rows (density filter) on the GPU's dc ---
        dcf = pr.filter("dc")
        hs = pr.get("hs")
        rows, hs_o = oracle.filter_rows(nelx, nely, nelz, p["rmin"], elems[:60])
        assert_rel(hs[elems[:60]], hs_o, 1e-14, "Hs rows")
        dcf_o = []
        for (cols, w) in rows:
            _, hs_cols = oracle.filter_rows(nelx, nely, nelz, p["rmin"], cols)
            dcf_o.append(np.sum(w * dc[cols] / hs_cols))
        assert_rel(dcf[elems[:60]], dcf_o, 1e-9, "dc~ rows")
        dvf = pr.get("dvf")
        x_before = pr.get("x")
        # --- A7: OC at the GPU's lambda, pointwise; volume property ---
        xnew, lam, chg, vol = pr.oc_step()
        xo = oracle.oc_xnew(x_before[elems], dcf[elems], dvf[elems], lam, p["move"])
        assert_rel(xnew[elems], xo, 1e-9, "xnew sampled")
        assert abs(vol - p["volfrac"]) <= 1e-6
        assert np.all((xnew >= 0) & (xnew <= 1))
        assert chg <= p["move"] + 1e-15


def test_fullsize_config2(topo):
    """Config 2 (obstacle, rmin 2.5): per-component parity of one SIMP
    iteration; the oracle solves with Jacobi-CG to a true residual of 1e-12."""
    p, f, fx, pas = make_problem(2)
    nelx, nely, nelz = p["nelx"], p["nely"], p["nelz"]
    KE = oracle.element_stiffness(p["nu"])
    D = pas == 0
    x0 = np.where(D, p["volfrac"], 0.0)
    E_o = p["Emin"] + x0 ** p["penal"] * (p["E0"] - p["Emin"])
    K = oracle.assemble(nelx, nely, nelz, KE, E_o)
    H, Hs = oracle.filter_matrix(nelx, nely, nelz, p["rmin"])
    with topo.Problem(p, f, fx, pas) as pr:
        u, info = pr.solve()
        c, ce, dc = pr.sensitivity()
        dcf = pr.filter("dc")
        dvf = pr.get("dvf")
        xnew, lam, chg, vol = pr.oc_step()
        xphys = pr.get("xphys")
    assert oracle.true_residual(K, u, f, fx) <= 1e-10
    uo, _ = oracle.solve_jacobi_cg(K, f, fx, rtol=1e-12)
    assert np.linalg.norm(u - uo) <= 1e-8 * np.linalg.norm(uo)
    edof = oracle.edof_matrix(nelx, nely, nelz)
    ce_o = oracle.element_energies(u, KE, edof)
    _, c_o, dc_o, dv_o = oracle.sensitivities(x0, ce_o, p["penal"], p["E0"], p["Emin"], pas)
    assert_rel(ce, ce_o, 1e-9, "ce")
    assert_rel(dc, dc_o, 1e-9, "dc")
    assert c == pytest.approx(c_o, rel=1e-9)     # north_star 1e-9 (ce); WHT vs dense quadratic form
    dcf_o = oracle.apply_filter(H, Hs, 0, "dc", dc)
    dvf_o = oracle.apply_filter(H, Hs, 0, "dv", dv_o)
    assert_rel(dcf, dcf_o, 1e-9, "dc~")
    assert_rel(dvf, dvf_o, 1e-13, "dv~")
    xn_o, lam_o, V_o, npass = oracle.oc_update(x0, dcf_o, dvf_o, p["volfrac"], p["move"], p["oc_tol"],
                                               p["oc_lmax"], 0, H, Hs, pas)
    assert lam == pytest.approx(lam_o, rel=1e-8)
    assert_rel(xnew, xn_o, 1e-9, "xnew")
    assert_rel(xphys, oracle.apply_filter(H, Hs, 0, "x", xn_o, passive=pas), 1e-9, "xPhys")
    assert abs(vol - p["volfrac"]) <= 1e-6
    assert np.all(xnew[~D] == 0) and np.all(xphys[~D] == 0)


def test_config2_history_vs_oracle_golden(topo, golden_dir):
    """Config 2 at full size, all 30 BASELINE iterations, against the oracle's
    own run (tests/golden/cfg2_oracle_history.npz, written by
    tools/make_golden_cfg2.py from oracle/ only): c history within 1e-6
    relative, x / xPhys after iterations 10 and 30 within 1e-6 (R#25 metric),
    volume within 1e-6 every iteration."""
    import os
    g = np.load(os.path.join(golden_dir, "cfg2_oracle_history.npz"))
    p, f, fx, pas = make_problem(2)
    with topo.Problem(p, f, fx, pas) as pr:
        c10, x10, _ = pr.optimize(10)
        xp10 = pr.get("xphys")
        vols = [pr.timings()["volume"]]
        c20, x30, nd = pr.optimize(20)
        xp30 = pr.get("xphys")
        vols.append(pr.timings()["volume"])
    c = np.concatenate([c10, c20])
    assert nd == 20 and c.size == 30
    assert_rel(c, g["c"], 1e-6, "config-2 c history (30 iterations)")
    assert_rel(c[:10], g["c"][:10], 1e-6, "config-2 c history (first 10)")
    assert_rel(x10, g["x_10"], 1e-6, "x after 10")
    assert_rel(xp10, g["xphys_10"], 1e-6, "xPhys after 10")
    assert_rel(x30, g["x_30"], 1e-6, "x after 30")
    assert_rel(xp30, g["xphys_30"], 1e-6, "xPhys after 30")
    assert all(abs(v - p["volfrac"]) <= 1e-6 for v in vols)
    assert np.all(xp30[pas != 0] == 0)
