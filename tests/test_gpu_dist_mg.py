"""Distributed multigrid levels on x-slabs (reading
M10): levels 1 .. k are cycled on each slab's OWNED node planes (ghost planes
exchanged, the K-cycle's dots allreduced, the restriction into the first
replicated level all-gathered plane-wise); below them the levels stay
replicated.  W in-process slabs (loopback: the halo and gather paths of the
NCCL transport as device copies) must give the single-slab V-cycle, solve and
SIMP history up to rounding (partition-dependent summation order of the dots).

TOPO_DIST_MIN_NODES=0 distributes every eligible level on these small grids
(the default distributes levels of > 150k nodes: levels 1-2 at config 4);
TOPO_DEEP_NODES=0 runs every stored level through the large-level kernels
(Jacobi + stencil apply) instead of the fused warp-split sweeps."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from workloads import config_params, cantilever_load, cantilever_fixed, cylinder_passive, random_density, \
    random_vector  # noqa: E402


@pytest.fixture(scope="module")
def topo():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_05604_b200 import topo as t
    return t


def assert_rel(a, b, tol, what=""):
    a, b = np.asarray(a, float), np.asarray(b, float)
    r2 = np.linalg.norm(a - b) / np.linalg.norm(b)
    rm = np.max(np.abs(a - b)) / np.max(np.abs(b))
    assert r2 <= tol and rm <= tol, f"{what}: relL2={r2:.3e} relmax={rm:.3e} tol={tol:g}"


DIMS, OBST = (128, 32, 16), (64.0, 16.0, 5.0)


def _case(fp32, seed=3):
    p = config_params(dict(nelx=DIMS[0], nely=DIMS[1], nelz=DIMS[2], volfrac=0.2, rmin=1.5, n_iter=4,
                           cg_rtol=1e-10, obstacle=OBST), precond="mg", mg_fp32=fp32, mg_cycle="K")
    f, fx = cantilever_load(*DIMS), cantilever_fixed(*DIMS)
    pas = cylinder_passive(*DIMS, *OBST)
    x = random_density(int(np.prod(DIMS)), seed=seed)
    x[pas != 0] = 0.0
    return p, f, fx, pas, x


def _run(topo, p, f, fx, pas, x, b, mode, world, n_iter=4):
    with topo.Problem(p, f, fx, pas, dist=dict(mode=mode, rank=0, world=world, device=0)) as pr:
        nd = pr.count("mg_dist")
        pr.set_xphys(x)
        z = pr.mg_vcycle(b)
        u, info = pr.solve()
        assert info["precond"] == "mg" and info["true_rel_res"] <= 1e-10
        pr.set_density(None)
        c, xo, _ = pr.optimize(n_iter)
        t = pr.timings()
        assert t["mg_fallbacks"] == 0 and t["mg_promotions"] == 0
    return nd, z, u, info["iters"], c, xo


@pytest.mark.parametrize("W", [2, 4, 8])
@pytest.mark.parametrize("fp32", [0, 1])
@pytest.mark.parametrize("deep_nodes", [None, "0"])
def test_dist_levels_loopback_match_single(topo, monkeypatch, W, fp32, deep_nodes):
    monkeypatch.setenv("TOPO_DIST_MIN_NODES", "0")
    if deep_nodes is not None:
        monkeypatch.setenv("TOPO_DEEP_NODES", deep_nodes)
    p, f, fx, pas, x = _case(fp32)
    b = np.where(fx == 0, random_vector(fx.size, seed=9), 0.0)
    n1, z1, u1, it1, c1, x1 = _run(topo, p, f, fx, pas, x, b, topo.TOPO_DIST_SINGLE, 1)
    nW, zW, uW, itW, cW, xW = _run(topo, p, f, fx, pas, x, b, topo.TOPO_DIST_LOOPBACK, W)
    assert n1 == 0 and nW == 2          # levels 1 and 2 distributed, level 3 (coarsest) replicated
    assert_rel(zW, z1, 1e-5 if fp32 else 1e-11, f"V-cycle W={W}")
    assert abs(itW - it1) <= 1
    assert_rel(uW, u1, 1e-7, f"u W={W}")
    assert_rel(cW, c1, 1e-9, f"c history W={W}")
    assert_rel(xW, x1, 1e-6, f"design W={W}")


def test_dist_levels_default_rule(topo):
    """Without the override only levels of > 150k nodes are distributed (none on
    this grid): the replicated design, level-1 allreduce included, still runs."""
    p, f, fx, pas, x = _case(1)
    with topo.Problem(p, f, fx, pas, dist=dict(mode=topo.TOPO_DIST_LOOPBACK, rank=0, world=2, device=0)) as pr:
        assert pr.count("mg_dist") == 0


def test_dist_levels_partition_rule(topo, monkeypatch):
    """A level is distributed only while every slab boundary sits on an even
    plane of it and each slab owns >= 2 of its element planes: 3 slabs of
    128 / 3 planes -> boundaries 42, 85 (odd) -> replicated."""
    monkeypatch.setenv("TOPO_DIST_MIN_NODES", "0")
    p, f, fx, pas, x = _case(1)
    with topo.Problem(p, f, fx, pas, dist=dict(mode=topo.TOPO_DIST_LOOPBACK, rank=0, world=3, device=0)) as pr:
        assert pr.count("mg_dist") == 0
    monkeypatch.setenv("TOPO_DIST_LEVELS", "1")
    with topo.Problem(p, f, fx, pas, dist=dict(mode=topo.TOPO_DIST_LOOPBACK, rank=0, world=4, device=0)) as pr:
        assert pr.count("mg_dist") == 1


@pytest.mark.parametrize("fp32", [0, 1])
def test_dist_code_path_one_slab(topo, monkeypatch, fp32):
    """TOPO_DIST_FORCE1: the distributed-level code path with ONE slab owning
    every plane (no exchanges) equals the replicated path: V-cycle to rounding
    (the K-cycle dots' summation order) and the solve's iteration count."""
    p, f, fx, pas, x = _case(fp32)
    b = np.where(fx == 0, random_vector(fx.size, seed=9), 0.0)
    n1, z1, u1, it1, c1, x1 = _run(topo, p, f, fx, pas, x, b, topo.TOPO_DIST_SINGLE, 1, n_iter=2)
    monkeypatch.setenv("TOPO_DIST_FORCE1", "1")
    monkeypatch.setenv("TOPO_DIST_MIN_NODES", "0")
    nF, zF, uF, itF, cF, xF = _run(topo, p, f, fx, pas, x, b, topo.TOPO_DIST_SINGLE, 1, n_iter=2)
    assert n1 == 0 and nF == 2
    assert_rel(zF, z1, 1e-6 if fp32 else 1e-12, "V-cycle")
    assert itF == it1
    assert_rel(cF, c1, 1e-10, "c history")


@pytest.mark.parametrize("W,r", [(2, 1), (4, 2)])
def test_solo_timing_mode_runs_fixed_iterations(topo, monkeypatch, W, r):
    """TOPO_DIST_SOLO (tools/solo_scale.py): rank r's slab alone, no transport;
    every solve runs exactly cg_max_iter PCG iterations with no breakdown exit and
    no Jacobi fallback, so the kernel sequence per iteration is the NCCL rank's."""
    monkeypatch.setenv("TOPO_DIST_MIN_NODES", "0")
    p, f, fx, pas, x = _case(1)
    p = dict(p, cg_max_iter=7)
    with topo.Problem(p, f, fx, pas, dist=dict(mode=topo.TOPO_DIST_SOLO, rank=r, world=W, device=0)) as pr:
        assert pr.count("mg_dist") == 2
        lo, hi = pr.owned_range()
        assert (lo, hi) == topo.partition(DIMS[0], p["rmin"], W, r)
        pr.optimize(2, want_x=False)
        t = pr.timings()
        assert t["cg_iters"] == 7 and t["cg_iters_total"] == 14
        assert t["mg_fallbacks"] == 0 and t["mg_promotions"] == 0 and t["mg_theta_cuts"] == 0


@pytest.mark.parametrize("W", [2, 4])
def test_dist_levels_face_layout_loopback(topo, monkeypatch, W):
    """Distributed level 1 with the face layout (forced): each slab writes the face
    sums of its own node planes only; loopback slabs reproduce one slab."""
    monkeypatch.setenv("TOPO_DIST_MIN_NODES", "0")
    monkeypatch.setenv("TOPO_L1_FACE", "1")
    p, f, fx, pas, x = _case(1)
    b = np.where(fx == 0, random_vector(fx.size, seed=9), 0.0)
    n1, z1, u1, it1, c1, x1 = _run(topo, p, f, fx, pas, x, b, topo.TOPO_DIST_SINGLE, 1)
    nW, zW, uW, itW, cW, xW = _run(topo, p, f, fx, pas, x, b, topo.TOPO_DIST_LOOPBACK, W)
    assert nW == 2
    assert_rel(zW, z1, 1e-5, f"V-cycle W={W}")
    assert abs(itW - it1) <= 1
    assert_rel(cW, c1, 1e-9, f"c history W={W}")
