"""Pins for oracle.loop: volume constraint each iteration, compliance descent,
z-mirror symmetry, passive integrity, energy identity.  SURVEY §8(c); SPEC
S:295-304."""
import numpy as np
import pytest

from oracle import run_optimization
from workloads import make_problem, config_params, cantilever_load, cantilever_fixed, cylinder_passive


def _zmirror(v, nelx, nely, nelz):
    return v.reshape(nelz, nelx, nely)[::-1].ravel()


@pytest.mark.parametrize("mode", [0, 1])
def test_config0_loop_invariants(mode):
    p, f, fixed, passive = make_problem(0, filter_mode=mode)
    r = run_optimization(p, f, fixed, passive, n_iter=20)
    c = r["c"]
    assert np.allclose(r["c"], r["fu"], rtol=1e-8)              # c = sum E ce = f^T u
    assert c[-1] < c[0]
    assert np.all(np.diff(c[1:]) < 0) or np.mean(np.diff(c[1:]) < 0) >= 0.9
    assert np.all(np.abs(r["vol"] - 0.3) <= 1e-6)               # north_star: volume to 1e-6
    assert np.all(r["change"] <= 0.2 + 1e-15)
    xp = r["xPhys"]
    assert np.max(np.abs(xp - _zmirror(xp, 30, 10, 2))) <= 1e-6   # S:304 (z-symmetric problem)


def test_obstacle_loop_passive_integrity():
    """Small cylinder-obstacle cantilever: passive elements stay 0, volume over D."""
    p = config_params(dict(nelx=24, nely=8, nelz=4, volfrac=0.2, rmin=1.5, n_iter=6,
                           cg_rtol=1e-10, obstacle=(12.0, 4.0, 2.0)))
    nelx, nely, nelz = 24, 8, 4
    f, fixed = cantilever_load(nelx, nely, nelz), cantilever_fixed(nelx, nely, nelz)
    passive = cylinder_passive(nelx, nely, nelz, 12.0, 4.0, 2.0)
    assert passive.sum() == 4 * 12
    for mode in (0, 1):
        p["filter_mode"] = mode
        r = run_optimization(p, f, fixed, passive, n_iter=6, record=True)
        for rec in r["records"]:
            assert np.all(rec["xPhys"][passive != 0] == 0)
            assert np.all(rec["xnew"][passive != 0] == 0)
            assert np.all(rec["dc"][passive != 0] == 0)
        assert np.all(np.abs(r["vol"] - 0.2) <= 1e-6)
        xp = r["xPhys"]
        assert np.max(np.abs(xp - _zmirror(xp, nelx, nely, nelz))) <= 1e-6


def test_config2_obstacle_count():
    """Reading #23: 208 passive elements per z-layer, 4160 in total."""
    from workloads import CONFIGS
    c = CONFIGS[2]
    pas = cylinder_passive(c["nelx"], c["nely"], c["nelz"], *c["obstacle"])
    assert pas.sum() == 4160
    assert pas.reshape(20, 120, 40)[0].sum() == 208
