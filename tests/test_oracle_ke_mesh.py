"""Pins for oracle.ke and oracle.mesh against closed forms and brute force
(not against the oracle itself).  SURVEY §8(c) "What pins each part"."""
import json
import os

import numpy as np
import pytest

from oracle import element_stiffness, lame, edof_matrix, edof_matrix_loops, element_centroids
from oracle.mesh import LOCAL_NODES

NUS = [0.0, 0.2, 0.3, 0.45]


def _field(fn):
    """Nodal vector [24] of a displacement field u(x,y,z) at the local nodes."""
    v = np.zeros(24)
    for a, (x, y, z) in enumerate(LOCAL_NODES):
        v[3 * a:3 * a + 3] = fn(float(x), float(y), float(z))
    return v


@pytest.mark.parametrize("nu", NUS)
def test_ke_symmetric_psd_six_rigid_modes(nu):
    KE = element_stiffness(nu)
    assert np.max(np.abs(KE - KE.T)) < 1e-14
    w = np.linalg.eigvalsh(KE)
    zero = np.abs(w) <= 1e-8 * w.max()
    assert zero.sum() == 6                    # S:94 exactly 6 rigid-body modes
    assert np.all(w[~zero] > 0)


@pytest.mark.parametrize("nu", NUS)
def test_ke_rigid_body_nullspace(nu):
    KE = element_stiffness(nu)
    modes = [lambda x, y, z: (1, 0, 0), lambda x, y, z: (0, 1, 0), lambda x, y, z: (0, 0, 1),
             lambda x, y, z: (-y, x, 0), lambda x, y, z: (0, -z, y), lambda x, y, z: (z, 0, -x)]
    for m in modes:
        assert np.max(np.abs(KE @ _field(m))) < 1e-14


@pytest.mark.parametrize("nu", NUS)
def test_ke_uniform_strain_energies_closed_form(nu):
    """u^T KE u = eps:D:eps on the unit cube (trilinear elements reproduce
    linear fields exactly)."""
    KE = element_stiffness(nu)
    lam, mu = lame(1.0, nu)
    e1 = _field(lambda x, y, z: (x, 0, 0))
    assert e1 @ KE @ e1 == pytest.approx(lam + 2 * mu, rel=1e-13)
    e2 = _field(lambda x, y, z: (y, 0, 0))
    assert e2 @ KE @ e2 == pytest.approx(mu, rel=1e-13)
    e3 = _field(lambda x, y, z: (x, -nu * y, -nu * z))           # uniaxial stress
    assert e3 @ KE @ e3 == pytest.approx(1.0, rel=1e-13)          # = E


@pytest.mark.parametrize("nu", NUS)
def test_ke_diagonal_closed_form(nu):
    """KE_ii = (lambda+2mu)/9 + 2 mu/9 = (lambda+4mu)/9 for every DOF."""
    lam, mu = lame(1.0, nu)
    assert np.allclose(np.diag(element_stiffness(nu)), (lam + 4 * mu) / 9.0, rtol=1e-14, atol=0)


@pytest.mark.parametrize("nu", NUS)
def test_ke_linear_eigenmodes_closed_form(nu):
    """Hydrostatic mode: eigenvalue (3 lambda + 2 mu)/2; pure and normal-deviatoric
    shear modes: eigenvalue mu (consistent nodal forces of a uniform stress)."""
    KE = element_stiffness(nu)
    lam, mu = lame(1.0, nu)
    h = _field(lambda x, y, z: (x - .5, y - .5, z - .5))
    assert np.allclose(KE @ h, (3 * lam + 2 * mu) / 2 * h, atol=1e-14)
    s = _field(lambda x, y, z: (y - .5, x - .5, 0))
    assert np.allclose(KE @ s, mu * s, atol=1e-14)
    d = _field(lambda x, y, z: (x - .5, -(y - .5), 0))
    assert np.allclose(KE @ d, mu * d, atol=1e-14)


def test_mesh_counts_paper_grid(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "paper_mesh_counts.json")))
    nelx, nely, nelz = g["nelx"], g["nely"], g["nelz"]
    edof = edof_matrix(nelx, nely, nelz)
    assert edof.shape[0] == g["n_el"]
    assert len(np.unique(edof[:, 0::3])) == g["n_nodes"]
    assert edof.max() + 1 == g["n_dofs"]
    from workloads import cantilever_fixed
    assert int(cantilever_fixed(nelx, nely, nelz).sum()) == g["fixed_dofs_left_face"]


@pytest.mark.parametrize("dims", [(1, 1, 1), (2, 1, 1), (3, 2, 4), (5, 3, 2)])
def test_edof_vectorised_equals_loops(dims):
    assert np.array_equal(edof_matrix(*dims), edof_matrix_loops(*dims))


def test_edof_face_sharing():
    edof = edof_matrix(2, 1, 1)
    assert len(set(edof[0]) & set(edof[1])) == 12
    assert edof_matrix(1, 1, 1).shape == (1, 24) and sorted(edof_matrix(1, 1, 1)[0]) == list(range(24))


def test_centroids():
    c = element_centroids(3, 3, 3)
    assert np.allclose(c[13], (1.5, 1.5, 1.5))
    c2 = element_centroids(2, 1, 1)
    assert np.isclose(np.linalg.norm(c2[0] - c2[1]), 1.0)
