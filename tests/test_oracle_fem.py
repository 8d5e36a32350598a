"""Pins for oracle.fem: patch test (closed form), brute-force dense solve,
energy identity, linearity, closed-form diagonal.  SURVEY §8(c)."""
import numpy as np
import pytest

from oracle import (element_stiffness, edof_matrix, assemble, solve_direct, solve_jacobi_cg,
                    element_energies, matvec_free, matvec_elementwise, true_residual)
from oracle.mesh import LOCAL_NODES
from workloads import (roller_patch_problem, cantilever_load, cantilever_fixed, random_density,
                       random_vector, n_nodes, node_id)

NU = 0.3


@pytest.mark.parametrize("dims", [(4, 3, 2), (3, 1, 1), (2, 2, 2)])
@pytest.mark.parametrize("method", ["direct", "cg"])
def test_roller_patch_test_exact(dims, method):
    """Uniaxial stress under consistent traction: u = (x, -nu y, -nu z) exactly,
    c = nelx*nely*nelz (traction 1 on a nely*nelz face, end displacement nelx)."""
    nelx, nely, nelz = dims
    f, fixed = roller_patch_problem(nelx, nely, nelz)
    KE = element_stiffness(NU)
    K = assemble(nelx, nely, nelz, KE, np.ones(nelx * nely * nelz))
    u = solve_direct(K, f, fixed) if method == "direct" else solve_jacobi_cg(K, f, fixed, rtol=1e-14)[0]
    exact = np.zeros_like(u)
    for iz in range(nelz + 1):
        for ix in range(nelx + 1):
            for iy in range(nely + 1):
                n = node_id(nelx, nely, nelz, ix, iy, iz)
                exact[3 * n:3 * n + 3] = (ix, -NU * iy, -NU * iz)
    assert np.max(np.abs(u - exact)) < 1e-10
    assert f @ u == pytest.approx(nelx * nely * nelz, rel=1e-12)


def _dense_bruteforce(nelx, nely, nelz, KE, E):
    """Dense K by explicit loops over elements and local entries."""
    nn = n_nodes(nelx, nely, nelz)
    K = np.zeros((3 * nn, 3 * nn))
    e = 0
    for ez in range(nelz):
        for ex in range(nelx):
            for ey in range(nely):
                dofs = []
                for (dx, dy, dz) in LOCAL_NODES:
                    n = node_id(nelx, nely, nelz, ex + dx, ey + dy, ez + dz)
                    dofs += [3 * n, 3 * n + 1, 3 * n + 2]
                for a in range(24):
                    for b in range(24):
                        K[dofs[a], dofs[b]] += E[e] * KE[a, b]
                e += 1
    return K


def test_bruteforce_dense_2x2x2():
    """north_star: brute-force dense solve on a 2x2x2 mesh (81 DOF; the x = 0 face
    fixes 9 nodes = 27 DOF, so 54 are free -- SURVEY §8(c) says 72, a slip)."""
    nelx = nely = nelz = 2
    KE = element_stiffness(NU)
    E = 1e-9 + random_density(8, seed=3) ** 3 * (1 - 1e-9)
    Kd = _dense_bruteforce(nelx, nely, nelz, KE, E)
    Ks = assemble(nelx, nely, nelz, KE, E)
    assert np.max(np.abs(Ks.toarray() - Kd)) < 1e-12
    f = cantilever_load(nelx, nely, nelz)
    fixed = cantilever_fixed(nelx, nely, nelz)
    free = fixed == 0
    assert free.sum() == 54
    ud = np.zeros(81)
    ud[free] = np.linalg.solve(Kd[np.ix_(free, free)], f[free])
    us = solve_direct(Ks, f, fixed)
    assert np.max(np.abs(us - ud)) <= 1e-12 * np.max(np.abs(ud))
    uc = solve_jacobi_cg(Ks, f, fixed, rtol=1e-13)[0]
    assert np.linalg.norm(uc - ud) <= 1e-8 * np.linalg.norm(ud)


def test_zero_load_and_quadratic_scaling():
    nelx, nely, nelz = 4, 2, 2
    KE = element_stiffness(NU)
    K = assemble(nelx, nely, nelz, KE, np.full(16, 0.5 ** 3))
    fixed = cantilever_fixed(nelx, nely, nelz)
    f = cantilever_load(nelx, nely, nelz)
    assert not np.any(solve_direct(K, 0 * f, fixed))
    c1 = f @ solve_direct(K, f, fixed)
    c2 = (2 * f) @ solve_direct(K, 2 * f, fixed)
    assert c2 == pytest.approx(4 * c1, rel=1e-12)


@pytest.mark.parametrize("dims", [(6, 3, 2), (5, 4, 3)])
def test_energy_identity(dims):
    """c = f^T u = sum_e E_e u_e^T KE u_e (north_star)."""
    nelx, nely, nelz = dims
    n_el = nelx * nely * nelz
    KE = element_stiffness(NU)
    E = 1e-9 + random_density(n_el, seed=5) ** 3
    K = assemble(nelx, nely, nelz, KE, E)
    f, fixed = cantilever_load(*dims), cantilever_fixed(*dims)
    u = solve_direct(K, f, fixed)
    ce = element_energies(u, KE, edof_matrix(*dims))
    assert np.sum(E * ce) == pytest.approx(f @ u, rel=1e-10)
    assert np.all(ce >= -1e-18)


def test_diagonal_closed_form():
    """diag(K)_n = (lambda+4mu)/9 * sum_{e ni n} E_e for all 3 components."""
    nelx, nely, nelz = 4, 3, 2
    n_el = nelx * nely * nelz
    KE = element_stiffness(NU)
    E = random_density(n_el, seed=7)
    d = assemble(nelx, nely, nelz, KE, E).diagonal()
    lam, mu = 0.3 / (1.3 * 0.4), 1 / 2.6
    kd = (lam + 4 * mu) / 9
    for iz in range(nelz + 1):
        for ix in range(nelx + 1):
            for iy in range(nely + 1):
                s = 0.0
                for ez in (iz - 1, iz):
                    for ex in (ix - 1, ix):
                        for ey in (iy - 1, iy):
                            if 0 <= ex < nelx and 0 <= ey < nely and 0 <= ez < nelz:
                                s += E[ez * nelx * nely + ex * nely + ey]
                n = node_id(nelx, nely, nelz, ix, iy, iz)
                assert np.allclose(d[3 * n:3 * n + 3], kd * s, rtol=1e-13)


def test_matvec_elementwise_equals_csr():
    dims = (7, 4, 3)
    n_el = 7 * 4 * 3
    KE = element_stiffness(NU)
    E = random_density(n_el, seed=2)
    K = assemble(*dims, KE, E)
    fixed = cantilever_fixed(*dims)
    p = random_vector(K.shape[0], seed=1)
    q1 = matvec_free(K, p, fixed)
    q2 = matvec_elementwise(*dims, KE, E, p, fixed, chunk=17)
    assert np.linalg.norm(q1 - q2) <= 1e-14 * np.linalg.norm(q1)
    assert not np.any(q1[fixed != 0])


def test_monotone_in_density():
    """Adding material never increases compliance."""
    dims = (6, 2, 2)
    n_el = 24
    KE = element_stiffness(NU)
    f, fixed = cantilever_load(*dims), cantilever_fixed(*dims)
    x = random_density(n_el, seed=11)
    c0 = f @ solve_direct(assemble(*dims, KE, 1e-9 + x ** 3), f, fixed)
    x2 = x.copy()
    x2[5] = min(1.0, x2[5] + 0.3)
    c1 = f @ solve_direct(assemble(*dims, KE, 1e-9 + x2 ** 3), f, fixed)
    assert c1 <= c0


def test_true_residual_of_direct_solve():
    dims = (8, 4, 2)
    KE = element_stiffness(NU)
    E = 1e-9 + random_density(64, seed=4) ** 3
    K = assemble(*dims, KE, E)
    f, fixed = cantilever_load(*dims), cantilever_fixed(*dims)
    assert true_residual(K, solve_direct(K, f, fixed), f, fixed) < 1e-10


def test_matvec_rows_equals_csr():
    dims = (6, 5, 4)
    KE = element_stiffness(NU)
    E = random_density(120, seed=8)
    K = assemble(*dims, KE, E)
    fixed = cantilever_fixed(*dims)
    p = random_vector(K.shape[0], seed=2)
    q = matvec_free(K, p, fixed)
    from oracle import matvec_rows
    nodes = np.arange(0, K.shape[0] // 3, 7)
    assert np.allclose(matvec_rows(*dims, KE, E, p, fixed, nodes), q.reshape(-1, 3)[nodes], rtol=0, atol=1e-14)


def test_element_energies_strain_form():
    """The strain form of ce (sum_gp eps^T D eps / 8) equals u_e^T KE u_e, and a
    rigid translation has zero energy in it to rounding (closed form)."""
    import oracle
    from oracle import element_energies_strain
    KE = oracle.element_stiffness(0.3)
    rng = np.random.default_rng(8)
    ue = rng.standard_normal((500, 24))
    ce1 = np.einsum("ei,ij,ej->e", ue, KE, ue)
    ce2 = element_energies_strain(ue, 0.3)
    assert np.allclose(ce2, ce1, rtol=1e-12, atol=0)
    t = np.tile([3.7, -1.1, 250.0], 8)[None, :]
    assert element_energies_strain(t, 0.3)[0] <= 1e-30 * float(t @ t.T)      # zero up to rounding
    # uniform strain u = (x, 0, 0): energy lambda + 2 mu (closed form, unit cube)
    from oracle.mesh import LOCAL_NODES
    lam, mu = oracle.lame(1.0, 0.3)
    u = np.zeros((1, 24))
    for a, (ax, ay, az) in enumerate(LOCAL_NODES):
        u[0, 3 * a] = ax
    assert element_energies_strain(u, 0.3)[0] == pytest.approx(lam + 2 * mu, rel=1e-14)
