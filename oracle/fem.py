"""FEM: assembly, boundary conditions, solve (oracle).  P:42 §2.2.

K = sum_e E_e * scatter(KE, edofMat[e]) (COO triplets -> CSR, duplicates
summed; "COO initially, converted to CSR").  Dirichlet BCs by
elimination: solve K_ff u_f = f_f, u = 0 on fixed DOFs ("modifying the
system matrix and load vector ... avoiding ... penalty methods"; R#8).
"""
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .mesh import edof_matrix


def assemble(nelx, nely, nelz, KE, E, edof=None):
    """Global K (CSR, all DOFs, pre-BC).  SPEC S:127."""
    if edof is None:
        edof = edof_matrix(nelx, nely, nelz)
    n_dof = 3 * (nelx + 1) * (nely + 1) * (nelz + 1)
    iK = np.repeat(edof, 24, axis=1).ravel()          # row index of KE[a,b] -> edof[e,a]
    jK = np.tile(edof, (1, 24)).ravel()               # col index            -> edof[e,b]
    sK = (KE.ravel()[None, :] * np.asarray(E, dtype=np.float64)[:, None]).ravel()
    return sp.coo_matrix((sK, (iK, jK)), shape=(n_dof, n_dof)).tocsr()


def solve_direct(K, f, fixed):
    """u with u_fixed = 0 and K_ff u_f = f_f, by sparse LU (SuperLU).  S:137."""
    free = np.flatnonzero(np.asarray(fixed) == 0)
    u = np.zeros(K.shape[0])
    if not np.any(f[free]):
        return u
    Kff = K[free][:, free].tocsc()
    u[free] = spla.spsolve(Kff, f[free])
    return u


def solve_jacobi_cg(K, f, fixed, rtol=1e-12, max_iter=None, u0=None):
    """Plain Jacobi-preconditioned CG on K_ff, stopping on the TRUE relative
    residual ||f_f - K_ff u_f|| <= rtol ||f_f|| (checked whenever the
    recursive residual passes).  SPEC S:160 (Jacobi-CG contract)."""
    free = np.flatnonzero(np.asarray(fixed) == 0)
    Kff = K[free][:, free].tocsr()
    b = f[free]
    nb = np.linalg.norm(b)
    u = np.zeros(K.shape[0])
    if nb == 0.0:
        return u, 0
    x = np.zeros_like(b) if u0 is None else u0[free].copy()
    Minv = 1.0 / Kff.diagonal()
    r = b - Kff @ x
    z = Minv * r
    p = z.copy()
    rz = r @ z
    max_iter = max_iter or 20 * len(b)
    it = 0
    while it < max_iter:
        if np.linalg.norm(r) <= rtol * nb:
            rt = b - Kff @ x
            if np.linalg.norm(rt) <= rtol * nb:
                break
            r = rt                                  # residual replacement
            z = Minv * r
            p = z.copy()
            rz = r @ z
        q = Kff @ p
        alpha = rz / (p @ q)
        x += alpha * p
        r -= alpha * q
        z = Minv * r
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
        it += 1
    u[free] = x
    return u, it


def solve(K, f, fixed, method="auto", rtol=1e-12):
    """Direct solve when small (configs 0-1), else Jacobi-CG to true residual."""
    n_free = int(np.sum(np.asarray(fixed) == 0))
    if method == "direct" or (method == "auto" and n_free <= 60000):
        return solve_direct(K, f, fixed)
    return solve_jacobi_cg(K, f, fixed, rtol=rtol)[0]


def compliance_fu(f, u):
    """c = F^T U.  SPEC S:147."""
    return float(f @ u)


def element_energies(u, KE, edof):
    """ce_e = u_e^T KE u_e (not E-scaled).  P:47 §2.3."""
    ue = u[edof]                                      # [n_el, 24]
    return np.einsum("ei,ij,ej->e", ue, KE, ue)


def element_energies_strain(ue, nu):
    """ce_e = sum over the 2x2x2 Gauss points of (1/8) eps^T D eps with eps = B u_e
    -- the element strain energy from its definition (§2.3: ce = u_e^T KE u_e,
    KE = sum_gp (1/8) B^T D B, oracle.ke), evaluated through the strains.  Equal
    to element_energies in exact arithmetic; better conditioned when u_e is
    nearly rigid (B annihilates translations exactly: the shape-gradient rows
    cancel pairwise), which is how large displacements with little strain look
    on a cantilever.  ue: [n, 24] element DOF vectors."""
    from .ke import constitutive, strain_displacement
    D = constitutive(1.0, nu)
    pts = (0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0))
    ce = np.zeros(ue.shape[0])
    for xi in pts:
        for eta in pts:
            for zeta in pts:
                eps = ue @ strain_displacement(xi, eta, zeta).T          # [n, 6]
                ce += 0.125 * np.einsum("ei,ij,ej->e", eps, D, eps)
    return ce


def matvec_free(K, p, fixed):
    """q = K p with the Dirichlet mask: q_f = K_ff p_f, q = 0 on fixed DOFs."""
    fx = np.asarray(fixed) != 0
    pm = np.where(fx, 0.0, p)
    q = K @ pm
    q[fx] = 0.0
    return q


def matvec_elementwise(nelx, nely, nelz, KE, E, p, fixed, chunk=1 << 18):
    """Same operator without a stored K: q = sum_e E_e scatter(KE p_e), element
    chunks (for grids whose CSR does not fit)."""
    fx = np.asarray(fixed) != 0
    pm = np.where(fx, 0.0, p)
    q = np.zeros_like(pm)
    n_el = nelx * nely * nelz
    nxy = (nelx + 1) * (nely + 1)
    from .mesh import LOCAL_NODES
    for s in range(0, n_el, chunk):
        e = np.arange(s, min(n_el, s + chunk))
        ez, rem = np.divmod(e, nelx * nely)
        ex, ey = np.divmod(rem, nely)
        dofs = []
        for (dx, dy, dz) in LOCAL_NODES:
            n = (ez + dz) * nxy + (ex + dx) * (nely + 1) + (ey + dy)
            dofs += [3 * n, 3 * n + 1, 3 * n + 2]
        dofs = np.stack(dofs, axis=1)
        qe = (pm[dofs] @ KE.T) * np.asarray(E)[e][:, None]
        np.add.at(q, dofs.ravel(), qe.ravel())
    q[fx] = 0.0
    return q


def diag_K(K):
    return K.diagonal().copy()


def true_residual(K, u, f, fixed):
    """||f_f - K_ff u_f|| / ||f_f||."""
    free = np.asarray(fixed) == 0
    r = (f - K @ np.where(free, u, 0.0))[free]
    return float(np.linalg.norm(r) / np.linalg.norm(f[free]))


def matvec_rows(nelx, nely, nelz, KE, E, p, fixed, nodes):
    """Rows q_n (3 per node) of the masked operator for a list of node ids,
    by brute force over each node's (up to 8) elements.  For sampled parity
    checks on grids whose full matvec is too large for the oracle."""
    from .mesh import LOCAL_NODES
    fx = np.asarray(fixed) != 0
    pm = np.where(fx, 0.0, p)
    nxy = (nelx + 1) * (nely + 1)
    out = np.zeros((len(nodes), 3))
    for k, n in enumerate(nodes):
        iz, rem = divmod(int(n), nxy)
        ix, iy = divmod(rem, nely + 1)
        for ez in (iz - 1, iz):
            for ex in (ix - 1, ix):
                for ey in (iy - 1, iy):
                    if not (0 <= ex < nelx and 0 <= ey < nely and 0 <= ez < nelz):
                        continue
                    e = ez * nelx * nely + ex * nely + ey
                    dofs = []
                    ln = None
                    for a, (dx, dy, dz) in enumerate(LOCAL_NODES):
                        m = (ez + dz) * nxy + (ex + dx) * (nely + 1) + (ey + dy)
                        if m == n:
                            ln = a
                        dofs += [3 * m, 3 * m + 1, 3 * m + 2]
                    out[k] += E[e] * (KE[3 * ln:3 * ln + 3] @ pm[dofs])
        for c in range(3):
            if fx[3 * n + c]:
                out[k, c] = 0.0
    return out
