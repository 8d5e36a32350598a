"""Hex8 element stiffness (oracle).  P:42 §2.2 "Element stiffness matrices are
pre-computed"; unit cube, unit modulus, isotropic linear
elasticity, 2x2x2 Gauss quadrature (exact for the trilinear integrand).
Reading R#1: the quadrature KE on the unit cube IS the KE (no extra factor).
"""
import numpy as np
from .mesh import LOCAL_NODES


def lame(E, nu):
    """Lamé constants (lambda, mu) of isotropic elasticity."""
    return E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), E / (2.0 * (1.0 + nu))


def constitutive(E, nu):
    """6x6 isotropic D in Voigt order (xx, yy, zz, xy, yz, zx), engineering shear."""
    lam, mu = lame(E, nu)
    D = np.zeros((6, 6))
    D[:3, :3] = lam
    for i in range(3):
        D[i, i] += 2.0 * mu
        D[3 + i, 3 + i] = mu
    return D


def shape_gradients(xi, eta, zeta):
    """dN_a/d(x,y,z) [8,3] of the trilinear unit-cube shape functions."""
    g = np.zeros((8, 3))
    for a, (ax, ay, az) in enumerate(LOCAL_NODES):
        nx, dnx = (xi, 1.0) if ax else (1.0 - xi, -1.0)
        ny, dny = (eta, 1.0) if ay else (1.0 - eta, -1.0)
        nz, dnz = (zeta, 1.0) if az else (1.0 - zeta, -1.0)
        g[a] = (dnx * ny * nz, nx * dny * nz, nx * ny * dnz)
    return g


def strain_displacement(xi, eta, zeta):
    """B [6,24] so that eps = B @ u_e (u_e = (ux,uy,uz) per local node)."""
    g = shape_gradients(xi, eta, zeta)
    B = np.zeros((6, 24))
    for a in range(8):
        dx, dy, dz = g[a]
        B[0, 3 * a + 0] = dx
        B[1, 3 * a + 1] = dy
        B[2, 3 * a + 2] = dz
        B[3, 3 * a + 0] = dy
        B[3, 3 * a + 1] = dx
        B[4, 3 * a + 1] = dz
        B[4, 3 * a + 2] = dy
        B[5, 3 * a + 0] = dz
        B[5, 3 * a + 2] = dx
    return B


def element_stiffness(nu, E=1.0):
    """KE [24,24] = sum_gp w B^T D B over 2x2x2 Gauss points of [0,1]^3 (w = 1/8)."""
    D = constitutive(E, nu)
    pts = (0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0))
    KE = np.zeros((24, 24))
    for xi in pts:
        for eta in pts:
            for zeta in pts:
                B = strain_displacement(xi, eta, zeta)
                KE += 0.125 * (B.T @ D @ B)
    return KE
