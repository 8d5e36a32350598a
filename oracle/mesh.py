"""Structured Hex8 mesh numbering (oracle).  P:42 §2.2 "edofMat".

node n(ix,iy,iz) = iz*(nelx+1)*(nely+1) + ix*(nely+1) + iy
element e(ex,ey,ez) = ez*nelx*nely + ex*nely + ey
local node order: (ex,ey,ez),(ex+1,ey,ez),(ex+1,ey+1,ez),(ex,ey+1,ez), then ez+1.
"""
import numpy as np

LOCAL_NODES = ((0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0),
               (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1))


def edof_matrix_loops(nelx, nely, nelz):
    """edofMat [n_el, 24] by explicit enumeration (S:64 brute force)."""
    nxy = (nelx + 1) * (nely + 1)
    edof = np.zeros((nelx * nely * nelz, 24), dtype=np.int64)
    for ez in range(nelz):
        for ex in range(nelx):
            for ey in range(nely):
                e = ez * nelx * nely + ex * nely + ey
                for a, (dx, dy, dz) in enumerate(LOCAL_NODES):
                    n = (ez + dz) * nxy + (ex + dx) * (nely + 1) + (ey + dy)
                    edof[e, 3 * a:3 * a + 3] = (3 * n, 3 * n + 1, 3 * n + 2)
    return edof


def edof_matrix(nelx, nely, nelz):
    """Same table, vectorised with numpy (checked against the loop version)."""
    nxy = (nelx + 1) * (nely + 1)
    ez, ex, ey = np.meshgrid(np.arange(nelz), np.arange(nelx), np.arange(nely), indexing="ij")
    ez, ex, ey = ez.ravel(), ex.ravel(), ey.ravel()   # external element order
    cols = []
    for (dx, dy, dz) in LOCAL_NODES:
        n = (ez + dz) * nxy + (ex + dx) * (nely + 1) + (ey + dy)
        cols += [3 * n, 3 * n + 1, 3 * n + 2]
    return np.stack(cols, axis=1).astype(np.int64)


def element_centroids(nelx, nely, nelz):
    """Centroid (ex+.5, ey+.5, ez+.5) per element in external order."""
    ez, ex, ey = np.meshgrid(np.arange(nelz), np.arange(nelx), np.arange(nely), indexing="ij")
    return np.stack([ex.ravel() + 0.5, ey.ravel() + 0.5, ez.ravel() + 0.5], axis=1)
