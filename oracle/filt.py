"""Cone (linear-decay) filter (oracle).  P:50 §2.4: weights "decaying linearly
with distance up to a specified filter radius (rmin)"; H stored sparse, applied
by sparse matrix multiplication.  SPEC S:183-216.

H_ij = max(0, rmin - ||c_i - c_j||) for ||c_i - c_j|| < rmin (R#12), centroids
(ex+.5, ey+.5, ez+.5); Hs_i = sum_j H_ij over in-domain j (R#13, truncated at
the boundary).  Modes (R#10, R#11):
  0 density filter      xPhys = (H x)/Hs (passive forced to 0 void / 1 solid, R27);
                        dc~ = H(dc/Hs); dv~ = H(dv/Hs)
  1 sensitivity filter  dc~_i = sum_j H_ij x_j dc_j / (Hs_i max(gamma, x_i)), gamma = 1e-3
  2 plain               dc~ = (H dc)/Hs
"""
import numpy as np
import scipy.sparse as sp

GAMMA = 1e-3


def filter_matrix(nelx, nely, nelz, rmin):
    """H (CSR, symmetric) by enumerating every lattice offset of the box
    |d| <= ceil(rmin) and keeping d < rmin; plus Hs = H 1."""
    n_el = nelx * nely * nelz
    ez, ex, ey = np.meshgrid(np.arange(nelz), np.arange(nelx), np.arange(nely), indexing="ij")
    ex, ey, ez = ex.ravel(), ey.ravel(), ez.ravel()
    e = np.arange(n_el)
    R = int(np.ceil(rmin))
    rows, cols, vals = [], [], []
    for dz in range(-R, R + 1):
        for dx in range(-R, R + 1):
            for dy in range(-R, R + 1):
                d = np.sqrt(float(dx * dx + dy * dy + dz * dz))
                if not d < rmin:
                    continue
                jx, jy, jz = ex + dx, ey + dy, ez + dz
                ok = (jx >= 0) & (jx < nelx) & (jy >= 0) & (jy < nely) & (jz >= 0) & (jz < nelz)
                j = jz * nelx * nely + jx * nely + jy
                rows.append(e[ok])
                cols.append(j[ok])
                vals.append(np.full(int(ok.sum()), rmin - d))
    H = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n_el, n_el)).tocsr()
    Hs = np.asarray(H.sum(axis=1)).ravel()
    return H, Hs


def filter_matrix_allpairs(centroids, rmin):
    """Dense O(N^2) all-pairs H (brute force cross-check)."""
    d = np.sqrt(((centroids[:, None, :] - centroids[None, :, :]) ** 2).sum(-1))
    return np.where(d < rmin, rmin - d, 0.0)


def apply_filter(H, Hs, mode, what, v, x=None, passive=None):
    """One filter application.
    what = "x"  : physical densities from design variables (mode 0), else identity
    what = "dc" : filtered sensitivities
    what = "dv" : filtered volume sensitivities
    """
    if what == "x":
        if mode != 0:
            return v.copy()
        out = (H @ v) / Hs
        if passive is not None:                     # R14, R27: passive value after filtering
            P = np.asarray(passive)
            out[P == 1] = 0.0
            out[P == 2] = 1.0
        return out
    if mode == 0:
        return H @ (v / Hs)
    if mode == 1:
        if what == "dv":
            return v.copy()
        return (H @ (x * v)) / (Hs * np.maximum(GAMMA, x))
    if mode == 2:
        if what == "dv":
            return v.copy()
        return (H @ v) / Hs
    raise ValueError(mode)


def filter_rows(nelx, nely, nelz, rmin, rows):
    """Rows of H for a list of element ids, by brute force over the offset box
    (for sampled checks on grids whose H does not fit).  Returns a list of
    (cols, weights) and the row sums Hs[rows]."""
    R = int(np.ceil(rmin))
    out, hs = [], []
    for e in rows:
        ez, rem = divmod(int(e), nelx * nely)
        ex, ey = divmod(rem, nely)
        cols, w = [], []
        for dz in range(-R, R + 1):
            for dx in range(-R, R + 1):
                for dy in range(-R, R + 1):
                    d = np.sqrt(float(dx * dx + dy * dy + dz * dz))
                    jx, jy, jz = ex + dx, ey + dy, ez + dz
                    if d < rmin and 0 <= jx < nelx and 0 <= jy < nely and 0 <= jz < nelz:
                        cols.append(jz * nelx * nely + jx * nely + jy)
                        w.append(rmin - d)
        out.append((np.array(cols), np.array(w)))
        hs.append(float(np.sum(w)))
    return out, np.array(hs)


def _offsets(rmin):
    """Ball offsets (dx, dy, dz) with |d| < rmin and weights rmin - |d| (R#12)."""
    R = int(np.ceil(rmin))
    o = [(dx, dy, dz, rmin - np.sqrt(float(dx * dx + dy * dy + dz * dz)))
         for dz in range(-R, R + 1) for dx in range(-R, R + 1) for dy in range(-R, R + 1)
         if np.sqrt(float(dx * dx + dy * dy + dz * dz)) < rmin]
    return [np.array(v) for v in zip(*o)]


def hs_elements(nelx, nely, nelz, rmin, elems):
    """Hs_e = sum of the in-domain weights of element e's ball (R#13), for a list of
    element ids, by enumerating the ball offsets -- row sums of H without H (the
    in-domain test is the same `0 <= j < n` per axis as filter_matrix)."""
    dx, dy, dz, w = _offsets(rmin)
    elems = np.asarray(elems, dtype=np.int64)
    ez, rem = np.divmod(elems, nelx * nely)
    ex, ey = np.divmod(rem, nely)
    hs = np.zeros(elems.size)
    for k in range(w.size):
        ok = ((ex + dx[k] >= 0) & (ex + dx[k] < nelx) & (ey + dy[k] >= 0) & (ey + dy[k] < nely)
              & (ez + dz[k] >= 0) & (ez + dz[k] < nelz))
        hs += np.where(ok, w[k], 0.0)
    return hs


def apply_filter_rows(nelx, nely, nelz, rmin, mode, what, rows, v, x=None, passive=None):
    """apply_filter(...)[rows] without forming H (for grids whose H does not fit):
    the same definitions as apply_filter, row by row over the ball offsets, with
    Hs from hs_elements.  v, x, passive are full-length arrays."""
    dx, dy, dz, w = _offsets(rmin)
    rows = np.asarray(rows, dtype=np.int64)
    ez, rem = np.divmod(rows, nelx * nely)
    ex, ey = np.divmod(rem, nely)
    hs_i = hs_elements(nelx, nely, nelz, rmin, rows)
    v = np.asarray(v)
    if what == "x" and mode != 0:
        return v[rows].copy()
    if what == "dv" and mode != 0:
        return v[rows].copy()
    acc = np.zeros(rows.size)
    hs_of = None
    if what in ("dc", "dv") and mode == 0:       # Hs of every neighbour, computed once per distinct element
        allj = []
        for k in range(w.size):
            jx, jy, jz = ex + dx[k], ey + dy[k], ez + dz[k]
            ok = (jx >= 0) & (jx < nelx) & (jy >= 0) & (jy < nely) & (jz >= 0) & (jz < nelz)
            allj.append((jz * nelx * nely + jx * nely + jy)[ok])
        uj = np.unique(np.concatenate(allj))
        hs_u = hs_elements(nelx, nely, nelz, rmin, uj)
        hs_of = lambda j: hs_u[np.searchsorted(uj, j)]  # noqa: E731
    for k in range(w.size):
        jx, jy, jz = ex + dx[k], ey + dy[k], ez + dz[k]
        ok = (jx >= 0) & (jx < nelx) & (jy >= 0) & (jy < nely) & (jz >= 0) & (jz < nelz)
        j = np.where(ok, jz * nelx * nely + jx * nely + jy, 0)
        if what in ("dc", "dv") and mode == 0:
            term = np.where(ok, v[j] / np.where(ok, hs_of(np.where(ok, j, uj[0])), 1.0), 0.0)   # H (v / Hs)
        elif mode == 1:
            term = np.asarray(x)[j] * v[j]                              # H (x v)
        else:
            term = v[j]
        acc += np.where(ok, w[k] * term, 0.0)
    if what in ("dc", "dv") and mode == 0:
        return acc
    if mode == 1:
        return acc / (hs_i * np.maximum(GAMMA, np.asarray(x)[rows]))
    out = acc / hs_i
    if what == "x" and passive is not None:
        P = np.asarray(passive)[rows]
        out[P == 1] = 0.0
        out[P == 2] = 1.0
    return out
