"""Pins for oracle.filt, oracle.oc (filter, sensitivities, OC): brute force,
KD-tree (the paper's method), closed-form interior stencils (sum of three
squares, OEIS A005875), finite differences, OC invariants.  SURVEY §8(c)."""
import json
import os

import numpy as np
import pytest
from scipy.spatial import cKDTree

from oracle import (filter_matrix, filter_matrix_allpairs, apply_filter, element_centroids,
                    oc_update, sensitivities, element_stiffness, assemble, solve_direct,
                    element_energies, edof_matrix)
from workloads import cantilever_load, cantilever_fixed, random_density, random_vector, cylinder_passive


@pytest.mark.parametrize("dims,rmin", [((3, 3, 3), 1.5), ((7, 6, 5), 2.5), ((8, 5, 4), 3.0),
                                       ((6, 4, 3), 1.0), ((9, 4, 3), 4.0), ((5, 5, 5), 1.2)])
def test_filter_equals_allpairs(dims, rmin):
    H, Hs = filter_matrix(*dims, rmin)
    Hd = filter_matrix_allpairs(element_centroids(*dims), rmin)
    assert np.array_equal(H.toarray() != 0, Hd != 0)
    assert np.max(np.abs(H.toarray() - Hd)) < 1e-15
    assert np.allclose(Hs, Hd.sum(1), rtol=1e-15)


def test_filter_equals_kdtree_sampled_paper_grid():
    """32x16x16, rmin 4.0, 20 sampled rows vs a KD-tree radius query."""
    dims, rmin = (32, 16, 16), 4.0
    H, _ = filter_matrix(*dims, rmin)
    c = element_centroids(*dims)
    tree = cKDTree(c)
    rows = np.random.default_rng(0).choice(len(c), 20, replace=False)
    for i in rows:
        nb = tree.query_ball_point(c[i], rmin - 1e-12)
        ref = {j: rmin - np.linalg.norm(c[i] - c[j]) for j in nb}
        row = H.getrow(i)
        got = dict(zip(row.indices, row.data))
        assert set(got) == set(ref)
        for j in ref:
            assert got[j] == pytest.approx(ref[j], abs=1e-14)


@pytest.mark.parametrize("rmin,points", [(1.5, 19), (2.5, 81), (3.0, 93), (4.0, 251)])
def test_interior_stencil_closed_form(golden_dir, rmin, points):
    """Interior rows: #points = sum_{n<rmin^2} r3(n); Hs = sum r3(n)(rmin - sqrt n)."""
    r3 = json.load(open(os.path.join(golden_dir, "sum_of_three_squares.json")))["r3"]
    npts = sum(r3[n] for n in range(len(r3)) if np.sqrt(n) < rmin)
    hs = sum(r3[n] * (rmin - np.sqrt(n)) for n in range(len(r3)) if np.sqrt(n) < rmin)
    assert npts == points
    dims = (11, 11, 11)
    H, Hs = filter_matrix(*dims, rmin)
    centre = 5 * 121 + 5 * 11 + 5
    assert H.getrow(centre).nnz == points
    assert Hs[centre] == pytest.approx(hs, rel=1e-14)


def test_filter_symmetry_identity_constants():
    dims = (6, 5, 4)
    H, Hs = filter_matrix(*dims, 2.5)
    assert abs(H - H.T).max() == 0.0
    assert np.allclose(H.diagonal(), 2.5)
    one = np.ones(H.shape[0])
    assert np.allclose(apply_filter(H, Hs, 2, "dc", 3.7 * one), 3.7, rtol=1e-15)
    assert np.allclose(apply_filter(H, Hs, 0, "x", 0.3 * one), 0.3, rtol=1e-15)
    H1, Hs1 = filter_matrix(*dims, 1.0)
    v = random_vector(H.shape[0])
    for mode in (0, 1, 2):
        assert np.allclose(apply_filter(H1, Hs1, mode, "dc", v, x=np.full_like(v, .5)), v, rtol=1e-15)


def test_density_filter_volume_identity():
    """sum_{i in D} xPhys_i = dv~ . x (H symmetric), used by the GPU's OC."""
    dims = (10, 6, 4)
    H, Hs = filter_matrix(*dims, 2.5)
    passive = cylinder_passive(*dims, 5, 3, 1.6)
    D = passive == 0
    x = np.where(D, random_density(H.shape[0], seed=9), 0.0)
    xp = apply_filter(H, Hs, 0, "x", x, passive=passive)
    dv = D.astype(float)
    dvf = apply_filter(H, Hs, 0, "dv", dv)
    assert np.sum(xp[D]) == pytest.approx(dvf @ x, rel=1e-13)


def test_sensitivities_finite_differences():
    """4x2x2, rho = 0.5, central FD h = 1e-6, rel < 1e-4."""
    dims = (4, 2, 2)
    n_el = 16
    KE, edof = element_stiffness(0.3), edof_matrix(*dims)
    f, fixed = cantilever_load(*dims), cantilever_fixed(*dims)
    E0, Emin, penal = 1.0, 1e-9, 3.0

    def comp(x):
        E = Emin + x ** penal * (E0 - Emin)
        return f @ solve_direct(assemble(*dims, KE, E), f, fixed)

    x = np.full(n_el, 0.5)
    E = Emin + x ** penal * (E0 - Emin)
    u = solve_direct(assemble(*dims, KE, E), f, fixed)
    _, c, dc, _ = sensitivities(x, element_energies(u, KE, edof), penal, E0, Emin)
    assert c == pytest.approx(f @ u, rel=1e-10)
    assert np.all(dc <= 0)
    h = 1e-6
    for e in range(n_el):
        xp, xm = x.copy(), x.copy()
        xp[e] += h
        xm[e] -= h
        fd = (comp(xp) - comp(xm)) / (2 * h)
        assert abs(fd - dc[e]) < 1e-4 * abs(dc[e])
    assert np.all(sensitivities(np.zeros(n_el), np.ones(n_el), penal, E0, Emin)[2] == 0)


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_oc_uniform_fixed_point(mode):
    """uniform x = volfrac with uniform dc, dv -> xnew = volfrac."""
    dims = (6, 4, 3)
    H, Hs = filter_matrix(*dims, 1.5)
    n = H.shape[0]
    x = np.full(n, 0.3)
    dc = np.full(n, -2.0)
    dv = apply_filter(H, Hs, mode, "dv", np.ones(n))
    if mode == 0:
        dc = apply_filter(H, Hs, 0, "dc", dc)
    xnew, lam, V, npass = oc_update(x, dc, dv, 0.3, 0.2, 1e-10, 1e9, mode, H, Hs)
    assert np.allclose(xnew, 0.3, atol=1e-8)


def test_oc_move_clamp_and_passive_and_volume():
    dims = (3, 3, 3)
    n = 27
    passive = np.zeros(n, dtype=np.uint8)
    passive[13] = 1                                  # one passive-void element
    D = passive == 0
    H, Hs = filter_matrix(*dims, 1.5)
    x = np.where(D, 0.3, 0.0)
    dc = -random_density(n, seed=2, lo=0.1, hi=5.0)
    dc[0] = -1e12                                    # huge -dc -> min(1, x+move)
    dc[passive != 0] = 0
    for mode in (0, 1):
        dv = apply_filter(H, Hs, mode, "dv", D.astype(float))
        dcf = apply_filter(H, Hs, mode, "dc", dc, x=x)
        trace = []
        xnew, lam, V, npass = oc_update(x, dcf, dv, 0.3, 0.2, 1e-10, 1e9, mode, H, Hs, passive,
                                        trace=trace)
        assert xnew[13] == 0.0
        assert np.all(np.abs(xnew - x)[D] <= 0.2 + 1e-15)
        assert np.all((xnew >= 0) & (xnew <= 1))
        if mode == 1:
            assert xnew[0] == pytest.approx(0.5)
            assert abs(xnew[D].mean() - 0.3) <= 1e-6                    # north_star 1e-6
        else:
            xp = apply_filter(H, Hs, 0, "x", xnew, passive=passive)
            assert abs(xp[D].mean() - 0.3) <= 1e-6
        # V(lambda) non-increasing along the bisection trace
        tr = sorted(trace)
        assert all(tr[i][1] >= tr[i + 1][1] - 1e-12 for i in range(len(tr) - 1))
        assert npass == len(trace) and npass > 30


def test_filter_rows_equal_matrix():
    dims, rmin = (7, 6, 5), 2.5
    H, Hs = filter_matrix(*dims, rmin)
    from oracle import filter_rows
    rows = [0, 17, 100, 209]
    rr, hs = filter_rows(*dims, rmin, rows)
    for (cols, w), i in zip(rr, rows):
        row = H.getrow(i)
        assert dict(zip(cols.tolist(), w.tolist())) == pytest.approx(dict(zip(row.indices.tolist(), row.data.tolist())))
    assert np.allclose(hs, Hs[rows], rtol=1e-15)


@pytest.mark.parametrize("dims,rmin", [((7, 6, 5), 2.5), ((9, 4, 3), 4.0), ((8, 5, 4), 3.0), ((6, 4, 3), 1.5)])
def test_apply_filter_rows_equals_matrix_filter(dims, rmin):
    """The row-wise (H-free) filter used at full size equals the sparse-H filter,
    every mode and operand, on every row; hs_elements equals H's row sums."""
    from oracle import apply_filter_rows, hs_elements
    from workloads import solid_block_passive
    H, Hs = filter_matrix(*dims, rmin)
    n = H.shape[0]
    rows = np.arange(n)
    assert np.allclose(hs_elements(*dims, rmin, rows), Hs, rtol=1e-14, atol=0)
    pas = solid_block_passive(*dims, (0, 2), (0, 2), (0, dims[2]), base=(dims[0] - 1.0, dims[1] - 1.0, 1.2))
    x = random_density(n, seed=21, lo=1e-4, hi=1.0)
    v = -random_density(n, seed=22, lo=0.1, hi=3.0)
    for mode in (0, 1, 2):
        for what in ("dc", "dv", "x"):
            ref = apply_filter(H, Hs, mode, what, v if what != "x" else x, x=x, passive=pas)
            got = apply_filter_rows(*dims, rmin, mode, what, rows, v if what != "x" else x, x=x, passive=pas)
            assert np.allclose(got, ref, rtol=1e-13, atol=1e-15), (mode, what)
