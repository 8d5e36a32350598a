"""top3d-style SIMP loop (oracle).  P:53 §2.5 "iterative optimization loop
involving FEM analysis, sensitivity computation, sensitivity filtering, design
variable update using OC"; SURVEY §8(a) A8.

x0 = volfrac on D, 0 on passive void, 1 on passive solid; xPhys0 = x0 (R#18, R27).  Fixed n_iter (R#19).
Per iteration: E(xPhys) -> K -> u -> ce, c = sum E ce -> dc, dv -> filter ->
OC -> x, xPhys.  c_hist[it] is the compliance of the design entering it.
"""
import numpy as np

from .mesh import edof_matrix
from .ke import element_stiffness
from .fem import assemble, solve, element_energies
from .filt import filter_matrix, apply_filter
from .oc import sensitivities, oc_update


def run_optimization(p, f, fixed, passive=None, n_iter=None, solver="auto", x0=None,
                     record=False):
    nelx, nely, nelz = p["nelx"], p["nely"], p["nelz"]
    n_iter = p["n_iter"] if n_iter is None else n_iter
    mode = p.get("filter_mode", 0)
    KE = element_stiffness(p["nu"])
    edof = edof_matrix(nelx, nely, nelz)
    H, Hs = filter_matrix(nelx, nely, nelz, p["rmin"])
    n_el = nelx * nely * nelz
    D = np.ones(n_el, dtype=bool) if passive is None else (np.asarray(passive) == 0)
    if x0 is None:
        x = np.where(D, p["volfrac"], 0.0)
        if passive is not None:
            x[np.asarray(passive) == 2] = 1.0       # R27: passive solid holds 1
    else:
        x = np.asarray(x0, dtype=np.float64).copy()
        if passive is not None:
            x[np.asarray(passive) == 1] = 0.0
            x[np.asarray(passive) == 2] = 1.0
    xPhys = x.copy()
    dv_f = None
    hist = dict(c=[], fu=[], change=[], lam=[], vol=[], n_oc=[])
    recs = []
    for it in range(n_iter):
        E = p["Emin"] + xPhys ** p["penal"] * (p["E0"] - p["Emin"])
        K = assemble(nelx, nely, nelz, KE, E, edof)
        u = solve(K, f, fixed, method=solver)
        ce = element_energies(u, KE, edof)
        E, c, dc, dv = sensitivities(xPhys, ce, p["penal"], p["E0"], p["Emin"], passive)
        dc_f = apply_filter(H, Hs, mode, "dc", dc, x=x, passive=passive)
        if dv_f is None or mode != 0:
            dv_f = apply_filter(H, Hs, mode, "dv", dv, x=x, passive=passive)
        xnew, lam, V, n_oc = oc_update(x, dc_f, dv_f, p["volfrac"], p["move"], p["oc_tol"],
                                       p["oc_lmax"], mode, H, Hs, passive)
        change = float(np.max(np.abs(xnew - x)[D]))
        if record:
            recs.append(dict(xPhys=xPhys.copy(), x=x.copy(), u=u, ce=ce, dc=dc, dc_f=dc_f,
                             dv_f=dv_f.copy(), xnew=xnew.copy(), lam=lam))
        x = xnew
        xPhys = apply_filter(H, Hs, mode, "x", x, passive=passive)
        hist["c"].append(c)
        hist["fu"].append(float(f @ u))
        hist["change"].append(change)
        hist["lam"].append(lam)
        hist["vol"].append(float(np.sum(xPhys[D])) / np.count_nonzero(D))
        hist["n_oc"].append(n_oc)
    out = dict(x=x, xPhys=xPhys, **{k: np.array(v) for k, v in hist.items()})
    if record:
        out["records"] = recs
    return out
