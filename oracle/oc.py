"""Sensitivities and the OC update (oracle).  P:44-47 §2.3.

SIMP: E_e = Emin + xPhys_e^p (E0 - Emin)
dc_e  = -p xPhys_e^(p-1) (E0 - Emin) ce_e on design elements, 0 on passive
dv_e  = 1 on design elements, 0 on passive                        S:272, R#9
OC:   xnew_j(l) = max(0, x_j - m, min(1, x_j + m, x_j sqrt(max(0, -dc~_j/(dv~_j l)))))
      on design elements; passive elements hold their passive value (0 void,
      1 solid, reading R27); bisection on l in [0, lmax]:
      lmid = (l1+l2)/2; V(lmid) > volfrac |D| -> l1 = lmid else l2 = lmid;
      repeat while (l2-l1)/(l1+l2) > tol; xnew from the last lmid.   P:47; R#15-17
Volume (mode 0): V = sum_{i in D} (H xnew / Hs)_i, computed literally.
Volume (mode 1, 2): V = sum_{i in D} xnew_i.
Passive mask values (R27): 0 design, 1 void (x = 0, "obstacle"),
2 solid (x = 1, "mandatory-solid").  If the target is unreachable for
every lambda even without move limits -- the volume with every design element
at 0 and the passive values held (mode 0: the filtered passive-solid spill into
design elements; modes 1/2: 0) already exceeds it -- the update fails with
BisectionFailure ("e.g., passive-solid volume already exceeds the target").
A target that only the move limits keep out of reach in this step is not a
failure: the bisection then ends at the lower clamps (l1 -> lmax), as in top3d.
"""
import numpy as np

VOID, SOLID = 1, 2


class BisectionFailure(RuntimeError):
    """the volume target cannot be met in [0, lmax]."""


def passive_value(passive, n):
    """Density forced on each element: NaN on design elements, 0 void, 1 solid."""
    v = np.full(n, np.nan)
    if passive is not None:
        P = np.asarray(passive)
        v[P == VOID] = 0.0
        v[P == SOLID] = 1.0
    return v


def sensitivities(xPhys, ce, penal, E0, Emin, passive=None):
    """(E, c, dc, dv) from physical densities and element energies."""
    E = Emin + xPhys ** penal * (E0 - Emin)
    c = float(np.sum(E * ce))
    dc = -penal * xPhys ** (penal - 1.0) * (E0 - Emin) * ce
    dv = np.ones_like(xPhys)
    if passive is not None:
        P = np.asarray(passive) != 0
        dc[P] = 0.0
        dv[P] = 0.0
    return E, c, dc, dv


def oc_xnew(x, dc_f, dv_f, lmid, move, passive=None):
    """xnew(lmid) on design elements, the passive value elsewhere (R15-R17, R27)."""
    D = np.ones(x.shape, dtype=bool) if passive is None else (np.asarray(passive) == 0)
    xs = np.zeros_like(x)
    if passive is not None:
        xs[np.asarray(passive) == SOLID] = 1.0
    xd, dcd, dvd = x[D], dc_f[D], dv_f[D]
    cand = xd * np.sqrt(np.maximum(0.0, -dcd / (dvd * lmid)))
    xs[D] = np.maximum(0.0, np.maximum(xd - move, np.minimum(1.0, np.minimum(xd + move, cand))))
    return xs


def oc_update(x, dc_f, dv_f, volfrac, move, tol, lmax, mode, H=None, Hs=None, passive=None,
              trace=None):
    """Returns (xnew, lmid_last, V_last, n_passes).  Literal bisection loop."""
    D = np.ones(x.shape, dtype=bool) if passive is None else (np.asarray(passive) == 0)
    target = volfrac * float(np.count_nonzero(D))
    if mode == 0 and passive is not None:          # volume at xnew = 0 on every design element
        floor = np.zeros_like(x)
        floor[np.asarray(passive) == SOLID] = 1.0
        V0 = float(np.sum(((H @ floor) / Hs)[D]))
        if V0 > target:
            raise BisectionFailure(f"passive-solid volume {V0:.6g} > target {target:.6g}")
    l1, l2 = 0.0, float(lmax)
    xnew, lmid, V, n = x.copy(), None, None, 0
    while (l2 - l1) / (l1 + l2) > tol:
        lmid = 0.5 * (l2 + l1)
        xnew = oc_xnew(x, dc_f, dv_f, lmid, move, passive)
        if mode == 0:
            xp = (H @ xnew) / Hs
            V = float(np.sum(xp[D]))
        else:
            V = float(np.sum(xnew[D]))
        if trace is not None:
            trace.append((lmid, V))
        if V > target:
            l1 = lmid
        else:
            l2 = lmid
        n += 1
    return xnew, lmid, V, n
