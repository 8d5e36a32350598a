"""Synthetic cantilever workloads (BASELINE.json `configs`).

Readings applied here:
  #4  load: f_y = -1/(nelz+1) on each of the nelz+1 nodes of the edge
      x = nelx, y = 0 (total -1)           [BASELINE.json configs; §3]
  #5  supports: all 3 DOFs of every node with ix = 0   [P:59 "left face"]
  #22 random x: default_rng(0).uniform(0.01, 1.0, n_el) [config 1]
  #23 obstacle: element passive iff (ex+.5-cx)^2 + (ey+.5-cy)^2 < r^2, all ez
"""
import numpy as np

# Parameters common to every BASELINE.json config (BASELINE.json configs[0]).
COMMON = dict(E0=1.0, Emin=1e-9, nu=0.3, penal=3.0, move=0.2,
              filter_mode=0, oc_tol=1e-10, oc_lmax=1e9)

# BASELINE.json `configs` (DOF counts recomputed).
CONFIGS = {
    0: dict(nelx=30, nely=10, nelz=2, volfrac=0.3, rmin=1.5, n_iter=20, cg_rtol=1e-10,
            obstacle=None),
    1: dict(nelx=60, nely=20, nelz=4, volfrac=0.3, rmin=1.5, n_iter=50, cg_rtol=1e-10,
            obstacle=None),
    2: dict(nelx=120, nely=40, nelz=20, volfrac=0.2, rmin=2.5, n_iter=30, cg_rtol=1e-10,
            obstacle=(60.0, 20.0, 8.0)),
    3: dict(nelx=256, nely=128, nelz=128, volfrac=0.15, rmin=3.0, n_iter=10, cg_rtol=1e-8,
            obstacle=None),
    4: dict(nelx=512, nely=256, nelz=256, volfrac=0.12, rmin=3.0, n_iter=5, cg_rtol=1e-8,
            obstacle=None),
}


# The paper's own benchmark protocol (§3, §4.2; SURVEY
# §8(f) NEXT f1): 32x16x16 cantilever, volfrac 0.2, penal 3.0, rmin 4.0,
# 200 iterations, left face fixed, a vertical point load at the centre of the
# free end's bottom edge, the paper's sensitivity filter.  The
# solve tolerance stands in for the paper's direct solver.
PAPER_PROTOCOL = dict(nelx=32, nely=16, nelz=16, volfrac=0.2, rmin=4.0, n_iter=200, cg_rtol=1e-10,
                      obstacle=None, filter_mode=1, load="point")
# ... with the section-3 cylinder obstacle (paper_obstacle below)
PAPER_PROTOCOL_OBSTACLE = dict(PAPER_PROTOCOL, obstacle="paper")


def config_params(cfg, **over):
    """Full parameter dict of a config (common values + config values + overrides)."""
    p = dict(COMMON)
    p.update(CONFIGS[cfg] if not isinstance(cfg, dict) else cfg)
    p.update(over)
    return p


def n_nodes(nelx, nely, nelz):
    return (nelx + 1) * (nely + 1) * (nelz + 1)


def n_elems(nelx, nely, nelz):
    return nelx * nely * nelz


def node_id(nelx, nely, nelz, ix, iy, iz):
    return iz * (nelx + 1) * (nely + 1) + ix * (nely + 1) + iy


def elem_id(nelx, nely, nelz, ex, ey, ez):
    return ez * nelx * nely + ex * nely + ey


def cantilever_load(nelx, nely, nelz):
    """f[3*n_nd]: -1/(nelz+1) in y on the nodes (nelx, 0, iz), iz = 0..nelz."""
    f = np.zeros(3 * n_nodes(nelx, nely, nelz))
    for iz in range(nelz + 1):
        n = node_id(nelx, nely, nelz, nelx, 0, iz)
        f[3 * n + 1] = -1.0 / (nelz + 1)
    return f


def cantilever_fixed(nelx, nely, nelz):
    """fixed[3*n_nd] (uint8): every DOF of every node with ix = 0."""
    fx = np.zeros(3 * n_nodes(nelx, nely, nelz), dtype=np.uint8)
    iz, iy = np.meshgrid(np.arange(nelz + 1), np.arange(nely + 1), indexing="ij")
    n = node_id(nelx, nely, nelz, 0, iy.ravel(), iz.ravel())
    for c in range(3):
        fx[3 * n + c] = 1
    return fx


def roller_patch_problem(nelx, nely, nelz, traction=1.0):
    """Roller-supported bar under uniform x-traction on the x = nelx face.

    Supports: u_x = 0 on x = 0, u_y = 0 on y = 0, u_z = 0 on z = 0.
    Load: consistent nodal forces of a uniform traction on unit bilinear faces
    (each face contributes traction/4 to each of its 4 nodes).
    Returns (f, fixed).  Used by the patch test (SURVEY §8(c) pins).
    """
    nn = n_nodes(nelx, nely, nelz)
    f = np.zeros(3 * nn)
    fixed = np.zeros(3 * nn, dtype=np.uint8)
    for iz in range(nelz + 1):
        for ix in range(nelx + 1):
            for iy in range(nely + 1):
                n = node_id(nelx, nely, nelz, ix, iy, iz)
                if ix == 0:
                    fixed[3 * n + 0] = 1
                if iy == 0:
                    fixed[3 * n + 1] = 1
                if iz == 0:
                    fixed[3 * n + 2] = 1
    for ez in range(nelz):
        for ey in range(nely):
            for (dy, dz) in ((0, 0), (1, 0), (0, 1), (1, 1)):
                n = node_id(nelx, nely, nelz, nelx, ey + dy, ez + dz)
                f[3 * n + 0] += traction / 4.0
    return f, fixed


def cylinder_passive(nelx, nely, nelz, cx, cy, r):
    """passive[n_el] (uint8): z-axis cylinder, centroid test (reading #23)."""
    ez, ex, ey = np.meshgrid(np.arange(nelz), np.arange(nelx), np.arange(nely), indexing="ij")
    inside = (ex + 0.5 - cx) ** 2 + (ey + 0.5 - cy) ** 2 < r * r
    return inside.ravel().astype(np.uint8)  # ravel order = (ez, ex, ey) = external numbering


def solid_block_passive(nelx, nely, nelz, xr, yr, zr, base=None):
    """Passive mask with values 0 design, 1 void, 2 solid (reading R27): elements
    with ex in [xr), ey in [yr), ez in [zr) are passive SOLID (2); if `base` =
    (cx, cy, r) is given, the z-cylinder of cylinder_passive is passive VOID (1)."""
    pas = np.zeros(n_elems(nelx, nely, nelz), dtype=np.uint8)
    if base is not None:
        pas[cylinder_passive(nelx, nely, nelz, *base) != 0] = 1
    ez, ex, ey = np.meshgrid(np.arange(nelz), np.arange(nelx), np.arange(nely), indexing="ij")
    box = ((ex >= xr[0]) & (ex < xr[1]) & (ey >= yr[0]) & (ey < yr[1]) & (ez >= zr[0]) & (ez < zr[1]))
    pas[box.ravel()] = 2
    return pas


def paper_obstacle(nelx, nely, nelz, radius=0.15):
    """The paper's section-3 obstacle ("A cylindrical obstacle region is
    defined within the domain where material is disallowed"), in the shape of
    SPEC's example: a cylinder with its axis along y through the domain
    centre, radius 0.15 and full height, in coordinates normalised per axis to
    [0, 1]; element passive VOID (1) iff its normalised centroid satisfies
    (xc - 0.5)^2 + (zc - 0.5)^2 < radius^2."""
    ez, ex, ey = np.meshgrid(np.arange(nelz), np.arange(nelx), np.arange(nely), indexing="ij")
    xc, zc = (ex + 0.5) / nelx, (ez + 0.5) / nelz
    return ((xc - 0.5) ** 2 + (zc - 0.5) ** 2 < radius * radius).ravel().astype(np.uint8)


def random_density(n_el, seed=0, lo=0.01, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, n_el)


def random_vector(n, seed=1):
    return np.random.default_rng(seed).standard_normal(n)


def point_load(nelx, nely, nelz):
    """f_y = -1 on the node at the centre of the free end's bottom edge:
    (ix, iy, iz) = (nelx, 0, nelz // 2)  ("vertical point load ... at the
    center of the free end's bottom edge"; vertical = -y as in the configs)."""
    f = np.zeros(3 * n_nodes(nelx, nely, nelz))
    f[3 * node_id(nelx, nely, nelz, nelx, 0, nelz // 2) + 1] = -1.0
    return f


def make_problem(cfg, **over):
    """(params, f, fixed, passive-or-None) for a BASELINE config index, "paper"
    (the paper's benchmark protocol), "paper_obstacle" (the same with the
    section-3 cylinder) or a dict."""
    if cfg == "paper":
        cfg = PAPER_PROTOCOL
    elif cfg == "paper_obstacle":
        cfg = PAPER_PROTOCOL_OBSTACLE
    p = config_params(cfg, **over)
    nelx, nely, nelz = p["nelx"], p["nely"], p["nelz"]
    f = point_load(nelx, nely, nelz) if p.get("load") == "point" else cantilever_load(nelx, nely, nelz)
    fixed = cantilever_fixed(nelx, nely, nelz)
    passive = None
    if p.get("obstacle") == "paper":
        passive = paper_obstacle(nelx, nely, nelz)
    elif p.get("obstacle"):
        cx, cy, r = p["obstacle"]
        passive = cylinder_passive(nelx, nely, nelz, cx, cy, r)
    return p, f, fixed, passive
