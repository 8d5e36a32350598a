"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no stiffness, no solve, no
filter, no OC).  It only defines problem inputs: grid sizes and parameters of
the BASELINE.json configs, the cantilever load / support masks, the config-2
cylinder obstacle and seeded random fields.  Both `oracle/` and the product
path may import it; neither imports the other.

Numbering (external, SPEC S:45 [mesh/build_mesh]):
  node    n(ix,iy,iz) = iz*(nelx+1)*(nely+1) + ix*(nely+1) + iy
  element e(ex,ey,ez) = ez*nelx*nely + ex*nely + ey
  DOFs of node n: 3n, 3n+1, 3n+2 = (ux, uy, uz)
"""
from .cantilever import (  # noqa: F401
    CONFIGS, COMMON, PAPER_PROTOCOL, PAPER_PROTOCOL_OBSTACLE, paper_obstacle, config_params, point_load, n_nodes, n_elems, node_id, elem_id,
    cantilever_load, cantilever_fixed, roller_patch_problem, cylinder_passive, solid_block_passive,
    random_density, random_vector, make_problem,
)
