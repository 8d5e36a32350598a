"""ORACLE — plain, slow, obviously-correct CPU reference of the SIMP hot path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import it.  The
product path (`paper_2504_05604_b200/`) never imports, calls or links it, and
this package never imports the product path.  The two share no code; only the
seeded input generators in `workloads/` serve both.

It follows the paper's own CPU pipeline (PAPER.md = P:line):
  mesh       edofMat by explicit enumeration         P:42 §2.2; SPEC S:45
  ke         H8 stiffness by 2x2x2 Gauss quadrature  P:42 §2.2; S:117
  fem        COO->CSR assembly, BC elimination, solve P:42 §2.2; S:124-142
  sens       ce = u_e^T KE u_e, dc                   P:45-47 §2.3; S:272
  filt       cone filter H, Hs (brute force)         P:50 §2.4
  oc         OC bisection with move limits, passive  P:47 §2.3; S:282
             void (0) / solid (1) regions            S:252, S:283 (reading R27)
  loop       top3d loop                              P:53 §2.5; S:292
  mg         geometric multigrid preconditioner      SURVEY §8(f) f2;
             (Galerkin, damped Jacobi, V-cycle)      readings M1-M6 in DESIGN.md
Arithmetic is fp64 throughout.  Readings where the paper is silent are listed in
DESIGN.md ("Readings") and cited as R#n below.

Parity-pin status: every function is pinned by a `-m "not gpu"` test in
tests/test_oracle_*.py (closed forms, invariants, brute force, finite
differences).  Parity unpinned: absolute agreement with the paper's own runs
(the paper prints no compliance values).
"""
from .mesh import edof_matrix, edof_matrix_loops, element_centroids  # noqa: F401
from .ke import element_stiffness, lame  # noqa: F401
from .fem import (assemble, solve, solve_direct, solve_jacobi_cg, compliance_fu,  # noqa: F401
                  element_energies, element_energies_strain, matvec_free, matvec_elementwise, matvec_rows, diag_K,
                  true_residual)
from .filt import (filter_matrix, filter_matrix_allpairs, apply_filter, filter_rows,  # noqa: F401
                   hs_elements, apply_filter_rows)
from .oc import oc_update, oc_xnew, sensitivities, BisectionFailure, passive_value  # noqa: F401
from .loop import run_optimization  # noqa: F401
from . import mg  # noqa: F401
