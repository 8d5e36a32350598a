/*
 * topo.h -- C ABI of the B200-native matrix-free SIMP hot path
 * (PyTopo3D, arXiv 2504.05604; PAPER.md = "P:line", SPEC.md = "S:line").
 *
 * One call per step of the paper's optimisation loop (§2.5):
 *   topo_init         problem statement: grid, material, loads, supports,
 *                     passive (obstacle) regions              P:42 §2.2, §2.3
 *   topo_set_density  design variables x (pseudo-densities)   P:45 §2.3
 *   topo_solve        K(x) u = f, matrix-free EbE PCG          P:42 §2.2
 *                     (Jacobi or geometric-multigrid preconditioner)
 *   topo_sensitivity  ce = u_e^T KE u_e, c, dc                P:47 §2.3
 *   topo_filter       rmin cone filter (density / sensitivity) P:50 §2.4
 *   topo_oc_step      OC bisection with move limits            P:44-47 §2.3
 *   topo_optimize     the whole loop for n_iter iterations      P:53 §2.5
 *
 * Conventions
 *  - Every call returns int: TOPO_OK (0) or a TOPO_E* code.  No call throws,
 *    aborts or exits.  topo_last_error(ctx) has a one-line explanation.
 *  - Arithmetic is IEEE binary64 throughout (the BASELINE configs say fp64).
 *  - Host arrays use the EXTERNAL numbering of SPEC S:45:
 *        node    n(ix,iy,iz) = iz*(nelx+1)*(nely+1) + ix*(nely+1) + iy
 *        element e(ex,ey,ez) = ez*nelx*nely + ex*nely + ey
 *        DOFs of node n: 3n, 3n+1, 3n+2 = (ux, uy, uz)
 *    The device layout is private (x-slab SoA).
 *  - Ownership: the caller owns every host buffer.  Inputs are copied before
 *    the call returns and never retained.  Outputs go to caller-allocated
 *    buffers of the documented length; a NULL output is skipped.  The context
 *    owns all device memory until topo_destroy.
 *  - Multi-GPU (x-slabs): with dist->mode == TOPO_DIST_NCCL each rank passes
 *    GLOBAL-size inputs; outputs are written only for that rank's owned
 *    elements [ex_begin, ex_end) x all y,z (and the matching node planes);
 *    entries of other ranks are left untouched (gathering is the caller's job).
 *    TOPO_DIST_LOOPBACK runs `world` slabs in ONE process on one GPU (tests
 *    the partition and halo logic); outputs are then complete.
 *    TOPO_DIST_HOST: like NCCL (one process per slab), host-staged transport.
 *  - Threading: one context per thread; distinct contexts are independent,
 *    except that the element stiffness, filter weights and multigrid tables
 *    live in __constant__ memory of the device: a context re-uploads its
 *    tables whenever another context on the same device ran since its last
 *    call, so contexts on one device must not run CONCURRENTLY (interleaved
 *    calls are fine).
 *  - Call order: init -> [set_density] -> solve -> sensitivity -> filter(dc)
 *    -> oc_step.  A call whose inputs are not ready returns TOPO_ESTATE.
 */
#ifndef TOPO_H
#define TOPO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes (mapped from SPEC's error kinds) ---------- */
#define TOPO_OK              0
#define TOPO_EINVAL          1  /* bad dims/params, load on a fixed DOF */
#define TOPO_ENOCONV         2  /* PCG hit cg_max_iter (S:138 SingularSystem)               */
#define TOPO_EBREAKDOWN      3  /* PCG p^T K p <= 0 or non-finite                           */
#define TOPO_EUNCONSTRAINED  4  /* no fixed DOF (S:138 InsufficientConstraints)             */
#define TOPO_EBISECT         5  /* volume target unreachable in [0, oc_lmax]         */
#define TOPO_EALLPASSIVE     6  /* no design element                                */
#define TOPO_ECUDA           7
#define TOPO_ENCCL           8
#define TOPO_ENOMEM          9
#define TOPO_ESTATE         10  /* call order / missing input                               */

/* ---- filter modes (§2.4; reading R#10) -------------------- */
#define TOPO_FILTER_DENSITY     0  /* xPhys = H x / Hs ; dc~ = H(dc/Hs) ; dv~ = H(dv/Hs)     */
#define TOPO_FILTER_SENSITIVITY 1  /* dc~_i = sum_j H_ij x_j dc_j / (Hs_i max(1e-3, x_i))   */
#define TOPO_FILTER_PLAIN       2  /* dc~ = H dc / Hs                                       */

/* topo_filter `what` */
#define TOPO_FILTER_X   0   /* design variables -> physical densities                */
#define TOPO_FILTER_DC  1   /* raw sensitivities -> filtered sensitivities            */

/* topo_get fields.  Element fields are [n_el], node fields [3*n_nd] (DOF
 * interleaved, like u) unless noted.                                        */
#define TOPO_FIELD_U        0  /* displacements [3*n_nd]                         */
#define TOPO_FIELD_X        1  /* design variables [n_el]                        */
#define TOPO_FIELD_XPHYS    2  /* physical densities [n_el]                      */
#define TOPO_FIELD_E        3  /* SIMP modulus E_e [n_el]                        */
#define TOPO_FIELD_CE       4  /* element energies u_e^T KE u_e [n_el]           */
#define TOPO_FIELD_DC       5  /* raw sensitivities [n_el]                       */
#define TOPO_FIELD_DCF      6  /* filtered sensitivities [n_el]                  */
#define TOPO_FIELD_DVF      7  /* filtered volume sensitivities [n_el]           */
#define TOPO_FIELD_XNEW     8  /* last OC result [n_el]                          */
#define TOPO_FIELD_HS       9  /* filter row sums Hs [n_el]                      */
#define TOPO_FIELD_INVDIAG 10  /* Jacobi inverse diagonal per DOF [3*n_nd], 0 on fixed */
#define TOPO_FIELD_R       11  /* PCG recursive residual [3*n_nd]               */

/* distribution modes */
#define TOPO_DIST_SINGLE   0
#define TOPO_DIST_NCCL     1   /* EXPERIMENTAL: the NCCL data plane has never run (every GPU box of
                                  this build has one GPU); its control flow is the HOST mode's,
                                  which is tested with 2-4 processes on one GPU                   */
#define TOPO_DIST_LOOPBACK 2
#define TOPO_DIST_HOST     3   /* one process per slab, host-staged shared-memory transport (tests) */
#define TOPO_DIST_SOLO     4   /* measurement only: rank `rank`'s slab of a `world`-slab run, alone on
                                  this GPU, every exchange / allreduce / all-gather omitted (the
                                  other ranks' moduli are this slab's, tiled).  The kernel sequence
                                  and sizes are one rank's of the NCCL run; the numbers are NOT a
                                  solution of the problem (the coupling is dropped) -- for per-rank
                                  compute time of a strong-scaling run (tools/solo_scale.py)      */

typedef struct topo_ctx topo_ctx;    /* opaque; owns all device state */

/* Problem parameters.  Fill with topo_params_default first. */
typedef struct {
  int32_t nelx, nely, nelz;   /* elements per axis, >= 1; unit cubes           */
  double  volfrac;            /* 0 < volfrac < 1: target mean density over design elements  */
  double  penal;              /* SIMP exponent p >= 1 ("commonly p = 3")              */
  double  rmin;               /* filter radius in element lengths, 0 < rmin <= 6     */
  double  E0, Emin;           /* 0 < Emin < E0                                       */
  double  nu;                 /* Poisson ratio 0 <= nu < 0.5                        */
  double  move;               /* OC move limit 0 < move <= 1 ("standard move limits")  */
  int32_t filter_mode;        /* TOPO_FILTER_*                                              */
  double  cg_rtol;            /* stop when ||r|| <= cg_rtol ||f_free|| (then true residual) */
  int64_t cg_max_iter;        /* <= 0 -> 10 * n_dof                                  */
  int32_t cg_warm_start;      /* 1: start PCG from the previous u                            */
  double  oc_tol;             /* bisection stops when (l2-l1)/(l1+l2) <= oc_tol              */
  double  oc_lmax;            /* initial bracket [0, oc_lmax]                                */
  int32_t deterministic;      /* reductions are always fixed-order; kept for the ABI */
  int32_t cg_check_every;     /* PCG iterations per CUDA-graph batch between host polls; <=0 auto */
  /* Preconditioner of the PCG solve (readings M1-M6).
   * TOPO_PRECOND_JACOBI: z = D^-1 r with the on-the-fly diagonal.
   * TOPO_PRECOND_MG: one V-cycle of geometric multigrid on the nested Hex8 grids
   *   (trilinear transfer, Galerkin coarse operators, damped-Jacobi smoothing,
   *   exact coarsest solve).  On x-slabs (world > 1) the fine level is
   *   slab-local, the coarse levels with > 150 k nodes are distributed over
   *   the slabs by coarsened plane ranges (ghost-plane exchanges, allreduced
   *   K-cycle dots) and the smaller ones are replicated on every rank (mg_nu
   *   == 1 only, reading M10).  EINVAL at init if the hierarchy cannot be built (fewer than 2
   *   levels, coarse Dirichlet DOFs that do not cover the fine ones: property Q
   *   of reading M4; or x-slabs with mg_nu > 1).
   * TOPO_PRECOND_AUTO (default): MG where it can be built, else Jacobi.         */
  int32_t precond;
  int32_t mg_nu;              /* damped-Jacobi sweeps before and after the coarse correction (>= 1) */
  double  mg_omega;           /* theta in (0, 2): level-l Jacobi weight w_l = theta / lam_l, lam_l the
                                 Rayleigh quotient of D^-1 A_l after 8 power steps (default 1.6:
                                 5-7 % fewer iterations than 1.4 on every BASELINE config; a
                                 breakdown lowers theta by 0.2, down to 1.2, for the rest of the
                                 run -- reading M7)                                               */
  int32_t mg_coarse_max;      /* coarsening stops at the first level with <= this many DOFs (24..8192;
                                 0 = auto: min(5000, max(1000, n_dof / 2000)))                     */
  int32_t mg_nu_deep;         /* sweeps on the small coarse levels (<= 150 000 nodes, level >= 1):
                                 0 (default) = auto: 8 when the fine grid has >= 2 M nodes (those
                                 levels cost little next to the fine level, and solving the deep
                                 coarse problem better cuts the PCG iterations by ~30 % at config
                                 4), else mg_nu;  >= 1: that many on those levels (reading M5)      */
  int32_t mg_fp32;            /* 1 (default): multigrid levels >= 1 (vectors, stencils, level-1 Galerkin
                                 operator) and the fine smoothing matvecs' element operator in fp32 --
                                 mixed precision; the PCG, its matvec and every
                                 result stay fp64.  Safety net: a breakdown of the fp32 V-cycle
                                 (indefinite preconditioner) promotes the hierarchy to fp64 for the
                                 rest of the run; none observed on the BASELINE configs or the
                                 paper protocol.  0: fp64 throughout                               */
  int32_t mg_cycle;           /* TOPO_MG_KCYCLE (default): every coarse level above the coarsest is solved
                                 by two flexible-CG steps preconditioned by its own cycle (Notay &
                                 Vassilevski's K-cycle, reading M8), and the outer PCG uses the
                                 flexible Polak-Ribiere beta (M9) -- near two-grid convergence on
                                 void-rich SIMP designs, where the V-cycle's iteration count grows
                                 with the stiffness contrast.  TOPO_MG_VCYCLE: one cycle per level,
                                 standard PCG (round-1 behaviour).  mg_nu > 1 forces the V-cycle.    */
  int32_t krylov_fp32;        /* 1: with the fp32 hierarchy on one slab, the multigrid PCG keeps its
                                 residual r and q = K p in fp32 (SURVEY §8(f) f3 "fp32 storage inside
                                 fp64 iterative refinement"): u, p and the matvec stay fp64, and the
                                 fp64 TRUE residual f - K u decides convergence -- when the fp32
                                 recursion meets cg_rtol, the true residual is checked and, if it has
                                 not, r is replaced by it and PCG restarts (iterative refinement).
                                 0 (default): fp64 r and q -- measured faster on the B200 (config 4:
                                 0.160 vs 0.167 s per SIMP iteration): the fine matvecs are issue-
                                 bound, not byte-bound, and the fp32 recursion costs restarts      */
} topo_params;

#define TOPO_MG_VCYCLE 0
#define TOPO_MG_KCYCLE 1

#define TOPO_PRECOND_JACOBI 0
#define TOPO_PRECOND_MG     1
#define TOPO_PRECOND_AUTO   2

typedef struct {
  int32_t mode;               /* TOPO_DIST_SINGLE / _NCCL / _LOOPBACK / _HOST / _SOLO       */
  int32_t rank, world;        /* NCCL: this rank, #ranks; LOOPBACK: world = #slabs          */
  int32_t device;             /* CUDA device ordinal of this rank                            */
  const uint8_t *nccl_id;     /* NCCL: 128-byte ncclUniqueId broadcast by the caller;
                                 HOST: the 128-byte id of topo_host_transport_id (same on
                                 every rank)                                                 */
} topo_dist;

typedef struct {
  int64_t iters;              /* PCG iterations of the last solve                            */
  double  rel_res;            /* recursive ||r||/||f_free|| at exit                          */
  double  true_rel_res;       /* ||f - K u||/||f_free|| recomputed at exit                   */
  double  ms;                 /* device time of the solve (CUDA events)                      */
  int32_t replacements;       /* residual replacements performed                             */
  int32_t precond;            /* preconditioner used: TOPO_PRECOND_JACOBI or TOPO_PRECOND_MG  */
  int32_t mg_levels;          /* multigrid levels (0 with Jacobi)                            */
} topo_solve_info;

typedef struct {              /* last SIMP iteration (CUDA-event ms) + cumulative counters  */
  double  ms_efield, ms_solve, ms_sens, ms_filter, ms_oc, ms_total;
  int64_t cg_iters;
  int32_t oc_passes;
  double  c, fu, volume, change, lambda;
  int64_t kernel_launches;    /* cumulative count of this library's kernel launches          */
  int64_t cg_iters_total;     /* cumulative PCG iterations                                   */
  int32_t mg_fallbacks;       /* solves where the multigrid PCG broke down and was redone with
                                 the Jacobi preconditioner (cumulative)                        */
  int32_t mg_promotions;      /* 1 once an fp32 hierarchy (mg_fp32) broke down and was promoted to
                                 fp64 for the rest of the run (that solve is redone)           */
  int32_t mg_theta_cuts;      /* breakdowns answered by lowering the smoother theta by 0.2 (down
                                 to 1.2) for the rest of the run (that solve is redone)        */
  double  ms_mg_setup;        /* multigrid setup of the last solve (part of ms_solve)          */
  int64_t host_bytes;         /* cumulative bytes of field arrays the library copied between host
                                 and device (host-pointer calls; the _d calls add nothing)     */
} topo_timings;

/* Fill defaults: BASELINE common values (E0 1, Emin 1e-9, nu 0.3, penal 3,
 * move 0.2, density filter, cg_rtol 1e-8, oc_tol 1e-10, oc_lmax 1e9). */
void topo_params_default(topo_params *p);

/* Create a context.  load: [3*n_nd] nodal forces (must be 0 on fixed DOFs).
 * fixed: [3*n_nd] 0/1 Dirichlet mask (u = 0 where 1, elimination).
 * passive: [n_el] non-design mask or NULL (reading R27):
 *   0 design element; 1 passive VOID ("obstacle": x = xPhys = 0, E = Emin);
 *   2 passive SOLID ("mandatory-solid region": x = xPhys = 1, E = E0).
 *   Passive elements stay in the FE mesh and the filter, are excluded from the
 *   update, from dv and from the volume (target = volfrac * #design elements);
 *   with the density filter the solid elements' filtered spill into design
 *   elements counts towards the design volume, so a solid region can make the
 *   target unreachable: topo_oc_step then returns TOPO_EBISECT.
 *   Any other value: EINVAL.
 * dist: NULL -> one GPU (current device).  Errors: EINVAL, EUNCONSTRAINED,
 * EALLPASSIVE, ENOMEM, ECUDA, ENCCL.  On error *out is NULL.              */
int topo_init(const topo_params *p, const double *load, const uint8_t *fixed,
              const uint8_t *passive, const topo_dist *dist, topo_ctx **out);

/* Bind the CUDA stream (cudaStream_t as void*) every later call launches
 * on.  NULL/0 -> the context's own non-blocking stream.                    */
int topo_set_stream(topo_ctx *ctx, void *stream);

/* x-slab partition without a context (host only, no GPU): rank `rank` of
 * `world` owns elements [ex_begin, ex_end) = [rank*nelx/world,
 * (rank+1)*nelx/world) (integer division) and node planes [ex_begin, ex_end)
 * plus ix = nelx on the last rank.  EINVAL if a slab would be thinner than
 * max(1, R), R = filter radius ceil(rmin)-1 (halo from one neighbour only). */
int topo_partition(int32_t nelx, double rmin, int32_t world, int32_t rank, int32_t *ex_begin,
                   int32_t *ex_end);

/* Owned element range along x of this rank: [ex_begin, ex_end).           */
int topo_owned_range(const topo_ctx *ctx, int32_t *ex_begin, int32_t *ex_end);

/* Design variables x [n_el] (host).  NULL -> volfrac on design elements.
 * Passive entries are forced to their value (0 void, 1 solid).  Sets xPhys = x (reading R#18: the first
 * iteration is unfiltered).                                                 */
int topo_set_density(topo_ctx *ctx, const double *x);

/* Set physical densities directly (xPhys, [n_el]); passive forced to 0 / 1. */
int topo_set_xphys(topo_ctx *ctx, const double *xphys);

/* Solve K(xPhys) u = f on free DOFs (PCG, matrix-free; preconditioner per
 * topo_params.precond).  Computes
 * E = Emin + xPhys^p (E0-Emin) first.  u: [3*n_nd] output or NULL.
 * Errors: ENOCONV, EBREAKDOWN (u keeps the last iterate).                   */
int topo_solve(topo_ctx *ctx, double *u, topo_solve_info *info);

/* After topo_solve: ce_e = u_e^T KE u_e, c = sum_e E_e ce_e,
 * dc_e = -p xPhys^(p-1) (E0-Emin) ce_e (0 on passive).  c: scalar out.
 * ce, dc: [n_el] or NULL.                                                   */
int topo_sensitivity(topo_ctx *ctx, double *c, double *ce, double *dc);

/* One filter application.  what = TOPO_FILTER_DC: in = raw dc [n_el] (NULL ->
 * the context's dc from topo_sensitivity), out = dc~ [n_el] or NULL; also
 * prepares dv~.  what = TOPO_FILTER_X: in = x [n_el] (NULL -> current x),
 * out = xPhys [n_el] or NULL, and the context's xPhys is replaced.          */
int topo_filter(topo_ctx *ctx, int32_t what, const double *in, double *out);

/* OC bisection on the context's x, dc~, dv~ (after topo_filter(DC)).
 * xnew: [n_el] or NULL.  Scalars: final lambda (last lmid), change =
 * max |xnew - x| over design elements, volume = mean design xPhys(xnew)
 * (mode 0) / mean design xnew (modes 1, 2).  Then x <- xnew and
 * xPhys <- filter(x).  Errors: EBISECT when no lambda can meet the target --
 * the volume with every design element at 0 (the filtered passive-solid
 * spill, density filter) already exceeds it; x is then unchanged.
 * A target that only the move limit keeps out of reach in this step is not an
 * error: xnew ends at the lower move limits (top3d behaviour).               */
int topo_oc_step(topo_ctx *ctx, double *xnew, double *lambda, double *change, double *volume);

/* The loop: n_iter x (solve, sensitivity, filter, oc).  c_hist [n_iter]
 * (compliance of the design entering each iteration), x_out [n_el] final
 * design, n_done iterations completed (partial on error).
 * change_tol > 0 stops early when change < change_tol.                      */
int topo_optimize(topo_ctx *ctx, int32_t n_iter, double change_tol, double *c_hist,
                  double *x_out, int32_t *n_done);

/* q = K(E) p with the Dirichlet mask (q = 0 on fixed DOFs, p read as 0
 * there), using the current E (topo_solve / topo_update_modulus).  Host
 * p, q: [3*n_nd].  Test / GDOF-s hook.                                      */
int topo_apply_K(topo_ctx *ctx, const double *p, double *q);

/* Recompute E (and the Jacobi diagonal) from the current xPhys.            */
int topo_update_modulus(topo_ctx *ctx);

/* Benchmark hooks (device-resident operands).  topo_matvec_load copies a
 * host p [3*n_nd] into the internal matvec operand; topo_matvec_run launches
 * `reps` back-to-back matvec kernels on the bound stream (no host sync).   */
int topo_matvec_load(topo_ctx *ctx, const double *p);
int topo_matvec_run(topo_ctx *ctx, int32_t reps);

/* Device-side checkpoint of the optimiser state (design x, xPhys and the
 * displacement u used as PCG warm start): topo_snapshot copies it into
 * context-owned backup buffers (allocated on first use), topo_restore copies
 * it back.  Used by bench.py to time the same SIMP iterations twice (device-
 * resident and end-to-end); also a cheap checkpoint/resume.                  */
int topo_snapshot(topo_ctx *ctx);
int topo_restore(topo_ctx *ctx);

/* Read a field (TOPO_FIELD_*) in external numbering.                        */
int topo_get(topo_ctx *ctx, int32_t field, double *out);

int topo_get_timings(const topo_ctx *ctx, topo_timings *t);

/* Live kernel timing inside the timed region: when enabled, the PCG driver
 * brackets one matvec launch per CUDA-graph batch with CUDA events on the
 * bound stream.  topo_kernel_time returns the mean matvec duration (ms) and
 * the number of samples since the last reset.                               */
int topo_profile(topo_ctx *ctx, int32_t enable);
int topo_kernel_time(topo_ctx *ctx, double *mean_ms, int64_t *samples);
/* Same for the fine-level matvec variants of a multigrid PCG iteration:
 * which = 0: the PCG matvec (as topo_kernel_time); 1: the V-cycle's first sweep
 * fused into the matvec (z = w D^-1 r, q = K z); 2: its last sweep fused into the
 * matvec epilogue (z + w D^-1 (r - K z), rho).                                */
int topo_kernel_time_k(topo_ctx *ctx, int32_t which, double *mean_ms, int64_t *samples);

/* The element stiffness the library uses (24x24 row-major, unit cube,
 * E = 1, 2x2x2 Gauss; "pre-computed").  No context needed.    */
int topo_element_stiffness(double nu, double *ke576);

/* Multigrid test hooks.  topo_mg_levels: *n_levels = L (0
 * if the context solves with Jacobi) and the element counts dims[3*l ..
 * 3*l+2] = (nelx_l, nely_l, nelz_l) for l < L (dims may be NULL; room for 16
 * levels).  topo_mg_apply: y = A_l x on level l (external numbering of level
 * l's grid, [3*(nelx_l+1)(nely_l+1)(nelz_l+1)], x read as 0 on fixed DOFs, y = 0
 * there), A_0 = K(E), A_{l+1} = P^T A_l P (Galerkin).  topo_mg_vcycle: z = V(b)
 * for a fine-level b [3*n_nd] (one V-cycle, the PCG preconditioner).  Both use
 * the current E (recomputed from xPhys if stale).  ESTATE without multigrid. */
int topo_mg_levels(topo_ctx *ctx, int32_t *n_levels, int32_t *dims);
int topo_mg_apply(topo_ctx *ctx, int32_t level, const double *x, double *y);
int topo_mg_vcycle(topo_ctx *ctx, const double *b, double *z);

/* Number of layout/grid facts for tests: n_dof, n_el, owned nodes, etc.    */
int64_t topo_count(const topo_ctx *ctx, int32_t what);
#define TOPO_COUNT_NDOF        0
#define TOPO_COUNT_NEL         1
#define TOPO_COUNT_NODES       2
#define TOPO_COUNT_DESIGN      3
#define TOPO_COUNT_STENCIL     4   /* filter stencil points                   */
#define TOPO_COUNT_DEVICE_BYTES 5  /* device memory held by the context        */
#define TOPO_COUNT_MG_DIST     6   /* x-slabs: multigrid levels 1..k cycled on
                                      each slab's owned planes (0: replicated) */

/* TOPO_DIST_HOST helper: a fresh 128-byte transport id (a POSIX shared-memory
 * name) that rank 0 creates and broadcasts to the other ranks.  The host
 * transport runs the same per-rank control flow as NCCL (one slab per process,
 * only owned planes) with every exchange staged through pinned host memory and
 * a process-shared barrier: stream-ordered and CUDA-graph capturable, for
 * testing the x-slab path with several processes on one GPU.  Timeouts (and
 * NCCL asynchronous errors) surface as TOPO_ENCCL after TOPO_COMM_TIMEOUT
 * seconds (env, default 300) instead of hanging.                            */
int topo_host_transport_id(uint8_t *out128);

/* NCCL mode helper: fill a 128-byte ncclUniqueId (rank 0 calls it and
 * broadcasts the bytes, e.g. with torch.distributed).  ENCCL if libnccl.so.2
 * cannot be loaded.                                                          */
int topo_nccl_unique_id(uint8_t *out128);

/* ---- _d variants: device pointers + CUDA stream (§4.1.3
 * "Python API ... as a library within larger Python projects") --------------
 * Same semantics as the host calls above, except:
 *  - every array argument is a CUDA DEVICE pointer (on the context's device) to
 *    the WHOLE external array (S:45 numbering, same lengths); multi-GPU
 *    (NCCL) ranks write only their owned planes, as with host arrays;
 *  - `stream` (a cudaStream_t as void*; NULL = the stream already bound) is
 *    bound to the context like topo_set_stream, and all work -- including the
 *    reads of inputs and the writes of outputs -- is ordered on it: a _d call
 *    can return before its outputs are written (use them in stream order), and
 *    inputs must stay valid until the stream reaches the call's work;
 *  - no field array passes through host memory (topo_timings.host_bytes does
 *    not grow); scalar results (c, lambda, change, volume, c_hist, solve info)
 *    are still host outputs, because the PCG and OC drivers poll device state;
 *  - topo_init_d copies load / fixed / passive to the host once (the partition,
 *    multigrid hierarchy and masks are set up on the host at init).
 * Errors: as the host calls, plus EINVAL for a pointer that is not device
 * memory of the context's device.                                           */
int topo_init_d(const topo_params *p, const double *load_d, const uint8_t *fixed_d,
                const uint8_t *passive_d, const topo_dist *dist, void *stream, topo_ctx **out);
int topo_set_density_d(topo_ctx *ctx, const double *x_d, void *stream);
int topo_set_xphys_d(topo_ctx *ctx, const double *xphys_d, void *stream);
int topo_solve_d(topo_ctx *ctx, double *u_d, topo_solve_info *info, void *stream);
int topo_sensitivity_d(topo_ctx *ctx, double *c, double *ce_d, double *dc_d, void *stream);
int topo_filter_d(topo_ctx *ctx, int32_t what, const double *in_d, double *out_d, void *stream);
int topo_oc_step_d(topo_ctx *ctx, double *xnew_d, double *lambda, double *change, double *volume,
                   void *stream);
int topo_optimize_d(topo_ctx *ctx, int32_t n_iter, double change_tol, double *c_hist,
                    double *x_out_d, int32_t *n_done, void *stream);
int topo_apply_K_d(topo_ctx *ctx, const double *p_d, double *q_d, void *stream);
int topo_get_d(topo_ctx *ctx, int32_t field, double *out_d, void *stream);

const char *topo_last_error(const topo_ctx *ctx);
const char *topo_strerror(int code);
const char *topo_version(void);
void topo_destroy(topo_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* TOPO_H */
