"""Thin ctypes binding of libtopo (include/topo.h).  Argument marshalling only:
every step of the hot path runs in the CUDA kernels of libtopo.so.  There is
no CPU fallback -- importing this module without the built library raises.

Functions keep the C names (topo_init, topo_solve, ...); `Problem` is a small
convenience wrapper around one context.
"""
import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtopo.so")

# ---- constants (mirror include/topo.h) --------------------------------------
TOPO_OK, TOPO_EINVAL, TOPO_ENOCONV, TOPO_EBREAKDOWN, TOPO_EUNCONSTRAINED = 0, 1, 2, 3, 4
TOPO_EBISECT, TOPO_EALLPASSIVE, TOPO_ECUDA, TOPO_ENCCL, TOPO_ENOMEM, TOPO_ESTATE = 5, 6, 7, 8, 9, 10
TOPO_FILTER_DENSITY, TOPO_FILTER_SENSITIVITY, TOPO_FILTER_PLAIN = 0, 1, 2
TOPO_FILTER_X, TOPO_FILTER_DC = 0, 1
FIELDS = dict(u=0, x=1, xphys=2, E=3, ce=4, dc=5, dcf=6, dvf=7, xnew=8, hs=9, invdiag=10, r=11)
NODE_FIELDS = {"u", "invdiag", "r"}
TOPO_DIST_SINGLE, TOPO_DIST_NCCL, TOPO_DIST_LOOPBACK, TOPO_DIST_HOST, TOPO_DIST_SOLO = 0, 1, 2, 3, 4
TOPO_PRECOND_JACOBI, TOPO_PRECOND_MG, TOPO_PRECOND_AUTO = 0, 1, 2
PRECOND = dict(jacobi=0, mg=1, auto=2)
COUNTS = dict(ndof=0, nel=1, nodes=2, design=3, stencil=4, device_bytes=5, mg_dist=6)

# Every symbol include/topo.h declares (checked by tests/test_abi.py).
EXPORTS = ["topo_params_default", "topo_init", "topo_set_stream", "topo_owned_range",
           "topo_set_density", "topo_set_xphys", "topo_solve", "topo_sensitivity", "topo_filter",
           "topo_oc_step", "topo_optimize", "topo_apply_K", "topo_update_modulus",
           "topo_matvec_load", "topo_matvec_run", "topo_get", "topo_get_timings", "topo_profile",
           "topo_kernel_time", "topo_element_stiffness", "topo_count", "topo_last_error",
           "topo_strerror", "topo_version", "topo_destroy", "topo_nccl_unique_id", "topo_partition", "topo_snapshot", "topo_restore",
           "topo_mg_levels", "topo_mg_apply", "topo_mg_vcycle", "topo_kernel_time_k",
           # _d variants: device pointers + cudaStream_t
           "topo_init_d", "topo_set_density_d", "topo_set_xphys_d", "topo_solve_d",
           "topo_sensitivity_d", "topo_filter_d", "topo_oc_step_d", "topo_optimize_d",
           "topo_apply_K_d", "topo_get_d", "topo_host_transport_id"]


class topo_params(C.Structure):
    _fields_ = [("nelx", C.c_int32), ("nely", C.c_int32), ("nelz", C.c_int32),
                ("volfrac", C.c_double), ("penal", C.c_double), ("rmin", C.c_double),
                ("E0", C.c_double), ("Emin", C.c_double), ("nu", C.c_double), ("move", C.c_double),
                ("filter_mode", C.c_int32), ("cg_rtol", C.c_double), ("cg_max_iter", C.c_int64),
                ("cg_warm_start", C.c_int32), ("oc_tol", C.c_double), ("oc_lmax", C.c_double),
                ("deterministic", C.c_int32), ("cg_check_every", C.c_int32),
                ("precond", C.c_int32), ("mg_nu", C.c_int32), ("mg_omega", C.c_double),
                ("mg_coarse_max", C.c_int32), ("mg_nu_deep", C.c_int32), ("mg_fp32", C.c_int32),
                ("mg_cycle", C.c_int32), ("krylov_fp32", C.c_int32)]


class topo_dist(C.Structure):
    _fields_ = [("mode", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32),
                ("device", C.c_int32), ("nccl_id", C.POINTER(C.c_uint8))]


class topo_solve_info(C.Structure):
    _fields_ = [("iters", C.c_int64), ("rel_res", C.c_double), ("true_rel_res", C.c_double),
                ("ms", C.c_double), ("replacements", C.c_int32), ("precond", C.c_int32),
                ("mg_levels", C.c_int32)]


class topo_timings(C.Structure):
    _fields_ = [("ms_efield", C.c_double), ("ms_solve", C.c_double), ("ms_sens", C.c_double),
                ("ms_filter", C.c_double), ("ms_oc", C.c_double), ("ms_total", C.c_double),
                ("cg_iters", C.c_int64), ("oc_passes", C.c_int32), ("c", C.c_double),
                ("fu", C.c_double), ("volume", C.c_double), ("change", C.c_double),
                ("lambda_", C.c_double), ("kernel_launches", C.c_int64),
                ("cg_iters_total", C.c_int64), ("mg_fallbacks", C.c_int32),
                ("mg_promotions", C.c_int32), ("mg_theta_cuts", C.c_int32), ("ms_mg_setup", C.c_double),
                ("host_bytes", C.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2504_05604_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, D, I, VP = C.POINTER, C.POINTER(C.c_double), C.c_int, C.c_void_p
    U8 = P(C.c_uint8)
    ctxp = C.c_void_p
    sig = {
        "topo_params_default": (None, [P(topo_params)]),
        "topo_init": (I, [P(topo_params), D, U8, U8, P(topo_dist), P(ctxp)]),
        "topo_set_stream": (I, [ctxp, VP]),
        "topo_owned_range": (I, [ctxp, P(C.c_int32), P(C.c_int32)]),
        "topo_set_density": (I, [ctxp, D]),
        "topo_set_xphys": (I, [ctxp, D]),
        "topo_solve": (I, [ctxp, D, P(topo_solve_info)]),
        "topo_sensitivity": (I, [ctxp, D, D, D]),
        "topo_filter": (I, [ctxp, C.c_int32, D, D]),
        "topo_oc_step": (I, [ctxp, D, D, D, D]),
        "topo_optimize": (I, [ctxp, C.c_int32, C.c_double, D, D, P(C.c_int32)]),
        "topo_apply_K": (I, [ctxp, D, D]),
        "topo_update_modulus": (I, [ctxp]),
        "topo_matvec_load": (I, [ctxp, D]),
        "topo_matvec_run": (I, [ctxp, C.c_int32]),
        "topo_get": (I, [ctxp, C.c_int32, D]),
        "topo_get_timings": (I, [ctxp, P(topo_timings)]),
        "topo_profile": (I, [ctxp, C.c_int32]),
        "topo_kernel_time": (I, [ctxp, D, P(C.c_int64)]),
        "topo_element_stiffness": (I, [C.c_double, D]),
        "topo_count": (C.c_int64, [ctxp, C.c_int32]),
        "topo_last_error": (C.c_char_p, [ctxp]),
        "topo_strerror": (C.c_char_p, [I]),
        "topo_version": (C.c_char_p, []),
        "topo_destroy": (None, [ctxp]),
        "topo_nccl_unique_id": (I, [U8]),
        "topo_host_transport_id": (I, [U8]),
        "topo_snapshot": (I, [ctxp]),
        "topo_restore": (I, [ctxp]),
        "topo_partition": (I, [C.c_int32, C.c_double, C.c_int32, C.c_int32, P(C.c_int32), P(C.c_int32)]),
        "topo_mg_levels": (I, [ctxp, P(C.c_int32), P(C.c_int32)]),
        "topo_mg_apply": (I, [ctxp, C.c_int32, D, D]),
        "topo_mg_vcycle": (I, [ctxp, D, D]),
        "topo_kernel_time_k": (I, [ctxp, C.c_int32, D, P(C.c_int64)]),
        "topo_init_d": (I, [P(topo_params), VP, VP, VP, P(topo_dist), VP, P(ctxp)]),
        "topo_set_density_d": (I, [ctxp, VP, VP]),
        "topo_set_xphys_d": (I, [ctxp, VP, VP]),
        "topo_solve_d": (I, [ctxp, VP, P(topo_solve_info), VP]),
        "topo_sensitivity_d": (I, [ctxp, D, VP, VP, VP]),
        "topo_filter_d": (I, [ctxp, C.c_int32, VP, VP, VP]),
        "topo_oc_step_d": (I, [ctxp, VP, D, D, D, VP]),
        "topo_optimize_d": (I, [ctxp, C.c_int32, C.c_double, D, VP, P(C.c_int32), VP]),
        "topo_apply_K_d": (I, [ctxp, VP, VP, VP]),
        "topo_get_d": (I, [ctxp, C.c_int32, VP, VP]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = _load()
globals().update({n: getattr(_lib, n) for n in EXPORTS})


class TopoError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_lib.topo_strerror(code).decode()} ({code}): {msg}")
        self.code = code


def _dp(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def _u8(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_uint8))


def _devptr(t, n, dtype="float64", what="array"):
    """Device pointer of a CUDA tensor-like object (torch.Tensor: .data_ptr(),
    .is_cuda, .dtype, .numel(), .is_contiguous()); None -> NULL.  Marshalling
    only: checks that the buffer is a contiguous CUDA array of n elements."""
    if t is None:
        return None
    if not getattr(t, "is_cuda", False):
        raise TopoError(TOPO_EINVAL, f"{what}: expected a CUDA tensor")
    if str(t.dtype).split(".")[-1] != dtype or t.numel() != n or not t.is_contiguous():
        raise TopoError(TOPO_EINVAL, f"{what}: expected a contiguous {dtype} CUDA tensor of {n} elements, got "
                                     f"{t.dtype} {tuple(t.shape)}")
    return C.c_void_p(t.data_ptr())


def _stream(stream):
    """cudaStream_t from a torch.cuda.Stream, an int handle or None (bound stream)."""
    if stream is None:
        return None
    return C.c_void_p(int(getattr(stream, "cuda_stream", stream)))


def element_stiffness(nu):
    out = np.zeros(576)
    rc = _lib.topo_element_stiffness(float(nu), _dp(out))
    if rc:
        raise TopoError(rc, "topo_element_stiffness")
    return out.reshape(24, 24)


def nccl_unique_id():
    buf = np.zeros(128, dtype=np.uint8)
    rc = _lib.topo_nccl_unique_id(_u8(buf))
    if rc:
        raise TopoError(rc, "topo_nccl_unique_id")
    return bytes(buf)


def host_transport_id():
    """128-byte id of a fresh host-staged transport (TOPO_DIST_HOST); rank 0
    creates it and passes it to every rank as dist["nccl_id"]."""
    buf = np.zeros(128, dtype=np.uint8)
    rc = _lib.topo_host_transport_id(_u8(buf))
    if rc:
        raise TopoError(rc, "topo_host_transport_id")
    return bytes(buf)


def partition(nelx, rmin, world, rank):
    """Owned element range [ex0, ex1) of `rank` (host-only, no GPU)."""
    a, b = C.c_int32(), C.c_int32()
    rc = _lib.topo_partition(int(nelx), float(rmin), int(world), int(rank), C.byref(a), C.byref(b))
    if rc:
        raise TopoError(rc, "topo_partition")
    return a.value, b.value


def make_params(p):
    """topo_params from a dict (keys as in workloads.config_params)."""
    prm = topo_params()
    _lib.topo_params_default(C.byref(prm))
    for k in ("nelx", "nely", "nelz", "filter_mode", "cg_warm_start", "deterministic",
              "cg_check_every", "mg_nu", "mg_coarse_max", "mg_nu_deep", "mg_fp32", "krylov_fp32"):
        if k in p:
            setattr(prm, k, int(p[k]))
    if "mg_cycle" in p:
        prm.mg_cycle = {"V": 0, "K": 1}.get(p["mg_cycle"], p["mg_cycle"]) if isinstance(p["mg_cycle"], str) \
            else int(p["mg_cycle"])
    if "precond" in p:
        prm.precond = PRECOND[p["precond"]] if isinstance(p["precond"], str) else int(p["precond"])
    for k in ("volfrac", "penal", "rmin", "E0", "Emin", "nu", "move", "cg_rtol", "oc_tol", "oc_lmax",
              "mg_omega"):
        if k in p:
            setattr(prm, k, float(p[k]))
    if "cg_max_iter" in p:
        prm.cg_max_iter = int(p["cg_max_iter"])
    return prm


class Problem:
    """One topo context.  Host arrays in external numbering (topo.h)."""

    def __init__(self, params, load, fixed, passive=None, dist=None, stream=None):
        """load/fixed/passive: host arrays (numpy), or CUDA tensors -> topo_init_d."""
        self.p = dict(params)
        self.prm = make_params(self.p)
        self.nelx, self.nely, self.nelz = self.prm.nelx, self.prm.nely, self.prm.nelz
        self.n_el = self.nelx * self.nely * self.nelz
        self.n_nd = (self.nelx + 1) * (self.nely + 1) * (self.nelz + 1)
        on_dev = getattr(load, "is_cuda", False)
        if not on_dev:
            load = np.ascontiguousarray(load, dtype=np.float64)
            fixed = np.ascontiguousarray(fixed, dtype=np.uint8)
            passive = None if passive is None else np.ascontiguousarray(passive, dtype=np.uint8)
        if not on_dev and min(self.nelx, self.nely, self.nelz) >= 1 and (
                load.size != 3 * self.n_nd or fixed.size != 3 * self.n_nd
                or (passive is not None and passive.size != self.n_el)):
            raise TopoError(TOPO_EINVAL, "array sizes do not match the grid")
        self._ctx = C.c_void_p()
        dptr = None
        self._id = None
        if dist is not None:
            d = topo_dist()
            d.mode, d.rank, d.world, d.device = (int(dist.get("mode", 0)), int(dist.get("rank", 0)),
                                                 int(dist.get("world", 1)), int(dist.get("device", 0)))
            if dist.get("nccl_id") is not None:
                self._id = np.frombuffer(bytes(dist["nccl_id"]), dtype=np.uint8).copy()
                d.nccl_id = _u8(self._id)
            dptr = C.byref(d)
        if on_dev:
            rc = _lib.topo_init_d(C.byref(self.prm), _devptr(load, 3 * self.n_nd, what="load"),
                                  _devptr(fixed, 3 * self.n_nd, "uint8", "fixed"),
                                  _devptr(passive, self.n_el, "uint8", "passive"), dptr, _stream(stream),
                                  C.byref(self._ctx))
        else:
            rc = _lib.topo_init(C.byref(self.prm), _dp(load), _u8(fixed), _u8(passive), dptr,
                                C.byref(self._ctx))
        if rc:
            raise TopoError(rc, "topo_init")

    # -- helpers --
    def _check(self, rc, what):
        if rc:
            raise TopoError(rc, f"{what}: {_lib.topo_last_error(self._ctx).decode()}")

    def close(self):
        if self._ctx:
            _lib.topo_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- API --
    def set_stream(self, stream_handle):
        self._check(_lib.topo_set_stream(self._ctx, C.c_void_p(int(stream_handle or 0))),
                    "topo_set_stream")

    def owned_range(self):
        a, b = C.c_int32(), C.c_int32()
        self._check(_lib.topo_owned_range(self._ctx, C.byref(a), C.byref(b)), "topo_owned_range")
        return a.value, b.value

    def set_density(self, x=None):
        x = None if x is None else np.ascontiguousarray(x, dtype=np.float64)
        self._check(_lib.topo_set_density(self._ctx, _dp(x)), "topo_set_density")

    def set_xphys(self, xphys):
        xphys = np.ascontiguousarray(xphys, dtype=np.float64)
        self._check(_lib.topo_set_xphys(self._ctx, _dp(xphys)), "topo_set_xphys")

    def solve(self, want_u=True, u_out=None):
        u = u_out if u_out is not None else (np.zeros(3 * self.n_nd) if want_u else None)
        info = topo_solve_info()
        self._check(_lib.topo_solve(self._ctx, _dp(u), C.byref(info)), "topo_solve")
        return u, dict(iters=info.iters, rel_res=info.rel_res, true_rel_res=info.true_rel_res,
                       ms=info.ms, replacements=info.replacements,
                       precond={0: "jacobi", 1: "mg"}[info.precond], mg_levels=info.mg_levels)

    def sensitivity(self, want=True):
        c = C.c_double()
        ce = np.zeros(self.n_el) if want else None
        dc = np.zeros(self.n_el) if want else None
        self._check(_lib.topo_sensitivity(self._ctx, C.byref(c), _dp(ce), _dp(dc)), "topo_sensitivity")
        return c.value, ce, dc

    def filter(self, what, inp=None, want=True):
        inp = None if inp is None else np.ascontiguousarray(inp, dtype=np.float64)
        out = np.zeros(self.n_el) if want else None
        w = TOPO_FILTER_DC if what in ("dc", TOPO_FILTER_DC) else TOPO_FILTER_X
        self._check(_lib.topo_filter(self._ctx, w, _dp(inp), _dp(out)), "topo_filter")
        return out

    def oc_step(self, want=True):
        xnew = np.zeros(self.n_el) if want else None
        lam, chg, vol = C.c_double(), C.c_double(), C.c_double()
        self._check(_lib.topo_oc_step(self._ctx, _dp(xnew), C.byref(lam), C.byref(chg),
                                      C.byref(vol)), "topo_oc_step")
        return xnew, lam.value, chg.value, vol.value

    def optimize(self, n_iter, change_tol=0.0, x_out=None, want_x=True):
        """n_iter SIMP iterations; returns (c history, x or None, iterations done).
        want_x=False skips the design download (x stays in HBM)."""
        c_hist = np.zeros(n_iter)
        x = x_out if x_out is not None else (np.zeros(self.n_el) if want_x else None)
        nd = C.c_int32()
        self._check(_lib.topo_optimize(self._ctx, int(n_iter), float(change_tol), _dp(c_hist),
                                       _dp(x) if x is not None else None, C.byref(nd)), "topo_optimize")
        return c_hist[:nd.value], x, nd.value

    def apply_K(self, p):
        p = np.ascontiguousarray(p, dtype=np.float64)
        q = np.zeros(3 * self.n_nd)
        self._check(_lib.topo_apply_K(self._ctx, _dp(p), _dp(q)), "topo_apply_K")
        return q

    def update_modulus(self):
        self._check(_lib.topo_update_modulus(self._ctx), "topo_update_modulus")

    def matvec_load(self, p):
        p = np.ascontiguousarray(p, dtype=np.float64)
        self._check(_lib.topo_matvec_load(self._ctx, _dp(p)), "topo_matvec_load")

    def matvec_run(self, reps=1):
        self._check(_lib.topo_matvec_run(self._ctx, int(reps)), "topo_matvec_run")

    def snapshot(self):
        self._check(_lib.topo_snapshot(self._ctx), "topo_snapshot")

    def restore(self):
        self._check(_lib.topo_restore(self._ctx), "topo_restore")

    def get(self, field):
        n = 3 * self.n_nd if field in NODE_FIELDS else self.n_el
        out = np.zeros(n)
        self._check(_lib.topo_get(self._ctx, FIELDS[field], _dp(out)), f"topo_get({field})")
        return out

    def timings(self):
        t = topo_timings()
        self._check(_lib.topo_get_timings(self._ctx, C.byref(t)), "topo_get_timings")
        d = {k: getattr(t, k) for k, _ in topo_timings._fields_}
        d["lambda"] = d.pop("lambda_")
        return d

    def profile(self, enable=True):
        self._check(_lib.topo_profile(self._ctx, int(bool(enable))), "topo_profile")

    def kernel_time(self):
        m, n = C.c_double(), C.c_int64()
        self._check(_lib.topo_kernel_time(self._ctx, C.byref(m), C.byref(n)), "topo_kernel_time")
        return m.value, n.value

    def mg_levels(self):
        """[(nelx_l, nely_l, nelz_l)] of the multigrid hierarchy ([] with Jacobi)."""
        n = C.c_int32()
        dims = np.zeros(48, dtype=np.int32)
        self._check(_lib.topo_mg_levels(self._ctx, C.byref(n),
                                        dims.ctypes.data_as(C.POINTER(C.c_int32))), "topo_mg_levels")
        return [tuple(int(v) for v in dims[3 * l:3 * l + 3]) for l in range(n.value)]

    def mg_apply(self, level, x):
        """y = A_level x on multigrid level `level` (external numbering of that grid)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros_like(x)
        self._check(_lib.topo_mg_apply(self._ctx, int(level), _dp(x), _dp(y)), "topo_mg_apply")
        return y

    def mg_vcycle(self, b):
        """z = V(b): one multigrid V-cycle on a fine-level vector."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        z = np.zeros(3 * self.n_nd)
        self._check(_lib.topo_mg_vcycle(self._ctx, _dp(b), _dp(z)), "topo_mg_vcycle")
        return z

    def kernel_time_k(self, which):
        """(mean ms, samples) of matvec variant `which` (0 PCG, 1 MG pre-sweep, 2 MG post-sweep)."""
        m, n = C.c_double(), C.c_int64()
        self._check(_lib.topo_kernel_time_k(self._ctx, int(which), C.byref(m), C.byref(n)),
                    "topo_kernel_time_k")
        return m.value, n.value

    def count(self, what):
        return int(_lib.topo_count(self._ctx, COUNTS[what]))

    # -- _d variants: CUDA tensors in / out (external numbering, whole arrays),
    #    work ordered on `stream` (torch.cuda.Stream, handle or None = bound) --
    def set_density_d(self, x=None, stream=None):
        self._check(_lib.topo_set_density_d(self._ctx, _devptr(x, self.n_el, what="x"), _stream(stream)),
                    "topo_set_density_d")

    def set_xphys_d(self, xphys, stream=None):
        self._check(_lib.topo_set_xphys_d(self._ctx, _devptr(xphys, self.n_el, what="xphys"), _stream(stream)),
                    "topo_set_xphys_d")

    def solve_d(self, u=None, stream=None):
        info = topo_solve_info()
        self._check(_lib.topo_solve_d(self._ctx, _devptr(u, 3 * self.n_nd, what="u"), C.byref(info),
                                      _stream(stream)), "topo_solve_d")
        return dict(iters=info.iters, rel_res=info.rel_res, true_rel_res=info.true_rel_res, ms=info.ms,
                    replacements=info.replacements, precond={0: "jacobi", 1: "mg"}[info.precond],
                    mg_levels=info.mg_levels)

    def sensitivity_d(self, ce=None, dc=None, stream=None):
        c = C.c_double()
        self._check(_lib.topo_sensitivity_d(self._ctx, C.byref(c), _devptr(ce, self.n_el, what="ce"),
                                            _devptr(dc, self.n_el, what="dc"), _stream(stream)),
                    "topo_sensitivity_d")
        return c.value

    def filter_d(self, what, inp=None, out=None, stream=None):
        w = TOPO_FILTER_DC if what in ("dc", TOPO_FILTER_DC) else TOPO_FILTER_X
        self._check(_lib.topo_filter_d(self._ctx, w, _devptr(inp, self.n_el, what="in"),
                                       _devptr(out, self.n_el, what="out"), _stream(stream)), "topo_filter_d")

    def oc_step_d(self, xnew=None, stream=None):
        lam, chg, vol = C.c_double(), C.c_double(), C.c_double()
        self._check(_lib.topo_oc_step_d(self._ctx, _devptr(xnew, self.n_el, what="xnew"), C.byref(lam),
                                        C.byref(chg), C.byref(vol), _stream(stream)), "topo_oc_step_d")
        return lam.value, chg.value, vol.value

    def optimize_d(self, n_iter, x_out=None, change_tol=0.0, stream=None):
        c_hist = np.zeros(n_iter)
        nd = C.c_int32()
        self._check(_lib.topo_optimize_d(self._ctx, int(n_iter), float(change_tol), _dp(c_hist),
                                         _devptr(x_out, self.n_el, what="x_out"), C.byref(nd),
                                         _stream(stream)), "topo_optimize_d")
        return c_hist[:nd.value], nd.value

    def apply_K_d(self, p, q, stream=None):
        self._check(_lib.topo_apply_K_d(self._ctx, _devptr(p, 3 * self.n_nd, what="p"),
                                        _devptr(q, 3 * self.n_nd, what="q"), _stream(stream)), "topo_apply_K_d")

    def get_d(self, field, out, stream=None):
        n = 3 * self.n_nd if field in NODE_FIELDS else self.n_el
        self._check(_lib.topo_get_d(self._ctx, FIELDS[field], _devptr(out, n, what=field), _stream(stream)),
                    f"topo_get_d({field})")
