"""The _d ABI variants (device pointers + cudaStream_t; SURVEY §8(b)
§4.1.3 "as a library within larger Python projects"): torch CUDA tensors in and
out, work on a caller-owned torch stream, and NO field array through host
memory (topo_timings.host_bytes stays constant).  Results must equal the host
API's bit for bit (same kernels, same order) and the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from workloads import make_problem, random_density, random_vector, solid_block_passive  # noqa: E402
import oracle  # noqa: E402


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_05604_b200 import topo as t
    return t, torch


def _host_run(topo, p, f, fx, pas, x, dist=None):
    with topo.Problem(p, f, fx, pas, dist=dist) as pr:
        pr.set_density(x)
        u, info = pr.solve()
        c, ce, dc = pr.sensitivity()
        dcf = pr.filter("dc")
        xnew, lam, chg, vol = pr.oc_step()
        xphys = pr.get("xphys")
        q = pr.apply_K(random_vector(3 * pr.n_nd, seed=1))
        chist, xo, _ = pr.optimize(3)
    return dict(u=u, c=c, ce=ce, dc=dc, dcf=dcf, xnew=xnew, lam=lam, xphys=xphys, q=q, chist=chist, xo=xo)


@pytest.mark.parametrize("world", [1, 2])
def test_device_api_equals_host_api(env, world):
    topo, torch = env
    p, f, fx, _ = make_problem(1)
    dims = (p["nelx"], p["nely"], p["nelz"])
    pas = solid_block_passive(*dims, (40, 46), (0, 4), (0, 4), base=(30.0, 10.0, 3.0))
    n_el = int(np.prod(dims))
    x = random_density(n_el, seed=7, lo=0.05, hi=0.5)
    dist = None if world == 1 else dict(mode=topo.TOPO_DIST_LOOPBACK, rank=0, world=world, device=0)
    ref = _host_run(topo, p, f, fx, pas, x, dist)
    dev = torch.device("cuda:0")
    T = lambda a, dt=torch.float64: torch.as_tensor(np.ascontiguousarray(a)).to(dev, dt)  # noqa: E731
    f_t, fx_t, pas_t, x_t = T(f), T(fx, torch.uint8), T(pas, torch.uint8), T(x)
    n_nd = f.size // 3
    torch.cuda.synchronize()          # inputs were written on the default stream
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with topo.Problem(p, f_t, fx_t, pas_t, dist=dist, stream=s) as pr:
            hb0 = pr.timings()["host_bytes"]
            u_t = torch.empty(3 * n_nd, dtype=torch.float64, device=dev)
            ce_t, dc_t, dcf_t, xn_t, xp_t = (torch.empty(n_el, dtype=torch.float64, device=dev) for _ in range(5))
            pr.set_density_d(x_t, stream=s)
            info = pr.solve_d(u_t, stream=s)
            c = pr.sensitivity_d(ce_t, dc_t, stream=s)
            pr.filter_d("dc", None, dcf_t, stream=s)
            lam, chg, vol = pr.oc_step_d(xn_t, stream=s)
            pr.get_d("xphys", xp_t, stream=s)
            q_t = torch.empty(3 * n_nd, dtype=torch.float64, device=dev)
            pr.apply_K_d(T(random_vector(3 * n_nd, seed=1)), q_t, stream=s)
            xo_t = torch.empty(n_el, dtype=torch.float64, device=dev)
            chist, nd = pr.optimize_d(3, xo_t, stream=s)
            assert pr.timings()["host_bytes"] == hb0      # no field array through host memory
        s.synchronize()
    assert info["true_rel_res"] <= p["cg_rtol"]
    out = dict(u=u_t, ce=ce_t, dc=dc_t, dcf=dcf_t, xnew=xn_t, xphys=xp_t, q=q_t, xo=xo_t)
    for k, t in out.items():
        assert np.array_equal(t.cpu().numpy(), ref[k]), k
    assert c == ref["c"] and lam == ref["lam"] and np.array_equal(chist, ref["chist"])
    # and the oracle (one SIMP step on identical inputs)
    H, Hs = oracle.filter_matrix(*dims, p["rmin"])
    dcf_o = oracle.apply_filter(H, Hs, 0, "dc", ref["dc"])
    assert np.allclose(dcf_t.cpu().numpy(), dcf_o, rtol=1e-9, atol=1e-9 * np.abs(dcf_o).max())


def test_device_api_rejects_host_pointer(env):
    topo, torch = env
    p, f, fx, _ = make_problem(0)
    import ctypes as C
    with topo.Problem(p, f, fx) as pr:
        host = np.zeros(pr.n_el)
        rc = topo._lib.topo_get_d(pr._ctx, topo.FIELDS["x"], C.c_void_p(host.ctypes.data), None)
        assert rc == topo.TOPO_EINVAL
        with pytest.raises(topo.TopoError):
            pr.get_d("x", torch.zeros(pr.n_el, dtype=torch.float32, device="cuda:0"))
