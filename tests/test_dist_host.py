"""The x-slab path with ONE PROCESS PER SLAB (north_star (3)),
through the host-staged transport TOPO_DIST_HOST: the same per-rank control
flow as the NCCL transport (each process owns one slab and only its planes;
halo exchanges, scalar allreduces, the multigrid level-1 allreduce and the
moduli all-gather go between processes), on one GPU.  NCCL itself cannot put
two ranks on one GPU; this runs everything else of the multi-process path.

Checks: the c history and design equal the in-process loopback slabs (same
partition, same fixed-order sums) and the oracle; a peer that never joins or
dies mid-run turns into TOPO_ENCCL after TOPO_COMM_TIMEOUT, not a hang."""
import multiprocessing as mp
import os
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _problem(kind, **over):
    from workloads import config_params, cantilever_load, cantilever_fixed, solid_block_passive, make_problem
    if kind == "cfg1":
        return make_problem(1, **over)
    if kind == "dist":   # 4 levels: levels 1-2 distributed over the slabs (TOPO_DIST_MIN_NODES=0)
        dims = (128, 32, 16)
        p = config_params(dict(nelx=dims[0], nely=dims[1], nelz=dims[2], volfrac=0.2, rmin=1.5, n_iter=3,
                               cg_rtol=1e-10, obstacle=None), **over)
        return p, cantilever_load(*dims), cantilever_fixed(*dims), None
    dims = (36, 12, 6)
    p = config_params(dict(nelx=dims[0], nely=dims[1], nelz=dims[2], volfrac=0.25, rmin=2.5, n_iter=5,
                           cg_rtol=1e-10, obstacle=None), **over)
    pas = solid_block_passive(*dims, (15, 21), (0, 4), (0, 6), base=(8.0, 6.0, 2.5))
    return p, cantilever_load(*dims), cantilever_fixed(*dims), pas


def _worker(rank, world, tid, kind, over, n_iter, q, die_after_init=False, timeout=None, env=None):
    try:
        os.environ.update(env or {})
        if timeout is not None:
            os.environ["TOPO_COMM_TIMEOUT"] = str(timeout)
        import torch
        torch.cuda.set_device(0)
        from paper_2504_05604_b200 import topo
        p, f, fx, pas = _problem(kind, **over)
        dist = dict(mode=topo.TOPO_DIST_HOST, rank=rank, world=world, device=0, nccl_id=tid)
        with topo.Problem(p, f, fx, pas, dist=dist) as pr:
            if die_after_init:
                os._exit(0)
            a, b = pr.owned_range()
            if env and "TOPO_DIST_MIN_NODES" in env:
                assert pr.count("mg_dist") == 2
            try:
                c, x, nd = pr.optimize(n_iter)
                q.put((rank, "ok", c.tolist(), (a, b), x, pr.timings()["cg_iters_total"]))
            except topo.TopoError as e:
                q.put((rank, "err", e.code, str(e), None, None))
    except Exception as e:   # noqa: BLE001
        code = getattr(e, "code", -1)
        q.put((rank, "exc", code, repr(e), None, None))


def _run(world, kind, over, n_iter=5, env=None, **kw):
    from paper_2504_05604_b200 import topo
    tid = topo.host_transport_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, tid, kind, over, n_iter, q),
                         kwargs=dict(kw.get("per_rank", {}).get(r, {}), env=env)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = {}
    t0 = time.time()
    while len(out) < world and time.time() - t0 < 600:
        try:
            r = q.get(timeout=5)
            out[r[0]] = r
        except Exception:   # noqa: BLE001
            if not any(p.is_alive() for p in procs) and q.empty():
                break
    for pr in procs:
        pr.join(timeout=30)
        if pr.is_alive():
            pr.kill()
    return out


def _loopback(world, kind, over, n_iter=5):
    from paper_2504_05604_b200 import topo
    p, f, fx, pas = _problem(kind, **over)
    with topo.Problem(p, f, fx, pas, dist=dict(mode=topo.TOPO_DIST_LOOPBACK, rank=0, world=world, device=0)) as pr:
        c, x, _ = pr.optimize(n_iter)
    return c, x


@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("world,kind,precond", [(2, "solid", "jacobi"), (2, "solid", "mg"), (3, "solid", "mg"),
                                                (2, "cfg1", "mg")])
def test_host_transport_matches_loopback_and_oracle(gpu, world, kind, precond):
    import oracle
    over = dict(precond=precond)
    out = _run(world, kind, over)
    assert sorted(out) == list(range(world)), out
    for r in range(world):
        assert out[r][1] == "ok", out[r]
    c0 = np.array(out[0][2])
    for r in range(1, world):
        assert np.array_equal(np.array(out[r][2]), c0)          # every rank sees the same allreduced c
    # stitch the owned slabs of the design together
    p, f, fx, pas = _problem(kind, **over)
    n_el = p["nelx"] * p["nely"] * p["nelz"]
    x = np.zeros(n_el).reshape(p["nelz"], p["nelx"], p["nely"])
    for r in range(world):
        a, b = out[r][3]
        x[:, a:b, :] = out[r][4].reshape(p["nelz"], p["nelx"], p["nely"])[:, a:b, :]
    cl, xl = _loopback(world, kind, over)
    np.testing.assert_allclose(c0, cl, rtol=1e-12, atol=0)
    np.testing.assert_allclose(x.ravel(), xl, rtol=0, atol=1e-12)
    ro = oracle.run_optimization(p, f, fx, pas, n_iter=5)
    assert np.max(np.abs(c0 - ro["c"]) / ro["c"]) <= 1e-6


@pytest.mark.parametrize("world", [2, 4])
def test_host_transport_distributed_levels(gpu, monkeypatch, world):
    """Multigrid levels 1-2 distributed over one process per slab (ghost-plane
    exchanges, K-cycle dot allreduces and the level-3 all-gather through the
    host transport): c history and design equal the loopback slabs (same
    partition) to 1e-12 and the single slab to 1e-9."""
    from paper_2504_05604_b200 import topo
    env = {"TOPO_DIST_MIN_NODES": "0"}
    over = dict(precond="mg")
    out = _run(world, "dist", over, n_iter=3, env=env)
    assert sorted(out) == list(range(world)), out
    for r in range(world):
        assert out[r][1] == "ok", out[r]
    c0 = np.array(out[0][2])
    p, f, fx, pas = _problem("dist", **over)
    x = np.zeros(p["nelx"] * p["nely"] * p["nelz"]).reshape(p["nelz"], p["nelx"], p["nely"])
    for r in range(world):
        a, b = out[r][3]
        x[:, a:b, :] = out[r][4].reshape(p["nelz"], p["nelx"], p["nely"])[:, a:b, :]
    monkeypatch.setenv("TOPO_DIST_MIN_NODES", "0")
    cl, xl = _loopback(world, "dist", over, n_iter=3)
    np.testing.assert_allclose(c0, cl, rtol=1e-12, atol=0)
    np.testing.assert_allclose(x.ravel(), xl, rtol=0, atol=1e-12)
    with topo.Problem(p, f, fx, pas) as pr:
        c1, x1, _ = pr.optimize(3)
    assert np.max(np.abs(c0 - c1) / c1) <= 1e-9


def test_host_transport_peer_never_joins(gpu):
    """world = 2 but only rank 0 starts: init fails with TOPO_ENCCL after the timeout."""
    from paper_2504_05604_b200 import topo
    tid = topo.host_transport_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pr = ctx.Process(target=_worker, args=(0, 2, tid, "solid", dict(precond="jacobi"), 1, q), kwargs=dict(timeout=4))
    t0 = time.time()
    pr.start()
    r = q.get(timeout=120)
    pr.join(timeout=30)
    assert r[1] in ("exc", "err") and r[2] == topo.TOPO_ENCCL, r
    assert time.time() - t0 < 100


def test_host_transport_peer_dies(gpu):
    """rank 1 exits right after init: rank 0's first exchange times out and the
    solve returns TOPO_ENCCL instead of hanging."""
    from paper_2504_05604_b200 import topo
    out = _run(2, "solid", dict(precond="jacobi"), n_iter=2,
               per_rank={0: dict(timeout=5), 1: dict(die_after_init=True, timeout=5)})
    assert 0 in out and out[0][1] == "err" and out[0][2] == topo.TOPO_ENCCL, out
