"""Multi-process (world_size 2 and 4, gloo, CPU) checks of the x-slab host
logic: every rank computes its slab with the library's host-only partition,
the ranks allgather the ranges and check they tile [0, nelx) exactly once;
the NCCL-id broadcast used by bench.py is exercised with gloo."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nelx, rmin, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_05604_b200 import topo
    a, b = topo.partition(nelx, rmin, world, rank)
    t = torch.tensor([a, b], dtype=torch.int64)
    out = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(out, t)
    obj = [bytes(range(128)) if rank == 0 else None]      # stands in for ncclGetUniqueId bytes
    dist.broadcast_object_list(obj, src=0)
    if rank == 0:
        q.put(([tuple(x.tolist()) for x in out], obj[0]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,nelx,rmin", [(2, 512, 3.0), (4, 512, 3.0), (2, 37, 2.5), (4, 9, 1.5)])
def test_partition_tiles_domain(world, nelx, rmin):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nelx, rmin, q)) for r in range(world)]
    for p in procs:
        p.start()
    ranges, idbytes = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ranges[0][0] == 0 and ranges[-1][1] == nelx
    for (a0, b0), (a1, b1) in zip(ranges, ranges[1:]):
        assert b0 == a1 and b0 > a0
    assert idbytes == bytes(range(128))


def test_partition_rejects_thin_slabs():
    from paper_2504_05604_b200 import topo
    with pytest.raises(topo.TopoError):
        topo.partition(8, 4.0, 4, 0)        # slabs of 2 planes < R = 3
    assert topo.partition(8, 1.5, 8, 7) == (7, 8)
