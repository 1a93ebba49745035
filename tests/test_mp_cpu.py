"""Host-side multi-process logic on CPU (gloo, world_size 2), no GPU:
the NCCL unique-id rendezvous through torch.distributed, bench.py's max-over-ranks
timing reduction and topology selection, and the schedule staying in lockstep
across ranks (every rank must issue the same collective sequence)."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import paper_2104_05588_b200 as daso
    uid = daso.rendezvous_unique_id()
    t = bench.max_over_ranks(float(rank + 1) * 1.5, world)

    class A:
        topology = ""
    topo = bench.topology(A(), world)
    sched = daso.Schedule(4, 1, 1, 1, 6, 8, 2)
    recs = [sched.next(1 if k % 8 == 0 else 0) for k in range(48)]
    q.put((rank, uid, t, topo, recs))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_rendezvous_and_timing():
    world, port = 2, _port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, uid0, t0, topo0, rec0), (_, uid1, t1, topo1, rec1) = out
    assert uid0 == uid1 and len(uid0) == 128            # one NCCL id for the whole world
    assert t0 == t1 == 3.0                                # max over ranks
    assert topo0 == topo1 == (2, 1)                       # N=2 -> 2 virtual nodes x 1 GPU
    assert rec0 == rec1                                   # schedules in lockstep
