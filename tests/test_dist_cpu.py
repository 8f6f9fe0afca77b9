"""World-size-2 gloo tests (CPU) of the multi-GPU setup path
(paper_1104_1824_b200/dist.py): the NCCL unique id created by libsnp.so on
rank 0 reaches every rank through torch.distributed (the one host exchange
outside the levels), and the level-0 partition.  The per-level protocol runs
inside libsnp.so (tests/test_gpu_dist.py)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1104_1824_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        uid = D.broadcast_unique_id()
        assert isinstance(uid, bytes) and len(uid) == 128
        got = [None] * world
        dist.all_gather_object(got, uid)
        assert all(g == uid for g in got)            # every rank holds rank 0's id
        assert any(uid)                               # a real id, not zeros
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as ex:  # report to the parent
        q.put((rank, repr(ex)))


@pytest.mark.parametrize("world", [2])
def test_gloo_unique_id_broadcast(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: "ok" for r in range(world)}


def test_level0_slices_partition():
    for F0 in (1, 7, 64, 1000, 4194304):
        for P in (1, 2, 3, 8):
            cuts = [D.level0_slice(F0, r, P) for r in range(P)]
            assert cuts[0][0] == 0 and cuts[-1][1] == F0
            assert all(cuts[r][1] == cuts[r + 1][0] for r in range(P - 1))
