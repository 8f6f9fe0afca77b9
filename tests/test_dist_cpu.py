"""World-size-2 gloo tests (CPU) of the multi-GPU driver's host logic: the
all-to-all-v key exchange, the verdict return path, the small collectives and
the level-0 partition (paper_1104_1824_b200/dist.py).  No GPU involved."""
import os
import socket

import pytest
import torch
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
        comm = D.TorchComm()
        dev = torch.device("cpu")
        # small collectives
        g = comm.all_gather_ints([rank, 10 * rank + 1], dev)
        assert g == [[r, 10 * r + 1] for r in range(world)]
        assert comm.all_reduce_int(rank + 1, dev) == sum(r + 1 for r in range(world))
        big = (1 << 64) - 5 if rank == 0 else 7
        assert comm.all_reduce_u64(big, dev) == ((1 << 64) - 5 + 7 * (world - 1)) % (1 << 64)
        # keys: row i of rank r is (r, i, owner); sent to owner, grouped by owner
        torch.manual_seed(rank)
        n = 11 + 5 * rank
        owners = torch.randint(0, world, (n,))
        order = torch.argsort(owners, stable=True)
        send = torch.stack([torch.full((n,), rank), torch.arange(n), owners], dim=1)[order].to(torch.int64)
        counts = [int((owners == r).sum()) for r in range(world)]
        recv, recv_counts = comm.exchange(send, counts)
        assert recv.shape[0] == sum(recv_counts)
        assert bool((recv[:, 2] == rank).all())          # every key reached its owner
        # verdict = (source rank + index) parity, returned to the producer
        verdict = ((recv[:, 0] + recv[:, 1]) % 2).to(torch.uint8)
        back = comm.exchange_back(verdict, recv_counts, counts)
        exp = ((send[:, 0] + send[:, 1]) % 2).to(torch.uint8)
        assert torch.equal(back, exp)                     # back in send order
        # empty sends are legal
        e = torch.empty((0, 3), dtype=torch.int64)
        r2, c2 = comm.exchange(e, [0] * world)
        assert r2.shape[0] == 0 and c2 == [0] * world
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as ex:  # report to the parent
        q.put((rank, repr(ex)))


@pytest.mark.parametrize("world", [2])
def test_gloo_exchange(world):
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
