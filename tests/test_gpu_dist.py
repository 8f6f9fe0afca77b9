"""Multi-GPU exploration logic on one B200: P logical ranks run the real
driver (paper_1104_1824_b200/dist.py) in P threads, each with its own engine
instance and CUDA stream, exchanging through an in-process communicator; and
a real 1-rank NCCL group.  Results must equal the 1-GPU engine and the oracle
(same per-level counters, same digest) for every P."""
import os
import socket
import threading

import numpy as np
import pytest
import torch

import oracle
from paper_1104_1824_b200 import workloads as W

pytestmark = pytest.mark.gpu
M64 = (1 << 64) - 1


class ThreadComm:
    """In-process stand-in for the collectives (test infrastructure)."""

    def __init__(self, shared, rank, P):
        self.sh, self.rank, self.P = shared, rank, P

    def _allgather(self, obj):
        self.sh["slots"][self.rank] = obj
        self.sh["barrier"].wait()
        out = list(self.sh["slots"])
        self.sh["barrier"].wait()
        return out

    def all_gather_ints(self, values, device):
        return self._allgather(list(values))

    def all_reduce_int(self, v, device):
        return sum(self._allgather(int(v)))

    def all_reduce_u64(self, v, device):
        return sum(self._allgather(int(v))) & M64

    def exchange(self, send, counts):
        parts = list(torch.split(send, list(counts)))
        got = self._allgather((parts, list(counts)))
        recv = torch.cat([got[r][0][self.rank] for r in range(self.P)])
        return recv, [got[r][1][self.rank] for r in range(self.P)]

    def exchange_back(self, verdict, recv_counts, send_counts):
        parts = list(torch.split(verdict, list(recv_counts)))
        got = self._allgather(parts)
        return torch.cat([got[r][self.rank] for r in range(self.P)])


def run_logical(w, L0, P, depth, cfg):
    from paper_1104_1824_b200 import dist as D
    from paper_1104_1824_b200 import snp
    shared = {"barrier": threading.Barrier(P), "slots": [None] * P}
    results, errors = [None] * P, []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            eng = snp.System(w, keep_tree=0, **cfg)
            ex = D.DistExplorer(eng, ThreadComm(shared, r, P))
            lo, hi = D.level0_slice(L0.shape[0], r, P)
            c, keep = snp.configs_from_host(np.ascontiguousarray(L0[lo:hi]))
            ex.begin(c)
            levels = [ex.advance() for _ in range(depth)]
            results[r] = (levels, ex.summary())
            eng.close()
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(repr(e))
            shared["barrier"].abort()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errors, errors
    return results


@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_logical_ranks_match_single_gpu(P):
    from paper_1104_1824_b200 import snp
    w = W.random_system(512, outdeg=8, k_nd=6, seed=17)
    L0 = W.level0_counts(w, 700, 17, dtype=np.uint8)
    L0 = np.concatenate([L0, L0[:50]])  # duplicates across ranks at level 0
    cfg = dict(count_bits=8, dedup=1, frontier_target=600)
    depth = 4
    one = snp.System(w, keep_tree=0, **cfg)
    one.begin(L0)
    ref_levels = [one.advance() for _ in range(depth)]
    ref_sum = one.summary()
    res = run_logical(w, L0, P, depth, cfg)
    orc = oracle.System.from_workload(w).explore(L0, depth=depth, dedup=1, count_bits=8, frontier_target=600)
    for r in range(P):
        levels, summ = res[r]
        assert [l["T"] for l in levels] == [l["T"] for l in ref_levels] == orc.counters.T.tolist()
        assert [l["n_new"] for l in levels] == [l["n_new"] for l in ref_levels] == orc.counters.new.tolist()
        assert [l["kept"] for l in levels] == [l["kept"] for l in ref_levels] == orc.counters.kept.tolist()
        assert summ == ref_sum


def test_nccl_single_rank_group():
    import torch.distributed as dist
    from paper_1104_1824_b200 import dist as D
    from paper_1104_1824_b200 import snp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        w = W.random_system(300, outdeg=8, k_nd=5, seed=23)
        L0 = W.level0_counts(w, 400, 23, dtype=np.uint8)
        cfg = dict(count_bits=8, dedup=1, frontier_target=500)
        one = snp.System(w, keep_tree=0, **cfg)
        one.begin(L0)
        for _ in range(3):
            one.advance()
        eng = snp.System(w, keep_tree=0, **cfg)
        ex = D.DistExplorer(eng)
        c, keep = snp.configs_from_host(L0)
        ex.begin(c)
        for _ in range(3):
            ex.advance()
        assert ex.summary() == one.summary()
    finally:
        dist.destroy_process_group()
