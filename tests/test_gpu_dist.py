"""Multi-GPU exploration through the library's own exchanges (include/snp.h
snp_dist_*) on one B200: P logical ranks = P engine handles in
P host threads joined by an in-process group (the same protocol, agreement
points and row redistribution as the NCCL transport), and a real 1-rank NCCL
communicator.  Results must equal the 1-GPU engine and the oracle (per-level
counters, digest, the concatenated frontier) for every P."""
import os
import socket
import threading

import numpy as np
import pytest
import torch

import oracle
from paper_1104_1824_b200 import workloads as W

pytestmark = pytest.mark.gpu


def run_logical(w, L0, P, depth, cfg, rebalance=1.1, env=None):
    """returns per rank (levels, summary, frontier rows, frontier edges) or the
    exception each rank raised"""
    from paper_1104_1824_b200 import dist as D
    from paper_1104_1824_b200 import snp
    grp = D.LocalGroup(P)
    out = [None] * P
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            eng = snp.System(w, keep_tree=0, **cfg)
            ex = D.DistExplorer(eng, (grp, r), rebalance=rebalance)
            lo, hi = D.level0_slice(L0.shape[0], r, P)
            c, keep = snp.configs_from_host(np.ascontiguousarray(L0[lo:hi]))
            ex.begin(c)
            levels = [ex.advance() for _ in range(depth)]
            summ = ex.summary()
            F, off, _moved = ex.local()
            rows = eng.level_columns(eng.depth, np.arange(F)) if F else np.zeros((0, w.m), np.int32)
            par, t, _h, fp = eng.level_edges(eng.depth, halting=False)
            out[r] = (levels, summ, rows, (par, t, fp, off))
            eng.close()
        except Exception as e:  # surfaced by the caller
            out[r] = e

    try:
        th = [threading.Thread(target=rank_main, args=(r,)) for r in range(P)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=600)
        assert not any(t.is_alive() for t in th), "a rank hung"
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        grp.close()
    return out


def _system(seed=17):
    w = W.random_system(512, outdeg=8, k_nd=6, seed=seed)
    L0 = W.level0_counts(w, 700, seed, dtype=np.uint8)
    return w, np.concatenate([L0, L0[:50]])  # duplicates across ranks at level 0


@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("rebalance", [1.1, 1.0001])
def test_logical_ranks_match_single_gpu(P, rebalance):
    from paper_1104_1824_b200 import snp
    w, L0 = _system()
    cfg = dict(count_bits=8, dedup=1, frontier_target=600)
    depth = 4
    one = snp.System(w, keep_tree=0, **cfg)
    one.begin(L0)
    ref_levels = [one.advance() for _ in range(depth)]
    ref_sum = one.summary()
    ref_rows = one.level_columns(depth, np.arange(one.level_size(depth)))
    ref_par, ref_t, _h, ref_fp = one.level_edges(depth, halting=False)
    res = run_logical(w, L0, P, depth, cfg, rebalance=rebalance)
    for r in range(P):
        assert not isinstance(res[r], Exception), res[r]
    orc = oracle.System.from_workload(w).explore(L0, depth=depth, dedup=1, count_bits=8, frontier_target=600)
    for r in range(P):
        levels, summ, _rows, _e = res[r]
        assert [l["T"] for l in levels] == [l["T"] for l in ref_levels] == orc.counters.T.tolist()
        assert [l["n_new"] for l in levels] == [l["n_new"] for l in ref_levels] == orc.counters.new.tolist()
        assert [l["kept"] for l in levels] == [l["kept"] for l in ref_levels] == orc.counters.kept.tolist()
        assert [l["halting"] for l in levels] == [l["halting"] for l in ref_levels]
        assert summ == ref_sum
    # the ranks' frontiers, in rank order, are the 1-GPU frontier (rows, global parents, t, fp)
    order = sorted(range(P), key=lambda r: res[r][3][3])
    rows = np.concatenate([res[r][2] for r in order])
    assert (rows == ref_rows).all()
    assert (np.concatenate([res[r][3][0] for r in order]) == ref_par).all()
    assert (np.concatenate([res[r][3][1] for r in order]) == ref_t).all()
    assert (np.concatenate([res[r][3][2] for r in order]) == ref_fp).all()
    if rebalance < 1.01 and P > 1:   # forced redistribution: every rank holds ⌊F/P⌋ or ⌈F/P⌉ rows
        sizes = [len(res[r][2]) for r in range(P)]
        assert max(sizes) - min(sizes) <= 1
        assert any(l["rebalanced_rows"] > 0 for r in range(P) for l in res[r][0])


@pytest.mark.parametrize("step", [1, 2, 3, 4, 5, 6])
def test_injected_fault_agreed_by_every_rank(step):
    """A rank that fails at any protocol step makes every rank return its
    status (no rank is left waiting inside an exchange)."""
    from paper_1104_1824_b200 import snp
    w, L0 = _system(19)
    cfg = dict(count_bits=8, dedup=1, frontier_target=600)
    res = run_logical(w, L0, 3, 3, cfg, env={"SNP_DIST_INJECT": f"1,{step}", "SNP_DIST_TIMEOUT_S": "60"})
    for r in range(3):
        assert isinstance(res[r], snp.SnpError), (r, res[r])
        assert res[r].status == snp.SNP_E_CAPACITY


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
        ref = [one.advance() for _ in range(3)]
        eng = snp.System(w, keep_tree=0, **cfg)
        ex = D.DistExplorer(eng)                       # NCCL communicator inside libsnp.so
        c, keep = snp.configs_from_host(L0)
        assert ex.begin(c) == one.level_size(0)
        got = [ex.advance() for _ in range(3)]
        assert [g["T"] for g in got] == [r["T"] for r in ref]
        assert [g["kept"] for g in got] == [r["kept"] for r in ref]
        assert ex.summary() == one.summary()
    finally:
        dist.destroy_process_group()
