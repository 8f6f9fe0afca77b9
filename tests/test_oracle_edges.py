"""Pins of the oracle's every-edge record (reading A17: the computation tree
of Fig. 4, with the edges to configurations already seen):
each transition (parent, t) of an expanded level reaches configuration
ref = the oracle's stored configuration equal to children(parent)[t] (the
child function is pinned by brute force in test_oracle_properties.py), -1
exactly when that child was stored nowhere (dropped by thinning, A19), and
every configuration's own first-discovery edge (parent, t) points at it."""
import numpy as np
import pytest

import oracle
from paper_1104_1824_b200 import workloads as W


def _check_edges(s, run, thinning):
    rows = {tuple(c): i for i, c in enumerate(run.configs.tolist())}
    for L, refs in enumerate(run.edge_ref):
        lo, hi = run.level_offsets[L], run.level_offsets[L + 1]
        e = 0
        for p in range(hi - lo):
            psi, _S, Cn = s.children(run.configs[lo + p])
            for t in range(psi):
                r = int(refs[e])
                child = tuple(Cn[t].tolist())
                if r >= 0:
                    assert tuple(run.configs[r].tolist()) == child
                    assert r < run.level_offsets[L + 2]          # earlier levels or the next one
                else:
                    assert thinning and child not in rows          # stored nowhere
                e += 1
        assert e == len(refs) == run.counters.T[L]
        # first-discovery edges point at their configuration
        base = np.concatenate([[0], np.cumsum([s.children(c)[0] for c in run.level(L)])])
        for q in range(run.level_offsets[L + 1], run.level_offsets[L + 2]):
            assert refs[base[run.parent[q]] + int(run.t[q])] == q


@pytest.mark.parametrize("seed", range(0, 40, 4))
def test_edges_tiny(seed):
    w = W.tiny_random_system(seed)
    s = oracle.System.from_workload(w)
    for dedup in (0, 1):
        run = s.explore(w.C0, 5, dedup=dedup)
        if run.status == 0:
            _check_edges(s, run, thinning=False)


@pytest.mark.parametrize("seed,target", [(1, 0), (2, 30), (3, 60)])
def test_edges_random_thinning(seed, target):
    w = W.random_system(24, outdeg=3, k_nd=6, seed=seed)
    L0 = W.level0_counts(w, 40, seed)
    s = oracle.System.from_workload(w)
    run = s.explore(L0, 3, dedup=1, frontier_target=target)
    assert run.status == 0
    _check_edges(s, run, thinning=target > 0)


def test_edges_pi_printed_run():
    # Π (simulator encoding): 212 -> {212, 112, ...}: the self-loop of 212 and
    # its edge back to 112 (reading A6) are recorded as edges to
    # the earlier configurations instead of being dropped
    w = W.pi_system("simulator")
    s = oracle.System.from_workload(w)
    run = s.explore(w.C0, 3)
    _check_edges(s, run, thinning=False)
    i212 = [tuple(c) for c in run.configs.tolist()].index((2, 1, 2))
    lvl = next(L for L in range(run.num_levels) if run.level_offsets[L] <= i212 < run.level_offsets[L + 1])
    refs = run.edge_ref[lvl]
    psi, _S, Cn = s.children(run.configs[i212])
    start = sum(s.children(c)[0] for c in run.configs[run.level_offsets[lvl]:i212])
    assert i212 in refs[start:start + psi].tolist()                  # the self-loop 212 -> 212
